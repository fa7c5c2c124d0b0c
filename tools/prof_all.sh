#!/bin/bash
# One ncu --set full capture per hot kernel at 256^3 (first launch of each
# kernel class inside a V-cycle / a short FGMRES run). Run on a B200 box;
# summarise with tools/ncu_summary.py.
set -x
O=gpurun_out
ncu --set full --clock-control none -k regex:k_vanka_update -s 0 -c 1 -o $O/prof_k_vanka python tools/prof_kernels.py --what cycle --reps 1 > $O/ncu_k1.log 2>&1
ncu --set full --clock-control none -k regex:k_restrict3 -s 0 -c 1 -o $O/prof_k_restrict python tools/prof_kernels.py --what cycle --reps 1 > $O/ncu_k2.log 2>&1
ncu --set full --clock-control none -k regex:k_prolong3 -s 12 -c 1 -o $O/prof_k_prolong python tools/prof_kernels.py --what cycle --reps 1 > $O/ncu_k3.log 2>&1
ncu --set full --clock-control none -k regex:k_gemv_rows -s 0 -c 1 -o $O/prof_k_gemv python tools/prof_kernels.py --what cycle --reps 1 > $O/ncu_k4.log 2>&1
ncu --set full --clock-control none -k regex:k_mgs -s 3 -c 1 -o $O/prof_k_mgs python tools/prof_kernels.py --what solve --reps 1 > $O/ncu_k5.log 2>&1
