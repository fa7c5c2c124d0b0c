set -x
V=_variants
python tools/ab_stencil.py $V/lib_rr.so $V/lib_sp82.so $V/lib_sp161.so $V/lib_sp121.so $V/lib_sp92.so --n 256 > gpurun_out/ab_sp_256.txt 2>&1
python tools/ab_stencil.py $V/lib_rr.so $V/lib_sp82.so $V/lib_sp161.so $V/lib_sp121.so $V/lib_sp92.so --n 128 --reps 50 > gpurun_out/ab_sp_128.txt 2>&1
python tools/ab_stencil.py $V/lib_rr.so $V/lib_sp82.so $V/lib_sp161.so $V/lib_sp92.so --n 64 --reps 100 > gpurun_out/ab_sp_64.txt 2>&1
cat gpurun_out/ab_sp_256.txt gpurun_out/ab_sp_128.txt gpurun_out/ab_sp_64.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/t_sp_parity.log 2>&1; tail -5 gpurun_out/t_sp_parity.log
