V=_variants
python tools/ab_stencil.py $V/lib_rr.so $V/lib_sp82.so $V/lib_sp161.so $V/lib_sp121.so --n 256 > gpurun_out/ab_sp3_256.txt 2>&1
python tools/ab_stencil.py $V/lib_rr.so $V/lib_sp82.so $V/lib_sp161.so $V/lib_sp121.so --n 128 --reps 50 > gpurun_out/ab_sp3_128.txt 2>&1
python tools/ab_stencil.py $V/lib_rr.so $V/lib_sp82.so $V/lib_sp121.so --n 40 --reps 50 > gpurun_out/ab_sp3_40.txt 2>&1
python tools/ab_stencil.py $V/lib_rr.so $V/lib_sp82.so $V/lib_sp121.so --n 64 --reps 50 > gpurun_out/ab_sp3_64.txt 2>&1
cat gpurun_out/ab_sp3_256.txt gpurun_out/ab_sp3_128.txt gpurun_out/ab_sp3_40.txt gpurun_out/ab_sp3_64.txt
for v in sp82; do
ncu --set full --import-source on --clock-control none -k regex:k_stencil3d -s 5 -c 1 -o gpurun_out/prof3_$v python tools/ab_stencil.py $V/lib_$v.so --n 256 --reps 1 --one > gpurun_out/ncu3_$v.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py -m gpu -x -q > gpurun_out/t_sp3_parity.log 2>&1; tail -3 gpurun_out/t_sp3_parity.log
