set -x
V=_variants
python tools/ab_stencil.py $V/lib_rr.so $V/lib_sp82.so $V/lib_sp161.so $V/lib_sp121.so --n 256 > gpurun_out/ab_sp2_256.txt 2>&1
python tools/ab_stencil.py $V/lib_rr.so $V/lib_sp82.so $V/lib_sp161.so $V/lib_sp121.so --n 128 --reps 50 > gpurun_out/ab_sp2_128.txt 2>&1
python tools/ab_stencil.py $V/lib_rr.so $V/lib_sp82.so $V/lib_sp121.so --n 40 --reps 50 > gpurun_out/ab_sp2_40.txt 2>&1
cat gpurun_out/ab_sp2_256.txt gpurun_out/ab_sp2_128.txt gpurun_out/ab_sp2_40.txt
for v in sp82 sp121; do
ncu --set full --import-source on --clock-control none -k regex:k_stencil3d -s 5 -c 1 -o gpurun_out/prof2_$v python tools/ab_stencil.py $V/lib_$v.so --n 256 --reps 1 --one > gpurun_out/ncu2_$v.log 2>&1
done
