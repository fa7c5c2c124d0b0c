set -x
V=_variants
for v in sp82 sp161; do
ncu --set full --import-source on --clock-control none -k regex:k_stencil3d -s 5 -c 1 -o gpurun_out/prof_$v python tools/ab_stencil.py $V/lib_$v.so --n 256 --reps 1 --one > gpurun_out/ncu_$v.log 2>&1
tail -2 gpurun_out/ncu_$v.log
done
