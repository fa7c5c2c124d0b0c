set -x
python -m pytest tests/test_gpu_configs.py -m gpu -q > gpurun_out/t2.log 2>&1
tail -5 gpurun_out/t2.log
python tools/explore_sources.py 2 > gpurun_out/explore_src2.jsonl 2> gpurun_out/explore_src2.err
cat gpurun_out/explore_src2.jsonl
python tools/prof_kernels.py --what apply --reps 2 > gpurun_out/pk.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_stencil3d_rr -s 1 -c 1 -o gpurun_out/prof_rr_r2a python tools/prof_kernels.py --what apply --reps 2 > gpurun_out/ncu_rr.log 2>&1
tail -3 gpurun_out/ncu_rr.log
