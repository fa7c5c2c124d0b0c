set -x
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_bench_launch.py -m gpu -x -q > gpurun_out/t5.log 2>&1
tail -3 gpurun_out/t5.log
timeout 900 python tools/dist_overhead.py 128 > gpurun_out/dist_overhead_128.json 2> gpurun_out/dist_overhead.err
cat gpurun_out/dist_overhead_128.json
python bench.py --steps 2 --warmup 1 --solve 0 --mixed 0 --no-cpu > gpurun_out/b5_small.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ehmg -c 3000 --csv --log-file gpurun_out/launches_r2b.csv python bench.py --steps 2 --warmup 1 --solve 0 --mixed 0 --no-cpu > gpurun_out/ncu_launch2.log 2>&1
tail -1 gpurun_out/ncu_launch2.log | cut -c1-200
