set -x
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_media_grf.py -m gpu -x -q > gpurun_out/t6.log 2>&1
tail -3 gpurun_out/t6.log
python bench.py --steps 2 --warmup 1 --solve 0 --mixed 0 --no-cpu > gpurun_out/b6_small.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 3000 --csv --log-file gpurun_out/launches_r2c.csv python bench.py --steps 2 --warmup 1 --solve 0 --mixed 0 --no-cpu > gpurun_out/ncu_launch3.log 2>&1
tail -1 gpurun_out/ncu_launch3.log | cut -c1-100
