set -x
python -m pytest tests/test_gpu_configs.py -m gpu -q > gpurun_out/t4.log 2>&1
tail -3 gpurun_out/t4.log
python bench.py --steps 20 --warmup 5 > gpurun_out/b4_full.json 2> gpurun_out/b4_full.err
tail -c 300 gpurun_out/b4_full.json
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/b4_ref.json 2> gpurun_out/b4_ref.err
tail -c 300 gpurun_out/b4_ref.json
python bench.py --steps 2 --warmup 1 --solve 0 --mixed 0 --no-cpu > gpurun_out/b4_small.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 2 --warmup 1 --solve 0 --mixed 0 --no-cpu > gpurun_out/ncu_launch.log 2>&1
tail -2 gpurun_out/ncu_launch.log
python bench.py --workload c3 --steps 5 --warmup 3 --solve 0 --mixed 0 --no-cpu > gpurun_out/b4_c3.json 2> gpurun_out/b4_c3.err
tail -c 300 gpurun_out/b4_c3.json
python bench.py --workload c4w --steps 5 --warmup 3 --mixed 0 --no-cpu > gpurun_out/b4_c4w.json 2> gpurun_out/b4_c4w.err
tail -c 300 gpurun_out/b4_c4w.json
