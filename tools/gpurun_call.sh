set -x
python -m pytest tests/test_media_grf.py tests/test_gpu_acceptance.py tests/test_bench_launch.py tests/test_abi.py -m gpu -x -q > gpurun_out/t1.log 2>&1
tail -5 gpurun_out/t1.log
python bench.py --workload c3 --cells 256 --steps 5 --warmup 3 --mixed 0 --no-cpu > gpurun_out/b_c3_256.json 2> gpurun_out/b_c3_256.err
tail -c 600 gpurun_out/b_c3_256.json
python bench.py --mode sources --sources 2 --steps 1 --warmup 1 > gpurun_out/b_src2.json 2> gpurun_out/b_src2.err
tail -c 800 gpurun_out/b_src2.json
python tools/ref_extrapolation.py > gpurun_out/refx.log 2>&1
tail -3 gpurun_out/refx.log
