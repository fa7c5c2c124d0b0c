set -x
python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_configs.py::test_config3_recipe_fgmres_vs_reference > gpurun_out/t3.log 2>&1
tail -5 gpurun_out/t3.log
python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/b3.json 2> gpurun_out/b3.err
tail -c 400 gpurun_out/b3.json
