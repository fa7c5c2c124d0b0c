O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests_r1q.log 2>&1; echo "tests exit $?" >> $O/gpu_tests_r1q.log
timeout 600 python bench.py > $O/bench_r1q.json 2> $O/bench_r1q.err; echo "bench exit $?" >> $O/bench_r1q.err
timeout 300 python tools/run_hetero3d.py --n 128 --levels 4 > $O/hetero_r1q.jsonl 2> $O/hetero_r1q.err
timeout 600 python tools/run_hetero3d.py --n 256 --levels 5 >> $O/hetero_r1q.jsonl 2>> $O/hetero_r1q.err
