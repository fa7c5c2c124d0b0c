O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests_r1r.log 2>&1; echo "tests exit $?" >> $O/gpu_tests_r1r.log
timeout 600 python bench.py > $O/bench_r1r.json 2> $O/bench_r1r.err; echo "bench exit $?" >> $O/bench_r1r.err
