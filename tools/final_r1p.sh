O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests_r1p.log 2>&1; echo "tests exit $?" >> $O/gpu_tests_r1p.log
timeout 500 python bench.py > $O/bench_r1p.json 2> $O/bench_r1p.err; echo "bench exit $?" >> $O/bench_r1p.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench_r1p.csv python bench.py --steps 2 --warmup 3 --no-cpu --solve 0 --mixed 0 > $O/ncu_launch.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gs_dots -s 6 -c 1 -o $O/prof_k_gs_dots python tools/prof_kernels.py --what solve --reps 2 > $O/ncu_gs1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gs_update -s 6 -c 1 -o $O/prof_k_gs_update python tools/prof_kernels.py --what solve --reps 2 > $O/ncu_gs2.log 2>&1
