# bench line + launch list + one full ncu capture of the hot kernels (configs[1])
set -x
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench exit $?"
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_b.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches exit $?"
timeout 300 python tools/one_query.py 2 > gpurun_out/plain_q.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_range_filter|k_leaf_points|k_verify_gather|k_verify_prep|k_project_tc" \
    -c 14 -o gpurun_out/prof_full python tools/one_query.py 2 > gpurun_out/ncu_full.log 2>&1; echo "ncu full exit $?"
