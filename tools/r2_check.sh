# round-2 check: full GPU test suite (no -x), smoke, short bench -> gpurun_out/
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; free -g | head -2
timeout 2400 python -m pytest tests -m gpu -q -rf ${PYTEST_K:+-k "$PYTEST_K"} -s > gpurun_out/gpu_tests.log 2>&1; echo "tests exit $?"; tail -15 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py --steps ${STEPS:-10} --no-cpu-baseline --recall-queries 50 > gpurun_out/bench_quick.log 2>&1; echo "bench exit $?"; tail -c 1500 gpurun_out/bench_quick.log
