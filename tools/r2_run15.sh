# session 15: baseline of HEAD after re-entry: smoke, default bench (configs[4]), configs[1] bench, GPU tests
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
make -s -j8 -C paper_2603_24920_b200 > /dev/null && make -s -C oracle > /dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke15.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/smoke15.log
( time timeout 1500 python bench.py ) > gpurun_out/bench15_c5.log 2>&1; echo "bench c5 exit $?"; tail -4 gpurun_out/bench15_c5.log
timeout 900 python bench.py --config 2 --steps 20 --warmup 5 > gpurun_out/bench15_c2.log 2>&1; echo "bench c2 exit $?"
( time timeout 3000 python -m pytest tests -m gpu -q -rf -x ) > gpurun_out/gpu_tests15.log 2>&1; echo "all gpu tests exit $?"; tail -5 gpurun_out/gpu_tests15.log
