# session 33 (final, part 1): smoke, all GPU tests, bench lines (configs[4] default, configs[1],
# configs[3], AMB-22 radius, reference arm)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
make -s -j8 -C paper_2603_24920_b200 > /dev/null && make -s -C oracle > /dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke33.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/smoke33.log
( time timeout 2400 python -m pytest tests -m gpu -q -rf ) > gpurun_out/gpu_tests33.log 2>&1; echo "all gpu tests exit $?"; tail -3 gpurun_out/gpu_tests33.log
timeout 1500 python bench.py > gpurun_out/bench33_c5.log 2>&1; echo "bench c5 exit $?"
timeout 900 python bench.py --config 2 --steps 20 --warmup 5 > gpurun_out/bench33_c2.log 2>&1; echo "bench c2 exit $?"
timeout 900 python bench.py --config 4 > gpurun_out/bench33_c4.log 2>&1; echo "bench c4 exit $?"
timeout 900 python bench.py --radius amb22 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench33_c5_amb22.log 2>&1; echo "bench c5 amb22 exit $?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench33_ref.log 2>&1; echo "bench ref exit $?"
