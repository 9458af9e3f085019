# session 35 (final): smoke, all GPU tests in the driver's form (-x -q), default bench line,
# launch list + full capture of the dominant kernel at configs[4], configs[1] bench line
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
make -s -j8 -C paper_2603_24920_b200 > /dev/null && make -s -C oracle > /dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke35.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/smoke35.log
( time timeout 1700 python -m pytest tests -m gpu -x -q -rf --durations=8 ) > gpurun_out/gpu_tests35.log 2>&1; echo "all gpu tests exit $?"; tail -14 gpurun_out/gpu_tests35.log
( time timeout 900 python bench.py ) > gpurun_out/bench35_c5.log 2>&1; echo "bench c5 exit $?"; grep '^{' gpurun_out/bench35_c5.log | cut -c1-600
export DATAGEN_CACHE_DIR=/tmp/dgc
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/launches35_c5.csv python tools/cfg_query.py 5 2000 > gpurun_out/ncu35_l5.log 2>&1; echo "ncu launches c5 exit $?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_leaf_points|k_tile_pairs" -s 6 -c 2 -o gpurun_out/full35_c5 python tools/cfg_query.py 5 2000 > gpurun_out/ncu35_f5.log 2>&1; echo "ncu full c5 exit $?"
timeout 400 python bench.py --config 2 --steps 20 --warmup 5 > gpurun_out/bench35_c2.log 2>&1; echo "bench c2 exit $?"; grep '^{' gpurun_out/bench35_c2.log | cut -c1-400
