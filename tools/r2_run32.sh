# session 32 (final measurements): smoke, bench lines (configs[4] default, configs[1], configs[3],
# AMB-22 radius, reference arm), launch lists and full captures of the dominant kernels, GPU tests
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
make -s -j8 -C paper_2603_24920_b200 > /dev/null && make -s -C oracle > /dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke32.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/smoke32.log
timeout 1500 python bench.py > gpurun_out/bench32_c5.log 2>&1; echo "bench c5 exit $?"
timeout 900 python bench.py --config 2 --steps 20 --warmup 5 > gpurun_out/bench32_c2.log 2>&1; echo "bench c2 exit $?"
timeout 900 python bench.py --config 4 > gpurun_out/bench32_c4.log 2>&1; echo "bench c4 exit $?"
timeout 900 python bench.py --radius amb22 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench32_c5_amb22.log 2>&1; echo "bench c5 amb22 exit $?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench32_ref.log 2>&1; echo "bench ref exit $?"
export DATAGEN_CACHE_DIR=/tmp/dgc
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/launches32_c5.csv python tools/cfg_query.py 5 2000 > gpurun_out/ncu32_l5.log 2>&1; echo "ncu launches c5 exit $?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_leaf_points|k_tile_pairs" -s 6 -c 2 -o gpurun_out/full32_c5 python tools/cfg_query.py 5 2000 > gpurun_out/ncu32_f5.log 2>&1; echo "ncu full c5 exit $?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_local_finish|k_leaf_layout16|k_project_tc" -c 4 -o gpurun_out/full32_c5b python tools/cfg_query.py 5 16 > gpurun_out/ncu32_f5b.log 2>&1; echo "ncu full c5 build exit $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_leaf_points|k_range_filter" -s 8 -c 2 -o gpurun_out/full32_c2 python tools/cfg_query.py 2 > gpurun_out/ncu32_f2.log 2>&1; echo "ncu full c2 exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches32_c2.csv python bench.py --config 2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu32_l2.log 2>&1; echo "ncu launches c2 exit $?"
unset DATAGEN_CACHE_DIR
( time timeout 3000 python -m pytest tests -m gpu -q -rf ) > gpurun_out/gpu_tests32.log 2>&1; echo "all gpu tests exit $?"; tail -3 gpurun_out/gpu_tests32.log
