# session 36 (final, part 2): hash-family bit-exactness at d = 960/1500, full captures of the build
# kernels at configs[4] and of the configs[1] filter kernels, configs[3] and AMB-22 bench lines
mkdir -p gpurun_out
make -s -j8 -C paper_2603_24920_b200 > /dev/null && make -s -C oracle > /dev/null
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -k "streamed_hash_matrix or hash_family" > gpurun_out/tests36.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/tests36.log
export DATAGEN_CACHE_DIR=/tmp/dgc
timeout 500 ncu --set full --import-source on --clock-control none -k regex:"k_local_finish|k_leaf_layout16|k_project_tc" -c 4 -o gpurun_out/full36_c5b python tools/cfg_query.py 5 16 > gpurun_out/ncu36_f5b.log 2>&1; echo "ncu full c5 build exit $?"
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_leaf_points|k_range_filter" -s 8 -c 2 -o gpurun_out/full36_c2 python tools/cfg_query.py 2 > gpurun_out/ncu36_f2.log 2>&1; echo "ncu full c2 exit $?"
timeout 300 python bench.py --config 4 --no-cpu-baseline > gpurun_out/bench36_c4.log 2>&1; echo "bench c4 exit $?"; grep '^{' gpurun_out/bench36_c4.log | cut -c1-300
timeout 600 python bench.py --radius amb22 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench36_c5_amb22.log 2>&1; echo "bench c5 amb22 exit $?"; grep '^{' gpurun_out/bench36_c5_amb22.log | cut -c1-300
