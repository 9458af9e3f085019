# session 16: pair-kernel two-stage bounds A/B (configs[4], 2000 queries), build local-finish
# settings A/B (configs[4]), full captures of the build's top kernels
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
make -s -j8 -C paper_2603_24920_b200 > /dev/null && make -s -C oracle > /dev/null
export DATAGEN_CACHE_DIR=/tmp/dgc
DETLSH_LP_STATS=1 timeout 1200 python tools/split_ab.py 5 2000 0,1,3,6,7 > gpurun_out/split16_c5.log 2>&1; echo "split c5 exit $?"; grep -v STATS gpurun_out/split16_c5.log | tail -10; grep STATS gpurun_out/split16_c5.log | tail -5
timeout 900 python tools/build_ab.py 5 "1536:256,3072:256,4096:256,4096:512,6144:512" > gpurun_out/build16_c5.log 2>&1; echo "build c5 exit $?"; tail -10 gpurun_out/build16_c5.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_local_finish|k_leaf_layout16|k_part_scatter|k_part_count|k_rs_scatter" -c 6 -o gpurun_out/full16_build python tools/build_ab.py 5 "1536:256" > gpurun_out/ncu16_b.log 2>&1; echo "ncu build exit $?"
timeout 600 python tools/split_ab.py 4 10000 0,1,3,6,7 > gpurun_out/split16_c4.log 2>&1; echo "split c4 exit $?"; tail -6 gpurun_out/split16_c4.log
timeout 600 python tools/split_ab.py 2 1000 0,1,3 > gpurun_out/split16_c2.log 2>&1; echo "split c2 exit $?"; tail -6 gpurun_out/split16_c2.log
