# session 22: pair-kernel occupancy (6 blocks/SM) and blocks-per-query A/B at configs[4]; bench
# lines of the current state (configs[4] default, configs[1], configs[3])
mkdir -p gpurun_out
make -s -j8 -C paper_2603_24920_b200 > /dev/null && make -s -C oracle > /dev/null
export DATAGEN_CACHE_DIR=/tmp/dgc
timeout 900 python tools/query_ab.py 5 2000 DETLSH_LP_OCC6 0,1 > gpurun_out/occ22_c5.log 2>&1; echo "occ c5 exit $?"; tail -4 gpurun_out/occ22_c5.log
timeout 900 python tools/query_ab.py 5 2000 DETLSH_LP_Y 16,8,32 > gpurun_out/lpy22_c5.log 2>&1; echo "lpy c5 exit $?"; tail -6 gpurun_out/lpy22_c5.log
unset DATAGEN_CACHE_DIR
timeout 1500 python bench.py > gpurun_out/bench22_c5.log 2>&1; echo "bench c5 exit $?"; tail -1 gpurun_out/bench22_c5.log | cut -c1-400
timeout 900 python bench.py --config 2 --steps 20 --warmup 5 > gpurun_out/bench22_c2.log 2>&1; echo "bench c2 exit $?"
timeout 900 python bench.py --config 4 > gpurun_out/bench22_c4.log 2>&1; echo "bench c4 exit $?"
