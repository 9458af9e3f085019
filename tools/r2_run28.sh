# session 28: FIFO sub-box queue with L2 prefetch of the point codes (DETLSH_LP_PF) A/B at configs[4]
# and configs[3]; switch test
mkdir -p gpurun_out
make -s -j8 -C paper_2603_24920_b200 > /dev/null && make -s -C oracle > /dev/null
export DATAGEN_CACHE_DIR=/tmp/dgc
timeout 900 python tools/query_ab.py 5 2000 DETLSH_LP_PF 0,1 > gpurun_out/pf28_c5.log 2>&1; echo "pf c5 exit $?"; tail -4 gpurun_out/pf28_c5.log
timeout 900 python tools/query_ab.py 4 10000 DETLSH_LP_PF 0,1 > gpurun_out/pf28_c4.log 2>&1; echo "pf c4 exit $?"; tail -4 gpurun_out/pf28_c4.log
unset DATAGEN_CACHE_DIR
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "switch" > gpurun_out/tests28.log 2>&1; echo "tests exit $?"; tail -3 gpurun_out/tests28.log
