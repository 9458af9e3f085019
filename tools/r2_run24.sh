# session 24: persistent pair kernel vs blocks per query (configs[4], configs[3]); switch test
mkdir -p gpurun_out
make -s -j8 -C paper_2603_24920_b200 > /dev/null && make -s -C oracle > /dev/null
export DATAGEN_CACHE_DIR=/tmp/dgc
export DETLSH_LP_Y=128
timeout 900 python tools/query_ab.py 5 2000 DETLSH_LP_PERSIST 0,1 > gpurun_out/pers24_c5.log 2>&1; echo "persist c5 exit $?"; tail -4 gpurun_out/pers24_c5.log
timeout 900 python tools/query_ab.py 5 2000 DETLSH_LP_Y 128,256,512 > gpurun_out/lpy24_c5.log 2>&1; echo "lpy c5 exit $?"; tail -6 gpurun_out/lpy24_c5.log
timeout 900 python tools/query_ab.py 4 10000 DETLSH_LP_PERSIST 0,1 > gpurun_out/pers24_c4.log 2>&1; echo "persist c4 exit $?"; tail -4 gpurun_out/pers24_c4.log
unset DETLSH_LP_Y
unset DATAGEN_CACHE_DIR
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "switch" > gpurun_out/tests24.log 2>&1; echo "tests exit $?"; tail -3 gpurun_out/tests24.log
