# session 23: pair-kernel blocks per query (DETLSH_LP_Y) and latency variants (DETLSH_LP_VAR: 4 sub-box
# offsets with the leaf's, 8 next take ahead, 12 both) A/B at configs[4], [3], [1]; switch test
mkdir -p gpurun_out
make -s -j8 -C paper_2603_24920_b200 > /dev/null && make -s -C oracle > /dev/null
export DATAGEN_CACHE_DIR=/tmp/dgc
timeout 900 python tools/query_ab.py 5 2000 DETLSH_LP_Y 32,48,64,128 > gpurun_out/lpy23_c5.log 2>&1; echo "lpy c5 exit $?"; tail -8 gpurun_out/lpy23_c5.log
export DETLSH_LP_Y=32
timeout 900 python tools/query_ab.py 5 2000 DETLSH_LP_VAR 0,4,8,12 > gpurun_out/var23_c5.log 2>&1; echo "var c5 exit $?"; tail -8 gpurun_out/var23_c5.log
unset DETLSH_LP_Y
timeout 900 python tools/query_ab.py 4 10000 DETLSH_LP_Y 16,32,64 > gpurun_out/lpy23_c4.log 2>&1; echo "lpy c4 exit $?"; tail -6 gpurun_out/lpy23_c4.log
timeout 900 python tools/query_ab.py 2 1000 DETLSH_LP_Y 16,32,64 > gpurun_out/lpy23_c2.log 2>&1; echo "lpy c2 exit $?"; tail -6 gpurun_out/lpy23_c2.log
unset DATAGEN_CACHE_DIR
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "switch" > gpurun_out/tests23.log 2>&1; echo "tests exit $?"; tail -3 gpurun_out/tests23.log
