# session 21: sub-box owner table A/B (configs[4], [3], [1]); two-tier local finish (build A/B);
# tree + switch-invariance tests
mkdir -p gpurun_out
make -s -j8 -C paper_2603_24920_b200 > /dev/null && make -s -C oracle > /dev/null
export DATAGEN_CACHE_DIR=/tmp/dgc
timeout 900 python tools/query_ab.py 5 2000 DETLSH_LP_LTAB 0,1 > gpurun_out/ltab21_c5.log 2>&1; echo "ltab c5 exit $?"; tail -4 gpurun_out/ltab21_c5.log
timeout 900 python tools/build_ab.py 5 "3072:0,1536:0,2048:0,4096:0" > gpurun_out/build21_c5.log 2>&1; echo "build c5 exit $?"; tail -4 gpurun_out/build21_c5.log
timeout 600 python tools/query_ab.py 4 10000 DETLSH_LP_LTAB 0,1 > gpurun_out/ltab21_c4.log 2>&1; echo "ltab c4 exit $?"; tail -4 gpurun_out/ltab21_c4.log
timeout 600 python tools/build_ab.py 4 "3072:0,1536:0" > gpurun_out/build21_c4.log 2>&1; echo "build c4 exit $?"; tail -2 gpurun_out/build21_c4.log
timeout 600 python tools/query_ab.py 2 1000 DETLSH_LP_LTAB 0,1 > gpurun_out/ltab21_c2.log 2>&1; echo "ltab c2 exit $?"; tail -4 gpurun_out/ltab21_c2.log
timeout 600 python tools/build_ab.py 2 "3072:0,1536:0" > gpurun_out/build21_c2.log 2>&1; echo "build c2 exit $?"; tail -2 gpurun_out/build21_c2.log
unset DATAGEN_CACHE_DIR
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "switch or split_paths" > gpurun_out/tests21.log 2>&1; echo "tests exit $?"; tail -3 gpurun_out/tests21.log
