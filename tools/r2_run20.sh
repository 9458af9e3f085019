# session 20: pipelined point-code loads A/B (configs[4], [3], [1]); local-finish size/threads A/B
mkdir -p gpurun_out
make -s -j8 -C paper_2603_24920_b200 > /dev/null && make -s -C oracle > /dev/null
export DATAGEN_CACHE_DIR=/tmp/dgc
timeout 900 python tools/query_ab.py 5 2000 DETLSH_LP_PIPE 0,1 > gpurun_out/pipe20_c5.log 2>&1; echo "pipe c5 exit $?"; tail -4 gpurun_out/pipe20_c5.log
timeout 900 python tools/build_ab.py 5 "3072:256,3072:512,2048:256,2048:512,1536:256" > gpurun_out/build20_c5.log 2>&1; echo "build c5 exit $?"; tail -5 gpurun_out/build20_c5.log
timeout 600 python tools/query_ab.py 4 10000 DETLSH_LP_PIPE 0,1 > gpurun_out/pipe20_c4.log 2>&1; echo "pipe c4 exit $?"; tail -4 gpurun_out/pipe20_c4.log
timeout 600 python tools/build_ab.py 4 "1536:256,3072:256,3072:512" > gpurun_out/build20_c4.log 2>&1; echo "build c4 exit $?"; tail -3 gpurun_out/build20_c4.log
timeout 600 python tools/query_ab.py 2 1000 DETLSH_LP_PIPE 0,1 > gpurun_out/pipe20_c2.log 2>&1; echo "pipe c2 exit $?"; tail -4 gpurun_out/pipe20_c2.log
timeout 600 python tools/build_ab.py 2 "1536:256,3072:256,3072:512" > gpurun_out/build20_c2.log 2>&1; echo "build c2 exit $?"; tail -3 gpurun_out/build20_c2.log
