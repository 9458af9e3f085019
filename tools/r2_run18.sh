# session 18: box_bound16 A/B (configs[4] 2000 queries, configs[3], configs[1]), build with the
# radix scatter rewrite (configs[4]), switch-invariance + tree tests
mkdir -p gpurun_out
make -s -j8 -C paper_2603_24920_b200 > /dev/null && make -s -C oracle > /dev/null
export DATAGEN_CACHE_DIR=/tmp/dgc
timeout 900 python tools/query_ab.py 5 2000 DETLSH_BOX16 0,1 > gpurun_out/box18_c5.log 2>&1; echo "box c5 exit $?"; cat gpurun_out/box18_c5.log | tail -6
timeout 900 python tools/build_ab.py 5 "1536:256,3072:256" > gpurun_out/build18_c5.log 2>&1; echo "build c5 exit $?"; tail -4 gpurun_out/build18_c5.log
timeout 600 python tools/query_ab.py 4 10000 DETLSH_BOX16 0,1 > gpurun_out/box18_c4.log 2>&1; echo "box c4 exit $?"; tail -4 gpurun_out/box18_c4.log
timeout 600 python tools/query_ab.py 2 1000 DETLSH_BOX16 0,1 > gpurun_out/box18_c2.log 2>&1; echo "box c2 exit $?"; tail -4 gpurun_out/box18_c2.log
unset DATAGEN_CACHE_DIR
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "switch or tree or split or sample or large_k or end_to_end" > gpurun_out/tests18.log 2>&1; echo "tests exit $?"; tail -3 gpurun_out/tests18.log
