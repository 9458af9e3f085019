# session 29: leaf layout with shared-memory sub-box boxes in the spread form: build times, tests
mkdir -p gpurun_out
make -s -j8 -C paper_2603_24920_b200 > /dev/null && make -s -C oracle > /dev/null
export DATAGEN_CACHE_DIR=/tmp/dgc
timeout 900 python tools/build_ab.py 5 "3072:0" > gpurun_out/build29_c5.log 2>&1; echo "build c5 exit $?"; tail -1 gpurun_out/build29_c5.log
timeout 600 python tools/build_ab.py 4 "3072:0" > gpurun_out/build29_c4.log 2>&1; echo "build c4 exit $?"; tail -1 gpurun_out/build29_c4.log
timeout 900 python tools/query_ab.py 5 2000 DETLSH_LP_PF 0 > gpurun_out/q29_c5.log 2>&1; echo "query c5 exit $?"; tail -1 gpurun_out/q29_c5.log
unset DATAGEN_CACHE_DIR
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "switch or split_paths or trees or end_to_end or config5" > gpurun_out/tests29.log 2>&1; echo "tests exit $?"; tail -3 gpurun_out/tests29.log
