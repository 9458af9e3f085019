# session 31: REDUX tally (build), L2 prefetch default, smaller round-buffer reservation: tests and times
mkdir -p gpurun_out
make -s -j8 -C paper_2603_24920_b200 > /dev/null && make -s -C oracle > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "split_paths or trees" > gpurun_out/tests31a.log 2>&1; echo "tree tests exit $?"; tail -2 gpurun_out/tests31a.log
export DATAGEN_CACHE_DIR=/tmp/dgc
timeout 900 python tools/build_ab.py 5 "3072:0" > gpurun_out/build31_c5.log 2>&1; echo "build c5 exit $?"; tail -1 gpurun_out/build31_c5.log
timeout 900 python tools/batch_ab.py 5 4000 0 > gpurun_out/q31_c5.log 2>&1; echo "query c5 exit $?"; tail -1 gpurun_out/q31_c5.log
timeout 900 python tools/batch_ab.py 4 10000 0 > gpurun_out/q31_c4.log 2>&1; echo "query c4 exit $?"; tail -1 gpurun_out/q31_c4.log
unset DATAGEN_CACHE_DIR
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "switch or end_to_end or config5 or batch" > gpurun_out/tests31b.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/tests31b.log
