# session 27: block-wide split-dimension tally in k_local_finish: tree tests, build times
mkdir -p gpurun_out
make -s -j8 -C paper_2603_24920_b200 > /dev/null && make -s -C oracle > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "split_paths or trees" > gpurun_out/tests27.log 2>&1; echo "tree tests exit $?"; tail -3 gpurun_out/tests27.log
export DATAGEN_CACHE_DIR=/tmp/dgc
timeout 900 python tools/build_ab.py 5 "3072:0,1536:0,4096:0,2048:0" > gpurun_out/build27_c5.log 2>&1; echo "build c5 exit $?"; tail -4 gpurun_out/build27_c5.log
timeout 600 python tools/build_ab.py 4 "3072:0,1536:0" > gpurun_out/build27_c4.log 2>&1; echo "build c4 exit $?"; tail -2 gpurun_out/build27_c4.log
timeout 600 python tools/build_ab.py 2 "3072:0,1536:0" > gpurun_out/build27_c2.log 2>&1; echo "build c2 exit $?"; tail -2 gpurun_out/build27_c2.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_local_finish" -c 2 -o gpurun_out/full27_lf python tools/build_ab.py 5 "3072:0" > gpurun_out/ncu27_lf.log 2>&1; echo "ncu lf exit $?"
