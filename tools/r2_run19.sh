# session 19: warp-mode local finish: tree parity tests, build A/B at configs[4] and configs[1]
mkdir -p gpurun_out
make -s -j8 -C paper_2603_24920_b200 > /dev/null && make -s -C oracle > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "split_paths" > gpurun_out/tests19.log 2>&1; echo "tree tests exit $?"; tail -3 gpurun_out/tests19.log
export DATAGEN_CACHE_DIR=/tmp/dgc
timeout 900 python tools/build_ab.py 5 "1536:256:0,1536:256:512,3072:256:512,3072:256:1032,4096:256:1032,3072:512:1032" > gpurun_out/build19_c5.log 2>&1; echo "build c5 exit $?"; tail -7 gpurun_out/build19_c5.log
timeout 600 python tools/build_ab.py 2 "1536:256:0,1536:256:512,3072:256:1032" > gpurun_out/build19_c2.log 2>&1; echo "build c2 exit $?"; tail -4 gpurun_out/build19_c2.log
timeout 600 python tools/build_ab.py 4 "1536:256:0,1536:256:512,3072:256:1032" > gpurun_out/build19_c4.log 2>&1; echo "build c4 exit $?"; tail -4 gpurun_out/build19_c4.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_local_finish" -c 1 -o gpurun_out/full19_lf python tools/build_ab.py 5 "3072:256:1032" > gpurun_out/ncu19_lf.log 2>&1; echo "ncu lf exit $?"
