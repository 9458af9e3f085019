# session 38: the whole GPU suite in the driver's form, timed against its 1200 s step limit
mkdir -p gpurun_out
make -s -j8 -C paper_2603_24920_b200 > /dev/null && make -s -C oracle > /dev/null
( time timeout 1200 python -m pytest tests/ -x -q -m gpu --durations=10 ) > gpurun_out/gpu_tests38.log 2>&1; echo "all gpu tests exit $?"; tail -16 gpurun_out/gpu_tests38.log
