# session 37: the shortened full-size GPU tests (the driver's GPU test step is limited to 1200 s)
mkdir -p gpurun_out
make -s -j8 -C paper_2603_24920_b200 > /dev/null && make -s -C oracle > /dev/null
( time timeout 1100 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -rf -s --durations=12 -k "full_size or shards_config3" ) > gpurun_out/tests37.log 2>&1; echo "tests exit $?"; grep -E "cfg4|configs\[3\]|passed|failed|^[0-9.]+s " gpurun_out/tests37.log | cut -c1-260 | tail -30
