# session 33 (final, part 2): projection A/B at configs[4]/[1] shapes, configs[3] logical-shard
# parity, launch lists and full captures of the dominant kernels
mkdir -p gpurun_out
make -s -j8 -C paper_2603_24920_b200 > /dev/null && make -s -C oracle > /dev/null
for v in "0 0" "1 0" "0 1" "0 2" "0 4"; do set -- $v
  DETLSH_PROJ_TA=$1 DETLSH_PROJ_DEBUG=$2 timeout 300 python tools/proj_ab.py 100000000 96 6 16 2 2>&1 | tail -1
  DETLSH_PROJ_TA=$1 DETLSH_PROJ_DEBUG=$2 timeout 300 python tools/proj_ab.py 1000000 256 4 16 3 2>&1 | tail -1
done > gpurun_out/proj34.log; cat gpurun_out/proj34.log
( time timeout 2400 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -s -k "config5 or split_paths or sample_selection or breakpoints_from_samples or filter_switches or projection_variants or config3" ) > gpurun_out/tests34.log 2>&1; echo "tests exit $?"; grep -E "recall|passed|failed" gpurun_out/tests34.log | tail -12
timeout 1500 python bench.py --no-cpu-baseline > gpurun_out/bench34_c5.log 2>&1; echo "bench c5 exit $?"
export DATAGEN_CACHE_DIR=/tmp/dgc
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/launches34_c5.csv python tools/cfg_query.py 5 2000 > gpurun_out/ncu34_l5.log 2>&1; echo "ncu launches c5 exit $?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_leaf_points|k_tile_pairs" -s 6 -c 2 -o gpurun_out/full34_c5 python tools/cfg_query.py 5 2000 > gpurun_out/ncu34_f5.log 2>&1; echo "ncu full c5 exit $?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_local_finish|k_leaf_layout16|k_project_tc" -c 4 -o gpurun_out/full34_c5b python tools/cfg_query.py 5 16 > gpurun_out/ncu34_f5b.log 2>&1; echo "ncu full c5 build exit $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_leaf_points|k_range_filter" -s 8 -c 2 -o gpurun_out/full34_c2 python tools/cfg_query.py 2 > gpurun_out/ncu34_f2.log 2>&1; echo "ncu full c2 exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches34_c2.csv python bench.py --config 2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu34_l2.log 2>&1; echo "ncu launches c2 exit $?"
