# session 14 (final measurements): full GPU test suite, the bench lines, launch lists and full
# captures of the dominant kernels -> gpurun_out/
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke14.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/smoke14.log
timeout 1500 python bench.py > gpurun_out/bench14_c5.log 2>&1; echo "bench c5 exit $?"
timeout 900 python bench.py --config 2 --steps 20 --warmup 5 > gpurun_out/bench14_c2.log 2>&1; echo "bench c2 exit $?"
timeout 900 python bench.py --config 4 > gpurun_out/bench14_c4.log 2>&1; echo "bench c4 exit $?"
timeout 900 python bench.py --radius amb22 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench14_c5_amb22.log 2>&1; echo "bench c5 amb22 exit $?"
export DATAGEN_CACHE_DIR=/tmp/dgc
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches14_c5.csv python tools/cfg_query.py 5 2000 > gpurun_out/ncu14_l5.log 2>&1; echo "ncu launches c5 exit $?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_leaf_points|k_tile_pairs|k_project_tc|k_leaf_layout16|k_local_finish" -s 2 -c 6 -o gpurun_out/full14_c5 python tools/cfg_query.py 5 2000 > gpurun_out/ncu14_f5.log 2>&1; echo "ncu full c5 exit $?"
unset DATAGEN_CACHE_DIR
timeout 3000 python -m pytest tests -m gpu -q -rf -s > gpurun_out/gpu_tests14.log 2>&1; echo "all gpu tests exit $?"; tail -3 gpurun_out/gpu_tests14.log
