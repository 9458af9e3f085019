# session 11: full GPU test suite, the three bench workloads, launch list + ncu --set full of the
# dominant kernels at configs[4] and configs[1] -> gpurun_out/
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke11.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/smoke11.log
timeout 1500 python bench.py > gpurun_out/bench11_c5.log 2>&1; echo "bench c5 exit $?"; tail -c 400 gpurun_out/bench11_c5.log; echo
timeout 900 python bench.py --config 2 --steps 20 --warmup 5 > gpurun_out/bench11_c2.log 2>&1; echo "bench c2 exit $?"
timeout 900 python bench.py --config 4 > gpurun_out/bench11_c4.log 2>&1; echo "bench c4 exit $?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench11_ref.log 2>&1; echo "ref exit $?"; tail -c 300 gpurun_out/bench11_ref.log; echo
export DATAGEN_CACHE_DIR=/tmp/dgc
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches11_c5.csv python tools/cfg_query.py 5 2000 > gpurun_out/ncu11_l5.log 2>&1; echo "ncu launches c5 exit $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches11_c2.csv python bench.py --config 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu11_l2.log 2>&1; echo "ncu launches c2 exit $?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_leaf_points|k_tile_pairs" -s 4 -c 2 -o gpurun_out/full11_c5 python tools/cfg_query.py 5 2000 > gpurun_out/ncu11_f5.log 2>&1; echo "ncu full c5 exit $?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_range_filter|k_leaf_points|k_project_tc" -s 6 -c 4 -o gpurun_out/full11_c2 python tools/cfg_query.py 2 > gpurun_out/ncu11_f2.log 2>&1; echo "ncu full c2 exit $?"
timeout 3000 python -m pytest tests -m gpu -q -rf -s > gpurun_out/gpu_tests11.log 2>&1; echo "all gpu tests exit $?"; tail -5 gpurun_out/gpu_tests11.log
