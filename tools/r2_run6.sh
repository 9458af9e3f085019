# session 6: build profiles, the default bench (configs[4]) end to end, launch list + full ncu of the top kernel
mkdir -p gpurun_out
FREE_GB=$(df -BG --output=avail /tmp | tail -1 | tr -dc 0-9)
if [ "${FREE_GB:-0}" -gt 120 ]; then export DATAGEN_CACHE_DIR=/tmp/dgc; echo "datagen cache on"; fi
for cfg in 2 5; do timeout 900 python tools/build_prof.py $cfg > gpurun_out/build_prof_c$cfg.json 2>&1; echo "build_prof $cfg exit $?"; head -c 1500 gpurun_out/build_prof_c$cfg.json; echo; done
unset DATAGEN_CACHE_DIR
timeout 1500 python bench.py > gpurun_out/bench6.log 2>&1; echo "bench exit $?"; tail -c 2500 gpurun_out/bench6.log
export DATAGEN_CACHE_DIR=/tmp/dgc
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c5.csv python tools/cfg_query.py 5 2000 > gpurun_out/ncu_launch6.log 2>&1; echo "ncu launches exit $?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_leaf_points -s 2 -c 1 -o gpurun_out/lp_full python tools/cfg_query.py 5 2000 > gpurun_out/ncu_full6.log 2>&1; echo "ncu full exit $?"; tail -3 gpurun_out/ncu_full6.log
