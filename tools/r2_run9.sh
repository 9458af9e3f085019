# session 9: first-layer keys from the projection, query locality sort; regression + tests
mkdir -p gpurun_out
FREE_GB=$(df -BG --output=avail /tmp | tail -1 | tr -dc 0-9)
if [ "${FREE_GB:-0}" -gt 120 ]; then export DATAGEN_CACHE_DIR=/tmp/dgc; echo "datagen cache on"; fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for qs in 1 0; do
  DETLSH_QSORT=$qs timeout 900 python tools/qsweep.py 5 3 "c5 qsort$qs" 2>&1 | grep '^{' >> gpurun_out/qsweep9.jsonl
  tail -1 gpurun_out/qsweep9.jsonl | cut -c1-500
done
timeout 900 python tools/qsweep.py 4 3 "c4 r9" 2>&1 | grep '^{' >> gpurun_out/qsweep9.jsonl; tail -1 gpurun_out/qsweep9.jsonl | cut -c1-400
timeout 900 python tools/qsweep.py 2 5 "c2 r9" 2>&1 | grep '^{' >> gpurun_out/qsweep9.jsonl; tail -1 gpurun_out/qsweep9.jsonl | cut -c1-400
for cfg in 5 2; do timeout 900 python tools/build_prof.py $cfg > gpurun_out/build_prof9_c$cfg.json 2>&1; echo "build_prof $cfg exit $?"; head -c 600 gpurun_out/build_prof9_c$cfg.json; echo; done
timeout 2400 python -m pytest tests -m "gpu and not slow" -q -rf -s > gpurun_out/gpu_tests9.log 2>&1; echo "fast tests exit $?"; tail -4 gpurun_out/gpu_tests9.log
