# session 8: regression check after the size rules; local-finish threshold sweep for the build
mkdir -p gpurun_out
FREE_GB=$(df -BG --output=avail /tmp | tail -1 | tr -dc 0-9)
if [ "${FREE_GB:-0}" -gt 120 ]; then export DATAGEN_CACHE_DIR=/tmp/dgc; echo "datagen cache on"; fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for cfg in 5 4 2; do
  timeout 900 python tools/qsweep.py $cfg 3 "c$cfg r8" 2>&1 | grep '^{' >> gpurun_out/qsweep8.jsonl
  tail -1 gpurun_out/qsweep8.jsonl | cut -c1-500
done
for lm in 1536 4096 8192; do
  DETLSH_LOCAL_MAX=$lm timeout 900 python tools/build_prof.py 5 > gpurun_out/build_prof8_lm$lm.json 2>&1; echo "build lm$lm exit $?"; head -c 900 gpurun_out/build_prof8_lm$lm.json; echo
done
DETLSH_LOCAL_MAX=4096 timeout 900 python tools/build_prof.py 2 > gpurun_out/build_prof8_c2_lm4096.json 2>&1; head -c 300 gpurun_out/build_prof8_c2_lm4096.json; echo
timeout 2400 python -m pytest tests -m "gpu and not slow" -q -rf -s > gpurun_out/gpu_tests8.log 2>&1; echo "fast tests exit $?"; tail -4 gpurun_out/gpu_tests8.log
