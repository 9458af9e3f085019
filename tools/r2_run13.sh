# session 13: clamp-free box bounds in the pair kernel; regression + tests
mkdir -p gpurun_out
FREE_GB=$(df -BG --output=avail /tmp | tail -1 | tr -dc 0-9)
if [ "${FREE_GB:-0}" -gt 120 ]; then export DATAGEN_CACHE_DIR=/tmp/dgc; echo "datagen cache on"; fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for cfg in 5 4 2; do
  timeout 900 python tools/qsweep.py $cfg 3 "c$cfg r13" 2>&1 | grep '^{' >> gpurun_out/qsweep13.jsonl
  tail -1 gpurun_out/qsweep13.jsonl | cut -c1-400
done
timeout 2400 python -m pytest tests -m "gpu and not slow" -q -rf -s > gpurun_out/gpu_tests13.log 2>&1; echo "fast tests exit $?"; tail -3 gpurun_out/gpu_tests13.log
