# session 5: within-leaf Morton order (sub-box tightness) at configs[4], [3], [1]; parity tests
mkdir -p gpurun_out
FREE_GB=$(df -BG --output=avail /tmp | tail -1 | tr -dc 0-9)
if [ "${FREE_GB:-0}" -gt 120 ]; then export DATAGEN_CACHE_DIR=/tmp/dgc; echo "datagen cache on"; fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for cfg in 5 4 2; do
  for mo in 0 1; do
    DETLSH_LEAF_MORTON=$mo timeout 900 python tools/qsweep.py $cfg 3 "c$cfg morton$mo" 2>&1 | grep '^{' >> gpurun_out/qsweep5.jsonl
    tail -1 gpurun_out/qsweep5.jsonl | cut -c1-600
  done
done
timeout 2400 python -m pytest tests -m "gpu and not slow" -q -rf -s > gpurun_out/gpu_tests5.log 2>&1; echo "fast tests exit $?"; tail -4 gpurun_out/gpu_tests5.log
