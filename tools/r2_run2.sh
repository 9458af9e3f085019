# round-2 GPU session: smoke, benches (configs[1] and configs[4], tile-screen variants), then the
# GPU test suite (fast tests first, the full-size slow ones last) -> gpurun_out/
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv,noheader
echo "nproc $(nproc)"; free -g | head -2; df -h /tmp | tail -1
FREE_GB=$(df -BG --output=avail /tmp | tail -1 | tr -dc 0-9)
if [ "${FREE_GB:-0}" -gt 120 ]; then export DATAGEN_CACHE_DIR=/tmp/dgc; echo "datagen cache on"; fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/smoke.log
summ() { python - "$1" <<'PY'
import json, sys
try:
    d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
except Exception as e:
    print(sys.argv[1], "no JSON line", e); sys.exit()
print(sys.argv[1], "value", round(d["value"]), "query_ms", round(d["query_ms_per_step"], 3), "build_ms", round(d["build"]["ms_per_step"], 3),
      "recall", d["recall_at_k"], "cand/q", round(d["candidates_per_query"]), "stops", d["stop_reasons"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
for k, v in list(d["kernels"].items())[:10]: print("   ", k, v["launches"], round(v["ms"] / d["steps"], 3), "ms/step")
print("   filter counts", d["filter_counts_per_query"])
PY
}
for cfg in 2 5; do
  for ts in 0 1; do
    f=gpurun_out/b_c${cfg}_ts${ts}.log
    DETLSH_RF_TSCREEN=$ts timeout 1500 python bench.py --config $cfg --steps ${STEPS:-5} --no-cpu-baseline --recall-queries 50 > $f 2>&1
    echo "bench cfg$cfg ts$ts exit $?"; summ $f
  done
done
timeout 2400 python -m pytest tests -m "gpu and not slow" -q -rf -s > gpurun_out/gpu_tests_fast.log 2>&1; echo "fast tests exit $?"; tail -12 gpurun_out/gpu_tests_fast.log
timeout 3000 python -m pytest tests -m "gpu and slow" -q -rf -s > gpurun_out/gpu_tests_slow.log 2>&1; echo "slow tests exit $?"; tail -12 gpurun_out/gpu_tests_slow.log
timeout 900 python tools/vcost_check.py 3 5 > gpurun_out/vcost.log 2>&1; echo "vcost exit $?"; tail -6 gpurun_out/vcost.log
timeout 2400 bash tools/sanitize.sh > gpurun_out/sanitize.log 2>&1; echo "sanitize exit $?"; cat gpurun_out/sanitize.log
