# quick GPU check: parity tests + a short bench (no cpu baseline) -> summary line
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps ${STEPS:-10} --no-cpu-baseline --recall-queries 50 > gpurun_out/bench_quick.log 2>&1; echo "bench exit $?"
python - <<'PY'
import json
d=json.loads([l for l in open("gpurun_out/bench_quick.log") if l.startswith("{")][-1])
print("value", round(d["value"]), "query_ms", round(d["query_ms_per_step"],3), "e2e", round(d["e2e"]["value"]), "build_ms", round(d["build"]["ms_per_step"],3), "recall", d["recall_at_k"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
for k,v in list(d["kernels"].items())[:8]: print("  ", k, v["launches"], round(v["ms"]/d["steps"],3), "ms/step")
PY
