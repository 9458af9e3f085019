# short bench (no tests, no cpu baseline) -> summary
timeout 600 python bench.py --steps ${STEPS:-10} --no-cpu-baseline --recall-queries 50 ${BENCH_ARGS} > gpurun_out/bench_quick.log 2>&1; echo "bench exit $?"
python - <<'PY'
import json
d=json.loads([l for l in open("gpurun_out/bench_quick.log") if l.startswith("{")][-1])
print("value", round(d["value"]), "query_ms", round(d["query_ms_per_step"],3), "e2e", round(d["e2e"]["value"]), "build_ms", round(d["build"]["ms_per_step"],3), "recall", d["recall_at_k"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
print(d["filter_counts_per_query"])
for k,v in list(d["kernels"].items())[:8]: print("  ", k, v["launches"], round(v["ms"]/d["steps"],3), "ms/step")
PY
python - <<'PY'
import json
d=json.loads([l for l in open("gpurun_out/bench_quick.log") if l.startswith("{")][-1])
for r in d["rooflines"]: print("  roof", r["kernel"], r["bound"], r["achieved"], r["unit"], r["frac"], r.get("traffic"), r.get("parts_ms"))
print("  dominant", d["roofline"]["kernel"], d["roofline"]["frac"], d["roofline"].get("share_of_step"))
PY
