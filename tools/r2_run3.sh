# round-2 GPU session 3: variants of the filter / projection at configs[4] and configs[1], the new
# tests, and a launch list of the configs[4] bench -> gpurun_out/
mkdir -p gpurun_out
FREE_GB=$(df -BG --output=avail /tmp | tail -1 | tr -dc 0-9)
if [ "${FREE_GB:-0}" -gt 120 ]; then export DATAGEN_CACHE_DIR=/tmp/dgc; echo "datagen cache on"; fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/smoke.log
summ() { python - "$1" <<'PY'
import json, sys
try:
    d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
except Exception as e:
    print(sys.argv[1], "no JSON line", e); sys.exit()
print(sys.argv[1], "value", round(d["value"]), "query_ms", round(d["query_ms_per_step"], 3), "build_ms", round(d["build"]["ms_per_step"], 3),
      "recall", d["recall_at_k"], "cand/q", round(d["candidates_per_query"]), "stops", d["stop_reasons"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
for k, v in list(d["kernels"].items())[:12]: print("   ", k, v["launches"], round(v["ms"] / d["steps"], 3), "ms/step")
print("   filter counts", d["filter_counts_per_query"])
PY
}
run() {   # run TAG CFG ENV...
  tag=$1; cfg=$2; shift 2
  f=gpurun_out/b3_${tag}.log
  env "$@" timeout 1500 python bench.py --config $cfg --steps ${STEPS:-5} --no-cpu-baseline --recall-queries 50 > $f 2>&1
  echo "bench $tag exit $?"; summ $f
}
run c5_base 5 DETLSH_TILE_PAIRS=0
run c5_tp 5 DETLSH_TILE_PAIRS=1
run c5_tp_ta 5 DETLSH_TILE_PAIRS=1 DETLSH_PROJ_TA=1
run c2_base 2 DETLSH_TILE_PAIRS=0
run c2_tp 2 DETLSH_TILE_PAIRS=1
run c2_ta 2 DETLSH_PROJ_TA=1
timeout 1800 python -m pytest tests -m gpu -q -rf -s -k "switches or projection_variants or breakpoints_from or trees_ or merge or sample" > gpurun_out/gpu_tests3.log 2>&1; echo "tests exit $?"; tail -8 gpurun_out/gpu_tests3.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,l1tex__t_sector_hit_rate.pct,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active
for tp in 0 1; do
  DETLSH_TILE_PAIRS=$tp timeout 1200 ncu --metrics $M --clock-control none -k regex:"k_leaf_points|k_range_filter|k_tile_pairs" -c 12 --csv \
     python tools/cfg_query.py 5 2000 > gpurun_out/ncu_c5_tp$tp.csv 2> gpurun_out/ncu_c5_tp$tp.err; echo "ncu tp$tp exit $?"
done
