"""Commit the oracle's configs[4] results (ORACLE ONLY): gpurun_out/cfg5.{json,npz}, written on the
GPU host by tools/make_cfg5_golden.py (which calls only datagen and oracle/), become
  tests/golden/cfg5_oracle.npz   -- the 200-query subset's oracle top-k / stats at r_min and r_bench
  bench_configs.json["5"]        -- r_min (AMB-22), the operating-point sweep and r_bench (AMB-32)
No value here comes from the CUDA path.
Usage: python tools/cfg5_to_configs.py [gpurun_out/cfg5]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "cfg5")
log = json.load(open(src + ".json"))
z = np.load(src + ".npz")
keep = {k: z[k] for k in z.files}
np.savez_compressed(os.path.join(ROOT, "tests", "golden", "cfg5_oracle.npz"), **keep)
cfgs = json.load(open(os.path.join(ROOT, "bench_configs.json")))
e = {"name": "deep100m_like", "how": "oracle (tools/make_cfg5_golden.py on the GPU host): lower median of r*_q "
                                     "over 50 held-out sample queries (AMB-22)",
     "r_min": log["r_min"], "sample_queries": len(log["rstar"]),
     "rstar_p10": float(np.quantile(log["rstar"], 0.1)), "rstar_p90": float(np.quantile(log["rstar"], 0.9)),
     "point_how": f"largest m in 1..3 with oracle recall@k >= 0.95 on {log.get('nsw', 24)} held-out sample queries",
     "point_sweep": log.get("point_sweep", []), "bench_m": log.get("bench_m", 0),
     "r_bench": log.get("r_bench", log["r_min"]), "bench_oracle_recall": log.get("bench_oracle_recall"),
     "oracle_full_size": {k: log[k] for k in ("build_points_per_s_1core", "rmin_query", "rbench_query", "nproc", "procs")
                          if k in log}}
cfgs["5"] = e
json.dump(cfgs, open(os.path.join(ROOT, "bench_configs.json"), "w"), indent=1, sort_keys=True)
print(json.dumps(e, indent=1, default=float))
