"""Query-phase timing of one BASELINE config under the current DETLSH_* switches (experiments):
build once, answer every query at r_bench `reps` times (CUDA events), print one JSON line with the
median ms, the per-kernel device times and the filter counters.
Usage: [DETLSH_...=...] python tools/qsweep.py CFG [REPS] [TAG]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen  # noqa: E402
import paper_2603_24920_b200 as P  # noqa: E402

cid = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
tag = sys.argv[3] if len(sys.argv) > 3 else ""
D = datagen.generate(cid)
c = D["cfg"]
r = json.load(open(os.path.join(ROOT, "bench_configs.json")))[str(cid)]["r_bench"]
st_ = torch.cuda.current_stream()
Xd = torch.from_numpy(D["X"]).cuda()
Qd = torch.from_numpy(D["Q"]).cuda()
o = P.default_opts(borrow_data=1, stream=st_.cuda_stream)
g = P.detlsh_build(Xd, c.L, c.K, c.N_r, c.index_seed, opts=o)
g.query(Qd, c.k, c.c, r, c.beta, opts=o)          # warm-up (arenas)
ts = []
P.profile_reset()
P.profile_filter("")
for i in range(reps):
    if i == reps - 1:
        P.profile_enable(True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st_)
    ids, dd, st = g.query(Qd, c.k, c.c, r, c.beta, opts=o, stats=True)
    b.record(st_)
    b.synchronize()
    ts.append(a.elapsed_time(b))
P.profile_enable(False)
prof = P.profile_read()
ker = {k: round(v[1], 3) for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])[:10]}
env = {k: v for k, v in os.environ.items() if k.startswith("DETLSH_")}
print(json.dumps({"tag": tag, "config": cid, "env": env, "query_ms": float(np.median(ts[:-1] if reps > 1 else ts)),
                  "qps": c.nq / (float(np.median(ts[:-1] if reps > 1 else ts)) / 1e3),
                  "cand_per_query": float(st["n_cand"].mean()), "kernels_ms_last_rep(profiled)": ker,
                  "counts": {k: float(st[k].mean()) for k in ("leaves_tested", "leaves_passed", "points_tested",
                                                            "subboxes_tested")}}), flush=True)
