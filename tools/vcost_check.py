"""Validate the verification-path choice (verify_impl 0 = auto cost model) against measurement:
per config and radius, the whole query batch timed with the tensor-core path forced (2), the
sparse gather forced (3) and auto (0); auto should be within a few % of the faster forced one.
Usage: python tools/vcost_check.py CFG [CFG ...]  -> gpurun_out/vcost.json (appends)"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen  # noqa: E402
import paper_2603_24920_b200 as P  # noqa: E402

out_path = os.path.join(ROOT, "gpurun_out", "vcost.json")
res = json.load(open(out_path)) if os.path.exists(out_path) else []
bc = json.load(open(os.path.join(ROOT, "bench_configs.json")))
for cid in [int(a) for a in sys.argv[1:]]:
    D = datagen.generate(cid)
    c = D["cfg"]
    nq = min(c.nq, 2000)
    Xd = torch.from_numpy(D["X"]).cuda()
    Qd = torch.from_numpy(D["Q"][:nq]).cuda()
    st_ = torch.cuda.current_stream()
    g = P.detlsh_build(Xd, c.L, c.K, c.N_r, c.index_seed, opts=P.default_opts(borrow_data=1, stream=st_.cuda_stream))
    e = bc.get(str(cid), {})
    radii = sorted({e.get("r_min"), e.get("r_bench")} - {None})
    for r in radii:
        row = {"config": cid, "n": c.n, "d": c.d, "nq": nq, "r": r}
        for vi in (2, 3, 0):
            o = P.default_opts(verify_impl=vi, stream=st_.cuda_stream)
            g.query(Qd, c.k, c.c, r, c.beta, opts=o)            # warm-up
            ts = []
            for _ in range(3):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st_)
                ids, dd, st = g.query(Qd, c.k, c.c, r, c.beta, opts=o, stats=True)
                b.record(st_)
                b.synchronize()
                ts.append(a.elapsed_time(b))
            row[f"ms_v{vi}"] = float(np.median(ts))
            row["cand_per_query"] = float(st["n_cand"].mean())
            row["rounds_mean"] = float(st["rounds"].mean())
        best = min(row["ms_v2"], row["ms_v3"])
        row["auto_over_best"] = row["ms_v0"] / best
        print(json.dumps(row), flush=True)
        res.append(row)
    del g
    torch.cuda.empty_cache()
json.dump(res, open(out_path, "w"), indent=1)
