"""Write bench_configs.json: the initial radius r_min of each config (AMB-22), computed by
the ORACLE only (oracle.estimate_rmin: lower median over seeded sample queries of the
smallest radius whose full round reaches |S| >= ceil(beta n)+k).  Both the CUDA
path and the oracle then receive this same r_min.

Operating point ("a sweep r_min c^-m (m = 0..6) may report the fastest point
with recall >= 0.9"): with --point, the oracle also answers the held-out sample queries at
r_min c^-m, m = 0..6, and records r_bench = r_min c^-m* for the largest m* whose oracle
recall@k (vs the oracle's exact kNN) is >= 0.95 -- a margin over the 0.9 target.  bench.py
(both arms) runs at r_bench.  Only oracle/ is called.
Usage: python tools/make_rmin.py [--point] 1 2 3
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
from oracle import oracle as O  # noqa: E402

NS = 50   # sample queries (datagen stream 3, held out from the query set)
OUT = os.path.join(ROOT, "bench_configs.json")


def operating_point(ix, D, c, r_min):
    Qs = D["Qs"]
    gt, _ = O.exact_knn(D["X"], Qs, c.k)
    pts = []
    for m in range(7):
        r = r_min * c.c ** (-m)
        ids, _, _ = ix.query(Qs, c.k, c.c, r, c.beta)
        rec = float(np.mean([len(set(ids[i]) & set(gt[i])) / c.k for i in range(len(Qs))]))
        pts.append({"m": m, "r": r, "oracle_recall": rec})
        print("   m", m, "r", r, "oracle recall", rec, flush=True)
    ok = [p for p in pts if p["oracle_recall"] >= 0.95]
    best = max(ok, key=lambda p: p["m"]) if ok else pts[0]
    return best, pts


def main(cfg_ids, point=False):
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for cid in cfg_ids:
        t0 = time.time()
        D = datagen.generate(cid, nq=1, with_sample_queries=NS)
        c = D["cfg"]
        ix = O.Index(D["X"], c.L, c.K, c.N_r, c.index_seed, c.max_size, c.sample_frac)
        med, rs = ix.estimate_rmin(D["Qs"], c.k, c.c, c.beta, return_all=True)
        data[str(cid)] = {"name": c.name, "r_min": med, "rstar_p10": float(sorted(rs)[NS // 10]),
                          "rstar_p90": float(sorted(rs)[(9 * NS) // 10]), "sample_queries": NS,
                          "how": "oracle.estimate_rmin (lower median of r*_q), tools/make_rmin.py"}
        if point:
            best, pts = operating_point(ix, D, c, med)
            data[str(cid)].update({"bench_m": best["m"], "r_bench": best["r"], "bench_oracle_recall": best["oracle_recall"],
                                   "point_sweep": pts,
                                   "point_how": "largest m in 0..6 with oracle recall@k >= 0.95 on the sample queries"})
        print(cid, data[str(cid)], f"{time.time() - t0:.1f}s", flush=True)
        json.dump(data, open(OUT, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    main([int(a) for a in args] or [1, 2, 3], point="--point" in sys.argv)
