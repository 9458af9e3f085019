"""Write bench_configs.json: the initial radius r_min of each config (AMB-22), computed by
the ORACLE only (oracle.estimate_rmin: lower median over seeded sample queries of the
smallest radius whose full round reaches |S| >= ceil(beta n)+k).  Both the CUDA
path and the oracle then receive this same r_min.  Usage: python tools/make_rmin.py 1 2 3
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
from oracle import oracle as O  # noqa: E402

NS = 50   # sample queries (datagen stream 3, held out from the query set)
OUT = os.path.join(ROOT, "bench_configs.json")


def main(cfg_ids):
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
        print(cid, data[str(cid)], f"{time.time() - t0:.1f}s", flush=True)
        json.dump(data, open(OUT, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 2, 3])
