"""A/B of a query switch the library reads per query call: one build of a BASELINE config, then
the same query batch per value of the environment variable VAR (e.g. DETLSH_BOX16); results must
be identical, device-synchronised wall time per call printed (two rounds).
Usage: python tools/query_ab.py CFG NQ VAR v1,v2,..."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen  # noqa: E402
import paper_2603_24920_b200 as P  # noqa: E402

cid, nq, var = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
vals = sys.argv[4].split(",")
D = datagen.generate(cid)
c = D["cfg"]
r = json.load(open(os.path.join(ROOT, "bench_configs.json")))[str(cid)]["r_bench"]
Xd = torch.from_numpy(D["X"]).cuda()
Qd = torch.from_numpy(D["Q"][:nq]).cuda()
g = P.detlsh_build(Xd, c.L, c.K, c.N_r, c.index_seed, opts=P.default_opts(borrow_data=1))
torch.cuda.synchronize()
ref = None
for rep in range(3):
    for v in vals:
        os.environ[var] = v
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ids, dists, st = g.query(Qd, c.k, c.c, r, c.beta, stats=True)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
        ids, dists = ids.cpu().numpy(), dists.cpu().numpy()
        same = None
        if ref is None:
            ref = (ids, dists)
        else:
            same = bool(np.array_equal(ids, ref[0]) and np.array_equal(dists, ref[1]))
        print(f"cfg {cid} nq {nq} {var}={v} rep {rep}: {ms:.1f} ms, {nq / ms * 1e3:.0f} q/s, "
              f"cand {float(st['n_cand'].mean()):.0f}, identical {same}", flush=True)
