"""Query batch size A/B: one build of a BASELINE config, the same queries with opts.query_batch
= each value (0 = sized from free memory); results must be identical.
Usage: python tools/batch_ab.py CFG NQ qb1,qb2,..."""
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

cid, nq = int(sys.argv[1]), int(sys.argv[2])
qbs = [int(v) for v in sys.argv[3].split(",")]
D = datagen.generate(cid)
c = D["cfg"]
r = json.load(open(os.path.join(ROOT, "bench_configs.json")))[str(cid)]["r_bench"]
Xd = torch.from_numpy(D["X"]).cuda()
Qd = torch.from_numpy(D["Q"][:nq]).cuda()
g = P.detlsh_build(Xd, c.L, c.K, c.N_r, c.index_seed, opts=P.default_opts(borrow_data=1))
torch.cuda.synchronize()
ref = None
for rep in range(2):
    for qb in qbs:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ids, dists = g.query(Qd, c.k, c.c, r, c.beta, opts=P.default_opts(query_batch=qb))
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
        ids, dists = ids.cpu().numpy(), dists.cpu().numpy()
        same = None
        if ref is None:
            ref = (ids, dists)
        else:
            same = bool(np.array_equal(ids, ref[0]) and np.array_equal(dists, ref[1]))
        print(f"cfg {cid} nq {nq} query_batch {qb} rep {rep}: {ms:.1f} ms, {nq / ms * 1e3:.0f} q/s, identical {same}",
              flush=True)
