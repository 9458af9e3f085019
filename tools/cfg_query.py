"""One build + one query batch of a BASELINE config at its bench radius (for ncu captures of the
query kernels).  Usage: python tools/cfg_query.py CFG [NQ]"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen  # noqa: E402
import paper_2603_24920_b200 as P  # noqa: E402

cid = int(sys.argv[1])
nq = int(sys.argv[2]) if len(sys.argv) > 2 else None
D = datagen.generate(cid)
c = D["cfg"]
r = json.load(open(os.path.join(ROOT, "bench_configs.json")))[str(cid)]["r_bench"]
Xd = torch.from_numpy(D["X"]).cuda()
Q = D["Q"] if nq is None else D["Q"][:nq]
g = P.detlsh_build(Xd, c.L, c.K, c.N_r, c.index_seed, opts=P.default_opts(borrow_data=1))
ids, dists, st = g.query(torch.from_numpy(Q).cuda(), c.k, c.c, r, c.beta, stats=True)
torch.cuda.synchronize()
print("ok", Q.shape[0], float(st["n_cand"].mean()))
