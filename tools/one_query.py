"""Build configs[1] once and run N queries of its 1000 queries (for ncu captures: the first query
is the warm-up; kernels of the second are the ones to capture)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import datagen, paper_2603_24920_b200 as P
cid = int(os.environ.get("CFG", "2"))
D = datagen.generate(cid)
c = D['cfg']
import json
_e = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "bench_configs.json")))[str(cid)]
rmin = _e.get("r_bench", _e["r_min"])
Xd = torch.from_numpy(D['X']).cuda(); Qd = torch.from_numpy(D['Q']).cuda()
o = P.default_opts(borrow_data=1)
g = P.detlsh_build(Xd, c.L, c.K, c.N_r, c.index_seed, opts=o)
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    g.query(Qd, c.k, c.c, rmin, c.beta, opts=o)
torch.cuda.synchronize()
print("ok")
