"""Diagnostic: host phase trace (DETLSH_TRACE) of repeated index builds at a config."""
import os, sys
os.environ["DETLSH_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import datagen, paper_2603_24920_b200 as P
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
D = datagen.generate(cid, nq=10)
c = D['cfg']
Xd = torch.from_numpy(D['X']).cuda()
o = P.default_opts(borrow_data=1)
for it in range(5):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    g = P.detlsh_build(Xd, c.L, c.K, c.N_r, c.index_seed, opts=o)
    b.record(); b.synchronize()
    print(f"=== build {it} device {a.elapsed_time(b):.3f} ms", file=sys.stderr, flush=True)
    g.free()
