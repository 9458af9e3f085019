"""Diagnostic: device timeline of one index build (every launch, gaps between kernels)."""
import os, sys
os.environ["DETLSH_PROFILE_RAW"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import datagen, paper_2603_24920_b200 as P
D = datagen.generate(2, nq=10)
c = D['cfg']
Xd = torch.from_numpy(D['X']).cuda()
o = P.default_opts(borrow_data=1)
for it in range(4):
    P.profile_reset(); P.profile_enable(True)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    g = P.detlsh_build(Xd, c.L, c.K, c.N_r, c.index_seed, opts=o)
    b.record(); b.synchronize()
    P.profile_enable(False)
    print(f"=== build {it} device {a.elapsed_time(b):.3f} ms", file=sys.stderr, flush=True)
    P.profile_read()
    g.free()
