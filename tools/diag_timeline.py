"""Diagnostic: device timeline (every launch) of repeated queries, to find stalls between kernels."""
import os, sys, time
os.environ["DETLSH_PROFILE_RAW"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import datagen, paper_2603_24920_b200 as P
D = datagen.generate(2)
c = D['cfg']
Xd = torch.from_numpy(D['X']).cuda(); Qd = torch.from_numpy(D['Q']).cuda()
st = torch.cuda.current_stream()
o = P.default_opts(borrow_data=1, stream=st.cuda_stream)
g = P.detlsh_build(Xd, c.L, c.K, c.N_r, c.index_seed, opts=o)
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    rebuild = len(sys.argv) > 2
    P.profile_reset(); P.profile_enable(True)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    if rebuild:
        g.free(); g = P.detlsh_build(Xd, c.L, c.K, c.N_r, c.index_seed, opts=o)
    g.query(Qd, c.k, c.c, 0.4999283734152251, c.beta, opts=o, stats=True)
    b.record(st); b.synchronize()
    P.profile_enable(False)
    print(f"=== iter {it} device {a.elapsed_time(b):.2f} ms", file=sys.stderr, flush=True)
    P.profile_read()
