import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import datagen, paper_2603_24920_b200 as P
D = datagen.generate(2, nq=1000)
c = D['cfg']
Xd = torch.from_numpy(D['X']).cuda(); Qd = torch.from_numpy(D['Q']).cuda()
o = P.default_opts(borrow_data=1)
for it in range(5):
    if it >= 3: os.environ['DETLSH_TRACE'] = '1'
    torch.cuda.synchronize(); t = time.perf_counter()
    g = P.detlsh_build(Xd, c.L, c.K, c.N_r, c.index_seed, opts=o)
    torch.cuda.synchronize(); tb = time.perf_counter() - t
    ids, d = g.query(Qd, c.k, c.c, 1.1248388401842566, c.beta, opts=o)
    torch.cuda.synchronize(); tq = time.perf_counter() - t - tb
    print(f'iter {it}: build {tb*1e3:.2f} ms, query {tq*1e3:.2f} ms', file=sys.stderr, flush=True)
    g.free()
