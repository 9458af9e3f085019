import os, sys
sys.path.insert(0, '.')
import numpy as np, torch, datagen, paper_2603_24920_b200 as P
D = datagen.generate(2); c = D['cfg']
Xd = torch.from_numpy(D['X']).cuda(); Qd = torch.from_numpy(D['Q']).cuda()
o = P.default_opts(borrow_data=1)
g = P.detlsh_build(Xd, c.L, c.K, c.N_r, c.index_seed, opts=o)
ids, d, st = g.query(Qd, c.k, c.c, 1.1248388401842566, c.beta, opts=o, stats=True)
for r in range(3):
    sel = st['reason'] == r
    print('reason', r, sel.sum(), 'trees_last', np.bincount(st['trees_last'][sel], minlength=5), 'rounds', np.bincount(st['rounds'][sel]))
print('ncand mean', st['n_cand'].mean())
