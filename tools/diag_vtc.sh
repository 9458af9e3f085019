for dbg in 0 1 2 3; do
DETLSH_VTC_DEBUG=$dbg python - <<'PY'
import os, sys, json
sys.path.insert(0, '.')
import torch, datagen, paper_2603_24920_b200 as P
D = datagen.generate(2); c = D['cfg']
Xd = torch.from_numpy(D['X']).cuda(); Qd = torch.from_numpy(D['Q']).cuda()
o = P.default_opts(borrow_data=1)
g = P.detlsh_build(Xd, c.L, c.K, c.N_r, c.index_seed, opts=o)
for it in range(4):
    if it == 2: P.profile_reset(); P.profile_enable(True)
    g.query(Qd, c.k, c.c, 1.1248388401842566, c.beta, opts=o)
torch.cuda.synchronize(); P.profile_enable(False)
pr = P.profile_read()
print("dbg", os.environ["DETLSH_VTC_DEBUG"], {k: round(v[1] / v[0], 3) for k, v in pr.items() if 'verify' in k})
PY
done
