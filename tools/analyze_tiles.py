"""CPU study (oracle index, no GPU): how many leaves/tiles a query's range filter must test at
the bench radius under different tile layouts.  Exact fp64 lower bounds, tree 0, a sample of
queries.  Usage: python tools/analyze_tiles.py [cid] [nq]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
from oracle import oracle as O  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 20
D = datagen.generate(cid, nq=nq)
c = D["cfg"]
t0 = time.time()
ix = O.Index(D["X"], c.L, c.K, c.N_r, c.index_seed, c.max_size, c.sample_frac)
print(f"oracle build {time.time() - t0:.1f} s", flush=True)
r = json.load(open(os.path.join(os.path.dirname(__file__), "..", "bench_configs.json")))[str(cid)]["r_bench"]
rho2 = (ix.eps * r) ** 2
Bp = ix.breakpoints().astype(np.float64)      # [LK][N_r+1]
codes = ix.codes()                              # [n][LK]
K, N_r = c.K, c.N_r
t = 0
tr = ix.tree(t)
off, perm = tr["leaf_off"], tr["perm"]
nl = len(off) - 1
tc = codes[perm][:, t * K:(t + 1) * K].astype(np.int64)       # tree order
lo = np.minimum.reduceat(tc, off[:-1], axis=0)
hi = np.maximum.reduceat(tc, off[:-1], axis=0)
first = np.zeros(nl, np.int64)                  # first-layer cell id of each leaf: MSB vector
for j in range(K):
    first = first * 2 + (lo[:, j] >> 7)
print(f"leaves {nl}, mean size {np.mean(np.diff(off)):.1f}, first-layer cells {len(np.unique(first))}")


def dtab(qp):
    """[K][N_r] squared distance from q'_j to region s of dim j."""
    b = Bp[t * K:(t + 1) * K]
    lo_ = np.concatenate([np.full((K, 1), -np.inf), b[:, 1:N_r]], axis=1)
    hi_ = np.concatenate([b[:, 1:N_r], np.full((K, 1), np.inf)], axis=1)
    x = qp[:, None]
    v = np.maximum(0, np.maximum(lo_ - x, x - hi_))
    return v * v


def box_lb(T, sx, blo, bhi):
    cl = np.clip(sx[None, :], blo, bhi)
    return T[np.arange(K)[None, :], cl].sum(1)


def tiles_fixed(size):
    b = np.arange(0, nl, size)
    return [(s, min(s + size, nl)) for s in b]


def tiles_cells(maxlen):
    out, s = [], 0
    while s < nl:
        e = s + 1
        while e < nl and e - s < maxlen and first[e] == first[s]:
            e += 1
        out.append((s, e))
        s = e
    return out


layouts = {"fixed32": tiles_fixed(32), "fixed16": tiles_fixed(16), "fixed8": tiles_fixed(8),
           "cell<=32": tiles_cells(32), "cell<=16": tiles_cells(16)}
stats = {k: [0, 0, 0] for k in layouts}   # tiles tested, tiles passed, leaves in passed tiles
hier = {"64>8>1": [64, 8], "128>16>1": [128, 16], "256>32>4>1": [256, 32, 4], "32>4>1": [32, 4], "16>1": [16],
        "512>64>8>1": [512, 64, 8]}
hstats = {k: 0 for k in hier}
lp = pt = pp = 0
for qi in range(nq):
    qp = ix.project_query(D["Q"][qi]).astype(np.float64)[t * K:(t + 1) * K]
    T = dtab(qp)
    sx = np.array([np.searchsorted(Bp[t * K + j, 1:N_r], qp[j], side="left") for j in range(K)])
    llb = box_lb(T, sx, lo, hi)
    lpass = llb <= rho2
    lp += lpass.sum()
    sizes = np.diff(off)
    pt += sizes[lpass].sum()
    pts = tc[np.repeat(lpass, sizes)]
    plb = T[np.arange(K)[None, :], pts].sum(1)
    pp += (plb <= rho2).sum()
    for name, tl in layouts.items():
        s_ = np.array([a for a, _ in tl]); e_ = np.array([b for _, b in tl])
        tlo = np.minimum.reduceat(lo, s_, axis=0)
        thi = np.maximum.reduceat(hi, s_, axis=0)
        tpass = box_lb(T, sx, tlo, thi) <= rho2
        st = stats[name]
        st[0] += len(tl)
        st[1] += tpass.sum()
        st[2] += (e_ - s_)[tpass].sum()
    for name, lv in hier.items():
        alive = np.ones(1, bool)         # root
        tested = 0
        prev = nl
        sizes_ = lv + [1]
        cur_alive = None
        for li, sz in enumerate(sizes_):
            starts = np.arange(0, nl, sz)
            if li == 0:
                cand = np.ones(len(starts), bool)
            else:
                cand = np.repeat(cur_alive, sizes_[li - 1] // sz)[:len(starts)]
            tested += cand.sum()
            blo = np.minimum.reduceat(lo, starts, axis=0)
            bhi = np.maximum.reduceat(hi, starts, axis=0)
            cur_alive = cand & (box_lb(T, sx, blo, bhi) <= rho2)
        hstats[name] += tested
print(f"per query (tree 0, {nq} queries): leaves passed {lp / nq:.0f}, points tested {pt / nq:.0f}, points passed {pp / nq:.0f}")
for name, (a, b, l_) in stats.items():
    print(f"  {name:9s} tiles {a / nq:7.0f}  passed {b / nq:7.0f}  leaves tested {l_ / nq:8.0f}  "
          f"(tile tests + leaf tests {(a + l_) / nq:8.0f})")
for name, v in hstats.items():
    print(f"  hier {name:12s} box tests {v / nq:8.0f}")
