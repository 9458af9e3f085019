"""A/B of build settings read per build call (DETLSH_LOCAL_MAX, DETLSH_LF_THREADS, DETLSH_PDL): one data
generation, one build per setting (device-resident X), wall time per build (after a warm-up
build), and tree 0 (perm, leaf offsets) compared with the first setting's.
Usage: python tools/build_ab.py CFG "LM:THREADS[:PDL],..." (THREADS 0: per tier; PDL default 1)"""
import hashlib
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen  # noqa: E402
import paper_2603_24920_b200 as P  # noqa: E402

cid = int(sys.argv[1])
sets = [tuple(int(v) for v in (s + ":1").split(":")[:3]) for s in sys.argv[2].split(",")]
D = datagen.generate(cid, nq=16)
c = D["cfg"]
Xd = torch.from_numpy(D["X"]).cuda()
del D
ref = None
for rep in range(2):
    for lm, nt, pdl in sets:
        os.environ["DETLSH_LOCAL_MAX"] = str(lm)
        os.environ["DETLSH_LF_THREADS"] = str(nt)
        os.environ["DETLSH_PDL"] = str(pdl)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g = P.detlsh_build(Xd, c.L, c.K, c.N_r, c.index_seed, opts=P.default_opts(borrow_data=1))
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
        h = None
        if rep == 1:
            tr = g.tree(0)
            h = hashlib.sha1(tr["perm"].tobytes() + tr["leaf_off"].tobytes()).hexdigest()[:12]
            if ref is None:
                ref = h
        print(f"cfg {cid} LM {lm} LF_THREADS {nt} PDL {pdl} rep {rep}: build {ms:.1f} ms, {Xd.shape[0] / ms / 1e3:.1f} M pts/s, "
              f"tree0 {h} same {h == ref if h else None}", flush=True)
        g.free()
        del g
