"""Multi-process (gloo, world_size 2, CPU) tests of the point-sharded glue.

The collectives of paper_2603_24920_b200.dist run here on gloo; the per-shard arithmetic is
stood in for by the oracle (no GPU in this container), so what is checked is the glue:
C1 row all-gather -> identical global breakpoints, and C2 top-k all-gather + merge ->
the oracle's own G-shard result (O9).
"""
import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import datagen
        from oracle import oracle as O
        from paper_2603_24920_b200 import dist as PD

        # allgather_rows with ragged sizes
        t = torch.full((rank + 2, 3), float(rank))
        allr = PD.allgather_rows(t)
        assert allr.shape == (5, 3) and allr[:2].eq(0).all() and allr[2:].eq(1).all()

        D = datagen.generate(1, n=3000, nq=12)
        X, Q = D["X"], D["Q"]
        n = X.shape[0]
        L, K, N_r, seed = 4, 16, 256, 42
        lo, hi = PD.shard_range(n, world, rank)
        sh = O.Index(X, L, K, N_r, seed, row_lo=lo, row_hi=hi)   # the oracle's shard g (O9)
        calls = []

        # The per-shard arithmetic the library does on the GPU, stood in for by the oracle; the
        # glue (C1 all-gather of ragged row sets, breakpoint hand-off, C2 all-gather + merge) is
        # dist.py's own code under the gloo process group.
        def sample_projections(X_shard, L_, K_, N_r_, seed_, frac, lo_, n_global, opts=None):
            assert (L_, K_, N_r_, seed_, lo_, n_global) == (L, K, N_r, seed, lo, n)
            assert X_shard.shape[0] == hi - lo
            sample = sh.sample()                  # global ids of the whole-dataset sample
            mine = sample[(sample >= lo) & (sample < hi)] - lo
            calls.append("sample")
            return sh.P()[mine]

        def breakpoints_from_samples(allp, N_r_, opts=None):
            calls.append(("bp", allp.shape[0]))
            allp = allp.numpy()
            return np.stack([O.breakpoints_sort(allp[:, r], N_r_) for r in range(allp.shape[1])])

        def build(X_shard, L_, K_, N_r_, seed_, opts=None, id_offset=0, n_global=None, breakpoints=None):
            assert id_offset == lo and n_global == n
            assert np.array_equal(breakpoints, sh.breakpoints())   # C1 result == the oracle shard's
            calls.append("build")
            return sh

        ix = PD.sharded_build(X[lo:hi], lo, n, L, K, N_r, seed, opts=SimpleNamespace(sample_frac=0.01),
                              build=build, sample_projections=sample_projections,
                              breakpoints_from_samples=breakpoints_from_samples)
        assert ix is sh and calls[0] == "sample" and calls[-1] == "build"
        assert calls[1] == ("bp", O.sample_size(n, N_r, 0.01))     # every rank saw the whole sample
        whole = O.Index(X, L, K, N_r, seed)
        assert np.array_equal(sh.breakpoints(), whole.breakpoints())
        # C2: local top-k with global ids, all-gather, merge
        mi, md = PD.sharded_query(ix, Q, 10, 1.5, 300.0, 0.1,
                                  merge=lambda gi, gd, k: O.merge_topk(gi.numpy(), gd.numpy(), k))
        ri, rd = O.sharded_query(X, world, Q, 10, 1.5, 300.0, 0.1, L, K, N_r, seed)
        assert np.array_equal(mi, ri) and np.array_equal(md, rd)
        out_q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        out_q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_sharded_glue_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def test_shard_ranges_partition():
    from paper_2603_24920_b200 import dist as PD
    for n in (1, 7, 1000, 10_000_001):
        for G in (1, 2, 3, 8):
            rs = [PD.shard_range(n, G, g) for g in range(G)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
