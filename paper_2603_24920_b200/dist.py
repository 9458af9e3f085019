"""Multi-GPU glue for the point-sharded index -- torch.distributed plumbing only.

One process per GPU; rank g owns global ids [floor(g n/G), floor((g+1) n/G)).
  C1 (build): every rank projects ITS rows of the global sample (the n_s smallest keyed
     hashes over [0, n), AMB-4), the rows are all-gathered (NCCL), and every rank sorts the
     identical multiset -> identical breakpoints, identical codes as a 1-GPU build.
  C2 (query): queries are replicated; each rank answers with its per-shard budget
     ceil(beta n_g)+k and reports global ids; the G local top-k lists are all-gathered and
     merged by (dist, id) (detlsh_merge_topk).
The collectives run on whatever backend the process group has (nccl on GPUs, gloo in the
CPU tests); the arithmetic stays in libdetlsh.so.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import detlsh as D


def shard_range(n: int, world: int, rank: int):
    return (rank * n) // world, ((rank + 1) * n) // world


def allgather_rows(t: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather a [m_g][c] tensor with per-rank m_g (padded to the max); rows concatenated by rank."""
    world = dist.get_world_size(group)
    m = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(m) for _ in range(world)]
    dist.all_gather(sizes, m, group=group)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes)
    pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return torch.cat([o[:s] for o, s in zip(outs, sizes)], 0)


def global_breakpoints(X_shard, lo: int, n_global: int, L: int, K: int, N_r: int, seed: int,
                       sample_frac: float, opts=None, group=None, sample_projections=None,
                       breakpoints_from_samples=None):
    """C1: breakpoints of the whole dataset from the sharded sample (same on every rank).

    `sample_projections` / `breakpoints_from_samples` default to the library's calls
    (detlsh_sample_projections / detlsh_breakpoints_from_samples); the CPU tests inject the
    oracle's so the collective glue itself runs under a real (gloo) process group."""
    sp = sample_projections or D.detlsh_sample_projections
    bfs = breakpoints_from_samples or D.detlsh_breakpoints_from_samples
    Ps = sp(X_shard, L, K, N_r, seed, sample_frac, lo, n_global, opts=opts)
    if not torch.is_tensor(Ps):
        Ps = torch.from_numpy(np.ascontiguousarray(Ps))
    allp = allgather_rows(Ps.contiguous(), group)
    return bfs(allp.contiguous(), N_r, opts=opts)


def sharded_build(X_shard, lo: int, n_global: int, L: int, K: int, N_r: int, seed: int,
                  opts=None, group=None, build=None, **c1):
    """This rank's index over global ids [lo, lo + len(X_shard)) with the global breakpoints (C1).
    `build` defaults to detlsh_build (with id_offset / n_global / breakpoints); `c1` is passed
    to global_breakpoints."""
    o = opts if opts is not None else D.default_opts()
    B = global_breakpoints(X_shard, lo, n_global, L, K, N_r, seed, o.sample_frac, o, group, **c1)
    b = build or D.detlsh_build
    return b(X_shard, L, K, N_r, seed, opts=o, id_offset=lo, n_global=n_global, breakpoints=B)


def merge_shard_topk(ids, dists, k: int, group=None, merge=None):
    """C2: all-gather the local top-k lists ([nq][k] ids int64 / dists f32) and merge them.
    On GPUs the gathered lists stay on the device and detlsh_merge_topk merges them there
    (k_merge_topk); `merge` (default detlsh_merge_topk) is injectable for the CPU tests."""
    ids_t = ids if torch.is_tensor(ids) else torch.from_numpy(np.ascontiguousarray(ids))
    d_t = dists if torch.is_tensor(dists) else torch.from_numpy(np.ascontiguousarray(dists))
    world = dist.get_world_size(group)
    gi = [torch.empty_like(ids_t) for _ in range(world)]
    gd = [torch.empty_like(d_t) for _ in range(world)]
    dist.all_gather(gi, ids_t.contiguous(), group=group)
    dist.all_gather(gd, d_t.contiguous(), group=group)
    m = merge or D.detlsh_merge_topk
    return m(torch.stack(gi), torch.stack(gd), k)


def sharded_query(index, Q, k: int, c: float, r_min: float, beta: float, opts=None, group=None, merge=None):
    """Replicated queries against this rank's shard (per-shard budget ceil(beta n_g) + k), then C2."""
    res = index.query(Q, k, c, r_min, beta, opts=opts) if opts is not None else index.query(Q, k, c, r_min, beta)
    return merge_shard_topk(res[0], res[1], k, group, merge)
