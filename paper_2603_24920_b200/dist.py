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
                       sample_frac: float, opts=None, group=None):
    """C1: breakpoints of the whole dataset from the sharded sample (same on every rank)."""
    Ps = D.detlsh_sample_projections(X_shard, L, K, N_r, seed, sample_frac, lo, n_global, opts=opts)
    if not torch.is_tensor(Ps):
        Ps = torch.from_numpy(np.ascontiguousarray(Ps))
    allp = allgather_rows(Ps.contiguous(), group)
    return D.detlsh_breakpoints_from_samples(allp.contiguous(), N_r, opts=opts)


def sharded_build(X_shard, lo: int, n_global: int, L: int, K: int, N_r: int, seed: int,
                  opts=None, group=None):
    o = opts if opts is not None else D.default_opts()
    B = global_breakpoints(X_shard, lo, n_global, L, K, N_r, seed, o.sample_frac, o, group)
    return D.detlsh_build(X_shard, L, K, N_r, seed, opts=o, id_offset=lo, n_global=n_global, breakpoints=B)


def merge_shard_topk(ids, dists, k: int, group=None):
    """C2: all-gather the local top-k lists ([nq][k] ids int64 / dists f32) and merge them."""
    ids_t = ids if torch.is_tensor(ids) else torch.from_numpy(np.ascontiguousarray(ids))
    d_t = dists if torch.is_tensor(dists) else torch.from_numpy(np.ascontiguousarray(dists))
    world = dist.get_world_size(group)
    gi = [torch.empty_like(ids_t) for _ in range(world)]
    gd = [torch.empty_like(d_t) for _ in range(world)]
    dist.all_gather(gi, ids_t.contiguous(), group=group)
    dist.all_gather(gd, d_t.contiguous(), group=group)
    return D.detlsh_merge_topk(torch.stack(gi).cpu().numpy(), torch.stack(gd).cpu().numpy(), k)


def sharded_query(index, Q, k: int, c: float, r_min: float, beta: float, opts=None, group=None):
    ids, dists = index.query(Q, k, c, r_min, beta, opts=opts)
    return merge_shard_topk(ids, dists, k, group)
