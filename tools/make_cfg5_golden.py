"""Oracle expected values for configs[4] (n = 100M, d = 96, L = 6, beta = 0.05) -- ORACLE ONLY.

configs[4] is "oracle checked on a seeded 200-query subset" (BASELINE.json; seed
2005).  The oracle's index needs ~95 GB of host RAM, so this script runs on the GPU host (196 GB,
16 cores) and writes its results under gpurun_out/; they are then committed as
tests/golden/cfg5_oracle.npz and bench_configs.json["5"].  Only datagen (inputs) and oracle/
(the method) are called -- nothing from the CUDA path.

Steps (each the oracle as it stands; queries are embarrassingly parallel, so P forked processes
answer disjoint queries of the one index, BASELINE.md §3 "oracle x P cores"):
  1. datagen configs[4]: X [1e8][96], the 10,000 queries, 50 held-out r_min sample queries.
  2. orc_build (single thread, timed: oracle build points/s on 1 core).
  3. r*_q of the 50 sample queries (AMB-22) -> r_min = lower median (tools/make_rmin.py's rule).
  4. exact kNN (orc_exact_knn) of the sweep sample queries and of the 200-query subset.
  5. operating point (AMB-32): oracle recall@k on the first NSW sample queries at r_min c^-m,
     m = 1..3; r_bench = r_min c^-m* for the largest m* with recall >= 0.95 (else r_min).
  6. orc_query of the 200-query subset at r_min, and of its first NB queries at r_bench.
Usage (GPU host): python tools/make_cfg5_golden.py [--procs 16] [--out gpurun_out/cfg5]
"""
import argparse
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
from oracle import oracle as O  # noqa: E402

NS = 50          # r_min sample queries (as tools/make_rmin.py)
SUBSET_SEED = 2005
SUBSET = 200

_G = {}          # the index and inputs, inherited by the forked workers


def _rstar(i):
    c = _G["cfg"]
    _, rs = _G["ix"].estimate_rmin(_G["Qs"][i:i + 1], c.k, c.c, c.beta, return_all=True)
    return i, float(rs[0])


def _knn(job):
    which, i = job
    Qm = _G["Qs"] if which == "s" else _G["Q"]
    ids, d = O.exact_knn(_G["X"], Qm[i:i + 1], _G["cfg"].k)
    return job, ids[0], d[0]


def _query(job):
    which, i, r = job
    c = _G["cfg"]
    Qm = _G["Qs"] if which == "s" else _G["Q"]
    t = time.perf_counter()
    ids, d, st = _G["ix"].query(Qm[i:i + 1], c.k, c.c, r, c.beta)
    return job, ids[0], d[0], st[0], time.perf_counter() - t


def pool_map(fn, jobs, procs):
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as p:
        return list(p.imap_unordered(fn, jobs, chunksize=1))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "cfg5"))
    ap.add_argument("--n", type=int, default=None, help="smaller n (dry run of the script)")
    ap.add_argument("--nsw", type=int, default=24, help="sample queries in the operating-point sweep")
    ap.add_argument("--nb", type=int, default=64, help="subset queries also answered at r_bench")
    ap.add_argument("--subset", type=int, default=SUBSET)
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    log = {"procs": a.procs, "nproc": os.cpu_count()}

    def save(**arrays):
        json.dump(log, open(a.out + ".json", "w"), indent=1, default=float)
        if arrays:
            np.savez(a.out + ".npz", **arrays)

    t0 = time.time()
    D = datagen.generate(5, n=a.n, with_sample_queries=NS)
    c = D["cfg"]
    X, Q, Qs = D["X"], D["Q"], D["Qs"]
    sel = np.sort(np.random.default_rng(SUBSET_SEED).choice(len(Q), a.subset, replace=False))
    log.update(n=int(X.shape[0]), d=int(X.shape[1]), gen_s=time.time() - t0, subset_seed=SUBSET_SEED)
    print("generated", X.shape, f"{time.time() - t0:.0f}s", flush=True)
    save()

    t = time.perf_counter()
    ix = O.Index(X, c.L, c.K, c.N_r, c.index_seed, c.max_size, c.sample_frac)
    log["build_s"] = time.perf_counter() - t
    log["build_points_per_s_1core"] = X.shape[0] / log["build_s"]
    print("oracle build", f"{log['build_s']:.0f}s", flush=True)
    save()
    _G.update(ix=ix, X=X, Q=Q, Qs=Qs, cfg=c)

    t = time.time()
    rs = np.empty(NS)
    for i, r in pool_map(_rstar, range(NS), a.procs):
        rs[i] = r
    r_min = float(np.sort(rs)[(NS - 1) // 2])            # lower median (orc_estimate_rmin)
    log.update(r_min=r_min, rstar=rs.tolist(), rstar_s=time.time() - t)
    print("r_min", r_min, f"{time.time() - t:.0f}s", flush=True)
    save()

    t = time.time()
    gts_i = np.empty((a.nsw, c.k), np.int64)
    gt_i = np.empty((len(sel), c.k), np.int64)
    gt_d = np.empty((len(sel), c.k), np.float64)
    jobs = [("s", i) for i in range(a.nsw)] + [("q", int(i)) for i in sel]
    pos = {int(q): j for j, q in enumerate(sel)}
    for (which, i), ids, d in pool_map(_knn, jobs, a.procs):
        if which == "s":
            gts_i[i] = ids
        else:
            gt_i[pos[i]], gt_d[pos[i]] = ids, d
    log["knn_s"] = time.time() - t
    print("exact kNN", f"{time.time() - t:.0f}s", flush=True)
    save(sel=sel, gt_ids=gt_i, gt_dists=gt_d)

    t = time.time()
    ms = [1, 2, 3]
    radii = {m: r_min * c.c ** (-m) for m in ms}
    rec = {m: [] for m in ms}
    for (_, i, r), ids, _, _, _ in pool_map(_query, [("s", i, radii[m]) for m in ms for i in range(a.nsw)], a.procs):
        m = next(m for m in ms if radii[m] == r)
        rec[m].append(len(set(ids.tolist()) & set(gts_i[i].tolist())) / c.k)
    sweep = [{"m": m, "r": radii[m], "oracle_recall": float(np.mean(rec[m]))} for m in ms]
    ok = [p for p in sweep if p["oracle_recall"] >= 0.95]
    best = max(ok, key=lambda p: p["m"]) if ok else {"m": 0, "r": r_min, "oracle_recall": None}
    log.update(point_sweep=sweep, bench_m=best["m"], r_bench=best["r"], bench_oracle_recall=best["oracle_recall"],
               sweep_s=time.time() - t)
    print("sweep", sweep, f"{time.time() - t:.0f}s", flush=True)
    save(sel=sel, gt_ids=gt_i, gt_dists=gt_d)

    out = {}
    passes = [("rmin", r_min, sel)] + ([("rbench", best["r"], sel[:a.nb])] if best["m"] > 0 else [])
    for tag, r, qs in passes:
        t = time.time()
        ids = np.empty((len(qs), c.k), np.int64)
        dists = np.empty((len(qs), c.k), np.float32)
        st = np.zeros(len(qs), O.QSTATS_DTYPE)
        secs = np.empty(len(qs))
        p = {int(q): j for j, q in enumerate(qs)}
        for (_, i, _), ii, dd, ss, sec in pool_map(_query, [("q", int(i), r) for i in qs], a.procs):
            ids[p[i]], dists[p[i]], st[p[i]], secs[p[i]] = ii, dd, ss, sec
        wall = time.time() - t
        out.update({f"{tag}_ids": ids, f"{tag}_dists": dists, f"{tag}_stats": st, f"{tag}_secs": secs})
        log[f"{tag}_query"] = {"queries": len(qs), "wall_s": wall, "qps_1core": len(qs) / secs.sum(),
                               "qps_procs": len(qs) / wall, "mean_n_cand": float(st["n_cand"].mean()),
                               "stops": np.bincount(st["reason"], minlength=3).tolist()}
        print(tag, log[f"{tag}_query"], flush=True)
        save(sel=sel, gt_ids=gt_i, gt_dists=gt_d, r_min=r_min, r_bench=best["r"], bench_m=best["m"], **out)
    log["total_s"] = time.time() - t0
    save(sel=sel, gt_ids=gt_i, gt_dists=gt_d, r_min=r_min, r_bench=best["r"], bench_m=best["m"], **out)
    print("done", f"{log['total_s']:.0f}s", flush=True)


if __name__ == "__main__":
    main()
