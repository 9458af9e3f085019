"""f3: the paper's parameter studies on synthetic configs[1], measured on the GPU.

  E9  recall vs queries/s as the budget beta and the initial radius r_min c^-m vary
  E11 effect of k
  E6  L and K study; r_min per (L, K) from the GPU estimator (AMB-22)

Every point: device-timed query of the 1000 queries (CUDA events, after a warm-up call),
recall@k against exact kNN on 200 sampled queries.  Output: profiles/r01_sweeps.json and a
markdown table on stdout.  Not a bench line (bench.py is the contract)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2603_24920_b200 as P  # noqa: E402
from bench import exact_knn_sample, recall  # noqa: E402


def timed_query(g, Qd, k, c, r, beta, opts):
    g.query(Qd, k, c, r, beta, opts=opts)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    ids, _, st = g.query(Qd, k, c, r, beta, opts=opts, stats=True)
    b.record()
    b.synchronize()
    return ids.cpu().numpy(), a.elapsed_time(b), st


def main():
    D = datagen.generate(2, with_sample_queries=50)
    cfg = D["cfg"]
    X, Q = D["X"], D["Q"]
    Xd, Qd = torch.from_numpy(X).cuda(), torch.from_numpy(Q).cuda()
    sel = np.random.default_rng(2).choice(cfg.nq, 200, replace=False)
    gt = {k: exact_knn_sample(X, Q, k, sel) for k in (1, 10, 50, 100)}
    rmin0 = json.load(open(os.path.join(ROOT, "bench_configs.json")))["2"]["r_min"]
    opts = P.default_opts(borrow_data=1)
    out = {"config": "configs[1] deep1m_like (1M x 256, 1000 queries)", "points": []}

    def point(study, g, k, r, beta, **extra):
        ids, ms, st = timed_query(g, Qd, k, cfg.c, r, beta, opts)
        rec = recall(ids[sel], gt[k])
        e = {"study": study, "k": k, "r_min": r, "beta": beta, "recall": round(rec, 4),
             "queries_per_s": round(cfg.nq / (ms / 1e3)), "ms": round(ms, 3),
             "candidates_per_query": float(st["n_cand"].mean()), "rounds_mean": float(st["rounds"].mean()), **extra}
        out["points"].append(e)
        print(json.dumps(e), flush=True)

    g = P.detlsh_build(Xd, cfg.L, cfg.K, cfg.N_r, cfg.index_seed, opts=opts)
    for m in range(0, 7):                                    # E9: r_min c^-m
        point("E9_rmin", g, cfg.k, rmin0 * cfg.c ** (-m), cfg.beta, m=m)
    for beta in (0.01, 0.02, 0.05, 0.1, 0.2):                # E9: budget
        point("E9_beta", g, cfg.k, rmin0, beta)
    for k in (1, 10, 50, 100):                               # E11
        point("E11_k", g, k, rmin0, cfg.beta)
    g.free()
    for L, K in [(2, 16), (3, 16), (4, 16), (5, 16), (6, 16), (4, 8), (4, 12), (4, 20), (4, 24)]:   # E6
        t0 = time.perf_counter()
        g = P.detlsh_build(Xd, L, K, cfg.N_r, cfg.index_seed, opts=opts)
        torch.cuda.synchronize()
        tb = time.perf_counter() - t0
        r = g.estimate_rmin(D["Qs"], cfg.k, cfg.beta)
        point("E6_LK", g, cfg.k, r, cfg.beta, L=L, K=K, build_s=round(tb, 4))
        g.free()
    # on a gpurun box only gpurun_out/ comes back: pass a path there and copy it to profiles/
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r01_sweeps.json")
    json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
