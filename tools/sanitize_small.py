"""Small build + query workload for compute-sanitizer (one tool per run): every kernel family of
the library -- tcgen05 projection (PROJ_IMPL=0, default) or SIMT (1), sample selection, radix
sorts, tree build (global levels and the shared-memory finish), range filter (SIMD chunks and the
pair kernel), all four verification paths, top-k, LB-ordered truncation, EXACT, (r,c)-ANN,
the r_min estimator and the device C2 merge."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import datagen  # noqa: E402
import paper_2603_24920_b200 as P  # noqa: E402

impl = int(os.environ.get("PROJ_IMPL", "0"))
for (n, d, L, K, Nr, ms) in [(3000, 128, 4, 16, 256, 128), (1500, 37, 2, 8, 16, 5), (777, 100, 3, 12, 64, 9)]:
    D = datagen.generate(1, n=n, nq=9, with_sample_queries=4)
    X = np.ascontiguousarray(D["X"][:, :d])
    Q = np.ascontiguousarray(D["Q"][:, :d])
    g = P.detlsh_build(X, L, K, Nr, 3, opts=P.default_opts(max_size=ms, sample_frac=0.1, proj_impl=impl,
                                                           keep_projections=1))
    r = 50.0
    for mode in (0, 1, 2):
        for vi in (0, 1, 2, 3):
            ids, dist, st = g.query(Q, 5, 1.5, r, 0.1, opts=P.default_opts(mode=mode, proj_impl=impl, query_batch=4,
                                                                           verify_impl=vi), stats=True)
    g.query(Q, 5, 1.5, r, 0.05, opts=P.default_opts(lb_order=1, proj_impl=impl))
    g.rc_ann(Q, r, 1.5, 0.1, opts=P.default_opts(proj_impl=impl))
    try:
        g.estimate_rmin(np.ascontiguousarray(D["Qs"][:, :d]), 5, 0.1, opts=P.default_opts(proj_impl=impl))
    except P.DetlshError as e:       # a zero median (few regions) is refused after the kernels ran
        print("estimate_rmin:", e)
    print(n, d, L, K, Nr, "ok", st["reason"].tolist(), flush=True)
# the 16-query SIMD filter and the pair kernel at K = 16 with a larger group count
D = datagen.generate(1, n=20000, nq=40)
g = P.detlsh_build(D["X"], 4, 16, 256, 42, opts=P.default_opts(proj_impl=impl))
for r in (30.0, 120.0):
    g.query(D["Q"], 10, 1.5, r, 0.1, opts=P.default_opts(proj_impl=impl))
ids, dists = g.query(D["Q"], 10, 1.5, 120.0, 0.1)
P.detlsh_merge_topk(np.stack([ids, ids]), np.stack([dists, dists]), 10)
print("ok")
