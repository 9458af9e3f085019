"""Small build+query workload for compute-sanitizer (one tool per run)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import datagen, paper_2603_24920_b200 as P
impl = int(os.environ.get("PROJ_IMPL", "1"))
for (n, d, L, K, Nr, ms) in [(3000, 128, 4, 16, 256, 128), (1500, 37, 2, 8, 16, 5), (777, 100, 3, 12, 64, 9)]:
    D = datagen.generate(1, n=n, nq=9)
    X = np.ascontiguousarray(D["X"][:, :d]); Q = np.ascontiguousarray(D["Q"][:, :d])
    g = P.detlsh_build(X, L, K, Nr, 3, opts=P.default_opts(max_size=ms, sample_frac=0.1, proj_impl=impl))
    for mode in (0, 1):
        ids, dist, st = g.query(Q, 5, 1.5, 50.0, 0.1, opts=P.default_opts(mode=mode, proj_impl=impl, query_batch=4), stats=True)
    print(n, d, L, K, Nr, "ok", st["reason"].tolist())
