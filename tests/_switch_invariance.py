"""Helper for test_filter_switches_do_not_change_results (run once per switch setting in a
subprocess: the library reads its DETLSH_* switches once per process).  Builds a mid-size index
and queries it at a small and a large radius; writes ids and distances to the .npz given."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2603_24920_b200 as P  # noqa: E402

D = datagen.generate(2, n=60000, nq=300)
c = D["cfg"]
g = P.detlsh_build(D["X"], c.L, c.K, c.N_r, c.index_seed)
out = {}
for tag, r in (("small", 0.45), ("large", 0.9)):
    ids, d = g.query(D["Q"], c.k, c.c, r, c.beta)
    out[tag + "_ids"], out[tag + "_d"] = ids, d
    # the same queries in batches of 37 (S bitmaps reused across batches: cleared by streaming
    # zeros or by their dirty words, DETLSH_DIRTY_CLEAR).  Verification by the sparse gather in
    # both (direct fp32 sums): the auto cost model may pick the tensor-core form for a batch of 37
    # and the gather for the whole set, and the two may order a near-tie at the k-th place
    # differently (AMB-31) -- that is not what is checked here.
    i1, d1, s1 = g.query(D["Q"], c.k, c.c, r, c.beta, opts=P.default_opts(verify_impl=3), stats=True)
    ids, d, st = g.query(D["Q"], c.k, c.c, r, c.beta, opts=P.default_opts(query_batch=37, verify_impl=3), stats=True)
    out[tag + "_b_ids"], out[tag + "_b_d"], out[tag + "_b_n"] = ids, d, st["n_cand"]
    assert np.array_equal(ids, i1) and np.array_equal(d, d1) and np.array_equal(st["n_cand"], s1["n_cand"]), tag
np.savez(sys.argv[1], **out)
print("OK")
