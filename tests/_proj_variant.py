"""Helper for test_projection_variants (one subprocess per DETLSH_PROJ_TA setting: the library
reads its switches once per process).  Projections (fused encode and plain), row norms and a
query batch over three shapes; writes them to the .npz given."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2603_24920_b200 as P  # noqa: E402

out = {}
for tag, (cid, n, d, L) in {"c1": (2, 20000, 256, 4), "c5": (5, 20000, 96, 6), "c2": (3, 6000, 960, 4),
                            "ragged": (1, 3001, 37, 3)}.items():
    D = datagen.generate(cid, n=n, nq=50)
    X = np.ascontiguousarray(D["X"][:, :d])
    Q = np.ascontiguousarray(D["Q"][:, :d])
    g = P.detlsh_build(X, L, 16, 256, 11)
    out[tag + "_P"] = g.project(X[:4000])
    out[tag + "_codes"] = g.codes()
    out[tag + "_A"] = g.A()
    out[tag + "_B"] = g.breakpoints()
    ids, dd = g.query(Q, 10, 1.5, 1e9, 2.0, opts=P.default_opts(verify_impl=2))   # exact kNN through the TC path
    out[tag + "_ids"], out[tag + "_d"] = ids, dd
np.savez(sys.argv[1], **out)
print("OK")
