"""Helper for test_sample_selection_paths (subprocess, so DETLSH_SEL16_CAP -- read once per
process -- can force the 8-pass fallback): the GPU's sample ids (B1, AMB-3/4) equal the oracle's
for several n / sample fractions / seeds.  Prints OK on success."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_24920_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402

rng = np.random.default_rng(3)
for n, frac, seed in [(300_000, 0.01, 7), (70_001, 0.2, 11), (5000, 0.5, 3), (200_000, 0.001, 99)]:
    X = rng.standard_normal((n, 4)).astype(np.float32)
    g = P.detlsh_build(X, 1, 4, 16, seed, opts=P.default_opts(sample_frac=frac))
    want = O.sample_ids(seed, n, P.detlsh_sample_size(n, 16, frac))
    got = np.sort(g.sample())
    assert np.array_equal(got, np.sort(want)), (n, frac, seed)
    g.free()
print("OK")
