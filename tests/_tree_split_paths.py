"""Helper for test_trees_split_paths (run in a subprocess so DETLSH_LOCAL_MAX, read once per
process by the library, can differ): builds trees from skewed codes on the GPU and compares
them with the oracle's Alg. 2 trees, bit for bit.  Prints OK on success."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_24920_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402

rng = np.random.default_rng(5)
n, L, K, N_r = 30000, 2, 8, 64
codes = rng.integers(0, N_r, (n, L * K)).astype(np.uint8)
# 60 % of the points share one first-layer cell (all MSBs clear) and a narrow range in the
# low bits, so one node holds ~18K points and needs several global levels before it is small
# enough to finish in shared memory; the rest spread over many small cells.
hot = rng.random(n) < 0.6
codes[hot] = rng.integers(0, 12, (int(hot.sum()), L * K)).astype(np.uint8)
# K = 16, N_r = 256 as well: the fused leaf layout (gather + Morton order + boxes) serves it when
# the Morton order is on (DETLSH_LEAF_MORTON); its exported perm must still be canonical
codes16 = rng.integers(0, 256, (n, 2 * 16)).astype(np.uint8)
codes16[hot] = rng.integers(0, 40, (int(hot.sum()), 2 * 16)).astype(np.uint8)
for cds, L_, K_, N_r_ in ((codes, L, K, N_r), (codes16, 2, 16, 256)):
    for ms in (128, 20):
        g = P.detlsh_build_from_codes(cds, L_, K_, N_r_, max_size=ms)
        for i in range(L_):
            o = O.Tree(cds[:, i * K_:(i + 1) * K_], K_, N_r_, ms, builder=1).export()
            t = g.tree(i)
            for key in ("leaf_off", "perm", "lo", "hi", "bits"):
                assert np.array_equal(t[key], o[key]), (K_, ms, i, key)
        g.free()
print("OK")
