"""C-ABI checks that need no GPU: the library builds, loads, exports every symbol the header
declares, and its host-side logic (Eq. 2 parameters, sample size, C2 merge, argument
validation) is right."""
import math
import os
import re

import numpy as np
import pytest

import paper_2603_24920_b200 as P
from paper_2603_24920_b200 import detlsh as D

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "detlsh.h")).read()
    declared = set(re.findall(r"\b(detlsh_[a-z_0-9]+)\s*\(", hdr))
    assert {"detlsh_build", "detlsh_query", "detlsh_free", "detlsh_last_error"} <= declared
    lib = P.lib()
    for name in sorted(declared):
        assert hasattr(lib, name), name


def test_params_match_eq2():
    """Lemma 3 / Eq. 2, library's own closed-form chi2, vs scipy."""
    import scipy.stats
    for K in (2, 3, 7, 16, 32):
        for L in (1, 4, 6):
            p = P.detlsh_params(K, L, 1.5)
            e2 = scipy.stats.chi2.isf(math.exp(-1 / L), K)
            assert abs(p["eps"] ** 2 - e2) < 1e-7 * e2
            a2 = scipy.stats.chi2.sf(e2 / 2.25, K)
            assert abs(p["alpha2"] - a2) < 1e-9
            assert abs(p["beta_theory"] - (2 - 2 * a2 ** L)) < 1e-8


def test_sample_size_rule():
    assert [P.detlsh_sample_size(n, 256, 0.01) for n in (10_000, 1_000_000, 10_000_000, 100_000_000, 300)] == \
        [8192, 10_000, 100_000, 1_000_000, 300]


@pytest.mark.gpu
def test_merge_topk_device():
    """C2 merge (k_merge_topk) vs a plain sort of the pooled (dist, id) pairs."""
    rng = np.random.default_rng(0)
    G, nq, k = 4, 6, 5
    d = rng.integers(0, 9, (G, nq, k)).astype(np.float32)
    ids = rng.permutation(G * nq * k).reshape(G, nq, k).astype(np.int64)
    o = np.lexsort((ids, d), axis=-1)          # each list sorted by (dist, id), as detlsh_query writes it
    d, ids = np.take_along_axis(d, o, -1), np.take_along_axis(ids, o, -1)
    ids[0, 0, 4] = -1
    d[0, 0, 4] = np.inf
    oi, od = P.detlsh_merge_topk(ids, d, k)
    for q in range(nq):
        pairs = sorted((float(d[g, q, e]), int(ids[g, q, e])) for g in range(G) for e in range(k) if ids[g, q, e] >= 0)[:k]
        assert oi[q].tolist() == [p[1] for p in pairs]
        assert od[q].tolist() == [p[0] for p in pairs]


@pytest.mark.parametrize("kw,msg", [
    (dict(n=0), "n must be"), (dict(K=33), "K must be"), (dict(N_r=3), "N_r must be"),
    (dict(N_r=512), "N_r must be"), (dict(L=0), "L must be"), (dict(d=0), "d must be")])
def test_build_argument_errors(kw, msg):
    args = dict(n=10, d=8, L=4, K=16, N_r=256)
    args.update(kw)
    data = np.zeros((max(args["n"], 1), max(args["d"], 1)), np.float32)
    import ctypes as C
    h = C.c_void_p()
    st = P.lib().detlsh_build(data.ctypes.data_as(C.c_void_p), args["n"], args["d"], args["L"], args["K"],
                              args["N_r"], 42, C.byref(h))
    assert st == D.DETLSH_EINVAL
    assert msg in P.lib().detlsh_last_error().decode()


def test_no_gpu_is_a_loud_error():
    """Without a device the product fails (ECUDA) -- there is no CPU fallback."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(P.DetlshError) as e:
        P.detlsh_build(np.zeros((100, 8), np.float32), 4, 16, 256, 42)
    assert e.value.status == D.DETLSH_ECUDA
