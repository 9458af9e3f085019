"""Pins of the oracle against things other than itself (CPU only, -m "not gpu").

Each test names the paper passage it checks and what it is pinned to: a worked
example of the paper (tests/golden/*.json), a closed form, a library routine,
a mathematical invariant, or brute force on a tiny input.
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.stats

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ----------------------------------------------------------------- O1 chi2 / Eq. 2
def test_chi2_closed_form_k2():
    """chi2(2) survival is e^{-y/2}, so chi2_alpha(2) = -2 ln alpha (Lemma 2)."""
    for a, y in gold("chi2_params.json")["k2_cases"]:
        assert abs(O.chi2_isf(a, 2) - y) < 1e-9
        assert abs(O.chi2_isf(a, 2) + 2 * math.log(a)) < 1e-9


def test_chi2_closed_form_k4():
    """chi2(4) survival is e^{-y/2}(1+y/2); solved here by an independent bisection."""
    for a in (0.05, 0.25, 0.5, 0.9):
        lo, hi = 0.0, 200.0
        for _ in range(200):
            mid = 0.5 * (lo + hi)
            if math.exp(-mid / 2) * (1 + mid / 2) > a:
                lo = mid
            else:
                hi = mid
        assert abs(O.chi2_isf(a, 4) - lo) < 1e-9


def test_chi2_vs_scipy():
    for K in (1, 3, 8, 16, 32):
        for a in (1e-6, 0.01, 0.3, 0.778801, 0.995, 0.999999):
            assert abs(O.chi2_isf(a, K) - scipy.stats.chi2.isf(a, K)) < 1e-8 * max(1, scipy.stats.chi2.isf(a, K))
            y = scipy.stats.chi2.isf(a, K)
            assert abs(O.chi2_sf(y, K) - a) < 1e-10


def test_params_eq2_vs_scipy():
    """Lemma 3 / Eq. 2: alpha1 = e^{-1/L}, eps^2 = chi2_{alpha1}(K) = c^2 chi2_{alpha2}(K)."""
    for L in (1, 2, 3, 4, 5, 6, 8):
        p = O.params(16, L, 1.5)
        a1 = math.exp(-1.0 / L)
        e2 = scipy.stats.chi2.isf(a1, 16)
        a2 = scipy.stats.chi2.sf(e2 / 1.5 ** 2, 16)
        assert abs(p["alpha1"] - a1) < 1e-15
        assert abs(p["eps"] ** 2 - e2) < 1e-8
        assert abs(p["alpha2"] - a2) < 1e-10
        assert abs(p["beta_theory"] - (2 - 2 * a2 ** L)) < 1e-9
        # Eq. 2 closure: c^2 chi2_{alpha2}(K) == eps^2
        assert abs(1.5 ** 2 * O.chi2_isf(p["alpha2"], 16) - p["eps"] ** 2) < 1e-6


def test_beta_decreasing_in_L():
    """Fig. betal: theoretical beta falls with L (K=16, c=1.5)."""
    b = [O.params(16, L, 1.5)["beta_theory"] for L in range(1, 9)]
    assert all(x > y for x, y in zip(b, b[1:]))
    assert 0.037 < b[3] < 0.039          # L = 4 default


# ----------------------------------------------------------------- O2 hash family
def test_splitmix64_reference_vector():
    seq = gold("chi2_params.json")["splitmix64_seed0_sequence"]
    g = 0x9E3779B97F4A7C15
    for m, h in enumerate(seq):
        assert O.splitmix64((m * g) % 2 ** 64) == int(h, 16)


def test_hash_family_moments_and_determinism():
    """Eq. 1: entries i.i.d. N(0,1). 10^6 entries: mean 0+-0.01, var 1+-0.01."""
    A = O.hash_family(7, 15625, 4, 16)
    assert A.size == 1_000_000
    assert abs(A.mean()) < 0.01
    assert abs(A.var() - 1) < 0.01
    assert abs(scipy.stats.kurtosis(A.ravel())) < 0.05                 # Gaussian tails
    assert np.array_equal(A, O.hash_family(7, 15625, 4, 16))           # regeneration
    assert not np.array_equal(A[:100], O.hash_family(8, 15625, 4, 16)[:100])
    assert np.all((A.view(np.uint32) & 0x1FFF) == 0)                   # TF32-exact (AMB-1)


def test_lemma1_lemma2_statistics():
    """Lemma 1: s'^2/s^2 ~ chi2(K); Lemma 2: Pr[s' > s sqrt(chi2_a(K))] = a."""
    K, G, d = 16, 100_000, 8
    A = O.hash_family(99, d, G, K)                                     # G independent H_i
    rng = np.random.default_rng(0)
    o = rng.normal(size=(2, d)).astype(np.float32)
    P = O.project(A, o).astype(np.float64)                             # [2][G*K]
    s2 = float(((o[0].astype(np.float64) - o[1]) ** 2).sum())
    sp2 = ((P[0] - P[1]).reshape(G, K) ** 2).sum(1)
    ratio = sp2 / s2
    assert 15.8 <= ratio.mean() <= 16.2
    for a in (0.1, 0.5, 0.9):
        frac = np.mean(np.sqrt(ratio) > math.sqrt(O.chi2_isf(a, K)))
        assert abs(frac - a) < 0.01


def test_projection_vs_numpy_and_linearity():
    """P:296 h_ij(o) = a_ij . o; pinned to numpy fp64 matmul (fp32 result within 1 ulp)."""
    rng = np.random.default_rng(1)
    A = O.hash_family(3, 37, 2, 5)
    X = rng.normal(size=(200, 37)).astype(np.float32) * 10
    P = O.project(A, X)
    ref = (X.astype(np.float64) @ A.T.astype(np.float64)).astype(np.float32)
    ulp = np.spacing(np.abs(ref))
    assert np.all(np.abs(P - ref) <= ulp)
    # linearity: exact double sums on small integers, so only the fp32 roundings differ
    Xi = rng.integers(-50, 50, size=(2, 37)).astype(np.float32)
    Pi = O.project(A, np.vstack([Xi, Xi[:1] + Xi[1:]])).astype(np.float64)
    assert np.all(np.abs(Pi[2] - (Pi[0] + Pi[1])) <= 2 * np.spacing(np.abs(Pi[2]).astype(np.float32)))
    assert np.all(O.project(A, np.zeros((1, 37), np.float32)) == 0)


# ----------------------------------------------------------------- O3 sample / breakpoints
def test_sample_size_rule():
    """AMB-3: n_s = min(n, max(ceil(f n), 32 N_r)) -- the configs' sizes."""
    assert [O.sample_size(n, 256, f) for n, f in [(10_000, 0.01), (1_000_000, 0.01),
            (10_000_000, 0.01), (100_000_000, 0.01), (5000, 0.01)]] == [8192, 10_000, 100_000, 1_000_000, 5000]


def test_sample_ids_are_smallest_keys():
    """AMB-4: the n_s ids with the smallest keyed hash; brute force with numpy sort."""
    n, ns, seed = 3000, 250, 42
    ids = O.sample_ids(seed, n, ns)
    s = seed ^ 0x53414D504C45
    keys = np.array([O.splitmix64(s ^ O.splitmix64(i)) for i in range(n)], dtype=np.uint64)
    ref = np.sort(np.lexsort((np.arange(n), keys))[:ns])
    assert np.array_equal(ids, ref)
    # roughly uniform over [0, n)
    h = np.bincount(ids * 10 // n, minlength=10)
    assert scipy.stats.chisquare(h).pvalue > 1e-4


def test_breakpoints_worked_example():
    g = gold("breakpoints_example.json")
    assert O.breakpoints_sort(g["values"], g["N_r"]).tolist() == g["breakpoints"]
    assert O.breakpoints_qselect(g["values"], g["N_r"]).tolist() == g["breakpoints"]


def test_breakpoints_degenerate_and_qselect_equivalence():
    """QuickSelect divide-and-conquer gives the same order statistics as a full sort."""
    assert np.all(O.breakpoints_sort([3.5] * 50, 256) == 3.5)
    rng = np.random.default_rng(2)
    for it in range(300):
        m = int(rng.integers(1, 3000))
        N_r = int(2 ** rng.integers(1, 9))
        v = rng.normal(size=m).astype(np.float32) if it % 3 else rng.integers(0, 5, m).astype(np.float32)
        a = O.breakpoints_sort(v, N_r)
        b = O.breakpoints_qselect(v, N_r)
        assert np.array_equal(a, b)
        assert a[0] == v.min() and a[-1] == v.max() and np.all(np.diff(a) >= 0)


def test_breakpoints_equal_regions():
    """regions hold equal numbers of (sample) points: m divisible by N_r, distinct values."""
    rng = np.random.default_rng(3)
    v = rng.permutation(4096).astype(np.float32) * 0.37
    b = O.breakpoints_sort(v, 256)
    codes = np.searchsorted(b[1:256], v, side="left")
    assert np.all(np.bincount(codes, minlength=256) == 16)


# ----------------------------------------------------------------- O4 encode
def test_encode_examples_and_searchsorted():
    g = gold("encode_example.json")
    for x, s in g["cases"]:
        assert O.encode_value(x, g["breakpoints"], g["N_r"]) == s
    rng = np.random.default_rng(4)
    b = np.sort(rng.normal(size=257).astype(np.float32))
    xs = np.concatenate([rng.normal(size=2000) * 2, b]).astype(np.float32)
    codes = np.array([O.encode_value(x, b, 256) for x in xs])
    assert np.array_equal(codes, np.searchsorted(b[1:256], xs, side="left"))
    order = np.argsort(xs, kind="stable")
    assert np.all(np.diff(codes[order]) >= 0)                         # monotone


# ----------------------------------------------------------------- O5 trees
def test_split_worked_example():
    g = gold("split_example.json")
    for builder in (0, 1):
        t = O.Tree(np.array(g["codes"], np.uint8), g["K"], g["N_r"], g["max_size"], builder).export()
        assert len(t["leaf_off"]) - 1 == len(g["leaves"])
        for i, lf in enumerate(g["leaves"]):
            assert t["perm"][t["leaf_off"][i]:t["leaf_off"][i + 1]].tolist() == lf["members"]
            assert t["lo"][i].tolist() == lf["lo"] and t["hi"][i].tolist() == lf["hi"]
            assert t["bits"][i].tolist() == lf["bits"]


def _py_literal_alg2(codes, K, nb, max_size):
    """Brute-force Alg. 2 in Python for tiny inputs, written independently:
    nodes are dicts; a leaf splits while it holds >= max_size entries."""
    def bit(s, b):
        return (s >> (nb - 1 - b)) & 1

    first = {}
    for z, cd in enumerate(codes):
        key = tuple(bit(int(c), 0) for c in cd)
        node = first.setdefault(key, {"bits": [1] * K, "pre": list(key), "ids": [], "kids": None})
        while True:
            while node["kids"] is not None:
                j = node["dim"]
                node = node["kids"][bit(int(cd[j]), node["bits"][j])]
            if len(node["ids"]) >= max_size:
                best = None
                for j in range(K):
                    if node["bits"][j] >= nb:
                        continue
                    ones = sum(bit(int(codes[e][j]), node["bits"][j]) for e in node["ids"])
                    imb = abs(len(node["ids"]) - 2 * ones)
                    if best is None or imb < best[0]:
                        best = (imb, j)
                if best is not None:
                    j = best[1]
                    kids = []
                    for b in (0, 1):
                        bits = list(node["bits"]); pre = list(node["pre"])
                        bits[j] += 1; pre[j] = pre[j] * 2 + b
                        kids.append({"bits": bits, "pre": pre, "ids": [], "kids": None})
                    for e in node["ids"]:
                        kids[bit(int(codes[e][j]), node["bits"][j])]["ids"].append(e)
                    node["kids"], node["dim"], node["ids"] = kids, j, []
                    continue
            break
        node["ids"].append(z)
    leaves = []

    def walk(nd):
        if nd["kids"] is None:
            if nd["ids"]:
                lo = [p << (nb - b) for p, b in zip(nd["pre"], nd["bits"])]
                leaves.append((nd["ids"], lo, nd["bits"]))
            return
        walk(nd["kids"][0]); walk(nd["kids"][1])
    for key in sorted(first):
        walk(first[key])
    return leaves


@pytest.mark.parametrize("alphabet,max_size,n", [(256, 4, 300), (4, 3, 200), (2, 5, 150), (16, 1, 120)])
def test_tree_vs_python_bruteforce(alphabet, max_size, n):
    rng = np.random.default_rng(alphabet + max_size)
    K, N_r = 4, 256
    nb = 8
    codes = rng.integers(0, alphabet, size=(n, K)).astype(np.uint8)
    if alphabet < 256:   # duplicate-heavy, exhausting code space, one-sided splits
        codes = (codes * (256 // alphabet)).astype(np.uint8)
    ref = _py_literal_alg2(codes, K, nb, max_size)
    for builder in (0, 1):
        t = O.Tree(codes, K, N_r, max_size, builder).export()
        assert len(t["leaf_off"]) - 1 == len(ref)
        for i, (ids, lo, bits) in enumerate(ref):
            assert t["perm"][t["leaf_off"][i]:t["leaf_off"][i + 1]].tolist() == ids
            assert t["lo"][i].tolist() == lo and t["bits"][i].tolist() == bits


def test_tree_invariants(tiny_oracle):
    """Alg. 2 invariants: every point in exactly one leaf; codes inside the box; size <= max_size
    unless the code space is exhausted; literal Alg. 2 == bulk rule (B6)."""
    ix = tiny_oracle
    codes = ix.codes()
    for i in range(ix.L):
        t = ix.tree(i)
        assert np.array_equal(np.sort(t["perm"]), np.arange(ix.n))
        sizes = np.diff(t["leaf_off"])
        assert sizes.min() >= 1
        leaf_of = np.repeat(np.arange(len(sizes)), sizes)
        c = codes[t["perm"], i * ix.K:(i + 1) * ix.K]
        assert np.all(c >= t["lo"][leaf_of]) and np.all(c <= t["hi"][leaf_of])
        over = sizes > 128
        assert np.all(t["bits"][over] == 8)
        for s, e in zip(t["leaf_off"][:-1], t["leaf_off"][1:]):
            assert np.all(np.diff(t["perm"][s:e]) > 0)
        lit = O.Tree(codes[:, i * ix.K:(i + 1) * ix.K], ix.K, 256, 128, 0).export()
        for key in ("leaf_off", "perm", "lo", "hi", "bits"):
            assert np.array_equal(lit[key], t[key])


def test_tree_edge_cases():
    rng = np.random.default_rng(5)
    one = O.Tree(rng.integers(0, 256, (1, 16)).astype(np.uint8), 16, 256, 128).export()
    assert one["leaf_off"].tolist() == [0, 1]
    codes = rng.integers(0, 256, (500, 16)).astype(np.uint8)
    t = O.Tree(codes, 16, 256, 500).export()          # max_size >= n: first layer only
    assert np.all(t["bits"] == 1)
    keys = (codes >> 7).astype(np.int64) @ (1 << np.arange(15, -1, -1))
    assert len(t["leaf_off"]) - 1 == len(np.unique(keys))


# ----------------------------------------------------------------- O6 bounds
def test_bounds_worked_example():
    g = gold("bounds_example.json")
    b = np.array([g["breakpoints_dim0"], g["breakpoints_dim1"]], np.float32)
    lb2, ub2 = O.box_bounds2(g["box_lo"], g["box_hi"], g["query"], b, g["N_r"])
    assert abs(math.sqrt(lb2) - g["lb"]) < 1e-12 and abs(math.sqrt(ub2) - g["ub"]) < 1e-12
    lb2, ub2 = O.box_bounds2(g["box_lo"], g["box_hi"], [1.5, 5.5], b, g["N_r"])
    assert lb2 == 0.0                                   # query inside the box
    lb2, ub2 = O.box_bounds2([0, 2], [3, 2], [-100, 5.5], b, g["N_r"])
    assert lb2 == 0.0 and ub2 == math.inf               # outer regions unbounded (AMB-7)


def test_bounds_sandwich(tiny_oracle, tiny):
    """leafLB <= cellLB <= ||q'-p'|| for every point, incl. values outside [b_0, b_Nr] (AMB-7)."""
    ix = tiny_oracle
    B = ix.breakpoints().astype(np.float64)
    P = ix.P().astype(np.float64)
    codes = ix.codes()
    Nr = ix.N_r
    for qi in range(10):
        qp = ix.project_query(tiny["Q"][qi]).astype(np.float64)
        for i in range(ix.L):
            sl = slice(i * ix.K, (i + 1) * ix.K)
            Bi, c, x = B[sl], codes[:, sl].astype(np.int64), qp[sl]
            rows = np.arange(ix.K)
            l = np.where(c >= 1, Bi[rows, c], -np.inf)
            u = np.where(c <= Nr - 2, Bi[rows, np.minimum(c + 1, Nr)], np.inf)
            cell2 = (np.maximum(0, np.maximum(l - x, x - u)) ** 2).sum(1)
            true2 = ((P[:, sl] - x) ** 2).sum(1)
            assert np.all(cell2 <= true2 * (1 + 1e-12) + 1e-12)
            t = ix.tree(i)
            for L_ in range(0, len(t["leaf_off"]) - 1, 37):
                lb2, ub2 = O.box_bounds2(t["lo"][L_], t["hi"][L_], qp[sl].astype(np.float32), ix.breakpoints()[sl], Nr)
                mem = t["perm"][t["leaf_off"][L_]:t["leaf_off"][L_ + 1]]
                assert np.all(lb2 <= cell2[mem] + 1e-9)
                assert np.all(true2[mem] <= ub2 * (1 + 1e-12) + 1e-9)


def test_lut_clamp_equals_interval(tiny_oracle, tiny):
    """The GPU's LUT trick (SURVEY §8(c) derived check): D[clamp(s_x, lo, hi)] equals the
    interval-formula LB_j^2 because D is unimodal with D[s_x] = 0."""
    ix = tiny_oracle
    B = ix.breakpoints()
    rng = np.random.default_rng(6)
    Nr = ix.N_r
    for _ in range(200):
        r = int(rng.integers(0, ix.L * ix.K))
        x = np.float32(ix.project_query(tiny["Q"][int(rng.integers(0, 100))])[r] * rng.uniform(0.5, 1.5))
        b = B[r].astype(np.float64)
        s = np.arange(Nr)
        l = np.where(s >= 1, b[s], -np.inf)
        u = np.where(s <= Nr - 2, b[np.minimum(s + 1, Nr)], np.inf)
        D = np.maximum(0, np.maximum(l - x, x - u)) ** 2
        sx = O.encode_value(x, B[r], Nr)
        assert D[sx] == 0 and np.all(np.diff(D[:sx + 1]) <= 0) and np.all(np.diff(D[sx:]) >= 0)
        lo, hi = sorted(rng.integers(0, Nr, 2))
        lb2, _ = O.box_bounds2([lo], [hi], [x], B[r:r + 1], Nr)
        assert abs(D[min(max(sx, lo), hi)] - lb2) <= 1e-12 * max(1, lb2)


# ----------------------------------------------------------------- O7 range query
def test_range_query_equals_scan(tiny_oracle, tiny):
    """Alg. 3 traversal (prune LB > r', whole leaf if UB <= r', else per point) equals a
    brute-force scan of the per-point predicate (AMB-12) -- S:300."""
    ix = tiny_oracle
    B = ix.breakpoints().astype(np.float64)
    P = ix.P().astype(np.float64)
    codes = ix.codes().astype(np.int64)
    rng = np.random.default_rng(7)
    Nr = ix.N_r
    for it in range(60):
        qp = ix.project_query(tiny["Q"][it % 100])
        i = it % ix.L
        sl = slice(i * ix.K, (i + 1) * ix.K)
        x = qp[sl].astype(np.float64)
        c = codes[:, sl]
        rows = np.arange(ix.K)
        l = np.where(c >= 1, B[sl][rows, c], -np.inf)
        u = np.where(c <= Nr - 2, B[sl][rows, np.minimum(c + 1, Nr)], np.inf)
        cell2 = (np.maximum(0, np.maximum(l - x, x - u)) ** 2).sum(1)
        true2 = ((P[:, sl] - x) ** 2).sum(1)
        rho = float(np.sqrt(np.quantile(cell2, rng.uniform(0.001, 0.5))))
        got = ix.range_query(i, qp[sl], rho, O.CELL)
        assert np.array_equal(got, np.nonzero(cell2 <= rho * rho)[0])
        got_e = ix.range_query(i, qp[sl], rho, O.EXACT)
        assert np.array_equal(got_e, np.nonzero(true2 <= rho * rho)[0])
        got_r = ix.range_query(i, qp[sl], rho, O.RELAXED)
        assert set(got.tolist()) <= set(got_r.tolist())
        bigger = ix.range_query(i, qp[sl], rho * 1.3, O.CELL)
        assert set(got.tolist()) <= set(bigger.tolist())                # radius-monotone


# ----------------------------------------------------------------- O8 driver
def _np_knn(X, Q, k):
    d2 = ((Q[:, None, :].astype(np.float64) - X[None, :, :]) ** 2).sum(-1)
    ids = np.array([np.lexsort((np.arange(X.shape[0]), row))[:k] for row in d2])
    return ids, np.sqrt(np.take_along_axis(d2, ids, 1))


def test_driver_reduces_to_exact_knn():
    """beta >= 1 and a radius past every bound: S = D after round one, so Alg. 5 returns the
    exact k nearest neighbours (the textbook routine), here numpy brute force."""
    import datagen
    D = datagen.generate(1, n=2000, nq=20)
    X, Q = D["X"], D["Q"]
    ix = O.Index(X, 4, 16, 256, 42)
    ids, dists, st = ix.query(Q, 10, 1.5, 1e9, 2.0)
    ref_i, ref_d = _np_knn(X, Q, 10)
    assert np.array_equal(ids, ref_i)
    assert np.allclose(dists, ref_d, rtol=1e-6)
    assert np.all(st["reason"] == 1) and np.all(st["n_cand"] == 2000)
    ei, ed = O.exact_knn(X, Q, 10)
    assert np.array_equal(ei, ref_i) and np.allclose(ed, ref_d, rtol=1e-12)


def test_driver_k_equals_n_and_query_in_data():
    import datagen
    D = datagen.generate(1, n=300, nq=3)
    X = D["X"]
    ix = O.Index(X, 4, 16, 256, 42, max_size=16)
    ids, dists, st = ix.query(X[[5, 77]], 300, 1.5, 1.0, 0.1)     # k = n: all points sorted
    ref_i, _ = _np_knn(X, X[[5, 77]], 300)
    assert np.array_equal(ids, ref_i)
    ids, dists, st = ix.query(X[[5, 77, 123]], 3, 1.5, 1e-3, 0.1)  # q in D: itself at distance 0
    assert ids[:, 0].tolist() == [5, 77, 123] and np.all(dists[:, 0] == 0)


def test_driver_budget_and_determinism(tiny_oracle, tiny):
    c = tiny["cfg"]
    rmin = tiny_oracle.estimate_rmin(tiny["Qs"], c.k, c.c, c.beta)
    a = tiny_oracle.query(tiny["Q"][:30], c.k, c.c, rmin, c.beta)
    b = tiny_oracle.query(tiny["Q"][:30], c.k, c.c, rmin, c.beta)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    st = a[2]
    budget = math.ceil(c.beta * c.n) + c.k
    assert np.all(st["n_cand"][st["reason"] == 0] >= budget)
    assert np.all(st["n_cand"][st["reason"] == 1] < budget)
    assert np.all(st["n_cand"] >= c.k)
    # ids sorted by (dist, id)
    ids, d = a[0], a[1]
    for q in range(30):
        assert all((d[q, e], ids[q, e]) < (d[q, e + 1], ids[q, e + 1]) for e in range(c.k - 1))


def test_driver_round_cap():
    import datagen
    D = datagen.generate(1, n=500, nq=2)
    ix = O.Index(D["X"], 4, 16, 256, 42)
    ids, d, st = ix.query(D["Q"], 5, 1.5, 1e-30, 0.1)
    assert np.all(st["reason"] == 2) and np.all(st["rounds"] == 64)
    assert np.all(ids == -1) and np.all(np.isinf(d))


def test_rmin_defining_conditions(tiny_oracle, tiny):
    """at r*_q a full round gives |S| >= beta n + k; at r*_q / c it gives fewer."""
    c = tiny["cfg"]
    ix = tiny_oracle
    med, rs = ix.estimate_rmin(tiny["Qs"][:5], c.k, c.c, c.beta, return_all=True)
    budget = math.ceil(c.beta * c.n) + c.k
    for q in range(5):
        qp = ix.project_query(tiny["Qs"][q])
        def full_round(r):
            S = set()
            for i in range(ix.L):
                S |= set(ix.range_query(i, qp[i * ix.K:(i + 1) * ix.K], ix.eps * r).tolist())
            return len(S)
        assert full_round(rs[q] * (1 + 1e-9)) >= budget
        assert full_round(rs[q] / c.c) < budget
    assert med == np.sort(rs)[(len(rs) - 1) // 2]


def test_guarantee_theorem2(tiny_oracle, tiny):
    """Theorem 2: c^2-k-ANN with probability >= 1/2 - 1/e = 0.1321."""
    c = tiny["cfg"]
    rmin = tiny_oracle.estimate_rmin(tiny["Qs"], c.k, c.c, c.beta)
    ids, d, st = tiny_oracle.query(tiny["Q"], c.k, c.c, rmin, c.beta)
    _, gd = O.exact_knn(tiny["X"], tiny["Q"], c.k)
    ok = np.all(d <= c.c ** 2 * gd * (1 + 1e-6), axis=1)
    assert ok.mean() >= 0.5 - 1 / math.e
    recall = np.mean([len(set(ids[q]) & set(O.exact_knn(tiny["X"], tiny["Q"][q:q + 1], c.k)[0][0])) / c.k
                      for q in range(10)])
    assert recall >= 0.9


# ----------------------------------------------------------------- O9 / O10
def test_merge_topk_vs_numpy():
    rng = np.random.default_rng(8)
    G, nq, k = 3, 5, 7
    d = np.sort(rng.integers(0, 20, (G, nq, k)).astype(np.float32), -1)
    ids = rng.permutation(G * nq * k).reshape(G, nq, k).astype(np.int64)
    oi, od = O.merge_topk(ids, d, k)
    for q in range(nq):
        allp = sorted(zip(d[:, q].ravel().tolist(), ids[:, q].ravel().tolist()))[:k]
        assert oi[q].tolist() == [p[1] for p in allp] and od[q].tolist() == [p[0] for p in allp]


def test_shard_mode_g1_equals_unsharded(tiny):
    import datagen
    D = datagen.generate(1, n=3000, nq=10)
    X, Q = D["X"], D["Q"]
    ix = O.Index(X, 4, 16, 256, 42)
    a = ix.query(Q, 10, 1.5, 300.0, 0.1)
    b = O.sharded_query(X, 1, Q, 10, 1.5, 300.0, 0.1, 4, 16, 256, 42)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    # shards share A, sample and breakpoints with the whole
    s1 = O.Index(X, 4, 16, 256, 42, row_lo=1500, row_hi=3000)
    assert np.array_equal(s1.breakpoints(), ix.breakpoints())
    assert np.array_equal(s1.codes(), ix.codes()[1500:])


def test_recall_ratio_definitions():
    """recall = |R n R*|/k; overall ratio = mean ||q,o_i||/||q,o_i*||."""
    R, Rs = [1, 2, 3, 4], [3, 4, 5, 6]
    assert len(set(R) & set(Rs)) / 4 == 0.5
    assert np.mean(np.array([1.0, 3.0]) / np.array([1.0, 2.0])) == 1.25


def test_rc_ann_pins(tiny_oracle, tiny):
    """(r,c)-ANN, Alg. 4 pinned three ways: (1) a radius past every bound makes tree 1's
    range query return all of D, so |S| = n >= beta n + 1 and the answer is the exact nearest
    neighbour (numpy fp64 brute force, ties by id); (2) beta >= 1 never meets the budget, and with
    S = D the nearest neighbour lies within c r: same answer; (3) r below every bound: S is
    empty, nothing is returned; (4) at a middle radius the answer equals the first round of the
    c^2-k-ANN driver (Alg. 5, k = 1, r_min = r) whenever that round stopped it, and is
    "nothing" exactly when Alg. 5 needed a second round."""
    X, Q = tiny["X"], tiny["Q"][:40]
    d2 = ((Q[:, None, :].astype(np.float64) - X[None].astype(np.float64)) ** 2).sum(-1)
    nn = np.array([np.lexsort((np.arange(len(X)), row))[0] for row in d2])
    ids, dists = tiny_oracle.rc_ann(Q, 1e9, 1.5, 0.1)
    assert np.array_equal(ids, nn)
    assert np.allclose(dists, np.sqrt(d2[np.arange(len(Q)), nn]), rtol=1e-6)
    ids2, _ = tiny_oracle.rc_ann(Q, 1e9, 1.5, 2.0)
    assert np.array_equal(ids2, nn)
    ids3, d3 = tiny_oracle.rc_ann(Q, 1e-6, 1.5, 0.1)
    assert np.all(ids3 == -1) and np.all(np.isinf(d3))
    c = tiny["cfg"]
    rmin = tiny_oracle.estimate_rmin(tiny["Qs"], 1, c.c, c.beta)
    for r in (0.5 * rmin, rmin, 1.5 * rmin):
        ri, rd = tiny_oracle.rc_ann(Q, r, c.c, c.beta)
        qi, qd, st = tiny_oracle.query(Q, 1, c.c, r, c.beta)
        one = st["rounds"] == 1
        assert np.array_equal(ri[one], qi[one, 0]) and np.array_equal(rd[one], qd[one, 0])
        assert np.all(ri[~one] == -1)
        assert 0 < one.sum() or r < rmin


def _lb_order_reference(o, X, q, k, c, r_min, beta, L, K, N_r):
    """Sec. 6.2.2(2) re-derived from the exported trees and the pinned box bounds: per
    round, per tree, the leaves with LB <= (eps r)^2 in ascending (LB, leaf position) order; a
    leaf contributes its points whose own cell bound is <= (eps r)^2 (all of them when the
    leaf's upper bound is); |S| >= ceil(beta n)+k is checked after each leaf; else the radius
    test of Alg. 5 line 9 after the round."""
    n = len(X)
    B = o.breakpoints()
    codes = o.codes()
    qp = o.project_query(q)
    budget = int(np.ceil(beta * n)) + k
    trees = [o.tree(i) for i in range(L)]
    inS = np.zeros(n, bool)
    S = []
    r = r_min
    for _ in range(64):
        rho2 = (o.eps * r) ** 2
        for i, t in enumerate(trees):
            bi = B[i * K:(i + 1) * K]
            leaves = []
            for l in range(len(t["leaf_off"]) - 1):
                lb2, ub2 = O.box_bounds2(t["lo"][l], t["hi"][l], qp[i * K:(i + 1) * K], bi, N_r)
                if lb2 <= rho2:
                    leaves.append((lb2, l, ub2))
            for lb2, l, ub2 in sorted(leaves):
                for pid in t["perm"][t["leaf_off"][l]:t["leaf_off"][l + 1]]:
                    cl = codes[pid, i * K:(i + 1) * K]
                    if ub2 <= rho2 or O.box_bounds2(cl, cl, qp[i * K:(i + 1) * K], bi, N_r)[0] <= rho2:
                        if not inS[pid]:
                            inS[pid] = True
                            S.append(pid)
                if len(S) >= budget:
                    return np.array(sorted(S)), 0
        d2 = ((X[S].astype(np.float64) - q) ** 2).sum(1)
        if (d2 <= (c * r) ** 2).sum() >= k:
            return np.array(sorted(S)), 1
        r *= c
    return np.array(sorted(S)), 2


def test_lb_order_truncation_pins():
    """f2 pinned against an independent re-derivation (Python, from the exported trees and the
    pinned box bounds) on a small index at budgets that truncate inside a tree; with beta >= 1 the
    order cannot matter and lb_order equals plain Alg. 5."""
    import datagen
    D = datagen.generate(1, n=1500, nq=6)
    X, Q = D["X"], D["Q"]
    o = O.Index(X, 2, 8, 16, 11, max_size=24)
    reasons = []
    for beta, r in ((0.02, 300.0), (0.05, 400.0), (0.1, 600.0), (0.02, 150.0)):
        for qi in range(len(Q)):
            ids, _, st = o.query(Q[qi:qi + 1], 5, 1.5, r, beta, lb_order=True)
            S_ref, reason = _lb_order_reference(o, X, Q[qi].astype(np.float64), 5, 1.5, r, beta, 2, 8, 16)
            assert st["n_cand"][0] == len(S_ref) and st["reason"][0] == reason
            reasons.append(reason)
            d2 = ((X[S_ref].astype(np.float64) - Q[qi]) ** 2).sum(1)
            ref = S_ref[np.lexsort((S_ref, d2))][:5]
            assert np.array_equal(ids[0][:len(ref)], ref)
    assert reasons.count(0) >= 12 and reasons.count(1) >= 3     # budget cuts inside a tree, and radius stops
    a = o.query(Q, 5, 1.5, 30.0, 2.0, lb_order=True)
    b = o.query(Q, 5, 1.5, 30.0, 2.0)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[2]["n_cand"], b[2]["n_cand"])


# ----------------------------------------------------------------- RELAXED (f1) and the Alg. 5 driver,
# pinned against tests/_alg5_ref.py (numpy brute force; shares nothing with the oracle's traversal)
def test_tree_boxes_are_prefix_boxes(tiny_oracle):
    """Every exported leaf box is the Alg. 2 prefix box of its members: per dim the
    members share the top `bits` bits and [lo, hi] is exactly that prefix's symbol range."""
    ix = tiny_oracle
    nb = int(math.log2(ix.N_r))
    codes = ix.codes().astype(np.int64)
    for i in range(ix.L):
        t = ix.tree(i)
        c = codes[:, i * ix.K:(i + 1) * ix.K]
        bits = t["bits"].astype(np.int64)
        assert np.all(bits <= nb)
        leaf_of = np.repeat(np.arange(len(t["leaf_off"]) - 1), np.diff(t["leaf_off"]))
        mem = c[t["perm"]]
        shift = nb - bits[leaf_of]
        pre = (mem >> shift) << shift
        assert np.array_equal(pre, t["lo"][leaf_of].astype(np.int64))
        assert np.array_equal(t["hi"].astype(np.int64), t["lo"].astype(np.int64) + (1 << (nb - bits)) - 1)
        assert np.array_equal(np.sort(t["perm"]), np.arange(ix.n))          # each point in one leaf


def test_relaxed_range_query_brute_force(tiny_oracle, tiny):
    """Sec. 6.2.2(1): RELAXED returns exactly the points of the leaves whose box
    lower bound is <= rho -- brute force over the exported leaves, numpy bounds (not O6)."""
    from _alg5_ref import relaxed_range
    ix = tiny_oracle
    B = ix.breakpoints()
    rng = np.random.default_rng(17)
    trees = [ix.tree(i) for i in range(ix.L)]
    hit_partial = 0
    for it in range(48):
        qp = ix.project_query(tiny["Q"][it % 100])
        i = it % ix.L
        sl = slice(i * ix.K, (i + 1) * ix.K)
        rho = float(rng.uniform(0.05, 1.2)) * ix.eps * 100.0
        got = ix.range_query(i, qp[sl], rho, O.RELAXED)
        ref = relaxed_range(trees[i], B[sl], qp[sl], rho, ix.N_r)
        assert np.array_equal(got, ref), (it, len(got), len(ref))
        cell = ix.range_query(i, qp[sl], rho, O.CELL)
        hit_partial += len(ref) > len(cell)
    assert hit_partial >= 10     # radii where RELAXED really takes more than CELL


@pytest.mark.parametrize("m", [0, 3])
def test_driver_equals_tree_granular_rederivation(tiny_oracle, tiny, m):
    """Alg. 5 re-run in numpy tree by tree: budget |S| >= ceil(beta n)+k tested after
    EACH tree (line 7), radius test after the round (line 9), r <- c r (line 11).  The
    oracle's stop (reason, round, tree), |S| and top-k must equal it for every query."""
    from _alg5_ref import Space, alg5
    ix = tiny_oracle
    c = tiny["cfg"]
    rmin = ix.estimate_rmin(tiny["Qs"], c.k, c.c, c.beta) * c.c ** (-m)
    Q = tiny["Q"][:40]
    ids, dists, st = ix.query(Q, c.k, c.c, rmin, c.beta)
    sp = Space(ix.breakpoints(), ix.codes(), ix.K, ix.N_r)
    mid_round = 0
    for q in range(len(Q)):
        ref = alg5(sp, ix.eps, tiny["X"], Q[q], ix.project_query(Q[q]), c.k, c.c, rmin, c.beta, ix.n)
        got = (int(st["reason"][q]), int(st["rounds"][q]), int(st["trees_last"][q]), int(st["n_cand"][q]))
        assert got == (ref["reason"], ref["rounds"], ref["trees_last"], ref["n_cand"]), (q, got, ref["reason"])
        assert st["r_final"][q] == ref["r_final"]
        assert np.array_equal(ids[q], ref["ids"])
        assert np.array_equal(dists[q], np.sqrt(ref["d2"]).astype(np.float32))
        mid_round += ref["reason"] == 0 and ref["trees_last"] < ix.L
    if m == 0:
        assert mid_round >= 5    # budget stops inside a round exercise the after-each-tree rule
