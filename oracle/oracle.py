"""ctypes wrapper over liboracle.so -- TEST INFRASTRUCTURE ONLY.

The oracle is a plain single-threaded fp64 C implementation of DET-LSH
(arxiv 2603.24920) written from the paper (see detlsh_oracle.c).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module.  It never imports the product
package ``paper_2603_24920_b200`` and the product never imports it.

Parity status of each function:
  chi2_sf / chi2_isf / params ...... pinned (closed forms K=2,4; scipy)
  hash_family ...................... pinned (N(0,1) moments, Lemma 1/2 stats)
  project .......................... pinned (numpy fp64 matmul, linearity)
  sample_ids ....................... pinned (brute-force sort in numpy)
  breakpoints_sort / _qselect ...... pinned (S:188 worked example, equal-count)
  encode_value ..................... pinned (S:197 examples, searchsorted)
  tree_build / export .............. pinned (P:359 example, invariants, literal == bulk)
  box_bounds2 ...................... pinned (P:581-584 example, sandwich)
  range_query ...................... pinned (brute-force scan of the predicate)
  query ............................ pinned (exact-kNN special case, k=n, q in D, budget)
  merge_topk / exact_knn ........... pinned (numpy argsort)
  estimate_rmin .................... partly pinned (defining conditions); the
                                     grid/median convention itself is unpinned
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

CELL, RELAXED, EXACT = 0, 1, 2


def build() -> str:
    """Compile liboracle.so with its Makefile (plain gcc)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        src = os.path.join(_HERE, "detlsh_oracle.c")
        if (not os.path.exists(_LIB_PATH)) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
            build()
        L = C.CDLL(_LIB_PATH)
        P = C.c_void_p
        i64, i32, f64, u64 = C.c_int64, C.c_int, C.c_double, C.c_uint64
        sig = {
            "orc_chi2_sf": (f64, [f64, i32]),
            "orc_chi2_isf": (f64, [f64, i32]),
            "orc_params": (None, [i32, i32, f64, P, P, P, P]),
            "orc_splitmix64": (u64, [u64]),
            "orc_hash_family": (None, [u64, i32, i32, i32, P]),
            "orc_project": (None, [P, i32, i32, P, i64, P]),
            "orc_sample_size": (i64, [i64, i32, f64]),
            "orc_sample_ids": (None, [u64, i64, i64, P]),
            "orc_breakpoints_sort": (None, [P, i64, i32, P]),
            "orc_breakpoints_qselect": (None, [P, i64, i32, P]),
            "orc_encode_value": (i32, [C.c_float, P, i32]),
            "orc_tree_build": (P, [P, i64, i64, i32, i32, i32, i32]),
            "orc_tree_free": (None, [P]),
            "orc_tree_num_leaves": (i64, [P]),
            "orc_tree_export": (None, [P, P, P, P, P, P]),
            "orc_box_bounds2": (None, [P, P, P, P, i32, i32, P, P]),
            "orc_build": (P, [P, i64, i32, i64, i64, i32, i32, i32, u64, i32, f64, i32]),
            "orc_index_free": (None, [P]),
            "orc_index_n": (i64, [P]),
            "orc_index_n_sample": (i64, [P]),
            "orc_index_A": (P, [P]),
            "orc_index_breakpoints": (P, [P]),
            "orc_index_P": (P, [P]),
            "orc_index_codes": (P, [P]),
            "orc_index_sample": (P, [P]),
            "orc_index_tree": (P, [P, i32]),
            "orc_index_eps": (f64, [P]),
            "orc_range_query": (i64, [P, i32, P, f64, i32, P]),
            "orc_query": (None, [P, P, i64, i32, f64, f64, f64, i32, P, P, P]),
            "orc_query_ex": (None, [P, P, i64, i32, f64, f64, f64, i32, i32, P, P, P]),
            "orc_project_query": (None, [P, P, P]),
            "orc_rc_ann": (None, [P, P, i64, f64, f64, f64, i32, P, P]),
            "orc_merge_topk": (None, [P, P, i32, i64, i32, P, P]),
            "orc_exact_knn": (None, [P, i64, i32, P, i64, i32, P, P]),
            "orc_estimate_rmin": (f64, [P, P, i64, i32, f64, f64, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


QSTATS_DTYPE = np.dtype([("rounds", np.int32), ("trees_last", np.int32), ("reason", np.int32),
                         ("pad", np.int32), ("n_cand", np.int64), ("r_final", np.float64)])


# ---------------------------------------------------------------- O1
def chi2_sf(y: float, K: int) -> float:
    return lib().orc_chi2_sf(float(y), int(K))


def chi2_isf(alpha: float, K: int) -> float:
    return lib().orc_chi2_isf(float(alpha), int(K))


def params(K: int, L: int, c: float = 1.5):
    out = [C.c_double() for _ in range(4)]
    lib().orc_params(K, L, float(c), *[C.byref(o) for o in out])
    a1, eps, a2, beta = (o.value for o in out)
    return {"alpha1": a1, "eps": eps, "alpha2": a2, "beta_theory": beta}


# ---------------------------------------------------------------- O2
def splitmix64(x: int) -> int:
    return lib().orc_splitmix64(x & 0xFFFFFFFFFFFFFFFF)


def hash_family(seed: int, d: int, L: int, K: int) -> np.ndarray:
    A = np.empty((L * K, d), np.float32)
    lib().orc_hash_family(seed, d, L, K, _p(A))
    return A


def project(A: np.ndarray, X: np.ndarray) -> np.ndarray:
    A = _c(A, np.float32)
    X = _c(X, np.float32)
    P = np.empty((X.shape[0], A.shape[0]), np.float32)
    lib().orc_project(_p(A), A.shape[0], A.shape[1], _p(X), X.shape[0], _p(P))
    return P


# ---------------------------------------------------------------- O3/O4
def sample_size(n: int, N_r: int, f: float) -> int:
    return lib().orc_sample_size(n, N_r, f)


def sample_ids(seed: int, n: int, n_s: int) -> np.ndarray:
    ids = np.empty(n_s, np.int64)
    lib().orc_sample_ids(seed, n, n_s, _p(ids))
    return ids


def breakpoints_sort(v, N_r: int) -> np.ndarray:
    v = _c(v, np.float32)
    out = np.empty(N_r + 1, np.float32)
    lib().orc_breakpoints_sort(_p(v), v.size, N_r, _p(out))
    return out


def breakpoints_qselect(v, N_r: int) -> np.ndarray:
    v = _c(v, np.float32)
    out = np.empty(N_r + 1, np.float32)
    lib().orc_breakpoints_qselect(_p(v), v.size, N_r, _p(out))
    return out


def encode_value(x: float, b, N_r: int) -> int:
    b = _c(b, np.float32)
    return lib().orc_encode_value(float(x), _p(b), N_r)


# ---------------------------------------------------------------- O5/O6
class Tree:
    """Handle over an oracle DE-Tree built from codes [n][stride] (first K used)."""

    def __init__(self, codes: np.ndarray, K: int, N_r: int, max_size: int, builder: int = 0):
        self._codes = _c(codes, np.uint8)
        n, stride = self._codes.shape
        self.K = K
        self._h = lib().orc_tree_build(_p(self._codes), n, stride, K, N_r, max_size, builder)
        self.n = n

    def export(self):
        nl = lib().orc_tree_num_leaves(self._h)
        off = np.empty(nl + 1, np.int64)
        perm = np.empty(self.n, np.int64)
        lo = np.empty((nl, self.K), np.uint8)
        hi = np.empty((nl, self.K), np.uint8)
        bits = np.empty((nl, self.K), np.uint8)
        lib().orc_tree_export(self._h, _p(off), _p(perm), _p(lo), _p(hi), _p(bits))
        return {"leaf_off": off, "perm": perm, "lo": lo, "hi": hi, "bits": bits}

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_tree_free(self._h)
            self._h = None


def tree_export_ptr(h, n: int, K: int):
    nl = lib().orc_tree_num_leaves(h)
    off = np.empty(nl + 1, np.int64)
    perm = np.empty(n, np.int64)
    lo = np.empty((nl, K), np.uint8)
    hi = np.empty((nl, K), np.uint8)
    bits = np.empty((nl, K), np.uint8)
    lib().orc_tree_export(h, _p(off), _p(perm), _p(lo), _p(hi), _p(bits))
    return {"leaf_off": off, "perm": perm, "lo": lo, "hi": hi, "bits": bits}


def box_bounds2(lo, hi, x, b, N_r: int):
    lo = _c(lo, np.uint8)
    hi = _c(hi, np.uint8)
    x = _c(x, np.float32)
    b = _c(b, np.float32)
    lb = C.c_double()
    ub = C.c_double()
    lib().orc_box_bounds2(_p(lo), _p(hi), _p(x), _p(b), lo.size, N_r, C.byref(lb), C.byref(ub))
    return lb.value, ub.value


# ---------------------------------------------------------------- index, O7-O10
class Index:
    """Oracle index over rows [row_lo,row_hi) of X (global hash family/sample/breakpoints)."""

    def __init__(self, X: np.ndarray, L: int, K: int, N_r: int, seed: int, max_size: int = 128,
                 sample_frac: float = 0.01, builder: int = 1, row_lo: int = 0, row_hi=None):
        self.X = _c(X, np.float32)
        n_global, d = self.X.shape
        row_hi = n_global if row_hi is None else row_hi
        self.n_global, self.d, self.L, self.K, self.N_r = n_global, d, L, K, N_r
        self.row_lo, self.row_hi = row_lo, row_hi
        self.n = row_hi - row_lo
        self._h = lib().orc_build(_p(self.X), n_global, d, row_lo, row_hi, L, K, N_r, seed,
                                  max_size, float(sample_frac), builder)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_index_free(self._h)
            self._h = None

    # exports (copies)
    def _arr(self, ptr, shape, dtype):
        n = int(np.prod(shape))
        buf = (C.c_byte * (n * np.dtype(dtype).itemsize)).from_address(ptr)
        return np.frombuffer(buf, dtype=dtype, count=n).reshape(shape).copy()

    @property
    def eps(self) -> float:
        return lib().orc_index_eps(self._h)

    def A(self):
        return self._arr(lib().orc_index_A(self._h), (self.L * self.K, self.d), np.float32)

    def breakpoints(self):
        return self._arr(lib().orc_index_breakpoints(self._h), (self.L * self.K, self.N_r + 1), np.float32)

    def P(self):
        return self._arr(lib().orc_index_P(self._h), (self.n, self.L * self.K), np.float32)

    def codes(self):
        return self._arr(lib().orc_index_codes(self._h), (self.n, self.L * self.K), np.uint8)

    def sample(self):
        ns = lib().orc_index_n_sample(self._h)
        return self._arr(lib().orc_index_sample(self._h), (ns,), np.int64)

    def tree(self, i: int):
        return tree_export_ptr(lib().orc_index_tree(self._h, i), self.n, self.K)

    def project_query(self, q) -> np.ndarray:
        q = _c(q, np.float32)
        qp = np.empty(self.L * self.K, np.float32)
        lib().orc_project_query(self._h, _p(q), _p(qp))
        return qp

    def range_query(self, i: int, qp_i, rho: float, mode: int = CELL) -> np.ndarray:
        qp_i = _c(qp_i, np.float32)
        out = np.empty(self.n, np.int64)
        cnt = lib().orc_range_query(self._h, i, _p(qp_i), float(rho), mode, _p(out))
        return out[:cnt].copy()

    def query(self, Q, k: int, c: float, r_min: float, beta: float, mode: int = CELL, lb_order: bool = False):
        """Alg. 5; lb_order: Sec. 6.2.2(2) leaves in (LB, leaf) order, budget checked per leaf."""
        Q = _c(Q, np.float32).reshape(-1, self.d)
        nq = Q.shape[0]
        ids = np.empty((nq, k), np.int64)
        dists = np.empty((nq, k), np.float32)
        st = np.zeros(nq, QSTATS_DTYPE)
        lib().orc_query_ex(self._h, _p(Q), nq, k, float(c), float(r_min), float(beta), mode, int(lb_order),
                           _p(ids), _p(dists), _p(st))
        return ids, dists, st

    def rc_ann(self, Q, r: float, c: float, beta: float, mode: int = CELL):
        """(r,c)-ANN, Alg. 4: per query (id, dist) or (-1, inf)."""
        Q = _c(Q, np.float32).reshape(-1, self.d)
        nq = Q.shape[0]
        ids = np.empty(nq, np.int64)
        dists = np.empty(nq, np.float32)
        lib().orc_rc_ann(self._h, _p(Q), nq, float(c), float(r), float(beta), mode, _p(ids), _p(dists))
        return ids, dists

    def estimate_rmin(self, Qs, k: int, c: float, beta: float, return_all: bool = False):
        Qs = _c(Qs, np.float32).reshape(-1, self.d)
        rs = np.empty(Qs.shape[0], np.float64)
        med = lib().orc_estimate_rmin(self._h, _p(Qs), Qs.shape[0], k, float(c), float(beta), _p(rs))
        return (med, rs) if return_all else med


def merge_topk(ids: np.ndarray, dists: np.ndarray, k: int):
    """ids/dists: [G][nq][k] -> merged [nq][k] by (dist, id)."""
    ids = _c(ids, np.int64)
    dists = _c(dists, np.float32)
    G, nq, _ = ids.shape
    oi = np.empty((nq, k), np.int64)
    od = np.empty((nq, k), np.float32)
    lib().orc_merge_topk(_p(ids), _p(dists), G, nq, k, _p(oi), _p(od))
    return oi, od


def exact_knn(X, Q, k: int):
    X = _c(X, np.float32)
    Q = _c(Q, np.float32).reshape(-1, X.shape[1])
    ids = np.empty((Q.shape[0], k), np.int64)
    dists = np.empty((Q.shape[0], k), np.float64)
    lib().orc_exact_knn(_p(X), X.shape[0], X.shape[1], _p(Q), Q.shape[0], k, _p(ids), _p(dists))
    return ids, dists


def sharded_query(X, G: int, Q, k, c, r_min, beta, L, K, N_r, seed, max_size=128,
                  sample_frac=0.01, mode=CELL):
    """O9: G shards over ids [floor(g n/G), floor((g+1) n/G)), per-shard budget, merge."""
    n = X.shape[0]
    all_ids, all_d = [], []
    for g in range(G):
        lo, hi = (g * n) // G, ((g + 1) * n) // G
        ix = Index(X, L, K, N_r, seed, max_size, sample_frac, row_lo=lo, row_hi=hi)
        i, d, _ = ix.query(Q, k, c, r_min, beta, mode)
        all_ids.append(i)
        all_d.append(d)
        del ix
    return merge_topk(np.stack(all_ids), np.stack(all_d), k)
