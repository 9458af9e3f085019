"""Thin ctypes binding of libdetlsh.so (include/detlsh.h) -- argument marshalling only.

Every step of DET-LSH runs inside the CUDA library; this module only converts numpy
arrays / torch tensors to pointers and raises on a non-OK status.  There is no CPU
fallback: if the library is missing or cannot load, ``lib()`` raises.

Buffers may be numpy arrays (host) or CUDA torch tensors (device); outputs are
allocated like the input (host in -> host out, device in -> device out) unless given.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdetlsh.so")

DETLSH_OK, DETLSH_EINVAL, DETLSH_ENOMEM, DETLSH_ECUDA, DETLSH_ENCCL, DETLSH_EINTERNAL = range(6)
MODE_CELL, MODE_RELAXED, MODE_EXACT = 0, 1, 2
_NAMES = {1: "EINVAL", 2: "ENOMEM", 3: "ECUDA", 4: "ENCCL", 5: "EINTERNAL"}


class DetlshError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"detlsh {_NAMES.get(status, status)}: {msg}")
        self.status = status


class detlsh_opts(C.Structure):
    _fields_ = [("max_size", C.c_int32), ("sample_frac", C.c_double), ("mode", C.c_int32),
                ("query_batch", C.c_int32), ("stream", C.c_uint64), ("borrow_data", C.c_int32),
                ("proj_impl", C.c_int32), ("mem_budget", C.c_int64),
                ("verify_impl", C.c_int32), ("keep_projections", C.c_int32), ("lb_order", C.c_int32),
                ("pad1", C.c_int32)]


class detlsh_kernel_time(C.Structure):
    _fields_ = [("name", C.c_char * 64), ("launches", C.c_int64), ("total_ms", C.c_double)]


class detlsh_query_stats(C.Structure):
    _fields_ = [("rounds", C.c_int32), ("trees_last", C.c_int32), ("reason", C.c_int32),
                ("pad", C.c_int32), ("n_cand", C.c_int64), ("r_final", C.c_double),
                ("leaves_tested", C.c_int64), ("leaves_passed", C.c_int64), ("points_tested", C.c_int64),
                ("points_passed", C.c_int64), ("subboxes_tested", C.c_int64)]


STATS_DTYPE = np.dtype([("rounds", np.int32), ("trees_last", np.int32), ("reason", np.int32),
                        ("pad", np.int32), ("n_cand", np.int64), ("r_final", np.float64),
                        ("leaves_tested", np.int64), ("leaves_passed", np.int64), ("points_tested", np.int64),
                        ("points_passed", np.int64), ("subboxes_tested", np.int64)])

_lib = None


def build(quiet: bool = True) -> str:
    """Compile libdetlsh.so in-tree (nvcc, sm_100a only)."""
    import subprocess
    subprocess.run(["make", "-s", "-j8", "-C", _HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)
    return LIB_PATH


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `make -C {_HERE}` (CUDA library required; no fallback)")
    L = C.CDLL(LIB_PATH)
    P, i64, i32, u64, f64, sz = C.c_void_p, C.c_int64, C.c_int32, C.c_uint64, C.c_double, C.c_size_t
    O = C.POINTER(detlsh_opts)
    sig = {
        "detlsh_default_opts": (None, [O]),
        "detlsh_build": (i32, [P, i64, i32, i32, i32, i32, u64, P]),
        "detlsh_build_ex": (i32, [P, i64, i32, i32, i32, i32, u64, O, i64, i64, P, P]),
        "detlsh_query": (i32, [P, P, i64, i32, f64, f64, f64, P, P]),
        "detlsh_query_ex": (i32, [P, P, i64, i32, f64, f64, f64, O, P, P, P]),
        "detlsh_query_candidates": (i32, [P, P, i64, i32, f64, f64, f64, O, P, P, P, P, i64]),
        "detlsh_free": (None, [P]),
        "detlsh_last_error": (C.c_char_p, []),
        "detlsh_params": (i32, [i32, i32, f64, P, P, P]),
        "detlsh_sample_size": (i64, [i64, i32, f64]),
        "detlsh_sample_projections": (i32, [P, i64, i32, i32, i32, i32, u64, f64, i64, i64, O, P, i64, P]),
        "detlsh_breakpoints_from_samples": (i32, [P, i64, i32, i32, O, P]),
        "detlsh_merge_topk": (i32, [P, P, i32, i64, i32, P, P]),
        "detlsh_project": (i32, [P, P, i64, P]),
        "detlsh_project_ex": (i32, [P, P, i64, i32, P]),
        "detlsh_debug_export": (i32, [P, i32, i32, P, sz, C.POINTER(sz)]),
        "detlsh_build_from_codes": (i32, [P, i64, i32, i32, i32, O, P]),
        "detlsh_launch_count": (i64, []),
        "detlsh_estimate_rmin": (i32, [P, P, i64, i32, f64, O, P, P]),
        "detlsh_rc_ann": (i32, [P, P, i64, f64, f64, f64, O, P, P, P]),
        "detlsh_save": (i32, [P, C.c_char_p]),
        "detlsh_load": (i32, [C.c_char_p, P]),
        "detlsh_index_info": (i32, [P, P]),
        "detlsh_profile_enable": (None, [i32]),
        "detlsh_profile_filter": (None, [C.c_char_p]),
        "detlsh_profile_reset": (None, []),
        "detlsh_release_workspace": (None, []),
        "detlsh_workspace_bytes": (i64, []),
        "detlsh_profile_read": (i32, [P, i32]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def _check(status: int):
    if status != DETLSH_OK:
        raise DetlshError(status, lib().detlsh_last_error().decode())


def _is_torch(x):
    return type(x).__module__.startswith("torch")


def _ptr(x):
    if x is None:
        return None
    if _is_torch(x):
        assert x.is_contiguous()
        return C.c_void_p(x.data_ptr())
    assert x.flags["C_CONTIGUOUS"]
    return x.ctypes.data_as(C.c_void_p)


def _like(ref, shape, np_dtype, torch_dtype=None):
    if _is_torch(ref) and ref.is_cuda:
        import torch
        return torch.empty(shape, dtype=torch_dtype, device=ref.device)
    return np.empty(shape, np_dtype)


def _f32(x):
    if _is_torch(x):
        import torch
        return x.to(torch.float32).contiguous()
    return np.ascontiguousarray(x, np.float32)


def default_opts(**kw) -> detlsh_opts:
    o = detlsh_opts()
    lib().detlsh_default_opts(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def launch_count() -> int:
    return int(lib().detlsh_launch_count())


def profile_enable(on: bool = True):
    lib().detlsh_profile_enable(1 if on else 0)


def release_workspace():
    lib().detlsh_release_workspace()


def workspace_bytes() -> int:
    return int(lib().detlsh_workspace_bytes())


def profile_filter(prefixes: str | None):
    lib().detlsh_profile_filter(prefixes.encode() if prefixes else None)


def profile_reset():
    lib().detlsh_profile_reset()


def profile_read() -> dict:
    """{kernel name: (launches, total_ms)} since the last reset."""
    n = lib().detlsh_profile_read(None, 0)
    arr = (detlsh_kernel_time * max(n, 1))()
    n = lib().detlsh_profile_read(C.cast(arr, C.c_void_p), n)
    return {arr[i].name.decode(): (int(arr[i].launches), float(arr[i].total_ms)) for i in range(n)}


def detlsh_params(K: int, L: int, c: float):
    e, a2, b = C.c_double(), C.c_double(), C.c_double()
    _check(lib().detlsh_params(K, L, c, C.byref(e), C.byref(a2), C.byref(b)))
    return {"eps": e.value, "alpha2": a2.value, "beta_theory": b.value}


def detlsh_sample_size(n: int, N_r: int, f: float) -> int:
    return int(lib().detlsh_sample_size(n, N_r, f))


class Index:
    """Owning handle of a device index (detlsh_index*)."""

    def __init__(self, handle, n, d, L, K, N_r, data_ref=None):
        self._h = handle
        self.n, self.d, self.L, self.K, self.N_r = n, d, L, K, N_r
        self._data_ref = data_ref   # keeps a borrowed device buffer alive

    def __del__(self):
        self.free()

    def free(self):
        if getattr(self, "_h", None):
            lib().detlsh_free(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    # ------------------------------------------------------------------ query
    def query(self, Q, k: int, c: float, r_min: float, beta: float, opts: detlsh_opts | None = None,
              stats: bool = False, out_ids=None, out_dists=None):
        return detlsh_query_ex(self, Q, k, c, r_min, beta, opts, stats, out_ids, out_dists)

    def save(self, path: str):
        _check(lib().detlsh_save(self._h, str(path).encode()))

    def rc_ann(self, Q, r: float, c: float, beta: float, opts: detlsh_opts | None = None, stats: bool = False):
        """(r,c)-ANN, Alg. 4: per query (id, dist), (-1, inf) for "nothing"."""
        Q = _f32(Q)
        nq = Q.shape[0]
        ids = _like(Q, (nq,), np.int64, _torch_i64())
        dists = _like(Q, (nq,), np.float32, _torch_f32())
        st = np.zeros(nq, STATS_DTYPE) if stats else None
        o = opts if opts is not None else default_opts()
        _check(lib().detlsh_rc_ann(self._h, _ptr(Q), nq, r, c, beta, C.byref(o), _ptr(ids), _ptr(dists), _ptr(st)))
        return (ids, dists, st) if stats else (ids, dists)

    # ------------------------------------------------------------------ debug / test exports
    def export(self, what: int, tree: int = 0):
        need = C.c_size_t()
        _check(lib().detlsh_debug_export(self._h, what, tree, None, 0, C.byref(need)))
        sc = np.empty(4, np.int64)
        _check(lib().detlsh_debug_export(self._h, 9, tree if what >= 4 else 0, sc.ctypes.data_as(C.c_void_p), 32, None))
        n, n_s, nl, d = (int(v) for v in sc)
        LK = self.L * self.K
        shapes = {0: ((LK, d), np.float32), 1: ((LK, self.N_r + 1), np.float32), 2: ((n, LK), np.uint8),
                  3: ((n_s,), np.int64), 4: ((n,), np.int64), 5: ((nl + 1,), np.int64),
                  6: ((nl, self.K), np.uint8), 7: ((nl, self.K), np.uint8), 8: ((nl, self.K), np.uint8)}
        shape, dt = shapes[what]
        out = np.empty(shape, dt)
        assert out.nbytes == need.value, (out.nbytes, need.value)
        _check(lib().detlsh_debug_export(self._h, what, tree, out.ctypes.data_as(C.c_void_p), out.nbytes, None))
        return out

    def A(self):
        return self.export(0)

    def breakpoints(self):
        return self.export(1)

    def codes(self):
        return self.export(2)

    def sample(self):
        return self.export(3)

    def tree(self, i: int):
        return {"perm": self.export(4, i), "leaf_off": self.export(5, i), "lo": self.export(6, i),
                "hi": self.export(7, i), "bits": self.export(8, i)}

    def estimate_rmin(self, Qs, k: int, beta: float, opts: detlsh_opts | None = None, return_all: bool = False):
        """GPU r_min estimator (AMB-22): lower median over sample queries of r*_q."""
        Qs = _f32(Qs)
        ns = Qs.shape[0]
        rs = np.empty(ns, np.float64)
        rm = C.c_double()
        o = opts if opts is not None else default_opts()
        _check(lib().detlsh_estimate_rmin(self._h, _ptr(Qs), ns, k, beta, C.byref(o), _ptr(rs), C.byref(rm)))
        return (rm.value, rs) if return_all else rm.value

    def project(self, X, proj_impl: int | None = None):
        X = _f32(X)
        m = X.shape[0]
        out = _like(X, (m, self.L * self.K), np.float32, _torch_f32())
        if proj_impl is None:
            _check(lib().detlsh_project(self._h, _ptr(X), m, _ptr(out)))
        else:
            _check(lib().detlsh_project_ex(self._h, _ptr(X), m, proj_impl, _ptr(out)))
        return out


def _torch_f32():
    try:
        import torch
        return torch.float32
    except ImportError:   # pragma: no cover
        return None


def _torch_i64():
    try:
        import torch
        return torch.int64
    except ImportError:   # pragma: no cover
        return None


def detlsh_build(data, L: int, K: int, N_r: int, seed: int, opts: detlsh_opts | None = None,
                 id_offset: int = 0, n_global: int | None = None, breakpoints=None) -> Index:
    data = _f32(data)
    n, d = data.shape
    h = C.c_void_p()
    bp = _f32(breakpoints) if breakpoints is not None else None
    if opts is None and id_offset == 0 and n_global is None and bp is None:
        _check(lib().detlsh_build(_ptr(data), n, d, L, K, N_r, seed, C.byref(h)))
    else:
        o = opts if opts is not None else default_opts()
        _check(lib().detlsh_build_ex(_ptr(data), n, d, L, K, N_r, seed, C.byref(o), id_offset,
                                     n if n_global is None else n_global, _ptr(bp), C.byref(h)))
    borrowed = data if (opts is not None and opts.borrow_data) else None
    return Index(h, n, d, L, K, N_r, borrowed)


def detlsh_query_ex(index: Index, Q, k, c, r_min, beta, opts=None, stats=False, out_ids=None, out_dists=None):
    Q = _f32(Q)
    nq = Q.shape[0]
    ids = out_ids if out_ids is not None else _like(Q, (nq, k), np.int64, _torch_i64())
    dists = out_dists if out_dists is not None else _like(Q, (nq, k), np.float32, _torch_f32())
    st = np.zeros(nq, STATS_DTYPE) if stats else None
    if opts is None and not stats:
        _check(lib().detlsh_query(index.handle, _ptr(Q), nq, k, c, r_min, beta, _ptr(ids), _ptr(dists)))
    else:
        o = opts if opts is not None else default_opts()
        _check(lib().detlsh_query_ex(index.handle, _ptr(Q), nq, k, c, r_min, beta, C.byref(o), _ptr(ids),
                                     _ptr(dists), _ptr(st)))
    return (ids, dists, st) if stats else (ids, dists)


def detlsh_query_candidates(index: Index, Q, k, c, r_min, beta, opts=None):
    """Test hook: ids, dists, stats and each query's final candidate set S as a [nq][ceil(n/32)] u32 bitmap."""
    Q = _f32(Q)
    nq = Q.shape[0]
    ids = np.empty((nq, k), np.int64)
    dists = np.empty((nq, k), np.float32)
    st = np.zeros(nq, STATS_DTYPE)
    w = (index.n + 31) // 32
    S = np.zeros((nq, w), np.uint32)
    o = opts if opts is not None else default_opts()
    _check(lib().detlsh_query_candidates(index.handle, _ptr(Q), nq, k, c, r_min, beta, C.byref(o), _ptr(ids),
                                         _ptr(dists), _ptr(st), _ptr(S), w))
    return ids, dists, st, S


def candidate_ids(S_row, n: int) -> np.ndarray:
    """Local ids whose bit is set in one exported S bitmap row (ascending)."""
    bits = np.unpackbits(np.ascontiguousarray(S_row, np.uint32).view(np.uint8), bitorder="little")
    return np.flatnonzero(bits[:n])


def detlsh_query(index: Index, Q, k, c, r_min, beta):
    return detlsh_query_ex(index, Q, k, c, r_min, beta)


def detlsh_load(path: str) -> Index:
    """Load an index written by Index.save (detlsh_load)."""
    h = C.c_void_p()
    _check(lib().detlsh_load(str(path).encode(), C.byref(h)))
    info = np.zeros(8, np.int64)
    _check(lib().detlsh_index_info(h, info.ctypes.data_as(C.c_void_p)))
    n, d, L, K, N_r = (int(v) for v in info[:5])
    return Index(h, n, d, L, K, N_r)


def detlsh_build_from_codes(codes, L: int, K: int, N_r: int, max_size: int = 128) -> Index:
    codes = np.ascontiguousarray(codes, np.uint8) if not _is_torch(codes) else codes.contiguous()
    n = codes.shape[0]
    h = C.c_void_p()
    o = default_opts(max_size=max_size)
    _check(lib().detlsh_build_from_codes(_ptr(codes), n, L, K, N_r, C.byref(o), C.byref(h)))
    return Index(h, n, 1, L, K, N_r)


def detlsh_merge_topk(ids, dists, k: int):
    """C2 merge of [G][nq][k'] per-shard lists on the device; torch CUDA tensors stay on the device."""
    if _is_torch(ids):
        import torch
        ids = ids.to(torch.int64).contiguous()
        dists = dists.to(device=ids.device, dtype=torch.float32).contiguous()
    else:
        ids = np.ascontiguousarray(ids, np.int64)
        dists = np.ascontiguousarray(dists, np.float32)
    G, nq, kk = ids.shape
    assert kk == k, "per-shard lists must hold k entries"
    oi = _like(ids, (nq, k), np.int64, _torch_i64())
    od = _like(ids, (nq, k), np.float32, _torch_f32())
    _check(lib().detlsh_merge_topk(_ptr(ids), _ptr(dists), G, nq, k, _ptr(oi), _ptr(od)))
    return oi, od


def detlsh_sample_projections(data, L, K, N_r, seed, sample_frac, id_offset, n_global, cap=None,
                              opts: detlsh_opts | None = None):
    data = _f32(data)
    n, d = data.shape
    cap = cap if cap is not None else detlsh_sample_size(n_global, N_r, sample_frac)
    out = _like(data, (max(cap, 1), L * K), np.float32, _torch_f32())
    got = C.c_int64()
    o = opts if opts is not None else default_opts()
    _check(lib().detlsh_sample_projections(_ptr(data), n, d, L, K, N_r, seed, sample_frac, id_offset, n_global,
                                           C.byref(o), _ptr(out), cap, C.byref(got)))
    return out[:got.value]


def detlsh_breakpoints_from_samples(samples, N_r: int, opts: detlsh_opts | None = None):
    samples = _f32(samples)
    m, LK = samples.shape
    out = _like(samples, (LK, N_r + 1), np.float32, _torch_f32())
    o = opts if opts is not None else default_opts()
    _check(lib().detlsh_breakpoints_from_samples(_ptr(samples), m, LK, N_r, C.byref(o), _ptr(out)))
    return out
