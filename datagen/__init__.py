"""Seeded synthetic inputs shaped like the paper's workloads (BASELINE.json configs).

This module is shared by the oracle tests and by the CUDA path's tests and bench.
It holds NONE of the method's arithmetic: only the data/query distributions and
the per-config parameters.  The paper's datasets (PAPER.md Table `table2`,
P:770-790) are not available; these mixtures stand in for them (DESIGN.md,
"Input recipe").

Every array is produced by numpy's PCG64 from a SeedSequence of
``[seed, stream]`` (stream 1 = data, 2 = queries, 3 = r_min sample queries),
drawing rows in fixed chunks of 2^20 so the bytes do not depend on memory.
Queries come from the same mixture (same centres) but a different stream, so
they are held out (AMB-27).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

CHUNK = 1 << 20


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    d: int
    nq: int
    k: int
    L: int
    K: int
    N_r: int
    c: float
    beta: float
    seed: int          # data seed
    kind: str          # mixture family
    comps: int
    index_seed: int = 42
    max_size: int = 128
    sample_frac: float = 0.01
    extra: dict = field(default_factory=dict)


CONFIGS = {
    1: Config("tiny", 10_000, 128, 100, 10, 4, 16, 256, 1.5, 0.1, 1001, "gauss_box", 100),
    2: Config("deep1m_like", 1_000_000, 256, 1000, 50, 4, 16, 256, 1.5, 0.1, 1002, "unit", 1000),
    3: Config("gist_like", 1_000_000, 960, 1000, 100, 4, 16, 256, 1.5, 0.1, 1003, "abs01", 500),
    4: Config("sift10m_like", 10_000_000, 128, 10_000, 100, 4, 16, 256, 1.5, 0.1, 1004, "int255", 10_000),
    5: Config("deep100m_like", 100_000_000, 96, 10_000, 100, 6, 16, 256, 1.5, 0.05, 1005, "unit", 100_000),
}


def _rng(seed: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, stream])))


def _centres(cfg: Config) -> np.ndarray:
    r = _rng(cfg.seed, 0)
    d, C = cfg.d, cfg.comps
    if cfg.kind == "gauss_box":          # centres ~ U[0,100]^d
        return r.uniform(0.0, 100.0, size=(C, d)).astype(np.float32)
    if cfg.kind == "unit":               # mu = g/||g||, g ~ N(0, I_d)
        g = r.standard_normal((C, d), dtype=np.float32)
        return g / np.linalg.norm(g, axis=1, keepdims=True)
    if cfg.kind == "abs01":              # mu ~ |N(0, I_d)|
        return np.abs(r.standard_normal((C, d), dtype=np.float32))
    if cfg.kind == "int255":             # mu ~ U(-85, 200)^d
        return r.uniform(-85.0, 200.0, size=(C, d)).astype(np.float32)
    raise ValueError(cfg.kind)


def _draw(cfg: Config, mu: np.ndarray, m: int, stream: int) -> np.ndarray:
    r = _rng(cfg.seed, stream)
    out = np.empty((m, cfg.d), np.float32)
    for s in range(0, m, CHUNK):
        e = min(m, s + CHUNK)
        out[s:e] = _draw_chunk(cfg, mu, r, e - s)
    return out


def _draw_chunk(cfg: Config, mu: np.ndarray, r: np.random.Generator, m: int) -> np.ndarray:
    """The next m rows of the stream r (one chunk)."""
    comp = r.integers(0, cfg.comps, size=m)
    z = r.standard_normal((m, cfg.d), dtype=np.float32)
    x = mu[comp]
    if cfg.kind == "gauss_box":      # sigma = 5
        x = x + 5.0 * z
    elif cfg.kind == "unit":         # noise norm ~0.3 ||mu||, then unit-normalised
        x = x + np.float32(0.3 / math.sqrt(cfg.d)) * z
        x = x / np.linalg.norm(x, axis=1, keepdims=True)
    elif cfg.kind == "abs01":        # |mu + 0.3 z| (scaled to [0,1] afterwards)
        x = np.abs(x + 0.3 * z)
    elif cfg.kind == "int255":       # clip(round(mu + 20 z), 0, 255), ~30% zeros
        x = np.clip(np.rint(x + 20.0 * z), 0.0, 255.0)
    return x


def _cached(cfg: Config, n: int, make):
    """Experiments only: with DATAGEN_CACHE_DIR set, the data rows of (config, n) are kept in that
    directory as .npy (memory-mapped on reuse), so one job can run several benchmarks of the 100M
    config without regenerating it.  Unset (the default, and every driver-run command) = no cache."""
    import os
    d = os.environ.get("DATAGEN_CACHE_DIR")
    if not d or n < 5_000_000:
        return make()
    path = os.path.join(d, f"{cfg.name}_{cfg.seed}_{n}.npy")
    if os.path.exists(path):
        return np.load(path, mmap_mode="r")
    X = make()
    os.makedirs(d, exist_ok=True)
    np.save(path + ".tmp.npy", X)
    os.replace(path + ".tmp.npy", path)
    return X


def generate_rows(cfg: Config | int, lo: int, hi: int, n: int | None = None) -> np.ndarray:
    """Rows [lo, hi) of the config's data X (the same bytes as generate(cfg, n)["X"][lo:hi]); the
    stream is drawn up to hi but only the requested rows are kept (a point shard's memory)."""
    if isinstance(cfg, int):
        cfg = CONFIGS[cfg]
    n = cfg.n if n is None else n
    mu = _centres(cfg)
    r = _rng(cfg.seed, 1)
    out = np.empty((hi - lo, cfg.d), np.float32)
    for s in range(0, hi, CHUNK):
        e = min(n, s + CHUNK)
        blk = _draw_chunk(cfg, mu, r, e - s)
        a, b = max(s, lo), min(e, hi)
        if a < b:
            out[a - lo:b - lo] = blk[a - s:b - s]
    if cfg.kind == "abs01":
        raise ValueError("generate_rows: the abs01 family is scaled by the global data max")
    return out


def generate(cfg: Config | int, n: int | None = None, nq: int | None = None,
             with_sample_queries: int = 0):
    """Return dict(X [n][d] f32, Q [nq][d] f32, Qs [ns][d] f32, cfg).

    ``n``/``nq`` override the sizes (smaller parity cases of the same mixture)."""
    if isinstance(cfg, int):
        cfg = CONFIGS[cfg]
    n = cfg.n if n is None else n
    nq = cfg.nq if nq is None else nq
    mu = _centres(cfg)
    X = _cached(cfg, n, lambda: _draw(cfg, mu, n, 1))
    Q = _draw(cfg, mu, nq, 2)
    Qs = _draw(cfg, mu, with_sample_queries, 3) if with_sample_queries else None
    if cfg.kind == "abs01":
        s = float(X.max())
        X = np.clip(X / s, 0.0, 1.0)
        Q = np.clip(Q / s, 0.0, 1.0)
        if Qs is not None:
            Qs = np.clip(Qs / s, 0.0, 1.0)
    return {"X": np.ascontiguousarray(X), "Q": np.ascontiguousarray(Q), "Qs": Qs, "cfg": cfg}

