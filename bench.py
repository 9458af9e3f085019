#!/usr/bin/env python
"""Benchmark of the DET-LSH hot path on B200 (contract: see DESIGN.md "Measurement").

A step = one pass of the whole hot path over one batch of synthetic input:
detlsh_build over the configuration's n points (B0-B6) + detlsh_query of its nq queries
(Q0-Q8).  Inputs are device-resident before the timed region (X >> L2, so no L2 flush is
needed); timing uses CUDA events on the library's stream, max over ranks.

Default workload: configs[4] (n = 100M, d = 96, L = 6, beta = 0.05, 10,000 queries) -- the
largest BASELINE configuration, which fits one B200 (38.4 GB of data); `--config 2` selects
configs[1] (1M x 256), `--config 4` configs[3] (10M x 128).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl reference]

N > 1 runs under torchrun: points are sharded (strong scaling of the fixed config),
breakpoints are global (C1 all-gather), every rank answers every query with its
per-shard budget and the local top-k lists are all-gathered (NCCL) and merged on the
device (C2, k_merge_topk).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402

METRIC = "queries/s at recall@k>=0.9"


def load_rmin(cid: int, which: str = "bench") -> float:
    """The radius both arms run at: r_bench = r_min c^-m* (the operating point the ORACLE picked,
    tools/make_rmin.py --point: largest m with oracle recall >= 0.95 on held-out sample queries;
    SURVEY 8(d)), else the AMB-22 r_min itself."""
    e = json.load(open(os.path.join(ROOT, "bench_configs.json")))[str(cid)]
    return float(e["r_min"] if which == "amb22" else e.get("r_bench", e["r_min"]))


def rmin_info(cid: int) -> dict:
    e = json.load(open(os.path.join(ROOT, "bench_configs.json"))).get(str(cid))
    if e is None:
        return {"r_choice": "no oracle operating point recorded for this config (--r-value experiment)"}
    return {"r_min_amb22": e["r_min"], "bench_m": e.get("bench_m", 0),
            "bench_oracle_recall": e.get("bench_oracle_recall"),
            "r_choice": "r_min c^-m, m = largest with oracle recall@k >= 0.95 on 50 held-out sample queries "
                        "(tools/make_rmin.py --point; SURVEY 8(d))"}


def workload_desc(c) -> str:
    return (f"configs[{c_index(c)}] {c.name}: n={c.n:,} d={c.d} fp32, nq={c.nq}, k={c.k}, L={c.L}, K={c.K}, "
            f"N_r={c.N_r}, c={c.c}, beta={c.beta}")


def c_index(c) -> int:
    for i, v in datagen.CONFIGS.items():
        if v == c:
            return i - 1
    return -1


# ---------------------------------------------------------------- ground truth and quality (harness)
def exact_knn_sample(Xd, Xs: np.ndarray, lo: int, Q: np.ndarray, k: int, sel: np.ndarray, world: int = 1):
    """Exact kNN of Q[sel] (harness, not the library) over the point-sharded data: every rank screens
    its own rows (device copy Xd = host rows Xs = global ids [lo, lo + len)) in fp32 with torch on
    its GPU (8M-row blocks, TF32 off), re-ranks its k + 64 best per query in fp64 on the host (ties
    by id), and the ranks' local top-k lists are all-gathered and merged by (distance, id).
    Returns (ids, dists) [len(sel)][k] (every rank)."""
    import torch
    torch.backends.cuda.matmul.allow_tf32 = False
    extra = k + 64
    qs = torch.from_numpy(np.ascontiguousarray(Q[sel])).to(Xd.device)
    cands = []
    for s0 in range(0, Xd.shape[0], 1 << 23):
        blk = Xd[s0:s0 + (1 << 23), :Q.shape[1]]
        d2 = (blk * blk).sum(1)[None, :] - 2.0 * (qs @ blk.T)
        cands.append((torch.topk(d2, min(extra, blk.shape[0]), dim=1, largest=False).indices + s0).cpu())
    cand = torch.cat(cands, 1).numpy()
    kk = min(k, Xs.shape[0])
    ids = np.full((len(sel), k), -1, np.int64)
    dists = np.full((len(sel), k), np.inf, np.float64)
    for r in range(len(sel)):
        cid = np.unique(cand[r])
        d2 = ((Xs[cid].astype(np.float64) - Q[sel[r]].astype(np.float64)) ** 2).sum(1)
        o = np.lexsort((cid, d2))[:kk]
        ids[r, :kk], dists[r, :kk] = cid[o] + lo, np.sqrt(d2[o])
    if world > 1:
        import torch.distributed as dist
        ti, td = torch.from_numpy(ids).to(Xd.device), torch.from_numpy(dists).to(Xd.device)
        gi = [torch.empty_like(ti) for _ in range(world)]
        gd = [torch.empty_like(td) for _ in range(world)]
        dist.all_gather(gi, ti)
        dist.all_gather(gd, td)
        ai = torch.cat(gi, 1).cpu().numpy()
        ad = torch.cat(gd, 1).cpu().numpy()
        for r in range(len(sel)):
            o = np.lexsort((ai[r], ad[r]))[:k]
            ids[r], dists[r] = ai[r][o], ad[r][o]
    return ids, dists


def recall(ids: np.ndarray, gt: np.ndarray) -> float:
    k = gt.shape[1]
    return float(np.mean([len(set(ids[i].tolist()) & set(gt[i].tolist())) / k for i in range(len(gt))]))


def quality(ids, dists, gt_ids, gt_d, c2):
    """BASELINE.md 3 quality next to the throughput: recall@k vs exact kNN, the overall
    ratio mean_i ||q,o_i|| / ||q,o_i*||, and the c^2-k-ANN success rate of Theorem 2
    (every returned o_i within c^2 ||q, o_i*||)."""
    d = dists.astype(np.float64)
    ok = np.all(d <= c2 * gt_d * (1 + 1e-6), axis=1)
    pos = gt_d > 0
    ratio = np.where(pos, d / np.where(pos, gt_d, 1.0), 1.0).mean(1)
    return {"recall_at_k": recall(ids, gt_ids), "overall_ratio": float(ratio.mean()),
            "c2_success_rate": float(ok.mean()), "theorem2_bound": 0.5 - 1 / np.e, "queries": int(len(gt_ids))}


def oracle_agreement(cid: int, ids: np.ndarray, dists: np.ndarray, radius: str):
    """GPU top-k vs the ORACLE's own answers where the repo holds them for this workload
    (tests/golden/cfg5_oracle.npz: configs[4], the seeded 200-query subset, written by the
    oracle-only tools/make_cfg5_golden.py): recall vs the oracle's ids and the largest relative
    distance difference on common ids."""
    path = os.path.join(ROOT, "tests", "golden", "cfg5_oracle.npz")
    if cid != 5 or not os.path.exists(path):
        return None
    z = np.load(path)
    sel = z["sel"]
    key = "rbench" if radius == "bench" and "rbench_ids" in z.files else "rmin"
    if radius == "bench" and key != "rbench" and int(z["bench_m"]) != 0:
        return None
    oi, od = z[f"{key}_ids"], z[f"{key}_dists"]
    sel = sel[:len(oi)]
    gi, gd = ids[sel], dists[sel]
    worst = 0.0
    for q in range(len(sel)):
        m = {int(i): float(v) for i, v in zip(oi[q], od[q])}
        for i, v in zip(gi[q], gd[q]):
            if int(i) in m and m[int(i)] > 0:
                worst = max(worst, abs(float(v) - m[int(i)]) / m[int(i)])
    return {"recall_vs_oracle": recall(gi, oi), "max_rel_dist_diff": worst, "queries": int(len(sel)),
            "source": "tests/golden/cfg5_oracle.npz (oracle-only, seed 2005 subset)"}


# ---------------------------------------------------------------- clocks sampler
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) >= 9 for i in range(4) if r[5 + i].strip() == "Active"})
        load = [s for s in sm if s > 300] or sm
        return {"sm_mhz": float(np.median(load)) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------- roofline models
def peaks():
    p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else None
    if p:
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained"), "measured (MEASURED_PEAKS.json)"
    return 6650.0, 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


def kernel_models(c, steps: int, st, n_local: int, nq: int, ld: int):
    """Algorithmic work of all launches of each modelled kernel in the timed region
    (DESIGN.md §5).  `st` = per-query stats of one step (the computation is deterministic,
    every step does the same work)."""
    d, LK, K = c.d, c.L * c.K, c.K
    ns = datagen_ns(c, n_local)
    ncand = float(st["n_cand"].sum())
    # leaf boxes are read once per 16-query group and tree ("leaf-box bytes /
    # query-batch"); everything else per query
    # two-level filter (large n, library default n >= 64 * 2^K): the pair kernel bounds each listed
    # tile's leaves per query, so their boxes count per query (2K), not per 16-query group
    box_share = 1.0 if n_local >= 64 * (1 << K) else 1.0 / 16
    filt = float((st["leaves_tested"] * 2 * K * box_share + st["leaves_passed"] * 8 + st["subboxes_tested"] * 2 * K
                  + st["points_tested"] * K + st["points_passed"] * 12 + st["n_cand"] * 4).sum())
    lookups = float((st["points_tested"] * K + st["leaves_tested"] * K + st["subboxes_tested"] * K).sum())
    proj_bytes = n_local * (4 * ld + LK) + (ns + nq) * (4 * ld + 4 * LK)
    proj_flops = 2.0 * 2 * (n_local + ns + nq) * ((LK + 15) // 16 * 16) * ld      # x_hi and x_lo MMAs
    return {
        FILTER_UNIT: {"bytes": steps * filt, "smem_bytes": steps * lookups * 2,
                      "unit": ("per query: leaves_tested*2K (box bounds read by the query itself: the two-level "
                               "filter's tile and leaf bounds)" if box_share == 1.0 else
                               "per query: leaves_tested*2K/16 (leaf boxes read once per 16-query group, SURVEY 8(d) K5)")
                              + " + leaves_passed*8 + subboxes_tested*2K + points_tested*K + "
                              "points_passed*12 + new*4 B (K6, with the sub-box boxes the pair kernel "
                              "reads), over both filter kernels "
                              "(k_range_filter: tile/leaf bounds + dense tiles; k_leaf_points: sparse tiles' "
                              "points), timed together"},
        "k_verify_rows": {"bytes": steps * ncand * (4 * d + 8), "unit": "per candidate 4d+8 B (row + id + d2)"},
        "k_verify_gather": {"bytes": steps * ncand * (4 * d + 8),
                            "unit": "per candidate 4d+8 B (row + id + d2); all candidates of the step are counted "
                                    "here, so rounds verified on the tensor cores would inflate it (none at the "
                                    "bench point: every round takes the gather)"},
        # tensor-core verification: per round a masked X.Q^T over all n rows x the round's active
        # queries; 3 tf32 MMAs (x.q, x.q_lo, x_lo.q) per product; active query-rounds = sum of rounds
        "k_verify_tc": {"bytes": steps * ncand * (4 * d + 8),
                        "flops": steps * 3.0 * 2.0 * n_local * ld * float(st["rounds"].sum()),
                        "tensor_only": True,
                        "unit": "per candidate 4d+8 B (the gather it replaces); tensor work 3 x 2 n ld per active "
                                "query-round (3xTF32)"},
        "k_project_tc": {"bytes": steps * proj_bytes, "flops": steps * proj_flops,
                         "unit": "per row 4*ld B read + codes (LK B) or projections (4LK B) written"},
    }


def build_roofline(c, n_local: int, pts_per_s: float, hbm: float) -> dict:
    """Whole-build roofline (SURVEY 8(d) "Build total"): ~4d + 9 L K + 100 L bytes per point
    (X read once by the projection, codes written and re-read by the sort / split / gathers,
    ~100 B per point per tree of key-value sort traffic)."""
    bpp = 4 * c.d + 9 * c.L * c.K + 100 * c.L
    ach = pts_per_s * bpp / 1e9
    return {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s", "frac": round(ach / hbm, 4),
            "bytes_per_point": bpp, "points": n_local,
            "model": "4d + 9LK + 100L B per point (SURVEY 8(d) Build total) x points/s"}


FILTER_UNIT = "filter"      # k_range_filter or k_tile_pairs + k_leaf_points (one unit of work: Alg. 3)
FILTER_KERNELS = ("k_range_filter", "k_tile_pairs", "k_leaf_points")


def group_filter(prof):
    """Profile entries with the two filter kernels merged into one unit (their launches of
    k_range_filter counted as the unit's launches: one per tree per round)."""
    out, fl, fms, parts = {}, 0, 0.0, {}
    for k, (nl, ms) in prof.items():
        if k.startswith(FILTER_KERNELS):
            fms += ms
            parts[k] = round(ms, 4)
            fl = max(fl, nl)          # one launch of each per (batch, round, tree)
        else:
            out[k] = (nl, ms)
    if parts:
        out[FILTER_UNIT] = (max(fl, 1), fms)
    return out, parts


def roofline_entry(name, model, ms, hbm, bf16, clocks, launches=1, traffic=None):
    ach = model["bytes"] / (ms / 1e3) / 1e9
    if traffic and name == FILTER_UNIT:
        tr = sum(v for k, v in traffic.items() if k.startswith(FILTER_KERNELS)) or None
    else:
        tr = traffic.get(name) if traffic else None
    e = {"kernel": name, "bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
         "frac": round(ach / hbm, 4), "traffic": tr, "algorithmic_bytes_per_launch": round(model["bytes"] / launches),
         "ms": round(ms, 4), "ms_per_launch": round(ms / launches, 4), "unit_of_work": model["unit"]}
    if model.get("tensor_only"):
        tf = model["flops"] / (ms / 1e3) / 1e12
        pk = round(bf16 / 2, 1)
        e.update({"bound": "tensor", "achieved": round(tf, 1), "peak": pk, "unit": "TFLOP/s", "frac": round(tf / pk, 4),
                  "peak_note": "measured bf16 / 2 (TF32 nominal ratio); executed 3xTF32 MMA flops",
                  "gather_equivalent_GBps": round(ach, 1)})
        return e
    if "smem_bytes" in model:
        sm = (clocks.get("sm_mhz") or 1965.0) * 1e6
        smem_peak = 148 * 128 * sm / 1e9
        e["limiter"] = "shared-memory LUT lookups (codes and leaf boxes are L2-resident)"
        e["smem"] = {"achieved": round(model["smem_bytes"] / (ms / 1e3) / 1e9, 1), "peak": round(smem_peak, 1),
                     "unit": "GB/s", "peak_note": "148 SMs x 128 B/clk x SM clock (derived)",
                     "counted": "one 16-bit quantised term per (query, dim) lookup"}
    if "flops" in model:
        tf = model["flops"] / (ms / 1e3) / 1e12
        e["tensor"] = {"achieved": round(tf, 1), "peak": round(bf16 / 2, 1), "unit": "TFLOP/s",
                       "peak_note": "measured bf16 / 2 (TF32 nominal ratio), 2 MMAs (x_hi, x_lo) per k-step"}
    return e


def traffic_path(cid: int) -> str:
    """This workload's `ncu --set full` summary (profiles/traffic_c<cid>.json, written by
    tools/ncu_summary.py from a capture of the same configuration), else the generic one."""
    p = os.path.join(ROOT, "profiles", f"traffic_c{cid}.json")
    return p if os.path.exists(p) else os.path.join(ROOT, "profiles", "traffic.json")


def load_traffic(cid: int):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of each modelled
    kernel, from the committed ncu capture of this configuration."""
    path = traffic_path(cid)
    if not os.path.exists(path):
        return None
    return {k: v["dram_bytes_per_launch"] for k, v in json.load(open(path)).get("kernels", {}).items()}


def load_pipes(cid: int):
    """ncu ALU-pipe and issue utilisation (% of peak) per kernel, from the same capture."""
    path = traffic_path(cid)
    if not os.path.exists(path):
        return {}
    return {k: {"alu_pct": v.get("alu_pct"), "issue_pct": v.get("issue_pct")}
            for k, v in json.load(open(path)).get("kernels", {}).items() if v.get("alu_pct") is not None}


def datagen_ns(c, n):
    return min(n, max(int(np.ceil(c.sample_frac * n)), 32 * c.N_r))


# ---------------------------------------------------------------- reference arm (the oracle)
ORACLE_FULL_MAX = 2_000_000      # configs up to this n: the oracle indexes all points
ORACLE_SAMPLE_N = 1_000_000      # larger configs: the oracle indexes this prefix of the data (a bounded sample)
_ORC = {}                        # forked oracle workers inherit the index


def oracle_points(cfg) -> int:
    return cfg.n if cfg.n <= ORACLE_FULL_MAX else ORACLE_SAMPLE_N


def oracle_sample_desc(cfg, n_o: int) -> str:
    if n_o == cfg.n:
        return f"oracle (single-thread fp64 C) index over all {cfg.n:,} points"
    return (f"oracle (single-thread fp64 C) index over the first {n_o:,} of the {cfg.n:,} points "
            f"(a bounded sample: its per-query work and budget beta n + k are those of a {n_o:,}-point index)")


def _orc_query_one(i):
    c = _ORC["cfg"]
    t = time.perf_counter()
    _ORC["ix"].query(_ORC["Q"][i:i + 1], c.k, c.c, _ORC["r"], c.beta)
    return time.perf_counter() - t


def run_reference(args, cfg):
    from oracle import oracle as O
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    r_min = load_rmin(args.config, args.radius)
    n_o = oracle_points(cfg)
    D = datagen.generate(cfg, n=n_o)
    X, Q = D["X"], D["Q"]
    t0 = time.perf_counter()
    ix = O.Index(X, cfg.L, cfg.K, cfg.N_r, cfg.index_seed, cfg.max_size, cfg.sample_frac)
    build_s = time.perf_counter() - t0
    per_step = args.ref_queries
    rng = np.random.default_rng(0)
    times = []
    for s in range(args.warmup + args.steps):
        sel = rng.choice(cfg.nq, per_step, replace=False)
        t = time.perf_counter()
        ix.query(Q[sel], cfg.k, cfg.c, r_min, cfg.beta)
        if s >= args.warmup:
            times.append(time.perf_counter() - t)
    qps = per_step * len(times) / sum(times)
    line = {"impl": "reference", "metric": METRIC, "value": qps, "unit": "queries/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": workload_desc(cfg), "r_min": r_min, **rmin_info(args.config)},
            "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": 1, "kind": "oracle",
                             "sample": f"{oracle_sample_desc(cfg, n_o)}; {per_step} random queries of the {cfg.nq} "
                                       f"per step (oracle build {n_o / build_s:.0f} points/s, 1 core)"},
            "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg, Q, r, nqs: int) -> dict:
    """The oracle as it stands on the box's host cores, on a bounded sample of the workload:
    build points/s on 1 core; queries/s on 1 core and with P = nproc forked processes answering
    disjoint queries of the same index ("oracle x P cores")."""
    import multiprocessing as mp
    from oracle import oracle as O
    n_o = oracle_points(cfg)
    Xo = datagen.generate(cfg, n=n_o, nq=1)["X"]
    t0 = time.perf_counter()
    ix = O.Index(Xo, cfg.L, cfg.K, cfg.N_r, cfg.index_seed, cfg.max_size, cfg.sample_frac)
    tb = time.perf_counter() - t0
    sel = np.random.default_rng(1).choice(cfg.nq, nqs, replace=False)
    _ORC.update(ix=ix, Q=Q, cfg=cfg, r=r)
    t1 = [_orc_query_one(int(i)) for i in sel]
    P = os.cpu_count() or 1
    sel_p = np.random.default_rng(3).choice(cfg.nq, min(cfg.nq, 2 * P), replace=False)
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(P) as pool:
        pool.map(_orc_query_one, [int(i) for i in sel_p], chunksize=1)
    wall = time.perf_counter() - t0
    _ORC.clear()
    return {"value": nqs / sum(t1), "unit": "queries/s", "cores": 1, "kind": "oracle",
            "sample": f"{oracle_sample_desc(cfg, n_o)}; {nqs} of the {cfg.nq} queries at the bench radius",
            "build_points_per_s": n_o / tb, "seconds": tb + sum(t1) + wall,
            "oracle_x_P_cores": {"value": len(sel_p) / wall, "unit": "queries/s", "cores": P,
                                 "how": f"{P} forked oracle processes answering {len(sel_p)} disjoint queries "
                                        "of the same index (embarrassingly parallel, no code change)"}}


# ---------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-queries", type=int, default=4)
    ap.add_argument("--cpu-queries", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--proj-impl", type=int, default=None)
    ap.add_argument("--recall-queries", type=int, default=200)
    ap.add_argument("--radius", default="bench", choices=["bench", "amb22"],
                    help="bench: the oracle-chosen operating point r_bench; amb22: the AMB-22 r_min itself")
    ap.add_argument("--r-value", type=float, default=None,
                    help="experiments only: run at this radius instead of bench_configs.json's")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    cfg = datagen.CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist
    import paper_2603_24920_b200 as P
    from paper_2603_24920_b200 import dist as PD

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    r_min = args.r_value if args.r_value is not None else load_rmin(args.config, args.radius)
    lo, hi = PD.shard_range(cfg.n, world, rank)
    if world == 1 or cfg.kind == "abs01":
        Dd = datagen.generate(cfg)
        Xs, Q = np.ascontiguousarray(Dd["X"][lo:hi]), Dd["Q"]
        del Dd
    else:       # each rank holds only its shard's rows (configs[4]: 38.4 GB in all)
        Xs = datagen.generate_rows(cfg, lo, hi)
        Q = datagen.generate(cfg, n=1)["Q"]
    Xd = torch.from_numpy(Xs).cuda()
    Qd = torch.from_numpy(Q).cuda()
    stream = torch.cuda.current_stream()
    opts = P.default_opts(stream=stream.cuda_stream, borrow_data=1)
    if args.proj_impl is not None:
        opts.proj_impl = args.proj_impl
    n_local = hi - lo

    def barrier():
        if world > 1:
            dist.barrier()

    def build():
        if world > 1:
            return PD.sharded_build(Xd, lo, cfg.n, cfg.L, cfg.K, cfg.N_r, cfg.index_seed, opts)
        return P.detlsh_build(Xd, cfg.L, cfg.K, cfg.N_r, cfg.index_seed, opts=opts)

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    results = {}

    def step(timed: bool):
        e0, e1, e2 = ev(), ev(), ev()
        e0.record(stream)
        idx = build()
        e1.record(stream)
        ids, dists, st = idx.query(Qd, cfg.k, cfg.c, r_min, cfg.beta, opts=opts, stats=True)
        if world > 1:
            ids, dists = PD.merge_shard_topk(ids, dists, cfg.k)
        e2.record(stream)
        results["ids"], results["dists"], results["stats"] = ids, dists, st
        idx.free()
        return e0, e1, e2

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clk = Clocks(local)
    clk.start()
    time.sleep(0.3)
    P.profile_reset()
    # CUDA events in the timed region around the dominant unit's kernels only (every timed
    # launch adds an event pair to the stream); the other modelled kernels are timed in one
    # extra, untimed step below
    P.profile_filter("k_range_filter,k_tile_pairs,k_leaf_points")
    P.profile_enable(True)
    l0 = P.launch_count()
    evs = [step(True) for _ in range(args.steps)]
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    launches = P.launch_count() - l0
    P.profile_enable(False)
    prof = P.profile_read()
    clocks = clk.stop()
    P.profile_reset()
    P.profile_filter("k_verify,k_project_tc,k_topk")
    P.profile_enable(True)
    step(False)
    torch.cuda.synchronize()
    P.profile_enable(False)
    prof_extra = P.profile_read()          # one untimed step: verification, projection, top-k
    build_ms = sum(a.elapsed_time(b) for a, b, _ in evs)
    query_ms = sum(b.elapsed_time(c) for _, b, c in evs)
    step_ms = sum(a.elapsed_time(c) for a, _, c in evs)
    t = torch.tensor([build_ms, query_ms, step_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    build_ms, query_ms, step_ms = t.tolist()

    st = results["stats"]

    # e2e through the public API with host (pinned) buffers: H2D of the queries and D2H of the results inside
    Qh = torch.from_numpy(Q).pin_memory()
    idh = torch.empty((cfg.nq, cfg.k), dtype=torch.int64).pin_memory()
    dh = torch.empty((cfg.nq, cfg.k), dtype=torch.float32).pin_memory()
    idx = build()
    e2e_ms = []
    for s in range(args.warmup + args.steps):
        a, b = ev(), ev()
        a.record(stream)
        idx.query(Qh.numpy(), cfg.k, cfg.c, r_min, cfg.beta, opts=opts, out_ids=idh.numpy(), out_dists=dh.numpy())
        b.record(stream)
        b.synchronize()
        if s >= args.warmup:
            e2e_ms.append(a.elapsed_time(b))
    idx.free()
    te = torch.tensor([float(np.mean(e2e_ms))], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)

    sel = np.random.default_rng(2).choice(cfg.nq, min(args.recall_queries, cfg.nq), replace=False)
    gt, gt_d = exact_knn_sample(Xd, Xs, lo, Q, cfg.k, sel, world)
    if rank == 0:
        ids, dists = results["ids"], results["dists"]
        ids = ids.cpu().numpy() if torch.is_tensor(ids) else ids
        dists = dists.cpu().numpy() if torch.is_tensor(dists) else dists
        qual = quality(ids[sel], dists[sel], gt, gt_d, cfg.c ** 2)
        rec = qual["recall_at_k"]
        agree = oracle_agreement(args.config, ids, dists, args.radius)
        hbm, bf16, bf16s, peak_src = peaks()
        kern = {k: {"launches": v[0], "ms": round(v[1], 4)} for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])}
        kern.update({k: {"launches": v[0], "ms": round(v[1] * args.steps, 4), "from": "one extra untimed step, x steps"}
                     for k, v in prof_extra.items()})
        units, filter_parts = group_filter(prof)
        # per-step ms of every unit: the filter from the timed region, the rest from the extra step
        unit_step_ms = {k: v[1] / args.steps for k, v in units.items()}
        unit_step_ms.update({k: v[1] for k, v in prof_extra.items()})
        dom = max(unit_step_ms.items(), key=lambda kv: kv[1])[0] if unit_step_ms else None
        models = kernel_models(cfg, args.steps, st, n_local, cfg.nq, (cfg.d + 7) // 8 * 8)
        models1 = kernel_models(cfg, 1, st, n_local, cfg.nq, (cfg.d + 7) // 8 * 8)
        roofs = []
        traffic = load_traffic(args.config)
        all_units = [(k, v, models, "timed region") for k, v in units.items()] + \
                    [(k, v, models1, "extra untimed step") for k, v in prof_extra.items()]
        for kname, (nl_, ms), mset, src in sorted(all_units, key=lambda x: -unit_step_ms[x[0]]):
            for prefix, model in mset.items():
                if kname.startswith(prefix):
                    e = roofline_entry(kname, model, ms, hbm, bf16, clocks, nl_, traffic)
                    e["timed_in"] = src
                    if kname == FILTER_UNIT:
                        e["parts_ms"] = filter_parts
                        pipes = load_pipes(args.config)
                        e["limiter"] = (f"see ncu_pipes (ALU-pipe and issue utilisation) and traffic (DRAM bytes "
                                        f"per launch) from the committed capture {os.path.basename(traffic_path(args.config))}")
                        e["ncu_pipes"] = {k: v for k, v in pipes.items() if k.startswith(FILTER_KERNELS)}
                    roofs.append(e)
                    break
        roof = next((r for r in roofs if r["kernel"] == dom), None)
        if roof is not None:
            roof["share_of_step"] = round(unit_step_ms[dom] * args.steps / step_ms, 4)
            roof["peak_source"] = peak_src
        line = {
            "metric": METRIC, "value": cfg.nq * args.steps / (query_ms / 1e3), "unit": "queries/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": workload_desc(cfg), "n": cfg.n, "d": cfg.d, "nq": cfg.nq, "k": cfg.k,
                       "r_min": r_min, **rmin_info(args.config), "parallelism": f"point-sharded x{world}",
                       "l2": f"no flush: X ({cfg.n * cfg.d * 4 / 1e9:.2f} GB) and the rebuilt index exceed L2 (126 MB)",
                       "proj_impl": int(opts.proj_impl)},
            "recall_at_k": rec, "recall_queries": int(len(sel)),
            "quality": qual, "vs_oracle": agree,
            "query_ms_per_step": query_ms / args.steps,
            "build": {"points_per_s": cfg.n * args.steps / (build_ms / 1e3), "ms_per_step": build_ms / args.steps,
                      "roofline": build_roofline(cfg, n_local, cfg.n * args.steps / (build_ms / 1e3) / world, hbm)},
            "candidates_per_query": float(st["n_cand"].mean()),
            "stop_reasons": np.bincount(st["reason"], minlength=3).tolist(),
            "filter_counts_per_query": {k_: float(st[k_].mean()) for k_ in
                                        ("leaves_tested", "leaves_passed", "points_tested", "points_passed",
                                         "subboxes_tested")},
            "roofline": roof,
            "rooflines": roofs,
            "e2e": {"value": cfg.nq / (float(te.item()) / 1e3), "unit": "queries/s",
                    "h2d_bytes_per_step": int(Q.nbytes), "d2h_bytes_per_step": int(cfg.nq * cfg.k * 12),
                    "how": "detlsh_query with pinned host query/output buffers (copies inside the timed call)"},
            "gpu_launches": int(launches), "clocks": clocks, "kernels": kern,
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(cfg, Q, r_min, args.cpu_queries)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
