"""Summarise ncu exports for profiles/ (run here, no GPU needed).

  python tools/ncu_summary.py launches <launches.csv>            -> share-of-time table (markdown)
  python tools/ncu_summary.py full <prof.ncu-rep> <out.json>      -> key counters per launch + traffic.json

traffic.json maps the library's profile names (DL_LAUNCH names, what bench.py sees) to the DRAM
bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the captured launches."""
import collections
import csv
import json
import subprocess
import sys

PROFILE_NAME = {"k_range_filter": "k_range_filter_sel", "k_verify_tc": "k_verify_tc", "k_project_tc": "k_project_tc",
                "k_topk": "k_topk", "k_verify_rows": "k_verify_rows", "k_verify_gather": "k_verify_gather_sel",
                "k_collect_cands": "k_collect_cands", "k_count_new": "k_count_new", "k_leaf_points": "k_leaf_points_sel",
                "k_tile_pairs": "k_tile_pairs"}
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
         "ms": 1.0, "msecond": 1.0, "s": 1e3, "nsecond": 1e-6}


def short(name):
    base = name.split("(")[0].replace("void ", "").strip()
    return base.split("::")[-1]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1.0)
        k = short(d["Kernel Name"])
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    print("| kernel | launches | ms | share |\n|---|---|---|---|")
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        if ms / tot >= 0.002:
            print(f"| {k} | {n} | {ms:.3f} | {100 * ms / tot:.1f}% |")
    print(f"| total | {sum(v[0] for v in agg.values())} | {tot:.3f} | 100% |")


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    res = []
    for r in data:
        e = {"kernel": short(r[idx["Kernel Name"]])}
        for k in KEYS:
            if k in idx and r[idx[k]] not in ("", "n/a"):
                try:
                    v = float(r[idx[k]].replace(",", ""))
                except ValueError:
                    continue
                u = units[idx[k]]
                if u in ("byte", "Kbyte", "Mbyte", "Gbyte", "Tbyte"):
                    v *= SCALE[u]
                    u = "byte"
                if k == "gpu__time_duration.sum":
                    v *= SCALE.get(u, 1.0)
                    u = "ms"
                e[k] = v
        res.append(e)
    traffic = {}
    for e in res:
        base = e["kernel"].split("<")[0]
        name = PROFILE_NAME.get(base)
        if name and "dram__bytes_read.sum" in e:
            t = traffic.setdefault(name, {"launches": [], "dram_bytes_per_launch": 0})
            t["launches"].append({"ms": e.get("gpu__time_duration.sum"),
                                  "dram_bytes": e["dram__bytes_read.sum"] + e.get("dram__bytes_write.sum", 0),
                                  "alu_pct": e.get("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
                                  "issue_pct": e.get("smsp__issue_active.avg.pct_of_peak_sustained_active")})
    for name, t in traffic.items():
        t["dram_bytes_per_launch"] = round(sum(x["dram_bytes"] for x in t["launches"]) / len(t["launches"]))
        for key in ("alu_pct", "issue_pct"):
            vals = [x[key] for x in t["launches"] if x.get(key) is not None]
            if vals:
                t[key] = round(sum(vals) / len(vals), 1)
    json.dump({"launches": res}, open(out, "w"), indent=1)
    return traffic


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        tr = full(sys.argv[2], sys.argv[3])
        if len(sys.argv) > 4:
            json.dump({"source": sys.argv[2], "kernels": tr}, open(sys.argv[4], "w"), indent=1)
        print(json.dumps(tr, indent=1)[:3000])
