"""Per-kernel device time of one index build (experiments): build once to warm up, then build
again with the library's per-launch event timing on, and print the kernels by total time plus
the wall time of the untimed build.  Usage: python tools/build_prof.py CFG"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen  # noqa: E402
import paper_2603_24920_b200 as P  # noqa: E402

cid = int(sys.argv[1])
D = datagen.generate(cid, nq=1)
c = D["cfg"]
st_ = torch.cuda.current_stream()
Xd = torch.from_numpy(D["X"]).cuda()
o = P.default_opts(borrow_data=1, stream=st_.cuda_stream)
times = []
for i in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st_)
    g = P.detlsh_build(Xd, c.L, c.K, c.N_r, c.index_seed, opts=o)
    b.record(st_)
    b.synchronize()
    times.append(a.elapsed_time(b))
    g.free()
P.profile_reset()
P.profile_filter("")
P.profile_enable(True)
g = P.detlsh_build(Xd, c.L, c.K, c.N_r, c.index_seed, opts=o)
torch.cuda.synchronize()
P.profile_enable(False)
prof = P.profile_read()
tot = sum(v[1] for v in prof.values())
print(json.dumps({"config": cid, "build_ms": times, "points_per_s": c.n / (min(times) / 1e3),
                  "kernel_sum_ms": round(tot, 3),
                  "kernels": {k: [v[0], round(v[1], 3)] for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])}}))
