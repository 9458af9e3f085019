"""Projection + encode timing at a configuration's shape (device-resident Gaussian X): the build's
k_project_tc launches timed by the library's own CUDA-event profile, per process (the kernel's
experiment switches DETLSH_PROJ_TA / DETLSH_PROJ_DEBUG are read once per process).
Usage: python tools/proj_ab.py N D L K [reps]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_24920_b200 as P  # noqa: E402

n, d, L, K = (int(v) for v in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
g0 = torch.Generator(device="cuda").manual_seed(1)
X = torch.randn(n, d, device="cuda", generator=g0)
tag = f"TA={os.environ.get('DETLSH_PROJ_TA', '0')} DBG={os.environ.get('DETLSH_PROJ_DEBUG', '0')}"
for rep in range(reps):
    P.profile_reset()
    P.profile_filter("k_project_tc")
    P.profile_enable(True)
    g = P.detlsh_build(X, L, K, 256, 7, opts=P.default_opts(borrow_data=1))
    torch.cuda.synchronize()
    P.profile_enable(False)
    prof = P.profile_read()
    g.free()
    del g
    for k, (nl, ms) in prof.items():
        gb = n * d * 4 / 1e9 + n * L * K / 1e9
        print(f"{tag} n={n} d={d} LK={L * K} rep {rep}: {k} launches {nl} total {ms:.3f} ms "
              f"(X + codes {gb:.2f} GB -> {gb / ms:.2f} TB/s over all launches)", flush=True)
