"""Diagnostic: query wall/device time under bench-like variants (stats, profiling, clocks sampler)."""
import os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import datagen, paper_2603_24920_b200 as P
D = datagen.generate(2)
c = D['cfg']
Xd = torch.from_numpy(D['X']).cuda(); Qd = torch.from_numpy(D['Q']).cuda()
st = torch.cuda.current_stream()
o = P.default_opts(borrow_data=1, stream=st.cuda_stream)
rmin = 1.1248388401842566
def run(tag, stats=False, prof=False, rebuild=True, n=6):
    g = P.detlsh_build(Xd, c.L, c.K, c.N_r, c.index_seed, opts=o)
    ts = []
    for it in range(n):
        if rebuild and it:
            g.free(); g = P.detlsh_build(Xd, c.L, c.K, c.N_r, c.index_seed, opts=o)
        if prof: P.profile_enable(True)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        t = time.perf_counter(); a.record(st)
        r = g.query(Qd, c.k, c.c, rmin, c.beta, opts=o, stats=stats)
        b.record(st); b.synchronize(); w = time.perf_counter() - t
        if prof: P.profile_enable(False)
        ts.append((a.elapsed_time(b), w * 1e3))
    g.free()
    print(tag, ' '.join(f'{x:.1f}/{y:.1f}' for x, y in ts), flush=True)
run('plain(no rebuild)', rebuild=False)
run('plain+rebuild')
run('stats')
run('stats+prof')
smi = subprocess.Popen(['nvidia-smi', '--query-gpu=clocks.sm', '--format=csv,noheader', '-lms', '100'], stdout=subprocess.DEVNULL)
run('stats+prof+smi')
smi.terminate()
run('after smi')
