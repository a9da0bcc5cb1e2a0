"""Wall-clock breakdown of the end-to-end job through the public API (c3 by default): init, T steps,
and each output call.  python tools/e2e_breakdown.py [config] [T]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1912_02949_b200 as scg
import scg_inputs as si

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 25
L = si.laplacian(cfg)
c = si.CONFIGS[cfg]
for rep in range(2):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    s = scg.SketchyCGAL(L, R=c["R"], seed=c["seed"], debug_log=(rep == 1))
    s.synchronize(); t.append(time.perf_counter())
    s.step(T); s.synchronize(); t.append(time.perf_counter())
    lg = s.iter_log(); t.append(time.perf_counter())
    _, lam, _ = s.reconstruct(want_U=False); s.synchronize(); t.append(time.perf_counter())
    obj = s.objective(); t.append(time.perf_counter())
    feas = s.feasibility(); t.append(time.perf_counter())
    chi, w = s.round(); t.append(time.perf_counter())
    s.close()
    names = ["init", "steps", "iter_log", "reconstruct", "objective", "feasibility", "round"]
    print(rep, {k: round(t[i + 1] - t[i], 4) for i, k in enumerate(names)}, flush=True)
