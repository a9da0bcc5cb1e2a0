import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
import scg_inputs as si
from oracle import phase as ph
from paper_1912_02949_b200 import phase as pr
import torch
n = int(sys.argv[1]); T = int(sys.argv[2]); flags = int(sys.argv[3]) if len(sys.argv) > 3 else 0
I = si.phase_instance(n, seed=0)
g = pr.PhaseRetrieval(I.psi, I.b, R=5, seed=0, profile=True, flags=flags)
print("scalars", g.scalars())
g.step(1); torch.cuda.synchronize(); g.reset_stats()
t0 = time.time(); g.step(T); torch.cuda.synchronize(); dt = time.time() - t0
print(f"flags={flags} n={n} T={T} (after 1 warm-up iteration) {T/dt:.1f} it/s")
for k in g.kernel_stats():
    if k["launches"]:
        avg = k["total_ms"] / k["launches"] * 1e3
        print(f"{k['name']:20s} {k['launches']:6d} {avg:10.1f} us  {k['bytes_per_launch']/avg/1e3 if avg>0 else 0:8.1f} GB/s")
