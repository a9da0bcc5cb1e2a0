"""Library baseline for the phase retrieval matvec (NOT the product path): the same operator
D x = x / sqrt(n) + sum_j kappa_j M_j^* (w_j o M_j x) written with torch.fft (cuFFT) and torch elementwise
kernels on one B200, timed with CUDA events, next to the fused FFT kernels of csrc/phase.cu
(scg_pr_apply_D's three kernels).  Usage: python tools/phase_cufft_baseline.py [n] [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import scg_inputs as si
from oracle import phase as ph
from paper_1912_02949_b200 import phase as prm

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
I = si.phase_instance(n, seed=4)
kappa, _ = ph.scaling(I.psi, I.b, 3.0 * n)
rng = np.random.default_rng(0)
x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
w = rng.standard_normal((12, n))
dev = torch.device("cuda")
psi = torch.from_numpy(I.psi).to(dev)
cpsi = psi.conj()
kw = torch.from_numpy(kappa[:, None] * w).to(dev)
xt = torch.from_numpy(x).to(dev)
rsn = 1.0 / np.sqrt(n)


def apply_torch(xv):
    Y = torch.fft.fft(cpsi * xv[None, :], dim=1)
    Y = Y * kw
    Z = torch.fft.ifft(Y, dim=1) * n
    return xv * rsn + (psi * Z).sum(dim=0)


for _ in range(3):
    yt = apply_torch(xt)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    yt = apply_torch(xt)
e1.record()
e1.synchronize()
torch_us = 1e3 * e0.elapsed_time(e1) / reps
ref = ph.apply_D(I.psi, kappa, w, x)
err_t = float(np.max(np.abs(yt.cpu().numpy() - ref)) / np.max(np.abs(ref)))

g = prm.PhaseRetrieval(I.psi, I.b, R=5, seed=4, profile=True)
yg = g.apply_D(w, x)
err_g = float(np.max(np.abs(yg - ref)) / np.max(np.abs(ref)))
g.step(3)
g.reset_stats()
g.step(3)
st = {s["name"]: s for s in g.kernel_stats()}
ours_us = sum(1e3 * st[k]["total_ms"] / st[k]["launches"] for k in ("k_pr_f1", "k_pr_b", "k_pr_c"))
print({"n": n, "torch_cufft_matvec_us": round(torch_us, 1), "fused_fft_matvec_us": round(ours_us, 1),
       "speedup": round(torch_us / ours_us, 2), "rel_err_torch": err_t, "rel_err_fused": err_g,
       "note": "torch.fft (cuFFT, complex128) + torch elementwise kernels vs k_pr_f1 + k_pr_b + k_pr_c"})
