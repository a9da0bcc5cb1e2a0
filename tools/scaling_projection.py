"""Projection of multi-GPU strong scaling from EMULATED shards (no multi-GPU box in this pool).

P row shards of configs[3] run inside one context on one B200 (the same kernels, halo peer
stores and mailbox collectives as one process per GPU; launched in turn on one stream).  The
sampled CUDA-event time of every kernel class, divided by the P shards that launched it, is
the per-GPU device time of one rank; the projection adds, per collective, a measured-nowhere
allowance (NVLINK_US below) for the flag round trip over NVLink.  This is a MODEL, printed as
such, not a multi-GPU measurement.
Usage: python tools/scaling_projection.py [P ...]   (default 1 2 4)"""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1912_02949_b200 as scg
import scg_inputs as si

NVLINK_US = 3.0  # assumed flag round trip per collective (publish + acquire over NVSwitch)
INLINE = os.environ.get("INLINE", "0") == "1"  # SCG_INLINE_PULL
cfg = os.environ.get("CFG", "c3")
L = si.laplacian(cfg)
c = si.CONFIGS[cfg]
W, K = 3, int(os.environ.get("STEPS", "60"))
res = {}
for P in [int(a) for a in sys.argv[1:]] or [1, 2, 4]:
    # (a) the emulated stream's device time without per-kernel events (CUDA events around step(K) only):
    # the P shards run in turn on one stream, so device time / P is one rank's device time
    st0 = torch.cuda.Stream()
    s = scg.SketchyCGAL(L, R=c["R"], seed=c["seed"], profile=False, shards=P, side_rng=False,
                        stream=ctypes.c_void_p(st0.cuda_stream), inline_pull=INLINE)
    s.step(W)
    s.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st0)
    s.step(K)
    e1.record(st0)
    e1.synchronize()
    s.synchronize()
    dev_ms = e0.elapsed_time(e1)
    s.close()
    # (b) per-kernel events for the breakdown (the events add a fixed cost to every launch)
    # the start vector drawn inside k_dual_sketch at every P (the side-stream draw of one GPU overlaps
    # other kernels, which a sum of per-kernel times cannot represent)
    s = scg.SketchyCGAL(L, R=c["R"], seed=c["seed"], profile=True, shards=P, side_rng=False, inline_pull=INLINE)
    s.step(W)
    s.synchronize()
    s.reset_stats()
    t0 = time.perf_counter()
    s.step(K)
    s.synchronize()
    wall = time.perf_counter() - t0
    st = {k["name"]: k for k in s.kernel_stats() if k["launches"] > 0}
    per_gpu_ms = 0.0
    for name, k in st.items():
        per_gpu_ms += k["total_ms"] / (P if name != "pull_collective" else P)
    pulls = st.get("pull_collective", {"launches": 0})["launches"] / max(P, 1)
    if INLINE and P > 1:  # collectives pulled inside the Lanczos kernels still cross NVLink once each
        pulls += (st.get("lanczos_a_spmv_dot", {"launches": 0})["launches"]
                  + st.get("lanczos_b_axpy_norm", {"launches": 0})["launches"]) / max(P, 1)
    proj_ms = per_gpu_ms + pulls * NVLINK_US / 1e3
    res[P] = {"emulated_wall_s": round(wall, 3), "per_gpu_device_ms": round(per_gpu_ms, 2),
              "stream_device_ms_per_rank": round(dev_ms / P, 2),
              "projected_stream_ms": round(dev_ms / P + pulls * NVLINK_US / 1e3, 2),
              "collectives": int(pulls), "projected_ms": round(proj_ms, 2),
              "projected_it_per_s": round(K / (proj_ms / 1e3), 2),
              "kernels_us_per_launch": {n: round(1e3 * k["total_ms"] / k["launches"], 1) for n, k in st.items()}}
    s.close()
    torch.cuda.empty_cache()
base = res[min(res)]["projected_it_per_s"]
bstream = res[min(res)]["projected_stream_ms"]
for P, r in res.items():
    r["projected_strong_efficiency"] = round(r["projected_it_per_s"] / (base * P), 3)
    r["projected_stream_efficiency"] = round(bstream / (P * r["projected_stream_ms"]), 3)
print(json.dumps({"config": cfg, "window": [W + 1, W + K], "nvlink_us_per_collective_assumed": NVLINK_US,
                  "inline_pull": INLINE,
                  "model": "per-GPU device time of the emulated shards + assumed NVLink flag latency per collective; "
                           "projected_stream_*: the emulated stream's device time (no per-kernel events) / P, "
                           "projected_*: the sum of per-kernel event times / P",
                  "P": res}, indent=1))
