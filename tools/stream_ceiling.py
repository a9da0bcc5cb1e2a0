"""Achievable HBM bandwidth of the access mixes of the hot-path kernels, measured with torch's
own elementwise kernels (fp64, 2^24 rows like c3): 1 read + 1 write (copy), 3 reads + 1 write
(k_lanczos_b's pattern: a, X_i, X_{i-1} -> X_{i+1})."""
import json
import torch

n = 1 << 24
dev = "cuda"
a, b, c, o = (torch.randn(n, dtype=torch.float64, device=dev) for _ in range(4))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def bench(fn, nbytes, reps=50):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    t = ts[len(ts) // 2] / 1e3
    return nbytes / t / 1e9, t * 1e6


res = {}
res["copy_1r1w"] = bench(lambda: o.copy_(a), 16 * n)
res["addcmul_3r1w"] = bench(lambda: torch.addcmul(a, b, c, out=o), 32 * n)
res["add_2r1w"] = bench(lambda: torch.add(a, b, out=o), 24 * n)
print(json.dumps({k: {"GB/s": round(v[0], 1), "us": round(v[1], 1)} for k, v in res.items()}))
