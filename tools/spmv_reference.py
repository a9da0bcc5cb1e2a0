"""Library reference point for the c3 SpMV: torch CSR (cuSPARSE) fp64 matvec y = A x on the same
off-diagonal pattern (input order), plus the diagonal term, timed with CUDA events; bytes
counted like k_lanczos_a's algorithmic model (int32 col + fp64 val per entry, int32 row pointer,
x read once, diagonal and y)."""
import json
import sys
import os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scg_inputs as si

L = si.laplacian(sys.argv[1] if len(sys.argv) > 1 else "c3")
n = L.n
rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(L.row_ptr))
off = L.col != rows
rp = np.zeros(n + 1, dtype=np.int64)
np.cumsum(np.bincount(rows[off], minlength=n), out=rp[1:])
dev = "cuda"
A = torch.sparse_csr_tensor(torch.from_numpy(rp.astype(np.int32)), torch.from_numpy(L.col[off].astype(np.int32)),
                            torch.from_numpy(-L.val[off]), size=(n, n), device=dev)
x = torch.randn(n, dtype=torch.float64, device=dev)
d = torch.randn(n, dtype=torch.float64, device=dev)
y = torch.empty_like(x)
nnz = int(off.sum())


def run():
    torch.addcmul(torch.mv(A, x), d, x, out=y)


run()
torch.cuda.synchronize()
ts = []
for _ in range(30):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.mv(A, x)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
t = ts[len(ts) // 2] / 1e3
bytes_model = 12.0 * nnz + 4.0 * (n + 1) + 8.0 * n + 8.0 * n  # matrix + x once + y (no diagonal)
print(json.dumps({"config": sys.argv[1] if len(sys.argv) > 1 else "c3", "n": n, "nnz": nnz,
                  "cusparse_mv_us": round(t * 1e6, 1), "algorithmic_GB/s": round(bytes_model / t / 1e9, 1)}))
