"""A/B of the context's L2 fetch granularity limit (cudaLimitMaxL2FetchGranularity) around bench.py:
python tools/l2_fetch_ab.py G <bench args...>  (G = 0: leave the default)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from cuda.bindings import runtime as rt

G = int(sys.argv[1])
torch.cuda.init()
torch.zeros(1, device="cuda")  # the primary context
lim = rt.cudaLimit.cudaLimitMaxL2FetchGranularity
if G:
    print("set", rt.cudaDeviceSetLimit(lim, G), file=sys.stderr)
print("L2 fetch granularity", rt.cudaDeviceGetLimit(lim), file=sys.stderr)
import bench
sys.argv = ["bench.py"] + sys.argv[2:]
bench.main()
print("L2 fetch granularity after", rt.cudaDeviceGetLimit(lim), file=sys.stderr)
