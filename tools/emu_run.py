"""Emulated-shard run for profiling: python tools/emu_run.py P [steps] (configs[3])."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_02949_b200 as scg
import scg_inputs as si
P = int(sys.argv[1]); T = int(sys.argv[2]) if len(sys.argv) > 2 else 3
L = si.laplacian(os.environ.get("CFG", "c3"))
s = scg.SketchyCGAL(L, R=10, seed=3, shards=P)
s.step(T)
s.synchronize()
print("ok", s.t)
