"""Time to the paper's accuracy (relative error below 1e-2) on one B200 for the
synthetic phase retrieval instances (R = 5, alpha = 3n): iterations and wall time until the signal
estimate chi = sqrt(lambda_1) u_1 is within 1e-2 of chi_nat (checked every `every` iterations).
python tools/phase_recovery.py [n ...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import scg_inputs as si
from oracle import phase as ph  # relative_error only (a closed form)
from paper_1912_02949_b200 import phase as prm

sizes = [int(a) for a in sys.argv[1:]] or [10000, 100000, 1000000]
for n in sizes:
    I = si.phase_instance(n, seed=0)
    t0 = time.perf_counter()
    g = prm.PhaseRetrieval(I.psi, I.b, R=5, seed=0)
    every = 250
    hist = []
    while g.scalars()[0] < 20000:
        g.step(every)
        g.reconstruct()
        err = ph.relative_error(g.signal(), I.chi)
        hist.append((int(g.scalars()[0]), err))
        if err < 1e-2:
            break
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(json.dumps({"n": n, "iterations": hist[-1][0], "rel_err": hist[-1][1], "seconds_incl_checks": round(dt, 2),
                      "history": hist}), flush=True)
    g.close()
