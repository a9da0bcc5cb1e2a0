#!/usr/bin/env python
"""Write the oracle's reference trajectories for the long GPU parity cases (tests/golden/*.json).

Every value in these fixtures comes from the CPU oracle (``oracle/``) run on the seeded synthetic
inputs of ``scg_inputs`` -- never from the CUDA path.  The GPU tests (tests/test_gpu_golden.py)
compare the CUDA path's iteration records with them bit for bit, the feedback-path state through
SHA-256 digests of its exact bytes, and the off-path sketch S at sampled rows to rounding.

Cases ("Next round" item 1):
  c3_t25   configs[3] (n = 2^24) t = 1..25 -- covers the window bench.py is timed on by the driver
  c2_t100  configs[2] (n = 2^20, power-law hubs: long rows) t = 1..100
  c4_t5    configs[4] (n = 2^25, weighted, random matching) t = 1..5 at its real R = 20
  c1_T5000 configs[1] (torus, +-1 weights) the whole run T = 5000, reconstruction, objective,
           feasibility and the rounded cut
  c1_q255  configs[1] with the fixed Lanczos bound q = 255 (sketchycgal_set_lanczos_q), t = 1..12:
           k_tridiag / k_combine / the Lanczos store at k > 127

usage: python tests/golden/make_golden.py [case ...]      (all cases by default; OpenMP on all cores)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import scg_inputs as si  # noqa: E402

CASES = {
    "c3_t25": dict(cfg="c3", T=25),
    "c2_t100": dict(cfg="c2", T=100),
    "c4_t5": dict(cfg="c4", T=5),
    "c1_T5000": dict(cfg="c1", T=5000, recon=True),
    "c1_q255": dict(cfg="c1", T=12, qfix=255),
}
N_SAMPLE = 512  # rows of S kept for the rounding-level comparison


def digest(x) -> str:
    return hashlib.sha256(np.ascontiguousarray(x, dtype="<f8").tobytes()).hexdigest()


def hexlist(x):
    return [float(v).hex() for v in np.asarray(x, dtype=np.float64).ravel()]


def sample_rows(n: int, seed: int) -> np.ndarray:
    return np.sort(np.random.default_rng(seed).choice(n, size=min(n, N_SAMPLE), replace=False))


def make(name: str) -> dict:
    spec = CASES[name]
    cfg = spec["cfg"]
    c = si.CONFIGS[cfg]
    R, T, seed, qfix = c["R"], spec["T"], c["seed"], spec.get("qfix", 0)
    t0 = time.time()
    L = si.laplacian(cfg)
    o = oracle.Oracle(L, R, seed=seed, logcap=T, qfix=qfix)
    t1 = time.time()
    o.step(T)
    t2 = time.time()
    rows = sample_rows(L.n, 1234)
    S = o.S
    out = dict(case=name, config=cfg, n=int(L.n), m=int(L.m), R=R, T=T, seed=seed, qfix=qfix,
               source="oracle/ (CPU, fp64) on scg_inputs.laplacian(config); written by tests/golden/make_golden.py",
               oracle_seconds=round(t2 - t1, 1), setup_seconds=round(t1 - t0, 1),
               log_fields=list(oracle.LOG_FIELDS) + ["gap", "bound"],
               log=[hexlist(r) for r in o.log],
               sha256={"z": digest(o.z), "y": digest(o.y), "v": digest(o.v), "Omega": digest(o.Omega)},
               S_rows=rows.tolist(), S_sample=hexlist(S[rows, :]), S_absmax=float(np.abs(S).max()).hex(),
               p=float(o.p).hex(), tau=float(o.tau).hex())
    if spec.get("recon"):
        U, Lam, err = oracle.nystrom_reconstruct(S, o.Omega, o.tau)
        unit = o.alpha_orig / o.alpha
        lam_tc = oracle.trace_correct(Lam, o.alpha) * unit
        chi, w, k = oracle.round_cut(L, U)
        out.update(Lambda_tc=hexlist(lam_tc), err=hexlist(err * unit),
                   objective_hat_tc=float(oracle.objective_hat(L, U, lam_tc)).hex(),
                   feasibility_hat_tc=hexlist(oracle.feasibility_hat(U, lam_tc)),
                   implicit_objective=float(o.implicit_objective()).hex(),
                   implicit_infeasibility=float(o.implicit_infeasibility()).hex(),
                   cut_weight=float(w).hex(), cut_col=int(k),
                   chi_sha256=hashlib.sha256(np.ascontiguousarray(chi, dtype=np.int8).tobytes()).hexdigest())
    return out


def main(argv):
    names = argv or list(CASES)
    oracle.set_threads(0)
    for name in names:
        t = time.time()
        res = make(name)
        with open(os.path.join(HERE, f"{name}.json"), "w") as f:
            json.dump(res, f, separators=(",", ":"))
            f.write("\n")
        print(f"{name}: {time.time() - t:.1f} s (oracle {res['oracle_seconds']} s)", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
