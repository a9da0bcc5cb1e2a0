"""Binding of the phase retrieval hot path (include/scg_phase.h).

ctypes marshalling only: every step of the iteration runs in the CUDA kernels of
``csrc/phase.cu`` (sm_100a).  There is no CPU fallback -- ``load()`` raises when the library is
missing.  Complex arrays cross the ABI as interleaved (re, im) doubles (numpy complex128).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import LIB_DIR, ROOT, STATUS, _HERE

PHASE_LIB = os.environ.get("SCG_PHASE_LIB") or os.path.join(LIB_DIR, "libscg_phase.so")
PHASE_SOURCES = [os.path.join(_HERE, "csrc", "phase.cu"), os.path.join(ROOT, "include", "scg_phase.h"),
                 os.path.join(ROOT, "include", "sketchycgal.h"),
                 os.path.join(ROOT, "scg_inputs", "include", "scg_rng.h")]
SCG_PR_PROFILE = 1 << 8

_lib = None


class Rec(ctypes.Structure):
    _fields_ = [("t", ctypes.c_int64), ("q", ctypes.c_int32), ("k", ctypes.c_int32), ("theta", ctypes.c_double),
                ("xi", ctypes.c_double), ("c", ctypes.c_double), ("p", ctypes.c_double),
                ("znorm", ctypes.c_double), ("gamma", ctypes.c_double), ("tau", ctypes.c_double),
                ("gap", ctypes.c_double), ("bound", ctypes.c_double)]


class KStat(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("launches", ctypes.c_int64), ("total_ms", ctypes.c_double),
                ("bytes_per_launch", ctypes.c_double)]


def nvcc_cmd(out: str) -> list[str]:
    return ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
            "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", PHASE_SOURCES[0], "-o", out]


def build(force: bool = False) -> str:
    """Compile csrc/phase.cu for sm_100a in-tree (nvcc cross-compiles without a GPU)."""
    os.makedirs(LIB_DIR, exist_ok=True)
    newest = max(os.path.getmtime(p) for p in PHASE_SOURCES)
    if not force and os.path.exists(PHASE_LIB) and os.path.getmtime(PHASE_LIB) >= newest:
        return PHASE_LIB
    tmp = PHASE_LIB + f".tmp{os.getpid()}"
    subprocess.check_call(nvcc_cmd(tmp))
    os.replace(tmp, PHASE_LIB)
    return PHASE_LIB


EXPORTS = ("scg_pr_init", "scg_pr_step", "scg_pr_iter_log", "scg_pr_get_state", "scg_pr_reconstruct",
           "scg_pr_signal", "scg_pr_apply_D", "scg_pr_measure", "scg_pr_kernel_stats", "scg_pr_reset_stats",
           "scg_pr_stream", "scg_pr_destroy")


def open_library(path: str = PHASE_LIB):
    """dlopen the library and declare the ABI (no GPU needed)."""
    lib = ctypes.CDLL(path)
    P, I32, I64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    lib.scg_pr_init.restype = ctypes.c_int
    lib.scg_pr_init.argtypes = [I64, I32, P, P, I32, D, D, ctypes.c_uint64, ctypes.c_uint32, ctypes.POINTER(P)]
    for name, args in [("scg_pr_step", [P, I64]), ("scg_pr_iter_log", [P, P, I64, ctypes.POINTER(I64)]),
                       ("scg_pr_get_state", [P, I32, P]), ("scg_pr_reconstruct", [P, P, P]),
                       ("scg_pr_signal", [P, P]), ("scg_pr_apply_D", [P, P, P, P]), ("scg_pr_measure", [P, P, P]),
                       ("scg_pr_kernel_stats", [P, P, I32, ctypes.POINTER(I32)]), ("scg_pr_reset_stats", [P]),
                       ("scg_pr_destroy", [P])]:
        getattr(lib, name).restype = ctypes.c_int
        getattr(lib, name).argtypes = args
    lib.scg_pr_stream.restype = P
    lib.scg_pr_stream.argtypes = [P]
    return lib


def load():
    """Load the CUDA library.  Fails loudly (no fallback) without the library."""
    global _lib
    if _lib is None:
        if not os.path.exists(PHASE_LIB):
            raise RuntimeError(f"CUDA library {PHASE_LIB} is missing: run __graft_entry__.build()")
        _lib = open_library(PHASE_LIB)
    return _lib


class PhaseError(RuntimeError):
    pass


def _c128(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class PhaseRetrieval:
    """SketchyCGAL on the phase retrieval SDP (scg_pr_init ... scg_pr_destroy), one GPU."""

    def __init__(self, psi, b, R: int = 5, alpha: float | None = None, beta0: float = 1.0, seed: int = 0,
                 profile: bool = False, device: int = 0, flags: int = 0):
        import torch  # device selection only
        torch.cuda.set_device(device)
        self.lib = load()
        psi = _c128(psi)
        b = _f64(b)
        self.L, self.n = psi.shape
        self.R = int(R)
        self.alpha = 3.0 * self.n if alpha is None else float(alpha)
        h = ctypes.c_void_p()
        st = self.lib.scg_pr_init(self.n, self.L, psi.ctypes.data, b.ctypes.data, self.R, self.alpha, float(beta0),
                                  int(seed), (SCG_PR_PROFILE if profile else 0) | int(flags), ctypes.byref(h))
        self._check(st, "scg_pr_init")
        self._h = h

    def _check(self, st, what):
        if st != 0:
            raise PhaseError(f"{what}: {STATUS.get(st, st)}")

    def step(self, T: int = 1):
        self._check(self.lib.scg_pr_step(self._h, int(T)), "scg_pr_step")

    def iter_log(self) -> np.ndarray:
        t = int(self.scalars()[0])
        recs = (Rec * max(t, 1))()
        cnt = ctypes.c_int64()
        self._check(self.lib.scg_pr_iter_log(self._h, recs, t, ctypes.byref(cnt)), "scg_pr_iter_log")
        return np.array([[r.t, r.q, r.k, r.theta, r.xi, r.c, r.p, r.znorm, r.gamma, r.tau, r.gap, r.bound]
                         for r in recs[:cnt.value]], dtype=np.float64).reshape(-1, 12)

    def state(self, which: str):
        n, L, R = self.n, self.L, self.R
        code, shape, dt = {"z": (0, (L, n), np.float64), "y": (1, (L, n), np.float64),
                           "v": (2, (n,), np.complex128), "S": (3, (R, n), np.complex128),
                           "Omega": (4, (R, n), np.complex128), "bt": (5, (L, n), np.float64),
                           "kappa": (6, (L,), np.float64), "scalars": (7, (8,), np.float64)}[which]
        out = np.empty(shape, dtype=dt)
        self._check(self.lib.scg_pr_get_state(self._h, code, out.ctypes.data), "scg_pr_get_state")
        return out.T.copy() if which in ("S", "Omega") else out

    def scalars(self):
        """(t, tau, p, ||A'||, n1, n2, alpha, beta0)."""
        return self.state("scalars")

    def reconstruct(self):
        U = np.empty((self.R, self.n), dtype=np.complex128)
        lam = np.empty(self.R)
        self._check(self.lib.scg_pr_reconstruct(self._h, U.ctypes.data, lam.ctypes.data), "scg_pr_reconstruct")
        return U.T.copy(), lam

    def signal(self):
        chi = np.empty(self.n, dtype=np.complex128)
        self._check(self.lib.scg_pr_signal(self._h, chi.ctypes.data), "scg_pr_signal")
        return chi

    def apply_D(self, w, x):
        w, x = _f64(w), _c128(x)
        y = np.empty(self.n, dtype=np.complex128)
        self._check(self.lib.scg_pr_apply_D(self._h, w.ctypes.data, x.ctypes.data, y.ctypes.data), "scg_pr_apply_D")
        return y

    def measure(self, x):
        x = _c128(x)
        h = np.empty((self.L, self.n))
        self._check(self.lib.scg_pr_measure(self._h, x.ctypes.data, h.ctypes.data), "scg_pr_measure")
        return h

    def kernel_stats(self):
        arr = (KStat * 32)()
        cnt = ctypes.c_int32()
        self._check(self.lib.scg_pr_kernel_stats(self._h, arr, 32, ctypes.byref(cnt)), "scg_pr_kernel_stats")
        return [dict(name=a.name.decode(), launches=a.launches, total_ms=a.total_ms,
                     bytes_per_launch=a.bytes_per_launch) for a in arr[:cnt.value]]

    def reset_stats(self):
        self._check(self.lib.scg_pr_reset_stats(self._h), "scg_pr_reset_stats")

    def stream_ptr(self) -> int:
        return int(self.lib.scg_pr_stream(self._h) or 0)

    def close(self):
        if getattr(self, "_h", None):
            self.lib.scg_pr_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
