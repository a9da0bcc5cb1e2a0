"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module holds no solver arithmetic (DESIGN.md "Random inputs" and
"Input recipe").  It builds ``libscg_inputs.so`` from ``graphs.c`` and exposes:

* ``laplacian(config)`` -- the weighted Laplacian CSR of one of the five
  BASELINE.json workloads (or a custom family), as numpy arrays;
* ``laplacian_from_edges`` -- Laplacian CSR of a caller edge list;
* ``normals`` -- draws of the normative Gaussian stream of ``include/scg_rng.h``
  (the Omega / Lanczos start-vector stream).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libscg_inputs.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "graphs.c")
    hdr = os.path.join(_HERE, "include", "scg_rng.h")
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= max(os.path.getmtime(src), os.path.getmtime(hdr))):
        return _LIB_PATH
    tmp = _LIB_PATH + f".tmp{os.getpid()}"
    cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
           "-fno-fast-math", src, "-o", tmp, "-lm"]
    subprocess.check_call(cmd)
    os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.scg_gen_graph.restype = ctypes.c_void_p
        lib.scg_gen_graph.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_double, ctypes.c_uint64]
        lib.scg_graph_from_edges.restype = ctypes.c_void_p
        lib.scg_graph_from_edges.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_void_p, ctypes.c_int]
        lib.scg_graph_info.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
        lib.scg_graph_copy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.scg_graph_free.argtypes = [ctypes.c_void_p]
        lib.scg_fill_normal.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64,
                                        ctypes.c_int64, ctypes.c_void_p]
        lib.scg_fill_uniform.argtypes = lib.scg_fill_normal.argtypes
        lib.scg_philox.argtypes = [ctypes.c_uint32] * 6 + [ctypes.c_void_p]
        _lib = lib
    return _lib


@dataclass
class CSR:
    """Symmetric Laplacian L in CSR, diagonal stored in place, columns ascending."""
    n: int
    row_ptr: np.ndarray  # int64[n+1]
    col: np.ndarray      # int32[nnz]
    val: np.ndarray      # float64[nnz]

    @property
    def nnz(self) -> int:
        return int(self.col.shape[0])

    @property
    def m(self) -> int:
        """Number of undirected edges (off-diagonal nonzeros / 2)."""
        return (self.nnz - self.n) // 2

    def dense(self) -> np.ndarray:
        L = np.zeros((self.n, self.n))
        for r in range(self.n):
            for k in range(self.row_ptr[r], self.row_ptr[r + 1]):
                L[r, self.col[k]] += self.val[k]
        return L

    def edges(self):
        """(i, j, w) with i < j, w = -L_ij."""
        rows = np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.row_ptr))
        mask = self.col > rows
        return rows[mask], self.col[mask].astype(np.int64), -self.val[mask]


def _take(ptr) -> CSR:
    lib = _load()
    if not ptr:
        raise MemoryError("graph generation failed")
    n = ctypes.c_int64()
    nnz = ctypes.c_int64()
    lib.scg_graph_info(ptr, ctypes.byref(n), ctypes.byref(nnz))
    rp = np.empty(n.value + 1, dtype=np.int64)
    col = np.empty(nnz.value, dtype=np.int32)
    val = np.empty(nnz.value, dtype=np.float64)
    lib.scg_graph_copy(ptr, rp.ctypes.data, col.ctypes.data, val.ctypes.data)
    lib.scg_graph_free(ptr)
    return CSR(int(n.value), rp, col, val)


FAMILY = {"er": 0, "torus": 1, "powerlaw": 2, "rgg": 3, "ring_matching": 4}


def generate(family: str, a: int, b: int = 0, p: float = 0.0, seed: int = 0) -> CSR:
    return _take(_load().scg_gen_graph(FAMILY[family], int(a), int(b), float(p), int(seed)))


def laplacian_from_edges(n: int, i, j, w, dedupe: bool = False) -> CSR:
    i = np.ascontiguousarray(i, dtype=np.int32)
    j = np.ascontiguousarray(j, dtype=np.int32)
    w = np.ascontiguousarray(w, dtype=np.float64)
    return _take(_load().scg_graph_from_edges(int(n), int(i.shape[0]), i.ctypes.data, j.ctypes.data,
                                              w.ctypes.data, 1 if dedupe else 0))


# The five BASELINE.json workloads (configs[0..4]); see DESIGN.md "Input recipe".
CONFIGS = {
    "c0": dict(family="er", a=800, p=0.06, seed=0, R=10, T=1000,
               desc="MaxCut SDP, Erdos-Renyi n=800 p=0.06, unit weights, R=10, T=1000, seed 0"),
    "c1": dict(family="torus", a=50, b=160, seed=1, R=10, T=5000,
               desc="MaxCut SDP, torus 50x160 (n=8000, m=16000), weights +-1, R=10, T=5000, seed 1"),
    "c2": dict(family="powerlaw", a=1 << 20, seed=2, R=10, T=2000,
               desc="MaxCut SDP, ER + Chung-Lu Zipf(2.1) n=2^20 avg deg ~8, unit weights, R=10, T=2000, seed 2"),
    "c3": dict(family="rgg", a=1 << 24, seed=3, R=10, T=1000,
               desc="MaxCut SDP, mutual k-NN (k=2..4) random geometric n=2^24 Morton order, unit weights, "
                    "R=10, T=1000, seed 3"),
    "c4": dict(family="ring_matching", a=1 << 25, seed=4, R=20, T=500,
               desc="MaxCut SDP, ring + random perfect matching n=2^25 (3-regular), w~U[0.5,1.5], R=20, T=500, "
                    "seed 4"),
}


def laplacian(config: str) -> CSR:
    c = CONFIGS[config]
    return generate(c["family"], c["a"], c.get("b", 0), c.get("p", 0.0), c["seed"])


def normals(seed: int, stream: int, sub: int, first: int, count: int) -> np.ndarray:
    out = np.empty(int(count), dtype=np.float64)
    _load().scg_fill_normal(int(seed), int(stream), int(sub), int(first), int(count), out.ctypes.data)
    return out


def uniforms(seed: int, stream: int, sub: int, first: int, count: int) -> np.ndarray:
    out = np.empty(int(count), dtype=np.float64)
    _load().scg_fill_uniform(int(seed), int(stream), int(sub), int(first), int(count), out.ctypes.data)
    return out


def philox(counter, key) -> np.ndarray:
    out = np.zeros(4, dtype=np.uint32)
    _load().scg_philox(*[int(x) for x in counter], *[int(x) for x in key], out.ctypes.data)
    return out


# ---------------------------------------------------------------------------
# Synthetic abstract phase retrieval instances.
SCG_STREAM_PHASE = 3  # include/scg_rng.h: sub 0 = unit phase, 1 = magnitude, 2 = signal
PHASE_L = 12  # d = 12 n coded-diffraction measurements


@dataclass
class PhaseInstance:
    """psi: (L, n) complex modulating waveforms; chi: (n,) the signal chi_natural;
    b: (L, n) real phaseless measurements, b[j, l] = |(W_n diag(psi_j)^* chi)_l|^2 (reading R36)."""
    n: int
    psi: np.ndarray
    chi: np.ndarray
    b: np.ndarray


def phase_psi(n: int, seed: int, L: int = PHASE_L) -> np.ndarray:
    """Coded diffraction waveforms: each entry is a uniform draw from {1, i, -1, -i}
    times an independent draw from {sqrt(2)/2, sqrt(3)} with probabilities 0.8 / 0.2."""
    cnt = L * n
    u_unit = uniforms(seed, SCG_STREAM_PHASE, 0, 0, cnt)
    u_mag = uniforms(seed, SCG_STREAM_PHASE, 1, 0, cnt)
    k = np.minimum((u_unit * 4.0).astype(np.int64), 3)
    unit = np.array([1.0 + 0.0j, 0.0 + 1.0j, -1.0 + 0.0j, 0.0 - 1.0j])[k]
    mag = np.where(u_mag < 0.8, np.sqrt(2.0) / 2.0, np.sqrt(3.0))
    return (unit * mag).reshape(L, n)


def phase_signal(n: int, seed: int) -> np.ndarray:
    """chi_natural from the complex standard normal distribution: real and imaginary
    parts independent N(0, 1/2), so E|chi_i|^2 = 1 (reading R36)."""
    g = normals(seed, SCG_STREAM_PHASE, 2, 0, 2 * n)
    return (g[0::2] + 1j * g[1::2]) * np.sqrt(0.5)


def phase_instance(n: int, seed: int = 0, L: int = PHASE_L) -> PhaseInstance:
    """One synthetic instance: psi, chi_natural and the d = L n measurements b.
    The measurement of the data recipe uses numpy's FFT (W_n(l, k) = exp(-2 pi i l k / n))."""
    psi = phase_psi(n, seed, L)
    chi = phase_signal(n, seed)
    b = np.abs(np.fft.fft(np.conj(psi) * chi[None, :], axis=1)) ** 2
    return PhaseInstance(n, psi, chi, b)


# Workloads of the phase retrieval experiment: n in {10^2, ..., 10^6}, d = 12 n,
# R = 5, alpha = 3 n.
PHASE_CONFIGS = {
    "p2": dict(n=100, seed=0, R=5),
    "p3": dict(n=1000, seed=1, R=5),
    "p4": dict(n=10000, seed=2, R=5),
    "p5": dict(n=100000, seed=3, R=5),
    "p6": dict(n=1000000, seed=4, R=5),
}
