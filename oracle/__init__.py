"""CPU oracle for the SketchyCGAL MaxCut hot path (arXiv 1912.02949).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
this package.  The product path (``paper_1912_02949_b200``) never imports it
and shares no code with it; both consume only the seeded input stream of
``scg_inputs``.

* ``scg_oracle.c`` -- the iteration (Alg. 4), randomized Lanczos
  (Alg. 2), tridiagonal eigensolve, exact sums (CAC-2), built with
  gcc -ffp-contract=off.
* this module -- ctypes wrapper plus the one-shot steps written with numpy /
  LAPACK library primitives: Nystrom reconstruction (Alg. 3 / SM3,
  P:1244-1253), error estimates, trace correction
  (Alg. 4 line 13), sign rounding, metrics.

Parity pins: tests/test_oracle_*.py.  Every oracle function is pinned; the
only "parity unpinned" item is the full trajectory at configs[2..4] sizes
(no external value exists).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

P = ctypes.c_void_p
I64 = ctypes.c_int64
D = ctypes.c_double


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "scg_oracle.c")
    hdr = os.path.join(_HERE, "..", "scg_inputs", "include", "scg_rng.h")
    if (not force and os.path.exists(_LIB)
            and os.path.getmtime(_LIB) >= max(os.path.getmtime(src), os.path.getmtime(hdr))):
        return _LIB
    tmp = _LIB + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
                           "-fno-fast-math", src, "-o", tmp, "-lm"])
    os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.oracle_xsum.restype = D
        lib.oracle_xsum.argtypes = [P, I64, ctypes.POINTER(ctypes.c_int)]
        lib.oracle_dot.restype = D
        lib.oracle_dot.argtypes = [P, P, I64]
        lib.oracle_apply.argtypes = [I64, P, P, P, P, P, P]
        lib.oracle_tridiag_mineig.restype = ctypes.c_int
        lib.oracle_tridiag_mineig.argtypes = [P, P, ctypes.c_int, ctypes.POINTER(D), P]
        lib.oracle_lanczos.restype = ctypes.c_int
        lib.oracle_lanczos.argtypes = [I64, P, P, P, P, P, ctypes.c_int, P, ctypes.POINTER(D),
                                       ctypes.POINTER(ctypes.c_int), P, P, P]
        lib.oracle_qt.restype = ctypes.c_int
        lib.oracle_qt.argtypes = [I64, I64]
        lib.oracle_gamma.restype = D
        lib.oracle_gamma.argtypes = [I64, D, D, D]
        lib.oracle_create.restype = P
        lib.oracle_create.argtypes = [I64, P, P, P, ctypes.c_int32, D, D, ctypes.c_uint64, ctypes.c_int,
                                      ctypes.c_int, I64, I64, ctypes.c_int]
        lib.oracle_destroy.argtypes = [P]
        lib.oracle_step.restype = ctypes.c_int
        lib.oracle_step.argtypes = [P, I64]
        lib.oracle_set_box.restype = ctypes.c_int
        lib.oracle_set_box.argtypes = [P, ctypes.c_double, ctypes.c_double]
        lib.oracle_set_ball.restype = ctypes.c_int
        lib.oracle_set_ball.argtypes = [P, ctypes.c_double]
        lib.oracle_set_l1_ball.restype = ctypes.c_int
        lib.oracle_proj.restype = ctypes.c_int
        lib.oracle_proj.argtypes = [P, P, P, ctypes.c_double, P]
        lib.oracle_set_l1_ball.argtypes = [P, ctypes.c_double]
        lib.oracle_t_done.restype = I64
        lib.oracle_t_done.argtypes = [P]
        lib.oracle_scalar.restype = D
        lib.oracle_scalar.argtypes = [P, ctypes.c_int]
        lib.oracle_get.argtypes = [P, ctypes.c_int, P]
        lib.oracle_set_threads.restype = ctypes.c_int
        lib.oracle_set_threads.argtypes = [ctypes.c_int]
        _lib = lib
    return _lib


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def set_threads(n: int = 0) -> int:
    """OpenMP threads of the oracle's row loops and exact sums (n <= 0: all cores).  The thread
    count never changes a bit of any result (exact sums; independent rows)."""
    return int(_load().oracle_set_threads(int(n)))


# ---------------------------------------------------------------- primitives
def xsum(p) -> float:
    """CAC-2: RNE of the exact sum of Q(p_r) (Q truncates at 2^-200)."""
    p = _f64(p)
    err = ctypes.c_int(0)
    r = _load().oracle_xsum(p.ctypes.data, p.shape[0], ctypes.byref(err))
    if err.value:
        raise OverflowError("xsum summand out of range")
    return r


def dot(a, b) -> float:
    a, b = _f64(a), _f64(b)
    return _load().oracle_dot(a.ctypes.data, b.ctypes.data, a.shape[0])


def apply(n, rp, col, m, d, x):
    """CAC-3 row chains of D = offdiag(m) + diag(d)."""
    rp = np.ascontiguousarray(rp, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    m, d, x = _f64(m), _f64(d), _f64(x)
    y = np.empty(n)
    _load().oracle_apply(n, rp.ctypes.data, col.ctypes.data, m.ctypes.data, d.ctypes.data, x.ctypes.data,
                         y.ctypes.data)
    return y


def tridiag_mineig(omega, rho):
    """CAC-5 minimum eigenpair of tridiag(rho, omega, rho) (Alg. 2 lines 11-12)."""
    om = _f64(omega)
    rh = _f64(rho) if len(rho) else np.zeros(1)
    k = om.shape[0]
    s = np.zeros(k)
    th = D()
    rc = _load().oracle_tridiag_mineig(om.ctypes.data, rh.ctypes.data, k, ctypes.byref(th), s.ctypes.data)
    if rc:
        raise ValueError("bad tridiagonal")
    return th.value, s


def qt(t: int, n: int) -> int:
    """Lanczos bound q_t = min(n-1, max(2, ceil(t^(1/4) ln n))) (reading A9)."""
    return _load().oracle_qt(t, n)


def gamma(t: int, alpha: float, beta0: float, nz: float) -> float:
    return _load().oracle_gamma(t, alpha, beta0, nz)


@dataclass
class LanczosResult:
    theta: float
    v: np.ndarray
    k: int
    omega: np.ndarray
    rho: np.ndarray
    s: np.ndarray


def offdiag_of_dense(M):
    """Split a dense symmetric M into (rp, col, m, d) for lanczos()/apply()."""
    n = M.shape[0]
    rp = [0]
    col, m = [], []
    for r in range(n):
        for c in range(n):
            if c != r and M[r, c] != 0.0:
                col.append(c)
                m.append(M[r, c])
        rp.append(len(col))
    return (np.array(rp, dtype=np.int64), np.array(col, dtype=np.int32), np.array(m, dtype=np.float64),
            np.ascontiguousarray(np.diag(M), dtype=np.float64))


def lanczos(n, rp, col, m, d, g, q) -> LanczosResult:
    """Alg. 2 ApproxMinEvec with start vector g (un-normalized randn) and bound q."""
    rp = np.ascontiguousarray(rp, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    m, d, g = _f64(m), _f64(d), _f64(g)
    v = np.zeros(n)
    om = np.zeros(int(q) + 1)
    rh = np.zeros(int(q) + 1)
    sv = np.zeros(int(q) + 1)
    th = D()
    k = ctypes.c_int()
    rc = _load().oracle_lanczos(n, rp.ctypes.data, col.ctypes.data, m.ctypes.data, d.ctypes.data, g.ctypes.data,
                                int(q), v.ctypes.data, ctypes.byref(th), ctypes.byref(k), om.ctypes.data,
                                rh.ctypes.data, sv.ctypes.data)
    if rc:
        raise RuntimeError(f"oracle lanczos failed rc={rc}")
    kk = k.value
    return LanczosResult(th.value, v, kk, om[:kk].copy(), rh[:max(kk - 1, 0)].copy(), sv[:kk].copy())


# ------------------------------------------------------------------ solver
LOG_FIELDS = ("t", "q", "k", "theta", "xi", "c", "p", "znorm", "gamma", "tau")


class Oracle:
    """Alg. 4 SketchyCGAL for MaxCut (C = -L, A = diag, b = 1, alpha = n)."""

    def __init__(self, L, R: int, alpha: float | None = None, beta0: float = 1.0, seed: int = 0,
                 scale: bool = True, qfix: int = 0, logcap: int = 0, vhist: int = 0, trace_le: bool = False,
                 ineq: bool = False, box: tuple | None = None, div_norm: bool = False, ball: float | None = None,
                 l1_ball: float | None = None):
        self.L = L
        self.n = L.n
        self.R = int(R)
        self.alpha_orig = float(L.n if alpha is None else alpha)
        self.scale = bool(scale)
        self.logcap = int(logcap)
        self.vhist_cap = int(vhist)
        self._rp = np.ascontiguousarray(L.row_ptr, dtype=np.int64)
        self._col = np.ascontiguousarray(L.col, dtype=np.int32)
        self._val = _f64(L.val)
        self._h = _load().oracle_create(self.n, self._rp.ctypes.data, self._col.ctypes.data, self._val.ctypes.data,
                                        self.R, self.alpha_orig, float(beta0), int(seed), 1 if scale else 0,
                                        int(qfix), self.logcap, self.vhist_cap,
                                        (1 if trace_le else 0) | (2 if ineq else 0) | (4 if div_norm else 0))
        self.trace_le = bool(trace_le)
        self.ineq = bool(ineq) or box is not None or ball is not None or l1_ball is not None
        if box is not None:  # K = {lo <= u <= hi}, original units
            if _load().oracle_set_box(self._h, float(box[0]), float(box[1])) != 0:
                raise ValueError("oracle_set_box: after the first step or lo > hi")
        if ball is not None:  # K = {||u - 1||_2 <= ball}, original units
            if _load().oracle_set_ball(self._h, float(ball)) != 0:
                raise ValueError("oracle_set_ball: after the first step or delta < 0")
        if l1_ball is not None:  # K = {||u - 1||_1 <= l1_ball}, original units
            if _load().oracle_set_l1_ball(self._h, float(l1_ball)) != 0:
                raise ValueError("oracle_set_l1_ball: after the first step or delta < 0")
        self.beta0 = float(beta0)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _load().oracle_destroy(h)
            self._h = None

    def step(self, T: int):
        rc = _load().oracle_step(self._h, int(T))
        if rc:
            raise RuntimeError("oracle: exact-sum range error")

    @property
    def t(self) -> int:
        return _load().oracle_t_done(self._h)

    def _get(self, which, shape):
        out = np.zeros(shape)
        _load().oracle_get(self._h, which, out.ctypes.data)
        return out

    @property
    def z(self):
        return self._get(0, self.n)

    @property
    def y(self):
        return self._get(1, self.n)

    @property
    def S(self):
        return self._get(2, self.n * self.R).reshape(self.R, self.n).T

    @property
    def Omega(self):
        return self._get(3, self.n * self.R).reshape(self.R, self.n).T

    @property
    def v(self):
        return self._get(4, self.n)

    @property
    def log(self) -> np.ndarray:
        return self._get(5, self.logcap * 12).reshape(self.logcap, 12)

    @property
    def vhist(self) -> np.ndarray:
        return self._get(6, self.vhist_cap * self.n).reshape(self.vhist_cap, self.n)

    @property
    def cdiag(self):
        return self._get(7, self.n)

    @property
    def p(self) -> float:
        return _load().oracle_scalar(self._h, 0)

    @property
    def tau(self) -> float:
        return _load().oracle_scalar(self._h, 1)

    @property
    def nrmL(self) -> float:
        return _load().oracle_scalar(self._h, 2)

    @property
    def alpha(self) -> float:
        return _load().oracle_scalar(self._h, 3)

    @property
    def b(self) -> float:
        return _load().oracle_scalar(self._h, 4)

    # ---- original-units monitors ("evaluated with respect to the original data")
    def project(self, z, y=None, beta: float = 1.0) -> np.ndarray:
        """proj_K(z + y / beta) onto the constraint set in effect, scaled units."""
        z = _f64(z)
        y = np.zeros_like(z) if y is None else _f64(y)
        w = np.empty_like(z)
        if _load().oracle_proj(self._h, z.ctypes.data, y.ctypes.data, float(beta), w.ctypes.data) != 0:
            raise ValueError("oracle_proj: no constraint set, or a range error in its exact sums")
        return w

    def implicit_objective(self) -> float:
        """tr(L X_t) of the implicit iterate from the tracked p_t = <C~, X~_t>."""
        if self.scale:
            return -self.p * self.nrmL * self.alpha_orig / self.alpha
        return -self.p

    def implicit_infeasibility(self) -> float:
        """||A X_t - b|| / (1 + ||b||) in original units."""
        unit = self.alpha_orig / self.alpha if self.scale else 1.0
        zb = (self.z - self.b) * unit
        return float(np.linalg.norm(zb) / (1.0 + np.sqrt(self.n)))


# --------------------------------------------------------- one-shot numpy steps
def matlab_eps(x: float) -> float:
    """MATLAB eps(x) = 2^(floor(log2 |x|) - 52) (reading A17)."""
    if x == 0.0:
        return 2.0 ** -1074
    m, e = np.frexp(abs(x))  # x = m 2^e, m in [0.5, 1)
    return float(2.0 ** (int(e) - 1 - 52))


def nystrom_reconstruct(S, Omega, tau: float | None = None, max_retry: int = 40):
    """NystromSketch.Reconstruct (Alg. 3; Alg. SM3).

    Returns (U, Lam, err): U n x R orthonormal, Lam descending >= 0, err_r = tau - cumsum(Lam)
    (None if tau is None).
    """
    n, R = S.shape
    nrm = float(np.linalg.norm(S, 2))
    if nrm == 0.0:
        U = np.linalg.qr(Omega)[0]
        Lam = np.zeros(R)
        return U, Lam, (None if tau is None else tau - np.cumsum(Lam))
    sigma = np.sqrt(n) * matlab_eps(nrm)                         # line 1
    for _ in range(max_retry):
        Ss = S + sigma * Omega                                     # line 2
        B = Omega.T @ Ss
        B = 0.5 * (B + B.T)
        try:
            Lc = np.linalg.cholesky(B)                             # line 3: B = Lc Lc^T, MATLAB R = Lc^T
            break
        except np.linalg.LinAlgError:
            sigma *= 2.0
    else:
        raise np.linalg.LinAlgError("Cholesky failed after 40 shift doublings")
    # line 4: S_sigma / R  with R upper (R^T R = B)  ->  Y = S_sigma R^{-1}
    Y = np.linalg.solve(Lc, Ss.T).T                                # Y R = S_sigma
    U, sv, _ = np.linalg.svd(Y, full_matrices=False)
    Lam = np.maximum(0.0, sv ** 2 - sigma)                         # line 5
    err = None if tau is None else tau - np.cumsum(Lam)            # SM3 line 6
    return U, Lam, err


def alpha_doubling(L, R: int, alpha0: float, T: int, rtol: float = 1e-2, max_rounds: int = 8,
                   beta0: float = 1.0, seed: int = 0, scale: bool = True):
    """Remark "Standard-form SDP", steps 1-4 as printed: solve the trace-bounded
    SDP tr X <= alpha_i for T iterations, stop when its primal objective equals
    the previous round's -- for these approximate solutions: within rtol relative (DESIGN.md
    reading R31) -- else alpha_{i+1} = 2 alpha_i.  Returns (last Oracle, alphas, objectives,
    converged); the objective is the implicit tr(L X_T) in original units."""
    alphas, objs = [], []
    alpha = float(alpha0)
    o = None
    for i in range(int(max_rounds)):
        o = Oracle(L, R, alpha=alpha, beta0=beta0, seed=seed, scale=scale, logcap=T, trace_le=True)
        o.step(T)
        alphas.append(alpha)
        objs.append(o.implicit_objective())
        if i > 0 and abs(objs[i] - objs[i - 1]) <= rtol * abs(objs[i]):
            return o, np.array(alphas), np.array(objs), True
        alpha = 2.0 * alpha
    return o, np.array(alphas), np.array(objs), False


def trace_correct(Lam, alpha: float):
    """Alg. 4 line 13: Lam + (alpha - tr Lam) I / R."""
    Lam = np.asarray(Lam, dtype=np.float64)
    return Lam + (alpha - Lam.sum()) / Lam.shape[0]


def cut_weight(L, chi) -> float:
    """Weight of the cut chi in {+-1}^n: (1/4) chi^T L chi (eqn:maxcut-sdp P:118-122)."""
    i, j, w = L.edges()
    chi = np.asarray(chi)
    return float(np.sum(w * (chi[i] != chi[j])))


def round_cut(L, U):
    """Best of the R sign cuts sgn(U[:, k]); sgn(0)=+1, ties lowest k, chi_0 = +1."""
    best_w, best_k, best_chi = -np.inf, -1, None
    for k in range(U.shape[1]):
        chi = np.where(U[:, k] >= 0.0, 1, -1).astype(np.int8)
        w = cut_weight(L, chi)
        if w > best_w:
            best_w, best_k, best_chi = w, k, chi
    if best_chi[0] < 0:
        best_chi = -best_chi
    return best_chi, best_w, best_k


def laplacian_quadratic(L, u) -> float:
    """u^T L u = sum_{ij in E} w_ij (u_i - u_j)^2 (eqn:comb-laplacian P:97-100)."""
    i, j, w = L.edges()
    return float(np.sum(w * (u[i] - u[j]) ** 2))


def objective_hat(L, U, Lam) -> float:
    """tr(L X^) = sum_k Lam_k u_k^T L u_k for X^ = U diag(Lam) U^T."""
    return float(sum(Lam[k] * laplacian_quadratic(L, U[:, k]) for k in range(U.shape[1])))


def feasibility_hat(U, Lam):
    """(||diag X^ - 1|| / ||1||, ||diag X^ - 1|| / (1 + ||1||)) (BASELINE)."""
    dX = (U * U) @ Lam
    r = np.linalg.norm(dX - 1.0)
    n = U.shape[0]
    return float(r / np.sqrt(n)), float(r / (1.0 + np.sqrt(n)))


def solve(L, R, T, seed=0, beta0=1.0, scale=True, trace_correction=True, logcap=None):
    """Full oracle run: Alg. 4 for T iterations, reconstruct, trace-correct, round.  Original units."""
    o = Oracle(L, R, seed=seed, beta0=beta0, scale=scale, logcap=T if logcap is None else logcap)
    o.step(T)
    U, Lam, err = nystrom_reconstruct(o.S, o.Omega, o.tau)
    unit = o.alpha_orig / o.alpha
    Lam_u = Lam * unit
    Lam_tc = trace_correct(Lam, o.alpha) * unit if trace_correction else Lam_u
    chi, w, k = round_cut(L, U)
    return dict(oracle=o, U=U, Lambda=Lam_u, Lambda_tc=Lam_tc, err=None if err is None else err * unit,
                objective=objective_hat(L, U, Lam_u), objective_tc=objective_hat(L, U, Lam_tc),
                feasibility=feasibility_hat(U, Lam_u), feasibility_tc=feasibility_hat(U, Lam_tc),
                chi=chi, cut_weight=w, cut_col=k,
                implicit_objective=o.implicit_objective(), implicit_infeasibility=o.implicit_infeasibility())
