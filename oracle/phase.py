"""CPU oracle for SketchyCGAL on the abstract phase retrieval SDP.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module.  The product path never
imports it and shares no code with it; both consume only the seeded inputs of ``scg_inputs``
(the instance psi, chi, b of P:4287-4305 and the Gaussian draws of ``include/scg_rng.h``).

Plain numpy, complex128 / float64, step by step in the paper's order and notation; numpy's FFT
(pocketfft) is the library primitive that applies the DFT matrix W_n.

Problem (eqn:numerics-phase-retrieval-sdp):

    minimize tr X  subject to  A X = b,  X psd,  tr X <= alpha,    A_i = a_i a_i^*,

with the coded-diffraction rows a_{(j-1)n+l}^* = W_n(l, :) diag(psi_j)^* (reading
R36), so (A X)_{j,l} = (M_j X M_j^*)_{ll} with M_j = W_n diag(conj psi_j), and
A^*(w) = sum_j M_j^* diag(w_j) M_j, M_j^* y = psi_j o (W_n^* y), W_n^* y = n ifft(y).

Scaling (eqn:problem-scaling; readings R37, R38): ||C||_F = ||A|| = alpha = 1 and
equal ||A_i||_F:  C~ = I / sqrt(n); every row of the modulation j is divided by
||A_i||_F = ||a_i||^2 = ||psi_j||^2 (c_j = 1 / ||psi_j||^2) and the whole map by its operator norm
s = ||A'||, so A~_i = kappa_j A_i with kappa_j = c_j / s;  b~ = kappa b / alpha;  X = alpha X~.

||A'|| (reading R38): A' splits over the circulant diagonals X_s = {X_{m+s, m}} of X (the rows of
M_j X M_j^* for different shifts s are orthogonal Fourier modes in l), so
||A'||^2 = n max_s lambda_max(H_s),  H_s(j, k) = c_j c_k sum_m conj(f_j^s(m)) f_k^s(m),
f_j^s(m) = conj(psi_j(m + s)) psi_j(m).  ``opnorm_exact`` evaluates every shift (FFT
autocorrelations); the path uses the s = 0 (diagonal) block, ``opnorm_diag`` =
sqrt(n lambda_max(G)), G(j, k) = c_j c_k <|psi_j|^2, |psi_k|^2>, which equals the exact norm on
the coded-diffraction distribution (uniform phases make the s != 0 blocks smaller; pinned by
tests/test_oracle_phase.py on the paper's instances).

Iteration (Alg. 4, with the trace-bounded LMO of P:3860-3868):
    beta_t = beta0 sqrt(t+1), eta_t = 2/(t+1), q_t = ceil(t^(1/4) ln n)
    w = y + beta_t (z - b~);  D_t = C~ + A~^*(w)
    (theta, v) = ApproxMinEvec(D_t; q_t)   (Alg. 2 over C^n; readings A1-A3)
    xi = v^* D_t v
    if xi < 0: H = vv^* (alpha~ = 1) else H = 0
    z <- (1 - eta) z + eta A~(H);  A~(vv^*)_{j,l} = kappa_j |(M_j v)_l|^2
    gamma = min(beta0, 4 beta0 / ((t+1)^{3/2} ||z - b~||^2))  (||A~|| = alpha~ = 1)
    y <- y + gamma (z - b~)
    S <- (1 - eta) S + eta v (v^* Omega)  [H = vv^*],  else (1 - eta) S
    tau <- (1 - eta) tau + eta ||v||^2 [H], p <- (1 - eta) p + eta v^* C~ v [H]
Rounding: chi = sqrt(lambda) u for the maximum eigenpair of X^ = alpha U Lam U^*,
relative error min_phi ||e^{i phi} chi - chi_nat|| / ||chi_nat||.
Random inputs: Omega[:, k] = N(seed, 0, k, 2i) + i N(seed, 0, k, 2i+1), the start vector of
iteration t g_i = N(seed, 1, t, 2i) + i N(seed, 1, t, 2i+1) (scg_rng.h streams 0 and 1).
"""
from __future__ import annotations

import numpy as np

import scg_inputs as si

from . import gamma as _gamma
from . import qt as _qt
from . import tridiag_mineig as _tridiag_mineig
from . import matlab_eps

LOG_FIELDS = ("t", "q", "k", "theta", "xi", "c", "p", "znorm", "gamma", "tau", "gap", "bound")


# ------------------------------------------------------------------ operators
def M(psi, x):
    """M_j x = W_n (conj(psi_j) o x) for every j (reading R36); returns (L, n)."""
    return np.fft.fft(np.conj(psi) * x[None, :], axis=1)


def Mstar(psi, Y):
    """sum_j M_j^* Y_j = sum_j psi_j o (W_n^* Y_j), W_n^* = n ifft."""
    n = psi.shape[1]
    return np.sum(psi * (n * np.fft.ifft(Y, axis=1)), axis=0)


def A_rank1(psi, kappa, v):
    """A~(v v^*)_{j,l} = kappa_j |(M_j v)_l|^2 (primitive 3 for phase retrieval)."""
    return kappa[:, None] * np.abs(M(psi, v)) ** 2


def Astar_apply(psi, kappa, w, x):
    """A~^*(w) x = sum_j kappa_j M_j^* (w_j o M_j x) (primitive 2)."""
    return Mstar(psi, kappa[:, None] * w * M(psi, x))


def apply_D(psi, kappa, w, x):
    """D x = C~ x + A~^*(w) x with C~ = I / sqrt(n) (eqn; primitive 1 + 2)."""
    n = psi.shape[1]
    return x / np.sqrt(n) + Astar_apply(psi, kappa, w, x)


# ------------------------------------------------------------------ scaling
def row_scale(psi):
    """c_j = 1 / ||A_i||_F = 1 / ||psi_j||^2 for the rows of modulation j."""
    return 1.0 / np.sum(np.abs(psi) ** 2, axis=1)


def opnorm_diag(psi, c):
    """||A'|| on the diagonal subspace: sqrt(n lambda_max(G)), G = P P^T, P_j = c_j |psi_j|^2."""
    n = psi.shape[1]
    P = c[:, None] * np.abs(psi) ** 2
    return float(np.sqrt(n * np.linalg.eigvalsh(P @ P.T)[-1]))


def opnorm_exact(psi, c):
    """Exact ||A'|| = sqrt(n max_s lambda_max(H_s)) over every circulant shift s (reading R38):
    H_s(j, k) = c_j c_k sum_m f_j^s(m) conj(f_k^s(m)) = c_j c_k sum_m u_jk(m + s) conj(u_jk(m)),
    u_jk(m) = conj(psi_j(m)) psi_k(m) -- the circular autocorrelation ifft(|fft(u_jk)|^2)[s].
    (For s != 0 the sup is taken over all complex x_s, an upper bound of the Hermitian case.)
    Returns (norm, argmax shift, lambda_max per shift)."""
    L, n = psi.shape
    H = np.empty((n, L, L), dtype=np.complex128)
    for j in range(L):
        for k in range(L):
            U = np.fft.fft(np.conj(psi[j]) * psi[k])
            H[:, j, k] = c[j] * c[k] * np.fft.ifft(U * np.conj(U))
    lam = np.linalg.eigvalsh(H)[:, -1]
    return float(np.sqrt(n * lam.max())), int(np.argmax(lam)), lam


def scaling(psi, b, alpha):
    """(kappa, b~): A~_i = kappa_j A_i with kappa_j = c_j / ||A'||, b~ = kappa b / alpha."""
    c = row_scale(psi)
    s = opnorm_diag(psi, c)
    kappa = c / s
    return kappa, kappa[:, None] * b / alpha


# ------------------------------------------------------------------ Lanczos (Alg. 2 over C^n)
def lanczos(apply, g, q):
    """ApproxMinEvec (Alg. 2) with stored vectors, start vector g (un-normalized),
    bound q; readings A1 (rho = ||v_{i+1}||), A2 (the q-th step needs no v_{q+1}) and A3 (break
    when rho <= 2^-45 (|omega| + rho_prev)) as in the MaxCut oracle.  Returns
    (theta, v, k, omega, rho, s)."""
    v = g / np.linalg.norm(g)                                   # lines 1-2
    V = [v]
    omega, rho = [], []
    vprev, rprev = np.zeros_like(v), 0.0
    k = q
    for i in range(1, q + 1):
        a = apply(v)
        om = float(np.real(np.vdot(v, a)))                      # line 5: Re(v_i^* M v_i)
        omega.append(om)
        if i == q:
            break
        u = a - om * v - rprev * vprev                          # line 6
        r = float(np.linalg.norm(u))                            # line 7
        rho.append(r)
        if r <= 2.0 ** -45 * (abs(om) + rprev):                 # line 8
            k = i
            break
        vprev, v, rprev = v, u / r, r                           # line 9
        V.append(v)
    k = len(omega)
    theta, s = _tridiag_mineig(np.array(omega), np.array(rho[:k - 1]))   # lines 11-12
    x = np.zeros_like(V[0])
    for j in range(k):
        x = x + s[j] * V[j]                                     # line 13
    x = x / np.linalg.norm(x)
    return theta, x, k, np.array(omega), np.array(rho[:k - 1]), s


def start_vector(seed, t, n):
    g = si.normals(seed, 1, t, 0, 2 * n)
    return g[0::2] + 1j * g[1::2]


def omega_matrix(seed, n, R):
    Om = np.empty((n, R), dtype=np.complex128)
    for k in range(R):
        g = si.normals(seed, 0, k, 0, 2 * n)
        Om[:, k] = g[0::2] + 1j * g[1::2]
    return Om


# ------------------------------------------------------------------ solver
class PhaseOracle:
    """Alg. 4 SketchyCGAL on the scaled phase retrieval SDP (module docstring)."""

    def __init__(self, psi, b, R: int, alpha: float | None = None, beta0: float = 1.0, seed: int = 0,
                 logcap: int = 0, keep_v: bool = False):
        self.psi = np.ascontiguousarray(psi, dtype=np.complex128)
        self.L, self.n = self.psi.shape
        n = self.n
        self.R = int(R)
        self.alpha = 3.0 * n if alpha is None else float(alpha)
        self.beta0 = float(beta0)
        self.seed = int(seed)
        self.kappa, self.bt = scaling(self.psi, np.asarray(b, dtype=np.float64), self.alpha)
        self.z = np.zeros((self.L, n))
        self.y = np.zeros((self.L, n))
        self.Omega = omega_matrix(self.seed, n, self.R)
        self.S = np.zeros((n, self.R), dtype=np.complex128)
        self.tau = 0.0
        self.p = 0.0
        self.t = 0
        self.log = []
        self.v = None
        self.keep_v = keep_v
        self.vhist = []

    def D(self, t):
        beta = self.beta0 * np.sqrt(t + 1.0)
        return self.y + beta * (self.z - self.bt)

    def step(self, T: int = 1):
        n = self.n
        rsn = 1.0 / np.sqrt(n)
        for _ in range(int(T)):
            t = self.t + 1
            beta = self.beta0 * np.sqrt(t + 1.0)                # line 5
            eta = 2.0 / (t + 1.0)
            q = _qt(t, n)
            # surrogate gap / posterior bound of the state before the update
            e = self.z - self.bt
            S_yz = float(np.sum(self.y * self.z))
            S_ez = float(np.sum(e * self.z))
            S_yb = float(np.sum(self.y * self.bt))
            S_ezb = float(np.sum(e * (self.z + self.bt)))
            p_t = self.p
            w = self.y + beta * e                               # line 6: D_t = C~ + A~^*(w)
            theta, v, k, _, _, _ = lanczos(lambda x: apply_D(self.psi, self.kappa, w, x),
                                           start_vector(self.seed, t, n), q)
            xi = float(np.real(np.vdot(v, apply_D(self.psi, self.kappa, w, v))))
            cval = float(np.real(np.vdot(v, v))) * rsn          # v^* C~ v
            on = xi < 0.0                                       # trace-bounded LMO
            if on:
                self.z = (1.0 - eta) * self.z + eta * A_rank1(self.psi, self.kappa, v)
            else:
                self.z = (1.0 - eta) * self.z
            e1 = self.z - self.bt
            nz = float(np.sum(e1 * e1))
            gam = _gamma(t, 1.0, self.beta0, nz)                # alpha~ = ||A~|| = 1
            self.y = self.y + gam * e1
            if on:
                g = np.conj(v) @ self.Omega                     # v^* Omega
                self.S = (1.0 - eta) * self.S + eta * np.outer(v, g)
                self.tau = (1.0 - eta) * self.tau + eta * float(np.real(np.vdot(v, v)))
                self.p = (1.0 - eta) * self.p + eta * cval
            else:
                self.S = (1.0 - eta) * self.S
                self.tau = (1.0 - eta) * self.tau
                self.p = (1.0 - eta) * self.p
            ax = min(xi, 0.0)
            gap = (p_t + S_yz) + beta * S_ez - ax
            bound = (p_t + S_yb) + 0.5 * beta * S_ezb - ax
            self.log.append((t, q, k, theta, xi, cval, self.p, np.sqrt(nz), gam, self.tau, gap, bound))
            self.v = v
            if self.keep_v:
                self.vhist.append(v.copy())
            self.t = t

    @property
    def logarr(self):
        return np.array(self.log, dtype=np.float64).reshape(-1, len(LOG_FIELDS))

    def reconstruct(self):
        """NystromSketch.Reconstruct over C^n (Alg. 3; SM3): (U, Lam) of the scaled
        X^ = U diag(Lam) U^*; no trace correction for the trace-bounded set (reading R37)."""
        return nystrom_reconstruct_c(self.S, self.Omega)

    def signal(self):
        """chi = sqrt(alpha lambda_1) u_1 in original units."""
        U, Lam = self.reconstruct()
        return np.sqrt(self.alpha * Lam[0]) * U[:, 0]

    def implicit_infeasibility(self):
        """||z - b~|| / ||b~|| (relative, scaled units)."""
        return float(np.linalg.norm(self.z - self.bt) / np.linalg.norm(self.bt))


def nystrom_reconstruct_c(S, Omega, max_retry: int = 40):
    """Alg. 3 over C^n: nu = sqrt(n) eps(||S||), S_nu = S + nu Omega, B = Omega^* S_nu (made
    Hermitian), C = chol(B) (B = C^* C), U Sigma ~ = svd(S_nu C^{-1}), Lam = max(Sigma^2 - nu, 0)."""
    n, R = S.shape
    nrm = float(np.linalg.norm(S, 2))
    if nrm == 0.0:
        return np.linalg.qr(Omega)[0], np.zeros(R)
    nu = np.sqrt(n) * matlab_eps(nrm)
    for _ in range(max_retry):
        Ss = S + nu * Omega
        B = Omega.conj().T @ Ss
        B = 0.5 * (B + B.conj().T)
        try:
            Lc = np.linalg.cholesky(B)                          # B = Lc Lc^*, C = Lc^*
            break
        except np.linalg.LinAlgError:
            nu *= 2.0
    else:
        raise np.linalg.LinAlgError("Cholesky failed after 40 shift doublings")
    Y = np.linalg.solve(Lc, Ss.conj().T).conj().T               # Y C = S_nu
    U, sv, _ = np.linalg.svd(Y, full_matrices=False)
    return U, np.maximum(0.0, sv ** 2 - nu)


def relative_error(chi, chi_nat):
    """min_phi ||e^{i phi} chi - chi_nat|| / ||chi_nat||, in closed form:
    ||chi||^2 + ||chi_nat||^2 - 2 |<chi, chi_nat>| at the minimizing phase."""
    a = float(np.real(np.vdot(chi, chi)))
    c = float(np.real(np.vdot(chi_nat, chi_nat)))
    return float(np.sqrt(max(a + c - 2.0 * abs(np.vdot(chi, chi_nat)), 0.0) / c))
