"""Pins of the CPU oracle against things other than itself.

Each test names the paper passage (P:<line> of PAPER.md) or SPEC.md worked
example (S:<line>) it checks, and the independent reference it uses: closed
forms, numpy/scipy dense eigensolvers, math.fsum / fractions, the dense
shadow CGAL iteration (Alg. 1), brute-force cut enumeration.
"""
import itertools
import math
from fractions import Fraction

import numpy as np
import pytest
import scipy.linalg as sla

import oracle
import scg_inputs as si


# ------------------------------------------------------------- CAC-2 exact sums
def test_xsum_equals_fsum_random_and_cancellation():
    rng = np.random.default_rng(0)
    for trial in range(50):
        n = int(rng.integers(1, 3000))
        scale = 10.0 ** rng.uniform(-30, 20, size=n)
        p = rng.standard_normal(n) * scale
        if trial % 3 == 0:  # heavy cancellation
            p = np.concatenate([p, -p[: n // 2], [1e-3]])
        assert oracle.xsum(p) == math.fsum(p)


def test_xsum_exact_cases():
    assert oracle.xsum([1e16, 1.0, -1e16]) == 1.0
    assert oracle.xsum([2.0 ** 53, 1.0, 1.0]) == 2.0 ** 53 + 2.0  # exact then one rounding
    assert oracle.xsum([2.0 ** 53, 1.0]) == 2.0 ** 53  # tie -> even
    assert oracle.xsum([2.0 ** 53 + 2.0, 1.0]) == 2.0 ** 53 + 4.0  # tie -> even (up)
    assert oracle.xsum([]) == 0.0
    # Q: truncation toward zero at 2^-200
    assert oracle.xsum([2.0 ** -210]) == 0.0
    assert oracle.xsum([-(2.0 ** -199 + 2.0 ** -230)]) == -(2.0 ** -199)
    x = 1.0 + 2.0 ** -52
    assert oracle.xsum([x * 2.0 ** -148]) == x * 2.0 ** -148  # last mantissa bit exactly 2^-200: kept
    assert oracle.xsum([x * 2.0 ** -149]) == 2.0 ** -149      # last bit 2^-201: truncated by Q
    with pytest.raises(OverflowError):
        oracle.xsum([2.0 ** 101])


def test_dot_is_exact_sum_of_rounded_products():
    rng = np.random.default_rng(1)
    a, b = rng.standard_normal(1000), rng.standard_normal(1000)
    assert oracle.dot(a, b) == math.fsum(a * b)
    exact = sum(Fraction(x) for x in a * b)
    assert abs(Fraction(oracle.dot(a, b)) - exact) <= Fraction(abs(float(exact))) * Fraction(2) ** -53


# ------------------------------------------------------------- CAC-3 row chains
def test_apply_integer_inputs_exact():
    # Small integers: every fma is exact, so the chain equals the dense product exactly.
    rng = np.random.default_rng(2)
    n = 40
    M = rng.integers(-5, 6, size=(n, n)).astype(float)
    M = M + M.T
    M[rng.random((n, n)) < 0.6] = 0.0
    M = np.triu(M, 1) + np.triu(M, 1).T + np.diag(np.diag(M))
    rp, col, m, d = oracle.offdiag_of_dense(M)
    x = rng.integers(-7, 8, size=n).astype(float)
    assert np.array_equal(oracle.apply(n, rp, col, m, d, x), M @ x)


def test_apply_rounding_bound():
    rng = np.random.default_rng(3)
    n = 30
    M = rng.standard_normal((n, n))
    M = M + M.T
    rp, col, m, d = oracle.offdiag_of_dense(M)
    x = rng.standard_normal(n)
    y = oracle.apply(n, rp, col, m, d, x)
    for r in range(n):
        exact = sum(Fraction(M[r, c]) * Fraction(x[c]) for c in range(n))
        bound = n * 2.0 ** -53 * float(np.sum(np.abs(M[r] * x))) * 1.01
        assert abs(float(Fraction(y[r]) - exact)) <= bound


def test_apply_long_rows_integer_exact_and_bounded():
    # Rows of > 32 entries take the strided partial chains (reading R27): still exact on
    # small integers, and within the summation rounding bound on real data.
    rng = np.random.default_rng(5)
    n = 300
    M = rng.integers(-5, 6, size=(n, n)).astype(float)
    M = np.triu(M, 1)
    M = M + M.T + np.diag(rng.integers(-9, 10, size=n).astype(float))
    rp, col, m, d = oracle.offdiag_of_dense(M)
    assert np.max(np.diff(rp)) > 200
    x = rng.integers(-7, 8, size=n).astype(float)
    assert np.array_equal(oracle.apply(n, rp, col, m, d, x), M @ x)
    Mr = rng.standard_normal((n, n))
    Mr = Mr + Mr.T
    rp, col, m, d = oracle.offdiag_of_dense(Mr)
    xr = rng.standard_normal(n)
    y = oracle.apply(n, rp, col, m, d, xr)
    for r in range(0, n, 37):
        exact = sum(Fraction(Mr[r, c]) * Fraction(xr[c]) for c in range(n))
        bound = n * 2.0 ** -53 * float(np.sum(np.abs(Mr[r] * xr))) * 1.01
        assert abs(float(Fraction(y[r]) - exact)) <= bound


def _fma(a, b, c):  # correctly rounded fma via exact rationals (float(Fraction) rounds to nearest)
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def test_apply_long_row_order_differs_from_single_chain():
    # The partial-chain order (R27) rounds differently from one left-to-right chain: on data
    # built to cancel the two orders give different bits, so the GPU parity tests pin the
    # order, not just the value.
    rng = np.random.default_rng(0)
    rng.standard_normal(69), rng.uniform(-20, 20, 69), rng.standard_normal(70)  # skip the first draw
    n = 70
    M = np.zeros((n, n))
    v = rng.standard_normal(n - 1) * np.exp(rng.uniform(-20, 20, n - 1))  # wide dynamic range
    M[0, 1:] = v
    M[1:, 0] = v
    x = rng.standard_normal(n)
    rp, col, m, d = oracle.offdiag_of_dense(M)
    y = oracle.apply(n, rp, col, m, d, x)
    acc = d[0] * x[0]
    for k in range(rp[0], rp[1]):
        acc = _fma(m[k], x[col[k]], acc)
    assert y[0] != acc


def test_apply_heavy_rows_integer_exact_and_bounded():
    # Rows of > 1024 entries take 256 strided partial chains (SURVEY CAC-2's W = 256 bin, reading
    # R27): exact on small integers, within the summation rounding bound on real data, and a
    # different rounding from the 32-chain order on cancelling data (so the bin boundary is pinned).
    rng = np.random.default_rng(8)
    n = 3000
    hub = rng.integers(-5, 6, size=n - 1).astype(float)
    hub[hub == 0] = 1.0
    i = np.zeros(n - 1, dtype=np.int64)
    j = np.arange(1, n)
    rp = np.zeros(n + 1, dtype=np.int64)
    rp[1] = n - 1
    rp[2:] = n - 1 + np.arange(1, n)
    col = np.concatenate([j, np.zeros(n - 1, dtype=np.int64)]).astype(np.int32)
    m = np.concatenate([hub, hub])
    d = rng.integers(-9, 10, size=n).astype(float)
    x = rng.integers(-7, 8, size=n).astype(float)
    y = oracle.apply(n, rp, col, m, d, x)
    assert y[0] == d[0] * x[0] + float(np.dot(hub, x[1:]))
    hr = rng.standard_normal(n - 1) * np.exp(rng.uniform(-15, 15, n - 1))
    xr = rng.standard_normal(n)
    mr = np.concatenate([hr, hr])
    y = oracle.apply(n, rp, col, mr, d, xr)
    exact = Fraction(d[0]) * Fraction(xr[0]) + sum(Fraction(a) * Fraction(b) for a, b in zip(hr, xr[1:]))
    bound = n * 2.0 ** -53 * (abs(d[0] * xr[0]) + float(np.sum(np.abs(hr * xr[1:])))) * 1.01
    assert abs(float(Fraction(y[0]) - exact)) <= bound
    L32 = [0.0] * 32  # the W = 32 order the row would take below the bin boundary
    for k in range(n - 1):
        L32[k % 32] = _fma(hr[k], xr[1 + k], L32[k % 32])
    off = 16
    while off >= 1:
        for l in range(off):
            L32[l] = L32[l] + L32[l + off]
        off //= 2
    assert y[0] != d[0] * xr[0] + L32[0]


# ------------------------------------------------------------- Laplacian
def test_laplacian_identities():
    L = si.laplacian("c0")
    Ld = L.dense()
    assert np.allclose(Ld @ np.ones(L.n), 0.0)
    rng = np.random.default_rng(4)
    x = rng.standard_normal(L.n)
    assert math.isclose(x @ Ld @ x, oracle.laplacian_quadratic(L, x), rel_tol=1e-12)
    # single edge and triangle (SPEC S:431-432 examples)
    L1 = si.laplacian_from_edges(2, [0], [1], [1.0])
    assert np.array_equal(L1.dense(), np.array([[1.0, -1.0], [-1.0, 1.0]]))
    L3 = si.laplacian_from_edges(3, [0, 0, 1], [1, 2, 2], [1.0, 1.0, 1.0])
    assert np.array_equal(L3.dense(), 3 * np.eye(3) - np.ones((3, 3)))


# ------------------------------------------------------------- schedules
def test_qt_schedule_examples():
    assert oracle.qt(1, 100) == 5
    assert oracle.qt(16, 100) == 10
    assert oracle.qt(7, 3) == 2     # S:144 (clip to n - 1)
    # config[0] / config[3] ranges quoted in SURVEY.md section 8
    assert oracle.qt(1, 800) == 7 and oracle.qt(1000, 800) == 38
    assert oracle.qt(1, 1 << 24) == 17 and oracle.qt(1000, 1 << 24) == 94


def test_gamma_examples():
    # eqn:sketchy-cgal-dual-step
    assert oracle.gamma(1, 1.0, 1.0, 1.0) == 1.0
    assert oracle.gamma(3, 1.0, 1.0, 2.0) == 0.25
    assert oracle.gamma(5, 1.0, 1.0, 0.0) == 1.0
    for t in (1, 10, 100):
        for nz in (1e-8, 1e-3, 1.0, 1e3):
            g = oracle.gamma(t, 1.0, 1.0, nz)
            assert 0.0 <= g <= 1.0
            assert g * nz <= 4.0 / (t + 1) ** 1.5 * (1 + 1e-15)


# ------------------------------------------------------------- tridiagonal (Alg. 2 lines 11-12)
def test_tridiag_worked_examples():
    th, s = oracle.tridiag_mineig([2.0], [])
    assert th == 2.0 and s[0] == 1.0
    th, s = oracle.tridiag_mineig([0.0, 0.0], [1.0])
    assert abs(th + 1.0) < 1e-15
    s = s / np.linalg.norm(s)
    assert np.allclose(np.abs(s), [2 ** -0.5, 2 ** -0.5], atol=1e-15) and s[0] * s[1] < 0
    th, s = oracle.tridiag_mineig([1.0, 2.0, 3.0], [0.0, 0.0])  # S:135 decoupled
    assert abs(th - 1.0) < 1e-15
    assert np.allclose(s / np.linalg.norm(s), [1.0, 0.0, 0.0], atol=1e-12)


def test_tridiag_toeplitz_closed_form():
    for k in (3, 10, 50, 94):
        a, b = 0.3, 0.7
        th, s = oracle.tridiag_mineig(np.full(k, a), np.full(k - 1, b))
        lam = a - 2 * b * math.cos(math.pi / (k + 1))
        assert abs(th - lam) <= 1e-14 * (abs(a) + 2 * b)
        j = np.arange(1, k + 1)
        ref = np.sin(j * k * math.pi / (k + 1))  # eigenvector of the smallest eigenvalue
        s = s / np.linalg.norm(s)
        ref = ref / np.linalg.norm(ref)
        assert min(np.linalg.norm(s - ref), np.linalg.norm(s + ref)) < 1e-10


def test_tridiag_vs_lapack():
    rng = np.random.default_rng(5)
    for trial in range(200):
        k = int(rng.integers(2, 95))
        om = rng.standard_normal(k) * 10 ** rng.uniform(-3, 3)
        rho = np.abs(rng.standard_normal(k - 1)) * 10 ** rng.uniform(-3, 3)
        th, s = oracle.tridiag_mineig(om, rho)
        w, V = sla.eigh_tridiagonal(om, rho)
        NT = max(np.abs(om).max() + 2 * rho.max(), 1e-300)
        assert abs(th - w[0]) <= 1e-12 * NT
        T = np.diag(om) + np.diag(rho, 1) + np.diag(rho, -1)
        sn = s / np.linalg.norm(s)
        assert np.linalg.norm(T @ sn - w[0] * sn) <= 1e-9 * NT
        jm = int(np.argmax(np.abs(s)))
        assert s[jm] > 0  # sign convention


# ------------------------------------------------------------- Lanczos (Alg. 2)
def _rand_sym(n, rng):
    A = rng.standard_normal((n, n))
    return (A + A.T) / 2


def test_lanczos_full_krylov_is_exact():
    # test-only q = n (reading A4): the Krylov space is everything -> theta = lambda_min
    rng = np.random.default_rng(6)
    for n in (3, 5, 8, 12):
        M = _rand_sym(n, rng)
        rp, col, m, d = oracle.offdiag_of_dense(M)
        g = rng.standard_normal(n)
        r = oracle.lanczos(n, rp, col, m, d, g, n)
        lam = np.linalg.eigvalsh(M)
        nrm = np.abs(lam).max()
        assert abs(r.theta - lam[0]) <= 1e-10 * nrm
        assert abs(r.v @ M @ r.v - lam[0]) <= 1e-9 * nrm
        assert abs(np.linalg.norm(r.v) - 1.0) < 1e-14


def test_lanczos_spec_examples():
    # S:125 diag(-2, 1, 5) with the full Krylov space -> (-2, +-e1)
    M = np.diag([-2.0, 1.0, 5.0])
    rp, col, m, d = oracle.offdiag_of_dense(M)
    r = oracle.lanczos(3, rp, col, m, d, np.array([0.3, -1.1, 0.7]), 3)
    assert abs(r.theta + 2.0) < 1e-12
    assert abs(abs(r.v[0]) - 1.0) < 1e-10
    # S:124 M = I: rho_1 = 0 up to rounding -> invariant subspace break (reading A3), xi = 1
    M = np.eye(3)
    rp, col, m, d = oracle.offdiag_of_dense(M)
    r = oracle.lanczos(3, rp, col, m, d, np.array([0.3, -1.1, 0.7]), 3)
    assert r.k == 1 and abs(r.theta - 1.0) <= 4e-16


def test_lanczos_matches_dense_rayleigh_ritz():
    # Before orthogonality is lost the Ritz value equals lambda_min of V^T M V with V the Krylov basis
    rng = np.random.default_rng(7)
    n, q = 300, 6
    M = _rand_sym(n, rng)
    rp, col, m, d = oracle.offdiag_of_dense(M)
    g = rng.standard_normal(n)
    r = oracle.lanczos(n, rp, col, m, d, g, q)
    K = np.empty((n, q))
    K[:, 0] = g
    for j in range(1, q):
        K[:, j] = M @ K[:, j - 1]
    Q, _ = np.linalg.qr(K)
    H = Q.T @ M @ Q
    lam = np.linalg.eigvalsh(H)[0]
    assert abs(r.theta - lam) <= 1e-10 * np.abs(np.linalg.eigvalsh(M)).max()
    # interlacing: never below lambda_min(M)
    assert r.theta >= np.linalg.eigvalsh(M)[0] - 1e-12 * np.abs(M).max()
    # the returned unit vector realises (close to) the Ritz value
    assert abs(r.v @ M @ r.v - r.theta) < 1e-9


def test_lanczos_fact_41_statistical():
    # Fact 4.1: n=100, eps=1, delta=1/4, q = ceil(1/2 + log(n/delta^2)) = 8
    rng = np.random.default_rng(8)
    n, q, trials, ok = 100, 8, 200, 0
    M = _rand_sym(n, rng)
    rp, col, m, d = oracle.offdiag_of_dense(M)
    lam = np.linalg.eigvalsh(M)
    nrm = np.abs(lam).max()
    for t in range(trials):
        r = oracle.lanczos(n, rp, col, m, d, si.normals(99, 1, t, 0, n), q)
        ok += (r.v @ M @ r.v) <= lam[0] + nrm / 8
    assert ok / trials >= 0.5


# ------------------------------------------------------------- Alg. 4 loop invariants
def _shadow_cgal(L, o, T, beta0=1.0):
    """Dense CGAL (Alg. 1) driven by the oracle's v_t; returns per-t shadow states."""
    n = L.n
    Lam = L.dense()
    nrm = np.sqrt((Lam ** 2).sum())
    C = -Lam / nrm
    alpha, b = 1.0, 1.0 / n
    X = np.zeros((n, n))
    y = np.zeros(n)
    V = o.vhist
    out = []
    for t in range(1, T + 1):
        beta = beta0 * math.sqrt(t + 1)
        eta = 2.0 / (t + 1)
        Dt = C + np.diag(y + beta * (np.diag(X) - b))
        lam_min = np.linalg.eigvalsh(Dt)[0]
        v = V[t - 1]
        X = (1 - eta) * X + eta * alpha * np.outer(v, v)
        zb = np.diag(X) - b
        nz = zb @ zb
        gam = beta0 if nz == 0 else min(beta0, 4 * alpha ** 2 * beta0 / ((t + 1) ** 1.5 * nz))
        y = y + gam * zb
        out.append(dict(X=X.copy(), y=y.copy(), lam_min=lam_min, C=C))
    return out


def test_loop_invariants_shadow_cgal():
    # eqn:loop-invariant: z = A X_t, S = X_t Omega, tau = tr X_t, p = <C, X_t>
    L = si.laplacian_from_edges(14, *zip(*[(i, j, 1.0) for i in range(14) for j in range(i + 1, 14)
                                            if (i * 7 + j * 3) % 5 < 2]))
    n, R, T = L.n, 4, 60
    o = oracle.Oracle(L, R, seed=11, logcap=T, vhist=T, qfix=n)  # full Krylov space -> exact min eigvec
    o.step(T)
    sh = _shadow_cgal(L, o, T)
    X = sh[-1]["X"]
    assert np.allclose(o.z, np.diag(X), atol=1e-14, rtol=1e-12)
    assert np.allclose(o.S, X @ o.Omega, atol=1e-13, rtol=1e-11)
    assert math.isclose(o.tau, np.trace(X), rel_tol=1e-13)
    assert math.isclose(o.p, float(np.sum(sh[-1]["C"] * X)), rel_tol=1e-11, abs_tol=1e-15)
    assert np.allclose(o.y, sh[-1]["y"], rtol=1e-9, atol=1e-13)
    lg = o.log
    for t in range(T):
        # with the full Krylov space the Ritz value is lambda_min(D_t) (D_t assembled densely)
        assert abs(lg[t, 3] - sh[t]["lam_min"]) <= 1e-9 * (1 + abs(sh[t]["lam_min"]))
        assert abs(lg[t, 4] - lg[t, 3]) <= 1e-9 * (1 + abs(lg[t, 3]))  # xi = v* D v
    # tr X_t = alpha for t >= 1 (eta_1 = 1)
    assert abs(o.z.sum() - 1.0) < 1e-13 and abs(o.tau - 1.0) < 1e-13


def test_unscaled_variant_invariants():
    L = si.laplacian("c0")
    o = oracle.Oracle(L, 5, seed=0, scale=False, logcap=30)
    o.step(30)
    assert math.isclose(o.z.sum(), L.n, rel_tol=1e-12)  # tr X = alpha = n
    assert o.b == 1.0 and o.alpha == L.n


# ------------------------------------------------------------- SDP value closed forms + brute force
def _edges_graph(n, edges):
    i, j = zip(*edges)
    return si.laplacian_from_edges(n, i, j, [1.0] * len(edges))


@pytest.mark.parametrize("name,n,edges,sdp", [
    ("C5", 5, [(k, (k + 1) % 5) for k in range(5)], 10 * (1 + math.cos(math.pi / 5))),  # odd cycle 2n(1+cos(pi/n))
    ("C8", 8, [(k, (k + 1) % 8) for k in range(8)], 4 * 8),  # bipartite: 4 sum w
    ("K6", 6, [(i, j) for i in range(6) for j in range(i + 1, 6)], 36.0),  # K_n: n^2
])
def test_sdp_value_closed_forms(name, n, edges, sdp):
    L = _edges_graph(n, edges)
    o = oracle.Oracle(L, 3, seed=5, logcap=1)
    o.step(3000)
    val = o.implicit_objective()
    assert abs(val - sdp) / sdp < 3e-3, (name, val, sdp)


def _brute_maxcut(L):
    i, j, w = L.edges()
    best = -1.0
    for bits in itertools.product([1, -1], repeat=L.n - 1):
        chi = np.array((1,) + bits)
        best = max(best, float(np.sum(w * (chi[i] != chi[j]))))
    return best


def test_rounded_cut_vs_brute_force():
    rng = np.random.default_rng(9)
    for trial in range(4):
        n = 12
        edges = [(a, b) for a in range(n) for b in range(a + 1, n) if rng.random() < 0.4]
        L = _edges_graph(n, edges)
        res = oracle.solve(L, R=4, T=400, seed=trial)
        opt = _brute_maxcut(L)
        assert res["cut_weight"] <= opt + 1e-9
        assert res["cut_weight"] >= 0.878 * opt * 0.9   # sign rounding gives a good cut here
        assert res["implicit_objective"] >= 4 * opt * (1 - 2e-2)  # relaxation dominates
    # bipartite: the rounded cut is the optimum (all edges)
    edges = [(a, b) for a in range(6) for b in range(6, 12) if (a + b) % 3]
    L = _edges_graph(12, edges)
    res = oracle.solve(L, R=4, T=400, seed=1)
    assert res["cut_weight"] == len(edges) == _brute_maxcut(L)


def test_weak_duality_certificate():
    # eqn:model-dual-function-supp: alpha lambda_min(C + A* y) - <y, b> <= p* (scaled, minimize)
    L = si.laplacian("c0")
    o = oracle.Oracle(L, 4, seed=0, logcap=1)
    o.step(300)
    C = -L.dense() / o.nrmL
    lb = 1.0 * np.linalg.eigvalsh(C + np.diag(o.y))[0] - o.y.sum() / L.n
    ub_orig = -lb * o.nrmL * L.n  # upper bound on max tr(L X)
    val = o.implicit_objective()
    assert ub_orig >= val * (1 - 5e-3)
    assert (ub_orig - val) / val < 5e-2


# ------------------------------------------------------------- Nystrom (Alg. 3 / SM3)
def test_matlab_eps():
    assert oracle.matlab_eps(1.0) == 2.0 ** -52
    assert oracle.matlab_eps(3.0) == 2.0 ** -51
    assert oracle.matlab_eps(0.75) == 2.0 ** -53


def test_nystrom_exact_recovery_low_rank():
    # rank(X) <= R -> X^ = X with probability one
    rng = np.random.default_rng(10)
    n, r, R = 60, 3, 6
    G = rng.standard_normal((n, r))
    X = G @ G.T
    Om = rng.standard_normal((n, R))
    U, Lam, err = oracle.nystrom_reconstruct(X @ Om, Om, np.trace(X))
    Xh = U @ np.diag(Lam) @ U.T
    assert np.linalg.norm(Xh - X) <= 1e-9 * np.linalg.norm(X)
    assert np.allclose(U.T @ U, np.eye(R), atol=1e-12)
    assert np.all(np.diff(Lam) <= 1e-12) and np.all(Lam >= 0)
    assert abs(err[r - 1]) <= 1e-9 * np.trace(X)


def test_nystrom_error_identity_and_trace_correction():
    rng = np.random.default_rng(11)
    n, R = 40, 8
    for trial in range(20):
        G = rng.standard_normal((n, n)) * (0.7 ** np.arange(n))
        X = G @ G.T
        Om = rng.standard_normal((n, R))
        U, Lam, err = oracle.nystrom_reconstruct(X @ Om, Om, np.trace(X))
        # err_r = ||X - [X^]_r||_* -- X - [X^]_r is psd so the nuclear norm is its trace
        for rr in (1, 3, R):
            Xr = U[:, :rr] @ np.diag(Lam[:rr]) @ U[:, :rr].T
            nuc = np.abs(np.linalg.eigvalsh(X - Xr)).sum()
            assert abs(err[rr - 1] - nuc) <= 1e-8 * np.trace(X)
        # err nonincreasing in r and bounds the best rank-r error
        assert np.all(np.diff(err) <= 1e-9 * np.trace(X))
        ev = np.sort(np.linalg.eigvalsh(X))[::-1]
        assert np.all(ev[R:].sum() <= err[-1] + 1e-9 * np.trace(X))
        # trace correction at most doubles the error
        Lt = oracle.trace_correct(Lam, np.trace(X))
        e_hat = np.abs(np.linalg.eigvalsh(X - U @ np.diag(Lam) @ U.T)).sum()
        e_til = np.abs(np.linalg.eigvalsh(X - U @ np.diag(Lt) @ U.T)).sum()
        assert e_til <= 2 * e_hat * (1 + 1e-9) + 1e-12
        assert math.isclose(Lt.sum(), np.trace(X), rel_tol=1e-13)


def test_trace_correct_example():
    assert np.allclose(oracle.trace_correct([0.5, 0.3], 1.0), [0.6, 0.4])


def test_fact_51_mean_bound():
    # Fact 5.1: E ||X - X^||_* <= (1 + r/(R-r-1)) ||X - [X]_r||_*
    rng = np.random.default_rng(12)
    n, R, r = 50, 12, 5
    G = rng.standard_normal((n, n)) * (0.8 ** np.arange(n))
    X = G @ G.T
    ev = np.sort(np.linalg.eigvalsh(X))[::-1]
    tail = ev[r:].sum()
    errs = []
    for t in range(300):
        Om = rng.standard_normal((n, R))
        U, Lam, _ = oracle.nystrom_reconstruct(X @ Om, Om)
        errs.append(np.abs(np.linalg.eigvalsh(X - U @ np.diag(Lam) @ U.T)).sum())
    assert np.mean(errs) <= (1 + r / (R - r - 1)) * tail * 1.1


# ------------------------------------------------------------- rounding
def test_rounding_examples():
    L3 = si.laplacian_from_edges(3, [0, 0, 1], [1, 2, 2], [1.0, 1.0, 1.0])
    assert oracle.cut_weight(L3, [1, 1, -1]) == 2.0  # SPEC triangle example
    chi = np.array([1, 1, -1])
    assert oracle.cut_weight(L3, chi) == 0.25 * chi @ L3.dense() @ chi
    P3 = si.laplacian_from_edges(3, [0, 1], [1, 2], [1.0, 1.0])
    c, w, k = oracle.round_cut(P3, np.array([[1.0], [-1.0], [1.0]]))
    assert w == 2.0 == _brute_maxcut(P3)
    c, w, k = oracle.round_cut(P3, np.array([[-0.0], [0.0], [0.0]]))  # sgn(0)=+1
    assert w == 0.0
    C5 = _edges_graph(5, [(k, (k + 1) % 5) for k in range(5)])
    K4 = _edges_graph(4, [(i, j) for i in range(4) for j in range(i + 1, 4)])
    assert _brute_maxcut(P3) == 2 and _brute_maxcut(C5) == 4 and _brute_maxcut(K4) == 4


# ------------------------------------------------------------- f2: gap and posterior bound
def test_posterior_bound_dominates_suboptimality():
    """eqn:scgal-posterior-error-bd: with the exact lambda_min(D_t), the bound
    p_t + <y_t, b> + beta_t/2 <z_t - b, z_t + b> - alpha lambda_min(D_t) is >= p_t - p_star,
    p_star from the closed-form SDP value of an odd cycle (2n(1+cos(pi/n))).  The logged bound
    uses xi_t >= lambda_min, so it is <= the exact one; gap - bound equals
    <y_t, z_t - b> + beta_t/2 ||z_t - b||^2 (P:1557 derivation)."""
    n = 5
    L = _edges_graph(n, [(k, (k + 1) % n) for k in range(n)])
    sdp = 2 * n * (1 + math.cos(math.pi / n))
    T = 600
    o = oracle.Oracle(L, 3, seed=11, logcap=T + 1)
    Ld = L.dense()
    prev_bound = None
    for t in (5, 50, 600):
        o.step(t - o.t)
        y, z, p, b, alpha = o.y.copy(), o.z.copy(), o.p, o.b, o.alpha
        p_star = -sdp / (n * o.nrmL)
        beta = 1.0 * math.sqrt(t + 2)  # beta of iteration t+1 (state before its update)
        D = -Ld / o.nrmL + np.diag(y + beta * (z - b))
        lam = float(np.linalg.eigvalsh(D)[0])
        bound_exact = p + b * y.sum() + 0.5 * beta * float(np.dot(z - b, z + b)) - alpha * lam
        assert p - p_star <= bound_exact + 1e-12, (t, p - p_star, bound_exact)
        if prev_bound is not None:
            assert bound_exact < prev_bound
        prev_bound = bound_exact
        # the record of iteration t+1 (same state) once that iteration has run
        o.step(1)
        rec = o.log[t]
        assert rec[11] <= bound_exact + 1e-12
        ident = float(np.dot(y, z - b)) + 0.5 * beta * float(np.dot(z - b, z - b))
        assert abs((rec[10] - rec[11]) - ident) <= 1e-12 * max(1.0, abs(rec[10]))


# ------------------------------------------------------------- f3: trace-bounded LMO
def test_trace_bounded_sdp_value_and_trace():
    """tr X <= 1.05 n with H = 0 when xi_t >= 0: diag X = 1 still forces
    tr X = n at the optimum, so the closed-form SDP value of C5 is recovered; the tracked trace
    tau_t = tr X_t never exceeds alpha; the H = 0 branch does fire."""
    n = 5
    L = _edges_graph(n, [(k, (k + 1) % n) for k in range(n)])
    sdp = 2 * n * (1 + math.cos(math.pi / n))
    o = oracle.Oracle(L, 3, seed=5, logcap=3000, alpha=1.05 * n, trace_le=True)
    o.step(3000)
    assert abs(o.implicit_objective() - sdp) / sdp < 3e-3
    assert np.all(o.log[:, 9] <= o.alpha * (1 + 1e-14))
    assert np.any(o.log[:, 4] >= 0.0)  # some iterations took H = 0
    # equality run for comparison: same limit
    oe = oracle.Oracle(L, 3, seed=5, logcap=1)
    oe.step(3000)
    assert abs(o.implicit_objective() - oe.implicit_objective()) / sdp < 3e-3


def test_alpha_doubling_standard_form_driver():
    """Remark "Standard-form SDP" on C5 (closed-form SDP value, P-independent):
    diag X = 1 forces tr X = n, so a bound alpha < n scales the optimum to (alpha / n) X* with
    objective (alpha / n) * SDP, and every alpha >= n gives the SDP itself.  From alpha0 = n/4 the
    driver doubles through n/4, n/2, n and stops at 2n (objective repeated within rtol) with the
    SDP value; from alpha0 >= n it stops after two rounds."""
    n = 5
    L = _edges_graph(n, [(k, (k + 1) % n) for k in range(n)])
    sdp = 2 * n * (1 + math.cos(math.pi / n))
    o, al, ob, conv = oracle.alpha_doubling(L, 3, alpha0=n / 4, T=3000, rtol=1e-2, seed=5)
    assert conv
    np.testing.assert_array_equal(al, (n / 4) * 2.0 ** np.arange(4))
    for a, v in zip(al, ob):
        assert abs(v - min(a / n, 1.0) * sdp) <= 3e-3 * sdp
    assert o.alpha_orig == 2 * n
    o2, al2, ob2, conv2 = oracle.alpha_doubling(L, 3, alpha0=1.05 * n, T=3000, rtol=1e-2, seed=5)
    assert conv2 and len(al2) == 2 and abs(ob2[-1] - sdp) <= 3e-3 * sdp
    # max_rounds caps an unconverged sequence
    _, al3, _, conv3 = oracle.alpha_doubling(L, 3, alpha0=n / 4, T=3000, rtol=1e-2, seed=5, max_rounds=2)
    assert not conv3 and len(al3) == 2


def test_inequality_template_closed_forms():
    """General template with K = {u <= b} (SCG_INEQ): MaxCut with
    diag X <= 1.  On C5 the optimum still has diag X = 1 (L is psd), so the closed-form SDP value
    is recovered; with tr X <= n/2 as well, the equality problem is infeasible while the
    inequality one has the vertex-transitive optimum (1/2) X*, value SDP/2, and a feasible
    iterate (z <= b).  The gap / bound records are the general-template ones (reading R33): finite,
    and the gap shrinks toward 0."""
    n = 5
    L = _edges_graph(n, [(k, (k + 1) % n) for k in range(n)])
    sdp = 2 * n * (1 + math.cos(math.pi / n))
    o = oracle.Oracle(L, 3, seed=5, logcap=3000, ineq=True)
    o.step(3000)
    assert abs(o.implicit_objective() - sdp) <= 3e-3 * sdp
    assert np.all(np.isfinite(o.log[:, 10:12]))
    assert abs(o.log[-1, 10]) < 0.05 * abs(o.log[4, 10])
    h = oracle.Oracle(L, 3, seed=5, logcap=3000, ineq=True, trace_le=True, alpha=n / 2)
    h.step(3000)
    assert abs(h.implicit_objective() - sdp / 2) <= 3e-3 * sdp
    z = h.z * (h.alpha_orig / h.alpha)  # diag X_T in original units
    assert np.all(z <= 1.0 + 1e-3) and abs(z.sum() - n / 2) <= 1e-2 * n


def test_box_constraint_set_closed_forms():
    """Box K = {lo <= u <= hi} (the l_inf ball |u - 1| <= delta of P:3915-3918): on C5 with
    diag X in [1 - delta, 1 + delta] and tr X <= 1.05 n (1 + delta) the optimum is (1 + delta) X*,
    value (1 + delta) SDP.  Special cases: lo = hi = 1 is the equality problem (every iterate bitwise,
    the general-template gap / bound equal to rounding), lo = -inf, hi = 1 is SCG_INEQ (bitwise)."""
    n = 5
    L = _edges_graph(n, [(k, (k + 1) % n) for k in range(n)])
    sdp = 2 * n * (1 + math.cos(math.pi / n))
    for d in (0.1, 0.3):
        o = oracle.Oracle(L, 3, seed=5, logcap=3000, box=(1 - d, 1 + d), trace_le=True, alpha=1.05 * n * (1 + d))
        o.step(3000)
        assert abs(o.implicit_objective() - (1 + d) * sdp) <= 3e-3 * sdp
        z = o.z * (o.alpha_orig / o.alpha)
        assert np.all(np.abs(z - (1 + d)) <= 5e-3)
    e = oracle.Oracle(L, 3, seed=5, logcap=300)
    e.step(300)
    b = oracle.Oracle(L, 3, seed=5, logcap=300, box=(1.0, 1.0))
    b.step(300)
    np.testing.assert_array_equal(b.log[:, :10], e.log[:, :10])
    np.testing.assert_array_equal(b.z, e.z)
    # the general-template gap / bound (reading R33) with w = b are the equality ones, up to rounding
    np.testing.assert_allclose(b.log[:, 10:12], e.log[:, 10:12], rtol=1e-11, atol=1e-14)
    i1 = oracle.Oracle(L, 3, seed=5, logcap=300, box=(-np.inf, 1.0))
    i1.step(300)
    i2 = oracle.Oracle(L, 3, seed=5, logcap=300, ineq=True)
    i2.step(300)
    np.testing.assert_array_equal(i1.log, i2.log)
    np.testing.assert_array_equal(i1.y, i2.y)


# ------------------------------------------------------------- one-shot metrics
def test_objective_and_feasibility_hat_bipartite_cut_closed_form():
    """X^ = chi chi^T for a cut chi of a bipartite graph with every edge crossing: tr(L X^) = chi^T L chi
    = sum_E w (chi_i - chi_j)^2 = 4 sum w (eqn:comb-laplacian P:97-100) and diag X^ = 1, so both
    infeasibility normalizations are 0 (BASELINE)."""
    rng = np.random.default_rng(4)
    a, b = 7, 9
    edges = [(i, a + j) for i in range(a) for j in range(b) if rng.random() < 0.5]
    i, j = zip(*edges)
    w = rng.uniform(0.5, 2.0, size=len(edges))
    L = si.laplacian_from_edges(a + b, i, j, w)
    chi = np.array([1.0] * a + [-1.0] * b)
    n = a + b
    U = (chi / np.sqrt(n))[:, None]
    Lam = np.array([float(n)])
    assert abs(oracle.objective_hat(L, U, Lam) - 4.0 * w.sum()) <= 1e-12 * 4.0 * w.sum()
    f1, f2 = oracle.feasibility_hat(U, Lam)
    assert f1 <= 1e-14 and f2 <= 1e-14


@pytest.mark.parametrize("a,b", [(3.0, 1.0), (0.5, 2.25), (4.0, 0.0)])
def test_objective_and_feasibility_hat_rank2_closed_form(a, b):
    """Hand-built rank-2 X^ on the 4-cycle C_4 (unit weights): u1 = 1/2 (1,1,1,1), u2 = 1/2 (1,-1,1,-1),
    Lambda = (a, b).  u1^T L u1 = 0 (L 1 = 0), u2^T L u2 = sum over the 4 edges of (u_i - u_j)^2 = 4,
    so tr(L X^) = 4 b; diag X^ = (a + b)/4 in every entry, so ||diag X^ - 1|| = 2 |(a + b)/4 - 1| and the
    two normalizations divide it by ||1|| = 2 and 1 + ||1|| = 3."""
    L = _edges_graph(4, [(0, 1), (1, 2), (2, 3), (3, 0)])
    U = 0.5 * np.array([[1.0, 1.0], [1.0, -1.0], [1.0, 1.0], [1.0, -1.0]])
    Lam = np.array([a, b])
    assert abs(oracle.objective_hat(L, U, Lam) - 4.0 * b) <= 1e-14 * max(1.0, 4.0 * b)
    r = 2.0 * abs((a + b) / 4.0 - 1.0)
    f1, f2 = oracle.feasibility_hat(U, Lam)
    assert abs(f1 - r / 2.0) <= 1e-15 and abs(f2 - r / 3.0) <= 1e-15


@pytest.mark.parametrize("n", [4, 6, 9])
def test_implicit_objective_and_infeasibility_star_closed_form(n):
    """Star K_{1,n-1}: L has eigenvalues 0, 1 (n-2 times) and n, with the simple top eigenvector
    (n-1, -1, ..., -1)/sqrt(n(n-1)).  At t = 1 (z = y = 0) D_1 = -L/||L||_F - beta_1 b I, whose minimum
    eigenvector is that top vector; the full Krylov space (q = n; three distinct eigenvalues, so the
    Krylov space is exhausted after 3 steps) gives it to rounding.  With eta_1 = 1 the implicit iterate is
    X_2 = alpha v v^T, so in original units z = n (v o v) = (n-1, 1/(n-1), ..., 1/(n-1)):
      ||z - 1|| / (1 + sqrt n) = sqrt((n-2)^2 + (n-1)(1/(n-1) - 1)^2) / (1 + sqrt n)
      tr(L X_2) = n lambda_max(L) = n^2."""
    L = _edges_graph(n, [(0, j) for j in range(1, n)])
    o = oracle.Oracle(L, 2, seed=11, qfix=n, logcap=1)
    o.step(1)
    want = math.sqrt((n - 2) ** 2 + (n - 1) * (1.0 / (n - 1) - 1.0) ** 2) / (1.0 + math.sqrt(n))
    assert abs(o.implicit_infeasibility() - want) <= 1e-12 * want
    assert abs(o.implicit_objective() - n * n) <= 1e-12 * n * n


def test_implicit_infeasibility_balanced_cycle_is_zero():
    """Even cycle C_8: the top eigenvector of L is the alternating vector (eigenvalue 4, simple), so
    v o v = 1/n exactly up to rounding at every t (z = b, y = 0 keep D_t = C - beta b I): the implicit
    iterate is feasible, ||z - b|| = 0 to rounding for all t."""
    L = _edges_graph(8, [(k, (k + 1) % 8) for k in range(8)])
    o = oracle.Oracle(L, 2, seed=3, qfix=8, logcap=5)
    o.step(5)
    assert o.implicit_infeasibility() <= 1e-11
    assert abs(o.implicit_objective() - 8 * 4.0) <= 1e-12 * 32.0


# ------------------------------------------------------------- reading R26 (normalization by a reciprocal)
def test_r26_reciprocal_normalization_within_noise_floor():
    """Reading R26 evaluates Alg. 2 line 9's v / rho as v * fl(1/rho) (<= 1 ulp per entry from the
    printed division).  Pin: the oracle with the literal division (div_norm) on configs[0] stays within
    the noise floor any rounding-level change produces without reorthogonalization (SURVEY.md Appendix A:
    two fp64 implementations differing in summation order agree to ~1e-12 in theta_t only for t <~ 20,
    the objective to ~1e-4): theta_t within 1e-10 relative for t <= 20, the implicit objective after
    T = 1000 within 1e-4, and the rounded cut weight within 0.5%."""
    L = si.laplacian("c0")
    T = 1000
    a = oracle.solve(L, 10, T, seed=0)
    o2 = oracle.Oracle(L, 10, seed=0, logcap=T, div_norm=True)
    o2.step(T)
    th, th2 = a["oracle"].log[:, 3], o2.log[:, 3]
    assert np.max(np.abs(th[:20] - th2[:20]) / np.abs(th[:20])) <= 1e-10
    assert not np.array_equal(th, th2)  # the two forms are different roundings
    o_a, o_b = a["implicit_objective"], o2.implicit_objective()
    assert abs(o_a - o_b) <= 1e-4 * abs(o_a)
    U2, lam2, _ = oracle.nystrom_reconstruct(o2.S, o2.Omega, o2.tau)
    _, w2, _ = oracle.round_cut(L, U2)
    assert abs(w2 - a["cut_weight"]) <= 5e-3 * a["cut_weight"]


# ------------------------------------------------------------- OpenMP (thread count is bitwise-neutral)
def test_thread_count_does_not_change_bits():
    """The exact sums (CAC-2) are integer sums, and the row loops are independent, so 1 thread and all
    cores give identical bits (checked on a graph above the oracle's 65536-row parallel threshold)."""
    L = si.generate("rgg", 1 << 17, seed=5)
    runs = []
    for th in (1, 0):
        oracle.set_threads(th)
        o = oracle.Oracle(L, 3, seed=5, logcap=2)
        o.step(2)
        runs.append((o.log.copy(), o.z, o.y, o.v, o.S))
    oracle.set_threads(0)
    for x, y in zip(*runs):
        np.testing.assert_array_equal(x, y)


def test_qt_has_no_cap():
    """q_t = min(n - 1, max(2, ceil(t^(1/4) ln n))) (reading A9) with no other bound: for
    n = 2^25 and t = 10^6 it is ceil(31.62... * 17.33...) = 549 (the earlier oracle capped it at 127)."""
    assert oracle.qt(10 ** 6, 1 << 25) == math.ceil(math.sqrt(math.sqrt(1e6)) * math.log(2.0 ** 25))
    assert oracle.qt(10 ** 6, 1 << 25) > 127
    assert oracle.qt(10 ** 6, 100) == 99


def test_lanczos_beyond_127_steps_dense_rayleigh_ritz():
    """Alg. 2 with q = 160 > 127 on a 400 x 400 matrix with a well separated bottom eigenvalue: theta is
    lambda_min (dense eigh) to 1e-10 ||D|| and the vector's Rayleigh quotient matches."""
    rng = np.random.default_rng(7)
    n = 400
    Q = np.linalg.qr(rng.standard_normal((n, n)))[0]
    ev = np.concatenate([[-3.0], rng.uniform(0.0, 1.0, n - 1)])
    M = (Q * ev) @ Q.T
    M = 0.5 * (M + M.T)
    rp, col, m, d = oracle.offdiag_of_dense(M)
    g = si.normals(3, 1, 1, 0, n)
    res = oracle.lanczos(n, rp, col, m, d, g, 160)
    lmin = np.linalg.eigvalsh(M)[0]
    assert res.k == 160 or res.k < 160  # no cap below q
    assert abs(res.theta - lmin) <= 1e-10 * np.abs(ev).max()
    assert abs(res.v @ M @ res.v - lmin) <= 1e-8


# ------------------------------------------------------------- golden fixtures come from the oracle
def test_golden_fixture_reproduces_from_oracle():
    """tests/golden/*.json are written by tests/golden/make_golden.py from oracle/ only; the cheap case
    is regenerated here and must match the stored fixture exactly (log, digests, S sample)."""
    import json
    import os
    import sys
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    sys.path.insert(0, here)
    import make_golden
    fresh = make_golden.make("c1_q255")
    with open(os.path.join(here, "c1_q255.json")) as f:
        stored = json.load(f)
    for k in ("log", "sha256", "S_rows", "S_sample", "S_absmax", "p", "tau", "R", "T", "qfix"):
        assert fresh[k] == stored[k], k
    assert max(int(float.fromhex(r[2])) for r in stored["log"]) > 127  # k beyond the old cap


def test_general_template_bound_dominates_suboptimality():
    """General template (reading R33): f_t(X) = <C,X> + min_{w in K} <y, AX - w> + beta/2 ||AX - w||^2
    is convex with gradient D_t = C + A*(y + beta (AX - w_t)), w_t = proj_K(AX + y/beta), and
    f_t(X_star) <= p_star, so the derivation of P:3100-3140 gives the bound
    p_t + <y_t, w_t> + beta_t/2 <z_t - w_t, z_t + w_t> - alpha min(lambda_min(D_t), 0) >= p_t - p_star
    (trace-bounded set).  Pin on C5 with the box diag X in [1 - delta, 1 + delta], whose optimum is
    (1 + delta) SDP (closed form, test_box_constraint_set_closed_forms); the logged bound (xi_t) is
    <= the exact one, and gap - bound = <y, z - w> + beta/2 ||z - w||^2."""
    n = 5
    L = _edges_graph(n, [(k, (k + 1) % n) for k in range(n)])
    sdp = 2 * n * (1 + math.cos(math.pi / n))
    d = 0.2
    alpha = 1.05 * n * (1 + d)
    o = oracle.Oracle(L, 3, seed=5, logcap=700, box=(1 - d, 1 + d), trace_le=True, alpha=alpha)
    Ld = L.dense()
    for t in (5, 50, 600):
        o.step(t - o.t)
        y, z, p, a_s = o.y.copy(), o.z.copy(), o.p, o.alpha
        lo, hi = (1 - d) / n, (1 + d) / n
        p_star = -(1 + d) * sdp / (n * o.nrmL)
        beta = math.sqrt(t + 2)
        w = np.minimum(np.maximum(z + y / beta, lo), hi)
        D = -Ld / o.nrmL + np.diag(y + beta * (z - w))
        lam = float(np.linalg.eigvalsh(D)[0])
        bound_exact = p + float(np.dot(y, w)) + 0.5 * beta * float(np.dot(z - w, z + w)) - a_s * min(lam, 0.0)
        assert p - p_star <= bound_exact + 1e-12, (t, p - p_star, bound_exact)
        o.step(1)
        rec = o.log[t]
        assert rec[11] <= bound_exact + 1e-12
        ident = float(np.dot(y, z - w)) + 0.5 * beta * float(np.dot(z - w, z - w))
        assert abs((rec[10] - rec[11]) - ident) <= 1e-12 * max(1.0, abs(rec[10]))


def test_l2_ball_constraint_set_closed_forms():
    """Norm constraint K = {u : ||u - 1||_2 <= delta} (projection reading R34).  On C5
    (vertex-transitive) the optimum of max tr(LX) with ||diag X - 1|| <= delta (and tr X <= alpha, large
    enough) has a uniform diagonal 1 + delta / sqrt(n), so its value is (1 + delta / sqrt n) SDP.
    delta = 0 is the equality problem: every iterate bitwise (the projection is then exactly b), the
    general-template gap / bound equal to rounding; the bound dominates the suboptimality (exact
    lambda_min) as for the box."""
    n = 5
    L = _edges_graph(n, [(k, (k + 1) % n) for k in range(n)])
    sdp = 2 * n * (1 + math.cos(math.pi / n))
    for d in (0.2, 0.6):
        c = 1 + d / math.sqrt(n)
        o = oracle.Oracle(L, 3, seed=5, logcap=3000, ball=d, trace_le=True, alpha=1.05 * n * c)
        o.step(3000)
        assert abs(o.implicit_objective() - c * sdp) <= 3e-3 * sdp
        z = o.z * (o.alpha_orig / o.alpha)
        assert abs(np.linalg.norm(z - 1.0) - d) <= 5e-3
    e = oracle.Oracle(L, 3, seed=5, logcap=300)
    e.step(300)
    b = oracle.Oracle(L, 3, seed=5, logcap=300, ball=0.0)
    b.step(300)
    np.testing.assert_array_equal(b.log[:, :10], e.log[:, :10])
    np.testing.assert_array_equal(b.z, e.z)
    np.testing.assert_allclose(b.log[:, 10:12], e.log[:, 10:12], rtol=1e-11, atol=1e-14)
    d = 0.4
    c = 1 + d / math.sqrt(n)
    alpha = 1.05 * n * c
    o = oracle.Oracle(L, 3, seed=5, logcap=700, ball=d, trace_le=True, alpha=alpha)
    Ld = L.dense()
    for t in (5, 50, 600):
        o.step(t - o.t)
        y, z, p = o.y.copy(), o.z.copy(), o.p
        beta = math.sqrt(t + 2)
        pt = z + y / beta
        ev = pt - 1.0 / n
        N = float(np.linalg.norm(ev))
        w = pt if N <= d / n else 1.0 / n + (d / n / N) * ev
        D = -Ld / o.nrmL + np.diag(y + beta * (z - w))
        lam = float(np.linalg.eigvalsh(D)[0])
        bound_exact = p + float(np.dot(y, w)) + 0.5 * beta * float(np.dot(z - w, z + w)) - o.alpha * min(lam, 0.0)
        assert p - (-c * sdp / (n * o.nrmL)) <= bound_exact + 1e-12


def _soft_threshold_bisect(e, delta):
    """Euclidean projection of e onto {||u||_1 <= delta} by bisection on the threshold theta of
    F(theta) = sum max(|e| - theta, 0) = delta (an algorithm independent of the oracle's sort)."""
    a = np.abs(e)
    if a.sum() <= delta:
        return e.copy()
    lo, hi = 0.0, float(a.max())
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if np.maximum(a - mid, 0).sum() > delta:
            lo = mid
        else:
            hi = mid
    return np.sign(e) * np.maximum(a - 0.5 * (lo + hi), 0)


def test_l1_ball_projection_pins():
    """l1-ball projection (reading R35) against values fixed by the definition: ties
    ([4,4,4,2] - 1 with delta 1: the top three share theta = 8/3), a uniform |e| (theta = |e| -
    delta / n), a point already inside (returned unchanged, bitwise), delta = 0 (b, bitwise), and
    random vectors against an independent bisection on the threshold (1e-12): the projection lies on
    the sphere ||w - b||_1 = delta and keeps the signs of e."""
    n = 6
    L = _edges_graph(n, [(k, (k + 1) % n) for k in range(n)])
    o = oracle.Oracle(L, 2, scale=False, l1_ball=1.0)
    w = o.project(np.array([4.0, 4.0, 4.0, 2.0, 1.0, 1.0]))
    np.testing.assert_allclose(w, [4 / 3, 4 / 3, 4 / 3, 1, 1, 1], rtol=1e-15)
    w = o.project(np.full(n, 1.5))  # |e| = 0.5, n |e| = 3 > 1: theta = 0.5 - 1/6
    np.testing.assert_allclose(w, np.full(n, 1 + 1 / 6), rtol=1e-15)
    w = o.project(np.full(n, 0.5))
    np.testing.assert_allclose(w, np.full(n, 1 - 1 / 6), rtol=1e-15)
    p = np.array([1.2, 1.0, 0.9, 1.0, 1.1, 0.95])  # ||p - 1||_1 = 0.45 <= 1
    np.testing.assert_array_equal(o.project(p), p)
    z = oracle.Oracle(L, 2, scale=False, l1_ball=0.0)
    np.testing.assert_array_equal(z.project(np.array([4.0, -1, 3, 2, 1, 0])), np.ones(n))
    rng = np.random.default_rng(7)
    n = 300
    L = _edges_graph(n, [(k, (k + 1) % n) for k in range(n)])
    for delta in (0.3, 5.0, 40.0):
        o = oracle.Oracle(L, 2, scale=False, l1_ball=delta)
        for _ in range(5):
            e = rng.standard_normal(n) * rng.choice([0.1, 1.0], n)
            e[rng.integers(0, n, 20)] = 0.25  # ties
            w = o.project(1.0 + e)
            want = 1.0 + _soft_threshold_bisect(e, delta)
            np.testing.assert_allclose(w, want, rtol=0, atol=1e-12)
            if np.abs(e).sum() > delta:
                assert abs(np.abs(w - 1.0).sum() - delta) <= 1e-12 * n
                assert np.all(np.sign(w - 1.0) * np.sign(e) >= 0)


def test_l1_ball_constraint_set_closed_forms():
    """Norm constraint K = {u : ||u - 1||_1 <= delta} (projection reading R35).  On C5
    (vertex-transitive; the ball is permutation invariant and the optimal value concave in the
    diagonal) the optimum of max tr(LX) with ||diag X - 1||_1 <= delta has the uniform diagonal
    1 + delta / n: value (1 + delta / n) SDP.  delta = 0 is the equality problem: every iterate bitwise,
    the general-template gap / bound equal to rounding; the bound dominates the suboptimality (exact
    lambda_min)."""
    n = 5
    L = _edges_graph(n, [(k, (k + 1) % n) for k in range(n)])
    sdp = 2 * n * (1 + math.cos(math.pi / n))
    for d in (0.3, 1.0):
        c = 1 + d / n
        o = oracle.Oracle(L, 3, seed=5, logcap=3000, l1_ball=d, trace_le=True, alpha=1.05 * n * c)
        o.step(3000)
        assert abs(o.implicit_objective() - c * sdp) <= 3e-3 * sdp
        z = o.z * (o.alpha_orig / o.alpha)
        assert abs(np.abs(z - 1.0).sum() - d) <= 1e-2
    e = oracle.Oracle(L, 3, seed=5, logcap=300)
    e.step(300)
    b = oracle.Oracle(L, 3, seed=5, logcap=300, l1_ball=0.0)
    b.step(300)
    np.testing.assert_array_equal(b.log[:, :10], e.log[:, :10])
    np.testing.assert_array_equal(b.z, e.z)
    np.testing.assert_allclose(b.log[:, 10:12], e.log[:, 10:12], rtol=1e-11, atol=1e-14)
    d = 0.5
    c = 1 + d / n
    o = oracle.Oracle(L, 3, seed=5, logcap=700, l1_ball=d, trace_le=True, alpha=1.05 * n * c)
    Ld = L.dense()
    for t in (5, 50, 600):
        o.step(t - o.t)
        y, z, p = o.y.copy(), o.z.copy(), o.p
        beta = math.sqrt(t + 2)
        w = 1.0 / n + _soft_threshold_bisect(z + y / beta - 1.0 / n, d / n)
        D = -Ld / o.nrmL + np.diag(y + beta * (z - w))
        lam = float(np.linalg.eigvalsh(D)[0])
        bound_exact = p + float(np.dot(y, w)) + 0.5 * beta * float(np.dot(z - w, z + w)) - o.alpha * min(lam, 0.0)
        assert p - (-c * sdp / (n * o.nrmL)) <= bound_exact + 1e-12
        np.testing.assert_allclose(o.project(z, y, beta), w, rtol=0, atol=1e-15)
