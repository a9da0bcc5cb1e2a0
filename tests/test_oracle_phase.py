"""Pins of the phase retrieval oracle (oracle/phase.py) against what the paper
and the mathematics fix: the printed coded-diffraction rows written out as a dense DFT matrix, the
adjoint identity, dense eigendecompositions, a dense shadow CGAL, exact Nystrom recovery, the
closed-form phase alignment, the exact operator norm over every circulant shift, and the paper's
recovery claim (relative error below 1e-2)."""
import numpy as np
import pytest

import oracle
import scg_inputs as si
from oracle import phase as ph


def dense_rows(psi):
    """r_i = a_i^* = W_n(l, :) diag(psi_j)^* written out entry by entry, with
    W_n(l, k) = exp(-2 pi i l k / n), 0-based l, k; stacked j-major: i = j n + l."""
    L, n = psi.shape
    rows = np.empty((L * n, n), dtype=np.complex128)
    for j in range(L):
        for l in range(n):
            for k in range(n):
                rows[j * n + l, k] = np.exp(-2j * np.pi * l * k / n) * np.conj(psi[j, k])
    return rows


def rand_herm(rng, n):
    G = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    return 0.5 * (G + G.conj().T)


def test_instance_distribution_and_measurements_match_printed_rows():
    n = 12
    I = si.phase_instance(n, seed=5)
    assert I.psi.shape == (12, n) and I.b.shape == (12, n)
    mags = np.abs(I.psi)
    assert np.all(np.isclose(mags, np.sqrt(2) / 2) | np.isclose(mags, np.sqrt(3)))
    units = I.psi / mags
    assert np.allclose(np.abs(np.round(units.real) + 1j * np.round(units.imag) - units), 0)
    r = dense_rows(I.psi)
    b_dense = np.abs(r @ I.chi) ** 2                  # b_i = |<a_i, chi>|^2
    np.testing.assert_allclose(I.b.reshape(-1), b_dense, rtol=1e-12, atol=1e-12)
    # the oracle's forward operator is the same map
    np.testing.assert_allclose(np.abs(ph.M(I.psi, I.chi)) ** 2, I.b, rtol=1e-12, atol=1e-12)


def test_waveform_statistics_large_sample():
    psi = si.phase_psi(20000, seed=3)
    mags = np.abs(psi)
    frac_small = np.mean(np.isclose(mags, np.sqrt(2) / 2))
    assert abs(frac_small - 0.8) < 0.01                # probabilities 0.8 / 0.2
    ph_idx = np.round(np.angle(psi) / (np.pi / 2)).astype(int) % 4
    counts = np.bincount(ph_idx.reshape(-1), minlength=4) / psi.size
    assert np.all(np.abs(counts - 0.25) < 0.01)        # uniform on {1, i, -1, -i}
    chi = si.phase_signal(200000, seed=3)
    assert abs(np.mean(np.abs(chi) ** 2) - 1.0) < 0.01  # complex standard normal
    assert abs(np.mean(chi.real * chi.imag)) < 0.01


def test_operators_match_dense_definition_and_adjoint():
    rng = np.random.default_rng(0)
    n = 10
    I = si.phase_instance(n, seed=1)
    r = dense_rows(I.psi)
    kappa = rng.uniform(0.5, 2.0, 12)
    kap_i = np.repeat(kappa, n)
    X = rand_herm(rng, n)
    AX_dense = kap_i * np.real(np.einsum("ik,kl,il->i", r, X, np.conj(r)))   # <A_i, X> = a_i^* X a_i
    v = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    np.testing.assert_allclose(ph.A_rank1(I.psi, kappa, v).reshape(-1),
                               kap_i * np.abs(r @ v) ** 2, rtol=1e-12)
    w = rng.standard_normal((12, n))
    Astar_dense = (r.conj().T * (kap_i * w.reshape(-1))) @ r          # sum_i w_i A_i
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    np.testing.assert_allclose(ph.Astar_apply(I.psi, kappa, w, x), Astar_dense @ x, rtol=1e-11, atol=1e-11)
    # adjoint identity <A X, w> = Re tr(X A^*(w))
    lhs = float(np.sum(AX_dense * w.reshape(-1)))
    rhs = float(np.real(np.trace(X @ Astar_dense)))
    assert abs(lhs - rhs) <= 1e-10 * abs(lhs)
    # D = I / sqrt(n) + A^*(w)
    np.testing.assert_allclose(ph.apply_D(I.psi, kappa, w, x), x / np.sqrt(n) + Astar_dense @ x,
                               rtol=1e-11, atol=1e-11)


def test_scaling_equalizes_rows_and_norm_is_exact():
    for n, seed in ((8, 0), (64, 1), (100, 0), (1000, 1)):
        I = si.phase_instance(n, seed=seed)
        c = ph.row_scale(I.psi)
        r = None
        if n <= 64:
            r = dense_rows(I.psi)
            fro = np.repeat(c, n) * np.sum(np.abs(r) ** 2, axis=1)      # ||c_j a_i a_i^*||_F
            np.testing.assert_allclose(fro, 1.0, rtol=1e-13)
        exact, shift, lam = ph.opnorm_exact(I.psi, c)
        diag = ph.opnorm_diag(I.psi, c)
        assert shift == 0 and abs(exact - diag) <= 1e-12 * exact          # reading R38
        assert np.sort(lam)[-2] < 0.5 * lam.max()
        if r is not None and n == 8:
            # brute-force power iteration on A'^* A' over Hermitian n x n matrices
            ci = np.repeat(c, n)
            X = np.eye(n, dtype=complex)
            for _ in range(500):
                AX = ci * np.real(np.einsum("ik,kl,il->i", r, X, np.conj(r)))
                Y = (r.conj().T * (ci * AX)) @ r
                X = Y / np.linalg.norm(Y)
            AX = ci * np.real(np.einsum("ik,kl,il->i", r, X, np.conj(r)))
            assert abs(np.linalg.norm(AX) - exact) <= 1e-9 * exact
        kappa, bt = ph.scaling(I.psi, I.b, 3.0 * n)
        # scaled signal satisfies A~(X~_nat) = b~ with X~_nat = chi chi^* / alpha
        np.testing.assert_allclose(ph.A_rank1(I.psi, kappa, I.chi) / (3.0 * n), bt, rtol=1e-11)


def test_complex_lanczos_full_krylov_and_ritz_bounds():
    rng = np.random.default_rng(2)
    n = 16
    I = si.phase_instance(n, seed=2)
    kappa, bt = ph.scaling(I.psi, I.b, 3.0 * n)
    w = rng.standard_normal((12, n)) * 0.3
    r = dense_rows(I.psi)
    Dd = np.eye(n) / np.sqrt(n) + (r.conj().T * (np.repeat(kappa, n) * w.reshape(-1))) @ r
    lam = np.linalg.eigvalsh(Dd)
    g = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    th, v, k, om, rho, s = ph.lanczos(lambda x: ph.apply_D(I.psi, kappa, w, x), g, n)
    assert abs(th - lam[0]) <= 1e-10 * abs(lam).max()
    assert np.linalg.norm(Dd @ v - th * v) <= 1e-7 * abs(lam).max()
    assert abs(np.linalg.norm(v) - 1.0) < 1e-14
    for q in (2, 4, 7):
        thq = ph.lanczos(lambda x: ph.apply_D(I.psi, kappa, w, x), g, q)[0]
        assert thq >= lam[0] - 1e-12 and thq <= lam[-1] + 1e-12
    # the tridiagonal built from omega / rho is the Rayleigh-Ritz matrix of the Krylov basis
    T = np.diag(om) + np.diag(rho, 1) + np.diag(rho, -1)
    np.testing.assert_allclose(np.sort(np.linalg.eigvalsh(T)), lam, rtol=1e-8, atol=1e-10)


def test_iterates_match_dense_shadow_cgal():
    """Loop invariants against a dense CGAL (Alg. 1 with the trace-bounded LMO) driven by the
    oracle's own v_t: z = A~(X_t), S = X_t Omega, tau = tr X_t, p = <C~, X_t>."""
    n, T = 16, 40
    I = si.phase_instance(n, seed=3)
    o = ph.PhaseOracle(I.psi, I.b, R=3, seed=3, keep_v=True)
    o.step(T)
    r = dense_rows(I.psi)
    X = np.zeros((n, n), dtype=complex)
    lg = o.logarr
    for t in range(1, T + 1):
        eta = 2.0 / (t + 1)
        v = o.vhist[t - 1]
        H = np.outer(v, v.conj()) if lg[t - 1, 4] < 0 else np.zeros((n, n))
        X = (1 - eta) * X + eta * H
    Az = np.repeat(o.kappa, n) * np.real(np.einsum("ik,kl,il->i", r, X, np.conj(r)))
    np.testing.assert_allclose(o.z.reshape(-1), Az, rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(o.S, X @ o.Omega, rtol=1e-10, atol=1e-13)
    assert abs(o.tau - np.real(np.trace(X))) < 1e-12
    assert abs(o.p - np.real(np.trace(X)) / np.sqrt(n)) < 1e-12
    assert np.any(lg[:, 4] < 0) and lg[0, 1] == oracle.qt(1, n)
    # the Ritz value of every step is >= lambda_min(D_t) and xi = v^* D v >= lambda_min
    assert np.all(lg[:, 4] >= lg[:, 3] - 1e-12)


def test_complex_nystrom_exact_recovery_of_low_rank():
    rng = np.random.default_rng(4)
    n, R, r = 40, 5, 3
    Q = np.linalg.qr(rng.standard_normal((n, r)) + 1j * rng.standard_normal((n, r)))[0]
    lam = np.array([3.0, 1.0, 0.25])
    X = (Q * lam) @ Q.conj().T
    Om = ph.omega_matrix(9, n, R)
    U, Lam = ph.nystrom_reconstruct_c(X @ Om, Om)
    Xh = (U * Lam) @ U.conj().T
    assert np.linalg.norm(Xh - X) <= 1e-10 * np.linalg.norm(X)
    np.testing.assert_allclose(Lam[:3], lam, rtol=1e-10)


def test_relative_error_closed_form_vs_phase_grid():
    rng = np.random.default_rng(5)
    chi_nat = rng.standard_normal(30) + 1j * rng.standard_normal(30)
    chi = np.exp(0.7j) * chi_nat + 0.1 * (rng.standard_normal(30) + 1j * rng.standard_normal(30))
    phis = np.linspace(0, 2 * np.pi, 200001)
    brute = min(np.linalg.norm(np.exp(1j * p) * chi - chi_nat) for p in phis[::100])
    fine = np.linspace(-0.01, 0.01, 2001) + phis[::100][np.argmin(
        [np.linalg.norm(np.exp(1j * p) * chi - chi_nat) for p in phis[::100]])]
    brute = min(brute, min(np.linalg.norm(np.exp(1j * p) * chi - chi_nat) for p in fine))
    assert abs(ph.relative_error(chi, chi_nat) - brute / np.linalg.norm(chi_nat)) < 1e-7
    assert ph.relative_error(np.exp(2.1j) * chi_nat, chi_nat) < 1e-7


def test_recovers_signal_to_paper_accuracy_n100():
    """SketchyCGAL (R = 5, alpha = 3n) recovers every instance to relative error
    below 1e-2; the implicit trace tends to ||chi||^2 / alpha (X_t -> chi chi^* / alpha)."""
    n = 100
    I = si.phase_instance(n, seed=0)
    o = ph.PhaseOracle(I.psi, I.b, R=5, seed=0)
    o.step(1000)
    err = ph.relative_error(o.signal(), I.chi)
    assert err < 1e-2, err
    assert abs(o.tau - np.vdot(I.chi, I.chi).real / (3.0 * n)) < 2e-2 * o.tau
    assert o.implicit_infeasibility() < 1e-2
    lg = o.logarr
    # posterior bound: bound_t >= p_t - p_star with p_star = ||chi||^2 / (alpha sqrt n)
    # (X_nat is the unique solution of the PhaseLift SDP for this instance; checked by recovery)
    pstar = np.vdot(I.chi, I.chi).real / (3.0 * n * np.sqrt(n))
    p_prev = np.concatenate([[0.0], lg[:-1, 6]])
    assert np.all(lg[:, 11] >= (p_prev - pstar) - 1e-12)
