"""GPU parity of the phase retrieval path (csrc/phase.cu through include/scg_phase.h) against the
CPU oracle (oracle/phase.py) on the same seeded instances.

Tolerances: the FFT is a different summation order than numpy's pocketfft,
so the comparisons are within floating-point bounds rather than bitwise -- operator entries within
1e-12 relative to the operator scale (an FFT of length n has error ~ eps log2 n), the Ritz values
within 1e-8 relative for the first iterations (BASELINE's per-iteration eigenvalue bound), the
state within 1e-6 after the window, and the recovered signal within the paper's 1e-2 accuracy."""
import numpy as np
import pytest

import scg_inputs as si
from oracle import phase as ph

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pr(gpu):
    from paper_1912_02949_b200 import phase as prm
    prm.load()
    return prm


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


# sizes: the paper's n = 10^2..10^6 plus ragged {2,3,5}-smooth shapes (odd radices, n1 != n2)
@pytest.mark.parametrize("n", [100, 360, 1000, 2 * 3 * 5 * 7 - 30, 4500, 10000, 100000, 1000000])
def test_operator_parity(pr, n):
    I = si.phase_instance(n, seed=11)
    ctx = pr.PhaseRetrieval(I.psi, I.b, R=5, seed=11)
    kappa, bt = ph.scaling(I.psi, I.b, 3.0 * n)
    np.testing.assert_allclose(ctx.state("kappa"), kappa, rtol=1e-12)
    np.testing.assert_allclose(ctx.state("bt"), bt, rtol=1e-11, atol=1e-14 * np.abs(bt).max())
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    assert _rel(ctx.measure(x), ph.A_rank1(I.psi, kappa, x)) < 1e-12
    w = rng.standard_normal((12, n))
    assert _rel(ctx.apply_D(w, x), ph.apply_D(I.psi, kappa, w, x)) < 1e-12
    # the signal itself: A~(chi chi^*) / alpha = b~
    assert _rel(ctx.measure(I.chi) / (3.0 * n), bt) < 1e-12
    ctx.close()


def _run_both(n, seed, T, R=5):
    from paper_1912_02949_b200 import phase as prm
    I = si.phase_instance(n, seed=seed)
    g = prm.PhaseRetrieval(I.psi, I.b, R=R, seed=seed)
    g.step(T)
    o = ph.PhaseOracle(I.psi, I.b, R=R, seed=seed)
    o.step(T)
    return I, g, o


@pytest.mark.parametrize("n,seed,T", [(100, 0, 60), (1000, 1, 40), (4500, 5, 25)])
def test_trajectory_parity(pr, n, seed, T):
    I, g, o = _run_both(n, seed, T)
    gl, ol = g.iter_log(), o.logarr
    assert gl.shape == ol.shape
    np.testing.assert_array_equal(gl[:, 1], ol[:, 1])               # q_t
    np.testing.assert_array_equal(gl[:, 2], ol[:, 2])               # k_t
    win = min(T, 20)
    scale = np.abs(ol[:win, 3]).max()
    assert np.max(np.abs(gl[:win, 3] - ol[:win, 3])) <= 1e-8 * scale   # theta_t
    assert np.max(np.abs(gl[:win, 4] - ol[:win, 4])) <= 1e-8 * scale   # xi_t
    np.testing.assert_array_equal(gl[:, 4] < 0, ol[:, 4] < 0)        # LMO branch
    for col in (6, 7, 9):                                            # p, ||z - b||, tau
        assert _rel(gl[:, col], ol[:, col]) < 1e-6
    assert _rel(g.state("z"), o.z) < 1e-6
    assert _rel(g.state("y"), o.y) < 1e-6
    assert _rel(g.state("S"), o.S) < 1e-6
    np.testing.assert_allclose(g.state("Omega"), o.Omega, rtol=0, atol=0)   # the same seeded draws
    # v up to a global phase (sign): |<v_gpu, v_oracle>| = 1
    v = g.state("v")
    assert abs(abs(np.vdot(v, o.v)) - 1.0) < 1e-6


def test_reconstruction_parity_on_gpu_sketch(pr):
    """Alg. 3 on the GPU against the oracle's Nystrom applied to the GPU's own S and Omega."""
    n = 1000
    I = si.phase_instance(n, seed=3)
    g = pr.PhaseRetrieval(I.psi, I.b, R=5, seed=3)
    g.step(80)
    U, lam = g.reconstruct()
    Uo, lamo = ph.nystrom_reconstruct_c(g.state("S"), g.state("Omega"))
    np.testing.assert_allclose(lam, lamo, rtol=1e-9, atol=1e-12 * lamo[0])
    assert np.allclose(U.conj().T @ U, np.eye(5), atol=1e-10)
    for k in range(2):          # the well separated leading columns, up to a phase
        assert abs(abs(np.vdot(U[:, k], Uo[:, k])) - 1.0) < 1e-8
    chi = g.signal()
    np.testing.assert_allclose(chi, np.sqrt(3.0 * n * lam[0]) * U[:, 0], rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("n,T", [(100, 1000), (1000, 1500)])
def test_recovers_signal_like_the_paper(pr, n, T):
    """relative error below 1e-2; the oracle's and the GPU's signals agree."""
    I, g, o = _run_both(n, 0, T)
    g.reconstruct()
    chi_g, chi_o = g.signal(), o.signal()
    eg, eo = ph.relative_error(chi_g, I.chi), ph.relative_error(chi_o, I.chi)
    assert eg < 1e-2 and eo < 1e-2, (eg, eo)
    assert ph.relative_error(chi_g, chi_o) < 1e-3
    gl = g.iter_log()
    assert abs(gl[-1, 9] - o.tau) < 1e-6 * o.tau


def test_full_size_first_iteration_p6(pr):
    """n = 10^6 (the paper's largest), the bench configuration: the first iteration's
    Ritz value, monitor and z against the oracle."""
    n = 1000000
    I = si.phase_instance(n, seed=4)
    g = pr.PhaseRetrieval(I.psi, I.b, R=5, seed=4)
    g.step(1)
    o = ph.PhaseOracle(I.psi, I.b, R=5, seed=4)
    o.step(1)
    gl, ol = g.iter_log(), o.logarr
    assert gl[0, 1] == ol[0, 1] and gl[0, 2] == ol[0, 2]
    assert abs(gl[0, 3] - ol[0, 3]) <= 1e-8 * abs(ol[0, 3])
    assert abs(gl[0, 4] - ol[0, 4]) <= 1e-8 * abs(ol[0, 4])
    assert _rel(g.state("z"), o.z) < 1e-6
    assert _rel(g.state("y"), o.y) < 1e-6


def test_reconstruct_before_any_rank_one_update(pr):
    """While xi_t >= 0 the trace-bounded LMO returns H = 0 and S stays 0: the
    reconstruction is X^ = 0 (Lam = 0, U an orthonormal basis), like the oracle's."""
    n = 100
    I = si.phase_instance(n, seed=0)
    g = pr.PhaseRetrieval(I.psi, I.b, R=5, seed=0)
    o = ph.PhaseOracle(I.psi, I.b, R=5, seed=0)
    g.step(3)
    o.step(3)
    assert np.all(o.logarr[:, 4] >= 0) and np.all(g.iter_log()[:, 4] >= 0)
    assert not np.any(g.state("S"))
    U, lam = g.reconstruct()
    Uo, lamo = o.reconstruct()
    assert np.all(lam == 0) and np.all(lamo == 0)
    assert np.allclose(U.conj().T @ U, np.eye(5), atol=1e-12)
    assert not np.any(g.signal())


@pytest.mark.parametrize("flags", [1 << 10, (1 << 11) | (1 << 12) | (1 << 13), 1 << 9])
def test_execution_options_agree(pr, flags):
    """SCG_PR_GENERIC (runtime radix plans), SCG_PR_NOPF_* (no next-tile prefetch) and SCG_PR_TM2 give
    the same operator and iterates within the FFT's rounding as the default kernels (n = 10^4: the
    compile-time 100 x 100 plan)."""
    n = 10000
    I = si.phase_instance(n, seed=6)
    a = pr.PhaseRetrieval(I.psi, I.b, R=5, seed=6)
    b = pr.PhaseRetrieval(I.psi, I.b, R=5, seed=6, flags=flags)
    rng = np.random.default_rng(1)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    w = rng.standard_normal((12, n))
    assert _rel(b.apply_D(w, x), a.apply_D(w, x)) < 1e-13
    assert _rel(b.measure(x), a.measure(x)) < 1e-13
    a.step(15)
    b.step(15)
    la, lb = a.iter_log(), b.iter_log()
    np.testing.assert_array_equal(la[:, 1:3], lb[:, 1:3])
    assert np.max(np.abs(la[:, 3] - lb[:, 3])) <= 1e-9 * np.abs(la[:, 3]).max()
    assert _rel(b.state("z"), a.state("z")) < 1e-8


@pytest.mark.parametrize("L,R", [(1, 1), (3, 2), (32, 16)])
def test_other_modulation_counts_and_ranks(pr, L, R):
    """The boundary's limits: L = 1..32 modulations, R = 1..16 (include/scg_phase.h), vs the oracle."""
    n = 360  # 18 x 20: runtime plans with radix 3
    psi = si.phase_psi(n, seed=9, L=L)
    chi = si.phase_signal(n, seed=9)
    b = np.abs(np.fft.fft(np.conj(psi) * chi[None, :], axis=1)) ** 2
    g = pr.PhaseRetrieval(psi, b, R=R, seed=9)
    o = ph.PhaseOracle(psi, b, R=R, seed=9)
    kappa, _ = ph.scaling(psi, b, 3.0 * n)
    np.testing.assert_allclose(g.state("kappa"), kappa, rtol=1e-12)
    g.step(20)
    o.step(20)
    gl, ol = g.iter_log(), o.logarr
    np.testing.assert_array_equal(gl[:, 1:3], ol[:, 1:3])
    assert np.max(np.abs(gl[:, 3] - ol[:, 3])) <= 1e-8 * np.abs(ol[:, 3]).max()
    assert _rel(g.state("z"), o.z) < 1e-6
    assert _rel(g.state("S"), o.S) < 1e-6 or not np.any(o.S)


def test_q_cap_on_tiny_n(pr):
    """n = 6 (2 x 3): from t ~ 64 on, q_t = min(n - 1, ...) caps the Lanczos steps (P:1451 with
    Alg. 2's min{q, n - 1}); GPU and oracle agree on q_t, k_t and theta_t."""
    n = 6
    I = si.phase_instance(n, seed=2)
    g = pr.PhaseRetrieval(I.psi, I.b, R=3, seed=2)
    o = ph.PhaseOracle(I.psi, I.b, R=3, seed=2)
    g.step(120)
    o.step(120)
    gl, ol = g.iter_log(), o.logarr
    np.testing.assert_array_equal(gl[:, 1:3], ol[:, 1:3])
    assert gl[:, 1].max() == n - 1 and np.sum(gl[:, 1] == n - 1) > 20
    assert np.max(np.abs(gl[:, 3] - ol[:, 3])) <= 1e-8 * np.abs(ol[:, 3]).max()


def test_zero_signal_and_degenerate_inputs(pr):
    """chi_nat = 0 gives b = 0: D_1 = I / sqrt(n) has xi > 0, the LMO returns H = 0 at every t and X
    stays 0 (GPU and oracle); a modulation that is identically zero is rejected (||A_i||_F = 0 leaves
    the row scaling of P:1811-1812 undefined)."""
    n = 100
    psi = si.phase_psi(n, seed=3)
    b = np.zeros((12, n))
    g = pr.PhaseRetrieval(psi, b, R=5, seed=3)
    o = ph.PhaseOracle(psi, b, R=5, seed=3)
    g.step(10)
    o.step(10)
    assert np.all(g.iter_log()[:, 4] > 0) and np.all(o.logarr[:, 4] > 0)
    assert not np.any(g.state("z")) and not np.any(g.state("S"))
    g.reconstruct()
    assert not np.any(g.signal())
    bad = psi.copy()
    bad[4] = 0.0
    with pytest.raises(pr.PhaseError):
        pr.PhaseRetrieval(bad, b, R=5, seed=3)


def test_hooks_leave_the_iteration_state_alone(pr):
    """apply_D / measure run on scratch buffers: the iterates, the eigenvector and the next iterations are
    those of a context without hook calls."""
    n = 1000
    I = si.phase_instance(n, seed=8)
    a = pr.PhaseRetrieval(I.psi, I.b, R=5, seed=8)
    b = pr.PhaseRetrieval(I.psi, I.b, R=5, seed=8)
    a.step(5)
    b.step(5)
    rng = np.random.default_rng(3)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    b.apply_D(rng.standard_normal((12, n)), x)
    b.measure(x)
    np.testing.assert_array_equal(a.state("v"), b.state("v"))
    a.step(5)
    b.step(5)
    np.testing.assert_array_equal(a.iter_log(), b.iter_log())
    np.testing.assert_array_equal(a.state("z"), b.state("z"))
