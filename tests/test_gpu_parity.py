"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar: the feedback path (theta_t, k_t, z, y, d, v) is
bitwise identical at every t; off-path quantities (S, xi, c, p) agree to
rounding; after T the reconstruction-based objective and feasibility agree to
1e-6 relative (BASELINE.json north_star) and the rounded cut on configs[0] is
identical.
"""
import numpy as np
import pytest

import oracle
import scg_inputs as si

pytestmark = pytest.mark.gpu


def _run_pair(gpu, L, R, T, seed, scale=True, regenerate=False, **opts):
    g = gpu.SketchyCGAL(L, R=R, seed=seed, scale=scale, regenerate=regenerate, **opts)
    g.step(T)
    o = oracle.Oracle(L, R, seed=seed, scale=scale, logcap=T)
    o.step(T)
    return g, o


def _assert_trajectory(g, o, T):
    gl, ol = g.iter_log(), o.log
    assert gl.shape == (T, 12)
    np.testing.assert_array_equal(gl[:, 10:12], ol[:, 10:12])     # surrogate gap, posterior bound bitwise
    np.testing.assert_array_equal(gl[:, 0:3], ol[:, 0:3])          # t, q, k
    np.testing.assert_array_equal(gl[:, 3], ol[:, 3])              # theta (Ritz) bitwise
    np.testing.assert_array_equal(gl[:, 8], ol[:, 8])              # gamma bitwise
    np.testing.assert_array_equal(gl[:, 7], ol[:, 7])              # ||z - b|| bitwise
    np.testing.assert_allclose(gl[:, 4], ol[:, 4], rtol=1e-13, atol=0)  # xi
    np.testing.assert_allclose(gl[:, 5:7], ol[:, 5:7], rtol=1e-13, atol=0)  # c, p
    np.testing.assert_array_equal(g.state("z"), o.z)
    np.testing.assert_array_equal(g.state("y"), o.y)
    np.testing.assert_array_equal(g.state("v"), o.v)
    np.testing.assert_array_equal(g.state("Omega"), o.Omega)
    S_o = o.S
    np.testing.assert_allclose(g.state("S"), S_o, rtol=0, atol=1e-13 * np.abs(S_o).max())


@pytest.mark.parametrize("resident", [True, False])
def test_config0_full_trajectory_and_cut(gpu, resident):
    """configs[0] (ER n=800, R=10, T=1000, seed 0): every iterate, the objective and the cut -- with
    the resident cluster kernel (one launch per iteration, the default below 2^16 rows) and with the
    multi-kernel iteration."""
    L = si.laplacian("c0")
    T = 1000
    g, o = _run_pair(gpu, L, 10, T, seed=0, resident=resident)
    _assert_trajectory(g, o, T)
    U, lam, err = g.reconstruct()
    Uo, lam_o, err_o = oracle.nystrom_reconstruct(o.S, o.Omega, o.tau)
    unit = L.n / o.alpha
    lam_tc = oracle.trace_correct(lam_o, o.alpha) * unit
    np.testing.assert_allclose(lam, lam_tc, rtol=1e-9)
    np.testing.assert_allclose(err, err_o * unit, rtol=1e-6, atol=1e-9 * L.n)
    obj = g.objective()
    obj_o = oracle.objective_hat(L, Uo, lam_tc)
    assert abs(obj[0] - o.implicit_objective()) <= 1e-12 * abs(obj[0])
    assert abs(obj[1] - obj_o) <= 1e-6 * abs(obj_o)
    fz = g.feasibility()
    f_o = oracle.feasibility_hat(Uo, lam_tc)
    assert abs(fz[0] - o.implicit_infeasibility()) <= 1e-10 * fz[0]
    assert abs(fz[1] - f_o[0]) <= 1e-6 * f_o[0] and abs(fz[2] - f_o[1]) <= 1e-6 * f_o[1]
    chi, w = g.round()
    chi_o, w_o, _ = oracle.round_cut(L, Uo)
    np.testing.assert_array_equal(chi, chi_o)
    assert w == w_o


@pytest.mark.parametrize("regenerate,resident", [(False, True), (False, False), (True, False)])
def test_config1_trajectory_signed_weights(gpu, regenerate, resident):
    """configs[1] shape (torus, +-1 weights), first 300 iterations bitwise, both Lanczos modes, with and
    without the resident cluster kernel."""
    L = si.laplacian("c1")
    g, o = _run_pair(gpu, L, 10, 300, seed=1, regenerate=regenerate, resident=resident)
    _assert_trajectory(g, o, 300)


def test_config0_regenerate_mode(gpu):
    """Storage-optimal two-pass Lanczos (Alg. 2 as printed) on configs[0], 400 iterations."""
    L = si.laplacian("c0")
    g, o = _run_pair(gpu, L, 10, 400, seed=0, regenerate=True)
    _assert_trajectory(g, o, 400)


def test_unscaled_variant(gpu):
    L = si.laplacian("c0")
    g, o = _run_pair(gpu, L, 5, 60, seed=3, scale=False)
    _assert_trajectory(g, o, 60)


@pytest.mark.parametrize("regenerate,resident", [(False, True), (False, False), (True, False)])
def test_breakdown_complete_graph(gpu, regenerate, resident):
    """K_8: D_1 has two eigenvalues -> invariant subspace after 2 steps (Alg. 2 line 8)."""
    n = 8
    i, j = np.triu_indices(n, 1)
    L = si.laplacian_from_edges(n, i, j, np.ones(len(i)))
    g, o = _run_pair(gpu, L, 3, 25, seed=2, regenerate=regenerate, resident=resident)
    assert o.log[0, 2] == 2 and o.log[0, 1] == 3  # k = 2 < q_1 = ceil(ln 8) = 3
    _assert_trajectory(g, o, 25)


@pytest.mark.parametrize("resident", [True, False])
@pytest.mark.parametrize("n", [2, 3, 5, 33, 257, 1000])
def test_small_and_ragged_sizes(gpu, n, resident):
    rng = np.random.default_rng(n)
    i = np.arange(n - 1)
    j = i + 1  # a path keeps the graph connected
    extra = rng.integers(0, n, size=(2 * n, 2))
    extra = extra[extra[:, 0] != extra[:, 1]]
    i = np.concatenate([i, extra[:, 0]])
    j = np.concatenate([j, extra[:, 1]])
    w = rng.uniform(0.5, 1.5, size=len(i))
    L = si.laplacian_from_edges(n, i, j, w)
    R = min(4, n)
    g, o = _run_pair(gpu, L, R, 40, seed=n, resident=resident)
    _assert_trajectory(g, o, 40)


def test_isolated_vertices_and_heavy_row(gpu):
    """A star (one row of degree n-50) plus isolated vertices: ragged rows, zero rows."""
    n = 3000
    i = np.zeros(n - 50, dtype=np.int64)
    j = np.arange(1, n - 49)
    L = si.laplacian_from_edges(n, i, j, np.ones(len(i)))
    g, o = _run_pair(gpu, L, 5, 30, seed=9)
    _assert_trajectory(g, o, 30)


@pytest.mark.parametrize("cfg,T,pdl", [("c0", 200, False), ("c2", 2, True)])
def test_launch_policy_forced_bitwise(gpu, cfg, T, pdl):
    """Programmatic dependent launches (default on) off (SCG_NO_PDL), and on: the same bitwise
    trajectory as the oracle."""
    L = si.laplacian(cfg)
    c = si.CONFIGS[cfg]
    g, o = _run_pair(gpu, L, c["R"], T, seed=c["seed"], pdl=pdl)
    _assert_trajectory(g, o, T)


@pytest.mark.parametrize("cfg,T", [("c1", 300), ("c3", 2), ("c4", 1)])
def test_sell_layout_where_ell_applies_bitwise(gpu, cfg, T):
    """Graphs whose rows all have <= 8 entries run the ELL-W SpMV by default; the SELL-32 layout
    (SCG_NO_ELL) gives the same bitwise trajectory on them."""
    L = si.laplacian(cfg)
    c = si.CONFIGS[cfg]
    R = 2 if cfg == "c4" else c["R"]
    g, o = _run_pair(gpu, L, R, T, seed=c["seed"], ell=False)
    _assert_trajectory(g, o, T)


@pytest.mark.parametrize("n", [8000, 8001, 8031])
def test_ell_ragged_tail_bitwise(gpu, n):
    """ELL-W with a row count that is not a multiple of the 32-row slice (signed weights, a ring plus
    chords: every row <= 4 entries), multi-kernel iteration."""
    i = np.arange(n)
    L = si.laplacian_from_edges(n, np.concatenate([i, i]), np.concatenate([(i + 1) % n, (i + 97) % n]),
                                np.concatenate([np.ones(n), -np.ones(n)]), dedupe=True)
    g, o = _run_pair(gpu, L, 4, 30, seed=6, resident=False)
    _assert_trajectory(g, o, 30)


@pytest.mark.parametrize("weights", ["unit", "signed", "valued"])
@pytest.mark.parametrize("resident", [False, True])
def test_ell_mixed_row_lengths_bitwise(gpu, weights, resident):
    """ELL-3 against the oracle on rows of 1-3 entries (most rows padded), a ragged last slice, unit
    weights (the sign-free positive layout), signed unit weights and general weights: the padding's
    -0 products leave every chain unchanged; with the resident cluster kernel (the ELL engine for
    W <= 4 as well)."""
    n = 8001
    i = np.arange(n)
    ch = i[i % 3 == 0]
    u, v = np.concatenate([i[i % 7 != 0], ch]), np.concatenate([(i[i % 7 != 0] + 1) % n, (ch + 97) % n])
    rng = np.random.default_rng(11)
    w = {"unit": np.ones(len(u)), "signed": np.where(rng.random(len(u)) < 0.5, -1.0, 1.0),
         "valued": rng.uniform(0.5, 1.5, len(u))}[weights]
    L = si.laplacian_from_edges(n, u, v, w, dedupe=True)
    lens = np.diff(np.asarray(L.row_ptr)) - 1
    assert lens.max() <= 4 and lens.min() <= 2
    g, o = _run_pair(gpu, L, 4, 30, seed=6, resident=resident)
    _assert_trajectory(g, o, 30)


def test_ell_far_columns_bitwise(gpu):
    """Unit-weight ELL (the sign-free positive layout) with columns n/2 rows away on every fifth vertex
    and short chords elsewhere, n = 100001 (ragged last slice), against the oracle."""
    n = 100001
    i = np.arange(n)
    far, near = i[i % 5 == 0], i[i % 5 == 2]
    u = np.concatenate([i, far, near])
    v = np.concatenate([(i + 1) % n, (far + n // 2) % n, (near + 300) % n])
    L = si.laplacian_from_edges(n, u, v, np.ones(len(u)), dedupe=True)
    g, o = _run_pair(gpu, L, 4, 12, seed=8)
    _assert_trajectory(g, o, 12)


@pytest.mark.parametrize("cfg,T", [("c0", 200), ("c3", 1)])
def test_tma_staged_recurrence_bitwise(gpu, cfg, T):
    """The opt-in TMA-staged recurrence kernel (SCG_TMA_B) gives the same bitwise trajectory."""
    L = si.laplacian(cfg)
    c = si.CONFIGS[cfg]
    g, o = _run_pair(gpu, L, c["R"], T, seed=c["seed"], tma_b=True)
    _assert_trajectory(g, o, T)


def test_sketch_rank_50(gpu):
    """R = 50 (BASELINE allows R <= 50) on configs[0]: the g = v^T Omega column loop in chunks of 16,
    the deferred sketch flush and the R x R reconstruction core at their largest."""
    L = si.laplacian("c0")
    T = 150
    g, o = _run_pair(gpu, L, 50, T, seed=0)
    _assert_trajectory(g, o, T)
    U, lam, _ = g.reconstruct()
    Uo, lam_o, _ = oracle.nystrom_reconstruct(o.S, o.Omega, o.tau)
    np.testing.assert_allclose(lam, oracle.trace_correct(lam_o, o.alpha) * (L.n / o.alpha), rtol=1e-8)


@pytest.mark.parametrize("cfg,T", [("c0", 300), ("c3", 1)])
def test_warp_specialized_spmv_engine_bitwise(gpu, cfg, T):
    """The opt-in warp-specialized TMA k_lanczos_a (SCG_WS_SPMV: producer warp + mbarrier ring)
    gives the same bitwise trajectory."""
    L = si.laplacian(cfg)
    c = si.CONFIGS[cfg]
    g, o = _run_pair(gpu, L, c["R"], T, seed=c["seed"], ws_spmv=True)
    _assert_trajectory(g, o, T)


@pytest.mark.parametrize("cfg,T", [("c0", 300), ("c2", 2), ("c3", 1)])
def test_fused_pass1_kernel_bitwise(gpu, cfg, T):
    """The opt-in persistent pass-1 kernel (SCG_FUSED_PASS1: all q Lanczos steps in one cooperative
    launch, grid barriers on the exact-sum tickets) gives the same bitwise trajectory."""
    L = si.laplacian(cfg)
    c = si.CONFIGS[cfg]
    g, o = _run_pair(gpu, L, c["R"], T, seed=c["seed"], fused_pass1=True)
    _assert_trajectory(g, o, T)


@pytest.mark.parametrize("P", [2, 3])
def test_warp_specialized_sharded_bitwise(gpu, P):
    """The warp-specialized SpMV under emulated row shards (odd row bases: the 16-byte aligned
    bulk copy of the own entries starts one element early; peer halo stores elsewhere)."""
    L = si.laplacian("c0")
    T = 200
    g = gpu.SketchyCGAL(L, R=10, seed=0, shards=P, ws_spmv=True)
    g.step(T)
    o = oracle.Oracle(L, 10, seed=0, logcap=T)
    o.step(T)
    _assert_trajectory(g, o, T)


@pytest.mark.parametrize("regenerate", [False, True])
def test_fused_pass1_breakdown_and_regenerate(gpu, regenerate):
    """Fused pass 1 through a Lanczos breakdown (K_8, k = 2 < q) in both Lanczos modes."""
    n = 8
    i, j = np.triu_indices(n, 1)
    L = si.laplacian_from_edges(n, i, j, np.ones(len(i)))
    g, o = _run_pair(gpu, L, 3, 25, seed=2, regenerate=regenerate, fused_pass1=True)
    _assert_trajectory(g, o, 25)


def test_steps_resume_equals_single_call(gpu):
    L = si.laplacian("c0")
    a = gpu.SketchyCGAL(L, R=4, seed=5)
    a.step(7)
    a.step(13)
    b = gpu.SketchyCGAL(L, R=4, seed=5)
    b.step(20)
    np.testing.assert_array_equal(a.iter_log(), b.iter_log())
    np.testing.assert_array_equal(a.state("y"), b.state("y"))


@pytest.mark.parametrize("cfg", ["c2", "c3", "c4"])
def test_full_size_apply_D_bitwise(gpu, cfg):
    """BASELINE sizes: every row of D x (the SpMV of the Lanczos kernels) equals the oracle's row chain."""
    L = si.laplacian(cfg)
    c = si.CONFIGS[cfg]
    g = gpu.SketchyCGAL(L, R=c["R"], seed=c["seed"])
    g.step(1)
    x = si.normals(123, 7, 0, 0, L.n)
    y = g.apply_D(x)
    # oracle row chains with the GPU-independent C~ (built by the oracle) and the same d
    o = oracle.Oracle(L, 1, seed=c["seed"], logcap=0)
    rows = np.repeat(np.arange(L.n, dtype=np.int64), np.diff(L.row_ptr))
    off = L.col != rows
    rp = np.zeros(L.n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows[off], minlength=L.n), out=rp[1:])
    m = (-L.val[off]) / o.nrmL
    d = g.state("d")
    y_o = oracle.apply(L.n, rp, L.col[off], m, d, x)
    np.testing.assert_array_equal(y, y_o)
    np.testing.assert_array_equal(g.state("cdiag"), o.cdiag)
    z = g.state("z")
    assert abs(z.sum() - 1.0) < 1e-12  # tr X_2 = alpha
    del o


@pytest.mark.parametrize("regenerate", [False, True])
def test_config2_first_iterations_bitwise(gpu, regenerate):
    L = si.laplacian("c2")
    g, o = _run_pair(gpu, L, 10, 3, seed=2, regenerate=regenerate)
    _assert_trajectory(g, o, 3)


def test_config3_first_iteration_bitwise(gpu):
    L = si.laplacian("c3")
    g, o = _run_pair(gpu, L, 10, 1, seed=3)
    _assert_trajectory(g, o, 1)


def test_config4_first_iteration_bitwise(gpu):
    """configs[4] at full size (n = 2^25, non-uniform weights, random matching edges): one whole
    iteration bitwise (R = 2 keeps the oracle's Omega work small; R does not enter the matvecs)."""
    L = si.laplacian("c4")
    g, o = _run_pair(gpu, L, 2, 1, seed=4)
    _assert_trajectory(g, o, 1)


def _xsum_cases():
    rng = np.random.default_rng(5)
    n = 200000
    wide = rng.standard_normal(n) * np.exp2(rng.integers(-300, 95, n).astype(float))
    cancel = np.concatenate([wide, -wide[::-1], [1e-300, 3.0]])
    mixed = rng.standard_normal(n) * np.exp2(rng.integers(-40, 40, n).astype(float))
    mixed[rng.integers(0, n, 500)] = 0.0
    mixed[rng.integers(0, n, 500)] = 5e-324  # subnormals (Q truncation at 2^-200)
    near = np.exp2(rng.uniform(90, 99.9, 1000)) * rng.choice([-1.0, 1.0], 1000)
    same = np.full(300000, 0.1)  # thousands of deposits per thread: the bins spill
    return {"wide": wide, "cancel": cancel, "mixed": mixed, "near_2^100": near, "same": same,
            "tiny": rng.standard_normal(n) * 1e-250, "empty": np.zeros(0)}


@pytest.mark.parametrize("case", ["wide", "cancel", "mixed", "near_2^100", "same", "tiny", "empty"])
@pytest.mark.parametrize("grid,block", [(296, 256), (1, 32), (3, 64)])
def test_exact_sum_accumulators(gpu, case, grid, block):
    """The kernels' per-thread exact accumulators (fp64 bins with spills, slow path, block and grid
    commits; CAC-2) against the oracle's independent integer exact sum, bitwise: magnitudes over 400
    binades, exact cancellation, zeros and subnormals (Q truncation), values near the 2^100 range
    limit, and 10^4 deposits per thread (grid 1 x 32)."""
    v = _xsum_cases()[case]
    s, rerr = gpu.selftest_xsum(v, grid=grid, block=block)
    want = oracle.xsum(v)
    assert rerr == 0
    assert float.hex(s) == float.hex(want), (s, want)
    bad = np.concatenate([v, [2.0 ** 100]])
    assert gpu.selftest_xsum(bad, grid=grid, block=block)[1] == 1


def test_shared_divisor_division_is_ieee(gpu):
    """div_rn (RN(1/b) + two fma corrections) must equal the hardware division bit for bit."""
    for seed in (1, 2, 3):
        assert gpu.selftest_division(1 << 26, seed) == 0


# ---------------------------------------------------------------- row-sharded path
# P ranks emulated inside one context on one device: the same kernels, halo peer
# stores and mailbox collectives as one process per GPU, checked bitwise against the
# oracle (the exact sums make the iterates independent of P).

@pytest.mark.parametrize("P", [2, 3])
def test_sharded_config0_trajectory_and_cut(gpu, P):
    L = si.laplacian("c0")
    T = 300
    g = gpu.SketchyCGAL(L, R=10, seed=0, shards=P)
    g.step(T)
    o = oracle.Oracle(L, 10, seed=0, logcap=T)
    o.step(T)
    _assert_trajectory(g, o, T)
    one = gpu.SketchyCGAL(L, R=10, seed=0)
    one.step(T)
    U1, lam1, _ = one.reconstruct()
    U, lam, _ = g.reconstruct()
    np.testing.assert_allclose(lam, lam1, rtol=1e-9)
    # the sharded reconstruction against the oracle's (Alg. 3 with LAPACK), not only the 1-GPU path
    Uo, lam_o, _ = oracle.nystrom_reconstruct(o.S, o.Omega, o.tau)
    lam_tc = oracle.trace_correct(lam_o, o.alpha) * (L.n / o.alpha)
    np.testing.assert_allclose(lam, lam_tc, rtol=1e-9)
    assert abs(g.objective()[1] - oracle.objective_hat(L, Uo, lam_tc)) <= 1e-6 * oracle.objective_hat(L, Uo, lam_tc)
    f_o = oracle.feasibility_hat(Uo, lam_tc)
    assert abs(g.feasibility()[1] - f_o[0]) <= 1e-6 * f_o[0]
    chi_o, w_o, _ = oracle.round_cut(L, Uo)
    chi_g, w_g = g.round()
    np.testing.assert_array_equal(chi_g, chi_o)
    assert w_g == w_o
    np.testing.assert_allclose(g.objective(), one.objective(), rtol=1e-9)
    np.testing.assert_allclose(g.feasibility(), one.feasibility(), rtol=1e-9)
    chi, w = g.round()
    chi1, w1 = one.round()
    np.testing.assert_array_equal(chi, chi1)
    assert abs(w - w1) <= 1e-9 * w1


@pytest.mark.parametrize("regenerate", [False, True])
def test_sharded_config1_signed_weights(gpu, regenerate):
    L = si.laplacian("c1")
    g = gpu.SketchyCGAL(L, R=10, seed=1, shards=4, regenerate=regenerate)
    g.step(120)
    o = oracle.Oracle(L, 10, seed=1, logcap=120)
    o.step(120)
    _assert_trajectory(g, o, 120)


@pytest.mark.parametrize("regenerate", [False, True])
def test_sharded_breakdown_complete_graph(gpu, regenerate):
    """Lanczos break (k < q) with P = 2: producers and pulls must skip together."""
    n = 8
    i, j = np.triu_indices(n, 1)
    L = si.laplacian_from_edges(n, i, j, np.ones(len(i)))
    g = gpu.SketchyCGAL(L, R=3, seed=2, shards=2, regenerate=regenerate)
    g.step(25)
    o = oracle.Oracle(L, 3, seed=2, logcap=25)
    o.step(25)
    _assert_trajectory(g, o, 25)


@pytest.mark.parametrize("n,P", [(3, 2), (33, 3), (257, 8), (1000, 5)])
def test_sharded_ragged_sizes(gpu, n, P):
    rng = np.random.default_rng(n)
    i = np.arange(n - 1)
    j = i + 1
    extra = rng.integers(0, n, size=(2 * n, 2))
    extra = extra[extra[:, 0] != extra[:, 1]]
    i = np.concatenate([i, extra[:, 0]])
    j = np.concatenate([j, extra[:, 1]])
    w = rng.uniform(0.5, 1.5, size=len(i))
    L = si.laplacian_from_edges(n, i, j, w)
    R = min(4, n)
    g = gpu.SketchyCGAL(L, R=R, seed=n, shards=P)
    g.step(40)
    o = oracle.Oracle(L, R, seed=n, logcap=40)
    o.step(40)
    _assert_trajectory(g, o, 40)


def test_sharded_heavy_row_and_explicit_splits(gpu):
    """A star centre (long row, warp engine) on the boundary between two uneven shards."""
    n = 3000
    i = np.zeros(n - 50, dtype=np.int64)
    j = np.arange(1, n - 49)
    L = si.laplacian_from_edges(n, i, j, np.ones(len(i)))
    g = gpu.SketchyCGAL(L, R=5, seed=9, shards=3, splits=np.array([0, 1, 1700, n]))
    g.step(30)
    o = oracle.Oracle(L, 5, seed=9, logcap=30)
    o.step(30)
    _assert_trajectory(g, o, 30)


@pytest.mark.parametrize("cfg,P,T", [("c2", 2, 2), ("c3", 2, 1)])
def test_sharded_full_size_first_iterations(gpu, cfg, P, T):
    L = si.laplacian(cfg)
    c = si.CONFIGS[cfg]
    g = gpu.SketchyCGAL(L, R=c["R"], seed=c["seed"], shards=P)
    g.step(T)
    o = oracle.Oracle(L, c["R"], seed=c["seed"], logcap=T)
    o.step(T)
    _assert_trajectory(g, o, T)


def _first_stop(log, n, nrmL, eps):
    """First t of a 12-column (scaled-units) iteration log meeting the stopping rule of
    PAPER.md:4044-4048 in original units (reading R28): objective x n ||L||_F, z x n, b = 1."""
    uz, uo = float(n), float(n) * nrmL
    nb = np.sqrt(n)
    for i in range(log.shape[0]):
        p_t = log[i - 1, 6] * uo if i > 0 else 0.0
        zres = log[i - 1, 7] * uz if i > 0 else nb
        if log[i, 11] * uo / (1.0 + abs(p_t)) <= eps and zres / (1.0 + nb) <= eps:
            return int(log[i, 0])
    return None


@pytest.mark.parametrize("shards", [1, 2])
def test_stopping_rule_run(gpu, shards):
    """sketchycgal_run stops at the first iteration meeting the paper's stopping rule (f2)."""
    L = si.laplacian("c0")
    o = oracle.Oracle(L, 10, seed=0, logcap=1000)
    o.step(1000)
    eps = 0.1
    t_o = _first_stop(o.log, L.n, o.nrmL, eps)
    assert t_o is not None and t_o > 1
    g = gpu.SketchyCGAL(L, R=10, seed=0, shards=shards)
    t = g.run(1000, eps=eps, check_every=37)
    assert t == t_o
    assert t_o <= g.t < t_o + 37


def _psd_cost_graph():
    """All-negative weights: C = -L is psd, so xi_t >= 0 (H = 0) happens early."""
    rng = np.random.default_rng(1)
    n = 60
    i, j = np.triu_indices(n, 1)
    keep = rng.random(len(i)) < 0.1
    return si.laplacian_from_edges(n, i[keep], j[keep], -np.ones(int(keep.sum())))


@pytest.mark.parametrize("graph,shards", [("psd", 1), ("psd", 3), ("c0", 1), ("c0", 2)])
def test_trace_bounded_lmo(gpu, graph, shards):
    """f3: tr X <= 1.05 n (SCG_TRACE_LE), H = 0 when xi_t >= 0: trajectory bitwise (the H = 0
    branch fires on the psd-cost graph), reconstruction trace-corrected to the tracked trace (R29)."""
    L = _psd_cost_graph() if graph == "psd" else si.laplacian("c0")
    T = 300
    R = 4 if graph == "psd" else 10
    alpha = 1.05 * L.n
    g = gpu.SketchyCGAL(L, R=R, seed=3, alpha=alpha, trace_le=True, shards=shards)
    g.step(T)
    o = oracle.Oracle(L, R, seed=3, alpha=alpha, trace_le=True, logcap=T)
    o.step(T)
    if graph == "psd":
        assert np.any(o.log[:, 4] >= 0.0)
    _assert_trajectory(g, o, T)
    U, lam, _ = g.reconstruct()
    Uo, lam_o, _ = oracle.nystrom_reconstruct(o.S, o.Omega, o.tau)
    lam_tc = oracle.trace_correct(lam_o, o.tau) * L.n
    np.testing.assert_allclose(lam, lam_tc, rtol=1e-9)
    assert abs(lam.sum() - o.tau * L.n) <= 1e-9 * abs(o.tau * L.n)


def test_sharded_rejects_asymmetric_pattern(gpu):
    """The halo plan is exact only for a symmetric pattern: an emulated-shard init rejects an
    asymmetric CSR (SCG_EINVAL), a single-GPU init accepts it."""
    L = si.laplacian("c1")
    rp, col, val = L.row_ptr.copy(), L.col.copy(), L.val.copy()
    # drop one off-diagonal entry of row 5 (not its transpose): structurally asymmetric
    r = 5
    a, b = int(rp[r]), int(rp[r + 1])
    k = next(k for k in range(a, b) if col[k] != r)
    keep = np.ones(len(col), dtype=bool)
    keep[k] = False
    rp2 = rp.copy()
    rp2[r + 1:] -= 1
    bad = si.CSR(L.n, rp2, col[keep], val[keep])
    with pytest.raises(gpu.ScgError):
        gpu.SketchyCGAL(bad, R=4, seed=1, shards=2)
    gpu.SketchyCGAL(bad, R=4, seed=1).close()


@pytest.mark.parametrize("resident,serial", [(False, False), (True, False), (False, True)])
def test_bench_launch_configuration_bitwise(gpu, resident, serial):
    """The configuration bench.py times -- torch's stream passed in (high priority), SCG_PROFILE event
    sampling, programmatic dependent launches, the side-stream start vectors (multi-kernel) or the
    resident cluster kernel -- gives the oracle's bits (configs[1] shape, 200 iterations)."""
    import ctypes
    import torch
    L = si.laplacian("c1")
    stream = torch.cuda.Stream(priority=-100)
    with torch.cuda.stream(stream):
        g = gpu.SketchyCGAL(L, R=10, seed=1, profile=True, stream=ctypes.c_void_p(stream.cuda_stream),
                            resident=resident, serial_rng=serial)
        g.step(3)
        g.synchronize()
        g.reset_stats()
        g.step(197)
        g.synchronize()
        stats = {s["name"]: s for s in g.kernel_stats()}
    main = "resident_iteration" if resident else "lanczos_a_spmv_dot"
    assert stats[main]["launches"] > 0 and stats[main]["total_ms"] > 0
    flow = stats["lanczos_pass1_in_flow"]  # whole passes 1 between one pair of events (every 8th iteration)
    if resident:
        assert flow["launches"] == 0
    else:  # t = 8, 16, ..., 200; a pass moves q k_lanczos_a + (q - 1) k_lanczos_b launches' bytes
        assert flow["launches"] == 25 and flow["total_ms"] > 0
        pair = stats["lanczos_a_spmv_dot"]["bytes_per_launch"] + stats["lanczos_b_axpy_norm"]["bytes_per_launch"]
        assert flow["bytes_per_launch"] > 10 * pair
    o = oracle.Oracle(L, 10, seed=1, logcap=200)
    o.step(200)
    _assert_trajectory(g, o, 200)


@pytest.mark.parametrize("graph,alpha0,T", [("c5", 1.25, 3000), ("c0", 400.0, 200)])
def test_alpha_doubling_driver_matches_oracle(gpu, graph, alpha0, T):
    """Standard-form driver through the C ABI against the oracle's: the same
    alpha sequence, stopping round and decision; per-round implicit objectives to rounding."""
    if graph == "c5":
        n = 5
        i = np.arange(n)
        L = si.laplacian_from_edges(n, i, (i + 1) % n, np.ones(n))
        R, seed = 3, 5
    else:
        L = si.laplacian("c0")
        R, seed = 10, 0
    g, al, ob, conv = gpu.SketchyCGAL.alpha_doubling(L, R, alpha0=alpha0, T=T, rtol=1e-2, max_rounds=5, seed=seed)
    o, al_o, ob_o, conv_o = oracle.alpha_doubling(L, R, alpha0=alpha0, T=T, rtol=1e-2, max_rounds=5, seed=seed)
    np.testing.assert_array_equal(al, al_o)
    assert conv == conv_o
    np.testing.assert_allclose(ob, ob_o, rtol=1e-12, atol=0)
    np.testing.assert_array_equal(g.state("z"), o.z)  # the last round's iterate, bitwise
    g.close()


@pytest.mark.parametrize("graph,shards,trace_le", [("c0", 1, False), ("c0", 2, False), ("c5", 1, True),
                                                   ("c1", 1, False)])
def test_inequality_template_bitwise(gpu, graph, shards, trace_le):
    """General template with K = {u <= b} (SCG_INEQ): slack w = min(z + y/beta, b) in
    D_t and in the dual update; every iterate bitwise against the oracle (sharded too)."""
    if graph == "c5":
        n = 5
        i = np.arange(n)
        L = si.laplacian_from_edges(n, i, (i + 1) % n, np.ones(n))
        R, seed, T, alpha = 3, 5, 400, 2.5
    else:
        L = si.laplacian(graph)
        c = si.CONFIGS[graph]
        R, seed, T, alpha = c["R"], c["seed"], 200, None
    g = gpu.SketchyCGAL(L, R=R, seed=seed, alpha=alpha, ineq=True, trace_le=trace_le, shards=shards)
    g.step(T)
    o = oracle.Oracle(L, R, seed=seed, alpha=alpha, logcap=T, ineq=True, trace_le=trace_le)
    o.step(T)
    _assert_trajectory(g, o, T)


@pytest.mark.parametrize("graph,box,shards", [("c0", (0.8, 1.2), 1), ("c0", (0.8, 1.2), 3), ("c5", (0.7, 1.3), 1)])
def test_box_constraint_set_bitwise(gpu, graph, box, shards):
    """Box K = {lo <= u <= hi} through sketchycgal_set_box: every iterate bitwise
    against the oracle; the setter refuses NaN / inverted bounds and calls after the first step."""
    if graph == "c5":
        n = 5
        i = np.arange(n)
        L = si.laplacian_from_edges(n, i, (i + 1) % n, np.ones(n))
        R, seed, T = 3, 5, 400
    else:
        L = si.laplacian(graph)
        R, seed, T = 10, 0, 200
    alpha = 1.05 * L.n * box[1]
    g = gpu.SketchyCGAL(L, R=R, seed=seed, alpha=alpha, trace_le=True, box=box, shards=shards)
    g.step(T)
    o = oracle.Oracle(L, R, seed=seed, alpha=alpha, logcap=T, trace_le=True, box=box)
    o.step(T)
    _assert_trajectory(g, o, T)
    assert g.lib.sketchycgal_set_box(g._h, 0.5, 1.5) != 0  # after the first step
    h = gpu.SketchyCGAL(L, R=R, seed=seed)
    assert h.lib.sketchycgal_set_box(h._h, 1.5, 0.5) != 0
    assert h.lib.sketchycgal_set_box(h._h, float("nan"), 1.0) != 0


@pytest.mark.parametrize("norm", ["l2", "l1"])
@pytest.mark.parametrize("graph,delta,shards", [("c0", 3.0, 1), ("c0", 3.0, 3), ("c0", 200.0, 1), ("c5", 0.4, 1),
                                                ("c5", 0.0, 2)])
def test_ball_constraint_sets_bitwise(gpu, graph, delta, shards, norm):
    """l2 / l1 balls K = {||u - 1|| <= delta} through sketchycgal_set_ball / _set_ball_l1 (P:3915-3918,
    readings R34, R35): the l2 scale is an exact-sum norm over all shards and the l1 threshold comes
    from an exact bisection over all shards, so every iterate is bitwise equal to the oracle's (which
    sorts) -- with the projection active (small delta), mostly inactive (delta = 200 on c0), and
    delta = 0 (the projection is then exactly b).  The setters refuse negative / NaN delta and calls
    after the first step."""
    if graph == "c5":
        n = 5
        i = np.arange(n)
        L = si.laplacian_from_edges(n, i, (i + 1) % n, np.ones(n))
        R, seed, T = 3, 5, 400 if norm == "l2" else 150
    else:
        L = si.laplacian(graph)
        R, seed, T = 10, 0, 200 if norm == "l2" else 60
    r = np.sqrt(L.n) if norm == "l2" else L.n
    alpha = 1.05 * L.n * (1 + delta / r)
    kw = {"ball": delta} if norm == "l2" else {"l1_ball": delta}
    g = gpu.SketchyCGAL(L, R=R, seed=seed, alpha=alpha, trace_le=True, shards=shards, **kw)
    g.step(T)
    o = oracle.Oracle(L, R, seed=seed, alpha=alpha, logcap=T, trace_le=True, **kw)
    o.step(T)
    _assert_trajectory(g, o, T)
    setter = g.lib.sketchycgal_set_ball if norm == "l2" else g.lib.sketchycgal_set_ball_l1
    assert setter(g._h, 1.0) != 0  # after the first step
    h = gpu.SketchyCGAL(L, R=R, seed=seed)
    setter = h.lib.sketchycgal_set_ball if norm == "l2" else h.lib.sketchycgal_set_ball_l1
    assert setter(h._h, -1.0) != 0
    assert setter(h._h, float("nan")) != 0


@pytest.mark.parametrize("P", [2, 3, 8])
def test_sharded_inline_pulls_bitwise(gpu, P):
    """SCG_INLINE_PULL: each Lanczos step's omega / rho collective pulled in the prologue of the kernel
    that consumes it (no k_pull launches inside pass 1) -- the oracle's bits (c0, 200 iterations), and
    the Lanczos breakdown of K_8 (k = 2 < q) sharded the same way."""
    L = si.laplacian("c0")
    T = 200
    g = gpu.SketchyCGAL(L, R=10, seed=0, shards=P, inline_pull=True)
    g.step(T)
    o = oracle.Oracle(L, 10, seed=0, logcap=T)
    o.step(T)
    _assert_trajectory(g, o, T)
    n = 8
    i, j = np.triu_indices(n, 1)
    K8 = si.laplacian_from_edges(n, i, j, np.ones(len(i)))
    g8 = gpu.SketchyCGAL(K8, R=3, seed=2, shards=min(P, 4), inline_pull=True)
    g8.step(25)
    o8 = oracle.Oracle(K8, 3, seed=2, logcap=25)
    o8.step(25)
    assert o8.log[0, 2] == 2
    _assert_trajectory(g8, o8, 25)
