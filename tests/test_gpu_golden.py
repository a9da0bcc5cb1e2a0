"""GPU parity on the long cases: the CUDA path (through the C ABI) against the oracle's
trajectories stored in tests/golden/ (written by tests/golden/make_golden.py, which calls only
oracle/ -- no value there comes from the CUDA path).

Bar: the feedback-path records (t, q, k, theta, ||z - b||, gamma, gap,
bound) are bitwise equal at every t, z / y / v / Omega are bitwise equal (SHA-256 of their bytes),
xi, c, p, tau agree to 1e-13 relative, S to 1e-13 max|S| at 512 sampled rows; after T the
reconstruction-based objective and feasibility agree to 1e-6 (BASELINE north_star) and the rounded
cut is identical.
"""
import ctypes
import hashlib
import json
import os

import numpy as np
import pytest

import scg_inputs as si

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
BITWISE_COLS = [0, 1, 2, 3, 7, 8, 10, 11]  # t q k theta znorm gamma gap bound
ROUNDING_COLS = [4, 5, 6, 9]                 # xi c p tau


def _golden(name):
    with open(os.path.join(HERE, "golden", f"{name}.json")) as f:
        return json.load(f)


def _unhex(a):
    return np.array([float.fromhex(v) for v in a], dtype=np.float64)


def _digest(x):
    return hashlib.sha256(np.ascontiguousarray(x, dtype="<f8").tobytes()).hexdigest()


def _check(g, ref):
    T, R = ref["T"], ref["R"]
    gl = g.iter_log()
    ol = np.array([_unhex(r) for r in ref["log"]])
    assert gl.shape == ol.shape == (T, 12)
    np.testing.assert_array_equal(gl[:, BITWISE_COLS], ol[:, BITWISE_COLS])
    np.testing.assert_allclose(gl[:, ROUNDING_COLS], ol[:, ROUNDING_COLS], rtol=1e-13, atol=0)
    for k in ("z", "y", "v", "Omega"):
        assert _digest(g.state(k)) == ref["sha256"][k], k
    S = g.state("S")
    rows = np.array(ref["S_rows"])
    want = _unhex(ref["S_sample"]).reshape(len(rows), R)
    np.testing.assert_allclose(S[rows, :], want, rtol=0, atol=1e-13 * float.fromhex(ref["S_absmax"]))
    assert abs(float(np.abs(S).max()) - float.fromhex(ref["S_absmax"])) <= 1e-13 * float.fromhex(ref["S_absmax"])


def test_config3_bench_window_t1_25_bitwise(gpu):
    """configs[3] (n = 2^24) t = 1..25 -- the window the driver's bench run times (W = 5, K = 20) -- in
    bench.py's launch configuration (torch's stream, SCG_PROFILE event sampling, programmatic launches);
    includes the deferred sketch flush at t = 16 on the full-size S."""
    import torch
    ref = _golden("c3_t25")
    L = si.laplacian("c3")
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        g = gpu.SketchyCGAL(L, R=ref["R"], seed=ref["seed"], profile=True, stream=ctypes.c_void_p(stream.cuda_stream))
        g.step(5)
        g.synchronize()
        g.reset_stats()
        g.step(20)
        g.synchronize()
    _check(g, ref)
    g.close()


def test_config2_t1_100_bitwise(gpu):
    """configs[2] (n = 2^20, Zipf hubs up to ~7.9k entries: long rows, dynamic slices) t = 1..100."""
    ref = _golden("c2_t100")
    g = gpu.SketchyCGAL(si.laplacian("c2"), R=ref["R"], seed=ref["seed"])
    g.step(ref["T"])
    _check(g, ref)
    g.close()


def test_config4_real_R20_t1_5_bitwise(gpu):
    """configs[4] (n = 2^25, weights U[0.5, 1.5], random matching) at its real sketch rank R = 20."""
    ref = _golden("c4_t5")
    assert ref["R"] == 20
    g = gpu.SketchyCGAL(si.laplacian("c4"), R=ref["R"], seed=ref["seed"])
    g.step(ref["T"])
    _check(g, ref)
    g.close()


def test_config1_whole_run_T5000_objective_feasibility_cut(gpu):
    """configs[1] for its whole run T = 5000: every record, the state, and after T the trace-corrected
    reconstruction, objective tr(L X^) and ||diag X^ - 1|| (1e-6, BASELINE), the implicit objective and
    infeasibility, and the identical rounded cut."""
    ref = _golden("c1_T5000")
    L = si.laplacian("c1")
    g = gpu.SketchyCGAL(L, R=ref["R"], seed=ref["seed"])
    g.step(ref["T"])
    _check(g, ref)
    U, lam, err = g.reconstruct()
    np.testing.assert_allclose(lam, _unhex(ref["Lambda_tc"]), rtol=1e-9)
    obj = g.objective()
    assert abs(obj[0] - float.fromhex(ref["implicit_objective"])) <= 1e-12 * abs(obj[0])
    o_hat = float.fromhex(ref["objective_hat_tc"])
    assert abs(obj[1] - o_hat) <= 1e-6 * abs(o_hat)
    fz = g.feasibility()
    f_o = _unhex(ref["feasibility_hat_tc"])
    assert abs(fz[0] - float.fromhex(ref["implicit_infeasibility"])) <= 1e-10 * fz[0]
    assert abs(fz[1] - f_o[0]) <= 1e-6 * f_o[0] and abs(fz[2] - f_o[1]) <= 1e-6 * f_o[1]
    chi, w = g.round()
    assert hashlib.sha256(np.ascontiguousarray(chi, dtype=np.int8).tobytes()).hexdigest() == ref["chi_sha256"]
    assert w == float.fromhex(ref["cut_weight"])
    g.close()


def test_fixed_q255_beyond_127_bitwise(gpu):
    """Fixed Lanczos bound q = 255 (sketchycgal_set_lanczos_q) on configs[1]: k_tridiag, k_combine and the
    grown Lanczos store at k > 127, every iterate bitwise."""
    ref = _golden("c1_q255")
    assert ref["qfix"] == 255
    g = gpu.SketchyCGAL(si.laplacian("c1"), R=ref["R"], seed=ref["seed"], qfix=255)
    g.step(ref["T"])
    _check(g, ref)
    assert int(g.iter_log()[:, 2].max()) > 127
    g.close()


def test_q_above_device_bound_is_an_error(gpu):
    """q beyond the device bound is refused (SCG_EINVAL), never silently truncated."""
    L = si.laplacian("c1")
    with pytest.raises(gpu.ScgError):
        gpu.SketchyCGAL(L, R=4, seed=1, qfix=256)
