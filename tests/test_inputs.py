"""Seeded input generators (scg_inputs): statistical and structural checks."""
import math

import numpy as np

import scg_inputs as si


def _u53(hi, lo):
    return ((int(hi) << 32) | int(lo)) >> 11


def test_normal_matches_box_muller_with_libm():
    # The fixed-polynomial ln / cos of scg_rng.h against libm Box-Muller on the same uniforms.
    seed, stream, sub = 12345, 1, 7
    g = si.normals(seed, stream, sub, 0, 2000)
    for i in range(0, 2000, 37):
        w = si.philox([i & 0xffffffff, i >> 32, sub, stream], [seed & 0xffffffff, seed >> 32])
        u1 = (_u53(w[0], w[1]) + 1) * 2.0 ** -53
        u2 = _u53(w[2], w[3]) * 2.0 ** -53
        ref = math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)
        assert abs(g[i] - ref) <= 4e-15 * max(1.0, abs(ref))


def test_normal_moments():
    g = si.normals(1, 0, 3, 0, 1_000_000)
    assert abs(g.mean()) < 5 / math.sqrt(1e6)
    assert abs(g.var() - 1.0) < 5 * math.sqrt(2 / 1e6)
    assert abs((g ** 3).mean()) < 5 * math.sqrt(15 / 1e6)
    assert abs((g ** 4).mean() - 3.0) < 5 * math.sqrt(96 / 1e6)
    # tail probabilities against the normal CDF
    for a in (1.0, 2.0, 3.0):
        p = (np.abs(g) > a).mean()
        ref = math.erfc(a / math.sqrt(2))
        assert abs(p - ref) < 5 * math.sqrt(ref * (1 - ref) / 1e6)


def test_streams_are_distinct_and_deterministic():
    a = si.normals(0, 0, 0, 0, 1000)
    b = si.normals(0, 1, 0, 0, 1000)
    c = si.normals(0, 0, 1, 0, 1000)
    assert np.array_equal(a, si.normals(0, 0, 0, 0, 1000))
    assert not np.allclose(a, b) and not np.allclose(a, c)
    # counter addressing: a window equals the slice of the full stream
    assert np.array_equal(si.normals(0, 0, 0, 500, 10), a[500:510])


def _check_laplacian(L):
    n = L.n
    rows = np.repeat(np.arange(n), np.diff(L.row_ptr))
    # symmetric, columns ascending, diagonal = weighted degree (L 1 = 0)
    for r in range(min(n, 2000)):
        c = L.col[L.row_ptr[r]:L.row_ptr[r + 1]]
        assert np.all(np.diff(c) > 0)
    rs = np.zeros(n)
    np.add.at(rs, rows, L.val)
    assert np.allclose(rs, 0.0, atol=1e-9)
    key = rows * n + L.col
    keyt = L.col.astype(np.int64) * n + rows
    o1, o2 = np.argsort(key), np.argsort(keyt)
    assert np.array_equal(key[o1], keyt[o2])
    assert np.array_equal(L.val[o1], L.val[o2])


def test_er_shape():
    L = si.laplacian("c0")
    _check_laplacian(L)
    m = L.m
    mu = 0.06 * 800 * 799 / 2
    assert abs(m - mu) < 5 * math.sqrt(mu)
    assert np.all(L.val[L.col != np.repeat(np.arange(L.n), np.diff(L.row_ptr))] == -1.0)


def test_torus_shape():
    L = si.laplacian("c1")
    _check_laplacian(L)
    assert L.n == 8000 and L.m == 16000
    assert np.all(np.diff(L.row_ptr) == 5)
    i, j, w = L.edges()
    assert set(np.unique(w)) == {-1.0, 1.0}
    assert abs((w > 0).mean() - 0.5) < 0.02


def test_small_families():
    L = si.generate("powerlaw", 1 << 14, seed=2)
    _check_laplacian(L)
    d = np.diff(L.row_ptr) - 1
    assert 6.0 < d.mean() < 9.0 and d.max() > 50
    L = si.generate("rgg", 1 << 16, seed=3)
    _check_laplacian(L)
    d = np.diff(L.row_ptr) - 1
    assert 2.2 < d.mean() < 2.6 and d.max() <= 4
    L = si.generate("ring_matching", 1 << 14, seed=4)
    _check_laplacian(L)
    d = np.diff(L.row_ptr) - 1
    assert d.max() == 3 and (d == 3).mean() > 0.99
    i, j, w = L.edges()
    assert w.min() >= 0.5 and w.max() <= 3.0


def test_laplacian_from_edges_merges_and_drops_loops():
    L = si.laplacian_from_edges(3, [0, 0, 1, 2], [1, 1, 2, 2], [1.0, 1.0, 1.0, 5.0])
    D = L.dense()
    assert np.array_equal(D, np.array([[2.0, -2.0, 0.0], [-2.0, 3.0, -1.0], [0.0, -1.0, 1.0]]))
