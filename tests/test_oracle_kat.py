"""Known-answer tests of the reference, restated against the CPU oracle.

Each test mirrors a doctest case of proj/tests/test_spectral.cpp or
proj/tests/test_mesh.cpp (file:line in the docstring) with the reference's own
tolerances; together they pin the oracle's spectral/mesh restatement to the
reference's published expectations.
"""
import math

import numpy as np
import pytest


def test_cheb_lobatto_nodes(oracle):
    """proj/tests/test_spectral.cpp:13-30"""
    assert list(oracle.cheb_lobatto(2)) == [1.0, -1.0]
    assert list(oracle.cheb_lobatto(3)) == [1.0, 0.0, -1.0]
    x5 = oracle.cheb_lobatto(5)
    for k in range(5):
        assert abs(x5[k] - math.cos(math.pi * k / 4)) < 1e-15
    assert x5[1] == pytest.approx(math.sqrt(2) / 2, rel=1e-15)


@pytest.mark.parametrize("p", [2, 5, 8, 13, 16])
def test_clenshaw_curtis(oracle, p):
    """proj/tests/test_spectral.cpp:32-43"""
    x, w = oracle.cheb_lobatto(p), oracle.cheb_weights(p)
    for deg in range(p):
        exact = 2.0 / (deg + 1) if deg % 2 == 0 else 0.0
        assert abs(np.sum(w * x ** deg) - exact) < 1e-13


def test_gauss_legendre(oracle):
    """proj/tests/test_spectral.cpp:45-69"""
    n1, w1 = oracle.gauss(1)
    assert n1[0] == 0.0 and w1[0] == pytest.approx(2.0, rel=1e-15)
    n2, w2 = oracle.gauss(2)
    assert n2[0] == pytest.approx(-1 / math.sqrt(3), rel=1e-15)
    assert n2[1] == pytest.approx(1 / math.sqrt(3), rel=1e-15)
    assert w2[0] == pytest.approx(1.0, rel=1e-14)
    n6, w6 = oracle.gauss(6)
    assert abs(np.sum(w6 * n6 ** 10) - 2 / 11) < 1e-14
    for n in [1, 2, 3, 6, 10, 14]:
        x, w = oracle.gauss(n)
        assert abs(w.sum() - 2.0) < 1e-14
        assert np.all(w > 0)
        for i in range(n):
            assert x[i] == pytest.approx(-x[n - 1 - i], rel=1e-14, abs=1e-300)


def test_diff_matrix(oracle):
    """proj/tests/test_spectral.cpp:71-99"""
    d2 = oracle.diff_matrix(2)
    assert np.allclose(d2, [[0.5, -0.5], [0.5, -0.5]], rtol=1e-15, atol=0)
    d8 = oracle.diff_matrix(8)
    assert np.abs(d8 @ np.ones(8)).max() < 1e-13
    x = oracle.cheb_lobatto(5)
    assert np.abs(oracle.diff_matrix(5) @ x ** 3 - 3 * x ** 2).max() < 1e-13
    for p in [6, 10, 16]:
        xs, d = oracle.cheb_lobatto(p), oracle.diff_matrix(p)
        for k in range(1, p):
            assert np.abs(d @ xs ** k - k * xs ** (k - 1)).max() < 1e-10


def test_barycentric(oracle):
    """proj/tests/test_spectral.cpp:101-119"""
    x = oracle.cheb_lobatto(7)
    assert np.abs(oracle.interp_matrix(x, x) - np.eye(7)).max() == 0.0
    g, _ = oracle.gauss(6)
    c8 = oracle.cheb_lobatto(8)
    m = oracle.interp_matrix(g, c8)
    assert np.abs(m.sum(axis=1) - 1).max() < 1e-13
    assert np.abs(m @ g ** 5 - c8 ** 5).max() < 1e-13
    with pytest.raises(RuntimeError):
        oracle.interp_matrix(np.array([0.5, 0.5]), c8)


def test_dtn_ops_2d(oracle):
    """proj/tests/test_spectral.cpp:121-166"""
    p, q = 8, 6
    P, Q = oracle.dtn_ops(2, p, 2.0)
    assert P.shape == (4 * p - 4, 4 * q) and Q.shape == (4 * q, p * p)
    assert np.abs(P @ np.ones(4 * q) - 1).max() < 1e-13
    pts = oracle.leaf_cheb_points([-1, -1], [1, 1], p, 2)
    qn = Q @ pts[:, 0]
    expect = np.concatenate([np.zeros(q), np.ones(q), np.zeros(q), -np.ones(q)])
    assert np.abs(qn - expect).max() < 1e-12
    x, y = pts[:, 0], pts[:, 1]
    q3 = Q @ (x ** 3 + x * y ** 2 - 2 * y ** 3)
    gp = oracle.gauss_boundary_points([-1, -1], [1, 1], q, 2)
    ux = lambda x, y: 3 * x * x + y * y
    uy = lambda x, y: 2 * x * y - 6 * y * y
    for s in range(4):
        for i in range(q):
            gx, gy = gp[s * q + i, 0], gp[s * q + i, 1]
            e = [-uy(gx, gy), ux(gx, gy), uy(gx, gy), -ux(gx, gy)][s]
            assert abs(q3[s * q + i] - e) < 1e-12


def test_dtn_ops_3d(oracle):
    """proj/tests/test_spectral.cpp:204-227"""
    p, q = 8, 6
    P, Q = oracle.dtn_ops(3, p, 2.0)
    assert P.shape == (296, 216) and Q.shape == (216, 512)
    assert np.abs(P @ np.ones(216) - 1).max() < 1e-12
    assert np.abs(Q @ np.ones(512)).max() < 1e-11
    pts = oracle.leaf_cheb_points([-1, -1, -1], [1, 1, 1], p, 3)
    qn = Q @ pts[:, 2]
    for f in range(6):
        e = {4: -1.0, 5: 1.0}.get(f, 0.0)
        assert np.abs(qn[f * q * q:(f + 1) * q * q] - e).max() < 1e-11


def test_refinement_and_face_projection(oracle):
    """proj/tests/test_spectral.cpp:229-271"""
    p = 4
    l8 = oracle.refinement_interpolant(p)
    assert l8.shape[0] == 8 * p ** 3
    assert np.abs(l8 @ np.ones(p ** 3) - 1).max() < 1e-13
    ref = oracle.leaf_cheb_points([-1, -1, -1], [1, 1, 1], p, 3)
    fine = l8 @ (ref[:, 0] * ref[:, 1] * ref[:, 2])
    off = [(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1)]
    idx = 0
    for c in range(8):
        lo = [0.0 if off[c][k] else -1.0 for k in range(3)]
        hi = [1.0 if off[c][k] else 0.0 for k in range(3)]
        for x in oracle.leaf_cheb_points(lo, hi, p, 3):
            assert abs(fine[idx] - x[0] * x[1] * x[2]) < 1e-14
            idx += 1
    q = 6
    refine, coarsen = oracle.face_projection(q)
    assert refine.shape == (4 * q * q, q * q) and coarsen.shape == (q * q, 4 * q * q)
    assert np.abs(refine @ np.ones(q * q) - 1).max() < 1e-13
    assert np.abs(coarsen @ np.ones(4 * q * q) - 1).max() < 1e-13
    g, _ = oracle.gauss(q)
    data = np.array([g[a] ** (q - 1) * g[b] ** (q - 2) + 0.25 * g[b] for a in range(q) for b in range(q)])
    assert np.abs(coarsen @ (refine @ data) - data).max() < 1e-13


@pytest.mark.parametrize("p", [6, 8, 12, 16])
def test_p_polynomial_exactness(oracle, p):
    """proj/tests/test_spectral.cpp:281-316"""
    q = p - 2
    P, _ = oracle.dtn_ops(2, p, 2.0)
    assert np.abs(P.sum(axis=1) - 1).max() < 1e-13
    poly = lambda t: t ** (q - 1) - 0.5 * t
    gp = oracle.gauss_boundary_points([-1, -1], [1, 1], q, 2)
    src = np.array([poly(gp[i, 0] if (i // q) in (0, 2) else gp[i, 1]) for i in range(4 * q)])
    dst = P @ src
    cpts = oracle.leaf_cheb_points([-1, -1], [1, 1], p, 2)
    _, ie = oracle.index_sets(p, 2)
    for r, idx in enumerate(ie):
        x = cpts[idx]
        on_sn = abs(abs(x[1]) - 1) < 1e-14
        on_ew = abs(abs(x[0]) - 1) < 1e-14
        if on_sn and on_ew:
            e = 0.5 * (poly(x[0]) + poly(x[1]))
        elif on_sn:
            e = poly(x[0])
        else:
            e = poly(x[1])
        assert abs(dst[r] - e) < 1e-12


def test_uniform_tree_counts(oracle):
    """proj/tests/test_mesh.cpp:18-35 (config 1: L=3, p=16 -> 64 leaves, N = 16,384)"""
    t1 = oracle.tree_info(2, 1, 8, [0, 0], [1, 1])
    assert t1["n_leaves"] == 4 and t1["total_points"] == 256
    t2 = oracle.tree_info(3, 0, 8, [0, 0, 0], [1, 1, 1])
    assert t2["n_leaves"] == 1 and t2["total_points"] == 512
    t3 = oracle.tree_info(2, 3, 16, [0, 0], [1, 1])
    assert t3["n_leaves"] == 64 and t3["total_points"] == 16384
    with pytest.raises(RuntimeError):
        oracle.tree_info(2, 1, 3, [0, 0], [1, 1])


def test_leaf_points(oracle):
    """proj/tests/test_mesh.cpp:37-77"""
    p2 = oracle.leaf_cheb_points([-1, -1], [1, 1], 2, 2)
    corners = {(x[0], x[1]) for x in p2}
    assert (-1, -1) in corners and (1, 1) in corners
    p3 = oracle.leaf_cheb_points([0, 0], [1, 1], 3, 2)
    assert set(p3[:, 0]) == {0.0, 0.5, 1.0}
    p8 = oracle.leaf_cheb_points([-1, -1], [1, 1], 8, 2)
    assert sum(1 for x in p8 if abs(x[0]) == 1.0 or abs(x[1]) == 1.0) == 28
    g2 = oracle.gauss_boundary_points([-1, -1], [1, 1], 6, 2)
    assert len(g2) == 24 and np.all(np.abs(g2[:, 0] * g2[:, 1]) < 1)
    assert len(oracle.gauss_boundary_points([0, 0, 0], [1, 1, 1], 6, 3)) == 216
    g1 = oracle.gauss_boundary_points([-1, -1], [1, 1], 1, 2)
    assert len(g1) == 4 and g1[0][0] == pytest.approx(0.0) and g1[0][1] == -1.0
    assert g1[1][0] == 1.0 and g1[1][1] == pytest.approx(0.0)
