"""CPU-side checks of the C-ABI boundary (include/hps_cuda.h / libhps_b200.so):
the library loads and exports every declared entry point, host-only geometry
(orderings of leaf and root-boundary points) matches the oracle bit-for-bit, and
the product fails loudly without a CUDA device (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2503_17535_b200 as H
from paper_2503_17535_b200 import hps as HP

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hps_cuda.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hpsg_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = H.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert b"sm_100a" in lib.hpsg_build_info()


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", HP.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", HP.LIB_PATH], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass  # FP64 tensor-core path
    assert "UCGABAR" in sass or "barrier.cluster" in sass or "CCTL" in sass or "MAPA" in sass  # cluster/DSMEM panel


def _tree(dim, p, L, lo, hi):
    return HP._Tree(dim, p, L, lo, hi)


@pytest.mark.parametrize("dim,p,L,lo,hi", [(2, 16, 3, -1.0, 1.0), (2, 8, 2, 0.1, 0.225), (3, 6, 2, 0.0, 1.0)])
def test_host_geometry_matches_oracle(oracle, dim, p, L, lo, hi):
    from paper_2503_17535_b200 import problems as PR
    from tests.oracle_problems import oracle_solver
    lib = H.lib()
    lib.hpsg_tree_leaf_points.argtypes = [C.POINTER(HP._Tree), C.POINTER(C.c_double)]
    lib.hpsg_tree_root_points.argtypes = [C.POINTER(HP._Tree), C.POINTER(C.c_double)]
    t = H.build_uniform_tree(lo, hi, L, dim, p)
    tr = _tree(dim, p, L, lo, hi)
    pts = np.zeros((t.n_leaves, p ** dim, 3))
    assert lib.hpsg_tree_leaf_points(C.byref(tr), HP._dp(pts)) == 0
    rp = np.zeros((t.root_boundary_size, 3))
    assert lib.hpsg_tree_root_points(C.byref(tr), HP._dp(rp)) == 0
    prob = PR.laplace_poly2d() if dim == 2 else PR.CATALOG["laplace3d"]()
    prob.lo, prob.hi = lo, hi
    o = oracle_solver(prob, p, L)
    o.build()
    assert np.array_equal(pts, o.leaf_points())
    assert np.array_equal(rp, o.root_points())
    info = oracle.tree_info(dim, L, p, [lo] * dim, [hi] * dim)
    assert info["n_leaves"] == t.n_leaves and info["total_points"] == t.total_points


def test_no_device_fails_loudly():
    if H.lib().hpsg_device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(H.HpsError) as e:
        H.HpsSolver(H.build_uniform_tree(-1, 1, 2, 2, 8), [H.Term(H.ROLE_LAPLACIAN, H.Field.const(1.0))])
    assert e.value.code == HP.HPSG_ERR_NO_DEVICE


def test_cpp_dropin_example_builds_and_fails_loudly_without_device():
    exe = os.path.join(ROOT, "examples", "solve_problem_b200")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2503_17535_b200"), "example"], check=True)
    if H.lib().hpsg_device_count() > 0:
        pytest.skip("a CUDA device is present (run by the gpu tests)")
    r = subprocess.run([exe, "2", "8"], capture_output=True, text=True)
    assert r.returncode == 1 and "no CUDA device" in r.stderr


def test_iti_leaf_operator_kats():
    """proj/tests/test_spectral.cpp:168-203 ("2D ItI leaf operators") on the product's host operators:
    G 1 = i eta on every walk point, QH 1 = Q H 1 = -i eta, QH x1 on the east side = 1 - i eta,
    G - Ntilde is exactly the i eta walk sampling (4p-4 entries)."""
    import ctypes as C
    import numpy as np
    import paper_2503_17535_b200 as H
    from paper_2503_17535_b200 import hps as HP
    p, q, eta = 8, 6, 2.5
    n, nbc, nb = p * p, 4 * p - 4, 4 * q
    L = H.lib()
    L.hpsg_iti_leaf_ops.argtypes = [C.c_int, C.c_double, C.c_double] + [C.POINTER(C.c_double)] * 5
    Gr, Gi, P = np.zeros((n, nbc)), np.zeros((n, nbc)), np.zeros((nb, nbc))
    QHr, QHi = np.zeros((n, nb)), np.zeros((n, nb))
    assert L.hpsg_iti_leaf_ops(p, eta, 2.0, *(HP._dp(a) for a in (Gr, Gi, P, QHr, QHi))) == 0
    G = (Gr + 1j * Gi).T            # column-major buffers -> (rows, cols)
    QH = (QHr + 1j * QHi).T
    P = P.T
    one = np.ones(n)
    assert np.abs(G @ one - 1j * eta).max() < 1e-12
    assert np.abs(QH @ one + 1j * eta).max() < 1e-12
    assert np.abs(P.sum(axis=1) - 1.0).max() < 1e-13          # Gauss -> walk interpolation of constants
    m = p - 1                                                    # cheb_lobatto_1d (spectral.cpp:14-26)
    cn = np.sin(np.pi * (m - 2 * np.arange(p)) / (2 * m))
    pts = np.zeros((n, 3))
    pts[:, 0] = cn[np.arange(n) // p]                            # x1 of tensor index i1*p + i2
    hu = QH @ pts[:, 0]
    assert np.abs(hu[q:2 * q] - (1.0 - 1j * eta)).max() < 1e-11   # east side (s = 1) rows
    assert (np.abs(Gi) > 0).sum() == 4 * p - 4 and np.allclose(Gi[Gi != 0], eta)


def test_fdm_leaf_operator_host_math():
    """Host side of the fast-diagonalisation leaf solve (hpsg_fdm_leaf_ops): A = s^2 a D2[int, int] has a real
    eigendecomposition A = V diag(lam) V^-1 to roundoff, and the separable factors reproduce the interior Q
    (the product's make_leaf_operators Q, itself checked against the reference in test_ref_parity) bit for bit."""
    import ctypes as C
    import numpy as np
    import paper_2503_17535_b200 as H
    from paper_2503_17535_b200 import hps as HP
    L = H.lib()
    dp = C.POINTER(C.c_double)
    L.hpsg_fdm_leaf_ops.argtypes = [C.c_int, C.c_double, C.c_double] + [dp] * 8
    for p, side, a in [(16, 2.0 / 256, 1.0), (12, 0.25, 2.5), (8, 2.0, -0.7)]:
        n1, q = p - 2, p - 2
        A, V, Vi = (np.zeros((n1, n1)) for _ in range(3))
        lam = np.zeros(n1)
        G, d = np.zeros((q, n1)), np.zeros((4, n1))
        ds = C.c_double()
        Qi = np.zeros((n1 * n1, 4 * q))
        assert L.hpsg_fdm_leaf_ops(p, side, a, HP._dp(A), HP._dp(lam), HP._dp(V), HP._dp(Vi), HP._dp(G), HP._dp(d),
                                   C.byref(ds), HP._dp(Qi)) == 0
        Qi = Qi.T                        # (4q, n1^2), interior column r = (i1-1) n1 + (i2-1)
        A, V, Vi = A.T, V.T, Vi.T        # column-major -> (rows, cols)
        scale = np.abs(A).max()
        assert np.abs(V @ np.diag(lam) @ Vi - A).max() < 1e-12 * scale
        assert np.abs(V @ Vi - np.eye(n1)).max() < 1e-12
        assert np.all(np.isreal(lam)) and len(set(lam.round(6))) == n1
        assert abs(ds.value - 2.0 / side) < 1e-15 * ds.value
        # the separable factors reproduce the dense interior Q exactly (one product per entry, same rounding)
        Qs = np.zeros_like(Qi)
        for sd in range(4):
            for i in range(q):
                for i1 in range(n1):
                    for i2 in range(n1):
                        m, k = (i1, i2) if sd in (0, 2) else (i2, i1)
                        Qs[sd * q + i, i1 * n1 + i2] = ds.value * (G[i, m] * d[sd, k])
        assert np.array_equal(Qs, Qi)
    assert L.hpsg_fdm_leaf_ops(3, 1.0, 1.0, *([None] * 8)) != 0
