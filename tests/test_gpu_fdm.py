"""The fast-diagonalisation leaf solve (csrc/leaf_fdm.cu) against the LU leaf kernel and the oracle.

The FDM path replaces the leaf LU (proj/src/local_solve.cpp:111-143) for operators whose second-order part
is one constant Laplacian term (the headline Helmholtz problem): L_ii = K + diag(c), solved by Richardson on the
true operator, preconditioned with the exactly diagonalisable K + cbar I.  Its fixed point is L_ii^-1 R, so the
leaf artifacts equal the LU ones to roundoff (tolerance 1e-12 relative; measured ~5e-15) and the solution meets
the north-star 1e-10 against the oracle.  Leaves that do not converge fall back to the LU kernel.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2503_17535_b200 as H  # noqa: E402
from paper_2503_17535_b200 import problems as PR  # noqa: E402
from tests.oracle_problems import oracle_solver  # noqa: E402

LEAF_PATH_FDM, LEAF_PATH_FDM_FALLBACK, LEAF_PATH_FUSED_LU = 2, 3, 0


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300))


def solver(prob, p, L, fdm=True, literal=True):
    tree = H.build_uniform_tree(prob.lo, prob.hi, L, prob.dim, p)
    s = H.HpsSolver(tree, prob.terms, prob.source, literal_sign=literal, root_implicit_S=True, fdm_leaf=fdm)
    s.build()
    return s


def test_fdm_path_selection():
    """Constant Laplacian + zeroth order -> FDM; variable first-order terms (poisson2d) -> LU kernel."""
    h = solver(PR.helmholtz_bumps(), 16, 4)
    assert h.stats()["leaf_path"] in (LEAF_PATH_FDM, LEAF_PATH_FDM_FALLBACK)
    assert h.stats()["leaf_exec_flops"] > 0
    p = solver(PR.poisson2d(), 16, 3)
    assert p.stats()["leaf_path"] == LEAF_PATH_FUSED_LU
    assert p.stats()["leaf_exec_flops"] == 0
    f = solver(PR.helmholtz_bumps(), 16, 4, fdm=False)
    assert f.stats()["leaf_path"] == LEAF_PATH_FUSED_LU


@pytest.mark.parametrize("p,L", [(16, 4), (16, 5), (12, 4), (8, 5)])
def test_fdm_leaf_artifacts_equal_lu(p, L):
    """[v | Y_i] and [h | T] of FDM leaves equal the LU kernel's to roundoff; the solutions agree."""
    prob = PR.helmholtz_bumps()
    a, b = solver(prob, p, L), solver(prob, p, L, fdm=False)
    assert a.stats()["leaf_path"] in (LEAF_PATH_FDM, LEAF_PATH_FDM_FALLBACK)
    n = a.tree.n_leaves
    for o in (0, 1, n // 3, n - 1):
        for x, y in zip(a.get_leaf(o), b.get_leaf(o)):
            assert rel(x, y) < 1e-12
    g = prob.boundary(a.root_boundary_points())
    assert rel(a.solve(g), b.solve(g)) < 1e-10


@pytest.mark.parametrize("p,L", [(16, 3), (16, 5), (12, 4)])
@pytest.mark.parametrize("literal", [True, False])
def test_fdm_solution_vs_oracle(p, L, literal):
    """North-star parity (1e-10) of the FDM build against the oracle, both sign conventions.  L = 3 at k = 30 has
    leaves whose Richardson contraction is too weak: they fall back to the LU kernel (leaf_path 3)."""
    prob = PR.helmholtz_bumps()
    s = solver(prob, p, L, literal=literal)
    o = oracle_solver(prob, p, L, literal=literal, root_implicit=True, parallel=True)
    o.build()
    g = prob.boundary(s.root_boundary_points())
    assert rel(s.solve(g), o.solve(g)) < 1e-10
    if (p, L) == (16, 3):
        assert s.stats()["leaf_path"] == LEAF_PATH_FDM_FALLBACK


def test_fdm_executed_flops_bounds():
    """Device DMMA count: every column runs its initial solve (2 passes of 16 DMMA.8x8x4 = 8192 FLOP each for
    the precomputed R^ columns, 4 for the source column) plus 1 .. kMaxSteps = 12 Richardson steps of 6 passes,
    and 24 DMMA for its [h | T] contraction."""
    prob = PR.helmholtz_bumps()
    s = solver(prob, 16, 5)   # L = 5: every leaf converges (no LU fallback)
    st = s.stats()
    assert st["leaf_path"] == LEAF_PATH_FDM
    ncol, nl = 57, s.tree.n_leaves
    per_pass = 16 * 512
    lo = nl * ncol * (2 + 6) * per_pass
    hi = nl * ncol * (4 + 6 * 12) * per_pass + nl * ncol * 24 * 512
    assert lo <= st["leaf_exec_flops"] <= hi


def test_fdm_repeated_builds_identical():
    """The leaf-independent right-hand side tables are prepared once per context: a second build is bitwise
    identical to the first."""
    prob = PR.helmholtz_bumps()
    s = solver(prob, 16, 4)
    g = prob.boundary(s.root_boundary_points())
    u0 = s.solve(g)
    s.build()
    assert np.array_equal(s.solve(g), u0)


def test_sampled_constant_laplacian_takes_fdm():
    """A host-sampled Laplacian coefficient that is one value everywhere (a std::function returning a constant,
    the C++ adapter's path) is recognised as that constant: the FDM leaf applies and the build is bitwise the
    built-in constant field's.  A sampled coefficient with one differing sample stays on the LU kernel."""
    prob = PR.helmholtz_bumps()
    tree = H.build_uniform_tree(prob.lo, prob.hi, 4, 2, 16)
    a = H.HpsSolver(tree, prob.terms, prob.source, root_implicit_S=True)
    a.build()
    lap = prob.terms[0].field.c[0]
    smp = np.full((tree.n_leaves, 16 * 16), lap)
    b = H.HpsSolver(tree, [H.Term(H.ROLE_LAPLACIAN, H.Field(H.FIELD_SAMPLED, samples=smp)), prob.terms[1]],
                    prob.source, root_implicit_S=True)
    b.build()
    assert b.stats()["leaf_path"] in (LEAF_PATH_FDM, LEAF_PATH_FDM_FALLBACK)
    g = prob.boundary(a.root_boundary_points())
    assert np.array_equal(a.solve(g), b.solve(g))
    smp2 = smp.copy()
    smp2[3, 7] = np.nextafter(lap, 2 * lap)
    c = H.HpsSolver(tree, [H.Term(H.ROLE_LAPLACIAN, H.Field(H.FIELD_SAMPLED, samples=smp2)), prob.terms[1]],
                    prob.source, root_implicit_S=True)
    c.build()
    assert c.stats()["leaf_path"] == LEAF_PATH_FUSED_LU


LEAF_PATH_ITI_ELIM, LEAF_PATH_ITI_LU_FALLBACK = 4, 5


@pytest.mark.parametrize("L,path", [(6, LEAF_PATH_ITI_ELIM), (3, LEAF_PATH_ITI_LU_FALLBACK)])
def test_iti_block_elimination_equals_lu(L, path):
    """ItI leaves by block elimination of [G; L_int] (fast-diagonalisation interior solve + the reduced
    4p-4 impedance system, local_solve.cpp:145-172) against the real-equivalent LU of the full leaf system:
    the radiation-closed scatter2d solutions agree to 1e-9 (measured 2.5e-10 at L = 6; the ItI parity floor of
    this suite is 5e-9, test_gpu_ref_parity.py, from complex vs real-equivalent pivoting).  At L = 3 (k = 40, leaf side 1/4) the interior
    Richardson iteration does not contract fast enough: the whole leaf stage falls back to the LU."""
    pr = PR.scatter2d(k=40.0)
    tree = H.build_uniform_tree(-1.0, 1.0, L, 2, 16)
    out = []
    for fdm in (True, False):
        s = H.HpsSolver(tree, pr.terms, pr.source_re, source_imag=pr.source_im, variant="iti", eta=pr.eta,
                        build_root_T=True, fdm_leaf=fdm)
        s.build()
        out.append((s.stats()["leaf_path"], s.solve_radiation()))
        s.close()
    assert out[0][0] == path and out[1][0] == 1
    assert rel(out[0][1], out[1][1]) < 1e-9


def test_iti_block_elimination_plane_wave():
    """Exact-solution gate of the eliminated ItI leaves: the impedance plane-wave problem to 1e-10 at p=16 L=4."""
    k, eta = 12.0, 12.0
    terms = [H.Term(H.ROLE_LAPLACIAN, H.Field.const(1.0)), H.Term(H.ROLE_ZEROTH, H.Field.const(k * k))]
    s = H.HpsSolver(H.build_uniform_tree(-1.0, 1.0, 4, 2, 16), terms, None, variant="iti", eta=eta)
    s.build()
    assert s.stats()["leaf_path"] == LEAF_PATH_ITI_ELIM
    from tests.test_gpu_parity import _impedance_data
    rp = s.root_boundary_points()
    kv = k * np.array([np.cos(0.7), np.sin(0.7)])
    u = lambda x: np.exp(1j * (x[..., 0] * kv[0] + x[..., 1] * kv[1]))
    du = lambda x: (1j * kv[0] * u(x), 1j * kv[1] * u(x))
    g = _impedance_data(rp, u, du, eta)
    ex = u(s.leaf_points())
    U = s.solve_complex(g)
    assert np.abs(U - ex).max() / np.abs(ex).max() < 1e-10


@pytest.mark.parametrize("p", [4, 5, 6, 7, 10])
def test_fdm_small_and_odd_orders(p):
    """Every compiled leaf order (the kernel is instantiated for p = 4..16) matches the LU leaf kernel."""
    prob = PR.helmholtz_bumps(k=6.0)
    a, b = solver(prob, p, 4), solver(prob, p, 4, fdm=False)
    assert a.stats()["leaf_path"] in (LEAF_PATH_FDM, LEAF_PATH_FDM_FALLBACK)
    for o in (0, a.tree.n_leaves - 1):
        for x, y in zip(a.get_leaf(o), b.get_leaf(o)):
            assert rel(x, y) < 1e-12
    g = prob.boundary(a.root_boundary_points())
    assert rel(a.solve(g), b.solve(g)) < 1e-10


def test_fdm_negative_laplacian_coefficient():
    """-Delta u + c u = f (a negative constant Laplacian coefficient, positive zeroth-order term): the
    eigendecomposition and the Richardson iteration are sign-agnostic."""
    terms = [H.Term(H.ROLE_LAPLACIAN, H.Field.const(-1.0)), H.Term(H.ROLE_ZEROTH, H.Field.const(4.0))]
    tree = H.build_uniform_tree(-1.0, 1.0, 4, 2, 12)
    out = []
    for fdm in (True, False):
        s = H.HpsSolver(tree, terms, H.Field.const(1.0), literal_sign=False, fdm_leaf=fdm)
        s.build()
        out.append((s.stats()["leaf_path"], s.solve(np.zeros(s.nb_root))))
    assert out[0][0] == LEAF_PATH_FDM
    assert rel(out[0][1], out[1][1]) < 1e-11
