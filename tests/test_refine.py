"""Product adaptive mesher (hpsg_refine_adaptive: refine_adaptive + enforce_level_restriction,
proj/src/mesh.cpp:141-318, host C++ in libhps_b200.so; no GPU needed) against the REFERENCE's own
refine_adaptive (oracle/_ref) and SPEC.md acceptance criterion 6 (level restriction holds exhaustively,
constant fields give single-leaf trees)."""
import numpy as np
import pytest

from paper_2503_17535_b200 import problems as PR
from paper_2503_17535_b200.hps import FIELD_CONST, FIELD_PB_EPS_GRAD, Field, mesh_json, refine_adaptive

R = pytest.importorskip("oracle.ref")


def same_tree(tr, t):
    return (np.array_equal(tr.depth, t["depth"]) and np.array_equal(tr.n_children, t["n_children"])
            and np.array_equal(tr.children, t["children"]) and np.array_equal(tr.lo, t["lo"])
            and np.array_equal(tr.hi, t["hi"]))


@pytest.mark.parametrize("p,tol,max_depth", [(8, 1e-2, 5), (8, 3e-4, 5), (6, 1e-3, 5)])
def test_wavefront_tree_equals_reference(p, tol, max_depth):
    if not R.available():
        pytest.skip("reference build not available")
    prob = PR.wavefront3d()
    tr, nu = refine_adaptive(0.0, 1.0, p, [prob.source], tol=tol, max_depth=max_depth)
    r = R.RefSolver(problem="wavefront3d", p=p, adaptive=True, tol=tol, max_depth=max_depth)
    assert tr.n_nodes == r.n_nodes and same_tree(tr, r.tree())
    assert nu == r.n_unresolved()


def test_poisson_boltzmann_tree_equals_reference():
    """config 5's mesher on the PB refinement fields (rho, eps, grad eps; make_poisson_boltzmann)."""
    if not R.available():
        pytest.skip("reference build not available")
    prob = PR.poisson_boltzmann3d()
    z = prob.source.centers
    c = prob.terms[0].field.c
    fields = [prob.source, prob.terms[0].field] + [Field(FIELD_PB_EPS_GRAD, tuple(c) + (float(a),), centers=z)
                                                    for a in range(3)]
    # the reference's refinement field rho is +rho; the product's source is -rho: same criterion (|.|-based)
    fields[0] = Field(prob.source.kind, (0.0, 1.0, prob.source.c[2]), centers=z)
    tr, _ = refine_adaptive(-1.0, 1.0, 6, fields, tol=1e-2, max_depth=3)
    r = R.RefSolver(problem="poisson_boltzmann3d", p=6, adaptive=True, tol=1e-2, max_depth=3, seed=20260810)
    assert tr.n_nodes == r.n_nodes and same_tree(tr, r.tree())


def max_face_gap(tr):
    """max_face_neighbor_depth_gap (mesh.cpp:403-439): brute force over all face-adjacent leaf pairs."""
    leaves = tr.leaves
    lo, hi, d = tr.lo[leaves], tr.hi[leaves], tr.depth[leaves]
    gap = 0
    for a in range(len(leaves)):
        touch = np.zeros(len(leaves), bool)
        for k in range(3):
            face = (np.isclose(hi[a, k], lo[:, k]) | np.isclose(lo[a, k], hi[:, k]))
            other = np.ones(len(leaves), bool)
            for m in range(3):
                if m != k:
                    other &= (np.minimum(hi[a, m], hi[:, m]) - np.maximum(lo[a, m], lo[:, m])) > 1e-14
            touch |= face & other
        if touch.any():
            gap = max(gap, int(np.abs(d[touch] - d[a]).max()))
    return gap


def test_level_restriction_and_constant_field():
    prob = PR.wavefront3d()
    tr, _ = refine_adaptive(0.0, 1.0, 8, [prob.source], tol=3e-4, max_depth=5)
    assert len(set(tr.depth[tr.leaves])) > 1          # genuinely nonuniform
    assert max_face_gap(tr) <= 1                       # 2:1 restriction (SPEC acceptance 6)
    one, _ = refine_adaptive(0.0, 1.0, 8, [Field(FIELD_CONST, (3.0,))], tol=1e-6, max_depth=5)
    assert one.n_nodes == 1 and one.n_leaves == 1


def test_mesh_json_equals_reference():
    """mesh_to_json (mesh.cpp:435-463) of an adaptive tree and of a 2D uniform tree: the product's text is
    byte-identical to the reference's (nlohmann dump(1))."""
    if not R.available():
        pytest.skip("reference build not available")
    prob = PR.wavefront3d()
    tr, _ = refine_adaptive(0.0, 1.0, 8, [prob.source], tol=1e-2, max_depth=5)
    r = R.RefSolver(problem="wavefront3d", p=8, adaptive=True, tol=1e-2, max_depth=5)
    assert mesh_json(tr) == r.mesh_json()
    from tests.test_gpu_general import uniform_as_general
    r2 = R.RefSolver(problem="poisson2d", p=16, L=2)
    assert mesh_json(uniform_as_general(2, 16, 2, -1.0, 1.0)) == r2.mesh_json()
