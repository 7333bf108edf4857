"""Memory-budgeted planner + transfer ledger (paper_2503_17535_b200/planner.py).

CPU: plan selection against an injected footprint model, ledger accounting, report/CSV shape.
GPU: the library footprint estimate equals what a context really allocates; SPEC's cross-strategy
equivalence example (none vs subtree on 2D L=4 p=8 within 1e-13); ledger totals and recomputed FLOPs.
"""
import math

import numpy as np
import pytest

from paper_2503_17535_b200 import hps as H
from paper_2503_17535_b200 import planner as PL


def model(tree):
    """Footprint stand-in: a part's bytes grow with its leaf count and its top-level interface."""
    nchild = 4 if tree.dim == 2 else 8

    def est(part):
        rd, _, cd = part if part is not None else (0, 0, tree.L)
        leaves = nchild ** (tree.L - rd) if cd == tree.L else nchild ** (cd - rd)
        return 1000.0 * leaves + 10.0 * 2 ** (tree.L - rd)
    return est


def test_plan_infinite_budget_is_one_subtree():
    tree = H.build_uniform_tree(-1, 1, 5, 2, 8)
    for strategy in ("none", "subtree"):
        p = PL.make_plan(tree, [], strategy=strategy, budget=math.inf, estimator=model(tree))
        assert p.cut_depth == 0 and p.n_subtrees == 0 and p.subtree_depth == tree.L


def test_plan_picks_largest_fitting_subtree():
    tree = H.build_uniform_tree(-1, 1, 5, 2, 8)
    est = model(tree)
    whole = est(None)
    for ds in range(1, tree.L):
        need = est((0, 0, ds)) + est((ds, 0, tree.L))
        p = PL.make_plan(tree, [], strategy="subtree", budget=need, estimator=est)
        # the smallest cut depth (largest subtrees) that fits; a looser budget never cuts deeper
        assert p.cut_depth <= ds and p.est_bytes["peak"] <= need
        assert p.n_subtrees == 4 ** p.cut_depth
    assert PL.make_plan(tree, [], strategy="subtree", budget=whole, estimator=est).cut_depth == 0
    with pytest.raises(PL.PlanError):
        PL.make_plan(tree, [], strategy="subtree", budget=10.0, estimator=est)
    with pytest.raises(PL.PlanError):
        PL.make_plan(tree, [], strategy="none", budget=whole / 2, estimator=est)


def test_plan_rejections():
    t2 = H.build_uniform_tree(-1, 1, 3, 2, 8)
    t3 = H.build_uniform_tree(0, 1, 2, 3, 6)
    with pytest.raises(PL.PlanError, match="3D"):
        PL.make_plan(t3, [], strategy="subtree", budget=1.0, estimator=model(t3))
    with pytest.raises(PL.PlanError, match="subtree"):
        PL.make_plan(t2, [], strategy="leaf", budget=1.0, estimator=model(t2))
    with pytest.raises(PL.PlanError):
        PL.make_plan(t2, [], strategy="bogus", estimator=model(t2))
    with pytest.raises(PL.PlanError):
        PL.make_plan(t2, [], strategy="none", budget=0.0, estimator=model(t2))


def test_ledger_and_report():
    led = PL.TransferLedger()
    assert PL.ledger_report(led)["bytes_in"] == 0 and PL.ledger_report(led)["bytes_out"] == 0
    led.add("create", "h2d", 800, "coefficient samples")
    led.add("solve", "h2d", 64, "root boundary data")
    led.add("solve", "d2h", 4096, "solution")
    with pytest.raises(ValueError):
        led.add("solve", "sideways", 1, "x")
    tree = H.build_uniform_tree(-1, 1, 4, 2, 8)
    plan = PL.make_plan(tree, [], strategy="none", estimator=model(tree))
    rep = PL.ledger_report(led, plan)
    assert rep["bytes_in"] == 864 and rep["bytes_out"] == 4096 and rep["stages"] == ["create", "solve"]
    assert rep["N"] == tree.total_points and rep["recomputed_flops"] == 0.0
    text = PL.report_csv([rep])
    assert text.splitlines()[0] == ",".join(PL.CSV_FIELDS) and text.splitlines()[1].startswith("none,4,8,")


@pytest.mark.gpu
def test_estimate_matches_allocation():
    from paper_2503_17535_b200 import problems as PR
    prob = PR.CATALOG["helmholtz_bumps"]()
    tree = H.build_uniform_tree(prob.lo, prob.hi, 4, 2, 16)
    for part in (None, (0, 0, 2), (2, 5, 4)):
        est = H.estimate_bytes(tree, prob.terms, prob.source, part=part, nrhs=1, literal_sign=False)
        s = H.HpsSolver(tree, prob.terms, prob.source, literal_sign=False, part=part)
        if s.n_cut:
            s.close()
            continue  # a cut part cannot be solved without its inputs; compare the build footprint
        s.build()
        s.solve(np.zeros(s.nb_root))
        assert s.stats()["device_bytes"] == est
        s.close()
    b0 = H.estimate_bytes(tree, prob.terms, prob.source, part=(0, 0, 2), nrhs=0)
    s = H.HpsSolver(tree, prob.terms, prob.source, part=(0, 0, 2))
    assert s.stats()["device_bytes"] == b0
    s.close()


@pytest.mark.gpu
def test_none_vs_subtree_equivalence():
    """SPEC.md planner example: strategy none vs subtree on L=4, p=8 2D -> identical within 1e-13."""
    from paper_2503_17535_b200 import problems as PR
    prob = PR.CATALOG["helmholtz_bumps"]()
    tree = H.build_uniform_tree(prob.lo, prob.hi, 4, 2, 8)
    p_none = PL.make_plan(tree, prob.terms, prob.source, strategy="none")
    # at this size the per-context fixed workspaces outweigh the saving, so the depth-2 plan is built
    # directly (the budget search itself is exercised at L=6 below)
    p_sub = PL.ExecutionPlan("subtree", 2, 8, 4, 2, 16, math.inf, {})
    u0, l0 = PL.execute(p_none, tree, prob.terms, prob.source, prob.boundary)
    u1, l1 = PL.execute(p_sub, tree, prob.terms, prob.source, prob.boundary)
    assert np.abs(u1 - u0).max() <= 1e-13 * np.abs(u0).max()
    r0, r1 = PL.ledger_report(l0, p_none), PL.ledger_report(l1, p_sub)
    assert r0["bytes_in"] == r1["bytes_in"] == 8 * 4 * 6 * 2 ** 4  # root boundary data only (device fields)
    assert r0["bytes_out"] == r1["bytes_out"] == tree.total_points * 8
    assert r0["recomputed_flops"] == 0.0 and r1["recomputed_flops"] > 0.0


@pytest.mark.gpu
def test_plan_budget_search_real_footprints():
    """L=6 p=16: the subtree plan under a budget below the store footprint cuts at the shallowest depth
    whose top part + one subtree part fit, and its peak really is below the whole-tree footprint."""
    from paper_2503_17535_b200 import problems as PR
    prob = PR.CATALOG["helmholtz_bumps"]()
    tree = H.build_uniform_tree(prob.lo, prob.hi, 6, 2, 16)
    whole = PL.make_plan(tree, prob.terms, prob.source, strategy="none").est_bytes["whole"]
    p = PL.make_plan(tree, prob.terms, prob.source, strategy="subtree", budget=0.5 * whole)
    assert p.cut_depth >= 1 and p.est_bytes["peak"] <= 0.5 * whole
    if p.cut_depth > 1:  # every shallower cut would not have fit
        d = p.cut_depth - 1
        need = (H.estimate_bytes(tree, prob.terms, prob.source, part=(0, 0, d)) +
                H.estimate_bytes(tree, prob.terms, prob.source, part=(d, 0, tree.L)))
        assert need > 0.5 * whole
