"""Memory-budgeted execution planner and transfer ledger (SPEC.md planner module).

The reference's `proj/src/planner.cpp` is a 4-line stub; SPEC.md:445-511 specifies it: choose among
no recomputation / subtree recomputation (Algs. 4-5 of the paper) under a device-memory budget, execute
the plan, and account every host<->device transfer in a ledger.  On the B200 the "arena" is the real
device: the footprint of each candidate context comes from the library's own allocation path
(`hpsg_estimate_bytes`, nothing allocated), execution uses the store path (`HpsSolver`) or
`SubtreeRecomputeSolver`, and the ledger records the transfers the run actually makes (coefficient
samples and boundary data in, the solution out -- every intermediate stays in HBM) plus the FLOPs
re-executed by recomputation (the library's counted build FLOPs of each recomputed subtree).

Strategies: "none" (store everything: one context) and "subtree" (largest complete subtrees whose
working set fits next to the top part; budget = inf -> one subtree = the whole tree).  The paper's
leaf recomputation (Alg. 4) exists to stream leaf outputs through a host round trip; with the whole
leaf stage resident it is the subtree strategy at a deeper cut, so "leaf" is refused with that message.
As SPEC.md requires, 3D problems never use recomputation (the paper's 3D path transfers per level).
"""
from __future__ import annotations

import csv
import io
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import hps as H

STRATEGIES = ("none", "subtree")
CSV_FIELDS = ("strategy", "L", "p", "N", "cut_depth", "bytes_in", "bytes_out", "recomputed_flops",
              "wall_seconds", "device_bytes")


class PlanError(ValueError):
    pass


@dataclass
class ExecutionPlan:
    strategy: str
    dim: int
    p: int
    L: int
    cut_depth: int       # depth of the subtree roots; 0 = one context for the whole tree
    n_subtrees: int      # subtrees recomputed during the solve (0 without recomputation)
    budget: float        # device bytes allowed
    est_bytes: dict      # {"whole": ..} or {"top": .., "subtree": .., "peak": ..}

    @property
    def subtree_depth(self):
        """Levels per subtree (the paper's subtree height)."""
        return self.L - self.cut_depth


@dataclass
class TransferLedger:
    events: list = field(default_factory=list)   # (stage, direction, bytes, tag)

    def add(self, stage, direction, nbytes, tag):
        if direction not in ("h2d", "d2h"):
            raise ValueError("direction must be h2d or d2h")
        self.events.append((stage, direction, int(nbytes), tag))

    def total(self, direction):
        return sum(b for _, d, b, _ in self.events if d == direction)


def _estimator(tree, terms, source, nrhs, opts):
    def est(part):
        return H.estimate_bytes(tree, terms, source, part=part, nrhs=nrhs, **opts)
    return est


def make_plan(tree: H.UniformTree, terms, source=None, strategy="subtree", budget=math.inf, nrhs=1,
              estimator=None, **opts) -> ExecutionPlan:
    """SPEC make_plan(tree, strategy, budget).  `estimator(part) -> bytes` defaults to the library's
    footprint of that part (part None = the whole tree)."""
    if strategy == "leaf":
        raise PlanError("leaf recomputation (Alg. 4) is the subtree strategy at a deeper cut on a device that "
                        "holds the whole leaf stage: use strategy='subtree'")
    if strategy not in STRATEGIES:
        raise PlanError(f"unknown strategy {strategy!r} (none | subtree)")
    if not budget > 0:
        raise PlanError("budget must be positive")
    est = estimator or _estimator(tree, terms, source, nrhs, opts)
    nchild = 4 if tree.dim == 2 else 8
    if strategy == "subtree" and tree.dim == 3:
        raise PlanError("3D problems do not use recomputation strategies (the paper's 3D path transfers "
                        "per merge level); use strategy='none'")
    whole = est(None)
    if strategy == "none" or whole <= budget:
        if whole > budget:
            raise PlanError(f"strategy 'none' needs {whole / 1e9:.2f} GB of device memory; budget {budget / 1e9:.2f} GB")
        return ExecutionPlan(strategy, tree.dim, tree.p, tree.L, 0, 0, budget, {"whole": whole})
    # subtree: the largest complete subtrees (smallest cut depth) whose part fits beside the top part
    for ds in range(1, tree.L):
        top = est((0, 0, ds))
        sub = est((ds, 0, tree.L))
        if top + sub <= budget:
            return ExecutionPlan("subtree", tree.dim, tree.p, tree.L, ds, nchild ** ds, budget,
                                 {"top": top, "subtree": sub, "peak": top + sub})
    raise PlanError(f"budget {budget / 1e9:.3f} GB is too small for one subtree of depth 1 next to the top part")


def _field_bytes(f, tree):
    if f is not None and f.kind == H.FIELD_SAMPLED and f.samples is not None:
        return tree.n_leaves * tree.p ** tree.dim * 8
    return 0


def execute(plan: ExecutionPlan, tree: H.UniformTree, terms, source, boundary, literal_sign=False,
            root_implicit_S=False, device=0):
    """SPEC execute(plan, tree, problem) -> (u, ledger).  `boundary(points) -> g` samples the root data;
    u is (n_leaves, p^d) on the host."""
    import torch
    from .recompute import SubtreeRecomputeSolver
    ledger = TransferLedger()
    for t in terms:
        if _field_bytes(t.field, tree):
            ledger.add("create", "h2d", _field_bytes(t.field, tree), "coefficient samples")
    if _field_bytes(source, tree):
        ledger.add("create", "h2d", _field_bytes(source, tree), "source samples")
    t0 = time.perf_counter()
    kw = dict(literal_sign=literal_sign, root_implicit_S=root_implicit_S, device=device)
    recomputed = 0.0
    if plan.cut_depth == 0:
        s = H.HpsSolver(tree, terms, source, **kw)
        s.build()
        g = np.ascontiguousarray(boundary(s.root_boundary_points()), dtype=np.float64)
        ledger.add("solve", "h2d", g.nbytes, "root boundary data")
        u = s.solve(g)
        ledger.add("solve", "d2h", u.nbytes, "solution")
        dev_bytes = s.stats()["device_bytes"]
        s.close()
    else:
        r = SubtreeRecomputeSolver(tree, terms, source, depth=plan.cut_depth, recompute=True, **kw)
        r.build()
        g = np.ascontiguousarray(boundary(r.root_boundary_points()), dtype=np.float64)
        ledger.add("solve", "h2d", g.nbytes, "root boundary data")
        g_dev = torch.from_numpy(g).to(torch.device("cuda", device))
        u_dev = r.solve_device(g_dev)
        u = u_dev[0].cpu().numpy()
        ledger.add("solve", "d2h", u.nbytes, "solution")
        sub_flops = r.work.stats()["build_flops"]
        recomputed = plan.n_subtrees * sub_flops      # every subtree is built a second time in the solve
        dev_bytes = r.top.stats()["device_bytes"] + r.work.stats()["device_bytes"]
        r.close()
    wall = time.perf_counter() - t0
    ledger.meta = {"recomputed_flops": recomputed, "wall_seconds": wall, "device_bytes": dev_bytes}
    return u, ledger


def ledger_report(ledger: TransferLedger, plan: ExecutionPlan | None = None) -> dict:
    """SPEC ledger_report -> {strategy, L, p, N, bytes_in, bytes_out, recomputed_flops, ...}."""
    meta = getattr(ledger, "meta", {})
    rep = {"strategy": plan.strategy if plan else None, "L": plan.L if plan else None, "p": plan.p if plan else None,
           "N": (4 if plan.dim == 2 else 8) ** plan.L * plan.p ** plan.dim if plan else None,
           "cut_depth": plan.cut_depth if plan else None,
           "bytes_in": ledger.total("h2d"), "bytes_out": ledger.total("d2h"),
           "recomputed_flops": float(meta.get("recomputed_flops", 0.0)),
           "wall_seconds": float(meta.get("wall_seconds", 0.0)), "device_bytes": float(meta.get("device_bytes", 0.0)),
           "stages": sorted({e[0] for e in ledger.events})}
    return rep


def report_csv(reports) -> str:
    """CSV rows (strategy, L, p, N, cut_depth, bytes_in, bytes_out, recomputed_flops, wall_seconds,
    device_bytes), the SPEC's external interface."""
    out = io.StringIO()
    w = csv.DictWriter(out, fieldnames=CSV_FIELDS, extrasaction="ignore")
    w.writeheader()
    for r in reports:
        w.writerow(r)
    return out.getvalue()
