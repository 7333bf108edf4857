"""Map product problem descriptors (paper_2503_17535_b200.problems) onto the reference build
oracle/_ref (the reference's own sources + the Eigen-API shim).  Test infrastructure only."""
import numpy as np

from oracle import oracle as O
from oracle import ref as R


def _field(f):
    return O.make_field(f.kind, f.c, f.centers, f.samples)


def ref_solver(prob, p, L, root_implicit=False, variant=0, eta=1.0, build_root_T=False, source_imag=None):
    keep, terms = [], []
    for t in prob.terms:
        f, k = _field(t.field)
        keep += k
        terms.append((t.role, t.axis, t.axis2, f))
    src = srci = None
    source = prob.source if variant == 0 else prob.source_re
    if source is not None:
        src, k = _field(source)
        keep += k
    if source_imag is not None:
        srci, k = _field(source_imag)
        keep += k
    return R.RefSolver(prob.dim, p, L, prob.lo, prob.hi, terms, src, source_imag=srci, variant=variant, eta=eta,
                       root_implicit=root_implicit, build_root_T=build_root_T, keep=keep)


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))

