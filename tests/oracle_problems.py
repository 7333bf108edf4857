"""Map product problem descriptors (paper_2503_17535_b200.problems) onto the CPU
oracle (test infrastructure only)."""
from oracle import oracle as O


def oracle_solver(prob, p, L, literal=True, root_implicit=False, parallel=False, source_override=None):
    keep, terms = [], []
    for t in prob.terms:
        f, k = O.make_field(t.field.kind, t.field.c, t.field.centers, t.field.samples)
        keep += k
        terms.append((t.role, t.axis, t.axis2, f))
    src = None
    s = source_override if source_override is not None else prob.source
    if s is not None:
        src, k = O.make_field(s.kind, s.c, s.centers, s.samples)
        keep += k
    return O.Solver(prob.dim, p, L, prob.lo, prob.hi, terms, src, literal_sign=literal, root_implicit=root_implicit,
                    parallel=parallel, keep=keep)
