"""Quick GPU sanity: product vs oracle on small problems (developer tool)."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_2503_17535_b200 as H
from paper_2503_17535_b200 import problems as PR
from oracle import oracle as O

def oracle_for(prob, p, L, literal):
    keep = []
    terms = []
    for t in prob.terms:
        f, k = O.make_field(t.field.kind, t.field.c, t.field.centers, t.field.samples); keep += k
        terms.append((t.role, t.axis, t.axis2, f))
    src = None
    if prob.source is not None:
        src, k = O.make_field(prob.source.kind, prob.source.c, prob.source.centers, prob.source.samples); keep += k
    s = O.Solver(prob.dim, p, L, prob.lo, prob.hi, terms, src, literal_sign=literal, keep=keep)
    s.build()
    return s

print(H.lib().hpsg_build_info().decode())
for name, p, L in [("laplace_poly2d", 8, 1), ("poisson2d", 16, 1), ("poisson2d", 16, 3), ("helmholtz_bumps", 16, 2)]:
    prob = PR.CATALOG[name]()
    tree = H.build_uniform_tree(prob.lo, prob.hi, L, prob.dim, p)
    for literal in (True, False):
        s = H.HpsSolver(tree, prob.terms, prob.source, literal_sign=literal)
        t0 = time.time(); s.build(); t1 = time.time()
        rp = s.root_boundary_points(); g = prob.boundary(rp)
        u = s.solve(g)
        o = oracle_for(prob, p, L, literal)
        orp = o.root_points(); uo = o.solve(prob.boundary(orp))
        lp = s.leaf_points()
        err_exact = PR.rel_linf(u, prob.exact(lp)) if prob.exact else None
        print(f"{name} p={p} L={L} literal={literal}: rootpts {np.abs(rp-orp).max():.1e} parity {PR.rel_linf(u, uo):.3e} "
              f"exact {err_exact:.3e} build {1e3*(t1-t0):.1f} ms stats {s.stats()['t_build_ms']:.2f} ms")
        Y, v, T, h = s.get_leaf(1); Yo, vo, To, ho = o.get_leaf(1)
        print("   leaf1 Y", np.abs(Y-Yo).max(), "v", np.abs(v-vo).max(), "T", np.abs(T-To).max()/np.abs(To).max(), "h", np.abs(h-ho).max())
        if L >= 2:
            S, gt, Tn, hn = s.get_node(1); So, gto, Tno, hno = o.get_node(1)
            print("   node1 S", np.abs(S-So).max(), "gt", np.abs(gt-gto).max(), "T", np.abs(Tn-Tno).max()/np.abs(Tno).max())
