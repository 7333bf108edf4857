"""FDM vs LU leaf path against the oracle restatement at one L (developer check; the headline problem)."""
import sys, json, os
sys.path.insert(0, '.')
import numpy as np
import paper_2503_17535_b200 as H
from paper_2503_17535_b200 import problems as PR
from oracle import oracle as O
from tests.oracle_problems import oracle_solver
L = int(sys.argv[1]) if len(sys.argv) > 1 else 8
k = float(sys.argv[2]) if len(sys.argv) > 2 else 30.0
prob = PR.helmholtz_bumps(k=k)
tree = H.build_uniform_tree(prob.lo, prob.hi, L, 2, 16)
us = {}
for fdm in (True, False):
    s = H.HpsSolver(tree, prob.terms, prob.source, literal_sign=False, root_implicit_S=True, fdm_leaf=fdm)
    s.build()
    us[fdm] = s.solve(prob.boundary(s.root_boundary_points()))
    ex = prob.exact(s.leaf_points())
    s.close()
O.set_threads(os.cpu_count())
o = oracle_solver(prob, 16, L, literal=False, root_implicit=True, parallel=True)
o.build()
uo = o.solve(prob.boundary(o.root_points()))
r = lambda a, b: float(np.abs(a - b).max() / np.abs(b).max())
print(json.dumps({"L": L, "k": k, "fdm_vs_oracle": r(us[True], uo), "lu_vs_oracle": r(us[False], uo),
                  "fdm_vs_lu": r(us[True], us[False]), "oracle_vs_exact": r(uo, ex), "fdm_vs_exact": r(us[True], ex),
                  "lu_vs_exact": r(us[False], ex)}))
