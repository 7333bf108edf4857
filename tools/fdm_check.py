"""FDM leaf path vs LU leaf path (developer check): leaf artifacts, solution, leaf-stage time."""
import sys, json
sys.path.insert(0, '.')
import numpy as np
import paper_2503_17535_b200 as H
from paper_2503_17535_b200 import problems as PR
L = int(sys.argv[1]) if len(sys.argv) > 1 else 5
prob = PR.helmholtz_bumps()
tree = H.build_uniform_tree(prob.lo, prob.hi, L, 2, 16)
out = {"L": L}
res = {}
for fdm in (True, False):
    s = H.HpsSolver(tree, prob.terms, prob.source, literal_sign=True, root_implicit_S=True, fdm_leaf=fdm)
    s.build(); s.build()
    st = s.stats()
    g = prob.boundary(s.root_boundary_points())
    u = s.solve(g)
    leaves = [s.get_leaf(i) for i in (0, 1, tree.n_leaves // 2 + 3)] if hasattr(s, "get_leaf") else []
    res[fdm] = (u, leaves)
    out["fdm" if fdm else "lu"] = {"leaf_path": st["leaf_path"], "t_leaf_ms": st["t_leaf_ms"], "t_build_ms": st["t_build_ms"],
                                   "min_rcond": st["min_rcond"]}
    s.close()
u1, l1 = res[True]; u0, l0 = res[False]
out["u_rel_diff"] = float(np.abs(u1 - u0).max() / np.abs(u0).max())
for k, (a, b) in enumerate(zip(l1, l0)):
    out[f"leaf{k}_rel"] = [float(np.abs(np.asarray(x) - np.asarray(y)).max() / max(1e-300, np.abs(np.asarray(y)).max())) for x, y in zip(a, b)]
print(json.dumps(out))
