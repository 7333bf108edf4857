"""Timing distribution of the implicit-root solve (developer tool)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2503_17535_b200 as H
from paper_2503_17535_b200 import problems as PR
prob = PR.helmholtz_bumps()
tree = H.build_uniform_tree(prob.lo, prob.hi, int(sys.argv[1]) if len(sys.argv) > 1 else 8, 2, 16)
s = H.HpsSolver(tree, prob.terms, prob.source, literal_sign=False, root_implicit_S=True)
s.build()
g = torch.tensor(prob.boundary(s.root_boundary_points()), device="cuda")
u = torch.empty((tree.n_leaves, 256), dtype=torch.float64, device="cuda")
ts = []
for it in range(30):
    s.solve_device(g.data_ptr(), 1, u.data_ptr())
    ts.append(s.stats()["t_solve_ms"])
print(" ".join(f"{t:.1f}" for t in ts))
