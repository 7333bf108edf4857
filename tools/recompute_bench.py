"""Subtree-recompute timing (developer tool): python tools/recompute_bench.py L depth."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2503_17535_b200 as H
from paper_2503_17535_b200 import problems as PR
from paper_2503_17535_b200.recompute import SubtreeRecomputeSolver
L = int(sys.argv[1]); ds = int(sys.argv[2])
prob = PR.helmholtz_bumps()
tree = H.build_uniform_tree(prob.lo, prob.hi, L, 2, 16)
rs = SubtreeRecomputeSolver(tree, prob.terms, prob.source, depth=ds, literal_sign=False, root_implicit_S=True)
g = torch.tensor(prob.boundary(rs.root_boundary_points()), device="cuda")
u = torch.empty((1, tree.n_leaves, 256), dtype=torch.float64, device="cuda")
rs.build(); rs.solve_device(g, u); torch.cuda.synchronize()
ts = []
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    rs.build(); rs.solve_device(g, u); torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
free, total = torch.cuda.mem_get_info()
pts = H.hps.tree_leaf_points_of(tree) if L <= 8 else None
err = None
if pts is not None:
    err = float(np.abs(u[0].cpu().numpy() - prob.exact(pts)).max() / np.abs(prob.exact(pts)).max())
print(json.dumps({"L": L, "depth": ds, "N": tree.total_points, "s_per_step": min(ts), "dof_per_s": tree.total_points / min(ts),
                  "device_used_gb": (total - free) / 1e9, "rel_linf_vs_exact": err}))
