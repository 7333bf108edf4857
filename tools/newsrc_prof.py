"""Config 3 (ii) developer profile: one 32-source solve_new_source on the L=8 keep_factors build, between
cudaProfilerStart/Stop."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2503_17535_b200 as H
from paper_2503_17535_b200 import problems as PR
prob = PR.helmholtz_bumps()
tree = H.build_uniform_tree(prob.lo, prob.hi, 8, 2, 16)
s = H.HpsSolver(tree, prob.terms, prob.source, literal_sign=False, root_implicit_S=True, keep_factors=True)
s.build()
chunk = 32
pts = torch.tensor(s.leaf_points(), device="cuda")
g = torch.tensor(prob.boundary(s.root_boundary_points()), device="cuda")
F = torch.empty((chunk, tree.n_leaves, 256), dtype=torch.float64, device="cuda")
for i in range(chunk):
    F[i] = torch.sin((1.0 + 0.1 * i) * pts[..., 0] - 0.5 * pts[..., 1] + 0.01 * i)
G = g.reshape(1, -1).repeat(chunk, 1).contiguous()
U = torch.empty_like(F)
for _ in range(2):
    s.solve_new_source_device(F.data_ptr(), G.data_ptr(), chunk, U.data_ptr())
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
s.solve_new_source_device(F.data_ptr(), G.data_ptr(), chunk, U.data_ptr())
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
