"""Config 3 (i) developer profile: one 64-RHS boundary solve on the L=8 build between cudaProfilerStart/Stop."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2503_17535_b200 as H
from paper_2503_17535_b200 import problems as PR
prob = PR.helmholtz_bumps()
tree = H.build_uniform_tree(prob.lo, prob.hi, 8, 2, 16)
s = H.HpsSolver(tree, prob.terms, prob.source, literal_sign=False, root_implicit_S=True)
s.build()
nrhs = int(sys.argv[1]) if len(sys.argv) > 1 else 64
G = torch.randn((nrhs, s.nb_root), dtype=torch.float64, device="cuda")
U = torch.empty((nrhs, tree.n_leaves, 256), dtype=torch.float64, device="cuda")
for _ in range(2):
    s.solve_device(G.data_ptr(), nrhs, U.data_ptr())
torch.cuda.synchronize()
print("t_solve_ms", s.stats()["t_solve_ms"])
torch.cuda.cudart().cudaProfilerStart()
s.solve_device(G.data_ptr(), nrhs, U.data_ptr())
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
