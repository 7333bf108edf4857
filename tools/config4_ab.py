"""Config-4 A/B (developer tool): 3D poisson3d_var p=8 L=4 build + solve through one libhps_b200 build; prints the
build times and saves u.  usage: python tools/config4_ab.py LIB OUT.npy"""
import sys, os, json
sys.path.insert(0, '.')
import numpy as np
import paper_2503_17535_b200.hps as hps
hps.LIB_PATH = os.path.abspath(sys.argv[1])
import paper_2503_17535_b200 as H
from paper_2503_17535_b200 import problems as PR
import torch
prob = PR.poisson3d_var()
tree = H.build_uniform_tree(prob.lo, prob.hi, 4, 3, 8)
s = H.HpsSolver(tree, prob.terms, prob.source, literal_sign=False, root_implicit_S=True)
g = torch.tensor(prob.boundary(s.root_boundary_points()), device="cuda")
u = torch.empty((tree.n_leaves, 8 ** 3), dtype=torch.float64, device="cuda")
out = []
for _ in range(2):
    s.build()
    s.solve_device(g.data_ptr(), 1, u.data_ptr())
    torch.cuda.synchronize()
    st = s.stats()
    out.append((round(st["t_build_ms"], 1), [round(x, 1) for x in st["t_level_ms"]]))
np.save(sys.argv[2], u.cpu().numpy())
print(json.dumps({"lib": sys.argv[1], "builds": out,
                  "rel_linf_vs_exact": PR.rel_linf(u.cpu().numpy(), prob.exact(s.leaf_points()))}))
