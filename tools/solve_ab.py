"""Solve-stage A/B (developer tool): the L=8 headline build + solve through one libhps_b200 build; writes u and
the solve time.  usage: python tools/solve_ab.py LIB OUT.npy"""
import sys, json, ctypes as C
sys.path.insert(0, '.')
import numpy as np
import os
import paper_2503_17535_b200.hps as hps
hps.LIB_PATH = os.path.abspath(sys.argv[1])   # load this build instead of the in-tree one
import paper_2503_17535_b200 as H
from paper_2503_17535_b200 import problems as PR
prob = PR.helmholtz_bumps()
tree = H.build_uniform_tree(prob.lo, prob.hi, 8, 2, 16)
s = H.HpsSolver(tree, prob.terms, prob.source, literal_sign=False, root_implicit_S=True)
builds = []
for _ in range(3):
    s.build()
    st = s.stats()
    builds.append((round(st["t_build_ms"], 2), [round(x, 2) for x in st["t_level_ms"]]))
import torch
g = prob.boundary(s.root_boundary_points())
g_dev = torch.tensor(g, device="cuda")
u_dev = torch.empty((tree.n_leaves, tree.p ** 2), dtype=torch.float64, device="cuda")
ts = []
for _ in range(5):
    s.solve_device(g_dev.data_ptr(), 1, u_dev.data_ptr())
    torch.cuda.synchronize()
    ts.append(s.stats()["t_solve_ms"])
np.save(sys.argv[2], u_dev.cpu().numpy())
if len(sys.argv) > 3:   # one solve between cudaProfilerStart/Stop (ncu --profile-from-start off)
    torch.cuda.cudart().cudaProfilerStart()
    s.solve_device(g_dev.data_ptr(), 1, u_dev.data_ptr())
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
print(json.dumps({"lib": sys.argv[1], "t_solve_ms": ts, "builds": builds[1:]}))
