import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2503_17535_b200 as H
from paper_2503_17535_b200 import problems as PR
prob = PR.helmholtz_bumps()
tree = H.build_uniform_tree(prob.lo, prob.hi, 8, 2, 16)
s = H.HpsSolver(tree, prob.terms, prob.source, literal_sign=False, root_implicit_S=True)
st = torch.cuda.current_stream(); s.set_stream(st.cuda_stream)
g = prob.boundary(s.root_boundary_points())
gp = torch.tensor(g).pin_memory(); up = torch.empty((tree.n_leaves, 256), dtype=torch.float64).pin_memory()
for it in range(4):
    t0 = time.time(); s.build(); torch.cuda.synchronize(); t1 = time.time()
    H.lib().hpsg_solve(s._h, H.hps._dp(gp.numpy()), 1, H.hps._dp(up.numpy()), None); t2 = time.time()
    print(f"build {1e3*(t1-t0):.1f} ms  solve(host) {1e3*(t2-t1):.1f} ms  stats solve {s.stats()['t_solve_ms']:.2f}", flush=True)
