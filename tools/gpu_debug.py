import sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2503_17535_b200 as H
from paper_2503_17535_b200 import problems as PR
from tests.oracle_problems import oracle_solver
prob = PR.helmholtz_bumps()
L = 4
tree = H.build_uniform_tree(-1, 1, L, 2, 16)
def run(rebuild=1, stream=False, device=False, implicit=True):
    s = H.HpsSolver(tree, prob.terms, prob.source, literal_sign=False, root_implicit_S=implicit)
    if stream: s.set_stream(torch.cuda.current_stream().cuda_stream)
    for _ in range(rebuild): s.build()
    g = prob.boundary(s.root_boundary_points())
    if device:
        gd = torch.tensor(g, device='cuda'); ud = torch.empty((tree.n_leaves, 256), dtype=torch.float64, device='cuda')
        s.solve_device(gd.data_ptr(), 1, ud.data_ptr()); torch.cuda.synchronize(); u = ud.cpu().numpy()
    else:
        u = s.solve(g)
    return PR.rel_linf(u, prob.exact(s.leaf_points()))
for kw in [dict(), dict(rebuild=2), dict(stream=True), dict(device=True), dict(rebuild=3, stream=True, device=True), dict(implicit=False, rebuild=2)]:
    print(kw, run(**kw), flush=True)
L = 6; tree = H.build_uniform_tree(-1, 1, L, 2, 16)
for kw in [dict(), dict(rebuild=2, stream=True, device=True)]: print(6, kw, run(**kw), flush=True)
# artifact mismatch
prob = PR.poisson2d()
s = H.HpsSolver(H.build_uniform_tree(-1, 1, 3, 2, 16), prob.terms, prob.source); s.build()
o = oracle_solver(prob, 16, 3); o.build()
for nid in [0, 1, 4, 5, 20]:
    got, ref = s.get_node(nid), o.get_node(nid)
    for name, a, b in zip("S gt T h".split(), got, ref):
        if b is not None: print(nid, name, np.abs(a-b).max(), np.abs(b).max())
