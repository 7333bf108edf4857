"""3D config 4 check (developer tool): poisson3d_var p=8 at L=3 vs the oracle, L=4 vs exact + timing."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np
import paper_2503_17535_b200 as H
from paper_2503_17535_b200 import problems as PR
prob = PR.poisson3d_var()
out = {}
for L in [int(a) for a in sys.argv[1:]] or [3, 4]:
    tree = H.build_uniform_tree(prob.lo, prob.hi, L, 3, 8)
    s = H.HpsSolver(tree, prob.terms, prob.source, literal_sign=False, root_implicit_S=True)
    for it in range(2):
        t0 = time.time(); s.build(); t1 = time.time()
        g = prob.boundary(s.root_boundary_points())
        u = s.solve(g); t2 = time.time()
    st = s.stats()
    ex = prob.exact(s.leaf_points())
    rec = {"L": L, "N": tree.total_points, "build_ms": st["t_build_ms"], "leaf_ms": st["t_leaf_ms"],
           "merge_ms": st["t_merge_ms"], "solve_ms": st["t_solve_ms"], "levels_ms": [round(x, 2) for x in st["t_level_ms"]],
           "top_D": st["top_D_size"], "rel_linf_vs_exact": float(np.abs(u - ex).max() / np.abs(ex).max()),
           "tflops": st["build_flops"] / st["t_build_ms"] / 1e9, "device_gb": st["device_bytes"] / 1e9}
    if L <= 3:
        from tests.oracle_problems import oracle_solver
        o = oracle_solver(prob, 8, L, literal=False, root_implicit=True, parallel=True)
        o.build()
        uo = o.solve(g)
        rec["rel_linf_vs_oracle"] = float(np.abs(u - uo).max() / np.abs(uo).max())
    print(json.dumps(rec), flush=True)
    del s
