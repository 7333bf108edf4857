"""ItI scatter2d timing (developer tool): python tools/iti_bench.py L k."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np
import paper_2503_17535_b200 as H
from paper_2503_17535_b200 import problems as PR
L = int(sys.argv[1]) if len(sys.argv) > 1 else 6
k = float(sys.argv[2]) if len(sys.argv) > 2 else 40.0
pr = PR.scatter2d(k=k)
tree = H.build_uniform_tree(-1.0, 1.0, L, 2, 16)
s = H.HpsSolver(tree, pr.terms, pr.source_re, source_imag=pr.source_im, variant="iti", eta=pr.eta, build_root_T=True)
for it in range(3):
    s.build()
    u = s.solve_radiation()
st = s.stats()
print(json.dumps({"L": L, "k": k, "N": tree.total_points, "build_ms": st["t_build_ms"], "leaf_ms": st["t_leaf_ms"],
                  "merge_ms": st["t_merge_ms"], "solve_ms": st["t_solve_ms"], "levels": [round(x, 2) for x in st["t_level_ms"]],
                  "device_gb": st["device_bytes"] / 1e9, "max_abs_u": float(np.abs(u).max())}))
