"""A/B timing of leaf-kernel variants: python tools/leaf_ab.py <path-to-libhps_b200.so> [L]
Builds the headline problem (2D Helmholtz p=16) at depth L through the given library and prints the live
leaf-kernel time (CUDA events) of the 3rd build and the solution error; the field is saved for comparison."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2503_17535_b200.hps as HH  # noqa: E402

path = sys.argv[1]
L = int(sys.argv[2]) if len(sys.argv) > 2 else 8
HH.LIB_PATH = os.path.abspath(path)
import paper_2503_17535_b200 as H  # noqa: E402
from paper_2503_17535_b200 import problems as PR  # noqa: E402

prob = PR.helmholtz_bumps()
tree = H.build_uniform_tree(prob.lo, prob.hi, L, 2, 16)
s = H.HpsSolver(tree, prob.terms, prob.source, literal_sign=False, root_implicit_S=True)
ts = []
for _ in range(3):
    s.build()
    ts.append(round(s.stats()["t_leaf_ms"], 2))
g = prob.boundary(s.root_boundary_points())
u = s.solve(g)
err = PR.rel_linf(u, prob.exact(s.leaf_points()))
print(f"{os.path.basename(path)} L={L}: leaf ms {ts}, build ms {s.stats()['t_build_ms']:.1f}, "
      f"rel_linf vs exact {err:.3e}, checksum {float(np.abs(u).sum()):.17g} {float(u[::97].sum()):.17g}", flush=True)
