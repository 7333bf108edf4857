for lib in paper_2503_17535_b200/libhps_b200.so build_ab/lib_w3.so build_ab/lib_w4.so; do
  timeout 300 python - $lib <<'PY'
import sys, os, json
sys.path.insert(0, '.')
import paper_2503_17535_b200.hps as hps
hps.LIB_PATH = os.path.abspath(sys.argv[1])
import numpy as np
import paper_2503_17535_b200 as H
from paper_2503_17535_b200 import problems as PR
prob = PR.helmholtz_bumps()
tree = H.build_uniform_tree(prob.lo, prob.hi, 8, 2, 16)
s = H.HpsSolver(tree, prob.terms, prob.source, literal_sign=False, root_implicit_S=True)
t = []
for _ in range(3):
    s.build(); t.append(s.stats()["t_leaf_ms"])
u = s.solve(prob.boundary(s.root_boundary_points()))
np.save("/tmp/u_%s.npy" % os.path.basename(sys.argv[1]), u)
a = np.load("/tmp/u_libhps_b200.so.npy")
print(json.dumps({"lib": sys.argv[1], "t_leaf_ms": t, "path": s.stats()["leaf_path"], "bitwise_vs_default": bool(np.array_equal(a, u))}))
PY
done
