for lib in paper_2503_17535_b200/libhps_b200.so build_ab/lib_tol16.so build_ab/lib_tol15.so; do
  python - $lib <<'PY'
import sys, os, json
sys.path.insert(0, '.')
import paper_2503_17535_b200.hps as hps
hps.LIB_PATH = os.path.abspath(sys.argv[1])
import numpy as np
import paper_2503_17535_b200 as H
from paper_2503_17535_b200 import problems as PR
from oracle import oracle as O
from tests.oracle_problems import oracle_solver
prob = PR.helmholtz_bumps()
tree = H.build_uniform_tree(prob.lo, prob.hi, 8, 2, 16)
s = H.HpsSolver(tree, prob.terms, prob.source, literal_sign=False, root_implicit_S=True)
s.build(); s.build()
st = s.stats()
u = s.solve(prob.boundary(s.root_boundary_points()))
np.save("/tmp/u_%s.npy" % os.path.basename(sys.argv[1]), u)
if not os.path.exists("/tmp/u_oracle.npy"):
    O.set_threads(os.cpu_count())
    o = oracle_solver(prob, 16, 8, literal=False, root_implicit=True, parallel=True)
    o.build()
    np.save("/tmp/u_oracle.npy", o.solve(prob.boundary(o.root_points())))
uo = np.load("/tmp/u_oracle.npy")
print(json.dumps({"lib": sys.argv[1], "t_leaf_ms": st["t_leaf_ms"], "exec_gflop": st["leaf_exec_flops"] / 1e9,
                  "vs_oracle": float(np.abs(u - uo).max() / np.abs(uo).max())}))
PY
done
