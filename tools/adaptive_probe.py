"""Adaptive 3D runs (Table 1 wavefront, SURVEY 8d config 5 Poisson-Boltzmann) on one B200:
mesh (product refine_adaptive), build, solve; sizes, times, device memory, error vs exact."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2503_17535_b200 as H  # noqa: E402
from paper_2503_17535_b200 import problems as PR  # noqa: E402
from paper_2503_17535_b200.hps import FIELD_PB_EPS_GRAD, Field, refine_adaptive  # noqa: E402


def run(prob, tree, label, **kw):
    s = H.HpsSolver(tree, prob.terms, prob.source, literal_sign=False, root_implicit_S=True)
    g = torch.tensor(prob.boundary(s.root_boundary_points()), device="cuda")
    u = torch.empty((tree.n_leaves, tree.p ** 3), dtype=torch.float64, device="cuda")
    s.build()
    s.solve_device(g.data_ptr(), 1, u.data_ptr())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.build()
    s.solve_device(g.data_ptr(), 1, u.data_ptr())
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    st = s.stats()
    out = dict(label=label, n_leaves=tree.n_leaves, N=tree.total_points, top_D=st["top_D_size"],
               build_ms=st["t_build_ms"], leaf_ms=st["t_leaf_ms"], merge_ms=st["t_merge_ms"], solve_ms=st["t_solve_ms"],
               wall_s=wall, device_gb=st["device_bytes"] / 1e9, torch_peak_gb=torch.cuda.max_memory_allocated() / 1e9,
               build_tflops=st["build_flops"] / st["t_build_ms"] / 1e9, **kw)
    if prob.exact is not None:
        out["rel_linf"] = PR.rel_linf(u.cpu().numpy(), prob.exact(s.leaf_points()))
    s.close()
    print(json.dumps(out), flush=True)
    return out


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("all", "wavefront"):
        prob = PR.wavefront3d()
        for L in (3, 4):
            from tests.test_gpu_general import uniform_as_general
            run(prob, uniform_as_general(3, 8, L, 0.0, 1.0), f"wavefront uniform p=8 L={L}")
        for tol in (1e-2, 1e-3, 3e-4, 1e-4, 3e-5):
            t0 = time.perf_counter()
            tree, nu = refine_adaptive(0.0, 1.0, 8, [prob.source], tol=tol, max_depth=6)
            run(prob, tree, f"wavefront adaptive p=8 tol={tol:g}", mesh_s=time.perf_counter() - t0, unresolved=nu)
    if which in ("all", "pb"):
        prob = PR.poisson_boltzmann3d()
        z = prob.source.centers
        c = prob.terms[0].field.c
        fields = [Field(prob.source.kind, (0.0, 1.0, prob.source.c[2]), centers=z), prob.terms[0].field]
        fields += [Field(FIELD_PB_EPS_GRAD, tuple(c) + (float(a),), centers=z) for a in range(3)]
        for p, tol, md in [(8, 1e-2, 5), (8, 3e-3, 5), (6, 1e-3, 5)]:
            t0 = time.perf_counter()
            tree, nu = refine_adaptive(-1.0, 1.0, p, fields, tol=tol, max_depth=md)
            run(prob, tree, f"poisson_boltzmann3d adaptive p={p} tol={tol:g}", mesh_s=time.perf_counter() - t0,
                unresolved=nu)


if __name__ == "__main__":
    main()
