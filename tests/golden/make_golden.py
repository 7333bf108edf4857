"""Generates tests/golden/*.npz from the REFERENCE build (oracle/_ref/libhps_ref.so: the reference's own
sources + the Eigen-API shim).  Run in the development container, where /root/reference exists:

    python tests/golden/make_golden.py

Each fixture holds the inputs a GPU test hands the product (root boundary data, leaf sources) and the
reference's outputs on them (solution field, leaf boundary data).  tests/test_gpu_ref_parity.py compares
the B200 path against these when the reference library is not present on the GPU box, and against the
live reference build when it is.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from paper_2503_17535_b200 import problems as PR  # noqa: E402
from tests.ref_problems import ref_solver  # noqa: E402
from oracle import ref as R  # noqa: E402

DTN = [("poisson2d", 16, 3, False), ("helmholtz_bumps", 16, 3, True), ("poisson3d_var", 6, 2, True)]


def dtn_case(name, p, L, implicit):
    prob = PR.CATALOG[name]()
    r = ref_solver(prob, p, L, root_implicit=implicit)
    r.build()
    g = prob.boundary(r.root_points())
    u, lg = r.solve(g, want_leaf_g=True)
    return dict(g=g, u=u, leaf_g=lg)


def iti_robin(L=3, p=16):
    r = R.RefSolver(problem="helmholtz_robin2d", p=p, L=L)
    r.build()
    g = r.sample_root_data()
    return dict(g=g, u=r.solve(g))


def scatter(L=3, p=16, k=20.0, seed=7):
    r = R.RefSolver(problem="scatter2d_bumps", p=p, L=L, k=k, seed=seed)
    r.build()
    return dict(u=r.solve_radiation())


def new_source(p=16, L=3):
    prob = PR.helmholtz_bumps()
    r = ref_solver(prob, p, L)
    r.build()
    pts = r.leaf_points()
    f = 2.0 * np.sin(1.5 * pts[..., 0] - 0.7 * pts[..., 1] + 0.2)
    g = prob.boundary(r.root_points()) * 1.1
    return dict(f=f, g=g, u=r.solve_new_source(f, g))


def main():
    for name, p, L, imp in DTN:
        np.savez_compressed(os.path.join(HERE, f"ref_{name}_p{p}_L{L}.npz"), **dtn_case(name, p, L, imp))
    np.savez_compressed(os.path.join(HERE, "ref_helmholtz_robin2d_p16_L3.npz"), **iti_robin())
    np.savez_compressed(os.path.join(HERE, "ref_scatter2d_bumps_k20_p16_L3.npz"), **scatter())
    np.savez_compressed(os.path.join(HERE, "ref_new_source_helmholtz_p16_L3.npz"), **new_source())
    print("written:", sorted(f for f in os.listdir(HERE) if f.endswith(".npz")))


if __name__ == "__main__":
    main()
