"""ItI variant check (developer tool): Helmholtz with a complex plane wave, impedance root data."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2503_17535_b200 as H
k, th = 12.0, 0.7
terms = [H.Term(H.ROLE_LAPLACIAN, H.Field.const(1.0)), H.Term(H.ROLE_ZEROTH, H.Field.const(k * k))]
for p, L in [(8, 1), (12, 2), (16, 3), (16, 4)]:
    tree = H.build_uniform_tree(-1.0, 1.0, L, 2, p)
    s = H.HpsSolver(tree, terms, None, literal_sign=False, variant="iti", eta=k)
    s.build()
    rp = s.root_boundary_points()
    kv = k * np.array([np.cos(th), np.sin(th)])
    u = lambda x: np.exp(1j * (x[..., 0] * kv[0] + x[..., 1] * kv[1]))
    nb = len(rp)
    side = np.repeat(np.arange(4), nb // 4)
    nrm = np.array([[0, -1], [1, 0], [0, 1], [-1, 0]], dtype=float)[side]
    du = 1j * (rp[:, :2] @ kv * 0 + (nrm @ kv)) * u(rp)
    g = du + 1j * k * u(rp)
    uh = s.solve_complex(g)
    ex = u(s.leaf_points())
    print(p, L, "rel Linf", np.abs(uh - ex).max() / np.abs(ex).max(), "build ms", round(s.stats()["t_build_ms"], 2), flush=True)
