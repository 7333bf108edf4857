"""ItI problems (developer tool): helmholtz_robin2d accuracy gate, scatter2d radiation closure."""
import sys, ctypes as C
sys.path.insert(0, '.')
import numpy as np
import paper_2503_17535_b200 as H
from paper_2503_17535_b200 import problems as PR
from paper_2503_17535_b200 import hps as HP
for L in (3, 4):
    tree = H.build_uniform_tree(-1.0, 1.0, L, 2, 16)
    pr = PR.helmholtz_robin2d(tree)
    s = H.HpsSolver(tree, pr.terms, pr.source_re, source_imag=pr.source_im, variant="iti", eta=pr.eta)
    s.build()
    u = s.solve_complex(pr.impedance(s.root_boundary_points()))
    ex = pr.exact(s.leaf_points())
    print("robin2d L", L, "rel Linf", np.abs(u - ex).max() / np.abs(ex).max(), flush=True)
pr = PR.scatter2d(k=20.0)
for L in (3, 4):
    tree = H.build_uniform_tree(-1.0, 1.0, L, 2, 16)
    s = H.HpsSolver(tree, pr.terms, pr.source_re, source_imag=pr.source_im, variant="iti", eta=pr.eta, build_root_T=True)
    s.build()
    u, g = s.solve_radiation(want_g=True)
    # outgoing impedance du/dn - i eta u of every boundary leaf face on the root boundary must vanish
    p, q = 16, 14
    QHr, QHi = np.zeros((p * p, 4 * q)), np.zeros((p * p, 4 * q))
    L_ = H.lib()
    L_.hpsg_iti_leaf_ops.argtypes = [C.c_int, C.c_double, C.c_double] + [C.POINTER(C.c_double)] * 5
    side = 2.0 / 2 ** L
    L_.hpsg_iti_leaf_ops(p, pr.eta, side, None, None, None, HP._dp(QHr), HP._dp(QHi))
    QH = (QHr + 1j * QHi).T
    lp = s.leaf_points()
    worst, scale = 0.0, np.abs(g).max()
    for l in range(tree.n_leaves):
        out = QH @ u[l]
        lo, hi = lp[l, :, 0].min(), lp[l, :, 0].max()
        blo, bhi = lp[l, :, 1].min(), lp[l, :, 1].max()
        for sd, on in ((0, blo < -1 + 1e-12), (1, hi > 1 - 1e-12), (2, bhi > 1 - 1e-12), (3, lo < -1 + 1e-12)):
            if on:
                worst = max(worst, np.abs(out[sd * q:(sd + 1) * q]).max())
    print("scatter2d L", L, "max |outgoing impedance| / max |g|", worst / scale, "max|u|", np.abs(u).max(), flush=True)
