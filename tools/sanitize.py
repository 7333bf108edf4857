"""compute-sanitizer driver (SURVEY §5 race-detection row): one small invocation of every kernel family.

Run as `compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python tools/sanitize.py [part]`.
Parts: leaf (fused leaf kernel + merges + downward pass, 2D p=16 L=3 and 3D p=6 L=2),
       lu (batched LU: single-CTA and 2/4-CTA DSMEM cluster panels, look-ahead, slab TRSM/TRSV),
       gemm (TMA DMMA GEMM + cp.async twin), all (default).
Sizes are small so racecheck finishes in minutes; the results go to profiles/r02_sanitizer_*.txt.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2503_17535_b200 as H  # noqa: E402
from paper_2503_17535_b200 import problems as PR  # noqa: E402
from tests.gpu_util import lib  # noqa: E402


def part_leaf():
    prob = PR.poisson2d()
    tree = H.build_uniform_tree(prob.lo, prob.hi, 3, 2, 16)
    s = H.HpsSolver(tree, prob.terms, prob.source)
    s.build()
    u = s.solve(prob.boundary(s.root_boundary_points()))
    print("leaf 2D: finite", bool(np.isfinite(u).all()))
    prob3 = PR.poisson3d_var() if hasattr(PR, "poisson3d_var") else None
    if prob3 is not None:
        t3 = H.build_uniform_tree(prob3.lo, prob3.hi, 2, 3, 6)
        s3 = H.HpsSolver(t3, prob3.terms, prob3.source)
        s3.build()
        u3 = s3.solve(prob3.boundary(s3.root_boundary_points()))
        print("leaf 3D: finite", bool(np.isfinite(u3).all()))


def part_lu():
    L = lib()
    for n, m, b in [(196, 57, 4), (896, 17, 1), (1792, 5, 1), (600, 1, 1)]:
        rng = np.random.default_rng(n)
        A = rng.standard_normal((b, n, n))
        R = rng.standard_normal((b, n, m))
        M = torch.tensor(np.ascontiguousarray(np.concatenate([A, R], axis=2).transpose(0, 2, 1)), device="cuda")
        piv = torch.zeros((b, n), dtype=torch.int32, device="cuda")
        st = torch.zeros((b, 3), dtype=torch.float64, device="cuda")
        assert L.hpsg_dev_getrf_aug(b, n, m, M.data_ptr(), n, n * (n + m), piv.data_ptr(), st.data_ptr()) == 0
        X = M.cpu().numpy().transpose(0, 2, 1)[:, :, n:]
        err = np.abs(X - np.linalg.solve(A, R)).max()
        R2 = torch.tensor(np.ascontiguousarray(R.transpose(0, 2, 1)), device="cuda")
        assert L.hpsg_dev_getrs(b, n, m, M.data_ptr(), n, n * (n + m), piv.data_ptr(), R2.data_ptr(), n, n * m) == 0
        print(f"lu n={n} m={m} b={b}: err {err:.1e}")


def part_gemm():
    L = lib()
    for m, n, k, b in [(256, 192, 96, 2), (56, 57, 196, 8)]:
        A = torch.randn((b, k, m), dtype=torch.float64, device="cuda")
        B = torch.randn((b, n, k), dtype=torch.float64, device="cuda")
        Cm = torch.randn((b, n, m), dtype=torch.float64, device="cuda")
        D = torch.zeros_like(Cm)
        assert L.hpsg_dev_dgemm(m, n, k, b, 1.0, A.data_ptr(), m, m * k, B.data_ptr(), k, k * n, 1.0,
                                Cm.data_ptr(), m, m * n, D.data_ptr(), m, m * n) == 0
        ref = A.transpose(1, 2) @ B.transpose(1, 2) + Cm.transpose(1, 2)
        print(f"gemm {m}x{n}x{k} b={b}: err {(D.transpose(1, 2) - ref).abs().max().item():.1e}")


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    for name, fn in [("leaf", part_leaf), ("lu", part_lu), ("gemm", part_gemm)]:
        if which in ("all", name):
            fn()
    torch.cuda.synchronize()
    print("sanitize: done")
