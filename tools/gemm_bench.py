"""DMMA DGEMM microbenchmark vs cuBLAS (torch float64) at the HPS shapes (developer tool)."""
import sys, json, os
sys.path.insert(0, '.')
import torch
from tests.gpu_util import lib
L = lib()
shapes = [  # (m, n, k, batch, label)
    (7168, 7169, 3584, 4, "d1 Schur [h|T]-=B[x|X]"),
    (3584, 3585, 1792, 16, "d2 Schur"),
    (6912, 7424, 256, 4, "d1 LU trailing k=256"),
    (6912, 256, 256, 1, "root LU trailing (late)"),
    (448, 449, 224, 1024, "d5 Schur"),
    (196, 57, 196, 65536, "leaf HT-like (m=56..196)"),
    (8192, 8192, 8192, 1, "square 8192"),
]
out = []
for m, n, k, b, label in shapes:
    A = torch.randn(b, k, m, dtype=torch.float64, device='cuda')
    B = torch.randn(b, n, k, dtype=torch.float64, device='cuda')
    C = torch.randn(b, n, m, dtype=torch.float64, device='cuda')
    def mine():
        L.hpsg_dev_dgemm(m, n, k, b, -1.0, A.data_ptr(), m, m*k, B.data_ptr(), k, k*n, 1.0, C.data_ptr(), m, m*n, C.data_ptr(), m, m*n)
    At, Bt = A.transpose(1, 2), B.transpose(1, 2)
    Ct = C.transpose(1, 2)
    def cub():
        torch.baddbmm(Ct, At, Bt, beta=1.0, alpha=-1.0, out=Ct)
    res = {"label": label, "m": m, "n": n, "k": k, "batch": b}
    for name, fn in [("dmma", mine), ("cublas", cub)]:
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        e0.record()
        for _ in range(reps): fn()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res[name + "_tflops"] = round(2.0 * m * n * k * b / ms / 1e9, 2)
    print(os.environ.get("HPS_GEMM_CFG", "auto"), label, res["dmma_tflops"], res["cublas_tflops"], flush=True)
