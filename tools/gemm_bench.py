"""DMMA GEMM (hpsg_dev_dgemm) vs cuBLAS DGEMM on merge-shaped problems (developer tool)."""
import sys, json
sys.path.insert(0, '.')
import torch
from tests.gpu_util import lib
L = lib()
shapes = [(7168, 7169, 256), (7168, 7169, 3584), (3584, 7169, 256), (3584, 3585, 1792), (4096, 4096, 4096),
          (1792, 1793, 256), (896, 897, 448), (448, 449, 224)]
for m, n, k in shapes:
    b = max(1, int(2 * 7168 * 7169 * 3584 / (2 * m * n * k) // 8)) if m < 3584 else 1
    b = min(b, 64)
    A = torch.randn((b, k, m), dtype=torch.float64, device="cuda").transpose(1, 2)
    B = torch.randn((b, n, k), dtype=torch.float64, device="cuda").transpose(1, 2)
    C = torch.randn((b, n, m), dtype=torch.float64, device="cuda").transpose(1, 2)
    D = torch.empty_like(C)
    def ours():
        L.hpsg_dev_dgemm(m, n, k, b, 1.0, A.data_ptr(), m, m * k, B.data_ptr(), k, k * n, 1.0, C.data_ptr(), m, m * n,
                         D.data_ptr(), m, m * n)
    def cub():
        torch.baddbmm(C, A, B, out=D)
    res = {"m": m, "n": n, "k": k, "batch": b}
    for name, f in (("dmma", ours), ("cublas", cub)):
        f(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            f()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        res[name + "_tflops"] = round(2 * m * n * k * b / ms / 1e9, 2)
    print(json.dumps(res))
