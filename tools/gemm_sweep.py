"""DMMA GEMM tile-config sweep at the HPS shapes (developer tool; HPS_GEMM_CFG per process)."""
import os, subprocess, sys, json
shapes = [(3328, 10497, 256, 4), (896, 7169, 1792, 4), (6912, 6913, 256, 1), (1536, 3841, 256, 16), (448, 449, 224, 256)]
code = r'''
import sys, json, torch
sys.path.insert(0, '.')
from tests.gpu_util import lib
L = lib()
out = []
for m, n, k, b in %r:
    A = torch.randn(b, k, m, dtype=torch.float64, device='cuda'); B = torch.randn(b, n, k, dtype=torch.float64, device='cuda')
    C = torch.randn(b, n, m, dtype=torch.float64, device='cuda')
    f = lambda: L.hpsg_dev_dgemm(m, n, k, b, -1.0, A.data_ptr(), m, m*k, B.data_ptr(), k, k*n, 1.0, C.data_ptr(), m, m*n, C.data_ptr(), m, m*n)
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): f()
    e1.record(); torch.cuda.synchronize()
    out.append(round(2.0*m*n*k*b*5/e0.elapsed_time(e1)/1e9, 1))
print(json.dumps(out))
''' % (shapes,)
for cfg in range(14):
    env = dict(os.environ, HPS_GEMM_CFG=str(cfg))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(cfg, r.stdout.strip() or r.stderr.strip()[-200:], flush=True)
