"""Single batched augmented LU timing (developer tool): python tools/lu_bench.py n m batch."""
import sys, json
sys.path.insert(0, '.')
import torch
from tests.gpu_util import lib
n, m, b = (int(x) for x in sys.argv[1:4])
L = lib()
g = torch.Generator(device="cuda").manual_seed(1)
M0 = torch.randn((b, n + m, n), dtype=torch.float64, device="cuda", generator=g)
piv = torch.zeros((b, n), dtype=torch.int32, device="cuda")
st = torch.zeros((b, 3), dtype=torch.float64, device="cuda")
M = M0.clone()
L.hpsg_dev_getrf_aug(b, n, m, M.data_ptr(), n, n * (n + m), piv.data_ptr(), st.data_ptr())
ts = []
for _ in range(3):
    M.copy_(M0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    L.hpsg_dev_getrf_aug(b, n, m, M.data_ptr(), n, n * (n + m), piv.data_ptr(), st.data_ptr())
    e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
fl = b * (2 / 3 * n ** 3 + 2 * n * n * m)
print(json.dumps({"n": n, "m": m, "batch": b, "ms": min(ts), "tflops": fl / min(ts) / 1e9}))
