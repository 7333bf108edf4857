"""Developer check of the batched DGEMM / LU primitives against numpy (GPU)."""
import sys, ctypes as C
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2503_17535_b200 as H
L = H.lib()
vp = C.c_void_p
L.hpsg_dev_dgemm.argtypes = [C.c_int]*4 + [C.c_double, vp, C.c_longlong, C.c_longlong, vp, C.c_longlong, C.c_longlong, C.c_double, vp, C.c_longlong, C.c_longlong, vp, C.c_longlong, C.c_longlong]
L.hpsg_dev_getrf_aug.argtypes = [C.c_int]*3 + [vp, C.c_longlong, C.c_longlong, vp, vp]
rng = np.random.default_rng(0)
for (m, n, k, b) in [(7, 5, 3, 2), (64, 64, 16, 1), (100, 57, 196, 3), (300, 301, 32, 2), (512, 520, 33, 1), (1024, 1024, 64, 2)]:
    A = torch.tensor(rng.standard_normal((b, k, m)), device='cuda')  # stored transposed => col-major m x k
    B = torch.tensor(rng.standard_normal((b, n, k)), device='cuda')
    Cm = torch.tensor(rng.standard_normal((b, n, m)), device='cuda')
    D = torch.zeros((b, n, m), dtype=torch.float64, device='cuda')
    rc = L.hpsg_dev_dgemm(m, n, k, b, -1.0, A.data_ptr(), m, m*k, B.data_ptr(), k, k*n, 0.5, Cm.data_ptr(), m, m*n, D.data_ptr(), m, m*n)
    ref = -(A.transpose(1,2) @ B.transpose(1,2)) + 0.5*Cm.transpose(1,2)
    print("gemm", m, n, k, b, rc, (D.transpose(1,2)-ref).abs().max().item() / ref.abs().max().item())
for (n, m, b) in [(5, 2, 3), (56, 113, 7), (196, 57, 5), (224, 449, 3), (448, 100, 2), (896, 64, 2), (1792, 10, 1), (3584, 4, 1)]:
    A = rng.standard_normal((b, n, n)) + 0*np.eye(n)
    R = rng.standard_normal((b, n, m))
    M = np.concatenate([A, R], axis=2)                 # row-major (b, n, n+m)
    Mt = torch.tensor(np.ascontiguousarray(M.transpose(0, 2, 1)), device='cuda')  # col-major
    piv = torch.zeros((b, n), dtype=torch.int32, device='cuda')
    st = torch.zeros((b, 3), dtype=torch.float64, device='cuda')
    rc = L.hpsg_dev_getrf_aug(b, n, m, Mt.data_ptr(), n, n*(n+m), piv.data_ptr(), st.data_ptr())
    X = Mt.cpu().numpy().transpose(0, 2, 1)[:, :, n:]
    Xref = np.linalg.solve(A, R)
    print("getrf", n, m, b, rc, np.abs(X - Xref).max() / np.abs(Xref).max(), st[0].tolist())
