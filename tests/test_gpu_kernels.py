"""Kernel-level parity of the batched FP64 primitives (DMMA GEMM, cluster-GEPP LU,
stored-factor solves) against a torch fp64 reference, through the C-ABI
device-pointer entry points of include/hps_cuda.h."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tests.gpu_util import lib  # noqa: E402


def colmajor(b, r, c, rng, ld=None):
    ld = ld or r
    x = torch.tensor(rng.standard_normal((b, c, ld)), device="cuda")
    return x  # x[b, j, i] = element (i, j); leading dimension ld


@pytest.mark.parametrize("m,n,k,b,ld_pad", [(7, 5, 3, 2, 0), (64, 64, 16, 1, 0), (100, 57, 196, 3, 1),
                                             (300, 301, 32, 2, 0), (512, 520, 33, 1, 3), (1024, 1024, 64, 2, 0),
                                             (2048, 1536, 96, 1, 0), (1000, 1000, 1000, 1, 2), (56, 57, 196, 300, 0)])
def test_dgemm(m, n, k, b, ld_pad):
    rng = np.random.default_rng(m * 7 + n)
    lda, ldb, ldc = m + ld_pad, k + ld_pad, m + ld_pad
    A, B, Cm = colmajor(b, m, k, rng, lda), colmajor(b, k, n, rng, ldb), colmajor(b, m, n, rng, ldc)
    D = torch.zeros_like(Cm)
    rc = lib().hpsg_dev_dgemm(m, n, k, b, -1.0, A.data_ptr(), lda, lda * k, B.data_ptr(), ldb, ldb * n, 0.5,
                              Cm.data_ptr(), ldc, ldc * n, D.data_ptr(), ldc, ldc * n)
    assert rc == 0
    At = A[:, :, :m].transpose(1, 2)
    Bt = B[:, :, :k].transpose(1, 2)
    ref = -(At @ Bt) + 0.5 * Cm[:, :, :m].transpose(1, 2)
    got = D[:, :, :m].transpose(1, 2)
    assert ((got - ref).abs().max() / ref.abs().max()).item() < 1e-13


def test_dgemm_broadcast_and_inplace():
    rng = np.random.default_rng(1)
    m, n, k, b = 56, 57, 196, 64
    A = colmajor(1, m, k, rng)            # shared operand (stride 0)
    B = colmajor(b, k, n, rng)
    Cm = colmajor(b, m, n, rng)
    ref = (A[0].T @ B.transpose(1, 2)) + Cm.transpose(1, 2)
    rc = lib().hpsg_dev_dgemm(m, n, k, b, 1.0, A.data_ptr(), m, 0, B.data_ptr(), k, k * n, 1.0, Cm.data_ptr(), m,
                              m * n, Cm.data_ptr(), m, m * n)
    assert rc == 0
    assert ((Cm.transpose(1, 2) - ref).abs().max() / ref.abs().max()).item() < 1e-13


@pytest.mark.parametrize("n,m,b", [(5, 2, 3), (56, 113, 7), (112, 225, 5), (196, 57, 9), (224, 449, 3),
                                   (448, 897, 2), (896, 64, 2), (896, 1793, 1), (1792, 33, 1), (3584, 4, 1),
                                   (600, 100, 3), (1000, 7, 2), (2000, 1, 1), (1100, 3, 1)])
def test_getrf_aug(n, m, b):
    rng = np.random.default_rng(n + m)
    A = rng.standard_normal((b, n, n))
    R = rng.standard_normal((b, n, m))
    M = torch.tensor(np.ascontiguousarray(np.concatenate([A, R], axis=2).transpose(0, 2, 1)), device="cuda")
    piv = torch.zeros((b, n), dtype=torch.int32, device="cuda")
    st = torch.zeros((b, 3), dtype=torch.float64, device="cuda")
    assert lib().hpsg_dev_getrf_aug(b, n, m, M.data_ptr(), n, n * (n + m), piv.data_ptr(), st.data_ptr()) == 0
    X = M.cpu().numpy().transpose(0, 2, 1)[:, :, n:]
    Xref = np.linalg.solve(A, R)
    assert np.abs(X - Xref).max() / np.abs(Xref).max() < 1e-10
    s = st.cpu().numpy()
    assert np.all(s[:, 2] == -1) and np.all(s[:, 0] > 0)
    # stored factors reproduce the solve (MergeArtifact::apply_Dinv path)
    R2 = torch.tensor(np.ascontiguousarray(R.transpose(0, 2, 1)), device="cuda")
    assert lib().hpsg_dev_getrs(b, n, m, M.data_ptr(), n, n * (n + m), piv.data_ptr(), R2.data_ptr(), n, n * m) == 0
    X2 = R2.cpu().numpy().transpose(0, 2, 1)
    assert np.abs(X2 - Xref).max() / np.abs(Xref).max() < 1e-10


def test_getrf_partial_pivoting_needed():
    """A matrix with a zero leading diagonal requires row exchanges."""
    n, m = 64, 3
    rng = np.random.default_rng(5)
    A = rng.standard_normal((n, n))
    A[0, 0] = 0.0
    A[:, 0] *= 1e-3
    A[17, 0] = 5.0
    R = rng.standard_normal((n, m))
    M = torch.tensor(np.ascontiguousarray(np.concatenate([A, R], axis=1).T), device="cuda")[None]
    piv = torch.zeros((1, n), dtype=torch.int32, device="cuda")
    st = torch.zeros((1, 3), dtype=torch.float64, device="cuda")
    assert lib().hpsg_dev_getrf_aug(1, n, m, M.data_ptr(), n, n * (n + m), piv.data_ptr(), st.data_ptr()) == 0
    assert piv[0, 0].item() == 17
    X = M[0].cpu().numpy().T[:, n:]
    assert np.abs(X - np.linalg.solve(A, R)).max() < 1e-10


def test_getrf_singular_reports_pivot():
    n, m = 40, 1
    A = np.random.default_rng(2).standard_normal((n, n))
    A[:, 7] = 0.0
    M = torch.tensor(np.ascontiguousarray(np.concatenate([A, np.ones((n, m))], axis=1).T), device="cuda")[None]
    piv = torch.zeros((1, n), dtype=torch.int32, device="cuda")
    st = torch.zeros((1, 3), dtype=torch.float64, device="cuda")
    assert lib().hpsg_dev_getrf_aug(1, n, m, M.data_ptr(), n, n * (n + m), piv.data_ptr(), st.data_ptr()) == 0
    assert st[0, 2].item() == 7


def test_getrf_aug_narrow_panels_large_n():
    """n beyond 16 CTAs x 864 rows: 16-column GEPP panels (2D L=9 / 3D L=4 roots); residual check on device."""
    import torch
    n, m = 14400, 3
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
    R = torch.randn((n, m), dtype=torch.float64, device="cuda", generator=g)
    M = torch.cat([A, R], dim=1).t().contiguous()   # column-major [A | R]
    piv = torch.zeros((1, n), dtype=torch.int32, device="cuda")
    st = torch.zeros((1, 3), dtype=torch.float64, device="cuda")
    assert lib().hpsg_dev_getrf_aug(1, n, m, M.data_ptr(), n, n * (n + m), piv.data_ptr(), st.data_ptr()) == 0
    X = M[n:].t()
    res = (A @ X - R).abs().max() / (A.abs().max() * X.abs().max() * n)
    assert res < 1e-14, float(res)
    assert st[0, 2].item() == -1


def test_gemm_live_timing():
    """hpsg_dev_gemm_timing (the bench's live GEMM roofline): records each launch's CUDA-event time and
    its 2mnk FLOPs while on, nothing while off."""
    import ctypes as C
    L = lib()
    L.hpsg_dev_gemm_timing.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                       C.POINTER(C.c_longlong)]
    rng = np.random.default_rng(5)
    m, n, k, b = 512, 384, 256, 3
    A, B, Cm = colmajor(b, m, k, rng), colmajor(b, k, n, rng), colmajor(b, m, n, rng)
    D = torch.zeros_like(Cm)

    def gemm():
        assert L.hpsg_dev_dgemm(m, n, k, b, 1.0, A.data_ptr(), m, m * k, B.data_ptr(), k, k * n, 0.0,
                                Cm.data_ptr(), m, m * n, D.data_ptr(), m, m * n) == 0

    ms, fl, nl = C.c_double(), C.c_double(), C.c_longlong()
    assert L.hpsg_dev_gemm_timing(1, None, None, None) == 0
    gemm()
    gemm()
    assert L.hpsg_dev_gemm_timing(2, C.byref(ms), C.byref(fl), C.byref(nl)) == 0
    assert nl.value == 2 and fl.value == 2 * 2.0 * m * n * k * b and ms.value > 0.0
    assert L.hpsg_dev_gemm_timing(0, None, None, None) == 0
    gemm()  # not recorded after stop
    assert L.hpsg_dev_gemm_timing(1, None, None, None) == 0
    assert L.hpsg_dev_gemm_timing(2, C.byref(ms), C.byref(fl), C.byref(nl)) == 0
    assert nl.value == 0 and fl.value == 0.0
    assert L.hpsg_dev_gemm_timing(0, None, None, None) == 0
