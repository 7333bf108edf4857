// lu.cu -- batched blocked LU with partial pivoting (see lu.cuh).
#include <algorithm>
#include <cfloat>
#include <climits>

#include "gemm.cuh"
#include "lu.cuh"

namespace hpsk {

namespace {

constexpr int kPanelThreads = 256;
constexpr int kRowsPerCta = 448;  // 448 x 32 doubles = 112 KiB of panel per CTA
constexpr int kMaxCluster = 16;   // non-portable cluster size (same GPC)
constexpr int kMaxRowsPerCta = 864;

struct PanelArgs {
  double* M;
  long long ld, stride;
  int n, j0, nb, rpc, cs;
  int* ipiv;
  double* stats;
};

HPS_DEV void argmax_merge(double& v, int& i, double v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}

// One panel (rows j0..n-1, columns j0..j0+nb-1) of one matrix per cluster.
__global__ void __launch_bounds__(kPanelThreads) panel_getrf_kernel(const PanelArgs a) {
  extern __shared__ __align__(16) double sm[];
  double* pan = sm;                          // [nb][rpc]
  double* urow = sm + (size_t)a.rpc * kLuNB; // pivot row (all nb cols)
  double* jrow = urow + kLuNB;               // displaced row j
  double* wv = jrow + kLuNB;                 // per-warp partial max
  int* wi = reinterpret_cast<int*>(wv + kPanelThreads / 32);
  double* cand_v = reinterpret_cast<double*>(wi + kPanelThreads / 32 + 2);  // 8-byte aligned slot
  int* cand_i = reinterpret_cast<int*>(cand_v + 1);
  int* s_piv = cand_i + 1;

  const int cs = a.cs;
  const int rank = cs > 1 ? (int)cluster_ctarank() : 0;
  const long long b = blockIdx.x / cs;
  double* M = a.M + b * a.stride;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rows_total = a.n - a.j0;
  const int r_begin = rank * a.rpc;
  const int nr = max(0, min(rows_total - r_begin, a.rpc));
  const int nb = a.nb;

  for (int e = tid; e < nr * nb; e += kPanelThreads) {
    const int r = e % nr, c = e / nr;
    pan[c * a.rpc + r] = M[(long long)(a.j0 + c) * a.ld + a.j0 + r_begin + r];
  }
  __syncthreads();

  double pmin = DBL_MAX, pmax = 0.0;
  int first_zero = -1;

  for (int j = 0; j < nb; ++j) {
    // ---- local argmax over panel rows >= j
    double bv = -1.0;
    int bi = INT_MAX;
    for (int r = tid; r < nr; r += kPanelThreads) {
      const int gr = r_begin + r;
      if (gr >= j) argmax_merge(bv, bi, fabs(pan[j * a.rpc + r]), gr);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      argmax_merge(bv, bi, v2, i2);
    }
    if (lane == 0) wv[warp] = bv, wi[warp] = bi;
    __syncthreads();
    if (warp == 0) {
      bv = lane < kPanelThreads / 32 ? wv[lane] : -1.0;
      bi = lane < kPanelThreads / 32 ? wi[lane] : INT_MAX;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
        argmax_merge(bv, bi, v2, i2);
      }
      if (lane == 0) *cand_v = bv, *cand_i = bi;
    }
    if (cs > 1) {
      cluster_sync();
      if (warp == 0) {
        bv = -1.0;
        bi = INT_MAX;
        if (lane < cs) {
          bv = dsmem_ld_f64(dsmem_map(cand_v, lane));
          bi = dsmem_ld_s32(dsmem_map(cand_i, lane));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
          const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
          argmax_merge(bv, bi, v2, i2);
        }
        if (lane == 0) *s_piv = (bi == INT_MAX) ? j : bi;
      }
    } else {
      if (tid == 0) *s_piv = (*cand_i == INT_MAX) ? j : *cand_i;
    }
    __syncthreads();
    const int piv = *s_piv;
    const int own_p = piv / a.rpc, own_j = j / a.rpc;

    // ---- fetch pivot row (and displaced row j for the pivot owner)
    for (int c = tid; c < nb; c += kPanelThreads) {
      const double* src = &pan[c * a.rpc + (piv - own_p * a.rpc)];
      urow[c] = (own_p == rank) ? *src : dsmem_ld_f64(dsmem_map(src, own_p));
      if (own_p == rank && piv != j) {
        const double* sj = &pan[c * a.rpc + (j - own_j * a.rpc)];
        jrow[c] = (own_j == rank) ? *sj : dsmem_ld_f64(dsmem_map(sj, own_j));
      }
    }
    if (cs > 1)
      cluster_sync();
    else
      __syncthreads();
    if (piv != j) {
      for (int c = tid; c < nb; c += kPanelThreads) {
        if (own_j == rank) pan[c * a.rpc + (j - r_begin)] = urow[c];
        if (own_p == rank) pan[c * a.rpc + (piv - r_begin)] = jrow[c];
      }
    }
    __syncthreads();

    const double pv = urow[j];
    const double apv = fabs(pv);
    if (!(apv > 0.0) || !isfinite(apv)) {
      if (first_zero < 0) first_zero = a.j0 + j;
    } else {
      pmin = fmin(pmin, apv);
      pmax = fmax(pmax, apv);
    }
    if (rank == 0 && tid == 0) a.ipiv[b * a.n + a.j0 + j] = a.j0 + piv;

    // ---- eliminate rows below j within this CTA's chunk
    if (apv > 0.0) {
      const double inv = 1.0 / pv;
      for (int r = tid; r < nr; r += kPanelThreads) {
        const int gr = r_begin + r;
        if (gr <= j) continue;
        const double l = pan[j * a.rpc + r] * inv;
        pan[j * a.rpc + r] = l;
        for (int c = j + 1; c < nb; ++c) pan[c * a.rpc + r] -= l * urow[c];
      }
    }
    __syncthreads();
  }

  for (int e = tid; e < nr * nb; e += kPanelThreads) {
    const int r = e % nr, c = e / nr;
    M[(long long)(a.j0 + c) * a.ld + a.j0 + r_begin + r] = pan[c * a.rpc + r];
  }
  if (rank == 0 && tid == 0 && a.stats) {
    double* s = a.stats + 3 * b;
    s[0] = fmin(s[0], pmin);
    s[1] = fmax(s[1], pmax);
    if (first_zero >= 0 && s[2] < 0) s[2] = first_zero;
  }
  if (cs > 1) cluster_sync();  // keep smem alive until remote readers are done
}

struct Seg {
  double* base;  // column 0 of the segment for matrix 0 (row index = matrix row)
  long long ld, stride;
  int ncols;
  int trsm;      // 1: apply L11^-1 to rows j0..j0+nb-1 after the swaps
};
struct SwapTrsmArgs {
  const double* L;  // matrix 0 of the factored matrices (for L11)
  long long ldL, strideL;
  const int* ipiv;
  int n, j0, nb;
  int nseg;
  int do_swaps;  // 0 when the rows were already permuted (bgetrs)
  Seg seg[3];
};

constexpr int kColThreads = 128;

// Row swaps of one panel applied to column segments, then U12 = L11^-1 A12
// (proj/src/local_solve.cpp:128 / merge.cpp:291: the forward half of the solve).
__global__ void __launch_bounds__(kColThreads) swap_trsm_kernel(const SwapTrsmArgs a) {
  __shared__ double L11[kLuNB][kLuNB + 1];
  __shared__ int piv[kLuNB];
  const long long b = blockIdx.x;
  const double* L = a.L + b * a.strideL;
  const int nb = a.nb;
  for (int e = threadIdx.x; e < nb * nb; e += kColThreads) {
    const int r = e % nb, c = e / nb;
    L11[r][c] = L[(long long)(a.j0 + c) * a.ldL + a.j0 + r];
  }
  for (int e = threadIdx.x; e < nb; e += kColThreads) piv[e] = a.ipiv[b * a.n + a.j0 + e];
  __syncthreads();

  int col = blockIdx.y * kColThreads + threadIdx.x;
  int s = 0;
  while (s < a.nseg && col >= a.seg[s].ncols) col -= a.seg[s++].ncols;
  if (s >= a.nseg) return;
  const Seg sg = a.seg[s];
  double* x = sg.base + b * sg.stride + (long long)col * sg.ld;
  for (int jj = 0; jj < (a.do_swaps ? nb : 0); ++jj) {
    const int r1 = a.j0 + jj, r2 = piv[jj];
    if (r2 != r1) {
      const double t = x[r1];
      x[r1] = x[r2];
      x[r2] = t;
    }
  }
  if (!sg.trsm) return;
  double v[kLuNB];
#pragma unroll
  for (int jj = 0; jj < kLuNB; ++jj) v[jj] = jj < nb ? x[a.j0 + jj] : 0.0;
#pragma unroll
  for (int jj = 1; jj < kLuNB; ++jj) {
    double acc = v[jj];
#pragma unroll
    for (int ii = 0; ii < jj; ++ii) acc -= L11[jj][ii] * v[ii];
    v[jj] = acc;
  }
#pragma unroll
  for (int jj = 0; jj < kLuNB; ++jj)
    if (jj < nb) x[a.j0 + jj] = v[jj];
}

struct TrsmUArgs {
  const double* U;
  long long ldU, strideU;
  int r0, nb;
  double* R;
  long long ldR, strideR;
  int ncols;
};

// X_blk = U_blk^-1 R_blk for one diagonal block of U (back substitution).
__global__ void __launch_bounds__(kColThreads) trsm_upper_kernel(const TrsmUArgs a) {
  __shared__ double U11[kLuNB][kLuNB + 1];
  const long long b = blockIdx.x;
  const double* U = a.U + b * a.strideU;
  const int nb = a.nb;
  for (int e = threadIdx.x; e < nb * nb; e += kColThreads) {
    const int r = e % nb, c = e / nb;
    U11[r][c] = U[(long long)(a.r0 + c) * a.ldU + a.r0 + r];
  }
  __syncthreads();
  const int col = blockIdx.y * kColThreads + threadIdx.x;
  if (col >= a.ncols) return;
  double* x = a.R + b * a.strideR + (long long)col * a.ldR + a.r0;
  double v[kLuNB];
#pragma unroll
  for (int jj = 0; jj < kLuNB; ++jj) v[jj] = jj < nb ? x[jj] : 0.0;
#pragma unroll
  for (int jj = kLuNB - 1; jj >= 0; --jj) {
    if (jj < nb) {
      double acc = v[jj];
#pragma unroll
      for (int ii = jj + 1; ii < kLuNB; ++ii)
        if (ii < nb) acc -= U11[jj][ii] * v[ii];
      v[jj] = acc / U11[jj][jj];
    }
  }
#pragma unroll
  for (int jj = 0; jj < kLuNB; ++jj)
    if (jj < nb) x[jj] = v[jj];
}

// Apply the complete pivot sequence of a factorization to R (LAPACK laswp), via the
// composite permutation built in shared memory: R[i, :] <- R[perm[i], :].
__global__ void laswp_perm_kernel(const int* ipiv, int n, double* R, long long ldR, long long strideR, int ncols,
                                  int cols_per_cta) {
  extern __shared__ __align__(16) double sbuf[];
  int* perm = reinterpret_cast<int*>(sbuf + n);
  const long long b = blockIdx.x;
  const int* pv = ipiv + b * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) perm[i] = i;
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 0; i < n; ++i) {
      const int j = pv[i];
      if (j != i) {
        const int t = perm[i];
        perm[i] = perm[j];
        perm[j] = t;
      }
    }
  __syncthreads();
  const int c0 = blockIdx.y * cols_per_cta, c1 = min(ncols, c0 + cols_per_cta);
  for (int c = c0; c < c1; ++c) {
    double* x = R + b * strideR + (long long)c * ldR;
    for (int i = threadIdx.x; i < n; i += blockDim.x) sbuf[i] = x[perm[i]];
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = sbuf[i];
    __syncthreads();
  }
}

__global__ void stats_init_kernel(double* s, int batch) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < batch) {
    s[3 * i + 0] = DBL_MAX;
    s[3 * i + 1] = 0.0;
    s[3 * i + 2] = -1.0;
  }
}

int cluster_for(int n) {
  int cs = (n + kRowsPerCta - 1) / kRowsPerCta;
  return std::max(1, cs);
}

cudaError_t launch_panel(int batch, int n, int j0, int nb, BatchedMat M, int* ipiv, double* stats, cudaStream_t st) {
  int cs = cluster_for(n);
  if (cs > kMaxCluster) cs = kMaxCluster;
  const int rows = n - j0;
  int rpc = (rows + cs - 1) / cs;
  if (rpc > kMaxRowsPerCta) return cudaErrorInvalidValue;
  if (cs == 1) rpc = rows;
  PanelArgs pa{M.p, M.ld, M.stride, n, j0, nb, rpc, cs, ipiv, stats};
  const size_t smem = (size_t)rpc * kLuNB * 8 + 2 * kLuNB * 8 + (kPanelThreads / 32) * 12 + 64;
  static size_t smem_set = 0;
  if (smem > smem_set) {
    cudaError_t e = cudaFuncSetAttribute(panel_getrf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)std::max<size_t>(smem, 48 * 1024));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(panel_getrf_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    smem_set = std::max<size_t>(smem, 48 * 1024);
  }
  if (cs == 1) {
    panel_getrf_kernel<<<batch, kPanelThreads, smem, st>>>(pa);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(batch * cs);
  cfg.blockDim = dim3(kPanelThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, panel_getrf_kernel, pa);
}

cudaError_t launch_swap_trsm(int batch, int n, int j0, int nb, const double* L, long long ldL, long long strideL,
                             const int* ipiv, const Seg* segs, int nseg, cudaStream_t st, int do_swaps = 1) {
  SwapTrsmArgs a{};
  a.do_swaps = do_swaps;
  a.L = L;
  a.ldL = ldL;
  a.strideL = strideL;
  a.ipiv = ipiv;
  a.n = n;
  a.j0 = j0;
  a.nb = nb;
  int total = 0;
  for (int i = 0; i < nseg; ++i) {
    if (segs[i].ncols <= 0) continue;
    a.seg[a.nseg++] = segs[i];
    total += segs[i].ncols;
  }
  if (total == 0) return cudaSuccess;
  dim3 grid(batch, (total + kColThreads - 1) / kColThreads);
  swap_trsm_kernel<<<grid, kColThreads, 0, st>>>(a);
  return cudaGetLastError();
}

// Blocked back substitution R <- U^-1 R, U = upper triangle of LU (n x n).
cudaError_t back_subst(int batch, int n, int m, const double* U, long long ldU, long long strideU, double* R,
                       long long ldR, long long strideR, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  const int nblk = (n + kLuNB - 1) / kLuNB;
  for (int jb = nblk - 1; jb >= 0; --jb) {
    const int r0 = jb * kLuNB, nb = std::min(kLuNB, n - r0);
    TrsmUArgs t{U, ldU, strideU, r0, nb, R, ldR, strideR, m};
    dim3 grid(batch, (m + kColThreads - 1) / kColThreads);
    trsm_upper_kernel<<<grid, kColThreads, 0, st>>>(t);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (r0 > 0) {
      GemmArgs g;
      g.m = r0;
      g.n = m;
      g.k = nb;
      g.batch = batch;
      g.A = U + (long long)r0 * ldU;
      g.lda = ldU;
      g.sA = strideU;
      g.B = R + r0;
      g.ldb = ldR;
      g.sB = strideR;
      g.C = R;
      g.ldc = ldR;
      g.sC = strideR;
      g.D = R;
      g.ldd = ldR;
      g.sD = strideR;
      g.alpha = -1.0;
      g.beta = 1.0;
      e = launch_dgemm(g, st);
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

}  // namespace

int bgetrf_max_n() { return kMaxCluster * kMaxRowsPerCta; }

cudaError_t lu_stats_init(double* stats, int batch, cudaStream_t st) {
  if (!stats || batch <= 0) return cudaSuccess;
  stats_init_kernel<<<(batch + 255) / 256, 256, 0, st>>>(stats, batch);
  return cudaGetLastError();
}

cudaError_t bgetrf_aug(int batch, int n, int m, BatchedMat M, int* ipiv, double* stats, cudaStream_t st) {
  if (batch <= 0 || n <= 0) return cudaSuccess;
  if (n > bgetrf_max_n()) return cudaErrorInvalidValue;
  cudaError_t e;
  for (int j0 = 0; j0 < n; j0 += kLuNB) {
    const int nb = std::min(kLuNB, n - j0);
    e = launch_panel(batch, n, j0, nb, M, ipiv, stats, st);
    if (e != cudaSuccess) return e;
    Seg segs[2];
    segs[0] = Seg{M.p, M.ld, M.stride, j0, 0};                                   // L columns: swaps only
    segs[1] = Seg{M.p + (long long)(j0 + nb) * M.ld, M.ld, M.stride, n + m - j0 - nb, 1};  // U12 | RHS
    e = launch_swap_trsm(batch, n, j0, nb, M.p, M.ld, M.stride, ipiv, segs, 2, st);
    if (e != cudaSuccess) return e;
    const int rows = n - j0 - nb, cols = n + m - j0 - nb;
    if (rows > 0 && cols > 0) {
      GemmArgs g;
      g.m = rows;
      g.n = cols;
      g.k = nb;
      g.batch = batch;
      g.A = M.p + (long long)j0 * M.ld + j0 + nb;
      g.lda = M.ld;
      g.sA = M.stride;
      g.B = M.p + (long long)(j0 + nb) * M.ld + j0;
      g.ldb = M.ld;
      g.sB = M.stride;
      double* C = M.p + (long long)(j0 + nb) * M.ld + j0 + nb;
      g.C = C;
      g.ldc = M.ld;
      g.sC = M.stride;
      g.D = C;
      g.ldd = M.ld;
      g.sD = M.stride;
      g.alpha = -1.0;
      g.beta = 1.0;
      e = launch_dgemm(g, st);
      if (e != cudaSuccess) return e;
    }
  }
  return back_subst(batch, n, m, M.p, M.ld, M.stride, M.p + (long long)n * M.ld, M.ld, M.stride, st);
}

cudaError_t bgetrs(int batch, int n, int m, BatchedMat LU, const int* ipiv, BatchedMat R, cudaStream_t st) {
  if (batch <= 0 || n <= 0 || m <= 0) return cudaSuccess;
  cudaError_t e;
  {
    const int cpc = 8;
    const size_t smem = (size_t)n * 12;
    static size_t smem_set = 0;
    if (smem > smem_set && smem > 48 * 1024) {
      e = cudaFuncSetAttribute(laswp_perm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      smem_set = smem;
    }
    laswp_perm_kernel<<<dim3(batch, (m + cpc - 1) / cpc), 256, smem, st>>>(ipiv, n, R.p, R.ld, R.stride, m, cpc);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  for (int j0 = 0; j0 < n; j0 += kLuNB) {
    const int nb = std::min(kLuNB, n - j0);
    Seg seg{R.p, R.ld, R.stride, m, 1};
    e = launch_swap_trsm(batch, n, j0, nb, LU.p, LU.ld, LU.stride, ipiv, &seg, 1, st, /*do_swaps=*/0);
    if (e != cudaSuccess) return e;
    const int rows = n - j0 - nb;
    if (rows > 0) {
      GemmArgs g;
      g.m = rows;
      g.n = m;
      g.k = nb;
      g.batch = batch;
      g.A = LU.p + (long long)j0 * LU.ld + j0 + nb;
      g.lda = LU.ld;
      g.sA = LU.stride;
      g.B = R.p + j0;
      g.ldb = R.ld;
      g.sB = R.stride;
      g.C = R.p + j0 + nb;
      g.ldc = R.ld;
      g.sC = R.stride;
      g.D = R.p + j0 + nb;
      g.ldd = R.ld;
      g.sD = R.stride;
      g.alpha = -1.0;
      g.beta = 1.0;
      e = launch_dgemm(g, st);
      if (e != cudaSuccess) return e;
    }
  }
  return back_subst(batch, n, m, LU.p, LU.ld, LU.stride, R.p, R.ld, R.stride, st);
}

}  // namespace hpsk
