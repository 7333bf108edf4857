// lu.cu -- batched blocked LU with partial pivoting (see lu.cuh).
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "gemm.cuh"
#include "gemv.cuh"
#include "lu.cuh"

namespace hpsk {

namespace {

#ifndef HPS_PANEL_THREADS
#define HPS_PANEL_THREADS 512
#endif
#ifndef HPS_PANEL_UNROLL
#define HPS_PANEL_UNROLL 4
#endif
constexpr int kPanelThreads = HPS_PANEL_THREADS;
constexpr int kPanelUnroll = HPS_PANEL_UNROLL;
#ifndef HPS_PANEL_ROWS
#define HPS_PANEL_ROWS 448
#endif
constexpr int kRowsPerCta = HPS_PANEL_ROWS;  // 448 x 32 doubles = 112 KiB of panel per CTA
constexpr int kMaxCluster = 16;   // non-portable cluster size (same GPC)
constexpr int kMaxRowsPerCta = 864;
constexpr int kTrsvMaxRhs = 4;    // few-RHS triangular solves (slab_trsv_kernel): right-hand sides per call

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
// Per column: one cluster barrier.  Every CTA publishes its best candidate (value, row and
// the whole candidate row) and, for the CTA owning row j, row j itself, into
// double-buffered shared slots; after the barrier warp 0 of every CTA reduces the cs
// candidates and pulls the pivot row (and row j for the pivot owner) through DSMEM.
// Remote CTAs only ever read the published slots, so the local swap/elimination needs no
// second barrier; slot reuse two columns later is ordered by the intervening barrier.
__global__ void __launch_bounds__(kPanelThreads) panel_getrf_kernel(const PanelArgs a) {
  extern __shared__ __align__(16) double sm[];
  double* pan = sm;                               // [nb][rpc]
  double* cand_row = sm + (size_t)a.rpc * a.nb;   // [2][kLuNB] published candidate row
  double* jrow_pub = cand_row + 2 * kLuNB;        // [2][kLuNB] published row j
  double* urow = jrow_pub + 2 * kLuNB;            // pivot row (local copy)
  double* jrow = urow + kLuNB;                    // row j (pivot owner's copy)
  double* wv = jrow + kLuNB;                      // per-warp partial max
  double* cand_v = wv + kPanelThreads / 32;       // [2]
  int* wi = reinterpret_cast<int*>(cand_v + 2);
  int* cand_i = wi + kPanelThreads / 32;          // [2]
  int* s_piv = cand_i + 2;

  const int cs = a.cs;
  const int rank = cs > 1 ? (int)cluster_ctarank() : 0;
  const long long b = blockIdx.x / cs;
  double* M = a.M + b * a.stride;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x;  // nthr <= kPanelThreads
  const int rows_total = a.n - a.j0;
  const int r_begin = rank * a.rpc;
  const int nr = max(0, min(rows_total - r_begin, a.rpc));
  const int nb = a.nb;

  for (int e = tid; e < nr * nb; e += nthr) {  // cp.async: all of a thread's loads in flight
    const int r = e % nr, c = e / nr;
    cp_async8(pan + c * a.rpc + r, M + (long long)(a.j0 + c) * a.ld + a.j0 + r_begin + r, true);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();

  double pmin = DBL_MAX, pmax = 0.0;
  int first_zero = -1;

  for (int j = 0; j < nb; ++j) {
    const int buf = j & 1;
    // ---- local argmax over panel rows >= j
    double bv = -1.0;
    int bi = INT_MAX;
    for (int r = tid; r < nr; r += nthr) {
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
    const int own_j = j / a.rpc;
    if (warp == 0) {
      bv = lane < nthr / 32 ? wv[lane] : -1.0;
      bi = lane < nthr / 32 ? wi[lane] : INT_MAX;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
        argmax_merge(bv, bi, v2, i2);
      }
      // publish the candidate (value, row, whole row) and, if owned here, row j
      if (lane == 0) cand_v[buf] = bv, cand_i[buf] = bi;
      if (lane < nb) {
        cand_row[buf * kLuNB + lane] = (bi != INT_MAX) ? pan[lane * a.rpc + (bi - r_begin)] : 0.0;
        if (own_j == rank) jrow_pub[buf * kLuNB + lane] = pan[lane * a.rpc + (j - r_begin)];
      }
    }
    if (cs > 1)
      cluster_sync();
    else
      __syncthreads();
    if (warp == 0) {
      double gv = -1.0;
      int gi = INT_MAX, gr = 0;
      if (lane < cs) {
        gv = cs > 1 ? dsmem_ld_f64(dsmem_map(&cand_v[buf], lane)) : cand_v[buf];
        gi = cs > 1 ? dsmem_ld_s32(dsmem_map(&cand_i[buf], lane)) : cand_i[buf];
        gr = lane;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, gv, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, gi, o);
        const int r2 = __shfl_xor_sync(0xffffffffu, gr, o);
        if (v2 > gv || (v2 == gv && i2 < gi)) gv = v2, gi = i2, gr = r2;
      }
      const int piv = (gi == INT_MAX) ? j : gi;
      const int own_p = (gi == INT_MAX) ? own_j : gr;
      if (lane == 0) *s_piv = piv;
      if (lane < nb) {
        const double* src = &cand_row[buf * kLuNB + lane];
        if (gi == INT_MAX) {  // no candidate anywhere (cannot happen for rows >= nb): pivot = row j
          const double* sj = &jrow_pub[buf * kLuNB + lane];
          urow[lane] = (own_j == rank || cs == 1) ? *sj : dsmem_ld_f64(dsmem_map(sj, own_j));
        } else {
          urow[lane] = (own_p == rank || cs == 1) ? *src : dsmem_ld_f64(dsmem_map(src, own_p));
        }
        if (own_p == rank && piv != j) {
          const double* sj = &jrow_pub[buf * kLuNB + lane];
          jrow[lane] = (own_j == rank || cs == 1) ? *sj : dsmem_ld_f64(dsmem_map(sj, own_j));
        }
      }
    }
    __syncthreads();
    const int piv = *s_piv;
    // Row exchange without a barrier: row j takes the pivot row (nobody reads row j again in this
    // column), and the owner of row piv eliminates from the old row j (jrow) instead of pan.
    if (piv != j && own_j == rank)
      for (int c = tid; c < nb; c += nthr) pan[c * a.rpc + (j - r_begin)] = urow[c];

    const double pv = urow[j];
    const double apv = fabs(pv);
    if (!(apv > 0.0) || !isfinite(apv)) {
      if (first_zero < 0) first_zero = a.j0 + j;
    } else {
      pmin = fmin(pmin, apv);
      pmax = fmax(pmax, apv);
    }
    if (rank == 0 && tid == 0) a.ipiv[b * a.n + a.j0 + j] = a.j0 + piv;

    // ---- eliminate rows below j within this CTA's chunk (LAPACK scales by the reciprocal).
    // Each thread only touches its own rows, and the next column reads other threads' rows only
    // after its first barrier, so no barrier closes the column.
    const double inv = apv > 0.0 ? 1.0 / pv : 0.0;
    for (int r = tid; r < nr; r += nthr) {
      const int gr = r_begin + r;
      if (gr <= j) continue;
      const bool swapped = (gr == piv && piv != j);
      if (swapped)  // the old row j moves here whole, its earlier multipliers included
        for (int c = 0; c < j; ++c) pan[c * a.rpc + r] = jrow[c];
      if (apv > 0.0) {
        const double l = (swapped ? jrow[j] : pan[j * a.rpc + r]) * inv;
        pan[j * a.rpc + r] = l;
#pragma unroll kPanelUnroll
        for (int c = j + 1; c < nb; ++c) pan[c * a.rpc + r] = (swapped ? jrow[c] : pan[c * a.rpc + r]) - l * urow[c];
      } else if (swapped) {
        for (int c = j; c < nb; ++c) pan[c * a.rpc + r] = jrow[c];
      }
    }
  }
  __syncthreads();

  for (int e = tid; e < nr * nb; e += nthr) {
    const int r = e % nr, c = e / nr;
    M[(long long)(a.j0 + c) * a.ld + a.j0 + r_begin + r] = pan[c * a.rpc + r];
  }
  if (rank == 0 && tid == 0 && a.stats) {
    double* s = a.stats + 3 * b;
    s[0] = fmin(s[0], pmin);
    s[1] = fmax(s[1], pmax);
    if (first_zero >= 0 && s[2] < 0) s[2] = first_zero;
  }
  if (cs > 1) cluster_sync();  // keep the published slots alive until remote readers are done
}

// Register-resident variant of panel_getrf_kernel for 32-column panels with <= kPanelThreads rows per CTA: each
// thread keeps its row of the panel in registers (the elimination reads and writes no shared memory; the column
// loop is unrolled so the row indexes registers), everything else is panel_getrf_kernel's protocol: warp
// candidates -> warp 0 -> published candidate row / row j -> one cluster barrier -> warp 0 pulls the cluster
// candidates and the pivot row through DSMEM -> one CTA barrier -> exchange + elimination.  Each warp's best lane
// writes its row to the warp's slot before the first barrier, so the CTA candidate row is in shared memory when
// warp 0 picks it.  Same pivots and arithmetic as panel_getrf_kernel (bit-identical factors).
#ifndef HPS_PANEL_REGROW
#define HPS_PANEL_REGROW 1
#endif
__global__ void __launch_bounds__(kPanelThreads) panel_getrf_regrow_kernel(const PanelArgs a) {
  constexpr int NB = kLuNB, NW = kPanelThreads / 32;
  __shared__ double wrow[NW][NB];           // each warp's candidate row
  __shared__ double cand_row[2][NB];        // published CTA candidate row (double-buffered by column parity)
  __shared__ double jrow_pub[2][NB];        // published row j
  __shared__ double urow[NB], jrow[NB];     // the pivot row, the old row j (pivot owner)
  __shared__ double wv[NW], cand_v[2];
  __shared__ int wi[NW], cand_i[2], s_piv;
  const int cs = a.cs;
  const int rank = cs > 1 ? (int)cluster_ctarank() : 0;
  const long long b = blockIdx.x / cs;
  double* M = a.M + b * a.stride;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int rows_total = a.n - a.j0;
  const int r_begin = rank * a.rpc;
  const int nr = max(0, min(rows_total - r_begin, a.rpc));
  const int gr = r_begin + tid;
  const bool have = tid < nr;
  double row[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) row[c] = have ? M[(long long)(a.j0 + c) * a.ld + a.j0 + gr] : 0.0;
  double pmin = DBL_MAX, pmax = 0.0;
  int first_zero = -1;
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const int buf = j & 1;
    double bv = (have && gr >= j) ? fabs(row[j]) : -1.0;
    int bi = (have && gr >= j) ? gr : INT_MAX;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      argmax_merge(bv, bi, v2, i2);
    }
    if (have && gr == bi) {
#pragma unroll
      for (int c = 0; c < NB; ++c) wrow[warp][c] = row[c];
    }
    const int own_j = j / a.rpc;
    if (have && gr == j) {
#pragma unroll
      for (int c = 0; c < NB; ++c) jrow_pub[buf][c] = row[c];
    }
    if (lane == 0) wv[warp] = bv, wi[warp] = bi;
    __syncthreads();
    if (warp == 0) {
      double cv = lane < nw ? wv[lane] : -1.0;
      int ci = lane < nw ? wi[lane] : INT_MAX, cw = lane;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, cv, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, ci, o);
        const int w2 = __shfl_xor_sync(0xffffffffu, cw, o);
        if (v2 > cv || (v2 == cv && i2 < ci)) cv = v2, ci = i2, cw = w2;
      }
      if (lane == 0) cand_v[buf] = cv, cand_i[buf] = ci;
      cand_row[buf][lane] = ci != INT_MAX ? wrow[cw][lane] : 0.0;
    }
    if (cs > 1)
      cluster_sync();
    else
      __syncthreads();
    if (warp == 0) {
      double gv = -1.0;
      int gi = INT_MAX, go = 0;
      if (lane < cs) {
        gv = cs > 1 ? dsmem_ld_f64(dsmem_map(&cand_v[buf], lane)) : cand_v[buf];
        gi = cs > 1 ? dsmem_ld_s32(dsmem_map(&cand_i[buf], lane)) : cand_i[buf];
        go = lane;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, gv, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, gi, o);
        const int o2 = __shfl_xor_sync(0xffffffffu, go, o);
        if (v2 > gv || (v2 == gv && i2 < gi)) gv = v2, gi = i2, go = o2;
      }
      const int piv = (gi == INT_MAX) ? j : gi;
      const int own_p = (gi == INT_MAX) ? own_j : go;
      if (lane == 0) s_piv = piv;
      if (gi == INT_MAX)
        urow[lane] = (own_j == rank || cs == 1) ? jrow_pub[buf][lane] : dsmem_ld_f64(dsmem_map(&jrow_pub[buf][lane], own_j));
      else
        urow[lane] = (own_p == rank || cs == 1) ? cand_row[buf][lane] : dsmem_ld_f64(dsmem_map(&cand_row[buf][lane], own_p));
      if (own_p == rank && piv != j)
        jrow[lane] = (own_j == rank || cs == 1) ? jrow_pub[buf][lane] : dsmem_ld_f64(dsmem_map(&jrow_pub[buf][lane], own_j));
    }
    __syncthreads();
    const int piv = s_piv;
    if (piv != j && have && gr == j) {
#pragma unroll
      for (int c = 0; c < NB; ++c) row[c] = urow[c];
    }
    const double pv = urow[j];
    const double apv = fabs(pv);
    if (!(apv > 0.0) || !isfinite(apv)) {
      if (first_zero < 0) first_zero = a.j0 + j;
    } else {
      pmin = fmin(pmin, apv);
      pmax = fmax(pmax, apv);
    }
    if (rank == 0 && tid == 0) a.ipiv[b * a.n + a.j0 + j] = a.j0 + piv;
    const double inv = apv > 0.0 ? 1.0 / pv : 0.0;
    if (have && gr > j) {
      const bool swapped = (gr == piv && piv != j);
      if (swapped) {  // the old row j moves here whole, its earlier multipliers included
#pragma unroll
        for (int c = 0; c < NB; ++c) row[c] = jrow[c];
      }
      if (apv > 0.0) {
        const double l = row[j] * inv;
        row[j] = l;
#pragma unroll
        for (int c = j + 1; c < NB; ++c) row[c] = row[c] - l * urow[c];
      }
    }
  }
#pragma unroll
  for (int c = 0; c < NB; ++c)
    if (have) M[(long long)(a.j0 + c) * a.ld + a.j0 + gr] = row[c];
  if (rank == 0 && tid == 0 && a.stats) {
    double* st = a.stats + 3 * b;
    st[0] = fmin(st[0], pmin);
    st[1] = fmax(st[1], pmax);
    if (first_zero >= 0 && st[2] < 0) st[2] = first_zero;
  }
  if (cs > 1) cluster_sync();  // keep the published slots alive until remote readers are done
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

#ifndef HPS_COL_THREADS
#define HPS_COL_THREADS 128
#endif
constexpr int kColThreads = HPS_COL_THREADS;

// Row swaps of one panel applied to column segments, then U12 = L11^-1 A12
// (proj/src/local_solve.cpp:128 / merge.cpp:291: the forward half of the solve).
__global__ void __launch_bounds__(kColThreads) swap_trsm_kernel(const SwapTrsmArgs a) {
  __shared__ double L11[kLuNB][kLuNB + 1];
  __shared__ int piv[kLuNB];
  const long long b = blockIdx.x;
  const double* L = a.L + b * a.strideL;
  const int nb = a.nb;
  for (int e = threadIdx.x; e < nb * nb; e += kColThreads) {  // cp.async: all loads in flight
    const int r = e % nb, c = e / nb;
    cp_async8(&L11[r][c], L + (long long)(a.j0 + c) * a.ldL + a.j0 + r, true);
  }
  cp_async_commit();
  for (int e = threadIdx.x; e < nb; e += kColThreads) piv[e] = a.ipiv[b * a.n + a.j0 + e];
  cp_async_wait<0>();
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
  // column-oriented (right-looking) substitution: the updates of one step are independent FMAs,
  // so the dependent chain is nb steps long instead of nb^2/2
#pragma unroll
  for (int ii = 0; ii < kLuNB - 1; ++ii)
#pragma unroll
    for (int jj = ii + 1; jj < kLuNB; ++jj) v[jj] -= L11[jj][ii] * v[ii];
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
  __shared__ double rdiag[kLuNB];
  for (int e = threadIdx.x; e < nb * nb; e += kColThreads) {  // cp.async: all loads in flight
    const int r = e % nb, c = e / nb;
    cp_async8(&U11[r][c], U + (long long)(a.r0 + c) * a.ldU + a.r0 + r, true);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  for (int r = threadIdx.x; r < nb; r += kColThreads) rdiag[r] = 1.0 / U11[r][r];
  __syncthreads();
  const int col = blockIdx.y * kColThreads + threadIdx.x;
  if (col >= a.ncols) return;
  double* x = a.R + b * a.strideR + (long long)col * a.ldR + a.r0;
  double v[kLuNB];
#pragma unroll
  for (int jj = 0; jj < kLuNB; ++jj) v[jj] = jj < nb ? x[jj] : 0.0;
  // column-oriented back substitution (independent FMAs per step; reciprocal of the diagonal)
#pragma unroll
  for (int jj = kLuNB - 1; jj >= 0; --jj) {
    if (jj < nb) {
      v[jj] *= rdiag[jj];
#pragma unroll
      for (int ii = 0; ii < jj; ++ii) v[ii] -= U11[ii][jj] * v[jj];
    }
  }
#pragma unroll
  for (int jj = 0; jj < kLuNB; ++jj)
    if (jj < nb) x[jj] = v[jj];
}

// Apply the complete pivot sequence of a factorization to R (LAPACK laswp), via the
// composite permutation built in shared memory: R[i, :] <- R[perm[i], :].
// Large n (perm + column no longer fit one CTA's shared memory together): the composite
// permutation goes to global memory first, then each column is gathered through shared memory.
__global__ void build_perm_kernel(const int* ipiv, int n, int* perm_out) {
  extern __shared__ int pm[];
  const long long b = blockIdx.x;
  const int* pv = ipiv + b * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) pm[i] = i;
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 0; i < n; ++i) {
      const int j = pv[i];
      if (j != i) {
        const int t = pm[i];
        pm[i] = pm[j];
        pm[j] = t;
      }
    }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) perm_out[b * n + i] = pm[i];
}

__global__ void apply_perm_cols_kernel(const int* perm, int n, double* R, long long ldR, long long strideR, int ncols) {
  extern __shared__ __align__(16) double col[];
  const long long b = blockIdx.x;
  const int c = blockIdx.y;
  if (c >= ncols) return;
  double* x = R + b * strideR + (long long)c * ldR;
  const int* pm = perm + b * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) col[i] = x[pm[i]];
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = col[i];
}

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
  if ((long long)rpc * nb > (long long)kMaxRowsPerCta * kLuNB) return cudaErrorInvalidValue;
  if (cs == 1) rpc = rows;
  PanelArgs pa{M.p, M.ld, M.stride, n, j0, nb, rpc, cs, ipiv, stats};
  const size_t smem = (size_t)rpc * nb * 8 + 6 * kLuNB * 8 + (kPanelThreads / 32) * 12 + 128;
  static PerDeviceFlag smem_set;
  const int dv = current_device();
  if (smem > smem_set.value[dv]) {
    cudaError_t e = cudaFuncSetAttribute(panel_getrf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)std::max<size_t>(smem, 48 * 1024));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(panel_getrf_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    smem_set.value[dv] = std::max<size_t>(smem, 48 * 1024);
  }
#ifndef HPS_REGROW_MIN_CS
#define HPS_REGROW_MIN_CS 4
#endif
#ifndef HPS_REGROW_SINGLE_MIN_ROWS
#define HPS_REGROW_SINGLE_MIN_ROWS 100000
#endif
  // measured: the register-resident panel pays from 4-CTA clusters up (the 2-CTA n = 896 panels are slower)
  const bool regrow = HPS_PANEL_REGROW && nb == kLuNB && rpc <= kPanelThreads &&
                      (cs >= HPS_REGROW_MIN_CS || (cs == 1 && rpc >= HPS_REGROW_SINGLE_MIN_ROWS));
  if (regrow) {
    static PerDeviceFlag rset;
    if (!(rset.set >> dv & 1)) {
      cudaError_t e = cudaFuncSetAttribute(panel_getrf_regrow_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
      rset.set |= 1ull << dv;
    }
  }
  if (cs == 1) {
    // single-CTA panels: one thread per row up to kPanelThreads (the 56- and 112-row panels of the
    // deep merge levels would otherwise run 4-6 warps with no rows through every barrier)
    const int threads = std::min(kPanelThreads, std::max(32, (rpc + 31) / 32 * 32));
    if (regrow)
      panel_getrf_regrow_kernel<<<batch, threads, 0, st>>>(pa);
    else
      panel_getrf_kernel<<<batch, threads, smem, st>>>(pa);
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
  if (regrow) {
    cfg.dynamicSmemBytes = 0;
    return cudaLaunchKernelEx(&cfg, panel_getrf_regrow_kernel, pa);
  }
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

// Two-level blocking: 32-column panels (GEPP in shared memory) inside 256-column
// outer blocks, so the bulk of every factorization and solve is one DMMA GEMM
// with k = 256 per outer block instead of a k = 32 update per panel (the
// trailing matrix is streamed from HBM 8x less often).
constexpr int kOuterNB = 256;

// GEPP panel width: 32 columns, or 16 when the panel of a matrix beyond 16 CTAs x 864 rows would
// not fit the cluster's shared memory (2D L=9 / 3D L=4 roots, n up to 27,648)
int panel_width(int n) { return n > kMaxCluster * kMaxRowsPerCta ? kLuNB / 2 : kLuNB; }

// C[rows, cols] += alpha * A[rows, k] * B[k, cols] on sub-blocks of strided batches.
cudaError_t gemm_sub(int batch, int rows, int cols, int k, double alpha, const double* A, long long lda, long long sA,
                     const double* B, long long ldb, long long sB, double* C, long long ldc, long long sC,
                     cudaStream_t st) {
  if (rows <= 0 || cols <= 0 || k <= 0) return cudaSuccess;
  GemmArgs g;
  g.m = rows;
  g.n = cols;
  g.k = k;
  g.batch = batch;
  g.A = A;
  g.lda = lda;
  g.sA = sA;
  g.B = B;
  g.ldb = ldb;
  g.sB = sB;
  g.C = C;
  g.ldc = ldc;
  g.sC = sC;
  g.D = C;
  g.ldd = ldc;
  g.sD = sC;
  g.alpha = alpha;
  g.beta = 1.0;
  return launch_dgemm(g, st);
}

#define HPS_TRY(x)                                                                      \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) {                                                            \
      return e_;                                                                        \
    }                                                                                   \
  } while (0)

// ---- slab triangular solves on the tensor cores (n >= slab_min_n()) -------------------------
// A 256-row slab solve X_slab <- T_slab^-1 X_slab (T unit-lower L or upper U of one outer
// block) as ONE launch instead of 8 x (32-column TRSM + k=32 GEMM): the inverses of the
// slab's 32x32 diagonal blocks are formed first (one warp per block), then every CTA keeps a
// 32-column strip of X in shared memory and runs the blocked substitution with DMMA:
// X_b = T_bb^-1 X_b, then X_i -= T_ib X_b for the remaining blocks i of the slab.
#ifndef HPS_SLAB_MIN_N
#define HPS_SLAB_MIN_N 64
#endif
constexpr int kSlabMinN = HPS_SLAB_MIN_N;  // measured: 64 beats 128 and 512 (d4-d6 merges) and 48 (d7)
int slab_min_n() { return kSlabMinN; }
constexpr int kSlabCW = 32;                 // strip width (4 column groups x 8 columns)
#ifndef HPS_SLAB_WARPS
#define HPS_SLAB_WARPS 8
#endif
constexpr int kSlabWarps = HPS_SLAB_WARPS;  // 4: one warp per column group; 8: two warps per group split the rows
constexpr int kSlabThreads = 32 * kSlabWarps;
constexpr int kSlabRowSplit = kSlabWarps / 4;
constexpr int kSlabLdX = kOuterNB + 4;      // 260 = 4 mod 16: conflict-free B fragments
constexpr int kSlabChunk = 64;              // rows of T staged per update step
constexpr int kSlabLdA = kSlabChunk + 4;    // 68

struct SlabArgs {
  const double* T;
  long long ldT, strideT;
  int r0, nbk;          // slab rows [r0, r0 + nbk), nbk <= kOuterNB; T_slab = T[r0.., r0..]
  double* X;            // X[(c) * ldX + r0 + i] for c < ncols
  long long ldX, strideX;
  int ncols;
  const double* Winv;   // [batch][kOuterNB / 32][32 x 32] diagonal-block inverses (column-major)
  bool vec2;            // T, X 16-byte aligned with even leading dimensions, strides and r0: pairs of rows move as one
                        // 16-byte cp.async / store
};

template <bool UPPER>
__global__ void __launch_bounds__(32) diag_inv_kernel(const double* T, long long ld, long long stride, int r0,
                                                      int nbk, double* Winv) {
  __shared__ double D[kLuNB][kLuNB + 1];
  const long long b = blockIdx.x;
  const int blk = blockIdx.y, lane = threadIdx.x;
  const int s0 = r0 + blk * kLuNB, nb = min(kLuNB, r0 + nbk - s0);
  const double* Tb = T + b * stride;
  for (int e = lane; e < kLuNB * kLuNB; e += 32) {
    const int r = e % kLuNB, c = e / kLuNB;
    D[r][c] = (r < nb && c < nb) ? Tb[(long long)(s0 + c) * ld + s0 + r] : (r == c ? 1.0 : 0.0);
  }
  __syncwarp();
  double x[kLuNB];  // column `lane` of the inverse
#pragma unroll
  for (int i = 0; i < kLuNB; ++i) x[i] = i == lane ? 1.0 : 0.0;
  if (!UPPER) {
#pragma unroll
    for (int k = 0; k < kLuNB - 1; ++k)
#pragma unroll
      for (int i = k + 1; i < kLuNB; ++i) x[i] -= D[i][k] * x[k];
  } else {
#pragma unroll
    for (int k = kLuNB - 1; k >= 0; --k) {
      x[k] /= D[k][k];
#pragma unroll
      for (int i = 0; i < k; ++i) x[i] -= D[i][k] * x[k];
    }
  }
  double* out = Winv + (b * (kOuterNB / kLuNB) + blk) * (kLuNB * kLuNB) + lane * kLuNB;
#pragma unroll
  for (int i = 0; i < kLuNB; ++i) out[i] = x[i];
}

// Work items of one slab solve, in order: for each diagonal block (top-down for L, bottom-up for
// U) one "diag" item (X_b <- T_bb^-1 X_b) and one "update" item per 64-row chunk of the rows still
// to be solved.  Every item's A operand (an inverse block or a T chunk) is staged by cp.async one
// item ahead into a two-slot ring, so its global latency hides behind the previous item's DMMAs.
template <bool UPPER>
struct SlabItems {
  int nblk, nbk;
  HPS_DEV int blk(int step) const { return UPPER ? nblk - 1 - step : step; }
  HPS_DEV int rows_lo(int bk) const { return UPPER ? 0 : (bk + 1) * kLuNB; }
  HPS_DEV int rows_hi(int bk) const { return UPPER ? bk * kLuNB : nbk; }
  HPS_DEV int nchunks(int bk) const { return (rows_hi(bk) - rows_lo(bk) + kSlabChunk - 1) / kSlabChunk; }
};

template <bool UPPER>
__global__ void __launch_bounds__(kSlabThreads, kSlabWarps >= 16 ? 2 : 1) slab_trsm_kernel(const SlabArgs a) {
  extern __shared__ __align__(16) double smem[];
  double* xs = smem;                          // [kSlabCW][kSlabLdX]: X strip, k-major per column
  double* ring = xs + kSlabCW * kSlabLdX;     // 2 x [kLuNB][kSlabLdA]: A operand ([k][m]) per item
  const long long b = blockIdx.x;
  const int c0 = blockIdx.y * kSlabCW;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const double* T = a.T + b * a.strideT;
  double* X = a.X + b * a.strideX;
  const SlabItems<UPPER> it{(a.nbk + kLuNB - 1) / kLuNB, a.nbk};
  const double* winv = a.Winv + b * (kOuterNB / kLuNB) * (kLuNB * kLuNB);

  // item cursor: (step, chunk) with chunk == -1 the diag item
  auto stage = [&](int step, int chunk, double* dst) {
    const int bk = it.blk(step);
    if (chunk < 0) {
      const double* inv = winv + bk * (kLuNB * kLuNB);  // column-major: (m, k) at m + 32 k
      for (int e = 2 * tid; e < kLuNB * kLuNB; e += 2 * blockDim.x)
        cp_async16(dst + (e / kLuNB) * kSlabLdA + e % kLuNB, inv + e, 16);
    } else {
      const int q0 = it.rows_lo(bk) + chunk * kSlabChunk, qn = min(kSlabChunk, it.rows_hi(bk) - q0);
      const double* src = T + (long long)(a.r0 + bk * kLuNB) * a.ldT + a.r0 + q0;
      if (a.vec2) {
        for (int e = tid; e < kLuNB * kSlabChunk / 2; e += blockDim.x) {
          const int mm = 2 * (e % (kSlabChunk / 2)), k = e / (kSlabChunk / 2);
          const int valid = max(0, min(2, qn - mm)) * 8;
          cp_async16(dst + k * kSlabLdA + mm, valid ? src + (long long)k * a.ldT + mm : src, valid);
        }
      } else {
        for (int e = tid; e < kLuNB * kSlabChunk; e += blockDim.x) {
          const int mm = e % kSlabChunk, k = e / kSlabChunk;
          cp_async8(dst + k * kSlabLdA + mm, mm < qn ? src + (long long)k * a.ldT + mm : src, mm < qn);
        }
      }
    }
    cp_async_commit();
  };
  auto next = [&](int& step, int& chunk) {
    if (chunk + 1 < it.nchunks(it.blk(step))) {
      ++chunk;
    } else {
      ++step;
      chunk = -1;
    }
  };

  int step = 0, chunk = -1, slot = 0;
  stage(step, chunk, ring);
  // cp.async: every load in flight; rows up to the 32-row padding of the last diagonal block (zero-filled
  // past nbk: the padded inverse blocks multiply them by zero)
  const int nbr = it.nblk * kLuNB;
  for (int c = warp; c < kSlabCW; c += kSlabWarps) {
    const bool okc = c0 + c < a.ncols;
    const double* xc = X + (long long)(c0 + c) * a.ldX + a.r0;
    if (a.vec2) {
      for (int r = 2 * lane; r < nbr; r += 64) {
        const int valid = okc ? max(0, min(2, a.nbk - r)) * 8 : 0;
        cp_async16(xs + c * kSlabLdX + r, valid ? xc + r : X, valid);
      }
    } else {
      for (int r = lane; r < nbr; r += 32) {
        const bool ok = okc && r < a.nbk;
        cp_async8(xs + c * kSlabLdX + r, ok ? xc + r : X, ok);
      }
    }
  }
  cp_async_commit();
  const int wc = (warp & 3) * 8;  // this warp's 8 columns of the strip
  const int rh = warp >> 2;       // its share of the rows (kSlabRowSplit > 1)
  while (step < it.nblk) {
    int ns = step, nc = chunk;
    next(ns, nc);
    cp_async_wait<0>();
    __syncthreads();  // item's operand landed; the other slot's previous item is consumed
    if (ns < it.nblk) stage(ns, nc, ring + (slot ^ 1) * (kLuNB * kSlabLdA));
    const double* A = ring + slot * (kLuNB * kSlabLdA);
    const int s0 = it.blk(step) * kLuNB;
    if (chunk < 0) {  // X_b <- T_bb^-1 X_b, in place (each warp reads and writes only its own columns)
      constexpr int kT = kLuNB / 8 / kSlabRowSplit;  // 8-row tiles of this warp
      double acc[kT][2];
#pragma unroll
      for (int i = 0; i < kT; ++i) acc[i][0] = acc[i][1] = 0.0;
#pragma unroll
      for (int kb = 0; kb < kLuNB; kb += 4) {
        const double bv = xs[(wc + g) * kSlabLdX + s0 + kb + t4];
#pragma unroll
        for (int i = 0; i < kT; ++i)
          dmma_8x8x4(acc[i][0], acc[i][1], A[(kb + t4) * kSlabLdA + (rh * kT + i) * 8 + g], bv);
      }
      if (kSlabRowSplit > 1)
        __syncthreads();  // the other row half has read X_b
      else
        __syncwarp();
#pragma unroll
      for (int i = 0; i < kT; ++i)
#pragma unroll
        for (int h = 0; h < 2; ++h) xs[(wc + 2 * t4 + h) * kSlabLdX + s0 + (rh * kT + i) * 8 + g] = acc[i][h];
    } else {  // X_q -= T_qb X_b for this chunk's rows
      const int q0 = it.rows_lo(it.blk(step)) + chunk * kSlabChunk;
      const int qn = min(kSlabChunk, it.rows_hi(it.blk(step)) - q0);
      double bneg[kLuNB / 4];
#pragma unroll
      for (int kb = 0; kb < kLuNB; kb += 4) bneg[kb / 4] = -xs[(wc + g) * kSlabLdX + s0 + kb + t4];
#ifndef HPS_SLAB_CHAINS
#define HPS_SLAB_CHAINS 4
#endif
      // kCh independent 8-row tiles per iteration (kCh DMMA accumulation chains in flight); tiles past the
      // chunk's last are computed on padding rows and not stored
      constexpr int kCh = HPS_SLAB_CHAINS;
      const int nmt = (qn + 7) / 8;
      for (int mt = kCh * rh; mt < nmt; mt += kCh * kSlabRowSplit) {
        const int r = q0 + mt * 8 + g;
        double c[kCh][2];
#pragma unroll
        for (int i = 0; i < kCh; ++i)
#pragma unroll
          for (int h = 0; h < 2; ++h) c[i][h] = xs[(wc + 2 * t4 + h) * kSlabLdX + r + 8 * i];
#pragma unroll
        for (int kb = 0; kb < kLuNB; kb += 4)
#pragma unroll
          for (int i = 0; i < kCh; ++i)
            dmma_8x8x4(c[i][0], c[i][1], A[(kb + t4) * kSlabLdA + (mt + i) * 8 + g], bneg[kb / 4]);
#pragma unroll
        for (int i = 0; i < kCh; ++i)
          if (mt + i < nmt)
#pragma unroll
            for (int h = 0; h < 2; ++h) xs[(wc + 2 * t4 + h) * kSlabLdX + r + 8 * i] = c[i][h];
      }
    }
    step = ns;
    chunk = nc;
    slot ^= 1;
  }
  __syncthreads();
  for (int c = warp; c < kSlabCW && c0 + c < a.ncols; c += kSlabWarps) {
    double* xc = X + (long long)(c0 + c) * a.ldX + a.r0;
    const double* sc = xs + c * kSlabLdX;
    if (a.vec2) {
      for (int r = 2 * lane; r < a.nbk; r += 64) {
        if (r + 1 < a.nbk)
          *reinterpret_cast<double2*>(xc + r) = *reinterpret_cast<const double2*>(sc + r);
        else
          xc[r] = sc[r];
      }
    } else {
      for (int r = lane; r < a.nbk; r += 32) xc[r] = sc[r];
    }
  }
}

long long slab_winv_elems(int batch) { return (long long)batch * (kOuterNB / kLuNB) * kLuNB * kLuNB; }

// grow a workspace array (contents are scratch); the bytes go to *total.  dry: count only (footprint
// estimation, hpsg_estimate_bytes), nothing is allocated.
template <class T>
cudaError_t ws_grow(T*& p, long long& cap, long long need, size_t* total, bool dry = false) {
  if (need <= cap) return cudaSuccess;
  if (!dry) {
    if (p) cudaFree(p);
    p = nullptr;
    cudaError_t e = cudaMalloc(&p, (size_t)need * sizeof(T));
    if (e != cudaSuccess) {
      if (total) *total -= (size_t)cap * sizeof(T);
      cap = 0;
      return e;
    }
  }
  if (total) *total += (size_t)(need - cap) * sizeof(T);
  cap = need;
  return cudaSuccess;
}

// X[r0:r0+nbk, 0:ncols] <- T_slab^-1 X[...] (unit-lower or upper slab of T), two launches
template <bool UPPER>
cudaError_t slab_trsm(int batch, const double* T, long long ldT, long long sT, int r0, int nbk, double* X,
                      long long ldX, long long sX, int ncols, LuWorkspace& ws, cudaStream_t st) {
  if (ncols <= 0 || nbk <= 0) return cudaSuccess;
  HPS_TRY(ws_grow(ws.winv, ws.winv_cap, slab_winv_elems(batch), ws.total));
  double* w = ws.winv;
  const int nblk = (nbk + kLuNB - 1) / kLuNB;
  diag_inv_kernel<UPPER><<<dim3(batch, nblk), 32, 0, st>>>(T, ldT, sT, r0, nbk, w);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const size_t smem = (size_t)(kSlabCW * kSlabLdX + 2 * kLuNB * kSlabLdA) * sizeof(double);
  static PerDeviceFlag attr;
  const int dv = current_device();
  if (!(attr.set >> dv & 1)) {
    e = cudaFuncSetAttribute(slab_trsm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(slab_trsm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr.set |= 1ull << dv;
  }
  const bool vec2 = ldT % 2 == 0 && sT % 2 == 0 && ldX % 2 == 0 && sX % 2 == 0 && r0 % 2 == 0 &&
                    reinterpret_cast<uintptr_t>(T) % 16 == 0 && reinterpret_cast<uintptr_t>(X) % 16 == 0;
  SlabArgs a{T, ldT, sT, r0, nbk, X, ldX, sX, ncols, w, vec2};
  const long long strips = (ncols + kSlabCW - 1) / kSlabCW;
  if (strips > 65535) return cudaErrorInvalidConfiguration;
  slab_trsm_kernel<UPPER><<<dim3(batch, (unsigned)strips), kSlabThreads, smem, st>>>(a);
  return cudaGetLastError();
}

// Blocked back substitution R <- U^-1 R, U = upper triangle of LU (n x n).
}  // namespace
template <bool UPPER>
cudaError_t trsv_blocked(const double* T, long long ldT, int n, double* X, long long ldX, int m, LuWorkspace& ws,
                         cudaStream_t st);
namespace {

cudaError_t back_subst(int batch, int n, int m, const double* U, long long ldU, long long strideU, double* R,
                       long long ldR, long long strideR, LuWorkspace& ws, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  // one large matrix with a few RHS (the implicit root's [D | h] factorization): the slab TRSV
  // (one CTA per 256-row slab + a streaming GEMV) instead of a chain of 32x32 TRSM + GEMM launches
  if (batch == 1 && m <= kTrsvMaxRhs && n >= 2 * kOuterNB) return trsv_blocked<true>(U, ldU, n, R, ldR, m, ws, st);
  const int nouter = (n + kOuterNB - 1) / kOuterNB;
  for (int ob = nouter - 1; ob >= 0; --ob) {
    const int r0 = ob * kOuterNB, r1 = std::min(n, r0 + kOuterNB);
    const int nsub = (r1 - r0 + kLuNB - 1) / kLuNB;
    if (n >= slab_min_n() && m >= kSlabCW) {
      HPS_TRY(slab_trsm<true>(batch, U, ldU, strideU, r0, r1 - r0, R, ldR, strideR, m, ws, st));
      HPS_TRY(gemm_sub(batch, r0, m, r1 - r0, -1.0, U + (long long)r0 * ldU, ldU, strideU, R + r0, ldR, strideR, R,
                       ldR, strideR, st));
      continue;
    }
    for (int sb = nsub - 1; sb >= 0; --sb) {
      const int s0 = r0 + sb * kLuNB, nb = std::min(kLuNB, r1 - s0);
      TrsmUArgs t{U, ldU, strideU, s0, nb, R, ldR, strideR, m};
      dim3 grid(batch, (m + kColThreads - 1) / kColThreads);
      trsm_upper_kernel<<<grid, kColThreads, 0, st>>>(t);
      HPS_TRY(cudaGetLastError());
      // rows of this outer block above the sub-block
      HPS_TRY(gemm_sub(batch, s0 - r0, m, nb, -1.0, U + (long long)s0 * ldU + r0, ldU, strideU, R + s0, ldR, strideR,
                       R + r0, ldR, strideR, st));
    }
    // everything above the outer block, k = outer block width
    HPS_TRY(gemm_sub(batch, r0, m, r1 - r0, -1.0, U + (long long)r0 * ldU, ldU, strideU, R + r0, ldR, strideR, R, ldR,
                     strideR, st));
  }
  return cudaSuccess;
}


// ---- look-ahead driver (n > 512): the next outer panel is factored on a side stream
// while the main stream runs the bulk of the current trailing update.  Row swaps that
// would touch columns outside the panel being factored are deferred and applied once per
// outer block from the block's composite permutation.

// moved-row list (dst, src) of the composite permutation of one outer block's pivots
__global__ void block_perm_kernel(const int* ipiv, int n, int J, int Jend, int* moved, int* nmoved) {
  extern __shared__ int perm[];  // perm[i]: original row (relative to J) now at row J + i
  __shared__ int cnt;
  const long long b = blockIdx.x;
  const int len = n - J;
  for (int i = threadIdx.x; i < len; i += blockDim.x) perm[i] = i;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  if (threadIdx.x == 0)
    for (int j = J; j < Jend; ++j) {
      const int p = ipiv[b * n + j];
      if (p != j) {
        const int t = perm[j - J];
        perm[j - J] = perm[p - J];
        perm[p - J] = t;
      }
    }
  __syncthreads();
  int* mv = moved + b * (4 * kOuterNB);
  for (int i = threadIdx.x; i < len; i += blockDim.x)
    if (perm[i] != i) {
      const int s = atomicAdd(&cnt, 1);
      mv[2 * s] = J + i;
      mv[2 * s + 1] = J + perm[i];
    }
  __syncthreads();
  if (threadIdx.x == 0) nmoved[b] = cnt;
}

// new[dst] = old[src] over the moved rows, one warp per column, columns [ca0,ca1) u [cb0,cb1)
__global__ void apply_perm_kernel(double* M, long long ld, long long stride, const int* moved, const int* nmoved,
                                  int ca0, int ca1, int cb0, int cb1) {
  const long long b = blockIdx.x;
  const int nm = nmoved[b];
  const int* mv = moved + b * (4 * kOuterNB);
  const int lane = threadIdx.x & 31;
  const int na = ca1 - ca0, ntot = na + (cb1 - cb0);
  for (int w = blockIdx.y * (blockDim.x / 32) + (threadIdx.x >> 5); w < ntot; w += gridDim.y * (blockDim.x / 32)) {
    const int c = w < na ? ca0 + w : cb0 + (w - na);
    double* col = M + b * stride + (long long)c * ld;
    double v[2 * kOuterNB / 32];
#pragma unroll
    for (int u = 0; u < 2 * kOuterNB / 32; ++u) {
      const int t = lane + 32 * u;
      if (t < nm) v[u] = col[mv[2 * t + 1]];
    }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 2 * kOuterNB / 32; ++u) {
      const int t = lane + 32 * u;
      if (t < nm) col[mv[2 * t]] = v[u];
    }
  }
}

cudaError_t lookahead_prepare(LuWorkspace& ws, int batch, int nev) {
  if (!ws.side) {
    // the panel stream outranks the trailing GEMMs so its few CTAs are scheduled as SMs free up
    int lo = 0, hi = 0;
    HPS_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    HPS_TRY(cudaStreamCreateWithPriority(&ws.side, cudaStreamNonBlocking, hi));
  }
  if (ws.n_ev < nev) {
    cudaEvent_t* ev = new cudaEvent_t[nev];
    for (int i = 0; i < ws.n_ev; ++i) ev[i] = ws.ev[i];
    for (int i = ws.n_ev; i < nev; ++i) HPS_TRY(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    delete[] ws.ev;
    ws.ev = ev;
    ws.n_ev = nev;
  }
  if (batch > ws.la_cap) {
    long long c1 = ws.la_cap * 4 * kOuterNB, c2 = ws.la_cap;
    HPS_TRY(ws_grow(ws.moved, c1, (long long)batch * 4 * kOuterNB, ws.total));
    HPS_TRY(ws_grow(ws.nmoved, c2, (long long)batch, ws.total));
    ws.la_cap = batch;
  }
  return cudaSuccess;
}

// inner loop of outer block [J, Jend): panels + in-block swaps/TRSM + in-block updates
cudaError_t factor_outer_panel(int batch, int n, int J, int Jend, BatchedMat M, int* ipiv, double* stats,
                               cudaStream_t s) {
  const long long ld = M.ld, sM = M.stride;
  double* A = M.p;
  auto at = [&](int r, int c) { return A + (long long)c * ld + r; };
  const int PW = panel_width(n);
  for (int j0 = J; j0 < Jend; j0 += PW) {
    const int nb = std::min(PW, Jend - j0);
    HPS_TRY(launch_panel(batch, n, j0, nb, M, ipiv, stats, s));
    Seg segs[2];
    segs[0] = Seg{at(0, J), ld, sM, j0 - J, 0};                  // in-block L columns: swaps only
    segs[1] = Seg{at(0, j0 + nb), ld, sM, Jend - j0 - nb, 1};     // rest of the outer panel: swaps + L11^-1
    HPS_TRY(launch_swap_trsm(batch, n, j0, nb, A, ld, sM, ipiv, segs, 2, s));
    HPS_TRY(gemm_sub(batch, n - j0 - nb, Jend - j0 - nb, nb, -1.0, at(j0 + nb, j0), ld, sM, at(j0, j0 + nb), ld, sM,
                     at(j0 + nb, j0 + nb), ld, sM, s));
  }
  return cudaSuccess;
}

cudaError_t bgetrf_aug_lookahead(int batch, int n, int m, BatchedMat M, int* ipiv, double* stats, LuWorkspace& ws,
                                 cudaStream_t st, bool keep_L) {
  const int K = (n + kOuterNB - 1) / kOuterNB;
  HPS_TRY(lookahead_prepare(ws, batch, 2 * K + 2));
  struct {
    cudaStream_t ps;
    int* moved;
    int* nmoved;
  } la{ws.side, ws.moved, ws.nmoved};
  cudaEvent_t* evP = ws.ev;      // panel k done (side stream)
  cudaEvent_t* evA = ws.ev + K;  // next panel's columns updated (main stream)
  cudaEvent_t evF = ws.ev[2 * K];
  const long long ld = M.ld, sM = M.stride;
  double* A = M.p;
  auto at = [&](int r, int c) { return A + (long long)c * ld + r; };
  const int ncol = n + m;
  static PerDeviceFlag perm_smem_set;
  const int dv = current_device();
  const size_t perm_smem = (size_t)n * sizeof(int);
  if (perm_smem > 48 * 1024 && perm_smem > perm_smem_set.value[dv]) {
    HPS_TRY(cudaFuncSetAttribute(block_perm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)perm_smem));
    perm_smem_set.value[dv] = perm_smem;
  }
  HPS_TRY(cudaEventRecord(evF, st));
  HPS_TRY(cudaStreamWaitEvent(la.ps, evF, 0));
  HPS_TRY(factor_outer_panel(batch, n, 0, std::min(n, kOuterNB), M, ipiv, stats, la.ps));
  HPS_TRY(cudaEventRecord(evP[0], la.ps));
  for (int k = 0; k < K; ++k) {
    const int J = k * kOuterNB, Jend = std::min(n, J + kOuterNB);
    HPS_TRY(cudaStreamWaitEvent(st, evP[k], 0));
    // deferred swaps of block k for every column outside [J, Jend)
    block_perm_kernel<<<batch, 256, (size_t)(n - J) * sizeof(int), st>>>(ipiv, n, J, Jend, la.moved, la.nmoved);
    HPS_TRY(cudaGetLastError());
    {
      const int left = keep_L ? J : 0;
      const int ncols = left + (ncol - Jend);
      const int gy = std::max(1, std::min(65535, (ncols + 7) / 8));
      apply_perm_kernel<<<dim3(batch, gy), 256, 0, st>>>(A, ld, sM, la.moved, la.nmoved, 0, left, Jend, ncol);
      HPS_TRY(cudaGetLastError());
    }
    // U12 = L11^-1 A12 over the block's row slab
    if (n >= slab_min_n() && Jend < ncol) {
      HPS_TRY(slab_trsm<false>(batch, A, ld, sM, J, Jend - J, at(0, Jend), ld, sM, ncol - Jend, ws, st));
    } else
    for (int j0 = J; j0 < Jend && Jend < ncol; j0 += kLuNB) {
      const int nb = std::min(kLuNB, Jend - j0);
      Seg seg{at(0, Jend), ld, sM, ncol - Jend, 1};
      HPS_TRY(launch_swap_trsm(batch, n, j0, nb, A, ld, sM, ipiv, &seg, 1, st, /*do_swaps=*/0));
      HPS_TRY(gemm_sub(batch, Jend - j0 - nb, ncol - Jend, nb, -1.0, at(j0 + nb, j0), ld, sM, at(j0, Jend), ld, sM,
                       at(j0 + nb, Jend), ld, sM, st));
    }
    if (Jend < n) {
      const int J2end = std::min(n, Jend + kOuterNB);
      // (a) the next outer panel's columns first, then hand them to the side stream
      HPS_TRY(gemm_sub(batch, n - Jend, J2end - Jend, Jend - J, -1.0, at(Jend, J), ld, sM, at(J, Jend), ld, sM,
                       at(Jend, Jend), ld, sM, st));
      HPS_TRY(cudaEventRecord(evA[k], st));
      HPS_TRY(cudaStreamWaitEvent(la.ps, evA[k], 0));
      HPS_TRY(factor_outer_panel(batch, n, Jend, J2end, M, ipiv, stats, la.ps));
      HPS_TRY(cudaEventRecord(evP[k + 1], la.ps));
      // (b) the rest of the trailing update, concurrently with that panel
      HPS_TRY(gemm_sub(batch, n - Jend, ncol - J2end, Jend - J, -1.0, at(Jend, J), ld, sM, at(J, J2end), ld, sM,
                       at(Jend, J2end), ld, sM, st));
    }
  }
  return back_subst(batch, n, m, A, ld, sM, at(0, n), ld, sM, ws, st);
}

}  // namespace

int bgetrf_max_n() { return kMaxCluster * kMaxRowsPerCta * (kLuNB / (kLuNB / 2)); }

cudaError_t lu_stats_init(double* stats, int batch, cudaStream_t st) {
  if (!stats || batch <= 0) return cudaSuccess;
  stats_init_kernel<<<(batch + 255) / 256, 256, 0, st>>>(stats, batch);
  return cudaGetLastError();
}

// look-ahead (panels of the next outer block on a high-priority side stream) from this n up; measured at
// L=8: d0 -1.7 ms, d1 -3 ms, d2 -1 ms (256 and 512 measured equal as the threshold)
#ifndef HPS_LOOKAHEAD_MIN_N
#define HPS_LOOKAHEAD_MIN_N (2 * kOuterNB)
#endif
constexpr int kLookaheadMinN = HPS_LOOKAHEAD_MIN_N;

cudaError_t bgetrf_aug(int batch, int n, int m, BatchedMat M, int* ipiv, double* stats, LuWorkspace& ws,
                       cudaStream_t st, bool keep_L) {
  if (batch <= 0 || n <= 0) return cudaSuccess;
  if (n > bgetrf_max_n()) return cudaErrorInvalidValue;
  if (ws.lookahead && n > kLookaheadMinN) return bgetrf_aug_lookahead(batch, n, m, M, ipiv, stats, ws, st, keep_L);
  const long long ld = M.ld, sM = M.stride;
  double* A = M.p;
  auto at = [&](int r, int c) { return A + (long long)c * ld + r; };
  const int ncol = n + m;
  for (int J = 0; J < n; J += kOuterNB) {
    const int Jend = std::min(n, J + kOuterNB);
    // (1) factor the outer panel columns [J, Jend); the row swaps go to every column at once,
    //     while columns right of the outer panel are otherwise left untouched
    for (int j0 = J; j0 < Jend; j0 += panel_width(n)) {
      const int nb = std::min(panel_width(n), Jend - j0);
      HPS_TRY(launch_panel(batch, n, j0, nb, M, ipiv, stats, st));
      Seg segs[3];
      segs[0] = keep_L ? Seg{A, ld, sM, j0, 0}                       // factored L columns: swaps only
                       : Seg{at(0, J), ld, sM, j0 - J, 0};          // (this outer block's only: the rest is dead)
      segs[1] = Seg{at(0, j0 + nb), ld, sM, Jend - j0 - nb, 1};      // rest of the outer panel: swaps + L11^-1
      segs[2] = Seg{at(0, Jend), ld, sM, ncol - Jend, 0};            // right of the outer panel: swaps only
      HPS_TRY(launch_swap_trsm(batch, n, j0, nb, A, ld, sM, ipiv, segs, 3, st));
      HPS_TRY(gemm_sub(batch, n - j0 - nb, Jend - j0 - nb, nb, -1.0, at(j0 + nb, j0), ld, sM, at(j0, j0 + nb), ld, sM,
                       at(j0 + nb, j0 + nb), ld, sM, st));
    }
    // (2) U12 = L11^-1 A12 over the outer block's row slab (blocked forward substitution)
    if (n >= slab_min_n() && Jend < ncol) {
      HPS_TRY(slab_trsm<false>(batch, A, ld, sM, J, Jend - J, at(0, Jend), ld, sM, ncol - Jend, ws, st));
    } else
    for (int j0 = J; j0 < Jend && Jend < ncol; j0 += kLuNB) {
      const int nb = std::min(kLuNB, Jend - j0);
      Seg seg{at(0, Jend), ld, sM, ncol - Jend, 1};
      HPS_TRY(launch_swap_trsm(batch, n, j0, nb, A, ld, sM, ipiv, &seg, 1, st, /*do_swaps=*/0));
      HPS_TRY(gemm_sub(batch, Jend - j0 - nb, ncol - Jend, nb, -1.0, at(j0 + nb, j0), ld, sM, at(j0, Jend), ld, sM,
                       at(j0 + nb, Jend), ld, sM, st));
    }
    // delayed trailing update with k = outer block width
    HPS_TRY(gemm_sub(batch, n - Jend, ncol - Jend, Jend - J, -1.0, at(Jend, J), ld, sM, at(J, Jend), ld, sM,
                     at(Jend, Jend), ld, sM, st));
  }
  return back_subst(batch, n, m, A, ld, sM, at(0, n), ld, sM, ws, st);
}

// ---- single-matrix, few-RHS triangular solves (the implicit-root solve: n = 7168, 1 RHS) --------
// Per 256-row slab: ONE CTA solves the slab (its eight 32x32 diagonal blocks one warp per RHS
// with shuffle broadcasts, the in-slab updates by the whole CTA), then one streaming GEMV applies
// the slab to every remaining row.  2 launches per slab instead of ~17.

template <bool UPPER>
__global__ void __launch_bounds__(256) slab_trsv_kernel(const double* T, long long ldT, int r0, int nbk, double* X,
                                                         long long ldX, int m) {
  // dynamic smem: tb[kLuNB][kOuterNB] (the sub-block's column block of the slab, all rows)
  extern __shared__ __align__(16) double tb[];
  __shared__ double xs[kTrsvMaxRhs][kOuterNB];
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  for (int e = tid; e < kTrsvMaxRhs * kOuterNB; e += 256) {
    const int c = e / kOuterNB, r = e % kOuterNB;
    xs[c][r] = (c < m && r < nbk) ? X[(long long)c * ldX + r0 + r] : 0.0;
  }
  const int nblk = (nbk + kLuNB - 1) / kLuNB;
  for (int step = 0; step < nblk; ++step) {
    const int bk = UPPER ? nblk - 1 - step : step;
    const int s0 = bk * kLuNB, nb = min(kLuNB, nbk - s0);
    const int ra = UPPER ? 0 : s0, rb = UPPER ? s0 + nb : nbk;  // rows touched: diag block + rest
    __syncthreads();
    // stage T[r0 + ra .. r0 + rb, r0 + s0 .. + nb) (column-major in tb: tb[k * kOuterNB + r])
    // cp.async: all 32 of a thread's loads in flight (a plain load/store loop waits one memory
    // latency per element; rows outside [ra, rb) are zero-filled and never read)
    for (int e = tid; e < kLuNB * kOuterNB; e += 256) {
      const int k = e / kOuterNB, r = e % kOuterNB;
      const bool ok = r >= ra && r < rb && k < nb;
      cp_async8(tb + e, ok ? T + (long long)(r0 + s0 + k) * ldT + r0 + r : T, ok);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    if (w < m) {
      double x = xs[w][s0 + lane < nbk ? s0 + lane : 0];
      if (!UPPER) {
        for (int k = 0; k < nb; ++k) {
          const double xk = __shfl_sync(0xffffffffu, x, k);
          if (lane > k && lane < nb) x -= tb[k * kOuterNB + s0 + lane] * xk;
        }
      } else {
        // reciprocal of the lane's pivot computed off the dependency chain: a divide on the
        // chain costs a full FP64 division sequence per column (measured 64 -> 38 us per slab)
        const double dinv = lane < nb ? 1.0 / tb[lane * kOuterNB + s0 + lane] : 0.0;
        for (int k = nb - 1; k >= 0; --k) {
          if (lane == k) x *= dinv;
          const double xk = __shfl_sync(0xffffffffu, x, k);
          if (lane < k) x -= tb[k * kOuterNB + s0 + lane] * xk;
        }
      }
      if (lane < nb) xs[w][s0 + lane] = x;
    }
    __syncthreads();
    const int ua = UPPER ? 0 : s0 + nb, ub = UPPER ? s0 : nbk;
    for (int r = ua + tid; r < ub; r += 256) {
      double acc[kTrsvMaxRhs] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 8
      for (int k = 0; k < nb; ++k) {
        const double t = tb[k * kOuterNB + r];
#pragma unroll
        for (int c = 0; c < kTrsvMaxRhs; ++c) acc[c] += t * xs[c][s0 + k];
      }
#pragma unroll
      for (int c = 0; c < kTrsvMaxRhs; ++c)
        if (c < m) xs[c][r] -= acc[c];
    }
  }
  __syncthreads();
  for (int e = tid; e < kTrsvMaxRhs * kOuterNB; e += 256) {
    const int c = e / kOuterNB, r = e % kOuterNB;
    if (c < m && r < nbk) X[(long long)c * ldX + r0 + r] = xs[c][r];
  }
}

// The same slab solve on a cluster of 8 CTAs: CTA j owns the slab's 32-row block j and loads its part of the
// slab's T at once (8 CTAs' loads in flight instead of one CTA staging 8 column blocks one after another).
// Step k (k = 0..7 for L, 7..0 for U): CTA k solves its diagonal block (the shuffle chain of slab_trsv_kernel)
// and publishes x_k; after one cluster barrier every CTA still to be solved pulls x_k through DSMEM and
// subtracts T_jk x_k.  Per row the subtractions happen in the same order with the same FMA chains as
// slab_trsv_kernel, so the results are bit-identical.
constexpr int kTrsvCluster = kOuterNB / kLuNB;  // 8
template <bool UPPER>
__global__ void __launch_bounds__(128) slab_trsv_cluster_kernel(const double* T, long long ldT, int r0, int nbk,
                                                                 double* X, long long ldX, int m) {
  extern __shared__ __align__(16) double tb[];  // [kOuterNB columns][kLuNB rows]: this CTA's rows of the slab
  __shared__ double xpub[kTrsvMaxRhs][kLuNB];
  const int j = (int)cluster_ctarank();
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int nblk = (nbk + kLuNB - 1) / kLuNB;
  const int rj0 = j * kLuNB, nbj = max(0, min(kLuNB, nbk - rj0));
  const int c_lo = UPPER ? rj0 : 0, c_hi = UPPER ? nbk : rj0 + nbj;
  if (nbj > 0) {
    for (int e = tid; e < (c_hi - c_lo) * kLuNB; e += blockDim.x) {
      const int c = c_lo + e / kLuNB, rr = e % kLuNB;
      const bool ok = rr < nbj;
      cp_async8(tb + c * kLuNB + rr, ok ? T + (long long)(r0 + c) * ldT + r0 + rj0 + rr : T, ok);
    }
  }
  cp_async_commit();
  double x = (w < m && lane < nbj) ? X[(long long)w * ldX + r0 + rj0 + lane] : 0.0;
  cp_async_wait<0>();
  __syncthreads();
  for (int step = 0; step < nblk; ++step) {
    const int k = UPPER ? nblk - 1 - step : step;
    if (j == k && w < m) {
      const int nb = nbj;
      if (!UPPER) {
        for (int kk = 0; kk < nb; ++kk) {
          const double xk = __shfl_sync(0xffffffffu, x, kk);
          if (lane > kk && lane < nb) x -= tb[(rj0 + kk) * kLuNB + lane] * xk;
        }
      } else {
        const double dinv = lane < nb ? 1.0 / tb[(rj0 + lane) * kLuNB + lane] : 0.0;
        for (int kk = nb - 1; kk >= 0; --kk) {
          if (lane == kk) x *= dinv;
          const double xk = __shfl_sync(0xffffffffu, x, kk);
          if (lane < kk) x -= tb[(rj0 + kk) * kLuNB + lane] * xk;
        }
      }
      xpub[w][lane] = x;
    }
    cluster_sync();
    if ((UPPER ? j < k : j > k) && w < m && nbj > 0) {
      const double xk = dsmem_ld_f64(dsmem_map(&xpub[w][lane], k));  // lane c: x_k[c]
      const int nbk_k = min(kLuNB, nbk - k * kLuNB);
      double acc = 0.0;
      for (int c = 0; c < nbk_k; ++c) {
        const double v = __shfl_sync(0xffffffffu, xk, c);
        acc += tb[(k * kLuNB + c) * kLuNB + lane] * v;
      }
      if (lane < nbj) x -= acc;
    }
  }
  if (w < m && lane < nbj) X[(long long)w * ldX + r0 + rj0 + lane] = x;
  cluster_sync();  // the last step's DSMEM reads are done before any CTA exits
}

// X <- T^-1 X for one matrix (unit-lower L or upper U of an LU), m <= kTrsvMaxRhs
constexpr long long kTrsvScratch = 1LL << 20;  // doubles of split-k partial sums (8 MB)

template <bool UPPER>
cudaError_t trsv_blocked(const double* T, long long ldT, int n, double* X, long long ldX, int m, LuWorkspace& ws,
                         cudaStream_t st) {
  HPS_TRY(ws_grow(ws.trsv, ws.trsv_cap, kTrsvScratch, ws.total));
  double* scratch = ws.trsv;
  const size_t scratch_elems = (size_t)kTrsvScratch;
  const int nouter = (n + kOuterNB - 1) / kOuterNB;
  for (int s = 0; s < nouter; ++s) {
    const int ob = UPPER ? nouter - 1 - s : s;
    const int J = ob * kOuterNB, Jend = std::min(n, J + kOuterNB);
    const size_t smem = (size_t)kLuNB * kOuterNB * sizeof(double);
    static PerDeviceFlag attr;
    const int dv = current_device();
    if (!(attr.set >> dv & 1)) {
      HPS_TRY(cudaFuncSetAttribute(slab_trsv_cluster_kernel<UPPER>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
      attr.set |= 1ull << dv;
    }
#ifndef HPS_TRSV_CLUSTER
#define HPS_TRSV_CLUSTER 1
#endif
    if (!HPS_TRSV_CLUSTER) {  // developer A/B: the one-CTA slab solve
      static PerDeviceFlag attr1;
      if (!(attr1.set >> dv & 1)) {
        HPS_TRY(cudaFuncSetAttribute(slab_trsv_kernel<UPPER>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr1.set |= 1ull << dv;
      }
      slab_trsv_kernel<UPPER><<<1, 256, smem, st>>>(T, ldT, J, Jend - J, X, ldX, m);
      HPS_TRY(cudaGetLastError());
    } else {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(kTrsvCluster);
      cfg.blockDim = dim3(128);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = kTrsvCluster;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      HPS_TRY(cudaLaunchKernelEx(&cfg, slab_trsv_cluster_kernel<UPPER>, T, ldT, J, Jend - J, X, ldX, m));
    }
    GemvArgs g;  // the rows outside the slab: X_rest -= T[rest, J:Jend] X_slab
    g.m = UPPER ? J : n - Jend;
    g.k = Jend - J;
    g.nv = m;
    g.A = T + (long long)J * ldT + (UPPER ? 0 : Jend);
    g.lda = ldT;
    g.x = X + J;
    g.ldx = ldX;
    g.y = X + (UPPER ? 0 : Jend);
    g.ldy = ldX;
    g.alpha = -1.0;
    g.beta = 1.0;
    if (g.m > 0) HPS_TRY(launch_gemv(g, scratch, scratch_elems, st, nullptr));
  }
  return cudaSuccess;
}

cudaError_t bgetrs(int batch, int n, int m, BatchedMat LU, const int* ipiv, BatchedMat R, LuWorkspace& ws,
                   cudaStream_t st) {
  if (batch <= 0 || n <= 0 || m <= 0) return cudaSuccess;
  const int dv = current_device();
  if ((size_t)n * 12 <= 200 * 1024) {
    const int cpc = 8;
    const size_t smem = (size_t)n * 12;
    static PerDeviceFlag smem_set;
    if (smem > smem_set.value[dv] && smem > 48 * 1024) {
      HPS_TRY(cudaFuncSetAttribute(laswp_perm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      smem_set.value[dv] = smem;
    }
    laswp_perm_kernel<<<dim3(batch, (m + cpc - 1) / cpc), 256, smem, st>>>(ipiv, n, R.p, R.ld, R.stride, m, cpc);
    HPS_TRY(cudaGetLastError());
  } else {
    HPS_TRY(ws_grow(ws.perm, ws.perm_cap, (long long)batch * n, ws.total));
    int* perm = ws.perm;
    static PerDeviceFlag attr;
    if (!(attr.set >> dv & 1)) {
      HPS_TRY(cudaFuncSetAttribute(build_perm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      HPS_TRY(cudaFuncSetAttribute(apply_perm_cols_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      attr.set |= 1ull << dv;
    }
    if ((size_t)n * 8 > 227 * 1024) return cudaErrorInvalidValue;
    build_perm_kernel<<<batch, 256, (size_t)n * sizeof(int), st>>>(ipiv, n, perm);
    HPS_TRY(cudaGetLastError());
    apply_perm_cols_kernel<<<dim3(batch, m), 512, (size_t)n * 8, st>>>(perm, n, R.p, R.ld, R.stride, m);
    HPS_TRY(cudaGetLastError());
  }
  const double* L = LU.p;
  if (batch == 1 && m <= kTrsvMaxRhs && n >= 1024) {
    HPS_TRY(trsv_blocked<false>(L, LU.ld, n, R.p, R.ld, m, ws, st));
    return trsv_blocked<true>(L, LU.ld, n, R.p, R.ld, m, ws, st);
  }
  for (int J = 0; J < n; J += kOuterNB) {
    const int Jend = std::min(n, J + kOuterNB);
    if (n >= slab_min_n() && m >= kSlabCW) {
      HPS_TRY(slab_trsm<false>(batch, L, LU.ld, LU.stride, J, Jend - J, R.p, R.ld, R.stride, m, ws, st));
    } else
    for (int j0 = J; j0 < Jend; j0 += kLuNB) {
      const int nb = std::min(kLuNB, Jend - j0);
      Seg seg{R.p, R.ld, R.stride, m, 1};
      HPS_TRY(launch_swap_trsm(batch, n, j0, nb, L, LU.ld, LU.stride, ipiv, &seg, 1, st, /*do_swaps=*/0));
      HPS_TRY(gemm_sub(batch, Jend - j0 - nb, m, nb, -1.0, L + (long long)j0 * LU.ld + j0 + nb, LU.ld, LU.stride,
                       R.p + j0, R.ld, R.stride, R.p + j0 + nb, R.ld, R.stride, st));
    }
    HPS_TRY(gemm_sub(batch, n - Jend, m, Jend - J, -1.0, L + (long long)J * LU.ld + Jend, LU.ld, LU.stride, R.p + J,
                     R.ld, R.stride, R.p + Jend, R.ld, R.stride, st));
  }
  return back_subst(batch, n, m, LU.p, LU.ld, LU.stride, R.p, R.ld, R.stride, ws, st);
}

size_t lu_workspace_need(int batch, int n, int m, bool factor, bool lookahead) {
  LuWorkspace ws;
  ws.lookahead = lookahead;
  size_t total = 0;
  ws.total = &total;
  lu_workspace_reserve(ws, batch, n, m, factor, /*dry=*/true);
  return total;
}

cudaError_t lu_workspace_reserve(LuWorkspace& ws, int batch, int n, int m, bool factor, bool dry) {
  if (batch <= 0 || n <= 0) return cudaSuccess;
  if (n >= kSlabMinN && (m >= kSlabCW || factor))
    HPS_TRY(ws_grow(ws.winv, ws.winv_cap, slab_winv_elems(batch), ws.total, dry));
  if (factor && ws.lookahead && n > kLookaheadMinN && batch > ws.la_cap) {
    long long c1 = ws.la_cap * 4 * kOuterNB, c2 = ws.la_cap;
    HPS_TRY(ws_grow(ws.moved, c1, (long long)batch * 4 * kOuterNB, ws.total, dry));
    HPS_TRY(ws_grow(ws.nmoved, c2, (long long)batch, ws.total, dry));
    ws.la_cap = batch;
  }
  if (!factor && (size_t)n * 12 > 200 * 1024)
    HPS_TRY(ws_grow(ws.perm, ws.perm_cap, (long long)batch * n, ws.total, dry));
  if (batch == 1 && m <= kTrsvMaxRhs && n >= 2 * kOuterNB)
    HPS_TRY(ws_grow(ws.trsv, ws.trsv_cap, kTrsvScratch, ws.total, dry));
  return cudaSuccess;
}

void lu_workspace_free(LuWorkspace& ws) {
  auto fr = [&](void* p, long long cap, size_t el) {
    if (p) cudaFree(p);
    if (ws.total) *ws.total -= (size_t)cap * el;
  };
  fr(ws.winv, ws.winv_cap, 8);
  fr(ws.moved, ws.la_cap * 4 * kOuterNB, 4);
  fr(ws.nmoved, ws.la_cap, 4);
  fr(ws.perm, ws.perm_cap, 4);
  fr(ws.trsv, ws.trsv_cap, 8);
  for (int i = 0; i < ws.n_ev; ++i) cudaEventDestroy(ws.ev[i]);
  delete[] ws.ev;
  if (ws.side) cudaStreamDestroy(ws.side);
  size_t* total = ws.total;
  const bool la = ws.lookahead;
  ws = LuWorkspace{};
  ws.total = total;
  ws.lookahead = la;
}

int lu_launch_count(int n, int m, bool factor) {
  // mirrors bgetrf_aug / bgetrs above (upper bound; zero-size GEMMs are skipped)
  int l = 1;  // stats init | laswp
  for (int J = 0; J < n; J += kOuterNB) {
    const int Jend = std::min(n, J + kOuterNB);
    if (factor)
      for (int j0 = J; j0 < Jend; j0 += panel_width(n)) {
        const int nb = std::min(panel_width(n), Jend - j0);
        l += 2 + (Jend - j0 - nb > 0 ? 1 : 0);
      }
    for (int j0 = J; j0 < Jend; j0 += kLuNB) {
      const int nb = std::min(kLuNB, Jend - j0);
      if (!factor || Jend < n + m) l += 1 + (Jend - j0 - nb > 0 ? 1 : 0);
    }
    if (Jend < n) l += 1;
  }
  if (m > 0)
    for (int r0 = 0; r0 < n; r0 += kOuterNB) {
      const int r1 = std::min(n, r0 + kOuterNB);
      for (int s0 = r0; s0 < r1; s0 += kLuNB) l += 1 + (s0 > r0 ? 1 : 0);
      if (r0 > 0) l += 1;
    }
  return l;
}

}  // namespace hpsk
