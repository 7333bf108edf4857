// leaf_fused.cu -- stage 1 (leaf-local solves) as ONE persistent kernel.
//
// Each CTA (16 warps) owns one SM and walks leaves blockIdx.x, +gridDim.x, ...
// For every leaf it runs the whole reference local solve
// (proj/src/local_solve.cpp:111-143 with discretize_operator :44-86) on an
// L2-resident per-CTA workspace W = [L_ii | sgn f_i | -L_ie P] (ni x (ni+1+nb)):
//   A. operator assembly + source sampling (leaf_common.cuh)
//   B. R = -L_ie P                      (block DMMA GEMM, P shared by all leaves)
//   C. blocked right-looking GEPP with the RHS riding along: 32-column panels
//      factored in shared memory (pivot = warp-shuffle argmax, ties -> lowest
//      row, the LAPACK/Eigen rule), composite-permutation row swaps, unit-lower
//      TRSM into a shared U12 tile, DMMA trailing update (A, B in smem)
//   D. blocked back substitution -> [v_i | Y_i]
//   E. [h | T] = Q_i [v_i | Y_i] + [0 | Q_e P]   (T = Q Y, h = Q v; :140-141)
// and writes only [v_i | Y_i] and [h | T] to HBM.  This replaces ~35 batched
// launches whose operands round-tripped through HBM with one launch whose
// working set (~0.4 MB per SM) stays in L2.
#include <cfloat>
#include <climits>

#include "leaf_common.cuh"

namespace hpsk {

namespace {

constexpr int kFT = 512;        // threads per CTA
constexpr int kFW = kFT / 32;   // warps
constexpr int kNB = 32;         // panel width
constexpr int kMaxNI = 208;     // interior points handled by the fused kernel (2D p <= 16)
constexpr int kMaxCols = 256;   // ni + 1 + nb
constexpr int kPLD = kMaxNI + 4;  // panel leading dim: (kPLD % 16) == 4 -> conflict-free A fragments
constexpr int kBLD = kNB + 4;     // U12 / X tile leading dim (k-major), (36 % 16) == 4

struct FusedSmem {
  LeafAsmSmem asmb;
  double pan[kNB * kPLD];       // panel [col][row] (also U_blk during back substitution)
  double tile[kMaxCols * kBLD]; // U12 (k x cols, k-major per column) or X block
  double red[4 * 1024];         // k-split reduction of the [h|T] product (<= 4 32x32 tiles)
  double wv[kFW];
  int wi[kFW];
  int piv[kNB];
  int moved_dst[2 * kNB], moved_src[2 * kNB];
  int n_moved;
  double pmin, pmax;
  int first_zero;
};

// D[m x n] (ldd) = alpha * A[m x k] (lda) * B[k x n] (ldb) + beta * C (ldc); generic pointers
// (shared or global), column-major, 32x32 warp tiles of DMMA.8x8x4 spread over the CTA.
// Fragment loads of one k4 slice (zero outside the matrix).
__device__ __forceinline__ void frag_load(double* af, double* bf, const double* A, int lda, const double* B, int ldb,
                                          int m, int n, int k, int m0, int n0, int kk, int g) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = m0 + i * 8 + g;
    af[i] = (r < m && kk < k) ? A[(long long)kk * lda + r] : 0.0;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int c = n0 + j * 8 + g;
    bf[j] = (c < n && kk < k) ? B[(long long)c * ldb + kk] : 0.0;
  }
}

// D[m x n] (ldd) = alpha * A[m x k] (lda) * B[k x n] (ldb) + beta * C (ldc); generic pointers
// (shared or global), column-major, 32x32 warp tiles of DMMA.8x8x4 spread over the CTA.
// Fragments are register double-buffered so global (L2) operand latency overlaps the DMMAs.
// With fewer tiles than warps and a scratch buffer `red` (>= tiles*1024 doubles of smem), the
// k range is split across warps and reduced with shared-memory atomics.
__device__ void block_dmma(int m, int n, int k, double alpha, const double* A, int lda, const double* B, int ldb,
                           double beta, const double* C, int ldc, double* D, int ldd, double* red = nullptr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int tm_n = (m + 31) / 32, tn_n = (n + 31) / 32, nt = tm_n * tn_n;
  int ks = 1;
  if (red && nt < kFW) ks = min(kFW / nt, (k + 15) / 16);
  const int kchunk = ((k + ks - 1) / ks + 3) / 4 * 4;
  if (ks > 1) {
    for (int e = threadIdx.x; e < nt * 1024; e += kFT) red[e] = 0.0;
    __syncthreads();
  }
  for (int t = warp; t < nt * ks; t += kFW) {
    const int tile = t % nt, z = t / nt;
    const int m0 = (tile % tm_n) * 32, n0 = (tile / tm_n) * 32;
    const int kb = z * kchunk, ke = min(k, kb + kchunk);
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    double af[2][4], bf[2][4];
    if (kb < ke) frag_load(af[0], bf[0], A, lda, B, ldb, m, n, ke, m0, n0, kb + t4, g);
    int cur = 0;
    for (int k0 = kb; k0 < ke; k0 += 4) {
      if (k0 + 4 < ke) frag_load(af[cur ^ 1], bf[cur ^ 1], A, lda, B, ldb, m, n, ke, m0, n0, k0 + 4 + t4, g);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[cur][i], bf[cur][j]);
      cur ^= 1;
    }
    if (ks > 1) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            atomicAdd(&red[tile * 1024 + (j * 8 + t4 * 2 + h) * 32 + i * 8 + g], acc[i][j][h]);
      continue;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = m0 + i * 8 + g;
      if (r >= m) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = n0 + j * 8 + t4 * 2 + h;
          if (c >= n) continue;
          double v = alpha * acc[i][j][h];
          if (beta != 0.0) v += beta * C[(long long)c * ldc + r];
          D[(long long)c * ldd + r] = v;
        }
    }
  }
  if (ks > 1) {
    __syncthreads();
    for (int e = threadIdx.x; e < m * n; e += kFT) {
      const int r = e % m, c = e / m;
      const int tile = (r / 32) + (c / 32) * tm_n;
      double v = alpha * red[tile * 1024 + (c % 32) * 32 + (r % 32)];
      if (beta != 0.0) v += beta * C[(long long)c * ldc + r];
      D[(long long)c * ldd + r] = v;
    }
  }
}

__device__ __forceinline__ void amax_merge(double& v, int& i, double v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) v = v2, i = i2;
}

// GEPP of the panel held in s.pan (rows [0, rows), columns [0, nb)); panel-relative pivots in s.piv.
__device__ void panel_gepp(FusedSmem& s, int rows, int nb, int j0) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int j = 0; j < nb; ++j) {
    double bv = -1.0;
    int bi = INT_MAX;
    for (int r = j + tid; r < rows; r += kFT) amax_merge(bv, bi, fabs(s.pan[j * kPLD + r]), r);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      amax_merge(bv, bi, v2, i2);
    }
    if (lane == 0) s.wv[warp] = bv, s.wi[warp] = bi;
    __syncthreads();
    if (warp == 0) {
      bv = lane < kFW ? s.wv[lane] : -1.0;
      bi = lane < kFW ? s.wi[lane] : INT_MAX;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
        amax_merge(bv, bi, v2, i2);
      }
      if (lane == 0) {
        const int p = bi == INT_MAX ? j : bi;
        s.piv[j] = p;
        const double apv = fabs(s.pan[j * kPLD + p]);
        if (!(apv > 0.0) || !isfinite(apv)) {
          if (s.first_zero < 0) s.first_zero = j0 + j;
        } else {
          s.pmin = fmin(s.pmin, apv);
          s.pmax = fmax(s.pmax, apv);
        }
      }
    }
    __syncthreads();
    const int p = s.piv[j];
    if (p != j)
      for (int c = tid; c < nb; c += kFT) {
        const double t = s.pan[c * kPLD + j];
        s.pan[c * kPLD + j] = s.pan[c * kPLD + p];
        s.pan[c * kPLD + p] = t;
      }
    __syncthreads();
    const double pv = s.pan[j * kPLD + j];
    if (fabs(pv) > 0.0) {
      const double inv = 1.0 / pv;
      for (int r = j + 1 + tid; r < rows; r += kFT) {
        const double l = s.pan[j * kPLD + r] * inv;
        s.pan[j * kPLD + r] = l;
        for (int c = j + 1; c < nb; ++c) s.pan[c * kPLD + r] -= l * s.pan[c * kPLD + j];
      }
    }
    __syncthreads();
  }
}

}  // namespace

__global__ void __launch_bounds__(kFT, 1) leaf_fused_kernel(const LeafFusedArgs f) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FusedSmem& s = *reinterpret_cast<FusedSmem*>(smem_raw);
  const LeafAsmArgs& a = f.a;
  const int ni = a.ni, ne = a.ne, nb = a.nb, ncol = ni + 1 + nb;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* W = f.scratch + (long long)blockIdx.x * f.scratch_stride;  // ni x ncol, ld ni
  double* E = W + (long long)ni * ncol;                               // ni x ne

  for (long long leaf = blockIdx.x; leaf < f.n_leaves; leaf += gridDim.x) {
    // ---- A. assembly
    leaf_assemble_block(a, leaf, W, ni, E, s.asmb);
    if (tid == 0) {
      a.bad_point[leaf] = s.asmb.bad;
      s.pmin = DBL_MAX;
      s.pmax = 0.0;
      s.first_zero = -1;
    }
    __syncthreads();
    // ---- B. R = -L_ie P into W[:, ni+1 : ni+1+nb]
    block_dmma(ni, nb, ne, -1.0, E, ni, f.P, ne, 0.0, nullptr, 0, W + (long long)(ni + 1) * ni, ni);
    __syncthreads();

    // ---- C. blocked GEPP, RHS columns ride along
    for (int j0 = 0; j0 < ni; j0 += kNB) {
      const int pnb = min(kNB, ni - j0), rows = ni - j0;
      for (int e = tid; e < rows * pnb; e += kFT) {
        const int r = e % rows, c = e / rows;
        s.pan[c * kPLD + r] = W[(long long)(j0 + c) * ni + j0 + r];
      }
      __syncthreads();
      panel_gepp(s, rows, pnb, j0);
      for (int e = tid; e < rows * pnb; e += kFT) {
        const int r = e % rows, c = e / rows;
        W[(long long)(j0 + c) * ni + j0 + r] = s.pan[c * kPLD + r];
      }
      // composite permutation of the panel's swaps over rows j0.. (LAPACK laswp order)
      if (tid == 0) {
        int nm = 0;
        // at most 2*pnb rows move; track them through the sequential swaps
        int rid[2 * kNB], src[2 * kNB];
        for (int jj = 0; jj < pnb; ++jj) {
          const int r1 = jj, r2 = s.piv[jj];
          if (r1 == r2) continue;
          int i1 = -1, i2 = -1;
          for (int t = 0; t < nm; ++t) {
            if (rid[t] == r1) i1 = t;
            if (rid[t] == r2) i2 = t;
          }
          if (i1 < 0) rid[nm] = r1, src[nm] = r1, i1 = nm++;
          if (i2 < 0) rid[nm] = r2, src[nm] = r2, i2 = nm++;
          const int t = src[i1];
          src[i1] = src[i2];
          src[i2] = t;
        }
        for (int t = 0; t < nm; ++t) s.moved_dst[t] = j0 + rid[t], s.moved_src[t] = j0 + src[t];
        s.n_moved = nm;
      }
      __syncthreads();
      // apply to all columns outside the panel: every (column, moved row) pair is loaded
      // first (one L2 round trip), then stored -- at most 256 x 64 = 32 pairs per thread
      {
        const int nm = s.n_moved, total = (ncol - pnb) * nm;
        if (total > 0) {
          double vals[32];
#pragma unroll
          for (int u = 0; u < 32; ++u) {
            const int e = tid + u * kFT;
            if (e < total) {
              const int cc = e / nm, mv = e % nm;
              const int c = cc < j0 ? cc : cc + pnb;
              vals[u] = W[(long long)c * ni + s.moved_src[mv]];
            }
          }
          __syncthreads();
#pragma unroll
          for (int u = 0; u < 32; ++u) {
            const int e = tid + u * kFT;
            if (e < total) {
              const int cc = e / nm, mv = e % nm;
              const int c = cc < j0 ? cc : cc + pnb;
              W[(long long)c * ni + s.moved_dst[mv]] = vals[u];
            }
          }
        }
      }
      __syncthreads();
      // U12 = L11^-1 A12 for columns right of the panel -> W and the smem tile (k-major)
      const int rc0 = j0 + pnb, nrc = ncol - rc0;
      for (int c = tid; c < nrc; c += kFT) {
        double* col = W + (long long)(rc0 + c) * ni + j0;
        double v[kNB];
#pragma unroll
        for (int jj = 0; jj < kNB; ++jj) v[jj] = jj < pnb ? col[jj] : 0.0;
#pragma unroll
        for (int jj = 1; jj < kNB; ++jj) {
          double acc = v[jj];
#pragma unroll
          for (int ii = 0; ii < jj; ++ii) acc -= s.pan[ii * kPLD + jj] * v[ii];
          v[jj] = acc;
        }
#pragma unroll
        for (int jj = 0; jj < kNB; ++jj)
          if (jj < pnb) {
            col[jj] = v[jj];
            s.tile[c * kBLD + jj] = v[jj];
          }
      }
      __syncthreads();
      // trailing update W[j0+pnb:, j0+pnb:] -= L21 (smem panel rows pnb..) x U12 (smem tile)
      if (rows > pnb && nrc > 0) {
        double* C = W + (long long)rc0 * ni + j0 + pnb;
        block_dmma(rows - pnb, nrc, pnb, -1.0, s.pan + pnb, kPLD, s.tile, kBLD, 1.0, C, ni, C, ni);
      }
      __syncthreads();
    }

    // ---- D. back substitution on the 1+nb RHS columns
    const int nr = 1 + nb;
    double* R = W + (long long)ni * ni;
    const int nblk = (ni + kNB - 1) / kNB;
    for (int jb = nblk - 1; jb >= 0; --jb) {
      const int r0 = jb * kNB, bnb = min(kNB, ni - r0);
      for (int e = tid; e < bnb * bnb; e += kFT) {
        const int r = e % bnb, c = e / bnb;
        s.pan[c * kPLD + r] = W[(long long)(r0 + c) * ni + r0 + r];
      }
      __syncthreads();
      for (int c = tid; c < nr; c += kFT) {
        double* col = R + (long long)c * ni + r0;
        double v[kNB];
#pragma unroll
        for (int jj = 0; jj < kNB; ++jj) v[jj] = jj < bnb ? col[jj] : 0.0;
#pragma unroll
        for (int jj = kNB - 1; jj >= 0; --jj) {
          if (jj < bnb) {
            double acc = v[jj];
#pragma unroll
            for (int ii = jj + 1; ii < kNB; ++ii)
              if (ii < bnb) acc -= s.pan[ii * kPLD + jj] * v[ii];
            v[jj] = acc / s.pan[jj * kPLD + jj];
          }
        }
#pragma unroll
        for (int jj = 0; jj < kNB; ++jj)
          if (jj < bnb) {
            col[jj] = v[jj];
            s.tile[c * kBLD + jj] = v[jj];
          }
      }
      __syncthreads();
      if (r0 > 0) block_dmma(r0, nr, bnb, -1.0, W + (long long)r0 * ni, ni, s.tile, kBLD, 1.0, R, ni, R, ni);
      __syncthreads();
    }

    // ---- E. [h | T] = Q_i [v | Y_i] + [0 | Q_e P]
    block_dmma(nb, nr, ni, 1.0, f.Qi, nb, R, ni, 1.0, f.ZQeP, nb, f.HT + leaf * f.strideHT, nb,
               ((nb + 31) / 32) * ((nr + 31) / 32) <= 4 ? s.red : nullptr);
    // ---- outputs: [v | Y_i] for the solve, pivot statistics
    double* Yv = f.Yv + leaf * f.strideYv;
    for (int e = tid; e < ni * nr; e += kFT) Yv[e] = R[e];
    if (tid == 0 && f.stats) {
      f.stats[3 * leaf + 0] = s.pmin;
      f.stats[3 * leaf + 1] = s.pmax;
      f.stats[3 * leaf + 2] = s.first_zero;
    }
    __syncthreads();
  }
}

bool leaf_fused_supported(int ni, int nb) { return ni <= kMaxNI && ni + 1 + nb <= kMaxCols; }

long long leaf_fused_scratch_per_cta(int ni, int ne, int nb) { return (long long)ni * (ni + 1 + nb) + (long long)ni * ne; }

cudaError_t launch_leaf_fused(const LeafFusedArgs& f, int grid, cudaStream_t st) {
  const size_t smem = sizeof(FusedSmem);
  static bool set = false;
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(leaf_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    set = true;
  }
  leaf_fused_kernel<<<grid, kFT, smem, st>>>(f);
  return cudaGetLastError();
}

}  // namespace hpsk
