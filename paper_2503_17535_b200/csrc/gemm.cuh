// gemm.cuh -- strided-batched FP64 GEMM on the B200 FP64 tensor cores (DMMA).
//
//   D[b] = alpha * A[b] * B[b] + beta * C[b]      (column-major, b = blockIdx.x)
//
// A is m x k, B is k x n, C/D are m x n; every operand is base + b*stride with
// an explicit leading dimension (stride 0 broadcasts one operand over the
// batch, e.g. the shared leaf operator Q).  Tiles are staged global->shared
// with cp.async (LDGSTS) through a STAGES-deep ring, and each warp issues
// mma.sync.m8n8k4.f64 (DMMA.8x8x4) on register fragments read from shared
// memory with conflict-free padding.  This is the workhorse of every stage:
// the leaf interface products (K4/K6), the Schur updates of the merges
// (K10, proj/src/merge.cpp:294-295), the trailing updates and back-substitution
// blocks of the batched LU (K2/K3/K8/K9), and the multi-RHS downward pass (K11/K13).
#pragma once

#include "common.cuh"

namespace hpsk {

struct GemmArgs {
  int m = 0, n = 0, k = 0, batch = 1;
  const double* A = nullptr;
  long long lda = 0, sA = 0;
  const double* B = nullptr;
  long long ldb = 0, sB = 0;
  const double* C = nullptr;  // may alias D; ignored when beta == 0
  long long ldc = 0, sC = 0;
  double* D = nullptr;
  long long ldd = 0, sD = 0;
  double alpha = 1.0, beta = 0.0;
  int seed_k_max = 0;  // set by launch_dgemm: accumulators seeded with C when k <= this
  const int* drow = nullptr;  // optional output row map: row r of the product goes to D row drow[r] (beta = 0)
  // optional batch map: launch batch i works on batch index bmap[i] (< bmap_extent) of A, B, C and D
  const int* bmap = nullptr;
  int bmap_extent = 0;
};

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool VEC>
struct GemmCfg {
  static constexpr int kWarpsM = BM / WM, kWarpsN = BN / WN;
  static constexpr int kThreads = 32 * kWarpsM * kWarpsN;
  static constexpr int kLdA = BM + 4;  // (BM+4) % 16 == 4 -> conflict-free A fragment loads
  static constexpr int kLdB = BK + 4;  // (BK+4) % 16 == 4 for BK % 16 == 0
  static constexpr int kStageA = BK * kLdA;
  static constexpr int kStageB = BN * kLdB;
  static constexpr int kSmemBytes = STAGES * (kStageA + kStageB) * 8;
  static constexpr int TM = WM / 8, TN = WN / 8;  // DMMA tiles per warp
  // two CTAs per SM when the register budget allows (<= 128 regs/thread at 256 threads)
  static constexpr int kMinBlocks = (kThreads >= 256) ? 1 : 4;
  static_assert(BM % WM == 0 && BN % WN == 0 && WM % 8 == 0 && WN % 8 == 0, "tile shape");
  static_assert(BK % 16 == 0 || BK == 8, "BK");
};

template <class Cfg, int BM, int BN, int BK, bool VEC>
HPS_DEV void gemm_load_stage(double* sA, double* sB, const double* A, long long lda, const double* B, long long ldb,
                             int m0, int n0, int k0, int m, int n, int k, int tid) {
  // A tile: BM rows x BK cols, column-major global -> sA[kk*ldA + mm]
  if (VEC) {
    constexpr int kVecA = BM / 2 * BK;
    for (int e = tid; e < kVecA; e += Cfg::kThreads) {
      const int mm = (e % (BM / 2)) * 2, kk = e / (BM / 2);
      const int gm = m0 + mm, gk = k0 + kk;
      const int valid = (gk < k) ? max(0, min(2, m - gm)) * 8 : 0;
      const double* src = valid ? A + (long long)gk * lda + gm : A;
      cp_async16(sA + kk * Cfg::kLdA + mm, src, valid);
    }
    constexpr int kVecB = BK / 2 * BN;
    for (int e = tid; e < kVecB; e += Cfg::kThreads) {
      const int kk = (e % (BK / 2)) * 2, nn = e / (BK / 2);
      const int gk = k0 + kk, gn = n0 + nn;
      const int valid = (gn < n) ? max(0, min(2, k - gk)) * 8 : 0;
      const double* src = valid ? B + (long long)gn * ldb + gk : B;
      cp_async16(sB + nn * Cfg::kLdB + kk, src, valid);
    }
  } else {
    for (int e = tid; e < BM * BK; e += Cfg::kThreads) {
      const int mm = e % BM, kk = e / BM;
      const int gm = m0 + mm, gk = k0 + kk;
      const bool ok = gm < m && gk < k;
      cp_async8(sA + kk * Cfg::kLdA + mm, ok ? A + (long long)gk * lda + gm : A, ok);
    }
    for (int e = tid; e < BK * BN; e += Cfg::kThreads) {
      const int kk = e % BK, nn = e / BK;
      const int gk = k0 + kk, gn = n0 + nn;
      const bool ok = gk < k && gn < n;
      cp_async8(sB + nn * Cfg::kLdB + kk, ok ? B + (long long)gn * ldb + gk : B, ok);
    }
  }
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool VEC>
__global__ void __launch_bounds__(GemmCfg<BM, BN, BK, WM, WN, STAGES, VEC>::kThreads,
                                  GemmCfg<BM, BN, BK, WM, WN, STAGES, VEC>::kMinBlocks)
    dgemm_dmma_kernel(const GemmArgs p) {
  using Cfg = GemmCfg<BM, BN, BK, WM, WN, STAGES, VEC>;
  extern __shared__ __align__(16) double smem[];
  double* sA = smem;
  double* sB = smem + STAGES * Cfg::kStageA;

  const int tiles_m = (p.m + BM - 1) / BM;
  const long long tile = (long long)blockIdx.z * gridDim.y + blockIdx.y;
  if (tile >= (long long)tiles_m * ((p.n + BN - 1) / BN)) return;
  const int tm = int(tile % tiles_m), tn = int(tile / tiles_m);
  const int m0 = tm * BM, n0 = tn * BN;
  const long long b = p.bmap ? __ldg(p.bmap + blockIdx.x) : blockIdx.x;  // batch in x (gridDim.y/z <= 65535)
  const double* A = p.A + b * p.sA;
  const double* B = p.B + b * p.sB;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % Cfg::kWarpsM, wn = warp / Cfg::kWarpsM;
  const int g = lane >> 2, t4 = lane & 3;

  // alpha = +-1 with beta in {0, 1} (the LU / Schur / solve products): the accumulators are
  // seeded with C up front (its latency hides under the cp.async prologue) and alpha's sign is
  // folded into the A fragments, so the epilogue is a plain store.
  const bool seeded = p.k <= p.seed_k_max && (p.alpha == 1.0 || p.alpha == -1.0) && (p.beta == 0.0 || p.beta == 1.0);
  const double asign = seeded ? p.alpha : 1.0;
  double acc[Cfg::TM][Cfg::TN][2];
  const double* Cs = (seeded && p.beta == 1.0) ? p.C + b * p.sC : nullptr;
#pragma unroll
  for (int i = 0; i < Cfg::TM; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::TN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = m0 + wm * WM + i * 8 + g, col = n0 + wn * WN + j * 8 + t4 * 2 + h;
        acc[i][j][h] = (Cs && row < p.m && col < p.n) ? Cs[(long long)col * p.ldc + row] : 0.0;
      }

  const int ktiles = (p.k + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles)
      gemm_load_stage<Cfg, BM, BN, BK, VEC>(sA + s * Cfg::kStageA, sB + s * Cfg::kStageB, A, p.lda, B, p.ldb, m0, n0,
                                            s * BK, p.m, p.n, p.k, tid);
    cp_async_commit();
  }

  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int pf = kt + STAGES - 1;
    if (pf < ktiles) {
      const int s = pf % STAGES;
      gemm_load_stage<Cfg, BM, BN, BK, VEC>(sA + s * Cfg::kStageA, sB + s * Cfg::kStageB, A, p.lda, B, p.ldb, m0, n0,
                                            pf * BK, p.m, p.n, p.k, tid);
    }
    cp_async_commit();

    const double* a_s = sA + (kt % STAGES) * Cfg::kStageA;
    const double* b_s = sB + (kt % STAGES) * Cfg::kStageB;
    // register double-buffered fragments: loads of k-slice kk+4 overlap the DMMAs of kk
    const double* a_w = a_s + t4 * Cfg::kLdA + wm * WM + g;
    const double* b_w = b_s + (wn * WN + g) * Cfg::kLdB + t4;
    double af[2][Cfg::TM], bf[2][Cfg::TN];
#pragma unroll
    for (int i = 0; i < Cfg::TM; ++i) af[0][i] = asign * a_w[i * 8];
#pragma unroll
    for (int j = 0; j < Cfg::TN; ++j) bf[0][j] = b_w[j * 8 * Cfg::kLdB];
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      const int cur = (kk / 4) & 1;
      if (kk + 4 < BK) {
#pragma unroll
        for (int i = 0; i < Cfg::TM; ++i) af[cur ^ 1][i] = asign * a_w[(kk + 4) * Cfg::kLdA + i * 8];
#pragma unroll
        for (int j = 0; j < Cfg::TN; ++j) bf[cur ^ 1][j] = b_w[j * 8 * Cfg::kLdB + kk + 4];
      }
#pragma unroll
      for (int i = 0; i < Cfg::TM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::TN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[cur][i], bf[cur][j]);
    }
  }
  cp_async_wait<0>();

  // epilogue: D = alpha*acc + beta*C
  const double* C = p.C ? p.C + b * p.sC : nullptr;
  double* D = p.D + b * p.sD;
#pragma unroll
  for (int i = 0; i < Cfg::TM; ++i) {
    const int row = m0 + wm * WM + i * 8 + g;
    if (row >= p.m) continue;
#pragma unroll
    for (int j = 0; j < Cfg::TN; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = n0 + wn * WN + j * 8 + t4 * 2 + h;
        if (col >= p.n) continue;
        double v = acc[i][j][h];
        if (!seeded) {
          v *= p.alpha;
          if (p.beta != 0.0) v += p.beta * C[(long long)col * p.ldc + row];
        }
        D[(long long)col * p.ldd + (p.drow ? __ldg(p.drow + row) : row)] = v;
      }
    }
  }
}

// Host launcher: picks a tile shape from the problem size.
cudaError_t launch_dgemm(const GemmArgs& a, cudaStream_t st);
// live timing of every launch_dgemm (developer/bench instrumentation; see hpsg_dev_gemm_timing)
void gemm_timing_enable(bool on);
bool gemm_timing_read(double* ms, double* flops, long long* launches);

}  // namespace hpsk
