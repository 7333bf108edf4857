// gemm_tma.cuh -- the strided-batched DMMA DGEMM of gemm.cuh with its operand tiles staged by
// TMA (cp.async.bulk.tensor) into an mbarrier-tracked ring instead of per-thread cp.async.
//
// Same smem layout as the cp.async kernel, so the DMMA fragment loop is unchanged: the TMA
// boxes are 4 elements taller than the tile (A box (BM+4) x BK, B box (BK+4) x BN), which
// reproduces the conflict-free padded leading dimensions (68 / 20); the extra elements are
// never read (out-of-bounds boxes are zero-filled by the TMA unit, which also handles edges).
// One thread arms each stage's mbarrier with the stage's byte count and issues the two box
// loads; every thread waits on the barrier's phase before using the stage.
#pragma once

#include <cuda.h>

#include "gemm.cuh"

namespace hpsk {

HPS_DEV void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
HPS_DEV void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
HPS_DEV void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
HPS_DEV void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES>
__global__ void __launch_bounds__(GemmCfg<BM, BN, BK, WM, WN, STAGES, true>::kThreads,
                                  GemmCfg<BM, BN, BK, WM, WN, STAGES, true>::kMinBlocks)
    dgemm_tma_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                     const GemmArgs p) {
  using Cfg = GemmCfg<BM, BN, BK, WM, WN, STAGES, true>;
  // TMA destinations need 128-byte alignment: every stage offset is a multiple of 128 bytes
  // (68 x 16 and 64 x 20 doubles), and the barriers sit after the ring
  extern __shared__ __align__(128) double tma_smem[];
  double* sA = tma_smem;
  double* sB = tma_smem + STAGES * Cfg::kStageA;
  uint64_t* bars = reinterpret_cast<uint64_t*>(tma_smem + STAGES * (Cfg::kStageA + Cfg::kStageB));

  const int tiles_m = (p.m + BM - 1) / BM;
  const long long tile = (long long)blockIdx.z * gridDim.y + blockIdx.y;
  if (tile >= (long long)tiles_m * ((p.n + BN - 1) / BN)) return;
  const int tm = int(tile % tiles_m), tn = int(tile / tiles_m);
  const int m0 = tm * BM, n0 = tn * BN;
  const int b = p.bmap ? __ldg(p.bmap + blockIdx.x) : blockIdx.x;
  const int bA = p.sA ? b : 0, bB = p.sB ? b : 0;  // stride-0 operands broadcast over the batch

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % Cfg::kWarpsM, wn = warp / Cfg::kWarpsM;
  const int g = lane >> 2, t4 = lane & 3;
  constexpr unsigned kStageBytes = (Cfg::kStageA + Cfg::kStageB) * sizeof(double);

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  const int ktiles = (p.k + BK - 1) / BK;
  auto issue = [&](int kt) {
    const int s = kt % STAGES;
    mbar_expect_tx(&bars[s], kStageBytes);
    tma_load_3d(sA + s * Cfg::kStageA, &mapA, &bars[s], m0, kt * BK, bA);
    tma_load_3d(sB + s * Cfg::kStageB, &mapB, &bars[s], kt * BK, n0, bB);
  };
  if (tid == 0)
    for (int s = 0; s < STAGES - 1 && s < ktiles; ++s) issue(s);

  const bool seeded = p.k <= p.seed_k_max && (p.alpha == 1.0 || p.alpha == -1.0) && (p.beta == 0.0 || p.beta == 1.0);
  const double asign = seeded ? p.alpha : 1.0;
  double acc[Cfg::TM][Cfg::TN][2];
  const double* Cs = (seeded && p.beta == 1.0) ? p.C + (long long)b * p.sC : nullptr;
#pragma unroll
  for (int i = 0; i < Cfg::TM; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::TN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = m0 + wm * WM + i * 8 + g, col = n0 + wn * WN + j * 8 + t4 * 2 + h;
        acc[i][j][h] = (Cs && row < p.m && col < p.n) ? Cs[(long long)col * p.ldc + row] : 0.0;
      }

  for (int kt = 0; kt < ktiles; ++kt) {
    const int s = kt % STAGES;
    // every thread is done with stage (kt-1) % STAGES before it is refilled for k-tile kt+STAGES-1
    __syncthreads();
    if (tid == 0 && kt + STAGES - 1 < ktiles) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      issue(kt + STAGES - 1);
    }
    mbar_wait(&bars[s], (kt / STAGES) & 1);
    const double* a_w = sA + s * Cfg::kStageA + t4 * Cfg::kLdA + wm * WM + g;
    const double* b_w = sB + s * Cfg::kStageB + (wn * WN + g) * Cfg::kLdB + t4;
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

  const double* C = p.C ? p.C + (long long)b * p.sC : nullptr;
  double* D = p.D + (long long)b * p.sD;
#pragma unroll
  for (int i = 0; i < Cfg::TM; ++i) {
    const int row = m0 + wm * WM + i * 8 + g;
    if (row >= p.m) continue;
#pragma unroll
    for (int j = 0; j < Cfg::TN; ++j)
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

// Launches the TMA variant when every operand satisfies the tensor-map rules (16-byte aligned
// bases, leading dimensions and batch strides multiple of 16 bytes); returns false otherwise.
bool launch_dgemm_tma(const GemmArgs& a, cudaStream_t st, cudaError_t* err);

}  // namespace hpsk
