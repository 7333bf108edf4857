// gemm.cu -- tile-shape dispatch for the strided-batched DMMA DGEMM (gemm.cuh).
#include "gemm.cuh"

namespace hpsk {

namespace {
template <int BM, int BN, int BK, int WM, int WN, int ST, bool VEC>
cudaError_t run(const GemmArgs& a, cudaStream_t st) {
  using Cfg = GemmCfg<BM, BN, BK, WM, WN, ST, VEC>;
  auto kern = dgemm_dmma_kernel<BM, BN, BK, WM, WN, ST, VEC>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const long long tiles = (long long)((a.m + BM - 1) / BM) * ((a.n + BN - 1) / BN);
  if (tiles > 65535) return cudaErrorInvalidConfiguration;
  dim3 grid(a.batch, (unsigned)tiles);
  kern<<<grid, Cfg::kThreads, Cfg::kSmemBytes, st>>>(a);
  return cudaGetLastError();
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
}  // namespace

cudaError_t launch_dgemm(const GemmArgs& a, cudaStream_t st) {
  if (a.m <= 0 || a.n <= 0 || a.batch <= 0) return cudaSuccess;
  // k <= 0 runs zero k-tiles: D = beta*C
  const bool vec = aligned16(a.A) && aligned16(a.B) && (a.lda % 2 == 0) && (a.ldb % 2 == 0) &&
                   (a.sA % 2 == 0) && (a.sB % 2 == 0);
  const long long work_tiles_big = (long long)((a.m + 127) / 128) * ((a.n + 127) / 128) * a.batch;
  // Large single/few-matrix products: 128x128 CTA tile, 8 warps of 32x64.
  if (a.m >= 256 && a.n >= 256 && work_tiles_big >= 148) {
    return vec ? run<128, 128, 16, 32, 64, 3, true>(a, st) : run<128, 128, 16, 32, 64, 3, false>(a, st);
  }
  // Everything else (batched small/medium matrices): 64x64 CTA tile, 4 warps of 32x32.
  return vec ? run<64, 64, 16, 32, 32, 3, true>(a, st) : run<64, 64, 16, 32, 32, 3, false>(a, st);
}

}  // namespace hpsk
