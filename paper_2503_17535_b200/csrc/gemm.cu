// gemm.cu -- tile-shape dispatch for the strided-batched DMMA DGEMM (gemm.cuh).
#include <vector>
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "gemm.cuh"
#include "gemm_tma.cuh"

#include <cudaTypedefs.h>

namespace hpsk {

namespace {
template <int BM, int BN, int BK, int WM, int WN, int ST, bool VEC>
cudaError_t run(const GemmArgs& a, cudaStream_t st) {
  using Cfg = GemmCfg<BM, BN, BK, WM, WN, ST, VEC>;
  auto kern = dgemm_dmma_kernel<BM, BN, BK, WM, WN, ST, VEC>;
  static PerDeviceFlag attr;  // per instantiation and device
  const int dv = current_device();
  if (!(attr.set >> dv & 1)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr.set |= 1ull << dv;
  }
  // tile index = blockIdx.z * gridDim.y + blockIdx.y (gridDim.y/z <= 65535; batch in x)
  const long long tiles = (long long)((a.m + BM - 1) / BM) * ((a.n + BN - 1) / BN);
  const unsigned ty = (unsigned)std::min<long long>(tiles, 65535), tz = (unsigned)((tiles + ty - 1) / ty);
  if (tz > 65535) return cudaErrorInvalidConfiguration;
  dim3 grid(a.batch, ty, tz);
  kern<<<grid, Cfg::kThreads, Cfg::kSmemBytes, st>>>(a);
  return cudaGetLastError();
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
}  // namespace

// CTA tile 64x64, k-step 16, four 32x32 warp tiles, 3-stage pipeline: the measured best of the round-1
// tile sweep (profiles/r01_ncu_summary.md) for every build shape.
template <bool V>
static cudaError_t run_default(const GemmArgs& a, cudaStream_t st) {
  return run<64, 64, 16, 32, 32, 3, V>(a, st);
}

namespace {
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3D map (rows, cols, batch) over a column-major strided batch; box (bx0, bx1, 1)
bool make_map(CUtensorMap* map, const double* base, long long rows, long long cols, long long ld, long long stride,
              int batch, unsigned bx0, unsigned bx1) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (ld * 8) % 16 || ld < rows) return false;
  const long long nb = stride ? batch : 1;
  if (stride && ((stride * 8) % 16 || stride < ld * cols)) return false;
  cuuint64_t dims[3] = {(cuuint64_t)rows, (cuuint64_t)cols, (cuuint64_t)nb};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 8), (cuuint64_t)((stride ? stride : ld * cols) * 8)};
  cuuint32_t box[3] = {bx0, bx1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

template <int BM, int BN, int BK, int WM, int WN, int ST>
bool run_tma(const GemmArgs& a, cudaStream_t st, cudaError_t* err) {
  using Cfg = GemmCfg<BM, BN, BK, WM, WN, ST, true>;
  if (a.k <= 0) return false;
  CUtensorMap mA, mB;
  const int extent = a.bmap ? a.bmap_extent : a.batch;  // the maps span every batch index the launch may touch
  if (!make_map(&mA, a.A, a.m, a.k, a.lda, a.sA, extent, BM + 4, BK)) return false;
  if (!make_map(&mB, a.B, a.k, a.n, a.ldb, a.sB, extent, BK + 4, BN)) return false;
  auto kern = dgemm_tma_kernel<BM, BN, BK, WM, WN, ST>;
  static PerDeviceFlag attr;  // per instantiation and device
  const int dv = current_device();
  if (!(attr.set >> dv & 1)) {
    *err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes + 64);
    if (*err != cudaSuccess) return true;
    attr.set |= 1ull << dv;
  }
  const long long tiles = (long long)((a.m + BM - 1) / BM) * ((a.n + BN - 1) / BN);
  const unsigned ty = (unsigned)std::min<long long>(tiles, 65535), tz = (unsigned)((tiles + ty - 1) / ty);
  if (tz > 65535) return false;
  kern<<<dim3(a.batch, ty, tz), Cfg::kThreads, Cfg::kSmemBytes + 64, st>>>(mA, mB, a);
  *err = cudaGetLastError();
  return true;
}

#ifndef HPS_GEMM_BM
#define HPS_GEMM_BM 64
#endif
#ifndef HPS_GEMM_BN
#define HPS_GEMM_BN 64
#endif
#ifndef HPS_GEMM_BK
#define HPS_GEMM_BK 16
#endif
#ifndef HPS_GEMM_ST
#define HPS_GEMM_ST 3
#endif
bool launch_dgemm_tma(const GemmArgs& a, cudaStream_t st, cudaError_t* err) {
  return run_tma<HPS_GEMM_BM, HPS_GEMM_BN, HPS_GEMM_BK, 32, 32, HPS_GEMM_ST>(a, st, err);
}

// Live GEMM timing (hpsg_dev_gemm_timing): while enabled, every launch is bracketed by CUDA events on
// its own stream and its algorithmic FLOPs (2 m n k per matrix) are recorded; the sums are read after
// the caller synchronises.  Off by default (no events on the product path).
namespace {
struct GemmTimer {
  bool on = false;
  std::vector<cudaEvent_t> ev;
  size_t used = 0;
  double flops = 0.0;
  long long launches = 0;
};
GemmTimer& gemm_timer() {
  static GemmTimer t;
  return t;
}
}  // namespace

void gemm_timing_enable(bool on) {
  GemmTimer& t = gemm_timer();
  t.on = on;
  t.used = 0;
  t.flops = 0.0;
  t.launches = 0;
}

bool gemm_timing_read(double* ms, double* flops, long long* launches) {
  GemmTimer& t = gemm_timer();
  double tot = 0.0;
  for (size_t i = 0; i + 1 < t.used; i += 2) {
    float x = 0.f;
    if (cudaEventElapsedTime(&x, t.ev[i], t.ev[i + 1]) != cudaSuccess) return false;
    tot += x;
  }
  *ms = tot;
  *flops = t.flops;
  *launches = t.launches;
  return true;
}

static cudaError_t launch_dgemm_impl(const GemmArgs& a, cudaStream_t st);

cudaError_t launch_dgemm(const GemmArgs& a, cudaStream_t st) {
  GemmTimer& t = gemm_timer();
  if (!t.on || a.m <= 0 || a.n <= 0 || a.batch <= 0) return launch_dgemm_impl(a, st);
  while (t.ev.size() < t.used + 2) {
    cudaEvent_t e;
    cudaError_t r = cudaEventCreate(&e);
    if (r != cudaSuccess) return r;
    t.ev.push_back(e);
  }
  cudaEventRecord(t.ev[t.used], st);
  const cudaError_t r = launch_dgemm_impl(a, st);
  cudaEventRecord(t.ev[t.used + 1], st);
  t.used += 2;
  t.flops += 2.0 * a.m * a.n * double(a.k) * a.batch;
  ++t.launches;
  return r;
}

static cudaError_t launch_dgemm_impl(const GemmArgs& a, cudaStream_t st) {
  if (a.m <= 0 || a.n <= 0 || a.batch <= 0) return cudaSuccess;
  // k <= 0 runs zero k-tiles: D = beta*C
  const bool vec = aligned16(a.A) && aligned16(a.B) && (a.lda % 2 == 0) && (a.ldb % 2 == 0) &&
                   (a.sA % 2 == 0) && (a.sB % 2 == 0);
  // accumulators seeded with C at every k (measured best inside the build: merges 256 -> 232 ms)
  GemmArgs b = a;
  b.seed_k_max = INT_MAX;
  // TMA-staged operands (same tiles); the cp.async twin when a tensor map is not legal for the operands
  cudaError_t e = cudaSuccess;
  if (launch_dgemm_tma(b, st, &e)) return e;
  return vec ? run_default<true>(b, st) : run_default<false>(b, st);
}

}  // namespace hpsk
