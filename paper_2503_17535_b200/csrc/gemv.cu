// gemv.cu -- strided-batched FP64 matrix x few-vectors product for the downward pass.
//
// The single-RHS solve (reference propagate/reconstruct_leaf, proj/src/solver.cpp:188-236)
// is a stream over every stored propagation block once: HBM-bound, 0.25 flop/byte.
// A DMMA tile wastes 7/8 of its work (and its loads) on an N=1 product, so for a few
// right-hand sides this kernel streams A column-major with one row per thread
// (coalesced 8-byte loads, 8 independent loads in flight per thread), keeps x in
// shared memory and splits long k ranges over CTAs with an ordered (deterministic)
// second-pass reduction.
#include <algorithm>
#include <cstdlib>

#include "gemv.cuh"

namespace hpsk {

namespace {

constexpr int kRows = 128;     // rows per CTA (one per thread)
constexpr int kKChunk = 1024;  // columns per CTA when k is split

template <int NV>
__global__ void __launch_bounds__(kRows) gemv_kernel(const GemvArgs a, double* partial, int nchunks) {
  __shared__ double xs[NV][kKChunk];
  const long long b = blockIdx.x;
  const int row = blockIdx.y * kRows + threadIdx.x;
  const int chunk = blockIdx.z;
  const int k0 = chunk * kKChunk, k1 = min(a.k, k0 + kKChunk);
  const double* A = a.A + b * a.sA;
  const double* X = a.x + b * a.sx;
  for (int v = 0; v < NV; ++v)  // cp.async: the x chunk's loads all in flight
    for (int kk = threadIdx.x; kk < k1 - k0; kk += kRows) cp_async8(&xs[v][kk], X + (long long)v * a.ldx + k0 + kk, true);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  if (row >= a.m) return;
  double acc[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) acc[v] = 0.0;
  const double* ap = A + (long long)k0 * a.lda + row;
  int kk = 0;
  for (; kk + 8 <= k1 - k0; kk += 8) {
    double t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) t[u] = ap[(long long)(kk + u) * a.lda];
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int v = 0; v < NV; ++v) acc[v] += t[u] * xs[v][kk + u];
  }
  for (; kk < k1 - k0; ++kk) {
    const double t = ap[(long long)kk * a.lda];
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[v] += t * xs[v][kk];
  }
  if (nchunks == 1) {
    double* Y = a.y + b * a.sy;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      double r = a.alpha * acc[v];
      if (a.beta != 0.0) r += a.beta * Y[(long long)v * a.ldy + row];
      Y[(long long)v * a.ldy + row] = r;
    }
  } else {
    // partial[b][chunk][v][row]
#pragma unroll
    for (int v = 0; v < NV; ++v) partial[((b * nchunks + chunk) * NV + v) * (long long)a.m + row] = acc[v];
  }
}

template <int NV>
__global__ void gemv_reduce_kernel(const GemvArgs a, const double* partial, int nchunks) {
  const long long total = (long long)a.batch * a.m * NV;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int row = int(e % a.m);
    const int v = int((e / a.m) % NV);
    const long long b = e / ((long long)a.m * NV);
    double s = 0.0;
    for (int c = 0; c < nchunks; ++c) s += partial[((b * nchunks + c) * NV + v) * (long long)a.m + row];
    double* Y = a.y + b * a.sy;
    double r = a.alpha * s;
    if (a.beta != 0.0) r += a.beta * Y[(long long)v * a.ldy + row];
    Y[(long long)v * a.ldy + row] = r;
  }
}

// Short-k, few-CTA shape (the root substitution's slab updates: m <= 7168 rows, k = 256): one
// row per thread makes every thread walk all k columns in dependent batches of 8 loads, so the
// launch is latency-bound (~29 us whatever m is). Here a CTA covers 32 rows with 16 warps, warp w
// streaming its own contiguous k range (coalesced 256-byte column segments, 16 loads in flight:
// k = 256 is one batch per thread), and the 16 partial sums are added in a fixed order through
// shared memory (deterministic).
constexpr int kWideRows = 32, kWideWarps = 16, kWideU = 16;

template <int NV>
__global__ void __launch_bounds__(kWideRows* kWideWarps) gemv_wide_kernel(const GemvArgs a) {
  __shared__ double part[kWideWarps][NV][kWideRows];
  const long long b = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int row = blockIdx.y * kWideRows + lane;
  const int kc = (a.k + kWideWarps - 1) / kWideWarps;
  const int k0 = min(a.k, warp * kc), k1 = min(a.k, k0 + kc);
  const double* X = a.x + b * a.sx;
  double acc[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) acc[v] = 0.0;
  if (row < a.m) {
    const double* ap = a.A + b * a.sA + row;
    int kk = k0;
    for (; kk + kWideU <= k1; kk += kWideU) {
      double t[kWideU];
#pragma unroll
      for (int u = 0; u < kWideU; ++u) t[u] = __ldg(ap + (long long)(kk + u) * a.lda);
#pragma unroll
      for (int u = 0; u < kWideU; ++u)
#pragma unroll
        for (int v = 0; v < NV; ++v) acc[v] += t[u] * __ldg(X + (long long)v * a.ldx + kk + u);
    }
    for (; kk < k1; ++kk) {
      const double t = __ldg(ap + (long long)kk * a.lda);
#pragma unroll
      for (int v = 0; v < NV; ++v) acc[v] += t * __ldg(X + (long long)v * a.ldx + kk);
    }
  }
#pragma unroll
  for (int v = 0; v < NV; ++v) part[warp][v][lane] = acc[v];
  __syncthreads();
  if (warp < NV && row < a.m) {
    const int v = warp;
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kWideWarps; ++w) s += part[w][v][lane];
    double* Y = a.y + b * a.sy;
    double r = a.alpha * s;
    if (a.beta != 0.0) r += a.beta * Y[(long long)v * a.ldy + row];
    Y[(long long)v * a.ldy + row] = r;
  }
}

template <int NV>
cudaError_t run(const GemvArgs& a, double* scratch, size_t scratch_elems, cudaStream_t st, int* launches) {
  const int row_tiles = (a.m + kRows - 1) / kRows;
  int nchunks = (a.k + kKChunk - 1) / kKChunk;
  // split k only when the grid would otherwise be too small to fill the GPU
  const long long ctas = (long long)a.batch * row_tiles;
  if (ctas < 296 && a.k <= kKChunk && a.k >= 2 * kWideWarps) {
    gemv_wide_kernel<NV><<<dim3(a.batch, (a.m + kWideRows - 1) / kWideRows), kWideRows * kWideWarps, 0, st>>>(a);
    if (launches) ++*launches;
    return cudaGetLastError();
  }
  if (ctas >= 296 || !scratch || (size_t)a.batch * nchunks * NV * a.m > scratch_elems) nchunks = 1;
  if (nchunks == 1 && a.k > kKChunk) {
    // single pass over all of k: loop over chunks inside one CTA
    for (int c0 = 0; c0 < a.k; c0 += kKChunk) {
      GemvArgs s = a;
      s.A = a.A + (long long)c0 * a.lda;
      s.x = a.x + c0;
      s.k = std::min(kKChunk, a.k - c0);
      if (c0 > 0) s.beta = 1.0, s.alpha = a.alpha;
      gemv_kernel<NV><<<dim3(a.batch, row_tiles, 1), kRows, 0, st>>>(s, nullptr, 1);
      if (launches) ++*launches;
    }
    return cudaGetLastError();
  }
  gemv_kernel<NV><<<dim3(a.batch, row_tiles, nchunks), kRows, 0, st>>>(a, scratch, nchunks);
  if (launches) ++*launches;
  if (nchunks > 1) {
    const long long total = (long long)a.batch * a.m * NV;
    gemv_reduce_kernel<NV><<<(unsigned)std::min<long long>((total + 255) / 256, 148 * 16), 256, 0, st>>>(a, scratch,
                                                                                                  nchunks);
    if (launches) ++*launches;
  }
  return cudaGetLastError();
}

}  // namespace

size_t gemv_scratch_elems(int m, int k, int batch, int nv) {
  const int nchunks = (k + kKChunk - 1) / kKChunk;
  return (size_t)batch * nchunks * nv * m;
}

cudaError_t launch_gemv(const GemvArgs& a, double* scratch, size_t scratch_elems, cudaStream_t st, int* launches) {
  if (a.m <= 0 || a.batch <= 0) return cudaSuccess;
  switch (a.nv) {
    case 1: return run<1>(a, scratch, scratch_elems, st, launches);
    case 2: return run<2>(a, scratch, scratch_elems, st, launches);
    case 3: return run<3>(a, scratch, scratch_elems, st, launches);
    case 4: return run<4>(a, scratch, scratch_elems, st, launches);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace hpsk
