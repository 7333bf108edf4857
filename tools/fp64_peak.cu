// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync f64 -> DMMA.8x8x4)
// and DFMA throughput. Writes one JSON line. Used to fill the FP64 roofline
// denominator that MEASURED_PEAKS.json lacks.
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void dmma_loop(double* out, int iters) {
  double acc[NACC][2];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int i = 0; i < NACC; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters) {
  double acc[NACC];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

// DMMA and DFMA issued together: even warps run the DMMA loop, odd warps the DFMA loop (MIX = 0), or every
// warp interleaves both (MIX = 1).  Answers whether the FP64 tensor pipe and the DFMA pipe add up.
template <int MIX>
__global__ void mixed_loop(double* out, int iters) {
  double acc[8][2], f[8];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int i = 0; i < 8; ++i) { acc[i][0] = 0; acc[i][1] = 0; f[i] = i; }
  const bool mma_warp = MIX == 1 || ((threadIdx.x >> 5) & 1) == 0;
  const bool fma_warp = MIX == 1 || ((threadIdx.x >> 5) & 1) == 1;
  for (int it = 0; it < iters; ++it) {
    if (mma_warp) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
    }
    if (fma_warp) {
#pragma unroll
      for (int i = 0; i < 8; ++i) f[i] = fma(f[i], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1] + f[i];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  float best_mma = 1e30f, best_fma = 1e30f;
  int blocks = nsm * 4, threads = 256;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dmma_loop<8><<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r && ms < best_mma) best_mma = ms;
    cudaEventRecord(e0);
    dfma_loop<8><<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (r && ms < best_fma) best_fma = ms;
  }
  float best_mix0 = 1e30f, best_mix1 = 1e30f;
  for (int r = 0; r < 5; ++r) {
    float ms;
    cudaEventRecord(e0);
    mixed_loop<0><<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (r && ms < best_mix0) best_mix0 = ms;
    cudaEventRecord(e0);
    mixed_loop<1><<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (r && ms < best_mix1) best_mix1 = ms;
  }
  double warps = blocks * threads / 32.0;
  // MIX 0: half the warps DMMA, half DFMA; MIX 1: every warp both
  double mix0 = (warps / 2 * iters * 8 * 512.0 + blocks * (double)threads / 2 * iters * 8 * 2.0) / best_mix0 / 1e9;
  double mix1 = (warps * iters * 8 * 512.0 + blocks * (double)threads * iters * 8 * 2.0) / best_mix1 / 1e9;
  printf("{\"mixed_split_warps_tflops\": %.3f, \"mixed_interleaved_tflops\": %.3f}\n", mix0, mix1);
  double mma_flops = warps * iters * 8 * 512.0;
  double fma_flops = blocks * (double)threads * iters * 8 * 2.0;
  printf("{\"sms\": %d, \"dmma_tflops\": %.3f, \"dfma_tflops\": %.3f, \"err\": \"%s\"}\n", nsm,
         mma_flops / best_mma / 1e9, fma_flops / best_fma / 1e9, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
