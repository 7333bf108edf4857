// Microbenchmark: cluster barrier latency vs cluster size and block size (developer tool).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void bar_kernel(long long* out, int iters, int mode) {
  __shared__ double buf[64];
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (mode == 0) {
      asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    } else if (mode == 1) {
      asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;\n" ::: "memory");
    } else {
      __syncthreads();
    }
    if (threadIdx.x == 0) buf[i & 63] = i;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / iters;
}
int main() {
  long long* d; cudaMalloc(&d, 1024 * 8);
  cudaFuncSetAttribute(bar_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int mode = 0; mode < 3; ++mode)
    for (int cs : {1, 2, 4, 8, 16})
      for (int thr : {128, 256, 512}) {
        if (mode == 2 && cs > 1) continue;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs); cfg.blockDim = dim3(thr);
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaLaunchKernelEx(&cfg, bar_kernel, d, 1000, mode);
        cudaEventRecord(e0);
        cudaLaunchKernelEx(&cfg, bar_kernel, d, 10000, mode);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        long long h[16]; cudaMemcpy(h, d, 8 * cs, cudaMemcpyDeviceToHost);
        printf("mode %d (%s) cs %2d thr %3d: %lld cycles/barrier, %.3f us/barrier  err=%s\n", mode,
               mode == 0 ? "release/acquire" : mode == 1 ? "relaxed" : "syncthreads", cs, thr, h[0], ms * 1e3 / 10000,
               cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
