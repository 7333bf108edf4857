// common.cuh -- shared device helpers for the B200 (sm_100a) HPS kernels.
//
// FP64 tensor-core math on Blackwell is the legacy mma.sync f64 path (there is
// no tcgen05 kind::f64); ptxas lowers mma.sync.m8n8k4.f64 to DMMA.8x8x4.
// Fragment layout of m8n8k4.f64 (PTX ISA "mma.m8n8k4 .f64"):
//   A (8x4, row)  : a0 = A[lane>>2][lane&3]
//   B (4x8, col)  : b0 = B[lane&3][lane>>2]
//   C (8x8)       : c{0,1} = C[lane>>2][(lane&3)*2 + {0,1}]
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define HPS_DEV __device__ __forceinline__

namespace hpsk {

// Host side: cudaFuncSetAttribute is per device, so one-time attribute flags are kept per device ordinal.
struct PerDeviceFlag {
  unsigned long long set = 0;  // bit d: done on device d
  size_t value[64] = {};       // e.g. the dynamic shared-memory size configured on device d
};
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d & 63;
}

HPS_DEV void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

HPS_DEV uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// cp.async (LDGSTS) with zero-fill when !pred.
HPS_DEV void cp_async8(void* dst, const void* src, bool pred) {
  const int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(sz));
}
HPS_DEV void cp_async16(void* dst, const void* src, int valid_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid_bytes));
}
HPS_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
HPS_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---- thread-block cluster helpers (DSMEM) --------------------------------
HPS_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
HPS_DEV uint32_t cluster_nctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;\n" : "=r"(r));
  return r;
}
HPS_DEV void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// map a local shared address to the same offset in CTA `rank` of the cluster
HPS_DEV uint32_t dsmem_map(const void* local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smem_u32(local)), "r"(rank));
  return r;
}
HPS_DEV double dsmem_ld_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];\n" : "=d"(v) : "r"(addr) : "memory");
  return v;
}
HPS_DEV int dsmem_ld_s32(uint32_t addr) {
  int v;
  asm volatile("ld.shared::cluster.s32 %0, [%1];\n" : "=r"(v) : "r"(addr) : "memory");
  return v;
}

}  // namespace hpsk
