// gemv.cuh -- strided-batched y = alpha * A x + beta * y for 1..4 vectors (see gemv.cu).
#pragma once

#include "common.cuh"

namespace hpsk {

struct GemvArgs {
  int m = 0, k = 0, batch = 1, nv = 1;  // A: m x k column-major; nv right-hand vectors
  const double* A = nullptr;
  long long lda = 0, sA = 0;
  const double* x = nullptr;  // k x nv, column stride ldx
  long long ldx = 0, sx = 0;
  double* y = nullptr;        // m x nv, column stride ldy
  long long ldy = 0, sy = 0;
  double alpha = 1.0, beta = 0.0;
};

// scratch: partial sums for split-k (may be null: no split); `launches` counts kernels issued
cudaError_t launch_gemv(const GemvArgs& a, double* scratch, size_t scratch_elems, cudaStream_t st, int* launches);
size_t gemv_scratch_elems(int m, int k, int batch, int nv);

}  // namespace hpsk
