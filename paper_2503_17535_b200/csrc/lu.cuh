// lu.cuh -- strided-batched LU with partial pivoting and augmented solves (FP64).
//
// Replaces Eigen::PartialPivLU::compute/solve at the reference's three hot
// call sites: the leaf interior factorization (proj/src/local_solve.cpp:125-137),
// the merge interface factorization (proj/src/merge.cpp:280-292) and the
// stored-factor solves (apply_Dinv, proj/src/merge.cpp:156-174).
//
// Blocked right-looking GETRF on M = [A | R] (n x (n+m), column-major):
//   per 32-column panel: (1) panel GEPP in shared memory -- one CTA, or a
//   thread-block cluster of up to 16 CTAs exchanging pivot candidates and
//   pivot rows through distributed shared memory for tall panels;
//   (2) row swaps + unit-lower TRSM of the panel's row block; (3) DMMA GEMM
//   trailing update.  The RHS columns ride along, so after the forward sweep
//   they hold L^-1 P R; a blocked back substitution (upper TRSM + DMMA GEMM)
//   leaves X = A^-1 R in place.  Pivot choice is the same max-|a| rule as
//   LAPACK/Eigen partial pivoting (ties -> lowest row).
#pragma once

#include "common.cuh"

namespace hpsk {

constexpr int kLuNB = 32;

struct BatchedMat {
  double* p = nullptr;      // matrix 0
  long long ld = 0;         // leading dimension
  long long stride = 0;     // elements between consecutive matrices
};

// Device scratch of the batched LU, OWNED BY THE CALLER (the solver context keeps one per context,
// sized at allocation time so its bytes count in hpsg_stats.device_bytes and hpsg_estimate_bytes):
//   winv        : inverses of the 32x32 diagonal blocks of one 256-row slab, batch x 8 x 32 x 32
//                 doubles (slab DMMA substitution, n >= kSlabMinN);
//   moved/nmoved: the look-ahead driver's composite row permutation per outer block (n > 512);
//   perm        : bgetrs row permutation when the LU is too tall for the shared-memory LASWP;
//   trsv        : split-k partial sums of the slab TRSV's streaming GEMV (batch 1, few RHS);
//   side, ev    : the look-ahead panel stream and its events (created on the context's device).
// Growth beyond the reserved sizes is allowed (the bytes are added to *total).
struct LuWorkspace {
  double* winv = nullptr;
  long long winv_cap = 0;  // doubles
  int* moved = nullptr;
  int* nmoved = nullptr;
  long long la_cap = 0;    // matrices
  int* perm = nullptr;
  long long perm_cap = 0;  // ints
  double* trsv = nullptr;
  long long trsv_cap = 0;  // doubles
  cudaStream_t side = nullptr;
  cudaEvent_t* ev = nullptr;
  int n_ev = 0;
  size_t* total = nullptr;  // byte counter of the owner
  bool lookahead = true;    // look-ahead driver for n > 512 (hpsg_options.no_lu_lookahead clears it)
};
// bytes of scratch bgetrf_aug (factor) or bgetrs (!factor) needs for one call shape
size_t lu_workspace_need(int batch, int n, int m, bool factor, bool lookahead = true);
// grow ws to cover one call shape (no-op when it already does); dry = count bytes only
cudaError_t lu_workspace_reserve(LuWorkspace& ws, int batch, int n, int m, bool factor, bool dry = false);
void lu_workspace_free(LuWorkspace& ws);

// per-matrix pivot statistics, 3 doubles: min |u_ii|, max |u_ii|, first zero pivot (-1 if none)
// (proj/src/local_solve.cpp:90-107 check_factorization; proj/src/merge.cpp:281-288)
cudaError_t lu_stats_init(double* stats, int batch, cudaStream_t st);

// Factor the leading n x n block of each M (pivots in ipiv[b*n + i], 0-based rows)
// and, if m > 0, overwrite the m RHS columns M[:, n:n+m] with A^-1 R.
// keep_L = false: the L factor is dead after the augmented solve (merge blocks whose X = D^-1 C is
// all that is kept), so row exchanges skip the L columns of finished outer blocks.
cudaError_t bgetrf_aug(int batch, int n, int m, BatchedMat M, int* ipiv, double* stats, LuWorkspace& ws,
                       cudaStream_t st, bool keep_L = true);

// Solve with stored factors: R <- A^-1 R for the LU in `LU` (from bgetrf_aug).
cudaError_t bgetrs(int batch, int n, int m, BatchedMat LU, const int* ipiv, BatchedMat R, LuWorkspace& ws,
                   cudaStream_t st);

// Largest n the panel kernel can handle (cluster limit x rows per CTA).
int bgetrf_max_n();

// kernel launches issued by bgetrf_aug (factor=true) / bgetrs (factor=false)
int lu_launch_count(int n, int m, bool factor);

}  // namespace hpsk
