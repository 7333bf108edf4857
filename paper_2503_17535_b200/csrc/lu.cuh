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

// per-matrix pivot statistics, 3 doubles: min |u_ii|, max |u_ii|, first zero pivot (-1 if none)
// (proj/src/local_solve.cpp:90-107 check_factorization; proj/src/merge.cpp:281-288)
cudaError_t lu_stats_init(double* stats, int batch, cudaStream_t st);

// Factor the leading n x n block of each M (pivots in ipiv[b*n + i], 0-based rows)
// and, if m > 0, overwrite the m RHS columns M[:, n:n+m] with A^-1 R.
// keep_L = false: the L factor is dead after the augmented solve (merge blocks whose X = D^-1 C is
// all that is kept), so row exchanges skip the L columns of finished outer blocks.
cudaError_t bgetrf_aug(int batch, int n, int m, BatchedMat M, int* ipiv, double* stats, cudaStream_t st,
                       bool keep_L = true);

// Solve with stored factors: R <- A^-1 R for the LU in `LU` (from bgetrf_aug).
cudaError_t bgetrs(int batch, int n, int m, BatchedMat LU, const int* ipiv, BatchedMat R, cudaStream_t st);

// Largest n the panel kernel can handle (cluster limit x rows per CTA).
int bgetrf_max_n();

// kernel launches issued by bgetrf_aug (factor=true) / bgetrs (factor=false)
int lu_launch_count(int n, int m, bool factor);

}  // namespace hpsk
