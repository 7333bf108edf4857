// leaf_fused.cu -- stage 1 (leaf-local solves) as ONE persistent kernel.
//
// Two CTAs (8 warps each) per SM walk leaves blockIdx.x, +gridDim.x, ...  For every
// leaf it runs the whole reference local solve (proj/src/local_solve.cpp:111-143
// with discretize_operator :44-86) on an L2-resident per-CTA workspace
// W = [L_ii | sgn f_i | -L_ie P] (ni x (ni+1+nb)), keeping every DMMA operand in
// shared memory:
//   A. operator assembly + source sampling (leaf_common.cuh, sparse grid lines);
//      the 2*dim exterior neighbours of each interior row go to a shared list
//   B. R = -L_ie P from that list (4 nonzeros per row in 2D instead of a dense GEMM)
//   C. blocked GEPP with the RHS riding along.  Per 32-column panel staged in shared
//      memory, warp 0 factors 8-column sub-panels (pivot = exact warp argmax on the
//      IEEE bits via REDUX, ties -> lowest current row, the LAPACK/Eigen rule; rows
//      exchanged across the whole panel) and all warps apply each sub-panel's TRSM
//      and k = 8 DMMA update; then one composite-permutation row exchange of the
//      other columns, unit-lower TRSM of U12, DMMA trailing update with L21 and U12
//      in shared memory (accumulators seeded from W)
//   D. blocked back substitution (U blocks staged in shared memory) -> [v_i | Y_i]
//   E. [h | T] = Q_i [v_i | Y_i] + [0 | Q_e P] over shared k-chunks, 8x8 DMMA
//      tiles distributed over all warps (T = Q Y, h = Q v; :140-141)
// Only [v_i | Y_i] and [h | T] reach HBM.
#include <cfloat>
#include <climits>

#include "leaf_common.cuh"

namespace hpsk {

namespace {

#ifndef HPS_LEAF_FT
#define HPS_LEAF_FT 256
#endif
constexpr int kFT = HPS_LEAF_FT;  // threads per CTA (256: two CTAs per SM)
constexpr int kFW = kFT / 32;     // warps
constexpr int kNB = 32;           // panel width / k chunk
constexpr int kMaxNI = 196;       // interior points (2D p <= 16)
constexpr int kMaxCols = 256;     // ni + 1 + nb
constexpr int kPLD = 196;         // A-operand leading dim: (kPLD % 16) == 4 -> conflict-free fragments
constexpr int kBLD = kNB + 4;     // B-operand (k-major) leading dim, (36 % 16) == 4
constexpr int kTileCols = 128;    // B-operand columns staged at a time
constexpr int kMaxNz = kMaxNI * 4;
constexpr int kRowsPerLane = (kMaxNI + 31) / 32;
#ifndef HPS_LEAF_SUB
#define HPS_LEAF_SUB 8
#endif
constexpr int kSub = HPS_LEAF_SUB;  // sub-panel width factored by one warp inside a panel
static_assert(kSub % 4 == 0, "sub-panel width: multiple of 4 (register GEPP write-back rounds)");
#ifndef HPS_LEAF_PAIR
#define HPS_LEAF_PAIR 1
#endif
constexpr bool kPairGepp = HPS_LEAF_PAIR;  // two-warp sub-panel GEPP for panels taller than 64 rows
#ifndef HPS_LEAF_REG_GEPP
#define HPS_LEAF_REG_GEPP 0  // 1: register-resident sub-panel (gepp_pair_regs): bit-identical, but measured
                             // slower at the 128-register cap (leaf 104.6 -> 120.6 ms, spills); kept for study
#endif

struct FusedSmem {
  LeafAsmSmemT<256, 16> asmb;
  double pan[kNB * kPLD];         // A operand: factored panel / U column block / Q_i chunk;
                                  // exterior-neighbour list during phases A-B
  double tile[kTileCols * kBLD];  // B operand: U12 chunk / X block / [v|Y] chunk; P during phase B
  double urow[kNB];
  double cv[kFW];
  int cp[kFW], ct[kFW];
  double rdiag[kNB];
  int prow[kMaxNI];
  int moved_dst[kMaxNI], moved_src[kMaxNI];
  int n_moved;
  double pmin, pmax;
  int first_zero;
};

// C[m x n] (global, ldc) = C - A[m x k] (smem, lda) * B[k x n] (smem, k-major ldb), k <= 32,
// (8 UM) x (8 UN) warp tiles; the accumulators are seeded with C so its load overlaps the fragment
// loads, and the fragments are double-buffered in registers (the loads of k-slice k0+4 are in
// flight while the DMMAs of k0 issue).
#ifndef HPS_LEAF_UM
#define HPS_LEAF_UM 4
#endif
#ifndef HPS_LEAF_UN
#define HPS_LEAF_UN 2
#endif
__device__ void update_smem(int m, int n, int k, const double* A, int lda, const double* B, int ldb, double* C,
                            int ldc) {
  constexpr int UM = HPS_LEAF_UM, UN = HPS_LEAF_UN;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int tm_n = (m + 8 * UM - 1) / (8 * UM), tn_n = (n + 8 * UN - 1) / (8 * UN);
  for (int t = warp; t < tm_n * tn_n; t += kFW) {
    const int m0 = (t % tm_n) * 8 * UM, n0 = (t / tm_n) * 8 * UN;
    double acc[UM][UN][2];
#pragma unroll
    for (int i = 0; i < UM; ++i)
#pragma unroll
      for (int j = 0; j < UN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = m0 + i * 8 + g, c = n0 + j * 8 + t4 * 2 + h;
          acc[i][j][h] = (r < m && c < n) ? C[(long long)c * ldc + r] : 0.0;
        }
    double af[2][UM], bf[2][UN];
#pragma unroll
    for (int i = 0; i < UM; ++i) af[0][i] = t4 < k ? -A[t4 * lda + m0 + i * 8 + g] : 0.0;
#pragma unroll
    for (int j = 0; j < UN; ++j) bf[0][j] = t4 < k ? B[(n0 + j * 8 + g) * ldb + t4] : 0.0;
#pragma unroll
    for (int k0 = 0; k0 < kNB; k0 += 4) {
      const int cur = (k0 / 4) & 1;
      if (k0 >= k) break;
      if (k0 + 4 < kNB) {
        const int kk = k0 + 4 + t4;
#pragma unroll
        for (int i = 0; i < UM; ++i) af[cur ^ 1][i] = kk < k ? -A[kk * lda + m0 + i * 8 + g] : 0.0;
#pragma unroll
        for (int j = 0; j < UN; ++j) bf[cur ^ 1][j] = kk < k ? B[(n0 + j * 8 + g) * ldb + kk] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < UM; ++i)
#pragma unroll
        for (int j = 0; j < UN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[cur][i], bf[cur][j]);
    }
#pragma unroll
    for (int i = 0; i < UM; ++i)
#pragma unroll
      for (int j = 0; j < UN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = m0 + i * 8 + g, c = n0 + j * 8 + t4 * 2 + h;
          if (r < m && c < n) C[(long long)c * ldc + r] = acc[i][j][h];
        }
  }
}

// One warp factors the rows x pnb panel in s.pan.  Lane-strided rows r = j + 1 + lane + 32 q; the
// slots past the last row are clamped onto it, so loads/stores need no predicates (the clamped
// lanes recompute and store exactly the owner's value).
// 1/x to full double precision (within 1 ulp) from the hardware approximation and two Newton steps:
// four dependent FMAs instead of the IEEE division subroutine on the pivot chain
#ifndef HPS_LEAF_FAST_RCP
#define HPS_LEAF_FAST_RCP 1
#endif
HPS_DEV double pivot_rcp(double x) {
#if HPS_LEAF_FAST_RCP
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
#else
  return 1.0 / x;
#endif
}

template <int NQ>
__device__ __forceinline__ void gepp_warp_body(FusedSmem& s, int rows, int sb, int se, int pnb, int j0) {
  const int lane = threadIdx.x & 31;
  double pmn = s.pmin, pmx = s.pmax;
  int fz = s.first_zero;
  for (int j = sb; j < se; ++j) {
    double* pj = s.pan + j * kPLD;
    double bv = -1.0;
    int bp = INT_MAX;
    {
      double a[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) a[q] = fabs(pj[min(j + lane + 32 * q, rows - 1)]);
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const double av = isnan(a[q]) ? INFINITY : a[q];
        if (j + lane + 32 * q < rows && av > bv) bv = av, bp = j + lane + 32 * q;
      }
    }
    {
      // warp argmax on the IEEE bits (non-negative doubles order as unsigned integers):
      // max of the high words, max of the low words among those, then the lowest row
      const unsigned long long key = bv >= 0.0 ? (unsigned long long)__double_as_longlong(bv) : 0ull;
      const unsigned hi = unsigned(key >> 32), lo = unsigned(key);
      const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
      const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
      bp = __reduce_min_sync(0xffffffffu, (hi == mh && lo == ml) ? bp : INT_MAX);
      bv = __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
    }
    if (bp != j) {
      if (lane < pnb) {
        const double t = s.pan[lane * kPLD + j];
        s.pan[lane * kPLD + j] = s.pan[lane * kPLD + bp];
        s.pan[lane * kPLD + bp] = t;
      }
      if (lane == 0) {
        const int t = s.prow[j];
        s.prow[j] = s.prow[bp];
        s.prow[bp] = t;
      }
    }
    // pivot statistics in registers (bv is warp-uniform), flushed once after the sub-panel
    if (!(bv > 0.0) || !isfinite(bv)) {
      if (fz < 0) fz = j0 + j;
    } else {
      pmn = fmin(pmn, bv);
      pmx = fmax(pmx, bv);
    }
    __syncwarp();
    const double pv = pj[j];
    if (fabs(pv) > 0.0 && j + 1 < rows) {
      const double rinv = pivot_rcp(pv);
      int off[NQ];
      double l[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) off[q] = min(j + 1 + lane + 32 * q, rows - 1);
#pragma unroll
      for (int q = 0; q < NQ; ++q) l[q] = pj[off[q]] * rinv;
      __syncwarp();
#pragma unroll
      for (int q = 0; q < NQ; ++q) pj[off[q]] = l[q];
      // rank-1 update, four columns at a time (4*NQ loads in flight per lane)
      int c = j + 1;
      for (; c + 4 <= se; c += 4) {
        const double* pc = s.pan + c * kPLD;
        double u[4], a[4][NQ];
#pragma unroll
        for (int k = 0; k < 4; ++k) u[k] = pc[k * kPLD + j];
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int q = 0; q < NQ; ++q) a[k][q] = pc[k * kPLD + off[q]];
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int q = 0; q < NQ; ++q) s.pan[(c + k) * kPLD + off[q]] = a[k][q] - l[q] * u[k];
      }
      for (; c < se; ++c) {
        double* pc = s.pan + c * kPLD;
        const double u = pc[j];
        double a[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) a[q] = pc[off[q]];
        __syncwarp();
#pragma unroll
        for (int q = 0; q < NQ; ++q) pc[off[q]] = a[q] - l[q] * u;
      }
    }
    __syncwarp();
  }
  if (lane == 0) s.pmin = pmn, s.pmax = pmx, s.first_zero = fz;
}

// Two-warp variant of gepp_warp_body for tall panels: warp w (0 or 1) owns the lane-strided row
// slots q = 2 qq + w, so each warp's pivot search and rank-1 update cover half the rows; per column
// the two warp candidates meet through shared memory under a 64-thread named barrier, warp 0
// exchanges the rows, a second named barrier publishes the exchange.  Stores are predicated (no
// clamped duplicates: a duplicate in the other warp would race with the owner).  Same pivot rule and
// arithmetic as gepp_warp_body.
HPS_DEV void pair_bar() { asm volatile("bar.sync 1, 64;\n" ::: "memory"); }
template <int NQH>
__device__ __forceinline__ void gepp_pair_body(FusedSmem& s, int rows, int sb, int se, int pnb, int j0) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double pmn = s.pmin, pmx = s.pmax;
  int fz = s.first_zero;
  for (int j = sb; j < se; ++j) {
    double* pj = s.pan + j * kPLD;
    double bv = -1.0;
    int bp = INT_MAX;
    {
      double a[NQH];
#pragma unroll
      for (int qq = 0; qq < NQH; ++qq) a[qq] = fabs(pj[min(j + lane + 32 * (2 * qq + w), rows - 1)]);
#pragma unroll
      for (int qq = 0; qq < NQH; ++qq) {
        const int r = j + lane + 32 * (2 * qq + w);
        const double av = isnan(a[qq]) ? INFINITY : a[qq];
        if (r < rows && av > bv) bv = av, bp = r;
      }
    }
    {
      const unsigned long long key = bv >= 0.0 ? (unsigned long long)__double_as_longlong(bv) : 0ull;
      const unsigned hi = unsigned(key >> 32), lo = unsigned(key);
      const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
      const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
      bp = __reduce_min_sync(0xffffffffu, (hi == mh && lo == ml) ? bp : INT_MAX);
      bv = bp == INT_MAX ? -1.0 : __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
    }
    if (lane == 0) s.cv[w] = bv, s.cp[w] = bp;
    pair_bar();
    {
      const double ov = s.cv[w ^ 1];
      const int op = s.cp[w ^ 1];
      if (ov > bv || (ov == bv && op < bp)) bv = ov, bp = op;
    }
    if (w == 0 && bp != j) {
      if (lane < pnb) {
        const double t = s.pan[lane * kPLD + j];
        s.pan[lane * kPLD + j] = s.pan[lane * kPLD + bp];
        s.pan[lane * kPLD + bp] = t;
      }
      if (lane == 0) {
        const int t = s.prow[j];
        s.prow[j] = s.prow[bp];
        s.prow[bp] = t;
      }
    }
    if (!(bv > 0.0) || !isfinite(bv)) {
      if (fz < 0) fz = j0 + j;
    } else {
      pmn = fmin(pmn, bv);
      pmx = fmax(pmx, bv);
    }
    pair_bar();
    const double pv = pj[j];
    if (fabs(pv) > 0.0 && j + 1 < rows) {
      const double rinv = pivot_rcp(pv);
      int off[NQH];
      bool own[NQH];
      double l[NQH];
#pragma unroll
      for (int qq = 0; qq < NQH; ++qq) {
        const int r = j + 1 + lane + 32 * (2 * qq + w);
        own[qq] = r < rows;
        off[qq] = min(r, rows - 1);
      }
#pragma unroll
      for (int qq = 0; qq < NQH; ++qq) l[qq] = pj[off[qq]] * rinv;
#pragma unroll
      for (int qq = 0; qq < NQH; ++qq)
        if (own[qq]) pj[off[qq]] = l[qq];
      int c = j + 1;
      for (; c + 4 <= se; c += 4) {
        const double* pc = s.pan + c * kPLD;
        double u[4], a[4][NQH];
#pragma unroll
        for (int k = 0; k < 4; ++k) u[k] = pc[k * kPLD + j];
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int qq = 0; qq < NQH; ++qq) a[k][qq] = pc[k * kPLD + off[qq]];
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int qq = 0; qq < NQH; ++qq)
            if (own[qq]) s.pan[(c + k) * kPLD + off[qq]] = a[k][qq] - l[qq] * u[k];
      }
      for (; c < se; ++c) {
        double* pc = s.pan + c * kPLD;
        const double u = pc[j];
        double a[NQH];
#pragma unroll
        for (int qq = 0; qq < NQH; ++qq) a[qq] = pc[off[qq]];
#pragma unroll
        for (int qq = 0; qq < NQH; ++qq)
          if (own[qq]) pc[off[qq]] = a[qq] - l[qq] * u;
      }
    }
    __syncwarp();
  }
  if (threadIdx.x == 0) s.pmin = pmn, s.pmax = pmx, s.first_zero = fz;
}

// Register-resident two-warp sub-panel GEPP (same pivot rule and arithmetic as gepp_pair_body): the
// sub-panel's rows live in registers (warp w owns the lane-strided row slots 2 qq + w) and are never
// moved between threads during the elimination -- each slot carries its current row position, a pivot
// exchange only swaps two positions, and the pivot row reaches the other slots through an 8-value shared
// broadcast.  The composite row permutation is applied to the panel's other columns once at the end.
// Per column: two 64-thread named barriers and no shared-memory streaming of the sub-panel.
template <int NQH>
__device__ __forceinline__ void gepp_pair_regs(FusedSmem& s, int rows, int sb, int se, int pnb, int j0) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int ncs = se - sb;
  double v[NQH][kSub];
  int pos[NQH], org[NQH];
  bool act[NQH];  // valid and not yet a pivot
#pragma unroll
  for (int qq = 0; qq < NQH; ++qq) {
    const int r = sb + lane + 32 * (2 * qq + w);
    act[qq] = r < rows;
    pos[qq] = r;
    const int rr = min(r, rows - 1);
    org[qq] = s.prow[rr];
#pragma unroll
    for (int c = 0; c < kSub; ++c) v[qq][c] = c < ncs ? s.pan[(sb + c) * kPLD + rr] : 0.0;
  }
  double pmn = s.pmin, pmx = s.pmax;
  int fz = s.first_zero;
#pragma unroll
  for (int jj = 0; jj < kSub; ++jj) {
    if (jj < ncs) {  // (no break: the loop must unroll so v[][jj] stays in registers)
    const int j = sb + jj;
    double bv = -1.0;
    int bp = INT_MAX;
#pragma unroll
    for (int qq = 0; qq < NQH; ++qq) {
      const double a = fabs(v[qq][jj]);
      const double av = isnan(a) ? INFINITY : a;
      if (act[qq] && (av > bv || (av == bv && pos[qq] < bp))) bv = av, bp = pos[qq];
    }
    {
      const unsigned long long key = bv >= 0.0 ? (unsigned long long)__double_as_longlong(bv) : 0ull;
      const unsigned hi = unsigned(key >> 32), lo = unsigned(key);
      const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
      const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
      bp = __reduce_min_sync(0xffffffffu, (hi == mh && lo == ml) ? bp : INT_MAX);
      bv = bp == INT_MAX ? -1.0 : __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
    }
    if (lane == 0) s.cv[w] = bv, s.cp[w] = bp;
    pair_bar();
    {
      const double ov = s.cv[w ^ 1];
      const int op = s.cp[w ^ 1];
      if (ov > bv || (ov == bv && op < bp)) bv = ov, bp = op;
    }
    if (!(bv > 0.0) || !isfinite(bv)) {
      if (fz < 0) fz = j0 + j;
    } else {
      pmn = fmin(pmn, bv);
      pmx = fmax(pmx, bv);
    }
    // the pivot slot publishes its row; positions j and bp trade places
#pragma unroll
    for (int qq = 0; qq < NQH; ++qq) {
      if (act[qq] && pos[qq] == bp) {
#pragma unroll
        for (int c = 0; c < kSub; ++c)
          if (c >= jj) s.urow[c] = v[qq][c];
      }
    }
#pragma unroll
    for (int qq = 0; qq < NQH; ++qq) {
      const int pq = pos[qq];
      pos[qq] = pq == j ? bp : (pq == bp ? j : pq);
      if (pos[qq] == j) act[qq] = false;  // the pivot slot now holds row j
    }
    pair_bar();
    const double pv = s.urow[jj];
    if (fabs(pv) > 0.0) {
      const double rinv = pivot_rcp(pv);
      double u[kSub];
#pragma unroll
      for (int c = 0; c < kSub; ++c) u[c] = c > jj && c < ncs ? s.urow[c] : 0.0;
#pragma unroll
      for (int qq = 0; qq < NQH; ++qq) {
        if (act[qq]) {
          const double l = v[qq][jj] * rinv;
          v[qq][jj] = l;
#pragma unroll
          for (int c = 0; c < kSub; ++c)
            if (c > jj) v[qq][c] -= l * u[c];
        }
      }
    }
    }
  }
  // write back: the sub-panel from registers; the panel's other columns get the same row permutation,
  // four columns per round (read all, barrier, write all, barrier)
#pragma unroll
  for (int qq = 0; qq < NQH; ++qq) {
    const int r = sb + lane + 32 * (2 * qq + w);
    if (r < rows) s.prow[pos[qq]] = org[qq];
  }
  for (int c0 = 0; c0 < pnb; c0 += 4) {
    if (c0 + 4 > sb && c0 < se) continue;  // sub-panel columns (kSub is a multiple of 4)
    double t[NQH][4];
#pragma unroll
    for (int qq = 0; qq < NQH; ++qq) {
      const int r = min(sb + lane + 32 * (2 * qq + w), rows - 1);
#pragma unroll
      for (int k = 0; k < 4; ++k) t[qq][k] = c0 + k < pnb ? s.pan[(c0 + k) * kPLD + r] : 0.0;
    }
    pair_bar();
#pragma unroll
    for (int qq = 0; qq < NQH; ++qq) {
      if (sb + lane + 32 * (2 * qq + w) < rows) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (c0 + k < pnb) s.pan[(c0 + k) * kPLD + pos[qq]] = t[qq][k];
      }
    }
    pair_bar();
  }
#pragma unroll
  for (int qq = 0; qq < NQH; ++qq) {
    if (sb + lane + 32 * (2 * qq + w) < rows) {
#pragma unroll
      for (int c = 0; c < kSub; ++c)
        if (c < ncs) s.pan[(sb + c) * kPLD + pos[qq]] = v[qq][c];
    }
  }
  if (threadIdx.x == 0) s.pmin = pmn, s.pmax = pmx, s.first_zero = fz;
}

// GEPP of panel columns [j0, j0+pnb) over rows [j0, ni) of W by ONE warp on the panel staged in
// s.pan (rows physically exchanged; lane-strided rows, no CTA barrier per column).  Pivot = max
// |a| with NaN ranked as +inf, ties -> lowest current row (the LAPACK/Eigen rule).  Writes the
// factored panel back to W and fills the moved-row list for the other columns.
__device__ void panel_gepp_warp(FusedSmem& s, double* W, int ni, int j0, int pnb, long long* prof = nullptr) {
  const int tid = threadIdx.x;
  long long t0 = prof ? clock64() : 0;
  auto tick = [&](int k) {
    if (prof) {
      const long long t = clock64();
      prof[k] += t - t0;
      t0 = t;
    }
  };
  const int rows = ni - j0;
  if (tid < rows) {  // thread = row (rows <= 196 < kFT); cp.async keeps all pnb loads in flight
    const double* src = W + (long long)j0 * ni + j0 + tid;
    for (int c = 0; c < pnb; ++c) cp_async8(s.pan + c * kPLD + tid, src + (long long)c * ni, true);
  }
  cp_async_commit();
  cp_async_wait<0>();
  for (int r = tid; r < rows; r += kFT) s.prow[r] = r;
  __syncthreads();
  tick(40);
  // kSub-column sub-panels: warp 0 factors one (swaps span the whole panel), then all warps apply
  // its L11^-1 to the sub-panel's rows of the later panel columns and the k <= kSub DMMA update
  const int nq = (rows + 31) / 32;
  for (int sb = 0; sb < pnb; sb += kSub) {
    const int se = min(sb + kSub, pnb);
    if (kPairGepp && nq >= 3) {
      if (tid < 64) {
#if HPS_LEAF_REG_GEPP
        switch (nq) {
          case 3: case 4: gepp_pair_regs<2>(s, rows, sb, se, pnb, j0); break;
          case 5: case 6: gepp_pair_regs<3>(s, rows, sb, se, pnb, j0); break;
          default: gepp_pair_regs<(kRowsPerLane + 1) / 2>(s, rows, sb, se, pnb, j0); break;
        }
#else
        switch (nq) {
          case 3: case 4: gepp_pair_body<2>(s, rows, sb, se, pnb, j0); break;
          case 5: case 6: gepp_pair_body<3>(s, rows, sb, se, pnb, j0); break;
          default: gepp_pair_body<(kRowsPerLane + 1) / 2>(s, rows, sb, se, pnb, j0); break;
        }
#endif
      }
    } else if (tid < 32) {
      switch (nq) {
        case 1: gepp_warp_body<1>(s, rows, sb, se, pnb, j0); break;
        case 2: gepp_warp_body<2>(s, rows, sb, se, pnb, j0); break;
        case 3: gepp_warp_body<3>(s, rows, sb, se, pnb, j0); break;
        case 4: gepp_warp_body<4>(s, rows, sb, se, pnb, j0); break;
        case 5: gepp_warp_body<5>(s, rows, sb, se, pnb, j0); break;
        case 6: gepp_warp_body<6>(s, rows, sb, se, pnb, j0); break;
        default: gepp_warp_body<kRowsPerLane>(s, rows, sb, se, pnb, j0); break;
      }
    }
    __syncthreads();
    tick(41);
    if (se >= pnb) break;
    // U12 rows [sb, se) of columns [se, pnb): unit-lower forward substitution
    for (int c = se + tid; c < pnb; c += kFT) {
      double* pc = s.pan + c * kPLD;
      double x[kSub];
#pragma unroll
      for (int i = 0; i < kSub; ++i) x[i] = sb + i < se ? pc[sb + i] : 0.0;
#pragma unroll
      for (int k = 0; k < kSub - 1; ++k)
#pragma unroll
        for (int i = k + 1; i < kSub; ++i) x[i] -= s.pan[(sb + k) * kPLD + sb + i] * x[k];
#pragma unroll
      for (int i = 0; i < kSub; ++i)
        if (sb + i < se) pc[sb + i] = x[i];
    }
    __syncthreads();
    tick(42);
    // rows [se, rows) x columns [se, pnb) -= L21 (k = se - sb) * U12: 8x8 DMMA tiles over all warps
    {
      const int lane = tid & 31, g = lane >> 2, t4 = lane & 3;
      const int tr = (rows - se + 7) / 8, tc = (pnb - se + 7) / 8;
      for (int t = tid >> 5; t < tr * tc; t += kFW) {
        const int r0 = se + (t % tr) * 8, c0 = se + (t / tr) * 8;
        const int r = r0 + g;
        double acc[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int cc = c0 + 2 * t4 + h;
          acc[h] = (r < rows && cc < pnb) ? s.pan[cc * kPLD + r] : 0.0;
        }
#pragma unroll
        for (int kb = 0; kb < kSub; kb += 4) {
          const int k = sb + kb + t4;
          const double av = (k < se && r < rows) ? -s.pan[k * kPLD + r] : 0.0;
          const double bv = (k < se && c0 + g < pnb) ? s.pan[(c0 + g) * kPLD + k] : 0.0;
          dmma_8x8x4(acc[0], acc[1], av, bv);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int cc = c0 + 2 * t4 + h;
          if (r < rows && cc < pnb) s.pan[cc * kPLD + r] = acc[h];
        }
      }
    }
    __syncthreads();
    tick(43);
  }
  if (tid == 0) s.n_moved = 0;
  __syncthreads();
  // only the U11 block goes back: L21 lives on in s.pan for the trailing update and is dead after
  for (int e = tid; e < pnb * pnb; e += kFT) {
    const int c = e / pnb, r = e - c * pnb;
    W[(long long)(j0 + c) * ni + j0 + r] = s.pan[c * kPLD + r];
  }
  for (int r = tid; r < rows; r += kFT)
    if (s.prow[r] != r) {
      const int slot = atomicAdd(&s.n_moved, 1);
      s.moved_dst[slot] = j0 + r;
      s.moved_src[slot] = j0 + s.prow[r];
    }
  __syncthreads();
}

}  // namespace

__global__ void __launch_bounds__(kFT, 512 / kFT) leaf_fused_kernel(const LeafFusedArgs f) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FusedSmem& s = *reinterpret_cast<FusedSmem*>(smem_raw);
  const LeafAsmArgs& a = f.a;
  const int ni = a.ni, ne = a.ne, nb = a.nb, ncol = ni + 1 + nb, nr = 1 + nb, dim = a.dim;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  double* W = f.scratch + (long long)blockIdx.x * f.scratch_stride;  // ni x ncol, ld ni
  double* R = W + (long long)ni * ni;                                 // [sgn f | -L_ie P] -> [v | Y_i]
  const bool p_in_smem = ne * nb <= kTileCols * kBLD;

  int iter = 0;
  const long long t_begin = clock64();
  auto stamp = [&](int k) {
    if (f.prof && blockIdx.x == 0 && tid == 0 && iter < 4) f.prof[iter * 8 + k] = clock64();
  };
  long long sub_t0 = 0;
  auto substamp = [&](int k) {  // accumulated sub-phases of the LU of leaf iteration 0 (slots 32..)
    if (f.prof && blockIdx.x == 0 && tid == 0 && iter == 0) {
      const long long t = clock64();
      if (k > 0) f.prof[32 + k] += t - sub_t0;
      sub_t0 = t;
    }
  };
  for (long long it = blockIdx.x; it < f.n_leaves; it += gridDim.x, ++iter) {
    const long long leaf = f.leaf_list ? f.leaf_list[it] : it;
    stamp(0);
    // ---- A. assembly (exterior neighbours into the shared list)
    double* nz_val = s.pan;
    int* nz_idx = reinterpret_cast<int*>(s.pan + kMaxNz);
    leaf_assemble_block(a, leaf, W, ni, nullptr, s.asmb, nz_idx, nz_val);
    if (tid == 0) {
      a.bad_point[leaf] = s.asmb.bad;
      s.pmin = DBL_MAX;
      s.pmax = 0.0;
      s.first_zero = -1;
    }
    if (p_in_smem) {
      for (int e = tid; e < ne * nb; e += kFT) cp_async8(s.tile + e, f.P + e, true);
      cp_async_commit();
      cp_async_wait<0>();
    }
    __syncthreads();
    stamp(1);
    // ---- B. R[:, 1 + j] = -sum over the row's exterior neighbours of L_ie * P[e, j]
    {
      const double* Pm = p_in_smem ? s.tile : f.P;
      const int nz = 2 * dim;
      // rows over the lanes, columns over the warps (no per-element index division); a row's
      // exterior neighbours are loaded once and reused for the warp's columns
      for (int r0 = 0; r0 < ni; r0 += 32) {
        const int r = r0 + lane;
        if (r >= ni) break;
        double zv[4];
        int zi[4];
#pragma unroll
        for (int z = 0; z < 4; ++z) {
          zv[z] = z < nz ? nz_val[z * ni + r] : 0.0;
          zi[z] = z < nz ? nz_idx[z * ni + r] : 0;
        }
        for (int j = warp; j < nb; j += kFW) {
          const double* Pj = Pm + j * ne;
          double acc = 0.0;
#pragma unroll
          for (int z = 0; z < 4; ++z)
            if (z < nz) acc += zv[z] * Pj[zi[z]];
          R[(long long)(1 + j) * ni + r] = -acc;
        }
      }
    }
    __syncthreads();

    stamp(2);
    // ---- C. blocked GEPP, RHS columns ride along
    for (int j0 = 0; j0 < ni; j0 += kNB) {
      const int pnb = min(kNB, ni - j0), rows = ni - j0;
      substamp(0);
      panel_gepp_warp(s, W, ni, j0, pnb, (f.prof && blockIdx.x == 0 && tid == 0 && iter == 0) ? f.prof : nullptr);
      substamp(1);
      // row exchange of every other column; chunks end on column boundaries
      {
        const int nm = s.n_moved;
        if (nm > 0) {
          constexpr int kPer = 8;
          const int cols_per_chunk = (kFT * kPer) / nm;
          // only columns right of the panel: the L columns left of it are dead (the
          // factors are not kept on this path), so their row order does not matter
          const int c_first = j0 + pnb, n_right = ncol - c_first;
          for (int cc0 = 0; cc0 < n_right; cc0 += cols_per_chunk) {
            const int total = min(cols_per_chunk, n_right - cc0) * nm;
            double vals[kPer];
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
              const int e = tid + u * kFT;
              if (e < total) {
                const int c = c_first + cc0 + e / nm, mv = e % nm;
                vals[u] = W[(long long)c * ni + s.moved_src[mv]];
              }
            }
            __syncthreads();
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
              const int e = tid + u * kFT;
              if (e < total) {
                const int c = c_first + cc0 + e / nm, mv = e % nm;
                W[(long long)c * ni + s.moved_dst[mv]] = vals[u];
              }
            }
            __syncthreads();
          }
        }
      }
      substamp(2);
      // per chunk of up to kTileCols columns right of the panel: stage A12 (k-major) in s.tile,
      // U12 = L11^-1 A12 in shared memory (one thread per column), then U12 back to W (coalesced)
      // alongside the DMMA trailing update that reads it from s.tile
      const int rc0 = j0 + pnb, nrc = ncol - rc0;
      for (int cc0 = 0; cc0 < nrc; cc0 += kTileCols) {
        const int ncc = min(kTileCols, nrc - cc0);
        for (int e = tid; e < ncc * kNB; e += kFT) {  // cp.async: all loads in flight, rows >= pnb zero
          const int kk = e % kNB, c = e / kNB;
          const bool ok = kk < pnb;
          cp_async8(s.tile + c * kBLD + kk, ok ? W + (long long)(rc0 + cc0 + c) * ni + j0 + kk : W, ok);
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        for (int c = tid; c < ncc; c += kFT) {
          double* col = s.tile + c * kBLD;
          double x[kNB];
#pragma unroll
          for (int jj = 0; jj < kNB; ++jj) x[jj] = col[jj];
#pragma unroll
          for (int ii = 0; ii < kNB - 1; ++ii)
#pragma unroll
            for (int jj = ii + 1; jj < kNB; ++jj) x[jj] -= s.pan[ii * kPLD + jj] * x[ii];
#pragma unroll
          for (int jj = 0; jj < kNB; ++jj)
            if (jj < pnb) col[jj] = x[jj];
        }
        __syncthreads();
        for (int e = tid; e < ncc * kNB; e += kFT) {
          const int kk = e % kNB, c = e / kNB;  // compile-time divisor
          if (kk < pnb) W[(long long)(rc0 + cc0 + c) * ni + j0 + kk] = s.tile[c * kBLD + kk];
        }
        if (rows > pnb)
          update_smem(rows - pnb, ncc, pnb, s.pan + pnb, kPLD, s.tile, kBLD,
                      W + (long long)(rc0 + cc0) * ni + j0 + pnb, ni);
        __syncthreads();
      }
      substamp(3);
      substamp(4);
    }

    stamp(3);
    // ---- D. back substitution on the 1+nb RHS columns.  Per 32-row block: the diagonal U block
    //      goes to the (dead) assembly buffer; warps 0-1 solve it for the <= 64 RHS columns while
    //      warps 2-7 stage the U column block above it (one barrier for both); then the DMMA update.
    {
      double* sDg = reinterpret_cast<double*>(&s.asmb);  // kNB x kNB diagonal block, ld kNB
      const int nblk = (ni + kNB - 1) / kNB;
      for (int jb = nblk - 1; jb >= 0; --jb) {
        const int r0 = jb * kNB, bnb = min(kNB, ni - r0);
        for (int c = warp; c < bnb; c += kFW)
          if (lane < bnb) {
            const double u = W[(long long)(r0 + c) * ni + r0 + lane];
            sDg[c * kNB + lane] = u;
            if (lane == c) s.rdiag[c] = 1.0 / u;
          }
        __syncthreads();
        if (tid < 64) {
          if (tid < nr) {
            double* col = R + (long long)tid * ni + r0;
            double x[kNB];
#pragma unroll
            for (int jj = 0; jj < kNB; ++jj) x[jj] = jj < bnb ? col[jj] : 0.0;
#pragma unroll
            for (int jj = kNB - 1; jj >= 0; --jj) {
              if (jj < bnb) {
                x[jj] *= s.rdiag[jj];
#pragma unroll
                for (int ii = 0; ii < jj; ++ii) x[ii] -= sDg[jj * kNB + ii] * x[jj];
              }
            }
#pragma unroll
            for (int jj = 0; jj < kNB; ++jj) {
              if (jj < bnb) col[jj] = x[jj];
              s.tile[tid * kBLD + jj] = jj < bnb ? x[jj] : 0.0;
            }
          }
        } else if (r0 > 0) {
          // U[0:r0, r0:r0+bnb] -> s.pan (A operand), one column per warp, rows over the lanes
          for (int c = warp - 2; c < bnb; c += kFW - 2) {
            const double* src = W + (long long)(r0 + c) * ni;
            for (int r = lane; r < r0; r += 32) cp_async8(s.pan + c * kPLD + r, src + r, true);
          }
          cp_async_commit();
          cp_async_wait<0>();
        }
        __syncthreads();
        if (r0 > 0) {
          update_smem(r0, nr, bnb, s.pan, kPLD, s.tile, kBLD, R, ni);
          __syncthreads();
        }
      }
    }

    stamp(4);
    // ---- E. [h | T] = Q_i [v | Y_i] + [0 | Q_e P]: 8x8 output tiles over all warps,
    //         k in shared chunks of 32 (A = Q_i chunk, B = [v|Y_i] chunk)
    {
      const int tmn = (nb + 7) / 8, tnn = (nr + 7) / 8, ntile = tmn * tnn;
      constexpr int kMaxT = 7;  // 8x8 tiles per warp: ceil(7*8 / 8) = 7 for nb = 56
      double acc[kMaxT][2];
#pragma unroll
      for (int u = 0; u < kMaxT; ++u) acc[u][0] = acc[u][1] = 0.0;
      // k chunks of kEK = 64 rows (4 barrier rounds instead of 7): Q_i chunk in s.pan (ld kEQ), [v|Y_i]
      // chunk in s.tile (ld kEQ); both leading dims are 4 mod 16 (conflict-free fragments)
      constexpr int kEK = 64, kEQ = 68;
      static_assert(kEK * kEQ <= kNB * kPLD && kEQ * 64 <= kTileCols * kBLD, "E-phase staging");
      for (int k0 = 0; k0 < ni; k0 += kEK) {
        const int kc = min(kEK, ni - k0);
        // cp.async staging: every element's load in flight at once
        for (int e = tid; e < nb * kc; e += kFT) {
          const int r = e % nb, kk = e / nb;
          cp_async8(s.pan + kk * kEQ + r, f.Qi + (long long)(k0 + kk) * nb + r, true);
        }
        for (int e = tid; e < nr * kEK; e += kFT) {
          const int kk = e % kEK, c = e / kEK;
          cp_async8(s.tile + c * kEQ + kk, kk < kc ? R + (long long)c * ni + k0 + kk : R, kk < kc);
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kMaxT; ++u) {
          const int t = warp + u * kFW;
          if (t < ntile) {
            const int m0 = (t % tmn) * 8, n0 = (t / tmn) * 8;
            for (int kk = 0; kk < kc; kk += 4) {
              const int kq = kk + t4;
              const double av = (kq < kc && m0 + g < nb) ? s.pan[kq * kEQ + m0 + g] : 0.0;
              const double bv = (kq < kc && n0 + g < nr) ? s.tile[(n0 + g) * kEQ + kq] : 0.0;
              dmma_8x8x4(acc[u][0], acc[u][1], av, bv);
            }
          }
        }
        __syncthreads();
      }
      double* HT = f.HT + leaf * f.strideHT;
#pragma unroll
      for (int u = 0; u < kMaxT; ++u) {
        const int t = warp + u * kFW;
        if (t < ntile) {
          const int m0 = (t % tmn) * 8, n0 = (t / tmn) * 8;
          const int r = m0 + g;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = n0 + t4 * 2 + h;
            if (r < nb && c < nr) __stcs(&HT[(long long)c * nb + r], acc[u][h] + f.ZQeP[(long long)c * nb + r]);
          }
        }
      }
    }
    stamp(5);
    // ---- outputs: [v | Y_i] for the solve, pivot statistics
    double* Yv = f.Yv + leaf * f.strideYv;
    for (int e0 = tid; e0 < ni * nr; e0 += 8 * kFT) {  // 8 loads in flight; streamed stores keep W in L2
      double t[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) t[u] = e0 + u * kFT < ni * nr ? R[e0 + u * kFT] : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (e0 + u * kFT < ni * nr) __stcs(&Yv[e0 + u * kFT], t[u]);
    }
    if (tid == 0 && f.stats) {
      f.stats[3 * leaf + 0] = s.pmin;
      f.stats[3 * leaf + 1] = s.pmax;
      f.stats[3 * leaf + 2] = s.first_zero;
    }
    __syncthreads();
  }
  if (f.prof && tid == 0) f.prof[64 + blockIdx.x] = clock64() - t_begin;
}

bool leaf_fused_supported(int n, int p, int ni, int nb, int dim, bool mixed_terms) {
  const int tmn = (nb + 7) / 8, tnn = (nb + 8) / 8;
  return !mixed_terms && dim == 2 && n <= 256 && p <= 16 && ni <= kMaxNI && ni <= kFT && ni + 1 + nb <= kMaxCols &&
         ni * 2 * dim <= kMaxNz && tmn * tnn <= 7 * kFW && 1 + nb <= kTileCols && nb <= 64 && 1 + nb <= 64 &&
         (size_t)kNB * kNB * 8 <= sizeof(LeafAsmSmemT<256, 16>);
}

long long leaf_fused_scratch_per_cta(int ni, int ne, int nb) { return (long long)ni * (ni + 1 + nb); }

// resident CTAs per SM of the fused kernel at its shared-memory size (the persistent grid is
// sized from this; the workspace footprint is grid * leaf_fused_scratch_per_cta)
int leaf_fused_ctas_per_sm() {
  const size_t smem = sizeof(FusedSmem);
  if (cudaFuncSetAttribute(leaf_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return 1;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, leaf_fused_kernel, kFT, smem) != cudaSuccess || n < 1) return 1;
  return n;
}

cudaError_t launch_leaf_fused(const LeafFusedArgs& f, int grid, cudaStream_t st) {
  const size_t smem = sizeof(FusedSmem);
  static PerDeviceFlag attr;
  const int dv = current_device();
  if (!(attr.set >> dv & 1)) {
    cudaError_t e = cudaFuncSetAttribute(leaf_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr.set |= 1ull << dv;
  }
  leaf_fused_kernel<<<grid, kFT, smem, st>>>(f);
  return cudaGetLastError();
}

}  // namespace hpsk
