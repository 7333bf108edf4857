// leaf_fdm.cu -- stage 1 (leaf-local solves) by fast diagonalisation, for operators whose second-order part
// is a constant Laplacian (a * Delta + c(x), any zeroth-order terms): the Helmholtz-type problems of the
// headline configuration.  One persistent kernel; the result is the reference's local solve
// (proj/src/local_solve.cpp:111-143: [v_i | Y_i] = L_ii^-1 [sgn f_i | -L_ie P], [h | T] = Q_i [v_i | Y_i] +
// [0 | Q_e P]) to roundoff, computed without an LU.
//
// On a uniform 2D tree every leaf has the same L_ii = K + diag(c), K = I (x) A + A (x) I with the 1D
// interior operator A = a (2/side)^2 D2[int, int] = V diag(lam) V^-1 (host eigendecomposition,
// geometry.cpp).  Per leaf, with cbar = (min c + max c) / 2 and K_c = K + cbar I (applied exactly through
// V: K_c^-1 U = V ((V^-1 U V^-T) / (lam_i + lam_j + cbar)) V^T on the 14 x 14 grid of a right-hand side),
// preconditioned Richardson on the TRUE operator
//     X_0 = K_c^-1 R,   X_{k+1} = X_k + K_c^-1 (R - K X_k - c o X_k)
// converges with rate rho = ||K_c^-1 (c - cbar)|| (about 1e-5 for the headline leaves: c varies by < 30
// across a leaf, the smallest |lam_i + lam_j| is 3.2e5), and its fixed point is L_ii^-1 R whatever the
// rounding of V.  A right-hand side stops when the predicted remaining error rho / (1 - rho) ||dX|| is
// below 1e-15 ||X|| (typically after 2-3 steps); a leaf that does not converge in kMaxSteps (resonant or
// strongly varying coefficients) raises the fail flag, and the host re-runs the LU leaf kernel.
//
// Data layout: every right-hand side is a 16 x 16 block (the 14 x 14 grid, zero padded) in shared memory,
// XOR-swizzled per column so DMMA fragment loads are conflict-free.  A warp owns whole blocks, so all
// passes of one right-hand side run without CTA barriers; each pass is "left-multiply by a 16 x 16 matrix
// held in registers (16 DMMA.8x8x4), store the block transposed", so two passes apply M U M^T.
#include <cfloat>
#include <climits>

#include "leaf_common.cuh"

namespace hpsk {

namespace {

#ifndef HPS_FDM_WARPS
#define HPS_FDM_WARPS 8
#endif
#ifndef HPS_FDM_MINB
#define HPS_FDM_MINB 2
#endif
constexpr int kT = 32 * HPS_FDM_WARPS, kW = kT / 32;
constexpr int kNC = kW;     // block slots (one per warp)
constexpr int kBlk = 256;   // 16 x 16 doubles
constexpr int kMaxSteps = 12;
#ifndef HPS_FDM_TOL
#define HPS_FDM_TOL 1e-18
#endif
constexpr double kTol = HPS_FDM_TOL;  // predicted remaining error / max|X| at which a right-hand side stops

#ifndef HPS_FDM_LPB
#define HPS_FDM_LPB 4
#endif
// leaves per CTA iteration: their columns are dealt to the warps as one sequence, so the end-of-iteration barrier
// waits for ceil(kLPB ncol / kW) columns per warp instead of kLPB ceil(ncol / kW) (L=8 leaf stage 17.3 -> 17.0 ms)
constexpr int kLPB = HPS_FDM_LPB;

struct FdmSmem {
  double R[kNC * kBlk], X[kNC * kBlk], W[kNC * kBlk];
  double cz[kLPB][kBlk];   // zeroth-order coefficient at the interior points (block layout), 0 in the padding
  double den[kLPB][kBlk];  // 1 / (lam_row + lam_col + cbar), 0 in the padding
  double fsrc[kLPB][2][256];  // source samples: real part (and the imaginary part in the ItI mode)
  int pos[256];      // tensor index -> interior r (>= 0) or -(exterior position) - 1
  double qDm[kBlk];  // separable Q_i as DMMA A operands (16 x 16 col-major, zero padded): rows s = d_s
  double qGm[kBlk];  // (side normal derivatives on the interior nodes) and G (Chebyshev -> Gauss, q x (p-2))
  double wmin[kLPB][kW], wmax[kLPB][kW];
  int bad[kLPB];
  int failed[kLPB];  // the leaf did not converge
  int ndmma[kLPB];   // DMMA.8x8x4 instructions issued for the leaf (executed-FLOP accounting)
  int ok[kLPB];      // the leaf takes the fast-diagonalisation path
};

// element (row, col) of a block: column-major 16 x 16, rows XOR-swizzled by the column with the bit-reversed
// low two column bits (x 4).  Conflict-free for the DMMA fragment loads (scalar, both orientations) and for the
// row-pair (double2) accesses of the transposed stores and the residual: within any quarter warp the columns
// g, g+1 of a pair land in opposite halves of the banks.
HPS_DEV int swx(int col) { return ((col & 1) << 3) | ((col & 2) << 1); }
HPS_DEV int swz(int row, int col) { return (col << 4) + (row ^ swx(col)); }

HPS_DEV void load_afrag(const double* M, double (&am)[2][4], int g, int t4) {
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) am[mt][ks] = M[(ks * 4 + t4) * 16 + mt * 8 + g];
}

// acc = M In, M from registers; In(k, n) read at swz(k, n) (TRANS = false) or swz(n, k) (TRANS = true).
// acc[mt][nt][h] is element (mt * 8 + g, nt * 8 + 2 t4 + h).  Ends with __syncwarp: the block may be
// overwritten in place after the call.
template <bool TRANS, bool SCALE = false>
HPS_DEV void mma_block(const double (&am)[2][4], const double* in, double (&acc)[2][2][2], int g, int t4,
                       const double* den = nullptr) {
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    double b[2];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int e = TRANS ? swz(nt * 8 + g, ks * 4 + t4) : swz(ks * 4 + t4, nt * 8 + g);
      b[nt] = SCALE ? in[e] * den[e] : in[e];
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) dmma_8x8x4(acc[mt][nt][0], acc[mt][nt][1], am[mt][ks], b[nt]);
  }
  __syncwarp();
}

// store acc transposed: element (m, n) to position (n, m), optionally scaled by den at that position
template <bool SCALE>
HPS_DEV void store_t(double* out, const double (&acc)[2][2][2], const double* den, int g, int t4) {
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int m = mt * 8 + g, n0 = nt * 8 + 2 * t4;
      const int p = swz(n0, m);  // (n0, m) and (n0 + 1, m) are adjacent
      double2 v = make_double2(acc[mt][nt][0], acc[mt][nt][1]);
      if (SCALE) {
        const double2 d = *reinterpret_cast<const double2*>(den + p);
        v.x *= d.x;
        v.y *= d.y;
      }
      *reinterpret_cast<double2*>(out + p) = v;
    }
  __syncwarp();
}

HPS_DEV double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// |v| to within a relative 2^-20 from above, as the high word of |v|: non-negative doubles order like their high
// words, so maxima reduce on the integer pipes (one redux per warp) and stay off the FP64 pipe the DMMAs use.
// The Richardson stopping tests only need these magnitudes as scales.
HPS_DEV unsigned abs_hi(double v) { return (unsigned)__double2hiint(v) & 0x7fffffffu; }
HPS_DEV double warp_max_hi(unsigned hi) {
  hi = __reduce_max_sync(0xffffffffu, hi);
  return hi == 0u ? 0.0 : __hiloint2double((int)hi, (int)0xffffffffu);
}

// Solve one right-hand side block: X <- L_ii^-1 R.  Returns false if it did not converge.
// hat: Xb already holds R^ = V^-1 R V^-T (the leaf-independent columns -L_ie P, precomputed once by
// leaf_fdm_prep_kernel); otherwise R^ is formed here from Rb (the source column).
HPS_DEV bool solve_block(const double* Rb, double* Xb, double* Wb, const double* cz, const double* den,
                         const double (&vi)[2][4], const double (&vv)[2][4], const double (&aa)[2][4], int g, int t4,
                         int& npass, bool hat) {
  double acc[2][2][2];
  // X_0 = K_c^-1 R = V (den o R^) V^T
  if (hat) {
    npass += 2;
    mma_block<false, true>(vv, Xb, acc, g, t4, den);
  } else {
    npass += 4;
    mma_block<false>(vi, Rb, acc, g, t4);
    store_t<false>(Wb, acc, nullptr, g, t4);
    mma_block<false>(vi, Wb, acc, g, t4);
    store_t<true>(Wb, acc, den, g, t4);
    mma_block<false>(vv, Wb, acc, g, t4);
  }
  store_t<false>(Wb, acc, nullptr, g, t4);
  mma_block<false>(vv, Wb, acc, g, t4);
  unsigned xm = 0u;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) xm = max(xm, max(abs_hi(acc[mt][nt][0]), abs_hi(acc[mt][nt][1])));
  store_t<false>(Xb, acc, nullptr, g, t4);
  double dprev = warp_max_hi(xm);
  bool contracted = false;
  // max|X_k| >= max|X_0| - sum of the corrections so far: the stopping tests use that lower bound as the
  // scale (one warp reduction per step)
  double xmax = dprev;
  if (dprev == 0.0) return true;
  for (int step = 0; step < kMaxSteps; ++step) {
    npass += 6;
    // W = R - A X - X A^T - c o X  (the residual of the true operator)
    mma_block<false>(aa, Xb, acc, g, t4);
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) Wb[swz(mt * 8 + g, nt * 8 + 2 * t4 + h)] = acc[mt][nt][h];
    __syncwarp();
    mma_block<true>(aa, Xb, acc, g, t4);  // (A X^T)(m, n) = (X A^T)(n, m)
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int p = swz(nt * 8 + 2 * t4, mt * 8 + g);
        const double2 r = *reinterpret_cast<const double2*>(Rb + p);
        const double2 w = *reinterpret_cast<const double2*>(Wb + p);
        const double2 x = *reinterpret_cast<const double2*>(Xb + p);
        const double2 c = *reinterpret_cast<const double2*>(cz + p);
        double2 o;
        o.x = r.x - w.x - acc[mt][nt][0] - c.x * x.x;
        o.y = r.y - w.y - acc[mt][nt][1] - c.y * x.y;
        *reinterpret_cast<double2*>(Wb + p) = o;
      }
    __syncwarp();
    // dX = K_c^-1 W; X += dX
    mma_block<false>(vi, Wb, acc, g, t4);
    store_t<false>(Wb, acc, nullptr, g, t4);
    mma_block<false>(vi, Wb, acc, g, t4);
    store_t<true>(Wb, acc, den, g, t4);
    mma_block<false>(vv, Wb, acc, g, t4);
    store_t<false>(Wb, acc, nullptr, g, t4);
    mma_block<false>(vv, Wb, acc, g, t4);
    unsigned dm = 0u;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int p = swz(nt * 8 + 2 * t4, mt * 8 + g);
        double2 x = *reinterpret_cast<const double2*>(Xb + p);
        x.x += acc[mt][nt][0];
        x.y += acc[mt][nt][1];
        *reinterpret_cast<double2*>(Xb + p) = x;
        dm = max(dm, max(abs_hi(acc[mt][nt][0]), abs_hi(acc[mt][nt][1])));
      }
    __syncwarp();
    const double dk = warp_max_hi(dm);
    xmax -= dk;
    if (dk == 0.0) return true;
    // measured contraction rho = dk / dprev; stop when the predicted remaining error rho / (1 - rho) dk is below
    // kTol xmax, or at the roundoff floor after a contraction (division-free forms)
    const bool contracts = 2.0 * dk < dprev;
    if (contracts && dk * dk <= kTol * xmax * (dprev - dk)) return true;
    if (dk <= 2e-15 * xmax && contracted) return true;
    contracted = contracted || contracts;
    dprev = dk;
  }
  return false;
}

template <int P>
__global__ void __launch_bounds__(kT, HPS_FDM_MINB) leaf_fdm_kernel(const LeafFdmArgs f) {
  constexpr int N1 = P - 2, NI = N1 * N1, NE = 4 * P - 4, NB = 4 * N1, NPT = P * P;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FdmSmem& s = *reinterpret_cast<FdmSmem*>(smem_raw);
  const LeafAsmArgs& a = f.a;
  // DtN: column 0 = sgn f_i, columns 1..NB = -L_ie P.  ItI mode: columns 0, 1 = Re f_i, Im f_i, columns
  // 2..NE+1 = -L_ie e_k (the prep tables were made with P = I), output Z = L_ii^-1 [f_i | -L_ie] only.
  // Source mode (f.src_cols > 0, the new-source pass of solve_new_source): every column is a source read from
  // f.Yv itself (sgn f_i in interior order, packed by the caller) and overwritten with L_ii^-1 of it.
  const bool srcmode = f.src_cols > 0;
  const int nsrc = srcmode ? f.src_cols : (f.iti ? 2 : 1);
  const int ncol = srcmode ? f.src_cols : nsrc + (f.iti ? 4 * P - 4 : NB);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t4 = lane & 3;
  double vi[2][4], vv[2][4], aa[2][4];
  load_afrag(f.Vinv, vi, g, t4);
  load_afrag(f.V, vv, g, t4);
  load_afrag(f.A, aa, g, t4);
  for (int r = tid; r < NI; r += kT) s.pos[a.interior[r]] = r;
  for (int r = tid; r < NE; r += kT) s.pos[a.exterior[r]] = -r - 1;
  for (int e = tid; e < kBlk; e += kT) {
    const int row = e & 15, col = e >> 4;
    s.qGm[e] = (!f.iti && row < N1 && col < N1) ? f.qG[row * N1 + col] : 0.0;   // G(i, m), q = N1
    s.qDm[e] = (!f.iti && row < 4 && col < N1) ? f.qd[row * N1 + col] : 0.0;    // d_s(k)
  }
  __syncthreads();

  // several leaves per iteration only when every CTA still gets many iterations (small trees: one leaf each)
  const int lpb = f.n_leaves >= (long long)gridDim.x * kLPB * 8 ? kLPB : 1;
  for (long long leaf0 = (long long)blockIdx.x * lpb; leaf0 < f.n_leaves; leaf0 += (long long)gridDim.x * lpb) {
    const int nl = (int)min((long long)lpb, f.n_leaves - leaf0);
    // ---- coefficients and source at the leaf points (leaf_cheb_points, discretize_operator's sampling)
    if (tid < kLPB) s.bad[tid] = INT_MAX, s.ndmma[tid] = 0, s.failed[tid] = 0;
    for (int e = tid; e < kLPB * kBlk; e += kT) s.cz[e / kBlk][e % kBlk] = 0.0;
    __syncthreads();
#pragma unroll
    for (int lf = 0; lf < kLPB; ++lf) {
      if (lf >= nl) break;
      const long long leaf = leaf0 + lf;
      const double* box = a.leaf_box + leaf * 6;
      double cmin = DBL_MAX, cmax = -DBL_MAX;
      for (int i = tid; i < NPT; i += kT) {
        const int i1 = i / P, i2 = i % P;
        double x[3] = {0.0, 0.0, 0.0};
        x[0] = __dadd_rn(__dmul_rn(0.5, __dadd_rn(box[0], box[3])), __dmul_rn(__dmul_rn(0.5, __dsub_rn(box[3], box[0])), a.cheb[i1]));
        x[1] = __dadd_rn(__dmul_rn(0.5, __dadd_rn(box[1], box[4])), __dmul_rn(__dmul_rn(0.5, __dsub_rn(box[4], box[1])), a.cheb[i2]));
        double cz = 0.0;
        for (int t = 0; t < a.nterms; ++t) {
          const double v = eval_field_t<2>(a.terms[t].f, x, leaf, i, NPT);
          if (!isfinite(v)) atomicMin(&s.bad[lf], i);
          if (a.terms[t].role == 2) cz = __dadd_rn(cz, v);
        }
        s.fsrc[lf][0][i] = (a.has_source && !srcmode) ? eval_field_t<2>(a.source, x, leaf, i, NPT) : 0.0;
        if (f.iti) s.fsrc[lf][1][i] = f.has_source_im ? eval_field_t<2>(f.source_im, x, leaf, i, NPT) : 0.0;
        const int r = s.pos[i];
        if (r >= 0) {
          s.cz[lf][swz(r % N1, r / N1)] = cz;
          cmin = fmin(cmin, cz);
          cmax = fmax(cmax, cz);
        }
      }
      cmin = -warp_max(-cmin);
      cmax = warp_max(cmax);
      if (lane == 0) s.wmin[lf][warp] = cmin, s.wmax[lf][warp] = cmax;
    }
    __syncthreads();
    double dmin[kLPB], dmax[kLPB];
#pragma unroll
    for (int lf = 0; lf < kLPB; ++lf) {
      dmin[lf] = DBL_MAX, dmax[lf] = 0.0;
      if (lf >= nl) continue;
      double cmin = s.wmin[lf][0], cmax = s.wmax[lf][0];
      for (int w = 1; w < kW; ++w) cmin = fmin(cmin, s.wmin[lf][w]), cmax = fmax(cmax, s.wmax[lf][w]);
      const double cbar = 0.5 * (cmin + cmax);
      if (!isfinite(cbar)) dmin[lf] = -1.0;  // not ok
      for (int e = tid; e < kBlk; e += kT) {
        const int col = e >> 4, row = (e & 15) ^ swx(col);
        double d = 0.0;
        if (row < N1 && col < N1) {
          const double ev = f.lam[row] + f.lam[col] + cbar;
          d = 1.0 / ev;
          dmin[lf] = fmin(dmin[lf], fabs(ev));
          dmax[lf] = fmax(dmax[lf], fabs(ev));
        }
        s.den[lf][e] = d;
      }
      dmin[lf] = -warp_max(-dmin[lf]);
      dmax[lf] = warp_max(dmax[lf]);
    }
    __syncthreads();  // everyone read s.wmin/wmax
#pragma unroll
    for (int lf = 0; lf < kLPB; ++lf)
      if (lane == 0 && lf < nl) s.wmin[lf][warp] = dmin[lf], s.wmax[lf][warp] = dmax[lf];
    __syncthreads();
    if (tid < nl) {
      const int lf = tid;
      const long long leaf = leaf0 + lf;
      double dn = s.wmin[lf][0], dx = s.wmax[lf][0];
      for (int w = 1; w < kW; ++w) dn = fmin(dn, s.wmin[lf][w]), dx = fmax(dx, s.wmax[lf][w]);
      // a negative dn marks a non-finite cbar (fmin keeps it negative)
      const bool ok = s.bad[lf] == INT_MAX && dn > 1e-12 * dx && dn >= 0.0;
      if (!srcmode) {
        a.bad_point[leaf] = s.bad[lf];
        f.stats[3 * leaf + 0] = dn;  // spectral analogue of the pivot statistics: min / max |lam_i + lam_j + cbar|
        f.stats[3 * leaf + 1] = dx;
        f.stats[3 * leaf + 2] = -1.0;
      }
      // non-finite samples (reported by the host) or a resonant leaf: the LU path takes over
      if (!ok && s.bad[lf] == INT_MAX) f.fail_list[atomicAdd(f.fail_count, 1)] = int(leaf);
      s.ok[lf] = ok;
    }
    __syncthreads();

    // ---- per warp: the iteration's columns t = warp + 1, warp + 1 + kW, ... over the leaves in turn (within a
    // leaf, column 0, the source, comes last), each solved, written and contracted to [h | T] without CTA barriers
    {
      double* Rb = s.R + warp * kBlk;
      double* Xb = s.X + warp * kBlk;
      double* Wb = s.W + warp * kBlk;
      for (int t = warp + 1; t <= nl * ncol; t += kW) {
        const int lf = (t - 1) / ncol, c = (t - 1) - lf * ncol + 1;
        if (!s.ok[lf]) continue;
        const long long leaf = leaf0 + lf;
        const int col = c == ncol ? 0 : c;
        int npass = 0, nout = 0;
        // right-hand side: the source column(s) (formed here); then -L_ie P (-L_ie in the ItI mode), the same for
        // every leaf (constant Laplacian): R and R^ = V^-1 R V^-T from the prep tables (L2-resident)
        if (col >= nsrc) {
          const double2* Rt = reinterpret_cast<const double2*>(f.Rtab + (long long)(col - nsrc) * kBlk);
          const double2* Rh = reinterpret_cast<const double2*>(f.Rhat + (long long)(col - nsrc) * kBlk);
#pragma unroll
          for (int e = lane; e < kBlk / 2; e += 32) {
            reinterpret_cast<double2*>(Rb)[e] = __ldg(Rt + e);
            reinterpret_cast<double2*>(Xb)[e] = __ldg(Rh + e);
          }
        } else if (srcmode) {
          const double* src = f.Yv + leaf * f.strideYv + (long long)col * NI;
          for (int e = lane; e < kBlk; e += 32) {
            const int cc = e >> 4, row = (e & 15) ^ swx(cc);
            Rb[e] = (row < N1 && cc < N1) ? src[cc * N1 + row] : 0.0;
          }
        } else {
          for (int e = lane; e < kBlk; e += 32) {
            const int cc = e >> 4, row = (e & 15) ^ swx(cc);
            Rb[e] = (row < N1 && cc < N1) ? a.fsign * s.fsrc[lf][col][(cc + 1) * P + row + 1] : 0.0;
          }
        }
        __syncwarp();
        const bool conv = solve_block(Rb, Xb, Wb, s.cz[lf], s.den[lf], vi, vv, aa, g, t4, npass, !srcmode && col >= nsrc);
        if (!conv && lane == 0) s.failed[lf] = 1;
        // [v_i | Y_i] column (interior index r = (i1-1) N1 + (i2-1)); ItI mode: the column of Z
        double* Yv = f.Yv + leaf * f.strideYv + (long long)col * NI;
#pragma unroll
        for (int r = lane; r < NI; r += 32) __stcs(&Yv[r], Xb[swz(r % N1, r / N1)]);
        if (!(f.iti || srcmode)) {
          // [h | T] = Q_i X + [0 | Q_e P] through the separable Q_i (geometry.cpp q_interior_factors), on DMMA:
          // U = Dm X (rows S, N: u_s(m) = sum_k d_s(k) X(k, m)) and Dm X^T (rows E, W), then H = G U^T, h = ds H.
          // Block element (row, col) = X(i1 = col + 1, i2 = row + 1).  U goes to Rb (free after the solve) as a
          // B operand: element (m, side) at swz(m, side); rows 4..7 of Dm are zero, so are those sides.
          double ad[4];
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) ad[ks] = s.qDm[(ks * 4 + t4) * 16 + g];
          double u[2][2][2];  // [pass][nt][h]: element (side g, m = nt * 8 + 2 t4 + h)
#pragma unroll
          for (int ps = 0; ps < 2; ++ps)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) u[ps][nt][0] = u[ps][nt][1] = 0.0;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
              dmma_8x8x4(u[0][nt][0], u[0][nt][1], ad[ks], Xb[swz(ks * 4 + t4, nt * 8 + g)]);   // Dm X
              dmma_8x8x4(u[1][nt][0], u[1][nt][1], ad[ks], Xb[swz(nt * 8 + g, ks * 4 + t4)]);   // Dm X^T
            }
          __syncwarp();
#pragma unroll
          for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h) Rb[swz(nt * 8 + 2 * t4 + h, g)] = (g & 1) ? u[1][nt][h] : u[0][nt][h];
          __syncwarp();
          double hh[2][2] = {{0.0, 0.0}, {0.0, 0.0}};  // [mt][h]: element (i = mt * 8 + g, side = 2 t4 + h)
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const double bv = Rb[swz(ks * 4 + t4, g)];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) dmma_8x8x4(hh[mt][0], hh[mt][1], s.qGm[(ks * 4 + t4) * 16 + mt * 8 + g], bv);
          }
          double* HT = f.HT + leaf * f.strideHT + (long long)col * NB;
          const double* zq = f.ZQeP + (long long)col * NB;
          if (t4 < 2)
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int i = mt * 8 + g, row = (2 * t4 + h) * N1 + i;
                if (i < N1) __stcs(&HT[row], f.qds * hh[mt][h] + __ldg(zq + row));
              }
          nout += 24;  // DMMA: two 8-row passes and one 8-column pass
        }
        __syncwarp();
        if (lane == 0 && npass) atomicAdd(&s.ndmma[lf], 16 * npass + nout);
      }
    }
    __syncthreads();
    if (tid < nl && s.ok[tid]) {
      const long long leaf = leaf0 + tid;
      if (s.failed[tid]) f.fail_list[atomicAdd(f.fail_count, 1)] = int(leaf);
      if (!srcmode) f.stats[3 * leaf + 2] = -1.0 - double(s.ndmma[tid]);  // < 0: no zero pivot; the LU fallback rewrites it
    }
  }
}

// The leaf-independent right-hand sides -L_ie P (constant Laplacian; the zeroth-order term only enters L_ii)
// in the block layout, and R^ = V^-1 R V^-T: one warp per column, the same arithmetic the leaf kernel used
// to run per leaf, so the results are unchanged.
template <int P>
__global__ void __launch_bounds__(32) leaf_fdm_prep_kernel(const LeafFdmArgs f) {
  constexpr int N1 = P - 2, NE = 4 * P - 4;
  __shared__ __align__(16) double R[kBlk], W[kBlk];
  __shared__ int pos[256];
  const LeafAsmArgs& a = f.a;
  const int lane = threadIdx.x, g = lane >> 2, t4 = lane & 3, rc = blockIdx.x + 1;
  const double s2 = a.scale * a.scale, clap = f.lap_coef;
  for (int r = lane; r < N1 * N1; r += 32) pos[a.interior[r]] = r;
  for (int r = lane; r < NE; r += 32) pos[a.exterior[r]] = -r - 1;
  __syncwarp();
  for (int q = lane; q < kBlk; q += 32) {
    const int col = q >> 4, row = (q & 15) ^ swx(col);
    double v = 0.0;
    if (row < N1 && col < N1) {
      const int i1 = col + 1, i2 = row + 1;
      // the row's exterior line neighbours in slot order (axis 0 node 0 / p-1, axis 1 node 0 / p-1), entries
      // s^2 (a D2(i, j)) as leaf_entry rounds them
      const double* Pj = f.P + (long long)(rc - 1) * NE;
      double acc = 0.0;
      acc += __dmul_rn(s2, __dmul_rn(clap, a.D2[0 * P + i1])) * Pj[-pos[0 * P + i2] - 1];
      acc += __dmul_rn(s2, __dmul_rn(clap, a.D2[(P - 1) * P + i1])) * Pj[-pos[(P - 1) * P + i2] - 1];
      acc += __dmul_rn(s2, __dmul_rn(clap, a.D2[0 * P + i2])) * Pj[-pos[i1 * P + 0] - 1];
      acc += __dmul_rn(s2, __dmul_rn(clap, a.D2[(P - 1) * P + i2])) * Pj[-pos[i1 * P + P - 1] - 1];
      v = -acc;
    }
    R[q] = v;
  }
  __syncwarp();
  double vi[2][4], acc[2][2][2];
  load_afrag(f.Vinv, vi, g, t4);
  mma_block<false>(vi, R, acc, g, t4);
  store_t<false>(W, acc, nullptr, g, t4);
  mma_block<false>(vi, W, acc, g, t4);
  store_t<false>(W, acc, nullptr, g, t4);
  for (int q = lane; q < kBlk; q += 32) {
    f.Rtab[(long long)(rc - 1) * kBlk + q] = R[q];
    f.Rhat[(long long)(rc - 1) * kBlk + q] = W[q];
  }
}

using FdmKernel = void (*)(const LeafFdmArgs);
FdmKernel fdm_kernel_for(int p) {
  switch (p) {
    case 4: return leaf_fdm_kernel<4>;
    case 5: return leaf_fdm_kernel<5>;
    case 6: return leaf_fdm_kernel<6>;
    case 7: return leaf_fdm_kernel<7>;
    case 8: return leaf_fdm_kernel<8>;
    case 9: return leaf_fdm_kernel<9>;
    case 10: return leaf_fdm_kernel<10>;
    case 11: return leaf_fdm_kernel<11>;
    case 12: return leaf_fdm_kernel<12>;
    case 13: return leaf_fdm_kernel<13>;
    case 14: return leaf_fdm_kernel<14>;
    case 15: return leaf_fdm_kernel<15>;
    case 16: return leaf_fdm_kernel<16>;
    default: return nullptr;
  }
}

}  // namespace

bool leaf_fdm_shape_ok(int p, int ni, int nb, int dim) {
  return dim == 2 && p >= 4 && p <= 16 && ni == (p - 2) * (p - 2) && nb <= 64 && p * p <= 256;
}

int leaf_fdm_ctas_per_sm(int p) {
  const size_t smem = sizeof(FdmSmem);
  FdmKernel k = fdm_kernel_for(p);
  if (!k || cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 1;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, kT, smem) != cudaSuccess || n < 1) return 1;
  return n;
}

cudaError_t launch_leaf_fdm_prep(const LeafFdmArgs& f, cudaStream_t st) {
  const int nb = f.iti ? 4 * f.a.p - 4 : 4 * (f.a.p - 2);
  switch (f.a.p) {
#define HPS_FDM_PREP(PP) \
  case PP: leaf_fdm_prep_kernel<PP><<<nb, 32, 0, st>>>(f); break;
    HPS_FDM_PREP(4) HPS_FDM_PREP(5) HPS_FDM_PREP(6) HPS_FDM_PREP(7) HPS_FDM_PREP(8) HPS_FDM_PREP(9) HPS_FDM_PREP(10)
    HPS_FDM_PREP(11) HPS_FDM_PREP(12) HPS_FDM_PREP(13) HPS_FDM_PREP(14) HPS_FDM_PREP(15) HPS_FDM_PREP(16)
#undef HPS_FDM_PREP
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_leaf_fdm(const LeafFdmArgs& f, int grid, cudaStream_t st) {
  const size_t smem = sizeof(FdmSmem);
  const int p = f.a.p;
  FdmKernel k = fdm_kernel_for(p);
  if (!k) return cudaErrorInvalidValue;
  static PerDeviceFlag attr[17];
  const int dv = current_device();
  if (!(attr[p].set >> dv & 1)) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr[p].set |= 1ull << dv;
  }
  k<<<grid, kT, smem, st>>>(f);
  return cudaGetLastError();
}

}  // namespace hpsk
