// leaf_common.cuh -- device-side leaf operator assembly shared by the batched
// (leaf_assemble_kernel) and fused (leaf_fused_kernel) leaf stages.
//
// Reference: discretize_operator (proj/src/local_solve.cpp:44-86) restricted to
// the interior rows, and the source sampling of HpsSolver::build_leaf
// (proj/src/solver.cpp:49-57).  Accumulation order per entry = term order, axis
// order, with the reference's s^k * (c_i * op_ij) rounding (no FMA contraction).
#pragma once

#include <climits>
#include <cmath>

#include "hps_kernels.cuh"

namespace hpsk {

constexpr int kLeafMaxPts = 512;  // p^d <= 512 (2D p <= 22, 3D p <= 8)
constexpr int kLeafMaxP = 24;

// Loops over the spatial axes are unrolled at compile time (DIM = 2 or 3) so the point and index
// arrays stay in registers; the runtime-dim entry points dispatch once.
template <int DIM>
__host__ __device__ __forceinline__ double leaf_bumps(const DevField& f, const double* x) {
  double s = 0.0;
  for (int j = 0; j < f.n_centers; ++j) {
    double r2 = 0.0;
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
      const double d = x[k] - f.centers[3 * j + k];
      r2 += d * d;
    }
    s += exp(-f.c[2] * r2);
  }
  return s;
}

// Evaluation of the built-in fields (hps_cuda.h HPSG_FIELD_*): on the device inside the leaf kernels, on the
// host for the adaptive-refinement criterion (hpsg_refine_adaptive).
template <int DIM>
__host__ __device__ __forceinline__ double eval_field_t(const DevField& f, const double* x, long long leaf, int pt,
                                                        int npts) {
  const double* c = f.c;
  switch (f.kind) {
    case 0: return c[0];
    case 1: return c[0] + c[1] * leaf_bumps<DIM>(f, x);
    case 2: return c[0] * sin(c[1] * x[0] + c[2] * x[1] + c[3] * x[2] + c[4]);
    case 3: return c[0] * cos(c[1] * x[0] + c[2] * x[1] + c[3] * x[2] + c[4]);
    case 4: return c[0] * leaf_bumps<DIM>(f, x) * sin(c[3] * x[0] + c[4] * x[1] + c[5] * x[2] + c[6]);
    case 5: {  // proj/src/problems.cpp:50-66
      const double X = x[0], Y = x[1];
      const double ux = 5.0 * exp(5.0 * X) * sin(5.0 * Y) + 10.0 * M_PI * cos(10.0 * M_PI * X) * sin(M_PI * Y);
      const double uy = 5.0 * exp(5.0 * X) * cos(5.0 * Y) + M_PI * sin(10.0 * M_PI * X) * cos(M_PI * Y);
      const double lap = -101.0 * M_PI * M_PI * sin(10.0 * M_PI * X) * sin(M_PI * Y);
      return lap - cos(5.0 * Y) * ux + sin(5.0 * Y) * uy;
    }
    case 6: return f.samples[leaf * npts + pt];
    case 7: {  // d/dx_a of the bump field
      const int ax = int(c[3]);
      double s = 0.0;
      for (int j = 0; j < f.n_centers; ++j) {
        double r2 = 0.0, dax = 0.0;
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
          const double d = x[k] - f.centers[3 * j + k];
          r2 += d * d;
          if (k == ax) dax = d;
        }
        s += -2.0 * c[2] * dax * exp(-c[2] * r2);
      }
      return c[1] * s;
    }
    case 8: {  // div(eps grad u), eps = c0 + c1 sum exp(-c2 r^2), u = prod_k sin(c3 x_k + c4)
      double sn[3], cs[3], u = 1.0;
#pragma unroll
      for (int k = 0; k < DIM; ++k) sn[k] = sin(c[3] * x[k] + c[4]), cs[k] = cos(c[3] * x[k] + c[4]), u *= sn[k];
      double eps = c[0], geps[3] = {0.0, 0.0, 0.0};
      for (int j = 0; j < f.n_centers; ++j) {
        double r2 = 0.0;
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
          const double d = x[k] - f.centers[3 * j + k];
          r2 += d * d;
        }
        const double e = exp(-c[2] * r2);
        eps += c[1] * e;
#pragma unroll
        for (int k = 0; k < DIM; ++k) geps[k] += c[1] * -2.0 * c[2] * (x[k] - f.centers[3 * j + k]) * e;
      }
      double f2 = -DIM * c[3] * c[3] * u * eps;
#pragma unroll
      for (int k = 0; k < DIM; ++k) {
        double du = c[3] * cs[k];
#pragma unroll
        for (int l = 0; l < DIM; ++l)
          if (l != k) du *= sn[l];
        f2 += geps[k] * du;
      }
      return f2;
    }
    case 9: {  // make_wavefront_3d source (proj/src/problems.cpp:154-179): Laplacian of atan(a rho^2 - 0.7)
      const double a = c[0];
      const double d0 = x[0] - c[1], d1 = x[1] - c[2], d2 = x[2] - c[3];
      const double r2 = d0 * d0 + d1 * d1 + d2 * d2;
      const double w = a * r2 - 0.7;
      const double s = 1.0 + w * w;
      return -2.0 * w / (s * s) * 4.0 * a * a * r2 + 6.0 * a / s;
    }
    case 10:    // PoissonBoltzmannSpec::eps, smooth (problems.cpp:187-191): eps0 + (eps_inf - eps0) exp(-A rho)
    case 11: {  // grad_eps[axis c4] (problems.cpp:200-205)
      double rho = 0.0, g[3] = {0.0, 0.0, 0.0};
      for (int j = 0; j < f.n_centers; ++j) {
        const double e0 = x[0] - f.centers[3 * j], e1 = x[1] - f.centers[3 * j + 1], e2 = x[2] - f.centers[3 * j + 2];
        const double e = exp(-c[3] * (e0 * e0 + e1 * e1 + e2 * e2));
        rho += e;
        const double t = -2.0 * c[3] * e;
        g[0] += t * e0;
        g[1] += t * e1;
        g[2] += t * e2;
      }
      if (f.kind == 10) return c[0] + (c[1] - c[0]) * exp(-c[2] * rho);
      const int ax = int(c[4]);
      return (c[1] - c[0]) * exp(-c[2] * rho) * (-c[2]) * (ax == 0 ? g[0] : ax == 1 ? g[1] : g[2]);
    }
    default: return NAN;
  }
}

__device__ __forceinline__ double eval_field(const DevField& f, const double* x, int dim, long long leaf, int pt,
                                             int npts) {
  return dim == 3 ? eval_field_t<3>(f, x, leaf, pt, npts) : eval_field_t<2>(f, x, leaf, pt, npts);
}

// v[i] for a runtime axis i < DIM without dynamic register indexing
template <int DIM>
__device__ __forceinline__ int pick(const int* v, int i) {
  int r = v[0];
#pragma unroll
  for (int k = 1; k < DIM; ++k) r = i == k ? v[k] : r;
  return r;
}

__device__ __forceinline__ void leaf_decode(int idx, int p, int dim, int* c) {
  if (dim == 2) {
    c[0] = idx / p;
    c[1] = idx % p;
    c[2] = 0;
  } else {
    c[0] = idx / (p * p);
    c[1] = (idx / p) % p;
    c[2] = idx % p;
  }
}

template <int MAXPTS, int MAXP>
struct LeafAsmSmemT {
  double coef[kMaxTerms][MAXPTS];
  double fsrc[MAXPTS];
  double D[MAXP * MAXP], D2[MAXP * MAXP];
  int pos[MAXPTS];  // tensor index -> interior position r (>= 0) or -(exterior position) - 1
  int bad;
};
using LeafAsmSmem = LeafAsmSmemT<kLeafMaxPts, kLeafMaxP>;

// Value of the operator entry L(gi, gj) accumulated in the reference order (term, then axis):
// proj/src/local_solve.cpp:63-83, each contribution rounded as s^k * (c_i * op_ij).
template <int DIM, class SM>
__device__ __forceinline__ double leaf_entry(const LeafAsmArgs& a, const SM& s, int gi, const int* ii, int gj,
                                             const int* jj) {
  const int p = a.p;
  const double s1 = a.scale, s2 = a.scale * a.scale;
  bool same[3];
#pragma unroll
  for (int k = 0; k < DIM; ++k) same[k] = ii[k] == jj[k];
  double val = 0.0;
  for (int t = 0; t < a.nterms; ++t) {
    const DevTerm& tm = a.terms[t];
    const double c = s.coef[t][gi];
    switch (tm.role) {
      case 0:  // laplacian: c s^2 sum_a D2_a
#pragma unroll
        for (int ax = 0; ax < DIM; ++ax) {
          bool ok = true;
#pragma unroll
          for (int k = 0; k < DIM; ++k)
            if (k != ax && !same[k]) ok = false;
          if (ok) val = __dadd_rn(val, __dmul_rn(s2, __dmul_rn(c, s.D2[jj[ax] * p + ii[ax]])));
        }
        break;
      case 1: {  // gradient: c s D_axis
        const int ax = tm.axis;
        bool ok = true;
#pragma unroll
        for (int k = 0; k < DIM; ++k)
          if (k != ax && !same[k]) ok = false;
        if (ok) val = __dadd_rn(val, __dmul_rn(s1, __dmul_rn(c, s.D[pick<DIM>(jj, ax) * p + pick<DIM>(ii, ax)])));
        break;
      }
      case 2:  // zeroth: diag(c)
        if (gi == gj) val = __dadd_rn(val, c);
        break;
      default: {  // second_order
        const int a1 = tm.axis, a2 = tm.axis2;
        const int j1 = pick<DIM>(jj, a1), i1 = pick<DIM>(ii, a1);
        if (a1 == a2) {
          bool ok = true;
#pragma unroll
          for (int k = 0; k < DIM; ++k)
            if (k != a1 && !same[k]) ok = false;
          if (ok) val = __dadd_rn(val, __dmul_rn(s2, __dmul_rn(c, s.D2[j1 * p + i1])));
        } else {
          bool ok = true;
#pragma unroll
          for (int k = 0; k < DIM; ++k)
            if (k != a1 && k != a2 && !same[k]) ok = false;
          if (ok) {
            const double d = __dmul_rn(s.D[j1 * p + i1], s.D[pick<DIM>(jj, a2) * p + pick<DIM>(ii, a2)]);
            val = __dadd_rn(val, __dmul_rn(s2, __dmul_rn(c, d)));
          }
        }
      }
    }
  }
  return val;
}

template <class SM>
__device__ __forceinline__ double leaf_entry(const LeafAsmArgs& a, const SM& s, int gi, const int* ii, int gj,
                                             const int* jj) {
  return a.dim == 3 ? leaf_entry<3>(a, s, gi, ii, gj, jj) : leaf_entry<2>(a, s, gi, ii, gj, jj);
}

// One CTA assembles one leaf: M[:, 0:ni] = L(I_i, I_i), M[:, ni] = sgn * f(I_i) (ld = ldM),
// E = L(I_i, I_e) (ld = ni).  Returns (via s.bad) the first non-finite coefficient point or INT_MAX.
// Without mixed second-order terms the operator row of point i is supported on the dim grid
// lines through i, so the block is zero-filled and only those (dim*(p-1)+1 per row) entries are
// evaluated; otherwise every entry is evaluated.
//
// enz_idx/enz_val (optional, operators without mixed terms only): instead of writing the
// exterior block E, record each interior row's 2*dim exterior line neighbours at slot
// (2*axis + (neighbour at node 0 ? 0 : 1)) * ni + r as (exterior position, value) -- row-fastest,
// so a warp reading one slot for consecutive rows hits consecutive banks.
template <int DIM, class SM>
__device__ __forceinline__ void leaf_assemble_block_t(const LeafAsmArgs& a, long long leaf, double* M, long long ldM,
                                                      double* E, SM& s, int* enz_idx, double* enz_val) {
  constexpr int dim = DIM;
  const int tid = threadIdx.x, nthr = blockDim.x, p = a.p, n = a.n;
  if (tid == 0) s.bad = INT_MAX;
  for (int e = tid; e < p * p; e += nthr) s.D[e] = a.D[e], s.D2[e] = a.D2[e];
  for (int r = tid; r < a.ni; r += nthr) s.pos[a.interior[r]] = r;
  for (int r = tid; r < a.ne; r += nthr) s.pos[a.exterior[r]] = -r - 1;
  __syncthreads();  // s.bad initialised before any atomicMin
  const double* box = a.leaf_box + leaf * 6;
  // leaf_cheb_points (proj/src/mesh.cpp:320-336): 0.5(lo+hi) + 0.5(hi-lo) t, no FMA contraction
  for (int i = tid; i < n; i += nthr) {
    int ci[3];
    leaf_decode(i, p, dim, ci);
    double x[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < dim; ++k)
      x[k] = __dadd_rn(__dmul_rn(0.5, __dadd_rn(box[k], box[3 + k])),
                       __dmul_rn(__dmul_rn(0.5, __dsub_rn(box[3 + k], box[k])), a.cheb[ci[k]]));
    for (int t = 0; t < a.nterms; ++t) {
      const double v = eval_field_t<DIM>(a.terms[t].f, x, leaf, i, n);
      s.coef[t][i] = v;
      if (!isfinite(v)) atomicMin(&s.bad, i);
    }
    s.fsrc[i] = a.has_source ? eval_field_t<DIM>(a.source, x, leaf, i, n) : 0.0;
  }
  bool mixed = false;
  for (int t = 0; t < a.nterms; ++t)
    if (a.terms[t].role == 3 && a.terms[t].axis != a.terms[t].axis2) mixed = true;
  const int ni = a.ni, ne = a.ne;
  if (mixed) {
    __syncthreads();
    for (int e = tid; e < ni * (ni + ne); e += nthr) {
      const int r = e % ni, cj = e / ni;
      const int gi = a.interior[r], gj = cj < ni ? a.interior[cj] : a.exterior[cj - ni];
      int ii[3], jj[3];
      leaf_decode(gi, p, dim, ii);
      leaf_decode(gj, p, dim, jj);
      const double v = leaf_entry<DIM>(a, s, gi, ii, gj, jj);
      if (cj < ni)
        M[(long long)cj * ldM + r] = v;
      else
        E[(long long)(cj - ni) * ni + r] = v;
    }
  } else {
    // zero fill (coalesced; 32-byte STG.256 stores where aligned, else 16-byte)
    if (ldM == ni && ((ni * ni) % 4) == 0 && ((reinterpret_cast<uintptr_t>(M) & 31) == 0)) {
      for (int e = tid; e < ni * ni / 4; e += nthr)
        asm volatile("st.global.v4.f64 [%0], {%1, %1, %1, %1};" ::"l"(M + 4 * (long long)e), "d"(0.0) : "memory");
    } else if (ldM == ni && (ni % 2) == 0 && ((reinterpret_cast<uintptr_t>(M) & 15) == 0)) {
      double2* m2 = reinterpret_cast<double2*>(M);
      for (int e = tid; e < ni * ni / 2; e += nthr) m2[e] = make_double2(0.0, 0.0);
    } else {
      for (int e = tid; e < ni * ni; e += nthr) M[(long long)(e / ni) * ldM + e % ni] = 0.0;
    }
    if (!enz_idx)
      for (int e = tid; e < ni * ne; e += nthr) E[e] = 0.0;
    __syncthreads();
    // entries on the grid lines through each interior point; the diagonal once
    const int per_row = dim * (p - 1) + 1;
    for (int e = tid; e < ni * per_row; e += nthr) {
      const int r = e % ni, w = e / ni;
      const int gi = a.interior[r];
      int ii[3], jj[3];
      leaf_decode(gi, p, dim, ii);
      jj[0] = ii[0], jj[1] = ii[1], jj[2] = ii[2];
      int ax = 0;
      if (w > 0) {
        ax = (w - 1) / (p - 1);
        const int k0 = (w - 1) % (p - 1);
#pragma unroll
        for (int k = 0; k < DIM; ++k)
          if (k == ax) jj[k] = k0 < ii[k] ? k0 : k0 + 1;  // skip the diagonal
      }
      const int gj = dim == 2 ? jj[0] * p + jj[1] : (jj[0] * p + jj[1]) * p + jj[2];
      const double v = leaf_entry<DIM>(a, s, gi, ii, gj, jj);
      const int q = s.pos[gj];
      if (q >= 0) {
        M[(long long)q * ldM + r] = v;
      } else if (enz_idx) {
        const int slot = (2 * ax + (pick<DIM>(jj, ax) == 0 ? 0 : 1)) * ni + r;
        enz_idx[slot] = -q - 1;
        enz_val[slot] = v;
      } else {
        E[(long long)(-q - 1) * ni + r] = v;
      }
    }
  }
  // RHS column 0 of the augmented block: sgn * f(I_i)
  for (int r = tid; r < ni; r += nthr) M[(long long)ni * ldM + r] = a.fsign * s.fsrc[a.interior[r]];
  __syncthreads();
}

template <class SM>
__device__ __forceinline__ void leaf_assemble_block(const LeafAsmArgs& a, long long leaf, double* M, long long ldM,
                                                    double* E, SM& s, int* enz_idx = nullptr,
                                                    double* enz_val = nullptr) {
  if (a.dim == 3)
    leaf_assemble_block_t<3>(a, leaf, M, ldM, E, s, enz_idx, enz_val);
  else
    leaf_assemble_block_t<2>(a, leaf, M, ldM, E, s, enz_idx, enz_val);
}

}  // namespace hpsk
