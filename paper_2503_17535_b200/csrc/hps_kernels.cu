// hps_kernels.cu -- see hps_kernels.cuh.
#include <climits>

#include "hps_kernels.cuh"

namespace hpsk {

namespace {

constexpr int kAsmThreads = 256;
constexpr int kMaxPts = 512;  // p^d <= 512 (2D p <= 22, 3D p <= 8)
constexpr int kMaxP = 24;

__device__ double bumps(const DevField& f, const double* x, int dim) {
  double s = 0.0;
  for (int j = 0; j < f.n_centers; ++j) {
    double r2 = 0.0;
    for (int k = 0; k < dim; ++k) {
      const double d = x[k] - f.centers[3 * j + k];
      r2 += d * d;
    }
    s += exp(-f.c[2] * r2);
  }
  return s;
}

// Device evaluation of the built-in fields (hps_cuda.h HPSG_FIELD_*).
__device__ double eval_field(const DevField& f, const double* x, int dim, long long leaf, int pt, int npts) {
  const double* c = f.c;
  switch (f.kind) {
    case 0: return c[0];
    case 1: return c[0] + c[1] * bumps(f, x, dim);
    case 2: return c[0] * sin(c[1] * x[0] + c[2] * x[1] + c[3] * x[2] + c[4]);
    case 3: return c[0] * cos(c[1] * x[0] + c[2] * x[1] + c[3] * x[2] + c[4]);
    case 4: return c[0] * bumps(f, x, dim) * sin(c[3] * x[0] + c[4] * x[1] + c[5] * x[2] + c[6]);
    case 5: {  // proj/src/problems.cpp:50-66
      const double X = x[0], Y = x[1];
      const double ux = 5.0 * exp(5.0 * X) * sin(5.0 * Y) + 10.0 * M_PI * cos(10.0 * M_PI * X) * sin(M_PI * Y);
      const double uy = 5.0 * exp(5.0 * X) * cos(5.0 * Y) + M_PI * sin(10.0 * M_PI * X) * cos(M_PI * Y);
      const double lap = -101.0 * M_PI * M_PI * sin(10.0 * M_PI * X) * sin(M_PI * Y);
      return lap - cos(5.0 * Y) * ux + sin(5.0 * Y) * uy;
    }
    case 6: return f.samples[leaf * npts + pt];
    default: return __longlong_as_double(0x7ff8000000000000ULL);
  }
}

__device__ __forceinline__ void decode(int idx, int p, int dim, int* c) {
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

__global__ void __launch_bounds__(kAsmThreads) leaf_assemble_kernel(const LeafAsmArgs a) {
  __shared__ double coef[kMaxTerms][kMaxPts];
  __shared__ double fsrc[kMaxPts];
  __shared__ double sD[kMaxP * kMaxP], sD2[kMaxP * kMaxP];
  __shared__ int bad;
  const long long leaf = blockIdx.x;
  const int tid = threadIdx.x, p = a.p, dim = a.dim, n = a.n;
  if (tid == 0) bad = INT_MAX;
  for (int e = tid; e < p * p; e += kAsmThreads) sD[e] = a.D[e], sD2[e] = a.D2[e];
  const double* box = a.leaf_box + leaf * 6;
  // leaf_cheb_points (proj/src/mesh.cpp:320-336): 0.5(lo+hi) + 0.5(hi-lo) t, no FMA contraction
  for (int i = tid; i < n; i += kAsmThreads) {
    int ci[3];
    decode(i, p, dim, ci);
    double x[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < dim; ++k)
      x[k] = __dadd_rn(__dmul_rn(0.5, __dadd_rn(box[k], box[3 + k])),
                       __dmul_rn(__dmul_rn(0.5, __dsub_rn(box[3 + k], box[k])), a.cheb[ci[k]]));
    for (int t = 0; t < a.nterms; ++t) {
      const double v = eval_field(a.terms[t].f, x, dim, leaf, i, n);
      coef[t][i] = v;
      if (!isfinite(v)) atomicMin(&bad, i);
    }
    fsrc[i] = a.has_source ? eval_field(a.source, x, dim, leaf, i, n) : 0.0;
  }
  __syncthreads();
  if (tid == 0) a.bad_point[leaf] = bad;  // INT_MAX: all samples finite

  const double s1 = a.scale, s2 = a.scale * a.scale;
  double* M = a.M + leaf * a.strideM;
  double* E = a.E + leaf * a.strideE;
  const int ni = a.ni, ncol = ni + a.ne;
  // L(ii, :) entry by entry; accumulation order = term order, axis order (local_solve.cpp:63-83)
  for (int e = tid; e < ni * ncol; e += kAsmThreads) {
    const int r = e % ni, cj = e / ni;
    const int gi = a.interior[r];
    const int gj = cj < ni ? a.interior[cj] : a.exterior[cj - ni];
    int ii[3], jj[3];
    decode(gi, p, dim, ii);
    decode(gj, p, dim, jj);
    bool same[3];
    for (int k = 0; k < 3; ++k) same[k] = ii[k] == jj[k];
    double val = 0.0;
    for (int t = 0; t < a.nterms; ++t) {
      const DevTerm& tm = a.terms[t];
      const double c = coef[t][gi];
      switch (tm.role) {
        case 0:  // laplacian: c s^2 sum_a D2_a
          for (int ax = 0; ax < dim; ++ax) {
            bool ok = true;
            for (int k = 0; k < dim; ++k)
              if (k != ax && !same[k]) ok = false;
            if (ok) val = __dadd_rn(val, __dmul_rn(s2, __dmul_rn(c, sD2[jj[ax] * p + ii[ax]])));
          }
          break;
        case 1: {  // gradient: c s D_axis
          const int ax = tm.axis;
          bool ok = true;
          for (int k = 0; k < dim; ++k)
            if (k != ax && !same[k]) ok = false;
          if (ok) val = __dadd_rn(val, __dmul_rn(s1, __dmul_rn(c, sD[jj[ax] * p + ii[ax]])));
          break;
        }
        case 2:  // zeroth: diag(c)
          if (gi == gj) val = __dadd_rn(val, c);
          break;
        default: {  // second_order
          const int a1 = tm.axis, a2 = tm.axis2;
          if (a1 == a2) {
            bool ok = true;
            for (int k = 0; k < dim; ++k)
              if (k != a1 && !same[k]) ok = false;
            if (ok) val = __dadd_rn(val, __dmul_rn(s2, __dmul_rn(c, sD2[jj[a1] * p + ii[a1]])));
          } else {
            bool ok = true;
            for (int k = 0; k < dim; ++k)
              if (k != a1 && k != a2 && !same[k]) ok = false;
            if (ok) {
              const double d = __dmul_rn(sD[jj[a1] * p + ii[a1]], sD[jj[a2] * p + ii[a2]]);
              val = __dadd_rn(val, __dmul_rn(s2, __dmul_rn(c, d)));
            }
          }
        }
      }
    }
    if (cj < ni)
      M[(long long)cj * ni + r] = val;
    else
      E[(long long)(cj - ni) * ni + r] = val;
  }
  // RHS column 0 of the augmented block: sgn * f(I_i)
  for (int r = tid; r < ni; r += kAsmThreads) M[(long long)ni * ni + r] = a.fsign * fsrc[a.interior[r]];
}

constexpr int kGatherThreads = 256;
constexpr int kGatherPerThread = 4;

__global__ void __launch_bounds__(kGatherThreads) gather_kernel(const GatherArgs a) {
  const long long node = blockIdx.x;
  const long long total = (long long)a.nrows * a.ncols;
  const int s = a.s;
  const int nslots = a.kind == 0 ? a.NI + 1 + a.NE : (a.kind == 1 ? a.NI : 1 + a.NE);
  double* dst = a.dst + node * a.stride;
  const double* ch0 = a.child_HT + node * a.nchild * a.child_stride;
  for (long long base = (long long)blockIdx.y * kGatherThreads * kGatherPerThread; base < total;
       base += (long long)gridDim.y * kGatherThreads * kGatherPerThread)
#pragma unroll
  for (int it = 0; it < kGatherPerThread; ++it) {
    const long long e = base + it * kGatherThreads + threadIdx.x;
    if (e >= total) break;
    const int r = int(e % a.nrows), col = int(e / a.nrows);
    const int rsec = r / s, rr = r % s;
    int slot, cc;
    if (a.kind == 0) {
      const int nd = a.NI * s;
      if (col < nd) {
        slot = col / s;
        cc = col % s;
      } else if (col == nd) {
        slot = a.NI;
        cc = 0;
      } else {
        const int c2 = col - nd - 1;
        slot = a.NI + 1 + c2 / s;
        cc = c2 % s;
      }
    } else if (a.kind == 1) {
      slot = col / s;
      cc = col % s;
    } else {
      if (col == 0) {
        slot = 0;
        cc = 0;
      } else {
        slot = 1 + (col - 1) / s;
        cc = (col - 1) % s;
      }
    }
    const int* tab = a.src + 2 * (rsec * nslots + slot);
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int code = tab[k];
      if (code < 0) continue;
      const int child = code >> 6, rf = (code >> 3) & 7, cfp1 = code & 7;
      const double* T = ch0 + child * a.child_stride;
      const long long hc = cfp1 == 0 ? 0 : 1 + (long long)(cfp1 - 1) * s + cc;
      v += T[hc * a.child_nb + rf * s + rr];
    }
    dst[(long long)col * a.ld + r] = v;
  }
}

__global__ void scatter_kernel(const ScatterArgs a) {
  const long long parent = blockIdx.x;
  const int child_nb = a.nface * a.s;
  const int rows = 1 + child_nb;
  const double* Gp = a.Gp + parent * a.strideGp;
  const double* GI = a.GI + parent * a.strideGI;
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < a.nchild * rows * a.nrhs; e += gridDim.y * blockDim.x) {
    const int r = e % rows;
    const int rhs = (e / rows) % a.nrhs;
    const int c = e / (rows * a.nrhs);
    double v;
    if (r == 0) {
      v = 1.0;
    } else {
      const int f = (r - 1) / a.s, i = (r - 1) % a.s;
      const int d = a.down[c * a.nface + f];
      v = d >= 0 ? Gp[(long long)rhs * a.ldGp + 1 + d + i] : GI[(long long)rhs * a.ldGI + (-d - 1) + i];
    }
    a.Gc[(parent * a.nchild + c) * a.strideGc + (long long)rhs * a.ldGc + r] = v;
  }
}

__global__ void neg_add_kernel(double* GI, const double* xh, int n, int nrhs, long long ld) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)n * nrhs) return;
  const int r = int(e % n), c = int(e / n);
  GI[c * ld + r] = -(GI[c * ld + r] + xh[r]);
}

__global__ void leaf_output_kernel(const LeafOutArgs a) {
  const long long total = (long long)a.n_leaves * a.npts * a.nrhs;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    // e indexes the output in [rhs][leaf][pos] order, pos over (interior | exterior)
    const int pos = int(e % a.npts);
    const long long lr = e / a.npts;
    const long long leaf = lr % a.n_leaves;
    const int rhs = int(lr / a.n_leaves);
    double v;
    int idx;
    if (pos < a.ni) {
      v = a.Ui[leaf * a.strideUi + (long long)rhs * a.ldUi + pos];
      idx = a.interior[pos];
    } else {
      v = a.Ue[leaf * a.strideUe + (long long)rhs * a.ldUe + pos - a.ni];
      idx = a.exterior[pos - a.ni];
    }
    a.u[((long long)rhs * a.n_leaves + leaf) * a.npts + idx] = v;
  }
}

__global__ void pack_root_kernel(double* G, const double* g, int nb, int nrhs) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int rows = nb + 1;
  if (e >= (long long)rows * nrhs) return;
  const int r = int(e % rows), c = int(e / rows);
  G[e] = r == 0 ? 1.0 : g[(long long)c * nb + r - 1];
}

__global__ void unpack_leaf_g_kernel(double* out, const double* G, int nb, int nrhs, int n_leaves) {
  const long long total = (long long)nb * nrhs * n_leaves;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = int(e % nb);
    const long long lr = e / nb;
    const long long leaf = lr % n_leaves;
    const int rhs = int(lr / n_leaves);
    out[e] = G[leaf * (long long)(nb + 1) * nrhs + (long long)rhs * (nb + 1) + 1 + r];
  }
}

}  // namespace

void launch_leaf_assemble(const LeafAsmArgs& a, int n_leaves, cudaStream_t st) {
  leaf_assemble_kernel<<<n_leaves, kAsmThreads, 0, st>>>(a);
}

void launch_gather(const GatherArgs& a, int n_nodes, cudaStream_t st) {
  const long long total = (long long)a.nrows * a.ncols;
  const long long per = kGatherThreads * kGatherPerThread;
  dim3 grid(n_nodes, (unsigned)std::min<long long>((total + per - 1) / per, 65535));
  gather_kernel<<<grid, kGatherThreads, 0, st>>>(a);
}

void launch_scatter(const ScatterArgs& a, int n_parents, cudaStream_t st) {
  const long long per_parent = (long long)a.nchild * (1 + a.nface * a.s) * a.nrhs;
  int gy = (int)std::min<long long>((per_parent + 255) / 256, 65535);
  scatter_kernel<<<dim3(n_parents, gy), 256, 0, st>>>(a);
}

void launch_neg_add(double* GI, const double* xh, int n, int nrhs, long long ld, cudaStream_t st) {
  const long long tot = (long long)n * nrhs;
  neg_add_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(GI, xh, n, nrhs, ld);
}

void launch_leaf_output(const LeafOutArgs& a, cudaStream_t st) {
  const long long total = (long long)a.n_leaves * a.npts * a.nrhs;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 64);
  leaf_output_kernel<<<blocks, 256, 0, st>>>(a);
}

void launch_pack_root(double* G, const double* g, int nb, int nrhs, cudaStream_t st) {
  const long long tot = (long long)(nb + 1) * nrhs;
  pack_root_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(G, g, nb, nrhs);
}

void launch_unpack_leaf_g(double* out, const double* G, int nb, int nrhs, int n_leaves, cudaStream_t st) {
  const long long total = (long long)nb * nrhs * n_leaves;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 64);
  unpack_leaf_g_kernel<<<blocks, 256, 0, st>>>(out, G, nb, nrhs, n_leaves);
}

}  // namespace hpsk
