// hps_kernels.cu -- see hps_kernels.cuh.
#include <climits>
#include <stdexcept>

#include "hps_kernels.cuh"
#include "leaf_common.cuh"

namespace hpsk {

namespace {

constexpr int kAsmThreads = 256;

__global__ void __launch_bounds__(kAsmThreads) leaf_assemble_kernel(const LeafAsmArgs a) {
  __shared__ LeafAsmSmem s;
  const long long leaf = blockIdx.x;
  leaf_assemble_block(a, leaf, a.M + leaf * a.strideM, a.ni, a.E + leaf * a.strideE, s);
  if (threadIdx.x == 0) a.bad_point[leaf] = s.bad;  // INT_MAX: all samples finite
}

__global__ void __launch_bounds__(kAsmThreads) iti_leaf_assemble_kernel(const ItiLeafArgs ia) {
  __shared__ LeafAsmSmem s;
  const LeafAsmArgs& a = ia.a;
  const long long leaf = blockIdx.x;
  const int tid = threadIdx.x, p = a.p, n = a.n, n2 = 2 * n, nbc = ia.nbc, nbq = ia.nbq;
  const long long ld = n2, ncol = n2 + 1 + 2 * nbq;
  double* M = a.M + leaf * a.strideM;
  // zero fill (16-byte stores)
  double2* m2 = reinterpret_cast<double2*>(M);
  for (long long e = tid; e < ld * ncol / 2; e += kAsmThreads) m2[e] = make_double2(0.0, 0.0);
  if (tid == 0) s.bad = INT_MAX;
  for (int e = tid; e < p * p; e += kAsmThreads) s.D[e] = a.D[e], s.D2[e] = a.D2[e];
  __syncthreads();
  // coefficients and source at the leaf Chebyshev points (leaf_cheb_points, mesh.cpp:320-336)
  const double* box = a.leaf_box + leaf * 6;
  for (int i = tid; i < n; i += kAsmThreads) {
    int ci[3];
    leaf_decode(i, p, 2, ci);
    double x[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < 2; ++k)
      x[k] = __dadd_rn(__dmul_rn(0.5, __dadd_rn(box[k], box[3 + k])),
                       __dmul_rn(__dmul_rn(0.5, __dsub_rn(box[3 + k], box[k])), a.cheb[ci[k]]));
    for (int t = 0; t < a.nterms; ++t) {
      const double v = eval_field(a.terms[t].f, x, 2, leaf, i, n);
      s.coef[t][i] = v;
      if (!isfinite(v)) atomicMin(&s.bad, i);
    }
    s.fsrc[i] = a.has_source ? eval_field(a.source, x, 2, leaf, i, n) : 0.0;
  }
  __syncthreads();
  // G rows (complex, shared by all leaves): [[Gr, -Gi], [Gi, Gr]]
  for (int e = tid; e < nbc * n; e += kAsmThreads) {
    const int r = e % nbc, c = e / nbc;
    const double gr = ia.Gr[(long long)c * nbc + r], gi = ia.Gi[(long long)c * nbc + r];
    M[(long long)c * ld + r] = gr;
    M[(long long)(n + c) * ld + r] = -gi;
    M[(long long)c * ld + n + r] = gi;
    M[(long long)(n + c) * ld + n + r] = gr;
  }
  // interior rows of the discretized operator (real), entries on the grid lines through the point
  const int per_row = 2 * (p - 1) + 1;
  for (int e = tid; e < a.ni * per_row; e += kAsmThreads) {
    const int k = e % a.ni, w = e / a.ni;
    const int gi = a.interior[k];
    int ii[3], jj[3];
    leaf_decode(gi, p, 2, ii);
    jj[0] = ii[0], jj[1] = ii[1], jj[2] = 0;
    ii[2] = 0;
    if (w > 0) {
      const int ax = (w - 1) / (p - 1), k0 = (w - 1) % (p - 1);
      jj[ax] = k0 < ii[ax] ? k0 : k0 + 1;
    }
    const int gj = jj[0] * p + jj[1];
    const double v = leaf_entry(a, s, gi, ii, gj, jj);
    M[(long long)gj * ld + nbc + k] = v;
    M[(long long)(n + gj) * ld + n + nbc + k] = v;
  }
  // source column (real f on the interior rows) and the Y right-hand sides [P; 0], i [P; 0]
  for (int k = tid; k < a.ni; k += kAsmThreads) {
    const int gi = a.interior[k];
    M[(long long)n2 * ld + nbc + k] = s.fsrc[gi];
    if (ia.has_source_im) {  // complex source: imaginary part on the imaginary rows
      int ci[3];
      leaf_decode(gi, p, 2, ci);
      double x[3] = {0.0, 0.0, 0.0};
      for (int q = 0; q < 2; ++q)
        x[q] = __dadd_rn(__dmul_rn(0.5, __dadd_rn(box[q], box[3 + q])),
                         __dmul_rn(__dmul_rn(0.5, __dsub_rn(box[3 + q], box[q])), a.cheb[ci[q]]));
      M[(long long)n2 * ld + n + nbc + k] = eval_field(ia.source_im, x, 2, leaf, gi, n);
    }
  }
  for (int e = tid; e < nbc * nbq; e += kAsmThreads) {
    const int r = e % nbc, j = e / nbc;
    const double pv = ia.P[(long long)j * nbc + r];
    M[(long long)(n2 + 1 + j) * ld + r] = pv;
    M[(long long)(n2 + 1 + nbq + j) * ld + n + r] = pv;
  }
  __syncthreads();
  if (tid == 0) a.bad_point[leaf] = s.bad;
}

__global__ void block_gather_kernel(const BlockGatherArgs a) {
  const long long node = blockIdx.x;
  const DevBlockCopy bc = a.blocks[blockIdx.y];
  double* dst = a.dst[bc.dst] + node * a.stride[bc.dst];
  const long long ld = a.ld[bc.dst];
  if (bc.child < 0) {
    for (int i = threadIdx.x; i < bc.rows; i += blockDim.x) dst[(long long)(bc.dc + i) * ld + bc.dr + i] = 1.0;
    return;
  }
  const double* src = a.child_HT + (node * a.nchild + bc.child) * a.child_stride;
  for (int e = threadIdx.x; e < bc.rows * bc.cols; e += blockDim.x) {
    const int r = e % bc.rows, c = e / bc.rows;
    dst[(long long)(bc.dc + c) * ld + bc.dr + r] = src[(long long)(bc.sc + c) * a.child_ld + bc.sr + r];
  }
}

__global__ void add_identity_kernel(double* A, int n, long long ld, long long stride) {
  double* a = A + (long long)blockIdx.x * stride;
  for (int i = threadIdx.x; i < n; i += blockDim.x) a[(long long)i * ld + i] += 1.0;
}

__global__ void copy_batched_kernel(double* dst, long long ldd, long long sd, const double* src, long long lds,
                                    long long ss, int rows, int cols) {
  const long long b = blockIdx.x;
  for (long long e = (long long)blockIdx.y * blockDim.x + threadIdx.x; e < (long long)rows * cols;
       e += (long long)gridDim.y * blockDim.x) {
    const int r = int(e % rows), c = int(e / rows);
    dst[b * sd + (long long)c * ldd + r] = src[b * ss + (long long)c * lds + r];
  }
}

__global__ void iti_leaf_output_kernel(double* u, const double* Ui, int n, int nrhs, int n_leaves) {
  const long long total = (long long)n_leaves * nrhs * n;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int pt = int(e % n);
    const long long lk = e / n;
    const long long leaf = lk % n_leaves;
    const int k = int(lk / n_leaves);
    const double* src = Ui + leaf * (2LL * n * nrhs) + (long long)k * 2 * n;
    u[2 * e] = src[pt];
    u[2 * e + 1] = src[n + pt];
  }
}

__global__ void complex_to_planar_kernel(double* g_re, const double* g, int nb, int nrhs) {
  const long long total = (long long)nb * nrhs;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = int(e % nb), k = int(e / nb);
    g_re[(long long)k * 2 * nb + r] = g[2 * e];
    g_re[(long long)k * 2 * nb + nb + r] = g[2 * e + 1];
  }
}

__global__ void evaluate_at_kernel(const EvalArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.npts) return;
  const int p = a.p, dim = a.dim, nchild = dim == 2 ? 4 : 8;
  double x[3] = {a.x[3 * i], a.x[3 * i + 1], a.x[3 * i + 2]};
  double lo[3] = {a.lo, a.lo, a.lo}, hi[3] = {a.hi, a.hi, a.hi};
  long long ord = 0;
  for (int l = 0; l < a.L; ++l) {  // locate_leaf: child slot of the offsets (downpass.cpp:13-27)
    int o[3] = {0, 0, 0};
    for (int k = 0; k < dim; ++k) {
      const double mid = 0.5 * (lo[k] + hi[k]);
      o[k] = x[k] >= mid ? 1 : 0;
      if (o[k]) lo[k] = mid; else hi[k] = mid;
    }
    const int q = (o[0] == 0 && o[1] == 0) ? 0 : (o[0] == 1 && o[1] == 0) ? 1 : (o[0] == 1 && o[1] == 1) ? 2 : 3;
    ord = ord * nchild + q + (dim == 3 && o[2] ? 4 : 0);
  }
  // barycentric weights of the Chebyshev-Lobatto interpolant (downpass.cpp:31-53)
  double w[3][kLeafMaxP];
  for (int k = 0; k < dim; ++k) {
    const double t = (2.0 * x[k] - lo[k] - hi[k]) / (hi[k] - lo[k]);
    int hit = -1;
    for (int j = 0; j < p; ++j)
      if (t == a.cheb[j]) hit = j;
    if (hit >= 0) {
      for (int j = 0; j < p; ++j) w[k][j] = j == hit ? 1.0 : 0.0;
      continue;
    }
    double den = 0.0;
    for (int j = 0; j < p; ++j) {
      double bw = (j % 2 == 0) ? 1.0 : -1.0;
      if (j == 0 || j == p - 1) bw *= 0.5;
      w[k][j] = bw / (t - a.cheb[j]);
      den += w[k][j];
    }
    for (int j = 0; j < p; ++j) w[k][j] /= den;
  }
  const long long np = dim == 2 ? (long long)p * p : (long long)p * p * p;
  const double* u = a.u + ord * np * (a.is_complex ? 2 : 1);
  double re = 0.0, im = 0.0;
  for (int i1 = 0; i1 < p; ++i1) {
    if (w[0][i1] == 0.0) continue;
    for (int i2 = 0; i2 < p; ++i2) {
      if (w[1][i2] == 0.0) continue;
      const double w12 = w[0][i1] * w[1][i2];
      for (int i3 = 0; i3 < (dim == 3 ? p : 1); ++i3) {
        const double ww = dim == 3 ? w12 * w[2][i3] : w12;
        const long long idx = dim == 3 ? ((long long)i1 * p + i2) * p + i3 : (long long)i1 * p + i2;
        if (a.is_complex) {
          re += ww * u[2 * idx];
          im += ww * u[2 * idx + 1];
        } else {
          re += ww * u[idx];
        }
      }
    }
  }
  if (a.is_complex) {
    a.out[2 * i] = re;
    a.out[2 * i + 1] = im;
  } else {
    a.out[i] = re;
  }
}

__global__ void __launch_bounds__(256) error_partials_kernel(const ErrArgs a) {
  __shared__ double red[4][256];
  const long long total = a.n_leaves * a.npts_leaf;
  double ninf = 0.0, dinf = 0.0, n2 = 0.0, d2 = 0.0;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long leaf = e / a.npts_leaf;
    const int pt = int(e % a.npts_leaf);
    int ci[3];
    leaf_decode(pt, a.p, a.dim, ci);
    const double* box = a.leaf_box + leaf * 6;
    double x[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < a.dim; ++k)
      x[k] = __dadd_rn(__dmul_rn(0.5, __dadd_rn(box[k], box[3 + k])),
                       __dmul_rn(__dmul_rn(0.5, __dsub_rn(box[3 + k], box[k])), a.cheb[ci[k]]));
    const double er = eval_field(a.ex_re, x, a.dim, leaf, pt, a.npts_leaf);
    const double ei = a.has_im ? eval_field(a.ex_im, x, a.dim, leaf, pt, a.npts_leaf) : 0.0;
    const double ur = a.is_complex ? a.u[2 * e] : a.u[e], ui = a.is_complex ? a.u[2 * e + 1] : 0.0;
    const double dr = ur - er, di = ui - ei;
    ninf = fmax(ninf, sqrt(dr * dr + di * di));
    dinf = fmax(dinf, sqrt(er * er + ei * ei));
    n2 += dr * dr + di * di;
    d2 += er * er + ei * ei;
  }
  red[0][threadIdx.x] = ninf, red[1][threadIdx.x] = dinf, red[2][threadIdx.x] = n2, red[3][threadIdx.x] = d2;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      red[0][threadIdx.x] = fmax(red[0][threadIdx.x], red[0][threadIdx.x + o]);
      red[1][threadIdx.x] = fmax(red[1][threadIdx.x], red[1][threadIdx.x + o]);
      red[2][threadIdx.x] += red[2][threadIdx.x + o];
      red[3][threadIdx.x] += red[3][threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x < 4) a.partial[blockIdx.x * 4 + threadIdx.x] = red[threadIdx.x][0];
}

constexpr int kGatherThreads = 256;

// One warp per destination column: (slot, cc) are uniform over the column and the rows of each
// section are a contiguous run in both source and destination, so loads and stores coalesce.  The
// column's per-section source offsets (at most 32 sections: NI, NE <= 24) are resolved once into shared
// memory; a row then costs one multiply-high (section = r / s) and one shared load per source.
__global__ void __launch_bounds__(kGatherThreads) gather_kernel(const GatherArgs a) {
  __shared__ long long soff[kGatherThreads / 32][32][2];
  const long long node = blockIdx.x;
  const int s = a.s;
  const int nslots = a.kind == 0 ? a.NI + 1 + a.NE : (a.kind == 1 ? a.NI : 1 + a.NE);
  double* dst = a.dst + node * a.stride + blockIdx.z * a.dst_rhs_stride;
  const double* ch0 = a.child_HT + node * a.nchild * a.child_stride + blockIdx.z * a.src_rhs_stride;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kGatherThreads / 32;
  const int nsec = (a.nrows + s - 1) / s;   // <= 32 (launch_gather)
  for (int dcolumn = blockIdx.y * nw + warp; dcolumn < a.ncols; dcolumn += gridDim.y * nw) {
    const int col = dcolumn + a.col_offset;
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
    } else if (col == 0) {
      slot = 0;
      cc = 0;
    } else {
      slot = 1 + (col - 1) / s;
      cc = (col - 1) % s;
    }
    __syncwarp();
    if (lane < nsec) {
      const int* tab = a.src + 2 * (lane * nslots + slot);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int code = __ldg(tab + k);
        long long o = -1;
        if (code >= 0) {
          const int child = code >> 6, rf = (code >> 3) & 7, cfp1 = code & 7;
          const long long hc = cfp1 == 0 ? 0 : 1 + (long long)(cfp1 - 1) * s + cc;
          o = child * a.child_stride + hc * a.child_nb + rf * s;
        }
        soff[warp][lane][k] = o;
      }
    }
    __syncwarp();
    double* dcol = dst + (long long)dcolumn * a.ld;
    // four rows per lane per batch: every operand load of the batch is issued before its stores
    // (the sources are read-only here, __ldg), so the loop is not one memory latency per row
    for (int r0 = lane; r0 < a.nrows; r0 += 128) {
      double v[4];
      bool nz[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = r0 + 32 * q;
        v[q] = 0.0;
        nz[q] = false;
        if (r < a.nrows) {
          const int rsec = a.smagic ? (int)__umulhi((unsigned)r, a.smagic) : r / s, rr = r - rsec * s;
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const long long o = soff[warp][rsec][k];
            if (o < 0) continue;
            nz[q] = true;
            v[q] += __ldg(ch0 + o + rr);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = r0 + 32 * q;
        if (r < a.nrows && (nz[q] || !a.skip_zero) &&
            (!a.row_mask || a.row_mask[node * nsec + (a.smagic ? (int)__umulhi((unsigned)r, a.smagic) : r / s)]))
          dcol[r] = v[q];
      }
    }
  }
}

// ItI real-equivalent columns of an imaginary unit are i times those of the matching real unit: for a complex
// column z stored as rows (re_row(o), im_row(o)), the column of i z holds (-im, re).  Fills columns
// [col_im0, col_im0 + ncols) from [col_re0, ...) of every node; half-blocked interface order (hc > 0:
// re_row(o) = o < hc ? o : 2 hc + (o - hc), im_row = re_row + hc) or plain exterior order (hc = 0:
// re_row(o) = o, im_row = o + nc).
__global__ void iti_fill_im_half_kernel(double* X, long long ld, long long stride, int nc, int hc, int col_re0,
                                        int col_im0, int ncols) {
  double* Xb = X + blockIdx.x * stride;
  const long long tot = (long long)nc * ncols;
  for (long long e = blockIdx.y * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.y * blockDim.x) {
    const int j = int(e / nc), o = int(e - (long long)j * nc);
    const int rr = hc ? (o < hc ? o : 2 * hc + (o - hc)) : o;
    const int ri = hc ? rr + hc : o + nc;
    const double re = Xb[(long long)(col_re0 + j) * ld + rr], im = Xb[(long long)(col_re0 + j) * ld + ri];
    Xb[(long long)(col_im0 + j) * ld + rr] = -im;
    Xb[(long long)(col_im0 + j) * ld + ri] = re;
  }
}

// ItI leaf by block elimination (run_leaf_stage): the leaf's [v | Y | iY] columns in real-equivalent tensor
// order from the interior solution U_i = W U_e (+ z on the source column) and the exterior solution U_e.
__global__ void iti_fdm_assemble_kernel(const ItiFdmAssembleArgs a) {
  const long long leaf = blockIdx.x;
  const double* Z = a.Z + leaf * a.stride;       // z_re, z_im: columns 0, 1 (nir each)
  const double* Ue = a.Ue + leaf * a.stride;     // 2 ne x mrhs, ld 2 ne
  const double* Ure = a.Ure + leaf * a.stride;   // nir x mrhs
  const double* Uim = a.Uim + leaf * a.stride;
  double* M = a.M + leaf * a.stride;             // [v | Y | iY]: 2n x mrhs, ld 2n
  const int n = a.n, ne = a.ne, nir = a.nir;
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < n * a.mrhs; e += gridDim.y * blockDim.x) {
    const int c = e / n, t = e - c * n;
    const int pos = a.pos[t];
    double re, im;
    if (pos >= 0) {
      re = Ure[(long long)c * nir + pos];
      im = Uim[(long long)c * nir + pos];
      if (c == 0) re += Z[pos], im += Z[nir + pos];
    } else {
      const int x = -pos - 1;
      re = Ue[(long long)c * 2 * ne + x];
      im = Ue[(long long)c * 2 * ne + ne + x];
    }
    M[(long long)c * 2 * n + t] = re;
    M[(long long)c * 2 * n + n + t] = im;
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
      v = a.lead;
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

__global__ void pack_root_kernel(double* G, const double* g, int nb, int nrhs, double lead) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int rows = nb + 1;
  if (e >= (long long)rows * nrhs) return;
  const int r = int(e % rows), c = int(e / rows);
  G[e] = r == 0 ? lead : g[(long long)c * nb + r - 1];
}

__global__ void unpack_leaf_g_kernel(double* out, const double* G, int nb, long long ldg, int nrhs, int n_leaves) {
  const long long total = (long long)nb * nrhs * n_leaves;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = int(e % nb);
    const long long lr = e / nb;
    const long long leaf = lr % n_leaves;
    const int rhs = int(lr / n_leaves);
    out[e] = G[leaf * ldg * nrhs + (long long)rhs * ldg + 1 + r];
  }
}

}  // namespace

void launch_iti_leaf_assemble(const ItiLeafArgs& a, int n_leaves, cudaStream_t st) {
  iti_leaf_assemble_kernel<<<n_leaves, kAsmThreads, 0, st>>>(a);
}
void launch_block_gather(const BlockGatherArgs& a, int n_nodes, cudaStream_t st) {
  if (a.nblocks <= 0 || n_nodes <= 0) return;
  block_gather_kernel<<<dim3(n_nodes, a.nblocks), 256, 0, st>>>(a);
}
void launch_add_identity(double* A, int n, long long ld, long long stride, int batch, cudaStream_t st) {
  if (batch > 0 && n > 0) add_identity_kernel<<<batch, 256, 0, st>>>(A, n, ld, stride);
}
void launch_copy_batched(double* dst, long long ldd, long long sd, const double* src, long long lds, long long ss,
                         int rows, int cols, int batch, cudaStream_t st) {
  if (batch <= 0 || rows <= 0 || cols <= 0) return;
  const long long e = (long long)rows * cols;
  const int gy = int(std::min<long long>(std::max<long long>(1, (148LL * 8 + batch - 1) / batch), (e + 255) / 256));
  copy_batched_kernel<<<dim3(batch, std::max(1, std::min(gy, 65535))), 256, 0, st>>>(dst, ldd, sd, src, lds, ss, rows,
                                                                                     cols);
}
void launch_iti_fill_im_half(double* X, long long ld, long long stride, int batch, int nc, int hc, int col_re0,
                             int col_im0, int ncols, cudaStream_t st) {
  const long long tot = (long long)nc * ncols;
  const int gy = (int)std::max<long long>(1, std::min<long long>((tot + 255) / 256, (148LL * 8 + batch - 1) / batch));
  iti_fill_im_half_kernel<<<dim3(batch, gy), 256, 0, st>>>(X, ld, stride, nc, hc, col_re0, col_im0, ncols);
}
void launch_iti_fdm_assemble(const ItiFdmAssembleArgs& a, int n_leaves, cudaStream_t st) {
  const int gy = std::max(1, std::min(64, (a.n * a.mrhs + 255) / 256));
  iti_fdm_assemble_kernel<<<dim3(n_leaves, gy), 256, 0, st>>>(a);
}
void launch_iti_leaf_output(double* u, const double* Ui, int n, int nrhs, int n_leaves, cudaStream_t st) {
  const long long total = (long long)n_leaves * nrhs * n;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 64);
  iti_leaf_output_kernel<<<blocks, 256, 0, st>>>(u, Ui, n, nrhs, n_leaves);
}
void launch_complex_to_planar(double* g_re, const double* g, int nb, int nrhs, cudaStream_t st) {
  const long long total = (long long)nb * nrhs;
  complex_to_planar_kernel<<<(unsigned)std::max<long long>(1, (total + 255) / 256), 256, 0, st>>>(g_re, g, nb, nrhs);
}

void launch_evaluate_at(const EvalArgs& a, cudaStream_t st) {
  if (a.npts <= 0) return;
  evaluate_at_kernel<<<(a.npts + 127) / 128, 128, 0, st>>>(a);
}
int launch_error_partials(const ErrArgs& a, cudaStream_t st) {
  const int blocks = 148 * 4;
  error_partials_kernel<<<blocks, 256, 0, st>>>(a);
  return blocks;
}

void launch_leaf_assemble(const LeafAsmArgs& a, int n_leaves, cudaStream_t st) {
  leaf_assemble_kernel<<<n_leaves, kAsmThreads, 0, st>>>(a);
}

void launch_gather(const GatherArgs& a0, int n_nodes, cudaStream_t st) {
  GatherArgs a = a0;
  if ((a.nrows + a.s - 1) / a.s > 32) throw std::runtime_error("gather: more than 32 row sections");
  // r / s as a multiply-high by ceil(2^32 / s): exact while r * s < 2^32
  a.smagic = (a.s > 1 && (long long)a.nrows * a.s < (1LL << 32)) ? unsigned(((1ULL << 32) + a.s - 1) / a.s) : 0u;
  const int nw = kGatherThreads / 32;
  // enough column groups to fill the GPU (~8 CTAs per SM over all nodes), each warp a column
  const long long want = std::max<long long>(1, (148LL * 8 + n_nodes - 1) / n_nodes);
  const long long groups = std::min<long long>((a.ncols + nw - 1) / nw, std::max<long long>(want, 1));
  dim3 grid(n_nodes, (unsigned)std::min<long long>(groups, 65535), a.nrhs);
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

void launch_pack_root(double* G, const double* g, int nb, int nrhs, cudaStream_t st, double lead) {
  const long long tot = (long long)(nb + 1) * nrhs;
  pack_root_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(G, g, nb, nrhs, lead);
}

namespace {
__global__ void pack_source_kernel(double* R, const double* f, const int* interior, int ni, int npts, int n_leaves,
                                   int nrhs, double sgn) {
  const long long total = (long long)n_leaves * nrhs * ni;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = int(e % ni);
    const long long lk = e / ni;
    const int k = int(lk % nrhs);
    const long long leaf = lk / nrhs;
    R[e] = sgn * f[((long long)k * n_leaves + leaf) * npts + interior[r]];
  }
}
__global__ void axpby_kernel(double* y, long long ldy, long long sy, const double* x, long long ldx, long long sx,
                             int n, int nrhs, long long batch, double a, double b) {
  const long long total = batch * nrhs * n;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = int(e % n);
    const long long lk = e / n;
    const int k = int(lk % nrhs);
    const long long i = lk / nrhs;
    double* yp = y + i * sy + (long long)k * ldy + r;
    *yp = a * *yp + b * x[i * sx + (long long)k * ldx + r];
  }
}
}  // namespace

void launch_pack_source(double* R, const double* f, const int* interior, int ni, int npts, int n_leaves, int nrhs,
                        double sgn, cudaStream_t st) {
  const long long total = (long long)n_leaves * nrhs * ni;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 32);
  pack_source_kernel<<<blocks, 256, 0, st>>>(R, f, interior, ni, npts, n_leaves, nrhs, sgn);
}

void launch_axpby(double* y, long long ldy, long long sy, const double* x, long long ldx, long long sx, int n,
                  int nrhs, long long batch, double a, double b, cudaStream_t st) {
  const long long total = batch * nrhs * n;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 32);
  axpby_kernel<<<blocks, 256, 0, st>>>(y, ldy, sy, x, ldx, sx, n, nrhs, batch, a, b);
}

void launch_unpack_leaf_g(double* out, const double* G, int nb, long long ldg, int nrhs, int n_leaves, cudaStream_t st) {
  const long long total = (long long)nb * nrhs * n_leaves;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 64);
  unpack_leaf_g_kernel<<<blocks, 256, 0, st>>>(out, G, nb, ldg, nrhs, n_leaves);
}

}  // namespace hpsk
