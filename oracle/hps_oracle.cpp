// hps_oracle.cpp -- TEST INFRASTRUCTURE ONLY (see hps_oracle.hpp header).
// CPU restatement of the reference HPS hot path; each function cites the
// reference file:line (relative to /root/reference/proj) it follows.
#include "hps_oracle.hpp"

#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <omp.h>
#include <sstream>

namespace hpso {

// ============================================================================
// BLAS / LAPACK binding (OpenBLAS shipped with scipy, LP64), naive fallback.
// ============================================================================
namespace {
using dgemm_t = void (*)(const char*, const char*, const int*, const int*, const int*, const double*,
                         const double*, const int*, const double*, const int*, const double*, double*,
                         const int*, size_t, size_t);
using dgetrf_t = void (*)(const int*, const int*, double*, const int*, int*, int*);
using dgetrs_t = void (*)(const char*, const int*, const int*, const double*, const int*, const int*,
                          double*, const int*, int*, size_t);
using setthr_t = void (*)(int);
struct Blas {
  dgemm_t dgemm = nullptr;
  dgetrf_t dgetrf = nullptr;
  dgetrs_t dgetrs = nullptr;
  setthr_t setthr = nullptr;
  bool ok = false;
};
Blas& blas() {
  static Blas b;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = std::getenv("HPSO_OPENBLAS");
    const char* path = env ? env :
#ifdef HPSO_OPENBLAS_PATH
                           HPSO_OPENBLAS_PATH;
#else
                           nullptr;
#endif
    if (std::getenv("HPSO_NO_BLAS") || !path) return;
    void* h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
    b.dgemm = (dgemm_t)dlsym(h, "scipy_dgemm_");
    b.dgetrf = (dgetrf_t)dlsym(h, "scipy_dgetrf_");
    b.dgetrs = (dgetrs_t)dlsym(h, "scipy_dgetrs_");
    b.setthr = (setthr_t)dlsym(h, "scipy_openblas_set_num_threads");
    b.ok = b.dgemm && b.dgetrf && b.dgetrs;
  });
  return b;
}
}  // namespace

int blas_available() { return blas().ok ? 1 : 0; }
void set_blas_threads(int n) {
  if (blas().ok && blas().setthr) blas().setthr(n);
}

void gemm(double alpha, const Mat& A, const Mat& B, double beta, Mat& C) {
  require(A.c == B.r && C.r == A.r && C.c == B.c, "gemm: shape mismatch");
  if (A.r == 0 || B.c == 0) return;
  if (A.c == 0) {
    for (double& x : C.a) x *= beta;
    return;
  }
  if (blas().ok) {
    const int m = A.r, n = B.c, k = A.c;
    blas().dgemm("N", "N", &m, &n, &k, &alpha, A.data(), &m, B.data(), &k, &beta, C.data(), &m, 1, 1);
    return;
  }
  for (int j = 0; j < C.c; ++j) {
    for (int i = 0; i < C.r; ++i) C(i, j) *= beta;
    for (int l = 0; l < A.c; ++l) {
      const double b = alpha * B(l, j);
      if (b == 0.0) continue;
      for (int i = 0; i < C.r; ++i) C(i, j) += A(i, l) * b;
    }
  }
}

Mat matmul(const Mat& A, const Mat& B) {
  Mat C(A.r, B.c);
  gemm(1.0, A, B, 0.0, C);
  return C;
}

// Eigen::PartialPivLU restated as LAPACK getrf (same partial-pivoting rule).
void LU::compute(const Mat& A) {
  require(A.r == A.c, "LU: square matrix required");
  lu = A;
  n = A.r;
  piv.assign(n, 0);
  if (n == 0) return;
  if (blas().ok) {
    int info = 0;
    blas().dgetrf(&n, &n, lu.data(), &n, piv.data(), &info);
    return;  // zero pivots are reported by the callers' pivot checks
  }
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = std::abs(lu(k, k));
    for (int i = k + 1; i < n; ++i)
      if (std::abs(lu(i, k)) > best) best = std::abs(lu(i, k)), p = i;
    piv[k] = p + 1;
    if (p != k)
      for (int j = 0; j < n; ++j) std::swap(lu(k, j), lu(p, j));
    const double d = lu(k, k);
    if (d == 0.0) continue;
    for (int i = k + 1; i < n; ++i) lu(i, k) /= d;
    for (int j = k + 1; j < n; ++j) {
      const double u = lu(k, j);
      if (u == 0.0) continue;
      for (int i = k + 1; i < n; ++i) lu(i, j) -= lu(i, k) * u;
    }
  }
}

Mat LU::solve(const Mat& B) const {
  require(B.r == n, "LU::solve: shape mismatch");
  Mat X = B;
  if (n == 0 || B.c == 0) return X;
  if (blas().ok) {
    int info = 0, nrhs = B.c;
    blas().dgetrs("N", &n, &nrhs, lu.data(), &n, piv.data(), X.data(), &n, &info, 1);
    return X;
  }
  for (int j = 0; j < X.c; ++j) {
    double* x = &X(0, j);
    for (int k = 0; k < n; ++k)
      if (piv[k] - 1 != k) std::swap(x[k], x[piv[k] - 1]);
    for (int k = 0; k < n; ++k)
      for (int i = k + 1; i < n; ++i) x[i] -= lu(i, k) * x[k];
    for (int k = n - 1; k >= 0; --k) {
      x[k] /= lu(k, k);
      for (int i = 0; i < k; ++i) x[i] -= lu(i, k) * x[k];
    }
  }
  return X;
}

Vec LU::solve(const Vec& b) const {
  Mat B(int(b.size()), 1);
  B.a = b;
  return solve(B).a;
}

// ============================================================================
// spectral: proj/src/spectral.cpp
// ============================================================================

// proj/src/spectral.cpp:14-26
Vec cheb_lobatto_1d(int p) {
  require(p >= 2, "cheb_lobatto_1d: p must be >= 2");
  const int n = p - 1;
  Vec x(p);
  for (int k = 0; k <= n / 2; ++k) {
    const double v = std::sin(M_PI * (n - 2 * k) / (2.0 * n));
    x[k] = v;
    x[n - k] = -v;
  }
  if (n % 2 == 0) x[n / 2] = 0.0;
  return x;
}

// proj/src/spectral.cpp:28-49
Vec cheb_lobatto_weights(int p) {
  const int n = p - 1;
  Vec w(p, 0.0);
  if (n == 0) fail("cheb_lobatto_weights: p must be >= 2");
  if (n == 1) {
    w[0] = w[1] = 1.0;
    return w;
  }
  const double endw = (n % 2 == 0) ? 1.0 / (n * n - 1.0) : 1.0 / (n * n);
  w[0] = endw;
  w[n] = endw;
  for (int j = 1; j < n; ++j) {
    const double theta = M_PI * j / n;
    double v = 1.0;
    for (int k = 1; k <= (n % 2 == 0 ? n / 2 - 1 : (n - 1) / 2); ++k)
      v -= 2.0 * std::cos(2.0 * k * theta) / (4.0 * k * k - 1.0);
    if (n % 2 == 0) v -= std::cos(n * theta) / (n * n - 1.0);
    w[j] = 2.0 * v / n;
  }
  return w;
}

// proj/src/spectral.cpp:51-85 (Newton on P_q, stored ascending)
GaussRule gauss_legendre_1d(int q) {
  require(q >= 1, "gauss_legendre_1d: q must be >= 1");
  GaussRule r;
  r.nodes.assign(q, 0.0);
  r.weights.assign(q, 0.0);
  for (int i = 0; i < (q + 1) / 2; ++i) {
    double x = std::cos(M_PI * (i + 0.75) / (q + 0.5));
    double pp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = x;
      for (int k = 2; k <= q; ++k) {
        const double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      const double pq = (q == 1) ? x : p1;
      pp = q * (x * pq - p0) / (x * x - 1.0);
      if (q == 1) pp = 1.0;
      const double dx = pq / pp;
      x -= dx;
      if (std::abs(dx) < 1e-15) break;
    }
    if (q == 1) x = 0.0;
    const double wgt = (q == 1) ? 2.0 : 2.0 / ((1.0 - x * x) * pp * pp);
    r.nodes[i] = -x;
    r.nodes[q - 1 - i] = x;
    r.weights[i] = wgt;
    r.weights[q - 1 - i] = wgt;
  }
  if (q % 2 == 1) r.nodes[q / 2] = 0.0;
  return r;
}

// proj/src/spectral.cpp:87-103
Mat cheb_diff_matrix(int p) {
  require(p >= 2, "cheb_diff_matrix: p must be >= 2");
  const Vec x = cheb_lobatto_1d(p);
  Mat d(p, p);
  auto c = [&](int i) { return (i == 0 || i == p - 1) ? 2.0 : 1.0; };
  for (int i = 0; i < p; ++i) {
    double rowsum = 0.0;
    for (int j = 0; j < p; ++j) {
      if (i == j) continue;
      const double sgn = ((i + j) % 2 == 0) ? 1.0 : -1.0;
      d(i, j) = (c(i) / c(j)) * sgn / (x[i] - x[j]);
      rowsum += d(i, j);
    }
    d(i, i) = -rowsum;
  }
  return d;
}

// proj/src/spectral.cpp:105-137
Mat barycentric_interp_matrix(const Vec& src, const Vec& dst) {
  const int n = int(src.size()), m = int(dst.size());
  require(n >= 1, "barycentric_interp_matrix: empty source grid");
  Vec w(n);
  for (int j = 0; j < n; ++j) {
    double prod = 1.0;
    for (int k = 0; k < n; ++k) {
      if (k == j) continue;
      const double diff = src[j] - src[k];
      require(diff != 0.0, "barycentric_interp_matrix: coincident source nodes");
      prod *= diff;
    }
    w[j] = 1.0 / prod;
  }
  Mat out(m, n);
  for (int i = 0; i < m; ++i) {
    int hit = -1;
    for (int j = 0; j < n; ++j)
      if (dst[i] == src[j]) {
        hit = j;
        break;
      }
    if (hit >= 0) {
      out(i, hit) = 1.0;
      continue;
    }
    double denom = 0.0;
    for (int j = 0; j < n; ++j) denom += w[j] / (dst[i] - src[j]);
    for (int j = 0; j < n; ++j) out(i, j) = (w[j] / (dst[i] - src[j])) / denom;
  }
  return out;
}

// proj/src/spectral.cpp:139-160
IndexSets leaf_index_sets(int p, int dim) {
  IndexSets s;
  if (dim == 2) {
    for (int i1 = 0; i1 < p; ++i1)
      for (int i2 = 0; i2 < p; ++i2) {
        const bool bnd = i1 == 0 || i1 == p - 1 || i2 == 0 || i2 == p - 1;
        (bnd ? s.exterior : s.interior).push_back(i1 * p + i2);
      }
  } else if (dim == 3) {
    for (int i1 = 0; i1 < p; ++i1)
      for (int i2 = 0; i2 < p; ++i2)
        for (int i3 = 0; i3 < p; ++i3) {
          const bool bnd = i1 == 0 || i1 == p - 1 || i2 == 0 || i2 == p - 1 || i3 == 0 || i3 == p - 1;
          (bnd ? s.exterior : s.interior).push_back((i1 * p + i2) * p + i3);
        }
  } else {
    fail("leaf_index_sets: dim must be 2 or 3");
  }
  return s;
}

// proj/src/spectral.cpp:162-168
Mat kron(const Mat& a, const Mat& b) {
  Mat out(a.r * b.r, a.c * b.c);
  for (int i = 0; i < a.r; ++i)
    for (int j = 0; j < a.c; ++j)
      for (int k = 0; k < b.r; ++k)
        for (int l = 0; l < b.c; ++l) out(i * b.r + k, j * b.c + l) = a(i, j) * b(k, l);
  return out;
}

namespace {
// proj/src/spectral.cpp:172-188 -- sides (S,E,N,W); node 0 carries +1
struct Side2d {
  int axis;
  double sign;
  int fixed_node;
};
Side2d side2d(int s, int p) {
  switch (s) {
    case 0: return {1, -1.0, p - 1};
    case 1: return {0, +1.0, 0};
    case 2: return {1, +1.0, 0};
    default: return {0, -1.0, p - 1};
  }
}
int t2(int i1, int i2, int p) { return i1 * p + i2; }
// proj/src/spectral.cpp:203-210
void normal_row_2d(int s, int run, int p, const Mat& d1, Mat& mat, int row) {
  const Side2d sd = side2d(s, p);
  for (int k = 0; k < p; ++k) {
    const int col = (sd.axis == 0) ? t2(k, run, p) : t2(run, k, p);
    mat(row, col) += sd.sign * d1(sd.fixed_node, k);
  }
}
// proj/src/spectral.cpp:232-246
struct Face3d {
  int axis;
  double sign;
  int fixed_node;
  int ua, va;
};
Face3d face3d(int f, int p) {
  const int axis = f / 2;
  const double sign = (f % 2 == 0) ? -1.0 : 1.0;
  const int fixed_node = (f % 2 == 0) ? p - 1 : 0;
  const int ua = (axis == 0) ? 1 : 0;
  const int va = (axis == 2) ? 1 : 2;
  return {axis, sign, fixed_node, ua, va};
}
int t3(int i1, int i2, int i3, int p) { return (i1 * p + i2) * p + i3; }
Vec reversed(const Vec& v) { return Vec(v.rbegin(), v.rend()); }
Mat scaled(Mat m, double s) {
  for (double& x : m.a) x *= s;
  return m;
}
}  // namespace

// proj/src/spectral.cpp:260-310
LeafOps assemble_dtn_ops_2d(int p, int q, double side) {
  require(q == p - 2, "assemble_dtn_ops_2d: requires q = p-2");
  LeafOps ops;
  ops.dim = 2;
  ops.p = p;
  ops.q = q;
  ops.side = side;
  ops.idx = leaf_index_sets(p, 2);
  const Vec cn = cheb_lobatto_1d(p);
  const GaussRule gr = gauss_legendre_1d(q);
  const Mat d1 = cheb_diff_matrix(p);
  const double dscale = 2.0 / side;
  const Mat cheb_to_gauss = barycentric_interp_matrix(reversed(cn), gr.nodes);

  const int ne = int(ops.idx.exterior.size());
  ops.P = Mat(ne, 4 * q);
  for (int r = 0; r < ne; ++r) {
    const int idx = ops.idx.exterior[r];
    const int i1 = idx / p, i2 = idx % p;
    std::vector<int> owners;
    if (i2 == p - 1) owners.push_back(0);
    if (i1 == 0) owners.push_back(1);
    if (i2 == 0) owners.push_back(2);
    if (i1 == p - 1) owners.push_back(3);
    const double wgt = 1.0 / owners.size();
    for (int s : owners) {
      const Side2d sd = side2d(s, p);
      const double t = (sd.axis == 0) ? cn[i2] : cn[i1];
      const Mat row = barycentric_interp_matrix(gr.nodes, Vec{t});
      for (int j = 0; j < q; ++j) ops.P(r, s * q + j) += wgt * row(0, j);
    }
  }
  ops.Q = Mat(4 * q, p * p);
  for (int s = 0; s < 4; ++s) {
    Mat nside(p, p * p);
    for (int r = 0; r < p; ++r) normal_row_2d(s, p - 1 - r, p, d1, nside, r);
    const Mat blk = scaled(matmul(cheb_to_gauss, nside), dscale);
    for (int i = 0; i < q; ++i)
      for (int j = 0; j < p * p; ++j) ops.Q(s * q + i, j) = blk(i, j);
  }
  return ops;
}

// proj/src/spectral.cpp:370-436
LeafOps assemble_dtn_ops_3d(int p, int q, double side) {
  require(q == p - 2, "assemble_dtn_ops_3d: requires q = p-2");
  LeafOps ops;
  ops.dim = 3;
  ops.p = p;
  ops.q = q;
  ops.side = side;
  ops.idx = leaf_index_sets(p, 3);
  const Vec cn = cheb_lobatto_1d(p);
  const GaussRule gr = gauss_legendre_1d(q);
  const Mat d1 = cheb_diff_matrix(p);
  const double dscale = 2.0 / side;
  const int pp = p * p * p;
  const Mat c2g = barycentric_interp_matrix(reversed(cn), gr.nodes);

  const int ne = int(ops.idx.exterior.size());
  ops.P = Mat(ne, 6 * q * q);
  for (int r = 0; r < ne; ++r) {
    const int idx = ops.idx.exterior[r];
    const int ijk[3] = {idx / (p * p), (idx / p) % p, idx % p};
    std::vector<int> owners;
    for (int a = 0; a < 3; ++a) {
      if (ijk[a] == p - 1) owners.push_back(2 * a);
      if (ijk[a] == 0) owners.push_back(2 * a + 1);
    }
    const double wgt = 1.0 / owners.size();
    for (int f : owners) {
      const Face3d fc = face3d(f, p);
      const Mat ru = barycentric_interp_matrix(gr.nodes, Vec{cn[ijk[fc.ua]]});
      const Mat rv = barycentric_interp_matrix(gr.nodes, Vec{cn[ijk[fc.va]]});
      for (int a = 0; a < q; ++a)
        for (int b = 0; b < q; ++b) ops.P(r, f * q * q + a * q + b) += wgt * ru(0, a) * rv(0, b);
    }
  }
  ops.Q = Mat(6 * q * q, pp);
  const Mat face_interp = kron(c2g, c2g);
  for (int f = 0; f < 6; ++f) {
    const Face3d fc = face3d(f, p);
    Mat nface(p * p, pp);
    for (int ru = 0; ru < p; ++ru)
      for (int rv = 0; rv < p; ++rv) {
        const int nu = p - 1 - ru, nv = p - 1 - rv;
        const int row = ru * p + rv;
        for (int k = 0; k < p; ++k) {
          int id[3];
          id[fc.axis] = k;
          id[fc.ua] = nu;
          id[fc.va] = nv;
          nface(row, t3(id[0], id[1], id[2], p)) += fc.sign * d1(fc.fixed_node, k);
        }
      }
    const Mat blk = scaled(matmul(face_interp, nface), dscale);
    for (int i = 0; i < q * q; ++i)
      for (int j = 0; j < pp; ++j) ops.Q(f * q * q + i, j) = blk(i, j);
  }
  return ops;
}

// proj/src/spectral.cpp:438-452
Mat refinement_interpolant(int p) {
  const Vec cn = cheb_lobatto_1d(p);
  Vec lo(p), hi(p);
  for (int i = 0; i < p; ++i) lo[i] = (cn[i] - 1.0) / 2.0, hi[i] = (cn[i] + 1.0) / 2.0;
  const Mat e[2] = {barycentric_interp_matrix(cn, lo), barycentric_interp_matrix(cn, hi)};
  const int pc = p * p * p;
  Mat out(8 * pc, pc);
  for (int c = 0; c < 8; ++c) {
    const Mat k3 = kron(e[child_offset[c][0]], kron(e[child_offset[c][1]], e[child_offset[c][2]]));
    for (int i = 0; i < pc; ++i)
      for (int j = 0; j < pc; ++j) out(c * pc + i, j) = k3(i, j);
  }
  return out;
}

// proj/src/spectral.cpp:454-483
FaceProjection face_projection_ops(int q) {
  const GaussRule gr = gauss_legendre_1d(q);
  Vec lo(q), hi(q);
  for (int i = 0; i < q; ++i) lo[i] = (gr.nodes[i] - 1.0) / 2.0, hi[i] = (gr.nodes[i] + 1.0) / 2.0;
  const Mat r1[2] = {barycentric_interp_matrix(gr.nodes, lo), barycentric_interp_matrix(gr.nodes, hi)};
  FaceProjection fp;
  const int qq = q * q;
  fp.refine = Mat(4 * qq, qq);
  for (int hu = 0; hu < 2; ++hu)
    for (int hv = 0; hv < 2; ++hv) {
      const Mat k = kron(r1[hu], r1[hv]);
      for (int i = 0; i < qq; ++i)
        for (int j = 0; j < qq; ++j) fp.refine((hu * 2 + hv) * qq + i, j) = k(i, j);
    }
  fp.coarsen = Mat(qq, 4 * qq);
  for (int iu = 0; iu < q; ++iu)
    for (int iv = 0; iv < q; ++iv) {
      const int hu = gr.nodes[iu] > 0.0 ? 1 : 0;
      const int hv = gr.nodes[iv] > 0.0 ? 1 : 0;
      const Mat ru = barycentric_interp_matrix(hu ? hi : lo, Vec{gr.nodes[iu]});
      const Mat rv = barycentric_interp_matrix(hv ? hi : lo, Vec{gr.nodes[iv]});
      for (int a = 0; a < q; ++a)
        for (int b = 0; b < q; ++b) fp.coarsen(iu * q + iv, (hu * 2 + hv) * qq + a * q + b) = ru(0, a) * rv(0, b);
    }
  return fp;
}

// ============================================================================
// mesh: proj/src/mesh.cpp
// ============================================================================
// proj/include/hps/mesh.hpp:24-25
const int child_offset[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                                {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};

long long Tree::total_points() const {
  long long per = 1;
  for (int k = 0; k < dim; ++k) per *= p;
  return per * n_leaves();
}

// proj/src/mesh.cpp:27-52
void Tree::split(int node_id) {
  require(nodes[node_id].is_leaf(), "split: node already has children");
  const int nchild = dim == 2 ? 4 : 8;
  Point mid;
  for (int k = 0; k < 3; ++k) mid[k] = 0.5 * (nodes[node_id].box.lo[k] + nodes[node_id].box.hi[k]);
  nodes[node_id].n_children = nchild;
  for (int c = 0; c < nchild; ++c) {
    const TreeNode& n = nodes[node_id];
    TreeNode ch;
    ch.id = int(nodes.size());
    ch.parent = node_id;
    ch.depth = n.depth + 1;
    for (int k = 0; k < 3; ++k) {
      ch.box.lo[k] = child_offset[c][k] ? mid[k] : n.box.lo[k];
      ch.box.hi[k] = child_offset[c][k] ? n.box.hi[k] : mid[k];
      ch.anchor[k] = 2 * n.anchor[k] + child_offset[c][k];
    }
    if (dim == 2) {
      ch.box.lo[2] = ch.box.hi[2] = 0.0;
      ch.anchor[2] = 0;
    }
    nodes[node_id].child[c] = ch.id;
    nodes.push_back(ch);
  }
}

// proj/src/mesh.cpp:54-71 (DFS leaf order, per-depth levels)
void Tree::finalize() {
  leaves.clear();
  levels.clear();
  const int nchild = dim == 2 ? 4 : 8;
  std::vector<int> stack{0};
  while (!stack.empty()) {
    const int id = stack.back();
    stack.pop_back();
    const TreeNode& n = nodes[id];
    if (int(levels.size()) <= n.depth) levels.resize(n.depth + 1);
    levels[n.depth].push_back(id);
    if (n.is_leaf())
      leaves.push_back(id);
    else
      for (int c = nchild - 1; c >= 0; --c) stack.push_back(n.child[c]);
  }
}

// proj/src/mesh.cpp:90-121
Tree build_uniform_tree(const Box& domain, int L, int dim, int p) {
  require(dim == 2 || dim == 3, "build_uniform_tree: dim must be 2 or 3");
  require(L >= 0, "build_uniform_tree: depth must be nonnegative");
  require(p >= 4, "build_uniform_tree: p must be >= 4");
  const double side = domain.hi[0] - domain.lo[0];
  require(side > 0, "build_uniform_tree: empty domain");
  for (int k = 1; k < dim; ++k)
    require(std::abs((domain.hi[k] - domain.lo[k]) - side) <= 1e-12 * std::abs(side),
            "build_uniform_tree: domain must be a square/cube");
  Tree t;
  t.dim = dim;
  t.p = p;
  t.q = p - 2;
  t.domain = domain;
  TreeNode root;
  root.id = 0;
  root.box = domain;
  if (dim == 2) root.box.lo[2] = root.box.hi[2] = 0.0;
  t.nodes.push_back(root);
  for (int level = 0; level < L; ++level) {
    std::vector<int> ids;
    for (const TreeNode& n : t.nodes)
      if (n.depth == level) ids.push_back(n.id);
    for (int id : ids) t.split(id);
  }
  t.finalize();
  return t;
}

// proj/src/mesh.cpp:320-336
std::vector<Point> leaf_cheb_points(const Box& box, int p, int dim) {
  const Vec cn = cheb_lobatto_1d(p);
  std::vector<Point> pts;
  auto map1 = [&](double t, int k) { return 0.5 * (box.lo[k] + box.hi[k]) + 0.5 * (box.hi[k] - box.lo[k]) * t; };
  if (dim == 2) {
    for (int i1 = 0; i1 < p; ++i1)
      for (int i2 = 0; i2 < p; ++i2) {
        Point x;
        x[0] = map1(cn[i1], 0);
        x[1] = map1(cn[i2], 1);
        pts.push_back(x);
      }
  } else {
    for (int i1 = 0; i1 < p; ++i1)
      for (int i2 = 0; i2 < p; ++i2)
        for (int i3 = 0; i3 < p; ++i3) {
          Point x;
          x[0] = map1(cn[i1], 0);
          x[1] = map1(cn[i2], 1);
          x[2] = map1(cn[i3], 2);
          pts.push_back(x);
        }
  }
  return pts;
}

// proj/src/mesh.cpp:342-375
std::vector<Point> leaf_gauss_boundary_points(const Box& box, int q, int dim) {
  const GaussRule gr = gauss_legendre_1d(q);
  std::vector<Point> pts;
  auto map1 = [&](double t, int k) { return 0.5 * (box.lo[k] + box.hi[k]) + 0.5 * (box.hi[k] - box.lo[k]) * t; };
  if (dim == 2) {
    for (int s = 0; s < 4; ++s)
      for (int i = 0; i < q; ++i) {
        const double t = gr.nodes[i];
        Point x;
        switch (s) {
          case 0: x[0] = map1(t, 0); x[1] = box.lo[1]; break;
          case 1: x[0] = box.hi[0]; x[1] = map1(t, 1); break;
          case 2: x[0] = map1(t, 0); x[1] = box.hi[1]; break;
          default: x[0] = box.lo[0]; x[1] = map1(t, 1); break;
        }
        pts.push_back(x);
      }
  } else {
    for (int f = 0; f < 6; ++f) {
      const int axis = f / 2;
      const int ua = (axis == 0) ? 1 : 0;
      const int va = (axis == 2) ? 1 : 2;
      const double fixed = (f % 2 == 0) ? box.lo[axis] : box.hi[axis];
      for (int iu = 0; iu < q; ++iu)
        for (int iv = 0; iv < q; ++iv) {
          Point x;
          x[axis] = fixed;
          x[ua] = map1(gr.nodes[iu], ua);
          x[va] = map1(gr.nodes[iv], va);
          pts.push_back(x);
        }
    }
  }
  return pts;
}

// ============================================================================
// layout: proj/src/layout.cpp
// ============================================================================
// proj/src/layout.cpp:10-15
int PanelLayout::npts() const {
  if (!split) return panel_pts();
  int n = 0;
  for (const auto& s : sub) n += s.npts();
  return n;
}
// proj/src/layout.cpp:24-31
bool PanelLayout::operator==(const PanelLayout& o) const {
  if (split != o.split || q != o.q || fdim != o.fdim) return false;
  if (!split) return true;
  for (size_t i = 0; i < sub.size(); ++i)
    if (!(sub[i] == o.sub[i])) return false;
  return true;
}
// proj/src/layout.cpp:33-40
PanelLayout PanelLayout::split_of(std::vector<PanelLayout> kids) {
  PanelLayout l;
  require(!kids.empty(), "PanelLayout::split_of: empty");
  l.q = kids[0].q;
  l.fdim = kids[0].fdim;
  l.split = true;
  l.sub = std::move(kids);
  return l;
}

namespace {
// proj/src/layout.cpp:89-119
void collect_points(const Box& box, int dim, int face, const PanelLayout& layout, std::vector<Point>& out) {
  if (!layout.split) {
    const auto pts = leaf_gauss_boundary_points(box, layout.q, dim);
    const int per = layout.panel_pts();
    for (int i = 0; i < per; ++i) out.push_back(pts[face * per + i]);
    return;
  }
  Point mid;
  for (int k = 0; k < 3; ++k) mid[k] = 0.5 * (box.lo[k] + box.hi[k]);
  if (dim == 2) {
    const int axis = (face == 0 || face == 2) ? 0 : 1;
    for (int h = 0; h < 2; ++h) {
      Box sb = box;
      (h ? sb.lo : sb.hi)[axis] = mid[axis];
      collect_points(sb, dim, face, layout.sub[h], out);
    }
  } else {
    const int fa = face / 2;
    const int ua = (fa == 0) ? 1 : 0;
    const int va = (fa == 2) ? 1 : 2;
    for (int hu = 0; hu < 2; ++hu)
      for (int hv = 0; hv < 2; ++hv) {
        Box sb = box;
        (hu ? sb.lo : sb.hi)[ua] = mid[ua];
        (hv ? sb.lo : sb.hi)[va] = mid[va];
        collect_points(sb, dim, face, layout.sub[hu * 2 + hv], out);
      }
  }
}
}  // namespace

// proj/src/layout.cpp:121-126
std::vector<Point> section_points(const Box& box, int dim, int face, const PanelLayout& layout) {
  std::vector<Point> out;
  collect_points(box, dim, face, layout, out);
  return out;
}

// ============================================================================
// local solve: proj/src/local_solve.cpp
// ============================================================================
namespace {
struct DiffOps {
  std::vector<Mat> d1, d2;
};
// proj/src/local_solve.cpp:21-40
DiffOps make_diff_ops(int p, int dim) {
  const Mat d = cheb_diff_matrix(p);
  const Mat dd = matmul(d, d);
  Mat id(p, p);
  for (int i = 0; i < p; ++i) id(i, i) = 1.0;
  DiffOps ops;
  if (dim == 2) {
    ops.d1 = {kron(d, id), kron(id, d)};
    ops.d2 = {kron(dd, id), kron(id, dd)};
  } else {
    ops.d1 = {kron(d, kron(id, id)), kron(id, kron(d, id)), kron(id, kron(id, d))};
    ops.d2 = {kron(dd, kron(id, id)), kron(id, kron(dd, id)), kron(id, kron(id, dd))};
  }
  return ops;
}
const DiffOps& diff_ops(int p, int dim) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<int, int>, DiffOps>> cache;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : cache)
    if (e.first == std::make_pair(p, dim)) return e.second;
  cache.emplace_back(std::make_pair(p, dim), make_diff_ops(p, dim));
  return cache.back().second;
}
}  // namespace

// proj/src/local_solve.cpp:44-86.  Dense n x n, row i scaled by c(x_i).
// (The loops skip structurally-zero entries of the kron operators; the
// arithmetic per nonzero entry is the reference's c_i * s^k * op(i,j).)
Mat discretize_operator(const Box& box, int leaf_ord, const std::vector<Term>& terms, int p, int dim) {
  const int n = dim == 2 ? p * p : p * p * p;
  const auto pts = leaf_cheb_points(box, p, dim);
  const DiffOps& ops = diff_ops(p, dim);
  const double scale = 2.0 / (box.hi[0] - box.lo[0]);
  Mat lmat(n, n);
  Vec c(n);
  auto add_scaled_rows = [&](double s, const Mat& op) {
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        const double o = op(i, j);
        if (o != 0.0) lmat(i, j) += s * (c[i] * o);
      }
  };
  for (const Term& term : terms) {
    for (int i = 0; i < n; ++i) {
      c[i] = term.eval(pts[i], leaf_ord, i);
      if (!std::isfinite(c[i])) {
        std::ostringstream os;
        os << "discretize_operator: non-finite coefficient sample on leaf " << leaf_ord << " at point ("
           << pts[i][0] << ", " << pts[i][1] << ", " << pts[i][2] << ")";
        fail(os.str());
      }
    }
    switch (term.role) {
      case Role::laplacian:
        for (int a = 0; a < dim; ++a) add_scaled_rows(scale * scale, ops.d2[a]);
        break;
      case Role::gradient:
        require(term.axis >= 0 && term.axis < dim, "discretize_operator: bad gradient axis");
        add_scaled_rows(scale, ops.d1[term.axis]);
        break;
      case Role::zeroth:
        for (int i = 0; i < n; ++i) lmat(i, i) += c[i];
        break;
      case Role::second_order:
        require(term.axis >= 0 && term.axis < dim && term.axis2 >= 0 && term.axis2 < dim,
                "discretize_operator: bad second_order axes");
        if (term.axis == term.axis2)
          add_scaled_rows(scale * scale, ops.d2[term.axis]);
        else
          add_scaled_rows(scale * scale, matmul(ops.d1[term.axis], ops.d1[term.axis2]));
        break;
    }
  }
  return lmat;
}

namespace {
// proj/src/local_solve.cpp:90-107
void check_factorization(const LU& fac, LeafSolution& out, const char* what) {
  double dmin = INFINITY, dmax = 0.0;
  for (int i = 0; i < fac.n; ++i) {
    const double a = std::abs(fac.lu(i, i));
    if (!std::isfinite(a) || a == 0.0) {
      std::ostringstream os;
      os << what << ": singular factorization (zero pivot at " << i << ")";
      fail(os.str());
    }
    dmin = std::min(dmin, a);
    dmax = std::max(dmax, a);
  }
  out.rcond = dmin / dmax;
  out.ill = out.rcond < 1e-12;
}
}  // namespace

// proj/src/local_solve.cpp:111-143
LeafSolution local_solve_dtn(const Mat& lmat, const Vec& fvec, const LeafOps& ops, bool literal_sign) {
  const auto& ii = ops.idx.interior;
  const auto& ie = ops.idx.exterior;
  const int n = lmat.r, ni = int(ii.size()), ne = int(ie.size()), nb = ops.P.c;
  Mat a_ii(ni, ni), a_ie(ni, ne);
  for (int r = 0; r < ni; ++r) {
    for (int c = 0; c < ni; ++c) a_ii(r, c) = lmat(ii[r], ii[c]);
    for (int c = 0; c < ne; ++c) a_ie(r, c) = lmat(ii[r], ie[c]);
  }
  LeafSolution sol;
  sol.fac.compute(a_ii);
  check_factorization(sol.fac, sol, "local_solve_dtn");
  const Mat x = sol.fac.solve(a_ie);
  sol.Y = Mat(n, nb);
  for (int r = 0; r < ne; ++r)
    for (int j = 0; j < nb; ++j) sol.Y(ie[r], j) = ops.P(r, j);
  Mat yi = matmul(x, ops.P);
  for (int r = 0; r < ni; ++r)
    for (int j = 0; j < nb; ++j) sol.Y(ii[r], j) = -yi(r, j);
  Vec fi(ni);
  for (int r = 0; r < ni; ++r) fi[r] = fvec[ii[r]];
  sol.v.assign(n, 0.0);
  const Vec vi = sol.fac.solve(fi);
  const double sgn = literal_sign ? -1.0 : 1.0;  // reference: -L_ii^-1 f_i (:137)
  for (int r = 0; r < ni; ++r) sol.v[ii[r]] = sgn * vi[r];
  sol.T = matmul(ops.Q, sol.Y);
  Mat vm(n, 1);
  vm.a = sol.v;
  sol.h = matmul(ops.Q, vm).a;
  return sol;
}

// ============================================================================
// merge: proj/src/merge.cpp (DtN, uniform children: identity interface transfers)
// ============================================================================
namespace {
struct Interface {
  int clo, flo, chi, fhi;
};
// proj/src/merge.cpp:20-33
const std::vector<Interface>& interfaces(int dim) {
  static const std::vector<Interface> if2d = {{0, 1, 1, 3}, {1, 2, 2, 0}, {3, 1, 2, 3}, {0, 2, 3, 0}};
  static const std::vector<Interface> if3d = {
      {0, 1, 1, 0}, {1, 3, 2, 2}, {3, 1, 2, 0}, {0, 3, 3, 2}, {4, 1, 5, 0}, {5, 3, 6, 2},
      {7, 1, 6, 0}, {4, 3, 7, 2}, {0, 5, 4, 4}, {1, 5, 5, 4}, {2, 5, 6, 4}, {3, 5, 7, 4},
  };
  return dim == 2 ? if2d : if3d;
}
struct ExtDest {
  int pface, qpos;
};
// proj/src/merge.cpp:41-56
ExtDest ext_dest(int dim, int child, int face) {
  const int* off = child_offset[child];
  if (dim == 2) {
    const int axis = (face == 1 || face == 3) ? 0 : 1;
    const int high = (face == 1 || face == 2) ? 1 : 0;
    if (off[axis] != high) return {-1, -1};
    const int run = axis == 0 ? 1 : 0;
    return {face, off[run]};
  }
  const int axis = face / 2, high = face % 2;
  if (off[axis] != high) return {-1, -1};
  const int ua = (axis == 0) ? 1 : 0;
  const int va = (axis == 2) ? 1 : 2;
  return {face, off[ua] * 2 + off[va]};
}
// proj/src/merge.cpp:58-64
int interface_of(int dim, int child, int face) {
  const auto& ifs = interfaces(dim);
  for (size_t t = 0; t < ifs.size(); ++t)
    if ((ifs[t].clo == child && ifs[t].flo == face) || (ifs[t].chi == child && ifs[t].fhi == face)) return int(t);
  return -1;
}
}  // namespace

// proj/src/merge.cpp:183-324 (with MergeGeom :90-152), uniform children.
MergeOut merge_dtn(int dim, const std::vector<ChildView>& ch, bool is_root, bool implicit_S) {
  const int nchild = dim == 2 ? 4 : 8, nface = 2 * dim;
  require(int(ch.size()) == nchild, "merge: wrong number of children");
  // --- MergeGeom (proj/src/merge.cpp:90-152)
  std::vector<std::array<int, 7>> child_off(nchild);
  for (int k = 0; k < nchild; ++k) {
    require(int(ch[k].sections->size()) == nface, "merge: bad child sections");
    child_off[k][0] = 0;
    for (int f = 0; f < nface; ++f) child_off[k][f + 1] = child_off[k][f] + (*ch[k].sections)[f].npts();
    require(ch[k].T->r == child_off[k][nface] && ch[k].T->c == child_off[k][nface],
            "merge: child T shape does not match its boundary layout");
  }
  const auto& ifs = interfaces(dim);
  std::vector<int> int_off(ifs.size()), int_len(ifs.size());
  int n_int = 0;
  for (size_t t = 0; t < ifs.size(); ++t) {
    const PanelLayout& la = (*ch[ifs[t].clo].sections)[ifs[t].flo];
    const PanelLayout& lb = (*ch[ifs[t].chi].sections)[ifs[t].fhi];
    require(la == lb, "merge: interface layout mismatch (oracle restates uniform merges only)");
    int_off[t] = n_int;
    int_len[t] = la.npts();
    n_int += la.npts();
  }
  std::vector<PanelLayout> parent_sections(nface);
  std::vector<int> parent_face_off(nface + 1, 0);
  std::vector<std::array<int, 6>> ext_off(nchild, {-1, -1, -1, -1, -1, -1});
  const int nquad = dim == 2 ? 2 : 4;
  for (int f = 0; f < nface; ++f) {
    std::vector<PanelLayout> quads(nquad);
    std::vector<int> owner(nquad, -1);
    for (int k = 0; k < nchild; ++k) {
      const ExtDest e = ext_dest(dim, k, f);
      if (e.pface != f) continue;
      quads[e.qpos] = (*ch[k].sections)[f];
      owner[e.qpos] = k;
    }
    int pos = parent_face_off[f];
    for (int qv = 0; qv < nquad; ++qv) {
      ext_off[owner[qv]][f] = pos;
      pos += quads[qv].npts();
    }
    parent_sections[f] = PanelLayout::split_of(std::move(quads));
    parent_face_off[f + 1] = pos;
  }
  const int n_ext = parent_face_off[nface];

  MergeOut out;
  Artifact& art = out.art;
  art.n_ext = n_ext;
  art.n_int = n_int;
  art.implicit = implicit_S;
  art.child_face_off = child_off;
  // --- block assembly (proj/src/merge.cpp:226-278)
  const bool need_ab = !is_root;
  Mat a, b, c, d(n_int, n_int);
  if (need_ab) a = Mat(n_ext, n_ext), b = Mat(n_ext, n_int);
  c = Mat(n_int, n_ext);
  Vec h_ext(n_ext, 0.0);
  art.h_int.assign(n_int, 0.0);
  for (int k = 0; k < nchild; ++k) {
    const Mat& tk = *ch[k].T;
    const Vec& hk = *ch[k].h;
    for (int rf = 0; rf < nface; ++rf) {
      const int r0 = child_off[k][rf], rn = child_off[k][rf + 1] - r0;
      const bool rext = ext_off[k][rf] >= 0;
      const int roff = rext ? ext_off[k][rf] : int_off[interface_of(dim, k, rf)];
      for (int i = 0; i < rn; ++i) (rext ? h_ext : art.h_int)[roff + i] += hk[r0 + i];
      for (int cf = 0; cf < nface; ++cf) {
        const int c0 = child_off[k][cf], cn = child_off[k][cf + 1] - c0;
        const bool cext = ext_off[k][cf] >= 0;
        const int coff = cext ? ext_off[k][cf] : int_off[interface_of(dim, k, cf)];
        Mat* dst = nullptr;
        if (rext && cext)
          dst = need_ab ? &a : nullptr;
        else if (rext && !cext)
          dst = need_ab ? &b : nullptr;
        else if (!rext && cext)
          dst = &c;
        else
          dst = &d;
        if (!dst) continue;
        for (int j = 0; j < cn; ++j)
          for (int i = 0; i < rn; ++i) (*dst)(roff + i, coff + j) += tk(r0 + i, c0 + j);
      }
    }
  }
  // --- factor + Schur (proj/src/merge.cpp:280-300)
  art.Dfac.compute(d);
  for (int i = 0; i < n_int; ++i) {
    const double piv = std::abs(art.Dfac.lu(i, i));
    if (!(piv > 0.0) || !std::isfinite(piv)) {
      std::ostringstream os;
      os << "merge_dtn: singular interface matrix D (pivot " << i << ")";
      fail(os.str());
    }
  }
  const Vec gsolve = art.Dfac.solve(art.h_int);
  art.gtilde.resize(n_int);
  for (int i = 0; i < n_int; ++i) art.gtilde[i] = -gsolve[i];
  if (!implicit_S) {
    Mat x = art.Dfac.solve(c);
    if (need_ab) {
      out.T = a;
      gemm(-1.0, b, x, 1.0, out.T);
      Mat gt(n_int, 1);
      gt.a = art.gtilde;
      Mat hm(n_ext, 1);
      hm.a = h_ext;
      gemm(1.0, b, gt, 1.0, hm);
      out.h = hm.a;
    }
    for (double& v : x.a) v = -v;
    art.S = std::move(x);
  } else {
    require(!need_ab, "merge_dtn: implicit_S requires is_root");
    art.C = std::move(c);
  }
  // --- downward-pass gather maps (proj/src/merge.cpp:302-320)
  art.child_maps.resize(nchild);
  for (int k = 0; k < nchild; ++k)
    for (int f = 0; f < nface; ++f) {
      FaceMap& m = art.child_maps[k][f];
      m.dst_len = child_off[k][f + 1] - child_off[k][f];
      if (ext_off[k][f] >= 0) {
        m.ext = true;
        m.offset = ext_off[k][f];
      } else {
        m.ext = false;
        m.offset = int_off[interface_of(dim, k, f)];
      }
      m.src_len = m.dst_len;
    }
  out.sections = parent_sections;
  return out;
}

// ============================================================================
// solver: proj/src/solver.cpp
// ============================================================================
// proj/src/solver.cpp:10-36
Solver::Solver(const Tree& tree, std::vector<Term> terms, std::function<double(const Point&, int, int)> source,
               SolverOptions opts)
    : tree_(&tree), terms_(std::move(terms)), source_(std::move(source)), opts_(opts) {
  const int n = int(tree.nodes.size());
  leaf_ord_.assign(n, -1);
  for (int i = 0; i < tree.n_leaves(); ++i) leaf_ord_[tree.leaves[i]] = i;
  leaf_.resize(tree.n_leaves());
  node_T_.resize(n);
  node_h_.resize(n);
  sections_.resize(n);
  art_.resize(n);
  const int nface = 2 * tree.dim;
  for (int id : tree.leaves) sections_[id] = std::vector<PanelLayout>(nface, PanelLayout::panel(tree.q, tree.dim - 1));
  // uniform trees: every leaf has the same side, one operator set (leaf_ops_cache)
  const double side = tree.leaf_side(tree.nodes[tree.leaves[0]]);
  ops_ = tree.dim == 2 ? assemble_dtn_ops_2d(tree.p, tree.q, side) : assemble_dtn_ops_3d(tree.p, tree.q, side);
}

// proj/src/solver.cpp:44-57
Mat Solver::leaf_operator(int ord, Vec* f) const {
  const TreeNode& leaf = tree_->nodes[tree_->leaves[ord]];
  require(std::abs(tree_->leaf_side(leaf) - ops_.side) == 0.0, "oracle: uniform trees only");
  if (f) {
    const auto pts = leaf_cheb_points(leaf.box, tree_->p, tree_->dim);
    f->assign(pts.size(), 0.0);
    for (size_t i = 0; i < pts.size(); ++i) (*f)[i] = source_ ? source_(pts[i], ord, int(i)) : 0.0;
  }
  return discretize_operator(leaf.box, ord, terms_, tree_->p, tree_->dim);
}

// proj/src/solver.cpp:44-65
void Solver::build_leaf(int ord) {
  Vec f;
  const Mat lmat = leaf_operator(ord, &f);
  leaf_[ord] = local_solve_dtn(lmat, f, ops_, opts_.literal_sign);
}

// proj/src/solver.cpp:77-97
std::vector<ChildView> Solver::child_views(int id) const {
  const TreeNode& n = tree_->nodes[id];
  const int nchild = tree_->dim == 2 ? 4 : 8;
  std::vector<ChildView> v(nchild);
  for (int c = 0; c < nchild; ++c) {
    const int cid = n.child[c];
    v[c].sections = &sections_[cid];
    const int ord = leaf_ord_[cid];
    if (ord >= 0) {
      v[c].T = &leaf_[ord].T;
      v[c].h = &leaf_[ord].h;
    } else {
      v[c].T = &node_T_[cid];
      v[c].h = &node_h_[cid];
    }
  }
  return v;
}

// proj/src/solver.cpp:99-135
void Solver::merge_internal(int id) {
  const bool is_root = id == 0;
  MergeOut out = merge_dtn(tree_->dim, child_views(id), is_root, is_root && opts_.root_implicit_S);
  sections_[id] = std::move(out.sections);
  art_[id] = std::move(out.art);
  if (!is_root) {
    node_T_[id] = std::move(out.T);
    node_h_[id] = std::move(out.h);
  }
}

// proj/src/solver.cpp:144-151 (serial loops; `parallel` = OpenMP over a level)
void Solver::build() {
  using clk = std::chrono::steady_clock;
  auto t0 = clk::now();
  const int nl = tree_->n_leaves();
  // "parallel oracle": OpenMP across independent leaves/merges with single-threaded BLAS
  // inside; levels with fewer nodes than threads run serially with threaded BLAS.
  const int nthr = omp_get_max_threads();
  if (opts_.parallel) {
    set_blas_threads(1);
    std::string err;
#pragma omp parallel for schedule(dynamic, 4)
    for (int i = 0; i < nl; ++i) {
      try {
        build_leaf(i);
      } catch (const std::exception& e) {
#pragma omp critical
        err = e.what();
      }
    }
    if (!err.empty()) fail(err);
  } else {
    for (int i = 0; i < nl; ++i) build_leaf(i);
  }
  for (int i = 0; i < nl; ++i) min_rcond_ = std::min(min_rcond_, leaf_[i].rcond);
  auto t1 = clk::now();
  for (int depth = tree_->max_depth() - 1; depth >= 0; --depth) {
    const auto& lev = tree_->levels[depth];
    const int cnt = int(lev.size());
    if (opts_.parallel && cnt >= nthr) {
      set_blas_threads(1);
      std::string err;
#pragma omp parallel for schedule(dynamic, 1)
      for (int i = 0; i < cnt; ++i) {
        if (tree_->nodes[lev[i]].is_leaf()) continue;
        try {
          merge_internal(lev[i]);
        } catch (const std::exception& e) {
#pragma omp critical
          err = e.what();
        }
      }
      if (!err.empty()) fail(err);
    } else {
      set_blas_threads(nthr);
      for (int id : lev)
        if (!tree_->nodes[id].is_leaf()) merge_internal(id);
    }
  }
  set_blas_threads(nthr);
  auto t2 = clk::now();
  t_leaf = std::chrono::duration<double>(t1 - t0).count();
  t_merge = std::chrono::duration<double>(t2 - t1).count();
}

// proj/src/solver.cpp:159-177
std::vector<Point> Solver::root_boundary_points() const {
  const TreeNode& n = tree_->nodes[0];
  std::vector<Point> pts;
  for (int f = 0; f < 2 * tree_->dim; ++f) {
    const auto fp = section_points(n.box, tree_->dim, f, sections_[0][f]);
    pts.insert(pts.end(), fp.begin(), fp.end());
  }
  return pts;
}

// proj/src/solver.cpp:188-252 (propagate + reconstruct_leaf + solve)
std::vector<Vec> Solver::solve(const Vec& g_root, std::vector<Vec>* leaf_g) const {
  const int nchild = tree_->dim == 2 ? 4 : 8, nface = 2 * tree_->dim;
  std::vector<Vec> g(tree_->nodes.size());
  g[0] = g_root;
  for (const auto& level : tree_->levels)
    for (int id : level) {
      const TreeNode& n = tree_->nodes[id];
      if (n.is_leaf()) continue;
      const Artifact& art = art_[id];
      require(art.n_int > 0, "propagate: missing merge artifact");
      const Vec& gj = g[id];
      Vec g_int(art.n_int);
      if (art.implicit) {
        // g_int = gtilde - D^-1 (C g)   (proj/src/solver.cpp:204-206)
        Mat gm(int(gj.size()), 1);
        gm.a = gj;
        const Mat cg = matmul(art.C, gm);
        const Vec y = art.Dfac.solve(cg.a);
        for (int i = 0; i < art.n_int; ++i) g_int[i] = art.gtilde[i] - y[i];
      } else {
        // g_int = S g + gtilde   (proj/src/solver.cpp:207-208)
        Mat gm(int(gj.size()), 1);
        gm.a = gj;
        const Mat sg = matmul(art.S, gm);
        for (int i = 0; i < art.n_int; ++i) g_int[i] = sg.a[i] + art.gtilde[i];
      }
      for (int c = 0; c < nchild; ++c) {
        const auto& offs = art.child_face_off[c];
        Vec& gc = g[n.child[c]];
        gc.assign(offs[nface], 0.0);
        for (int f = 0; f < nface; ++f) {
          const FaceMap& m = art.child_maps[c][f];
          const Vec& src = m.ext ? gj : g_int;
          for (int i = 0; i < m.dst_len; ++i) gc[offs[f] + i] = src[m.offset + i];
        }
      }
      if (id != 0) g[id].clear();
    }
  std::vector<Vec> u(tree_->n_leaves());
  if (leaf_g) leaf_g->resize(tree_->n_leaves());
  for (int i = 0; i < tree_->n_leaves(); ++i) {
    const Vec& gl = g[tree_->leaves[i]];
    const LeafSolution& sol = leaf_[i];
    Mat gm(int(gl.size()), 1);
    gm.a = gl;
    Mat um = matmul(sol.Y, gm);
    for (size_t j = 0; j < um.a.size(); ++j) um.a[j] += sol.v[j];
    u[i] = std::move(um.a);
    if (leaf_g) (*leaf_g)[i] = gl;
  }
  return u;
}

}  // namespace hpso
