// geometry.cpp -- host precompute for the B200 HPS solver (see geometry.hpp).
#include "geometry.hpp"

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <functional>
#include <stdexcept>

namespace hpsg {

std::string fmt(const char* f, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, f);
  vsnprintf(buf, sizeof buf, f, ap);
  va_end(ap);
  return buf;
}

static const int kChildOffset[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                                       {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};

// Chebyshev-Lobatto nodes, descending, antisymmetric by construction (spectral.cpp:14-26).
std::vector<double> cheb_nodes(int p) {
  const int n = p - 1;
  std::vector<double> x(p);
  for (int k = 0; k <= n / 2; ++k) {
    const double v = std::sin(M_PI * (n - 2 * k) / (2.0 * n));
    x[k] = v;
    x[n - k] = -v;
  }
  if (n % 2 == 0) x[n / 2] = 0.0;
  return x;
}

// Gauss-Legendre by Newton on the three-term recurrence (spectral.cpp:51-85).
void gauss_rule(int q, std::vector<double>& xs, std::vector<double>& ws) {
  xs.assign(q, 0.0);
  ws.assign(q, 0.0);
  for (int i = 0; i < (q + 1) / 2; ++i) {
    double x = std::cos(M_PI * (i + 0.75) / (q + 0.5)), dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = x;
      for (int k = 2; k <= q; ++k) {
        const double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      const double pq = q == 1 ? x : p1;
      dp = q == 1 ? 1.0 : q * (x * pq - p0) / (x * x - 1.0);
      const double dx = pq / dp;
      x -= dx;
      if (std::fabs(dx) < 1e-15) break;
    }
    if (q == 1) x = 0.0;
    const double w = q == 1 ? 2.0 : 2.0 / ((1.0 - x * x) * dp * dp);
    xs[i] = -x;
    xs[q - 1 - i] = x;
    ws[i] = ws[q - 1 - i] = w;
  }
  if (q % 2 == 1) xs[q / 2] = 0.0;
}

// Chebyshev differentiation with the negative-sum diagonal (spectral.cpp:87-103).
HostMat cheb_diff(int p) {
  const std::vector<double> x = cheb_nodes(p);
  HostMat d(p, p);
  for (int i = 0; i < p; ++i) {
    const double ci = (i == 0 || i == p - 1) ? 2.0 : 1.0;
    double sum = 0.0;
    for (int j = 0; j < p; ++j) {
      if (j == i) continue;
      const double cj = (j == 0 || j == p - 1) ? 2.0 : 1.0;
      d(i, j) = (ci / cj) * (((i + j) % 2 == 0) ? 1.0 : -1.0) / (x[i] - x[j]);
      sum += d(i, j);
    }
    d(i, i) = -sum;
  }
  return d;
}

// Barycentric Lagrange interpolation src -> dst (spectral.cpp:105-137).
HostMat bary_interp(const std::vector<double>& src, const std::vector<double>& dst) {
  const int n = int(src.size()), m = int(dst.size());
  std::vector<double> w(n);
  for (int j = 0; j < n; ++j) {
    double prod = 1.0;
    for (int k = 0; k < n; ++k)
      if (k != j) prod *= src[j] - src[k];
    w[j] = 1.0 / prod;
  }
  HostMat out(m, n);
  for (int i = 0; i < m; ++i) {
    int hit = -1;
    for (int j = 0; j < n && hit < 0; ++j)
      if (dst[i] == src[j]) hit = j;
    if (hit >= 0) {
      out(i, hit) = 1.0;
      continue;
    }
    double den = 0.0;
    for (int j = 0; j < n; ++j) den += w[j] / (dst[i] - src[j]);
    for (int j = 0; j < n; ++j) out(i, j) = (w[j] / (dst[i] - src[j])) / den;
  }
  return out;
}

static HostMat matmul(const HostMat& a, const HostMat& b) {
  HostMat c(a.r, b.c);
  for (int j = 0; j < b.c; ++j)
    for (int k = 0; k < a.c; ++k) {
      const double bk = b(k, j);
      if (bk == 0.0) continue;
      for (int i = 0; i < a.r; ++i) c(i, j) += a(i, k) * bk;
    }
  return c;
}

LeafOperators make_leaf_operators(int dim, int p, double side) {
  if (dim != 2 && dim != 3) throw std::runtime_error("make_leaf_operators: dim must be 2 or 3");
  if (p < 4) throw std::runtime_error("make_leaf_operators: p must be >= 4");
  LeafOperators op;
  op.dim = dim;
  op.p = p;
  op.q = p - 2;
  op.side = side;
  const int q = op.q;
  op.n = dim == 2 ? p * p : p * p * p;
  // interior / exterior tensor indices, increasing (spectral.cpp:139-160)
  for (int idx = 0; idx < op.n; ++idx) {
    int c[3] = {idx / p, idx % p, 0};
    if (dim == 3) c[0] = idx / (p * p), c[1] = (idx / p) % p, c[2] = idx % p;
    bool bnd = false;
    for (int a = 0; a < dim; ++a) bnd = bnd || c[a] == 0 || c[a] == p - 1;
    (bnd ? op.exterior : op.interior).push_back(idx);
  }
  op.ni = int(op.interior.size());
  op.ne = int(op.exterior.size());
  op.nb = dim == 2 ? 4 * q : 6 * q * q;

  const std::vector<double> cn = cheb_nodes(p);
  std::vector<double> gx, gw;
  gauss_rule(q, gx, gw);
  op.D = cheb_diff(p);
  op.D2 = matmul(op.D, op.D);
  const double ds = 2.0 / side;
  const std::vector<double> cheb_up(cn.rbegin(), cn.rend());
  const HostMat c2g = bary_interp(cheb_up, gx);  // q x p, ascending Chebyshev -> Gauss

  op.P = HostMat(op.ne, op.nb);
  op.Q = HostMat(op.nb, op.n);
  if (dim == 2) {
    // side s: normal axis, outward sign, Chebyshev node on the normal axis (spectral.cpp:172-188)
    const int nax[4] = {1, 0, 1, 0};
    const double sgn[4] = {-1, 1, 1, -1};
    const int fixed[4] = {p - 1, 0, 0, p - 1};
    for (int r = 0; r < op.ne; ++r) {
      const int i1 = op.exterior[r] / p, i2 = op.exterior[r] % p;
      int own[2], no = 0;
      if (i2 == p - 1) own[no++] = 0;
      if (i1 == 0) own[no++] = 1;
      if (i2 == 0) own[no++] = 2;
      if (i1 == p - 1) own[no++] = 3;
      for (int o = 0; o < no; ++o) {
        const int s = own[o];
        const double t = nax[s] == 0 ? cn[i2] : cn[i1];
        const HostMat row = bary_interp(gx, {t});
        for (int j = 0; j < q; ++j) op.P(r, s * q + j) += (1.0 / no) * row(0, j);
      }
    }
    for (int s = 0; s < 4; ++s) {
      HostMat ns(p, op.n);
      for (int r = 0; r < p; ++r) {
        const int run = p - 1 - r;
        for (int k = 0; k < p; ++k) {
          const int col = nax[s] == 0 ? k * p + run : run * p + k;
          ns(r, col) += sgn[s] * op.D(fixed[s], k);
        }
      }
      const HostMat blk = matmul(c2g, ns);
      for (int i = 0; i < q; ++i)
        for (int j = 0; j < op.n; ++j) op.Q(s * q + i, j) = ds * blk(i, j);
    }
  } else {
    auto face = [&](int f, int& axis, double& sg, int& fixed_node, int& ua, int& va) {
      axis = f / 2;
      sg = (f % 2 == 0) ? -1.0 : 1.0;
      fixed_node = (f % 2 == 0) ? p - 1 : 0;
      ua = axis == 0 ? 1 : 0;
      va = axis == 2 ? 1 : 2;
    };
    for (int r = 0; r < op.ne; ++r) {
      const int idx = op.exterior[r];
      const int ijk[3] = {idx / (p * p), (idx / p) % p, idx % p};
      int own[3], no = 0;
      for (int a = 0; a < 3; ++a) {
        if (ijk[a] == p - 1) own[no++] = 2 * a;
        if (ijk[a] == 0) own[no++] = 2 * a + 1;
      }
      for (int o = 0; o < no; ++o) {
        int axis, fx, ua, va;
        double sg;
        face(own[o], axis, sg, fx, ua, va);
        const HostMat ru = bary_interp(gx, {cn[ijk[ua]]}), rv = bary_interp(gx, {cn[ijk[va]]});
        for (int a = 0; a < q; ++a)
          for (int b = 0; b < q; ++b) op.P(r, own[o] * q * q + a * q + b) += (1.0 / no) * ru(0, a) * rv(0, b);
      }
    }
    HostMat fi(q * q, p * p);  // kron(c2g, c2g)
    for (int a = 0; a < q; ++a)
      for (int b = 0; b < q; ++b)
        for (int i = 0; i < p; ++i)
          for (int j = 0; j < p; ++j) fi(a * q + b, i * p + j) = c2g(a, i) * c2g(b, j);
    for (int f = 0; f < 6; ++f) {
      int axis, fx, ua, va;
      double sg;
      face(f, axis, sg, fx, ua, va);
      HostMat nf(p * p, op.n);
      for (int ru = 0; ru < p; ++ru)
        for (int rv = 0; rv < p; ++rv)
          for (int k = 0; k < p; ++k) {
            int id[3];
            id[axis] = k;
            id[ua] = p - 1 - ru;
            id[va] = p - 1 - rv;
            nf(ru * p + rv, (id[0] * p + id[1]) * p + id[2]) += sg * op.D(fx, k);
          }
      const HostMat blk = matmul(fi, nf);
      for (int i = 0; i < q * q; ++i)
        for (int j = 0; j < op.n; ++j) op.Q(f * q * q + i, j) = ds * blk(i, j);
    }
  }
  op.Qi = HostMat(op.nb, op.ni);
  HostMat Qe(op.nb, op.ne);
  for (int i = 0; i < op.nb; ++i) {
    for (int j = 0; j < op.ni; ++j) op.Qi(i, j) = op.Q(i, op.interior[j]);
    for (int j = 0; j < op.ne; ++j) Qe(i, j) = op.Q(i, op.exterior[j]);
  }
  op.QeP = matmul(Qe, op.P);
  return op;
}

void q_interior_factors(const LeafOperators& op, std::vector<double>& G, std::vector<double>& d, double& ds) {
  const int p = op.p, q = op.q, n1 = p - 2;
  std::vector<double> gx, gw;
  gauss_rule(q, gx, gw);
  const std::vector<double> cn = cheb_nodes(p);
  const std::vector<double> cheb_up(cn.rbegin(), cn.rend());
  const HostMat c2g = bary_interp(cheb_up, gx);  // the same interpolant make_leaf_operators uses
  const double sgn[4] = {-1, 1, 1, -1};
  const int fixed[4] = {p - 1, 0, 0, p - 1};
  G.assign(size_t(q) * n1, 0.0);
  d.assign(size_t(4) * n1, 0.0);
  for (int i = 0; i < q; ++i)
    for (int m = 0; m < n1; ++m) G[size_t(i) * n1 + m] = c2g(i, p - 2 - m);
  for (int s = 0; s < 4; ++s)
    for (int k = 0; k < n1; ++k) d[size_t(s) * n1 + k] = sgn[s] * op.D(fixed[s], k + 1);
  ds = 2.0 / op.side;
}

long long UniformTree::level_first_id(int d) const {
  // reference id of the first node at part depth d (breadth-first ids of the FULL tree, mesh.cpp:113-118)
  long long id = 0, cnt = 1;
  for (int k = 0; k < root_depth + d; ++k) id += cnt, cnt *= nchild;
  long long off = root_index;
  for (int k = 0; k < d; ++k) off *= nchild;
  return id + off;
}
long long UniformTree::level_count(int d) const {
  long long c = 1;
  for (int k = 0; k < d; ++k) c *= nchild;
  return c;
}

UniformTree make_part_tree(int dim, int p, int L_full, double lo, double hi, int root_depth, long long root_index,
                           int cut_depth) {
  if (!(hi > lo)) throw std::runtime_error("build_uniform_tree: empty domain");
  if (root_depth < 0 || cut_depth <= root_depth || cut_depth > L_full)
    throw std::runtime_error("tree part: need 0 <= root_depth < cut_depth <= L");
  UniformTree t;
  t.dim = dim;
  t.p = p;
  t.q = p - 2;
  t.L = cut_depth - root_depth;
  t.L_full = L_full;
  t.root_depth = root_depth;
  t.root_index = root_index;
  t.cut = cut_depth < L_full;
  t.lo = lo;
  t.hi = hi;
  t.nchild = dim == 2 ? 4 : 8;
  t.nface = 2 * dim;
  if (root_index < 0 || root_index >= t.level_count(root_depth))
    throw std::runtime_error("tree part: root index out of range");
  // part root box: repeated midpoint splits along the path from the domain root (mesh.cpp:31-43)
  double blo[3] = {lo, lo, dim == 3 ? lo : 0.0}, bhi[3] = {hi, hi, dim == 3 ? hi : 0.0};
  long long div = t.level_count(root_depth);
  for (int l = 0; l < root_depth; ++l) {
    div /= t.nchild;
    const int c = int((root_index / div) % t.nchild);
    for (int k = 0; k < dim; ++k) {
      const double mid = 0.5 * (blo[k] + bhi[k]);
      if (kChildOffset[c][k])
        blo[k] = mid;
      else
        bhi[k] = mid;
    }
  }
  for (int k = 0; k < 3; ++k) t.rlo[k] = blo[k], t.rhi[k] = bhi[k];
  if (!t.cut) {
    const long long nl = t.level_count(t.L);
    t.leaf_lo.assign(size_t(nl) * 6, 0.0);  // lo[3], hi[3] per leaf, DFS order within the part
    for (long long o = 0; o < nl; ++o) {
      double a[3] = {t.rlo[0], t.rlo[1], t.rlo[2]}, b[3] = {t.rhi[0], t.rhi[1], t.rhi[2]};
      long long dv = nl;
      for (int l = 0; l < t.L; ++l) {
        dv /= t.nchild;
        const int c = int((o / dv) % t.nchild);
        for (int k = 0; k < dim; ++k) {
          const double mid = 0.5 * (a[k] + b[k]);
          if (kChildOffset[c][k])
            a[k] = mid;
          else
            b[k] = mid;
        }
      }
      for (int k = 0; k < 3; ++k) t.leaf_lo[size_t(o) * 6 + k] = a[k], t.leaf_lo[size_t(o) * 6 + 3 + k] = b[k];
    }
  }
  t.leaf_side = (hi - lo) / double(1LL << L_full);
  return t;
}

UniformTree make_uniform_tree(int dim, int p, int L, double lo, double hi) {
  return make_part_tree(dim, p, L, lo, hi, 0, 0, L);
}

const std::vector<Iface>& ifaces(int dim) {
  // proj/src/merge.cpp:20-33
  static const std::vector<Iface> i2 = {{0, 1, 1, 3}, {1, 2, 2, 0}, {3, 1, 2, 3}, {0, 2, 3, 0}};
  static const std::vector<Iface> i3 = {{0, 1, 1, 0}, {1, 3, 2, 2}, {3, 1, 2, 0}, {0, 3, 3, 2},
                                        {4, 1, 5, 0}, {5, 3, 6, 2}, {7, 1, 6, 0}, {4, 3, 7, 2},
                                        {0, 5, 4, 4}, {1, 5, 5, 4}, {2, 5, 6, 4}, {3, 5, 7, 4}};
  return dim == 2 ? i2 : i3;
}
// exterior position (parent face, quadrant) of a child face, or -1 (merge.cpp:41-56)
int ext_qpos(int dim, int c, int f) {
  const int* off = kChildOffset[c];
  if (dim == 2) {
    const int axis = (f == 1 || f == 3) ? 0 : 1, high = (f == 1 || f == 2) ? 1 : 0;
    if (off[axis] != high) return -1;
    return off[axis == 0 ? 1 : 0];
  }
  const int axis = f / 2, high = f % 2;
  if (off[axis] != high) return -1;
  const int ua = axis == 0 ? 1 : 0, va = axis == 2 ? 1 : 2;
  return off[ua] * 2 + off[va];
}

bool face_on_domain_boundary(int dim, int d, long long idx, int f) {
  const int nchild = dim == 2 ? 4 : 8;
  const int axis = dim == 2 ? ((f == 1 || f == 3) ? 0 : 1) : f / 2;
  const int high = dim == 2 ? ((f == 1 || f == 2) ? 1 : 0) : f % 2;
  long long pos = 0;  // the node's grid position along `axis` at depth d (child digits, most significant first)
  for (int k = 0; k < d; ++k) {
    long long div = 1;
    for (int j = k + 1; j < d; ++j) div *= nchild;
    const int c = int((idx / div) % nchild);
    pos = 2 * pos + kChildOffset[c][axis];
  }
  return high ? pos == (1LL << d) - 1 : pos == 0;
}

MergeTables make_merge_tables(int dim, int s) {
  MergeTables m;
  m.dim = dim;
  m.s = s;
  m.nchild = dim == 2 ? 4 : 8;
  m.nface = 2 * dim;
  const int nquad = dim == 2 ? 2 : 4;
  const auto& ifs = ifaces(dim);
  m.NI = int(ifs.size());
  m.NE = m.nface * nquad;
  m.sec.assign(m.nchild * m.nface, 0);
  for (int c = 0; c < m.nchild; ++c)
    for (int f = 0; f < m.nface; ++f) {
      const int qp = ext_qpos(dim, c, f);
      if (qp >= 0) {
        m.sec[c * m.nface + f] = f * nquad + qp;
      } else {
        int t = -1;
        for (int k = 0; k < m.NI; ++k)
          if ((ifs[k].clo == c && ifs[k].flo == f) || (ifs[k].chi == c && ifs[k].fhi == f)) t = k;
        if (t < 0) throw std::runtime_error("make_merge_tables: unmatched face");
        m.sec[c * m.nface + f] = -t - 1;
      }
    }
  const int mdc = m.NI + 1 + m.NE, ahc = 1 + m.NE;
  m.md_src.assign(m.NI * mdc * 2, -1);
  m.b_src.assign(m.NE * m.NI * 2, -1);
  m.ah_src.assign(m.NE * ahc * 2, -1);
  auto add = [](std::vector<int>& tab, int slot, int code) {
    if (tab[2 * slot] < 0)
      tab[2 * slot] = code;
    else if (tab[2 * slot + 1] < 0)
      tab[2 * slot + 1] = code;
    else
      throw std::runtime_error("make_merge_tables: more than two contributions");
  };
  // MD = [D | h_int | C] (rows: interfaces), B (ext x int), AH = [h_ext | A]
  for (int c = 0; c < m.nchild; ++c)
    for (int rf = 0; rf < m.nface; ++rf) {
      const int rs = m.sec[c * m.nface + rf];
      for (int cf = -1; cf < m.nface; ++cf) {
        const int code = c * 64 + rf * 8 + (cf + 1);
        if (cf < 0) {
          if (rs >= 0)
            add(m.ah_src, rs * ahc + 0, code);
          else
            add(m.md_src, (-rs - 1) * mdc + m.NI, code);
          continue;
        }
        const int cs = m.sec[c * m.nface + cf];
        if (rs >= 0 && cs >= 0)
          add(m.ah_src, rs * ahc + 1 + cs, code);
        else if (rs >= 0)
          add(m.b_src, rs * m.NI + (-cs - 1), code);
        else if (cs >= 0)
          add(m.md_src, (-rs - 1) * mdc + m.NI + 1 + cs, code);
        else
          add(m.md_src, (-rs - 1) * mdc + (-cs - 1), code);
      }
    }
  m.down.assign(m.nchild * m.nface, 0);
  for (int c = 0; c < m.nchild; ++c)
    for (int f = 0; f < m.nface; ++f) {
      const int sc = m.sec[c * m.nface + f];
      m.down[c * m.nface + f] = sc >= 0 ? sc * s : -((-sc - 1) * s) - 1;
    }
  return m;
}

namespace {
// proj/src/layout.cpp:89-119 for uniform layouts of depth `levels`
void collect(double lo[3], double hi[3], int dim, int face, int levels, int q, const std::vector<double>& gx,
             std::vector<double>& out) {
  if (levels == 0) {
    auto map1 = [&](double t, int k) { return 0.5 * (lo[k] + hi[k]) + 0.5 * (hi[k] - lo[k]) * t; };
    if (dim == 2) {
      for (int i = 0; i < q; ++i) {
        double x[3] = {0, 0, 0};
        switch (face) {
          case 0: x[0] = map1(gx[i], 0); x[1] = lo[1]; break;
          case 1: x[0] = hi[0]; x[1] = map1(gx[i], 1); break;
          case 2: x[0] = map1(gx[i], 0); x[1] = hi[1]; break;
          default: x[0] = lo[0]; x[1] = map1(gx[i], 1); break;
        }
        out.insert(out.end(), x, x + 3);
      }
    } else {
      const int axis = face / 2, ua = axis == 0 ? 1 : 0, va = axis == 2 ? 1 : 2;
      const double fixed = face % 2 == 0 ? lo[axis] : hi[axis];
      for (int iu = 0; iu < q; ++iu)
        for (int iv = 0; iv < q; ++iv) {
          double x[3];
          x[axis] = fixed;
          x[ua] = map1(gx[iu], ua);
          x[va] = map1(gx[iv], va);
          out.insert(out.end(), x, x + 3);
        }
    }
    return;
  }
  double mid[3];
  for (int k = 0; k < 3; ++k) mid[k] = 0.5 * (lo[k] + hi[k]);
  if (dim == 2) {
    const int axis = (face == 0 || face == 2) ? 0 : 1;
    for (int h = 0; h < 2; ++h) {
      double sl[3] = {lo[0], lo[1], lo[2]}, sh[3] = {hi[0], hi[1], hi[2]};
      (h ? sl : sh)[axis] = mid[axis];
      collect(sl, sh, dim, face, levels - 1, q, gx, out);
    }
  } else {
    const int fa = face / 2, ua = fa == 0 ? 1 : 0, va = fa == 2 ? 1 : 2;
    for (int hu = 0; hu < 2; ++hu)
      for (int hv = 0; hv < 2; ++hv) {
        double sl[3] = {lo[0], lo[1], lo[2]}, sh[3] = {hi[0], hi[1], hi[2]};
        (hu ? sl : sh)[ua] = mid[ua];
        (hv ? sl : sh)[va] = mid[va];
        collect(sl, sh, dim, face, levels - 1, q, gx, out);
      }
  }
}
}  // namespace

// ---- ItI --------------------------------------------------------------------------------------
namespace {
// side2d (spectral.cpp:172-188): normal axis, outward sign, fixed Chebyshev node
void side2d(int s, int p, int& axis, double& sign, int& fixed) {
  switch (s) {
    case 0: axis = 1, sign = -1.0, fixed = p - 1; break;
    case 1: axis = 0, sign = +1.0, fixed = 0; break;
    case 2: axis = 1, sign = +1.0, fixed = 0; break;
    default: axis = 0, sign = -1.0, fixed = p - 1; break;
  }
}
// normal_row_2d (spectral.cpp:204-211)
void normal_row(int s, int run, int p, const HostMat& d1, HostMat& mat, int row) {
  int axis, fixed;
  double sign;
  side2d(s, p, axis, sign, fixed);
  for (int k = 0; k < p; ++k) {
    const int col = axis == 0 ? k * p + run : run * p + k;
    mat(row, col) += sign * d1(fixed, k);
  }
}
// walk_tensor_idx (spectral.cpp:224-227)
int walk_idx(int s, int run, int p) {
  int axis, fixed;
  double sign;
  side2d(s, p, axis, sign, fixed);
  return axis == 0 ? fixed * p + run : run * p + fixed;
}
}  // namespace

ItiLeafOperators make_iti_leaf_operators(int p, double eta, double side) {
  if (p < 4) throw std::runtime_error("assemble_iti_ops_2d: p must be >= 4");
  if (!(eta > 0.0)) throw std::runtime_error("assemble_iti_ops_2d: eta must be positive");
  ItiLeafOperators op;
  op.p = p;
  op.q = p - 2;
  op.n = p * p;
  op.nbc = 4 * p - 4;
  op.nb = 4 * op.q;
  op.eta = eta;
  op.side = side;
  for (int idx = 0; idx < op.n; ++idx) {
    const int i1 = idx / p, i2 = idx % p;
    if (i1 > 0 && i1 < p - 1 && i2 > 0 && i2 < p - 1) op.interior.push_back(idx);
  }
  op.ni = int(op.interior.size());
  const int q = op.q;
  const std::vector<double> cn = cheb_nodes(p);
  std::vector<double> gx, gw;
  gauss_rule(q, gx, gw);
  const HostMat d1 = cheb_diff(p);
  const double dscale = 2.0 / side;
  const std::vector<double> cheb_asc(cn.rbegin(), cn.rend());
  const HostMat c2g = bary_interp(cheb_asc, gx);  // q x p
  // N and the sampling rows on the 4p double-counted layout (spectral.cpp:333-342)
  HostMat N(4 * p, op.n), samp(4 * p, op.n);
  for (int s = 0; s < 4; ++s)
    for (int r = 0; r < p; ++r) {
      const int run = p - 1 - r;
      normal_row(s, run, p, d1, N, s * p + r);
      samp(s * p + r, walk_idx(s, run, p)) = 1.0;
    }
  // the 4p-4 walk (iti_walk, spectral.cpp:214-222): Ntilde, G = Ntilde + i eta samp_walk, P
  std::vector<std::pair<int, int>> walk;
  for (int i1 = p - 1; i1 >= 1; --i1) walk.emplace_back(0, i1);
  for (int i2 = p - 1; i2 >= 1; --i2) walk.emplace_back(1, i2);
  for (int i1 = 0; i1 <= p - 2; ++i1) walk.emplace_back(2, i1);
  for (int i2 = 0; i2 <= p - 2; ++i2) walk.emplace_back(3, i2);
  op.Gr = HostMat(op.nbc, op.n);
  op.Gi = HostMat(op.nbc, op.n);
  op.P = HostMat(op.nbc, op.nb);
  for (int r = 0; r < op.nbc; ++r) {
    const int s = walk[r].first, run = walk[r].second;
    normal_row(s, run, p, d1, op.Gr, r);
    op.Gi(r, walk_idx(s, run, p)) = eta;
    const HostMat row = bary_interp(gx, {cn[run]});
    for (int j = 0; j < q; ++j) op.P(r, s * q + j) = row(0, j);
  }
  for (double& v : op.Gr.a) v *= dscale;
  // QH = Q (N dscale - i eta samp), Q block-diagonal per side (spectral.cpp:362-366)
  op.QHr = HostMat(op.nb, op.n);
  op.QHi = HostMat(op.nb, op.n);
  for (int s = 0; s < 4; ++s)
    for (int i = 0; i < q; ++i)
      for (int j = 0; j < op.n; ++j) {
        double nr = 0.0, ni = 0.0;
        for (int r = 0; r < p; ++r) {
          nr += c2g(i, r) * N(s * p + r, j);
          ni += c2g(i, r) * samp(s * p + r, j);
        }
        op.QHr(s * q + i, j) = dscale * nr;
        op.QHi(s * q + i, j) = -eta * ni;
      }
  return op;
}

ItiMergeTables make_iti_merge_tables(int s) {
  const MergeTables g = make_merge_tables(2, s);  // exterior sections and interface ids (MergeGeom)
  ItiMergeTables t;
  t.s = s;
  const int nint_c = 8 * s, next_c = 8 * s, nbc_c = 4 * s;
  t.n_int = 2 * nint_c;
  t.n_ext = 2 * next_c;
  t.child_nb = 2 * nbc_c;
  auto ext_off = [&](int c, int f) { const int v = g.sec[c * 4 + f]; return v >= 0 ? v * s : -1; };
  // slots grouped {a, c} then {b, d}, each child's interfaces by id (merge.cpp:351-375)
  int slot_off[4][4];
  for (auto& r : slot_off)
    for (int& v : r) v = -1;
  struct Slot { int k, of, nb, nbf, off; };
  std::vector<Slot> slots;
  const auto& ifs = ifaces(2);
  int pos = 0;
  for (int k : {0, 2, 1, 3})
    for (size_t i = 0; i < ifs.size(); ++i) {
      int of, nb, nbf;
      if (ifs[i].clo == k) {
        of = ifs[i].flo, nb = ifs[i].chi, nbf = ifs[i].fhi;
      } else if (ifs[i].chi == k) {
        of = ifs[i].fhi, nb = ifs[i].clo, nbf = ifs[i].flo;
      } else {
        continue;
      }
      slots.push_back({k, of, nb, nbf, pos});
      slot_off[k][of] = pos;
      pos += s;
    }
  // Real-equivalent index of interface unknown o (complex offset) and part q (0 re, 1 im): half-blocked,
  // [re(top); im(top); re(bottom); im(bottom)] with top = the {a, c} slots, so that D = [[I, D12], [D21, I]]
  // keeps its complex 2 x 2 block structure and merge_iti's W = I - D12 D21 (merge.cpp:447-463) is a
  // contiguous real-equivalent block.  Exterior vectors stay [re; im].
  const int hc = nint_c / 2;
  auto ri = [&](int q, int o) { return o < hc ? q * hc + o : nint_c + q * hc + (o - hc); };
  auto xi = [&](int q, int o) { return q * next_c + o; };
  // complex s x s block of child k's T (faces rf, cf) or h (cf < 0) into matrix dst: rows at complex offset r
  // (interface rows when rint), columns at complex offset c (interface columns when cint) after column base cb
  auto tblock = [&](int dst, bool rint, bool cint, int cb, int r, int c, int k, int rf, int cf) {
    for (int qr = 0; qr < 2; ++qr)
      for (int qc = 0; qc < 2; ++qc)
        t.blocks.push_back({dst, rint ? ri(qr, r) : xi(qr, r), cb + (cint ? ri(qc, c) : xi(qc, c)), k,
                            qr * nbc_c + rf * s, 1 + qc * nbc_c + cf * s, s, s});
  };
  auto hblock = [&](int dst, bool rint, int col, int r, int k, int rf) {
    for (int qr = 0; qr < 2; ++qr)
      t.blocks.push_back({dst, rint ? ri(qr, r) : xi(qr, r), col, k, qr * nbc_c + rf * s, 0, s, 1});
  };
  // exterior rows: h_ext, A, B from each child's exterior faces (merge.cpp:386-415)
  for (int k = 0; k < 4; ++k)
    for (int rf = 0; rf < 4; ++rf) {
      const int roff = ext_off(k, rf);
      if (roff < 0) continue;
      hblock(2, false, 0, roff, k, rf);
      for (int cf = 0; cf < 4; ++cf) {
        if (ext_off(k, cf) >= 0)
          tblock(2, false, false, 1, roff, ext_off(k, cf), k, rf, cf);  // A in [h_ext | A]
        else
          tblock(1, false, true, 0, roff, slot_off[k][cf], k, rf, cf);  // B
      }
    }
  // interface rows: g_owner + neighbour's outgoing data = 0 (merge.cpp:417-447)
  for (const Slot& sl : slots) {
    hblock(0, true, 2 * nint_c, sl.off, sl.nb, sl.nbf);  // h_int column of [D | h_int | C]
    for (int qr = 0; qr < 2; ++qr) t.blocks.push_back({0, ri(qr, sl.off), ri(qr, sl.off), -1, 0, 0, s, s});
    for (int cf = 0; cf < 4; ++cf) {
      if (ext_off(sl.nb, cf) >= 0)
        tblock(0, true, false, 2 * nint_c + 1, sl.off, ext_off(sl.nb, cf), sl.nb, sl.nbf, cf);  // C
      else
        tblock(0, true, true, 0, sl.off, slot_off[sl.nb][cf], sl.nb, sl.nbf, cf);  // D
    }
  }
  // downward scatter per (child, real-equivalent face): real parts then imaginary parts
  t.down.assign(4 * 8, 0);
  for (int c = 0; c < 4; ++c)
    for (int f = 0; f < 4; ++f) {
      const int e = ext_off(c, f);
      t.down[c * 8 + f] = e >= 0 ? xi(0, e) : -ri(0, slot_off[c][f]) - 1;
      t.down[c * 8 + 4 + f] = e >= 0 ? xi(1, e) : -ri(1, slot_off[c][f]) - 1;
    }
  return t;
}

std::vector<double> root_boundary_points(const UniformTree& t) {
  std::vector<double> gx, gw, out;
  gauss_rule(t.q, gx, gw);
  for (int f = 0; f < t.nface; ++f) {
    double lo[3] = {t.rlo[0], t.rlo[1], t.rlo[2]}, hi[3] = {t.rhi[0], t.rhi[1], t.rhi[2]};
    collect(lo, hi, t.dim, f, t.L_full - t.root_depth, t.q, gx, out);
  }
  return out;
}


namespace {
// x <- M^-1 b for a dense n x n M (column-major copy), partial pivoting; false if singular
bool dense_solve(std::vector<double> M, int n, std::vector<double>& b) {
  for (int k = 0; k < n; ++k) {
    int r = k;
    for (int i = k + 1; i < n; ++i)
      if (std::fabs(M[size_t(k) * n + i]) > std::fabs(M[size_t(k) * n + r])) r = i;
    if (M[size_t(k) * n + r] == 0.0) return false;
    if (r != k) {
      for (int j = 0; j < n; ++j) std::swap(M[size_t(j) * n + k], M[size_t(j) * n + r]);
      std::swap(b[size_t(k)], b[size_t(r)]);
    }
    for (int i = k + 1; i < n; ++i) {
      const double l = M[size_t(k) * n + i] / M[size_t(k) * n + k];
      for (int j = k + 1; j < n; ++j) M[size_t(j) * n + i] -= l * M[size_t(j) * n + k];
      b[size_t(i)] -= l * b[size_t(k)];
    }
  }
  for (int k = n - 1; k >= 0; --k) {
    double s = b[size_t(k)];
    for (int j = k + 1; j < n; ++j) s -= M[size_t(j) * n + k] * b[size_t(j)];
    b[size_t(k)] = s / M[size_t(k) * n + k];
  }
  return true;
}
}  // namespace

bool real_eigendecomposition(const std::vector<double>& A, int n, std::vector<double>& lam, std::vector<double>& V,
                             std::vector<double>& Vinv) {
  auto at = [n](std::vector<double>& M, int i, int j) -> double& { return M[size_t(j) * n + i]; };
  std::vector<double> H = A;
  double anorm = 0.0;
  for (double v : A) anorm = std::max(anorm, std::fabs(v));
  if (!(anorm > 0.0) || !std::isfinite(anorm)) return false;
  // Householder reduction to upper Hessenberg form
  for (int k = 0; k + 2 < n; ++k) {
    double alpha = 0.0;
    for (int i = k + 1; i < n; ++i) alpha += at(H, i, k) * at(H, i, k);
    alpha = std::sqrt(alpha);
    if (alpha == 0.0) continue;
    if (at(H, k + 1, k) > 0) alpha = -alpha;
    std::vector<double> v(size_t(n), 0.0);
    v[size_t(k + 1)] = at(H, k + 1, k) - alpha;
    for (int i = k + 2; i < n; ++i) v[size_t(i)] = at(H, i, k);
    double vn = 0.0;
    for (double x : v) vn += x * x;
    if (vn == 0.0) continue;
    for (int j = 0; j < n; ++j) {  // H <- (I - 2vv'/v'v) H
      double s = 0.0;
      for (int i = k + 1; i < n; ++i) s += v[size_t(i)] * at(H, i, j);
      s = 2.0 * s / vn;
      for (int i = k + 1; i < n; ++i) at(H, i, j) -= s * v[size_t(i)];
    }
    for (int i = 0; i < n; ++i) {  // H <- H (I - 2vv'/v'v)
      double s = 0.0;
      for (int j = k + 1; j < n; ++j) s += at(H, i, j) * v[size_t(j)];
      s = 2.0 * s / vn;
      for (int j = k + 1; j < n; ++j) at(H, i, j) -= s * v[size_t(j)];
    }
  }
  // shifted QR (Givens) on the active leading block; deflate from the bottom
  lam.assign(size_t(n), 0.0);
  int m = n - 1, iters = 0;
  while (m >= 0) {
    if (m == 0) {
      lam[0] = at(H, 0, 0);
      break;
    }
    const double sub = std::fabs(at(H, m, m - 1));
    if (sub <= 1e-16 * (std::fabs(at(H, m, m)) + std::fabs(at(H, m - 1, m - 1)))) {
      lam[size_t(m)] = at(H, m, m);
      --m;
      iters = 0;
      continue;
    }
    if (++iters > 200) return false;
    // Wilkinson shift: eigenvalue of the trailing 2x2 closest to H(m, m); complex pair -> no real decomposition
    const double a = at(H, m - 1, m - 1), b = at(H, m - 1, m), c = at(H, m, m - 1), d = at(H, m, m);
    const double tr = 0.5 * (a - d), disc = tr * tr + b * c;
    if (disc < 0.0 && iters > 20) return false;
    double mu = d;
    if (disc >= 0.0) {
      const double r = std::sqrt(disc);
      mu = d - b * c / (tr + (tr >= 0 ? r : -r));
      if (!std::isfinite(mu)) mu = d;
    }
    for (int i = 0; i <= m; ++i) at(H, i, i) -= mu;
    std::vector<double> cs(static_cast<size_t>(m)), sn(static_cast<size_t>(m));
    for (int k = 0; k < m; ++k) {  // H = QR
      const double x = at(H, k, k), y = at(H, k + 1, k);
      const double r = std::hypot(x, y);
      const double cc = r == 0.0 ? 1.0 : x / r, ss = r == 0.0 ? 0.0 : y / r;
      cs[size_t(k)] = cc, sn[size_t(k)] = ss;
      for (int j = k; j <= m; ++j) {
        const double t1 = at(H, k, j), t2 = at(H, k + 1, j);
        at(H, k, j) = cc * t1 + ss * t2;
        at(H, k + 1, j) = -ss * t1 + cc * t2;
      }
    }
    for (int k = 0; k < m; ++k) {  // H = RQ
      const double cc = cs[size_t(k)], ss = sn[size_t(k)];
      for (int i = 0; i <= std::min(k + 1, m); ++i) {
        const double t1 = at(H, i, k), t2 = at(H, i, k + 1);
        at(H, i, k) = cc * t1 + ss * t2;
        at(H, i, k + 1) = -ss * t1 + cc * t2;
      }
    }
    for (int i = 0; i <= m; ++i) at(H, i, i) += mu;
  }
  std::vector<double> sorted = lam;
  std::sort(sorted.begin(), sorted.end());
  for (int i = 1; i < n; ++i)
    if (!(std::fabs(sorted[size_t(i)] - sorted[size_t(i - 1)]) > 1e-10 * anorm)) return false;  // distinct
  // eigenvectors by inverse iteration on the original matrix
  V.assign(size_t(n) * n, 0.0);
  for (int e = 0; e < n; ++e) {
    std::vector<double> M = A;
    const double shift = lam[size_t(e)] + 1e-12 * anorm;
    for (int i = 0; i < n; ++i) M[size_t(i) * n + i] -= shift;
    std::vector<double> x(size_t(n), 1.0);
    for (int it = 0; it < 3; ++it) {
      if (!dense_solve(M, n, x)) return false;
      double mx = 0.0;
      for (double v : x) mx = std::max(mx, std::fabs(v));
      if (!(mx > 0.0) || !std::isfinite(mx)) return false;
      for (double& v : x) v /= mx;
    }
    for (int i = 0; i < n; ++i) V[size_t(e) * n + i] = x[size_t(i)];
  }
  // V^-1 column by column, then the residual checks
  Vinv.assign(size_t(n) * n, 0.0);
  for (int j = 0; j < n; ++j) {
    std::vector<double> col(size_t(n), 0.0);
    col[size_t(j)] = 1.0;
    if (!dense_solve(V, n, col)) return false;
    for (int i = 0; i < n; ++i) Vinv[size_t(j) * n + i] = col[size_t(i)];
  }
  double res = 0.0, idr = 0.0;
  for (int i = 0; i < n; ++i)
    for (int e = 0; e < n; ++e) {
      double s = 0.0, t = 0.0;
      for (int k = 0; k < n; ++k) {
        s += A[size_t(k) * n + i] * V[size_t(e) * n + k];
        t += Vinv[size_t(k) * n + i] * V[size_t(e) * n + k];
      }
      res = std::max(res, std::fabs(s - lam[size_t(e)] * V[size_t(e) * n + i]));
      idr = std::max(idr, std::fabs(t - (i == e ? 1.0 : 0.0)));
    }
  return res <= 1e-11 * anorm && idr <= 1e-11;
}

}  // namespace hpsg
