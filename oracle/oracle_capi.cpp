// oracle_capi.cpp -- TEST INFRASTRUCTURE ONLY: extern "C" face of the CPU oracle.
#include "oracle_capi.h"

#include <cmath>
#include <cstring>
#include <memory>
#include <random>
#include <string>

#include "field_eval.hpp"
#include "hps_oracle.hpp"

using namespace hpso;
using hpso_fields::FieldEval;

namespace {
thread_local std::string g_err;

int guard(const std::function<void()>& fn) {
  try {
    fn();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

std::shared_ptr<FieldEval> make_field(const oracle_field& f, int dim, int npts, int n_leaves) {
  auto fe = std::make_shared<FieldEval>();
  fe->f = f;
  fe->dim = dim;
  fe->npts = npts;
  if (f.n_centers > 0) fe->centers.assign(f.centers, f.centers + 3 * f.n_centers);
  if (f.kind == ORACLE_FIELD_SAMPLED) {
    require(f.samples != nullptr, "oracle: sampled field without samples");
    fe->samples.assign(f.samples, f.samples + size_t(npts) * n_leaves);
  }
  fe->f.centers = nullptr;
  fe->f.samples = nullptr;
  return fe;
}

struct Handle {
  Tree tree;
  std::unique_ptr<Solver> solver;
  std::vector<std::shared_ptr<FieldEval>> fields;
  bool built = false;
};

void copy_mat(const Mat& m, double* out) {
  if (out) std::memcpy(out, m.data(), sizeof(double) * m.a.size());
}
void copy_vec(const Vec& v, double* out) {
  if (out) std::memcpy(out, v.data(), sizeof(double) * v.size());
}
Box make_box(const double* lo, const double* hi, int dim) {
  Box b;
  for (int k = 0; k < dim; ++k) b.lo[k] = lo[k], b.hi[k] = hi[k];
  return b;
}
}  // namespace

extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }
int oracle_blas_available(void) { return blas_available(); }
void oracle_set_threads(int n) { set_blas_threads(n); }

void oracle_bump_centers(unsigned long long seed, int n, int dim, double* out) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(-0.5, 0.5);
  for (int i = 0; i < n; ++i) {
    out[3 * i + 0] = dist(rng);
    out[3 * i + 1] = dist(rng);
    out[3 * i + 2] = dim == 3 ? dist(rng) : 0.0;
  }
}

void oracle_cheb_lobatto(int p, double* out) { copy_vec(cheb_lobatto_1d(p), out); }
void oracle_cheb_weights(int p, double* out) { copy_vec(cheb_lobatto_weights(p), out); }
int oracle_gauss(int q, double* nodes, double* weights) {
  return guard([&] {
    const GaussRule g = gauss_legendre_1d(q);
    copy_vec(g.nodes, nodes);
    copy_vec(g.weights, weights);
  });
}
void oracle_diff_matrix(int p, double* out) { copy_mat(cheb_diff_matrix(p), out); }
int oracle_interp_matrix(const double* src, int n, const double* dst, int m, double* out) {
  return guard([&] { copy_mat(barycentric_interp_matrix(Vec(src, src + n), Vec(dst, dst + m)), out); });
}
int oracle_dtn_ops(int dim, int p, double side, double* P, double* Q, int* pr, int* pc, int* qr, int* qc) {
  return guard([&] {
    const LeafOps ops = dim == 2 ? assemble_dtn_ops_2d(p, p - 2, side) : assemble_dtn_ops_3d(p, p - 2, side);
    *pr = ops.P.r;
    *pc = ops.P.c;
    *qr = ops.Q.r;
    *qc = ops.Q.c;
    copy_mat(ops.P, P);
    copy_mat(ops.Q, Q);
  });
}
int oracle_index_sets(int p, int dim, int* interior, int* exterior) {
  return guard([&] {
    const IndexSets s = leaf_index_sets(p, dim);
    if (interior) std::memcpy(interior, s.interior.data(), sizeof(int) * s.interior.size());
    if (exterior) std::memcpy(exterior, s.exterior.data(), sizeof(int) * s.exterior.size());
  });
}
void oracle_leaf_cheb_points(const double* lo, const double* hi, int p, int dim, double* out) {
  const auto pts = leaf_cheb_points(make_box(lo, hi, dim), p, dim);
  for (size_t i = 0; i < pts.size(); ++i)
    for (int k = 0; k < 3; ++k) out[3 * i + k] = pts[i][k];
}
void oracle_gauss_boundary_points(const double* lo, const double* hi, int q, int dim, double* out) {
  const auto pts = leaf_gauss_boundary_points(make_box(lo, hi, dim), q, dim);
  for (size_t i = 0; i < pts.size(); ++i)
    for (int k = 0; k < 3; ++k) out[3 * i + k] = pts[i][k];
}
int oracle_face_projection(int q, double* refine, double* coarsen) {
  return guard([&] {
    const FaceProjection fp = face_projection_ops(q);
    copy_mat(fp.refine, refine);
    copy_mat(fp.coarsen, coarsen);
  });
}
int oracle_refinement_interpolant(int p, double* out) {
  return guard([&] { copy_mat(refinement_interpolant(p), out); });
}
int oracle_tree_info(int dim, int L, int p, const double* lo, const double* hi, int* n_nodes, int* n_leaves,
                     long long* total_points, int* leaf_ids, int* node_depth, int* node_parent) {
  return guard([&] {
    const Tree t = build_uniform_tree(make_box(lo, hi, dim), L, dim, p);
    *n_nodes = int(t.nodes.size());
    *n_leaves = t.n_leaves();
    *total_points = t.total_points();
    if (leaf_ids) std::memcpy(leaf_ids, t.leaves.data(), sizeof(int) * t.leaves.size());
    for (size_t i = 0; i < t.nodes.size(); ++i) {
      if (node_depth) node_depth[i] = t.nodes[i].depth;
      if (node_parent) node_parent[i] = t.nodes[i].parent;
    }
  });
}

void* oracle_create(int dim, int p, int L, double lo, double hi, const oracle_term* terms, int n_terms,
                    const oracle_field* source, int literal_sign, int root_implicit, int parallel) {
  Handle* h = nullptr;
  const int rc = guard([&] {
    auto hp = std::make_unique<Handle>();
    Box dom;
    for (int k = 0; k < dim; ++k) dom.lo[k] = lo, dom.hi[k] = hi;
    hp->tree = build_uniform_tree(dom, L, dim, p);
    const int npts = dim == 2 ? p * p : p * p * p;
    std::vector<Term> tv;
    for (int i = 0; i < n_terms; ++i) {
      auto fe = make_field(terms[i].field, dim, npts, hp->tree.n_leaves());
      hp->fields.push_back(fe);
      Term t;
      t.role = Role(terms[i].role);
      t.axis = terms[i].axis;
      t.axis2 = terms[i].axis2;
      t.eval = [fe](const Point& x, int leaf, int pt) { return (*fe)(x, leaf, pt); };
      tv.push_back(t);
    }
    std::function<double(const Point&, int, int)> src;
    if (source) {
      auto fe = make_field(*source, dim, npts, hp->tree.n_leaves());
      hp->fields.push_back(fe);
      src = [fe](const Point& x, int leaf, int pt) { return (*fe)(x, leaf, pt); };
    }
    SolverOptions o;
    o.literal_sign = literal_sign != 0;
    o.root_implicit_S = root_implicit != 0;
    o.parallel = parallel != 0;
    hp->solver = std::make_unique<Solver>(hp->tree, std::move(tv), src, o);
    h = hp.release();
  });
  return rc == 0 ? h : nullptr;
}

void oracle_destroy(void* h) { delete static_cast<Handle*>(h); }

int oracle_build(void* hv) {
  auto* h = static_cast<Handle*>(hv);
  return guard([&] {
    require(h->tree.n_leaves() > 1, "oracle: L >= 1 required");
    h->solver->build();
    h->built = true;
  });
}
int oracle_n_leaves(void* hv) { return static_cast<Handle*>(hv)->tree.n_leaves(); }
int oracle_n_nodes(void* hv) { return int(static_cast<Handle*>(hv)->tree.nodes.size()); }
int oracle_root_bsize(void* hv) {
  auto* h = static_cast<Handle*>(hv);
  const int L = h->tree.max_depth();
  const int q = h->tree.q;
  return h->tree.dim == 2 ? 4 * q * (1 << L) : 6 * q * q * (1 << (2 * L));
}
int oracle_root_points(void* hv, double* xyz) {
  auto* h = static_cast<Handle*>(hv);
  return guard([&] {
    require(h->built, "oracle_root_points: build first");
    const auto pts = h->solver->root_boundary_points();
    for (size_t i = 0; i < pts.size(); ++i)
      for (int k = 0; k < 3; ++k) xyz[3 * i + k] = pts[i][k];
  });
}
int oracle_leaf_points(void* hv, double* xyz) {
  auto* h = static_cast<Handle*>(hv);
  return guard([&] {
    size_t pos = 0;
    for (int id : h->tree.leaves) {
      const auto pts = leaf_cheb_points(h->tree.nodes[id].box, h->tree.p, h->tree.dim);
      for (const auto& x : pts)
        for (int k = 0; k < 3; ++k) xyz[pos++] = x[k];
    }
  });
}
int oracle_discretize(void* hv, int ord, double* lmat, double* f) {
  auto* h = static_cast<Handle*>(hv);
  return guard([&] {
    require(ord >= 0 && ord < h->tree.n_leaves(), "oracle_discretize: bad ordinal");
    Vec fv;
    const Mat l = h->solver->leaf_operator(ord, &fv);
    copy_mat(l, lmat);
    copy_vec(fv, f);
  });
}
int oracle_solve(void* hv, const double* g_root, double* u, double* leaf_g) {
  auto* h = static_cast<Handle*>(hv);
  return guard([&] {
    require(h->built, "oracle_solve: build first");
    const int nb = oracle_root_bsize(hv);
    std::vector<Vec> lg;
    const auto uu = h->solver->solve(Vec(g_root, g_root + nb), leaf_g ? &lg : nullptr);
    size_t pos = 0;
    for (const auto& v : uu) {
      std::memcpy(u + pos, v.data(), sizeof(double) * v.size());
      pos += v.size();
    }
    if (leaf_g) {
      pos = 0;
      for (const auto& v : lg) {
        std::memcpy(leaf_g + pos, v.data(), sizeof(double) * v.size());
        pos += v.size();
      }
    }
  });
}
int oracle_get_leaf(void* hv, int ord, double* Y, double* v, double* T, double* hh) {
  auto* h = static_cast<Handle*>(hv);
  return guard([&] {
    require(h->built && ord >= 0 && ord < h->tree.n_leaves(), "oracle_get_leaf: bad ordinal");
    const LeafSolution& s = h->solver->leaf(ord);
    copy_mat(s.Y, Y);
    copy_vec(s.v, v);
    copy_mat(s.T, T);
    copy_vec(s.h, hh);
  });
}
int oracle_node_sizes(void* hv, int id, int* n_ext, int* n_int) {
  auto* h = static_cast<Handle*>(hv);
  return guard([&] {
    const Artifact& a = h->solver->artifact(id);
    *n_ext = a.n_ext;
    *n_int = a.n_int;
  });
}
int oracle_get_node(void* hv, int id, double* S, double* gtilde, double* T, double* hh) {
  auto* h = static_cast<Handle*>(hv);
  return guard([&] {
    const Artifact& a = h->solver->artifact(id);
    require(a.n_int > 0, "oracle_get_node: node not merged");
    copy_mat(a.S, S);
    copy_vec(a.gtilde, gtilde);
    if (id != 0) {
      copy_mat(h->solver->node_T(id), T);
      copy_vec(h->solver->node_h(id), hh);
    }
  });
}
int oracle_level_nodes(void* hv, int depth, int* ids) {
  auto* h = static_cast<Handle*>(hv);
  if (depth < 0 || depth > h->tree.max_depth()) return -1;
  const auto& lv = h->tree.levels[depth];
  if (ids) std::memcpy(ids, lv.data(), sizeof(int) * lv.size());
  return int(lv.size());
}
double oracle_min_rcond(void* hv) { return static_cast<Handle*>(hv)->solver->min_rcond(); }
void oracle_times(void* hv, double* t_leaf, double* t_merge) {
  auto* h = static_cast<Handle*>(hv);
  *t_leaf = h->solver->t_leaf;
  *t_merge = h->solver->t_merge;
}

}  // extern "C"
