// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY: extern "C" wrapper over the reference's own public API.
//
// Linked with the unmodified reference sources (oracle/Makefile.ref) into oracle/_ref/libhps_ref.so.
// Nothing here re-implements an HPS stage: every number comes out of hps::HpsSolver / hps::solve_problem
// (/root/reference/proj/src/solver.cpp, problems.cpp).  The only local logic is argument marshalling and
// the closed-form fields of the oracle_field descriptors (field_eval.hpp), handed to the reference as
// std::function closures exactly as a reference user would.
#include "ref_capi.h"

#include <chrono>
#include <complex>
#include <cstring>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "field_eval.hpp"
#include "hps/problems.hpp"
#include "hps/solver.hpp"

namespace {

using hps::Complex;
using hps::Real;
using hpso_fields::FieldEval;

thread_local std::string g_err;

template <class F>
int guard(F&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct RefHandle {
  std::shared_ptr<hps::DiscretizationTree> tree;
  std::unique_ptr<hps::HpsSolver<Real>> sr;
  std::unique_ptr<hps::HpsSolver<Complex>> sc;
  std::optional<hps::ProblemSpec> prob;
  std::vector<std::shared_ptr<FieldEval>> fields;
  double t_build = 0.0, t_solve = 0.0;
  int n_unresolved = 0;
  bool built = false;

  bool cplx() const { return sc != nullptr; }
  int npts_leaf() const { return tree->dim == 2 ? tree->p * tree->p : tree->p * tree->p * tree->p; }
};

RefHandle* H(void* h) {
  if (!h) throw std::runtime_error("ref: null handle");
  return static_cast<RefHandle*>(h);
}

std::shared_ptr<FieldEval> make_field(const oracle_field& f, int dim) {
  if (f.kind == ORACLE_FIELD_SAMPLED)
    throw std::runtime_error("ref: sampled fields are not supported (the reference takes point functions)");
  auto fe = std::make_shared<FieldEval>();
  fe->f = f;
  fe->dim = dim;
  if (f.n_centers > 0) fe->centers.assign(f.centers, f.centers + 3 * f.n_centers);
  fe->f.centers = nullptr;
  fe->f.samples = nullptr;
  return fe;
}

template <class S>
hps::Vec<S> vec_from(const double* p, int n) {
  hps::Vec<S> v(n);
  std::memcpy(v.data(), p, sizeof(S) * n);
  return v;
}
template <class M>
void copy_out(const M& m, double* out) {
  if (out && m.size()) std::memcpy(out, m.data(), sizeof(typename M::Scalar) * m.size());
}

template <class S>
void solve_into(RefHandle* r, const hps::HpsSolver<S>& s, const double* g_root, double* u, double* leaf_g) {
  const int nb = hps::node_boundary_size(*r->tree, 0);
  const hps::Vec<S> g = vec_from<S>(g_root, nb);
  std::vector<hps::Vec<S>> lg;
  const double t0 = now_s();
  const hps::SolutionField<S> field = s.solve(g, leaf_g ? &lg : nullptr);
  r->t_solve = now_s() - t0;
  const int n = r->npts_leaf();
  for (int i = 0; i < r->tree->n_leaves(); ++i) std::memcpy(u + size_t(i) * n * sizeof(S) / 8, field.u[i].data(), sizeof(S) * n);
  if (leaf_g) {
    size_t off = 0;
    for (const auto& v : lg) {
      std::memcpy(leaf_g + off, v.data(), sizeof(S) * v.size());
      off += v.size() * sizeof(S) / 8;
    }
  }
}

template <class S>
hps::SolutionField<S> field_from(RefHandle* r, const double* u) {
  hps::SolutionField<S> f;
  f.tree = r->tree.get();
  const int n = r->npts_leaf();
  f.u.resize(r->tree->n_leaves());
  for (int i = 0; i < r->tree->n_leaves(); ++i) f.u[i] = vec_from<S>(u + size_t(i) * n * sizeof(S) / 8, n);
  return f;
}

template <class S>
void get_leaf(const hps::HpsSolver<S>& s, int ord, double* Y, double* v, double* T, double* hh) {
  const auto& ls = s.leaf_solutions().at(ord);
  copy_out(ls.Y, Y);
  copy_out(ls.v, v);
  copy_out(ls.T, T);
  copy_out(ls.h, hh);
}

template <class S>
void get_node(const hps::HpsSolver<S>& s, int id, double* S_out, double* gt, double* T, double* hh) {
  const auto& art = s.artifact(id);
  copy_out(art.S_mat, S_out);
  copy_out(art.gtilde, gt);
  if (id == 0) {
    copy_out(s.root_T(), T);
    copy_out(s.root_h(), hh);
  } else {
    copy_out(s.node_T(id), T);
    copy_out(s.node_h(id), hh);
  }
}

void make_solver(RefHandle* r, hps::Variant var, double eta, std::vector<hps::CoefficientField> terms,
                 std::function<Complex(const hps::Point&)> src, hps::SolverOptions opts) {
  if (var == hps::Variant::iti)
    r->sc = std::make_unique<hps::HpsSolver<Complex>>(*r->tree, var, eta, std::move(terms), std::move(src), opts);
  else
    r->sr = std::make_unique<hps::HpsSolver<Real>>(*r->tree, var, eta, std::move(terms), std::move(src), opts);
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void ref_set_threads(int n) {
  auto& b = Eigen::shim::blas();
  if (b.ok && b.set_threads) b.set_threads(n);
}

void* ref_create(int dim, int p, int L, double lo, double hi, const oracle_term* terms, int n_terms,
                 const oracle_field* source, const oracle_field* source_imag, int variant, double eta,
                 int root_implicit, int build_root_T) {
  auto r = std::make_unique<RefHandle>();
  const int rc = guard([&] {
    hps::Box dom;
    dom.lo = hps::Point(lo, lo, dim == 3 ? lo : 0.0);
    dom.hi = hps::Point(hi, hi, dim == 3 ? hi : 0.0);
    r->tree = std::make_shared<hps::DiscretizationTree>(hps::build_uniform_tree(dom, L, dim, p));
    std::vector<hps::CoefficientField> cf;
    for (int i = 0; i < n_terms; ++i) {
      auto fe = make_field(terms[i].field, dim);
      r->fields.push_back(fe);
      hps::CoefficientField t;
      t.role = static_cast<hps::CoefficientField::Role>(terms[i].role);
      t.axis = terms[i].axis;
      t.axis2 = terms[i].axis2;
      t.eval = [fe](const hps::Point& x) { return (*fe)(x, 0, 0); };
      cf.push_back(std::move(t));
    }
    std::function<Complex(const hps::Point&)> src;
    if (source) {
      auto re = make_field(*source, dim);
      std::shared_ptr<FieldEval> im = source_imag ? make_field(*source_imag, dim) : nullptr;
      src = [re, im](const hps::Point& x) { return Complex((*re)(x, 0, 0), im ? (*im)(x, 0, 0) : 0.0); };
    }
    hps::SolverOptions opts;
    opts.root_implicit_S = root_implicit != 0;
    opts.build_root_T = build_root_T != 0;
    opts.quiet_warnings = true;
    make_solver(r.get(), variant ? hps::Variant::iti : hps::Variant::dtn, eta, std::move(cf), std::move(src), opts);
  });
  return rc == 0 ? r.release() : nullptr;
}

void* ref_create_problem(const char* name, double k, unsigned seed, int p, int adaptive, int L, double tol,
                         int max_depth, int keep_T) {
  auto r = std::make_unique<RefHandle>();
  const int rc = guard([&] {
    r->prob = hps::problem_by_name(name, k, seed);
    const hps::ProblemSpec& prob = *r->prob;
    // tree and options exactly as solve_problem (problems.cpp:365-388)
    if (adaptive) {
      hps::RefinementCriterion crit;
      crit.tol = tol;
      crit.p = p;
      crit.test_fields = prob.refinement_fields;
      std::vector<int> unresolved;
      r->tree = std::make_shared<hps::DiscretizationTree>(
          hps::refine_adaptive(prob.domain, crit, max_depth, &unresolved));
      r->n_unresolved = static_cast<int>(unresolved.size());
    } else {
      r->tree = std::make_shared<hps::DiscretizationTree>(hps::build_uniform_tree(prob.domain, L, prob.dim, p));
    }
    hps::SolverOptions opts;
    opts.quiet_warnings = true;
    if (prob.dim == 3) {
      opts.root_implicit_S = true;
      opts.free_T_after_merge = keep_T == 0;
    }
    if (prob.root_bc == hps::RootBC::radiation) opts.build_root_T = true;
    make_solver(r.get(), prob.variant, prob.eta, prob.terms, prob.source, opts);
  });
  return rc == 0 ? r.release() : nullptr;
}

void ref_destroy(void* h) { delete static_cast<RefHandle*>(h); }

int ref_build(void* h) {
  return guard([&] {
    RefHandle* r = H(h);
    const double t0 = now_s();
    if (r->cplx())
      r->sc->build();
    else
      r->sr->build();
    r->t_build = now_s() - t0;
    r->built = true;
  });
}

int ref_is_complex(void* h) { return H(h)->cplx() ? 1 : 0; }
int ref_n_leaves(void* h) { return H(h)->tree->n_leaves(); }
int ref_n_nodes(void* h) { return static_cast<int>(H(h)->tree->nodes.size()); }
int ref_dim(void* h) { return H(h)->tree->dim; }
int ref_p(void* h) { return H(h)->tree->p; }
int ref_root_bsize(void* h) { return hps::node_boundary_size(*H(h)->tree, 0); }
int ref_top_D_size(void* h) { return hps::top_merge_D_size(*H(h)->tree); }
int ref_n_unresolved(void* h) { return H(h)->n_unresolved; }

int ref_tree(void* h, int* depth, int* parent, int* n_children, int* children, double* lo, double* hi,
             long long* anchor, int* leaves) {
  return guard([&] {
    const auto& t = *H(h)->tree;
    for (size_t i = 0; i < t.nodes.size(); ++i) {
      const auto& n = t.nodes[i];
      if (depth) depth[i] = n.depth;
      if (parent) parent[i] = n.parent;
      if (n_children) n_children[i] = n.n_children;
      for (int c = 0; c < 8; ++c)
        if (children) children[8 * i + c] = n.child[c];
      for (int k = 0; k < 3; ++k) {
        if (lo) lo[3 * i + k] = n.box.lo[k];
        if (hi) hi[3 * i + k] = n.box.hi[k];
        if (anchor) anchor[3 * i + k] = n.anchor[k];
      }
    }
    if (leaves)
      for (int i = 0; i < t.n_leaves(); ++i) leaves[i] = t.leaves[i];
  });
}

int ref_root_points(void* h, double* xyz) {
  return guard([&] {
    RefHandle* r = H(h);
    const auto pts = r->cplx() ? r->sc->root_boundary_points() : r->sr->root_boundary_points();
    for (size_t i = 0; i < pts.size(); ++i)
      for (int k = 0; k < 3; ++k) xyz[3 * i + k] = pts[i][k];
  });
}

int ref_leaf_points(void* h, double* xyz) {
  return guard([&] {
    const auto& t = *H(h)->tree;
    size_t o = 0;
    for (int id : t.leaves)
      for (const auto& x : hps::leaf_cheb_points(t, t.nodes[id]))
        for (int k = 0; k < 3; ++k) xyz[o++] = x[k];
  });
}

int ref_sample_root_data(void* h, double* g) {
  return guard([&] {
    RefHandle* r = H(h);
    if (!r->prob) throw std::runtime_error("ref_sample_root_data: not a problem handle");
    if (r->cplx())
      copy_out(hps::sample_boundary_data(*r->sc, *r->prob), g);
    else
      copy_out(hps::sample_boundary_data(*r->sr, *r->prob), g);
  });
}

int ref_solve(void* h, const double* g_root, double* u, double* leaf_g) {
  return guard([&] {
    RefHandle* r = H(h);
    if (r->cplx())
      solve_into(r, *r->sc, g_root, u, leaf_g);
    else
      solve_into(r, *r->sr, g_root, u, leaf_g);
  });
}

int ref_solve_radiation(void* h, double* u) {
  return guard([&] {
    RefHandle* r = H(h);
    if (!r->cplx()) throw std::runtime_error("ref_solve_radiation: ItI handles only");
    const double t0 = now_s();
    const auto field = r->sc->solve_radiation();
    r->t_solve = now_s() - t0;
    const int n = r->npts_leaf();
    for (int i = 0; i < r->tree->n_leaves(); ++i) std::memcpy(u + size_t(i) * 2 * n, field.u[i].data(), 16 * n);
  });
}

int ref_solve_new_source(void* h, const double* leaf_f, int radiation, const double* g_root, double* u) {
  return guard([&] {
    RefHandle* r = H(h);
    const int n = r->npts_leaf(), nl = r->tree->n_leaves(), nb = hps::node_boundary_size(*r->tree, 0);
    auto run = [&](auto& s, auto tag) {
      using S = decltype(tag);
      std::vector<hps::Vec<S>> f(nl);
      for (int i = 0; i < nl; ++i) f[i] = vec_from<S>(leaf_f + size_t(i) * n * sizeof(S) / 8, n);
      std::optional<hps::Vec<S>> g;
      if (g_root) g = vec_from<S>(g_root, nb);
      const double t0 = now_s();
      const auto field =
          s.solve_new_source(f, radiation ? hps::RootBC::radiation : hps::RootBC::dirichlet, g ? &*g : nullptr);
      r->t_solve = now_s() - t0;
      for (int i = 0; i < nl; ++i) std::memcpy(u + size_t(i) * n * sizeof(S) / 8, field.u[i].data(), sizeof(S) * n);
    };
    if (r->cplx())
      run(*r->sc, Complex());
    else
      run(*r->sr, Real());
  });
}

int ref_get_leaf(void* h, int ord, double* Y, double* v, double* T, double* hh) {
  return guard([&] {
    RefHandle* r = H(h);
    if (r->cplx())
      get_leaf(*r->sc, ord, Y, v, T, hh);
    else
      get_leaf(*r->sr, ord, Y, v, T, hh);
  });
}

int ref_node_sizes(void* h, int id, int* n_ext, int* n_int) {
  return guard([&] {
    RefHandle* r = H(h);
    const int ne = r->cplx() ? r->sc->artifact(id).n_ext : r->sr->artifact(id).n_ext;
    const int ni = r->cplx() ? r->sc->artifact(id).n_int : r->sr->artifact(id).n_int;
    *n_ext = ne;
    *n_int = ni;
  });
}

int ref_get_node(void* h, int id, double* S, double* gtilde, double* T, double* hh) {
  return guard([&] {
    RefHandle* r = H(h);
    if (r->cplx())
      get_node(*r->sc, id, S, gtilde, T, hh);
    else
      get_node(*r->sr, id, S, gtilde, T, hh);
  });
}

int ref_error_report(void* h, const double* u, double* rel_linf, double* rel_l2) {
  return guard([&] {
    RefHandle* r = H(h);
    if (!r->prob || !r->prob->has_exact) throw std::runtime_error("ref_error_report: no exact solution");
    const hps::ErrorReport e = r->cplx() ? hps::error_report(field_from<Complex>(r, u), r->prob->exact)
                                         : hps::error_report(field_from<Real>(r, u), r->prob->exact);
    *rel_linf = e.rel_linf;
    *rel_l2 = e.rel_l2;
  });
}

double ref_min_rcond(void* h) {
  RefHandle* r = H(h);
  double m = 1.0;
  if (r->cplx())
    for (const auto& l : r->sc->leaf_solutions()) m = std::min(m, l.rcond);
  else
    for (const auto& l : r->sr->leaf_solutions()) m = std::min(m, l.rcond);
  return m;
}

int ref_any_ill_conditioned(void* h) {
  RefHandle* r = H(h);
  return (r->cplx() ? r->sc->any_ill_conditioned() : r->sr->any_ill_conditioned()) ? 1 : 0;
}

void ref_times(void* h, double* t_build_s, double* t_solve_s) {
  RefHandle* r = H(h);
  if (t_build_s) *t_build_s = r->t_build;
  if (t_solve_s) *t_solve_s = r->t_solve;
}

int ref_solve_problem(const char* name, double k, unsigned seed, int p, int adaptive, int L, double tol,
                      int max_depth, double* out) {
  return guard([&] {
    hps::Discretization disc;
    disc.p = p;
    disc.adaptive = adaptive != 0;
    disc.L = L;
    disc.tol = tol;
    disc.max_depth = max_depth;
    hps::SolverOptions opts;
    opts.quiet_warnings = true;
    const hps::SolveRun run = hps::solve_problem(hps::problem_by_name(name, k, seed), disc, opts);
    const hps::SolveReport& rep = run.report;
    const double v[8] = {rep.err.rel_linf, rep.err.rel_l2, double(rep.n_leaves), double(rep.N),
                         double(rep.top_D_size), double(rep.tree_depth), rep.t_build_s, rep.t_solve_s};
    std::memcpy(out, v, sizeof v);
  });
}

long long ref_mesh_json(void* h, char* buf, long long cap) {
  long long n = -1;
  guard([&] {
    const std::string s = hps::mesh_to_json(*H(h)->tree);
    n = (long long)s.size();
    if (buf && cap > n) std::memcpy(buf, s.c_str(), s.size() + 1);
  });
  return n;
}

int ref_dump_solution(void* h, const double* u, const char* json_path, const char* bin_path, const char* tree_ref) {
  return guard([&] {
    RefHandle* r = H(h);
    if (r->cplx())
      hps::dump_solution(field_from<Complex>(r, u), json_path, bin_path, tree_ref);
    else
      hps::dump_solution(field_from<Real>(r, u), json_path, bin_path, tree_ref);
  });
}

int ref_bench_sample(int p, int L, int m, double lo, double hi, const oracle_term* terms, int n_terms,
                     const oracle_field* source, int root_implicit, double* out) {
  return guard([&] {
    if (m < 1 || m > L) throw std::runtime_error("ref_bench_sample: need 1 <= m <= L");
    const int top = L - m;  // depths 0 .. top-1 are sampled one node each
    // (1) one depth-`top` subtree, end to end, by the reference solver
    const double side = (hi - lo) / double(1 << top);
    void* sub = ref_create(2, p, m, lo, lo + side, terms, n_terms, source, nullptr, 0, 1.0, 0, 0);
    if (!sub) throw std::runtime_error(g_err);
    std::unique_ptr<RefHandle> hs(static_cast<RefHandle*>(sub));
    double t0 = now_s();
    hs->sr->build();
    const double t_build = now_s() - t0;
    const int nb = hps::node_boundary_size(*hs->tree, 0);
    hps::VecR g = hps::VecR::Zero(nb);
    for (int i = 0; i < nb; ++i) g[i] = std::sin(0.37 * i);
    t0 = now_s();
    const auto field = hs->sr->solve(g);
    const double t_solve = now_s() - t0;
    double est = std::pow(4.0, top) * (t_build + t_solve);
    out[1] = t_build;
    out[2] = t_solve;
    out[3] = hs->tree->n_leaves();
    // (2) one merge + propagate per top depth, children of the true size
    hps::Box dom;
    dom.lo = hps::Point(lo, lo, 0.0);
    dom.hi = hps::Point(hi, hi, 0.0);
    const hps::DiscretizationTree full = hps::build_uniform_tree(dom, L, 2, p);
    for (int d = top - 1; d >= 0; --d) {
      const int nid = full.levels[d][0];
      const hps::TreeNode& node = full.nodes[nid];
      std::vector<std::vector<hps::PanelLayout>> secs(4);
      std::vector<hps::MatR> T(4);
      std::vector<hps::VecR> h(4);
      std::vector<hps::ChildView<Real>> views(4);
      for (int c = 0; c < 4; ++c) {
        const int cid = node.child[c];
        for (int f = 0; f < 4; ++f) secs[c].push_back(hps::node_section_layout(full, cid, f));
        const int n = hps::node_boundary_size(full, cid);
        T[c] = hps::MatR(n, n);
        h[c] = hps::VecR(n);
        for (int j = 0; j < n; ++j) {
          h[c][j] = std::cos(0.11 * j + c);
          for (int i = 0; i < n; ++i) T[c](i, j) = std::sin(1.7 * i + 0.3 * j + c) + (i == j ? 4.0 : 0.0);
        }
        views[c].T = &T[c];
        views[c].h = &h[c];
        views[c].sections = &secs[c];
        views[c].node_id = cid;
      }
      hps::MergeOptions mo;
      mo.is_root = d == 0;
      mo.implicit_S = d == 0 && root_implicit;
      t0 = now_s();
      hps::MergeOutput<Real> mout = hps::merge_node<Real>(2, hps::Variant::dtn, views, nullptr, mo);
      const double t_merge = now_s() - t0;
      // the propagate step of this node (solver.cpp:199-212): g_int, then the scatter into the children
      const hps::MergeArtifact<Real>& art = mout.art;
      hps::VecR gj = hps::VecR::Zero(art.n_ext);
      for (int i = 0; i < art.n_ext; ++i) gj[i] = std::sin(0.21 * i);
      t0 = now_s();
      hps::VecR g_int = art.implicit ? hps::VecR(art.gtilde - art.apply_Dinv(hps::artifact_apply_C(art, views, gj)))
                                     : hps::VecR(art.S_mat * gj + art.gtilde);
      std::vector<hps::VecR> gc(4);
      for (int c = 0; c < 4; ++c) {
        const auto& offs = art.child_face_off[c];
        gc[c].resize(offs[4]);
        for (int f = 0; f < 4; ++f) {
          const auto& mp = art.child_maps[c][f];
          gc[c].segment(offs[f], mp.dst_len) =
              mp.ext ? gj.segment(mp.offset, mp.src_len).eval() : g_int.segment(mp.offset, mp.src_len).eval();
        }
      }
      const double t_prop = now_s() - t0;
      out[4 + 2 * d] = t_merge;
      out[5 + 2 * d] = t_prop;
      est += std::pow(4.0, d) * (t_merge + t_prop);
    }
    out[0] = est;
  });
}

}  // extern "C"
