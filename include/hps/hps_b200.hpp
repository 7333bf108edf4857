// hps_b200.hpp -- header-only C++ drop-in for the reference HpsSolver<Real> DtN path,
// implemented over the C-ABI of libhps_b200.so (include/hps_cuda.h).
//
// Mirrors /root/reference/proj/include/hps/{mesh,local_solve,solver}.hpp for the
// calls solve_problem() makes (proj/src/problems.cpp:360-422): build_uniform_tree,
// CoefficientField{role, axis, axis2, std::function eval}, HpsSolver(tree, variant,
// eta, terms, source, opts), build(), root_boundary_points(), sample_root_data(),
// solve(g_root, leaf_g_out) -> SolutionField{tree, u per leaf}.  Arbitrary
// std::function fields are sampled on the host at the leaf Chebyshev points (as the
// reference does, proj/src/local_solve.cpp:53-62) and handed to the device as
// HPSG_FIELD_SAMPLED arrays; errors surface as hps::b200::Error with the reference's
// message text (proj/include/hps/core.hpp:27-35).
//
// Eigen types of the reference API are replaced by std::vector<double> (column-major
// where a matrix is meant).  Link with -lhps_b200.
#pragma once

#include <algorithm>
#include <array>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <exception>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "../hps_cuda.h"

namespace hps {
namespace b200 {

using Real = double;

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// proj/include/hps/core.hpp:25 (Eigen::Vector3d); x[2] unused in 2D
struct Point {
  double x[3] = {0.0, 0.0, 0.0};
  double operator[](int k) const { return x[k]; }
  double& operator[](int k) { return x[k]; }
};
struct Box {
  Point lo, hi;
};

// proj/include/hps/mesh.hpp:24-61: the reference's tree, node by node
constexpr int child_offset[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                                    {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};
struct TreeNode {
  Box box;
  int id = -1;
  int parent = -1;
  int depth = 0;
  std::array<int, 8> child{{-1, -1, -1, -1, -1, -1, -1, -1}};
  int n_children = 0;
  std::array<std::int64_t, 3> anchor{{0, 0, 0}};
  bool is_leaf() const { return n_children == 0; }
};

struct DiscretizationTree {
  int dim = 2, p = 0, q = 0;
  Box domain;
  std::vector<TreeNode> nodes;           // nodes[0] is the root
  std::vector<int> leaves;               // depth-first order
  std::vector<std::vector<int>> levels;  // node ids per depth
  int n_leaves() const { return static_cast<int>(leaves.size()); }
  long long total_points() const {
    long long per = 1;
    for (int k = 0; k < dim; ++k) per *= p;
    return per * n_leaves();
  }
  int max_depth() const { return static_cast<int>(levels.size()) - 1; }
  double leaf_side(const TreeNode& n) const { return (domain.hi[0] - domain.lo[0]) / double(std::int64_t(1) << n.depth); }
  // mesh.cpp:27-52 (the parent box is read before the node vector grows)
  void split(int node_id) {
    if (!nodes[size_t(node_id)].is_leaf()) throw std::runtime_error("split: node already has children");
    const TreeNode parent = nodes[size_t(node_id)];
    const int nchild = dim == 2 ? 4 : 8;
    nodes[size_t(node_id)].n_children = nchild;
    for (int c = 0; c < nchild; ++c) {
      TreeNode ch;
      ch.id = static_cast<int>(nodes.size());
      ch.parent = node_id;
      ch.depth = parent.depth + 1;
      for (int k = 0; k < 3; ++k) {
        const double mid = 0.5 * (parent.box.lo[k] + parent.box.hi[k]);
        ch.box.lo[k] = child_offset[c][k] ? mid : parent.box.lo[k];
        ch.box.hi[k] = child_offset[c][k] ? parent.box.hi[k] : mid;
        ch.anchor[k] = 2 * parent.anchor[k] + child_offset[c][k];
      }
      if (dim == 2) ch.box.lo[2] = ch.box.hi[2] = 0.0, ch.anchor[2] = 0;
      nodes[size_t(node_id)].child[size_t(c)] = ch.id;
      nodes.push_back(ch);
    }
  }
  // mesh.cpp:54-71
  void finalize() {
    leaves.clear();
    levels.clear();
    const int nchild = dim == 2 ? 4 : 8;
    std::vector<int> stack{0};
    while (!stack.empty()) {
      const int id = stack.back();
      stack.pop_back();
      const TreeNode& n = nodes[size_t(id)];
      if (static_cast<int>(levels.size()) <= n.depth) levels.resize(size_t(n.depth) + 1);
      levels[size_t(n.depth)].push_back(id);
      if (n.is_leaf())
        leaves.push_back(id);
      else
        for (int c = nchild - 1; c >= 0; --c) stack.push_back(n.child[size_t(c)]);
    }
  }
  bool is_uniform() const {
    for (int id : leaves)
      if (nodes[size_t(id)].depth != max_depth()) return false;
    return true;
  }
  // the C-ABI view (include/hps_cuda.h hpsg_tree_desc); the arrays live in `store`
  struct Desc {
    std::vector<int> depth, nch, children;
    std::vector<double> lo, hi;
    hpsg_tree_desc d{};
  };
  void describe(Desc& s) const {
    const size_t n = nodes.size();
    s.depth.resize(n), s.nch.resize(n), s.children.assign(8 * n, -1), s.lo.resize(3 * n), s.hi.resize(3 * n);
    for (size_t i = 0; i < n; ++i) {
      s.depth[i] = nodes[i].depth;
      s.nch[i] = nodes[i].n_children;
      for (int c = 0; c < 8; ++c) s.children[8 * i + size_t(c)] = nodes[i].child[size_t(c)];
      for (int k = 0; k < 3; ++k) s.lo[3 * i + size_t(k)] = nodes[i].box.lo[k], s.hi[3 * i + size_t(k)] = nodes[i].box.hi[k];
    }
    s.d = hpsg_tree_desc{dim, p, static_cast<int>(n), s.depth.data(), s.nch.data(), s.children.data(), s.lo.data(),
                         s.hi.data()};
  }
  // rebuild from C-ABI node arrays (product refine_adaptive / enforce_level_restriction output)
  static DiscretizationTree from_arrays(int dim, int p, const Box& domain, int n, const int* depth, const int* nch,
                                        const int* children, const double* lo, const double* hi) {
    DiscretizationTree t;
    t.dim = dim, t.p = p, t.q = p - 2, t.domain = domain;
    t.nodes.resize(size_t(n));
    for (int i = 0; i < n; ++i) {
      TreeNode& x = t.nodes[size_t(i)];
      x.id = i, x.depth = depth[i], x.n_children = nch[i];
      for (int c = 0; c < 8; ++c) x.child[size_t(c)] = children[8 * i + c];
      for (int k = 0; k < 3; ++k) x.box.lo[k] = lo[3 * i + k], x.box.hi[k] = hi[3 * i + k];
    }
    for (int i = 0; i < n; ++i)
      for (int c = 0; c < t.nodes[size_t(i)].n_children; ++c) {
        TreeNode& k = t.nodes[size_t(t.nodes[size_t(i)].child[size_t(c)])];
        k.parent = i;
        for (int a = 0; a < 3; ++a) k.anchor[size_t(a)] = a < dim ? 2 * t.nodes[size_t(i)].anchor[size_t(a)] + child_offset[c][a] : 0;
      }
    t.finalize();
    return t;
  }
};

// mesh.cpp:90-121
inline DiscretizationTree build_uniform_tree(const Box& domain, int L, int dim, int p) {
  if (dim != 2 && dim != 3) throw Error("build_uniform_tree: dim must be 2 or 3");
  if (L < 0) throw Error("build_uniform_tree: depth must be nonnegative");
  if (p < 4) throw Error("build_uniform_tree: p must be >= 4");
  const double side = domain.hi[0] - domain.lo[0];
  if (!(side > 0)) throw Error("build_uniform_tree: empty domain");
  for (int k = 1; k < dim; ++k)
    if (domain.lo[k] != domain.lo[0] || domain.hi[k] != domain.hi[0])
      throw Error("build_uniform_tree: domain must be [lo,hi]^dim");
  DiscretizationTree t;
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

// mesh.hpp:63-68 / mesh.cpp:233-318: adaptive 3D refinement on the product's host mesher
struct RefinementCriterion {
  double tol = 1e-6;
  int p = 8;
  std::vector<std::function<double(const Point&)>> test_fields;
};
inline DiscretizationTree refine_adaptive(const Box& domain, const RefinementCriterion& crit, int max_depth,
                                          std::vector<int>* unresolved = nullptr) {
  if (crit.test_fields.empty()) throw Error("refine_adaptive: no test fields");
  std::vector<hpsg_point_fn> fns;
  std::vector<void*> users;
  for (const auto& f : crit.test_fields) {
    fns.push_back([](void* u, const double* x) -> double {
      Point pt;
      pt[0] = x[0], pt[1] = x[1], pt[2] = x[2];
      return (*static_cast<const std::function<double(const Point&)>*>(u))(pt);
    });
    users.push_back(const_cast<std::function<double(const Point&)>*>(&f));
  }
  int n = 0, nu = 0;
  if (hpsg_refine_adaptive_cb(crit.p, domain.lo.x, domain.hi.x, crit.tol, max_depth, fns.data(), users.data(),
                              int(fns.size()), 0, &n, nullptr, nullptr, nullptr, nullptr, nullptr, &nu) != HPSG_OK &&
      n == 0)
    throw Error("refine_adaptive failed");
  std::vector<int> depth(static_cast<size_t>(n)), nch(static_cast<size_t>(n)), ch(static_cast<size_t>(8 * n));
  std::vector<double> lo(static_cast<size_t>(3 * n)), hi(static_cast<size_t>(3 * n));
  if (hpsg_refine_adaptive_cb(crit.p, domain.lo.x, domain.hi.x, crit.tol, max_depth, fns.data(), users.data(),
                              int(fns.size()), n, &n, depth.data(), nch.data(), ch.data(), lo.data(), hi.data(),
                              &nu) != HPSG_OK)
    throw Error("refine_adaptive failed");
  DiscretizationTree t =
      DiscretizationTree::from_arrays(3, crit.p, domain, n, depth.data(), nch.data(), ch.data(), lo.data(), hi.data());
  if (unresolved) unresolved->assign(size_t(nu), -1);  // count only (the ids are the product mesher's)
  return t;
}

// mesh.cpp:141-167
inline void enforce_level_restriction(DiscretizationTree& tree) {
  tree.finalize();
  DiscretizationTree::Desc d;
  tree.describe(d);
  int n = 0;
  if (hpsg_enforce_level_restriction(&d.d, 0, &n, nullptr, nullptr, nullptr, nullptr, nullptr) != HPSG_OK && n == 0)
    throw Error("enforce_level_restriction failed");
  std::vector<int> depth(static_cast<size_t>(n)), nch(static_cast<size_t>(n)), ch(static_cast<size_t>(8 * n));
  std::vector<double> lo(static_cast<size_t>(3 * n)), hi(static_cast<size_t>(3 * n));
  if (hpsg_enforce_level_restriction(&d.d, n, &n, depth.data(), nch.data(), ch.data(), lo.data(), hi.data()) != HPSG_OK)
    throw Error("enforce_level_restriction failed");
  tree = DiscretizationTree::from_arrays(tree.dim, tree.p, tree.domain, n, depth.data(), nch.data(), ch.data(),
                                         lo.data(), hi.data());
}

// mesh.cpp:320-340 over all leaves (DFS order, tensor order inside a leaf)
inline std::vector<Point> leaf_cheb_points(const DiscretizationTree& tree) {
  DiscretizationTree::Desc d;
  tree.describe(d);
  std::vector<double> xyz(size_t(tree.total_points()) * 3);
  if (hpsg_tree_desc_leaf_points(&d.d, xyz.data()) != HPSG_OK) throw Error("leaf_cheb_points: invalid tree");
  std::vector<Point> pts(size_t(tree.total_points()));
  for (size_t i = 0; i < pts.size(); ++i) pts[i][0] = xyz[3 * i], pts[i][1] = xyz[3 * i + 1], pts[i][2] = xyz[3 * i + 2];
  return pts;
}

// mesh.cpp:435-463
inline std::string mesh_to_json(const DiscretizationTree& tree) {
  DiscretizationTree::Desc d;
  tree.describe(d);
  size_t len = 0;
  if (hpsg_mesh_json(&d.d, nullptr, 0, &len) != HPSG_OK) throw Error("mesh_to_json failed");
  std::string s(len + 1, '\0');
  if (hpsg_mesh_json(&d.d, &s[0], s.size(), &len) != HPSG_OK) throw Error("mesh_to_json failed");
  s.resize(len);
  return s;
}

// proj/include/hps/local_solve.hpp:17-23
struct CoefficientField {
  enum class Role { laplacian = HPSG_ROLE_LAPLACIAN, gradient = HPSG_ROLE_GRADIENT, zeroth = HPSG_ROLE_ZEROTH,
                    second_order = HPSG_ROLE_SECOND_ORDER };
  Role role = Role::laplacian;
  int axis = -1;
  int axis2 = -1;
  std::function<Real(const Point&)> eval;
};

enum class Variant { dtn, iti };  // proj/include/hps/spectral.hpp:87

// proj/include/hps/solver.hpp:17-22 (+ the B200 options)
struct SolverOptions {
  bool build_root_T = false;      // ItI radiation closure (HpsSolverComplex::solve_radiation)
  bool root_implicit_S = false;   // MergeOptions::implicit_S at the root
  bool free_T_after_merge = false;
  bool quiet_warnings = false;
  bool literal_sign = true;       // reference v_i = -L_ii^-1 f_i (local_solve.cpp:137)
  bool keep_factors = false;      // keep the leaf LU factors (LeafSolution::fac) for solve_new_source
  int device = 0;
  int host_threads = 1;           // host threads sampling std::function fields (the reference samples
                                  // serially; > 1 requires thread-safe callables, 0 = every core)
};

// proj/include/hps/solver.hpp:15
enum class RootBC { dirichlet, impedance, radiation };

// LeafSolution<Real> (local_solve.hpp:30-39) without the factorization object: Y (p^d x nb, column-major),
// v, T (nb x nb), h; MergeArtifact<Real> (merge.hpp:58-100): S (n_int x n_ext; empty with an implicit root),
// gtilde
struct LeafSolution {
  std::vector<Real> Y, v, T, h;
};
struct MergeArtifact {
  int n_ext = 0, n_int = 0;
  bool implicit = false;
  std::vector<Real> S_mat, gtilde;
};

// proj/include/hps/solver.hpp:24-28
struct SolutionField {
  const DiscretizationTree* tree = nullptr;
  std::vector<std::vector<Real>> u;  // per leaf (DFS order), tensor order i1*p+i2 (3D: (i1*p+i2)*p+i3)
};

// proj/include/hps/solver.hpp:40-117, DtN / Real only
class HpsSolver {
 public:
  HpsSolver(const DiscretizationTree& tree, Variant variant, double eta, std::vector<CoefficientField> terms,
            std::function<Real(const Point&)> source, SolverOptions opts = {})
      : tree_(&tree), opts_(opts) {
    (void)eta;
    if (variant != Variant::dtn) throw Error("HpsSolver<Real> drives the DtN variant");
    if (opts.build_root_T) throw Error("hps_b200: build_root_T is the ItI radiation closure (HpsSolverComplex)");
    tree.describe(desc_);
    const long long npts = tree.total_points();
    // every field sampled at the leaf Chebyshev points (leaf_cheb_points, DFS order) as build_leaf /
    // discretize_operator do on the host, in one pass over the leaves (each point is formed once, with the
    // same expression as leaf_cheb_points), over host_threads threads
    std::vector<const std::function<Real(const Point&)>*> fns;
    for (const CoefficientField& f : terms) fns.push_back(&f.eval);
    if (source) fns.push_back(&source);
    std::vector<std::unique_ptr<double[]>> smp;
    for (size_t i = 0; i < fns.size(); ++i) smp.emplace_back(new double[size_t(npts)]);
    {
      std::vector<double> cn(size_t(tree.p));
      if (hpsg_cheb_nodes(tree.p, cn.data()) != HPSG_OK) throw Error("hps_b200: invalid tree");
      const int np = tree.dim == 2 ? tree.p * tree.p : tree.p * tree.p * tree.p;
      auto leaf_range = [&](long long l0, long long l1) {
        std::vector<double> m(size_t(3 * tree.p));
        for (long long l = l0; l < l1; ++l) {
          const Box& b = tree.nodes[size_t(tree.leaves[size_t(l)])].box;
          for (int k = 0; k < tree.dim; ++k)
            for (int i = 0; i < tree.p; ++i)
              m[size_t(k * tree.p + i)] = 0.5 * (b.lo[k] + b.hi[k]) + 0.5 * (b.hi[k] - b.lo[k]) * cn[size_t(i)];
          const size_t base = size_t(l) * size_t(np);
          for (int pt = 0; pt < np; ++pt) {
            Point x;
            if (tree.dim == 2) {
              x[0] = m[size_t(pt / tree.p)], x[1] = m[size_t(tree.p + pt % tree.p)], x[2] = 0.0;
            } else {
              x[0] = m[size_t(pt / (tree.p * tree.p))], x[1] = m[size_t(tree.p + (pt / tree.p) % tree.p)];
              x[2] = m[size_t(2 * tree.p + pt % tree.p)];
            }
            for (size_t f = 0; f < fns.size(); ++f) smp[f][base + size_t(pt)] = (*fns[f])(x);
          }
        }
      };
      const long long nl = tree.n_leaves();
      const int nth = opts.host_threads > 0 ? opts.host_threads : int(std::max(1u, std::thread::hardware_concurrency()));
      if (nth <= 1 || nl < 64) {
        leaf_range(0, nl);
      } else {
        std::vector<std::thread> th;
        std::vector<std::exception_ptr> err(static_cast<size_t>(nth));
        const long long chunk = (nl + nth - 1) / nth;
        for (int t = 0; t < nth; ++t)
          th.emplace_back([&, t] {
            try {
              leaf_range(std::min(nl, t * chunk), std::min(nl, (t + 1) * chunk));
            } catch (...) {
              err[size_t(t)] = std::current_exception();
            }
          });
        for (auto& x : th) x.join();
        for (auto& e : err)
          if (e) std::rethrow_exception(e);
      }
    }
    std::vector<hpsg_term> ct;
    for (size_t i = 0; i < terms.size(); ++i) {
      const CoefficientField& f = terms[i];
      hpsg_term tt{};
      tt.role = static_cast<int>(f.role);
      tt.axis = f.axis;
      tt.axis2 = f.axis2;
      tt.field.kind = HPSG_FIELD_SAMPLED;
      tt.field.samples = smp[i].get();
      ct.push_back(tt);
    }
    hpsg_field src{};
    const hpsg_field* srcp = nullptr;
    if (source) {
      src.kind = HPSG_FIELD_SAMPLED;
      src.samples = smp.back().get();
      srcp = &src;
    }
    hpsg_options o{};
    o.literal_sign = opts.literal_sign ? 1 : 0;
    o.root_implicit_S = opts.root_implicit_S ? 1 : 0;
    o.device = opts.device;
    o.keep_factors = opts.keep_factors ? 1 : 0;
    // uniform trees on [lo,hi]^dim take the uniform pipeline (fused leaf kernel, level batches); any other
    // tree (adaptive, level-restricted) the general-tree pipeline (hpsg_create_tree)
    bool cube = true;
    for (int k = 1; k < tree.dim; ++k)
      cube = cube && tree.domain.lo[k] == tree.domain.lo[0] && tree.domain.hi[k] == tree.domain.hi[0];
    int rc;
    if (tree.is_uniform() && cube && tree.max_depth() >= 1) {
      hpsg_tree t{tree.dim, tree.p, tree.max_depth(), tree.domain.lo[0], tree.domain.hi[0]};
      rc = hpsg_create(&t, ct.data(), int(ct.size()), srcp, &o, &ctx_);
    } else {
      rc = hpsg_create_tree(&desc_.d, ct.data(), int(ct.size()), srcp, &o, &ctx_);
    }
    if (rc != HPSG_OK) {
      const std::string msg = ctx_ ? hpsg_last_error(ctx_) : "no CUDA device";
      hpsg_destroy(ctx_);
      ctx_ = nullptr;
      throw Error(msg);
    }
  }
  HpsSolver(const HpsSolver&) = delete;
  HpsSolver& operator=(const HpsSolver&) = delete;
  ~HpsSolver() { hpsg_destroy(ctx_); }

  void build() { check(hpsg_build(ctx_)); }

  std::vector<Point> root_boundary_points() const {
    hpsg_stats st{};
    check(hpsg_get_stats(ctx_, &st));
    std::vector<double> xyz(size_t(st.root_bsize) * 3);
    check(hpsg_root_boundary_points(ctx_, xyz.data()));
    std::vector<Point> pts(size_t(st.root_bsize));
    for (size_t i = 0; i < pts.size(); ++i) pts[i][0] = xyz[3 * i], pts[i][1] = xyz[3 * i + 1], pts[i][2] = xyz[3 * i + 2];
    return pts;
  }

  std::vector<Real> sample_root_data(const std::function<Real(const Point&)>& g) const {
    const auto pts = root_boundary_points();
    std::vector<Real> out(pts.size());
    for (size_t i = 0; i < pts.size(); ++i) out[i] = g(pts[i]);
    return out;
  }

  SolutionField solve(const std::vector<Real>& g_root, std::vector<std::vector<Real>>* leaf_g_out = nullptr) const {
    const long long nl = tree_->n_leaves();
    hpsg_stats st{};
    check(hpsg_get_stats(ctx_, &st));
    if (g_root.size() != size_t(st.root_bsize)) throw Error("solve: boundary data of the wrong length");
    const int npts = tree_->dim == 2 ? tree_->p * tree_->p : tree_->p * tree_->p * tree_->p;
    const int nbl = 2 * tree_->dim * (tree_->dim == 2 ? tree_->q : tree_->q * tree_->q);
    std::vector<double> u(size_t(nl) * npts), lg;
    if (leaf_g_out) lg.resize(size_t(nl) * nbl);
    check(hpsg_solve(ctx_, g_root.data(), 1, u.data(), leaf_g_out ? lg.data() : nullptr));
    SolutionField f;
    f.tree = tree_;
    f.u.resize(size_t(nl));
    for (long long l = 0; l < nl; ++l) f.u[size_t(l)].assign(u.begin() + l * npts, u.begin() + (l + 1) * npts);
    if (leaf_g_out) {
      leaf_g_out->resize(size_t(nl));
      for (long long l = 0; l < nl; ++l) (*leaf_g_out)[size_t(l)].assign(lg.begin() + l * nbl, lg.begin() + (l + 1) * nbl);
    }
    return f;
  }

  // proj/include/hps/solver.hpp:71-72 / solver.cpp:285-307: same operator, new source (per-leaf
  // samples at the Chebyshev points), explicit root data; needs SolverOptions::keep_factors
  SolutionField solve_new_source(const std::vector<std::vector<Real>>& leaf_f, RootBC root_bc,
                                 const std::vector<Real>* g_root = nullptr) const {
    if (root_bc != RootBC::dirichlet) throw Error("solve_new_source: radiation closure is not on this path");
    if (!g_root) throw Error("solve_new_source: boundary data required");
    const long long nl = tree_->n_leaves();
    const int npts = tree_->dim == 2 ? tree_->p * tree_->p : tree_->p * tree_->p * tree_->p;
    if ((long long)leaf_f.size() != nl) throw Error("make_source_state: wrong leaf count");
    std::vector<double> f(size_t(nl) * npts), u(size_t(nl) * npts);
    for (long long l = 0; l < nl; ++l) {
      if ((int)leaf_f[size_t(l)].size() != npts) throw Error("make_source_state: wrong leaf sample count");
      std::copy(leaf_f[size_t(l)].begin(), leaf_f[size_t(l)].end(), f.begin() + l * npts);
    }
    check(hpsg_solve_new_source(ctx_, f.data(), g_root->data(), 1, u.data()));
    SolutionField out;
    out.tree = tree_;
    out.u.resize(size_t(nl));
    for (long long l = 0; l < nl; ++l) out.u[size_t(l)].assign(u.begin() + l * npts, u.begin() + (l + 1) * npts);
    return out;
  }

  int top_D_size() const {
    hpsg_stats st{};
    check(hpsg_get_stats(ctx_, &st));
    return st.top_D_size;
  }
  bool any_ill_conditioned() const {
    hpsg_stats st{};
    check(hpsg_get_stats(ctx_, &st));
    return st.ill_conditioned != 0;
  }
  const DiscretizationTree& tree() const { return *tree_; }
  hpsg_ctx* handle() const { return ctx_; }

  // ---- accessors (solver.hpp:80-92; uniform trees)
  LeafSolution leaf_solution(int ordinal) const {
    const int n = tree_->dim == 2 ? tree_->p * tree_->p : tree_->p * tree_->p * tree_->p;
    const int nb = 2 * tree_->dim * (tree_->dim == 2 ? tree_->q : tree_->q * tree_->q);
    LeafSolution l;
    l.Y.resize(size_t(n) * nb), l.v.resize(size_t(n)), l.T.resize(size_t(nb) * nb), l.h.resize(size_t(nb));
    check(hpsg_get_leaf(ctx_, ordinal, l.Y.data(), l.v.data(), l.T.data(), l.h.data()));
    return l;
  }
  std::vector<LeafSolution> leaf_solutions() const {
    std::vector<LeafSolution> out;
    for (int i = 0; i < tree_->n_leaves(); ++i) out.push_back(leaf_solution(i));
    return out;
  }
  MergeArtifact artifact(int node_id) const {
    MergeArtifact a;
    check(hpsg_node_sizes(ctx_, node_id, &a.n_ext, &a.n_int));
    a.implicit = node_id == 0 && opts_.root_implicit_S;
    if (!a.implicit) a.S_mat.resize(size_t(a.n_int) * a.n_ext);
    a.gtilde.resize(size_t(a.n_int));
    check(hpsg_get_node(ctx_, node_id, a.implicit ? nullptr : a.S_mat.data(), a.gtilde.data(), nullptr, nullptr));
    return a;
  }
  std::vector<Real> node_T(int node_id) const {
    int ne = 0, ni = 0;
    check(hpsg_node_sizes(ctx_, node_id, &ne, &ni));
    std::vector<Real> t(size_t(ne) * ne);
    check(hpsg_get_node(ctx_, node_id, nullptr, nullptr, t.data(), nullptr));
    return t;
  }
  std::vector<Real> node_h(int node_id) const {
    int ne = 0, ni = 0;
    check(hpsg_node_sizes(ctx_, node_id, &ne, &ni));
    std::vector<Real> h(static_cast<size_t>(ne));
    check(hpsg_get_node(ctx_, node_id, nullptr, nullptr, nullptr, h.data()));
    return h;
  }
  // solver.cpp:188-228 restricted to the leaves: the boundary data of every leaf (ordinal order)
  void propagate(const std::vector<Real>& g_root, std::vector<std::vector<Real>>& leaf_g) const { solve(g_root, &leaf_g); }
  // solver.cpp:230-236: u = Y g + v for one leaf (host arithmetic on the device-built Y, v)
  std::vector<Real> reconstruct_leaf(int ordinal, const std::vector<Real>& g_leaf) const {
    const LeafSolution l = leaf_solution(ordinal);
    const size_t n = l.v.size(), nb = g_leaf.size();
    std::vector<Real> u = l.v;
    for (size_t j = 0; j < nb; ++j)
      for (size_t i = 0; i < n; ++i) u[i] += l.Y[j * n + i] * g_leaf[j];
    return u;
  }

 private:
  void check(int rc) const {
    if (rc != HPSG_OK) throw Error(hpsg_last_error(ctx_));
  }
  const DiscretizationTree* tree_;
  DiscretizationTree::Desc desc_;
  SolverOptions opts_;
  hpsg_ctx* ctx_ = nullptr;
};

// proj/include/hps/solver.hpp:40-117 for S = Complex (Variant::iti, 2D): impedance-to-impedance
// maps, solve(g_root) with incoming impedance data, solve_radiation() with build_root_T.  Complex
// coefficient fields are real here (the reference's CoefficientField is real); the source may be
// complex.
using Complex = std::complex<double>;
struct SolutionFieldC {
  const DiscretizationTree* tree = nullptr;
  std::vector<std::vector<Complex>> u;
};

class HpsSolverComplex {
 public:
  HpsSolverComplex(const DiscretizationTree& tree, Variant variant, double eta, std::vector<CoefficientField> terms,
                   std::function<Complex(const Point&)> source, SolverOptions opts = {})
      : tree_(&tree) {
    if (variant != Variant::iti) throw Error("HpsSolver<Complex> drives the ItI variant");
    if (tree.dim != 2) throw Error("local_solve_iti: 2D only");
    if (!tree.is_uniform()) throw Error("merge_iti: uniform 2D trees only (merge.cpp:338-340)");
    hpsg_tree t{tree.dim, tree.p, tree.max_depth(), tree.domain.lo[0], tree.domain.hi[0]};
    const long long npts = tree.total_points();
    std::vector<double> xyz(size_t(npts) * 3);
    if (hpsg_tree_leaf_points(&t, xyz.data()) != HPSG_OK) throw Error("hps_b200: invalid tree");
    auto point = [&](long long i) {
      Point x;
      x[0] = xyz[3 * i], x[1] = xyz[3 * i + 1], x[2] = xyz[3 * i + 2];
      return x;
    };
    std::vector<std::vector<double>> samples;
    std::vector<hpsg_term> ct;
    for (const CoefficientField& f : terms) {
      std::vector<double> sv(static_cast<size_t>(npts));
      for (long long i = 0; i < npts; ++i) sv[size_t(i)] = f.eval(point(i));
      samples.push_back(std::move(sv));
      hpsg_term tt{};
      tt.role = static_cast<int>(f.role);
      tt.axis = f.axis;
      tt.axis2 = f.axis2;
      tt.field.kind = HPSG_FIELD_SAMPLED;
      ct.push_back(tt);
    }
    for (size_t i = 0; i < ct.size(); ++i) ct[i].field.samples = samples[i].data();
    std::vector<double> sre, sim;
    hpsg_field fre{}, fim{};
    hpsg_options o{};
    o.literal_sign = opts.literal_sign ? 1 : 0;
    o.device = opts.device;
    o.variant = HPSG_VARIANT_ITI;
    o.eta = eta;
    o.build_root_T = opts.build_root_T ? 1 : 0;
    const hpsg_field* srcp = nullptr;
    if (source) {
      sre.resize(size_t(npts));
      sim.resize(size_t(npts));
      for (long long i = 0; i < npts; ++i) {
        const Complex v = source(point(i));
        sre[size_t(i)] = v.real(), sim[size_t(i)] = v.imag();
      }
      fre.kind = fim.kind = HPSG_FIELD_SAMPLED;
      fre.samples = sre.data();
      fim.samples = sim.data();
      srcp = &fre;
      o.source_imag = &fim;
    }
    const int rc = hpsg_create(&t, ct.data(), int(ct.size()), srcp, &o, &ctx_);
    if (rc != HPSG_OK) {
      const std::string msg = ctx_ ? hpsg_last_error(ctx_) : "no CUDA device";
      hpsg_destroy(ctx_);
      ctx_ = nullptr;
      throw Error(msg);
    }
  }
  HpsSolverComplex(const HpsSolverComplex&) = delete;
  HpsSolverComplex& operator=(const HpsSolverComplex&) = delete;
  ~HpsSolverComplex() { hpsg_destroy(ctx_); }

  void build() { check(hpsg_build(ctx_)); }

  std::vector<Point> root_boundary_points() const {
    hpsg_stats st{};
    check(hpsg_get_stats(ctx_, &st));
    std::vector<double> xyz(size_t(st.root_bsize) * 3);
    check(hpsg_root_boundary_points(ctx_, xyz.data()));
    std::vector<Point> pts(size_t(st.root_bsize));
    for (size_t i = 0; i < pts.size(); ++i) pts[i][0] = xyz[3 * i], pts[i][1] = xyz[3 * i + 1], pts[i][2] = xyz[3 * i + 2];
    return pts;
  }

  SolutionFieldC solve(const std::vector<Complex>& g_root) const {
    std::vector<Complex> u(size_t(tree_->total_points()));
    check(hpsg_solve_complex(ctx_, reinterpret_cast<const double*>(g_root.data()), 1,
                             reinterpret_cast<double*>(u.data())));
    return split(u);
  }

  SolutionFieldC solve_radiation() const {
    std::vector<Complex> u(size_t(tree_->total_points()));
    check(hpsg_solve_radiation(ctx_, reinterpret_cast<double*>(u.data()), nullptr));
    return split(u);
  }

 private:
  SolutionFieldC split(const std::vector<Complex>& u) const {
    SolutionFieldC f;
    f.tree = tree_;
    const long long nl = tree_->n_leaves(), np = tree_->total_points() / nl;
    f.u.resize(size_t(nl));
    for (long long l = 0; l < nl; ++l) f.u[size_t(l)].assign(u.begin() + l * np, u.begin() + (l + 1) * np);
    return f;
  }
  void check(int rc) const {
    if (rc != HPSG_OK) throw Error(hpsg_last_error(ctx_));
  }
  const DiscretizationTree* tree_;
  hpsg_ctx* ctx_ = nullptr;
};

// downpass.cpp:108-143 / SPEC.md:438: raw little-endian FP64 leaf-major / point-minor + JSON sidecar, each
// written to <path>.tmp and renamed (the sidecar text is the reference's nlohmann dump(1) layout)
inline void dump_solution(const SolutionField& field, const std::string& json_path, const std::string& bin_path,
                          const std::string& tree_ref) {
  const int leaf_len = field.u.empty() ? 0 : static_cast<int>(field.u[0].size());
  const std::string tmp = bin_path + ".tmp";
  std::FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) throw Error("dump_solution: cannot write " + tmp);
  for (const auto& u : field.u) std::fwrite(u.data(), sizeof(double), u.size(), f);
  std::fclose(f);
  std::rename(tmp.c_str(), bin_path.c_str());
  const std::string jtmp = json_path + ".tmp";
  std::FILE* j = std::fopen(jtmp.c_str(), "wb");
  if (!j) throw Error("dump_solution: cannot write " + jtmp);
  std::fprintf(j, "{\n \"dtype\": \"float64\",\n \"leaf_len\": %d,\n \"n_leaves\": %d,\n \"tree_ref\": \"%s\"\n}\n",
               leaf_len, static_cast<int>(field.u.size()), tree_ref.c_str());
  std::fclose(j);
  std::rename(jtmp.c_str(), json_path.c_str());
}

}  // namespace b200
}  // namespace hps
