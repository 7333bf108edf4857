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
#include <functional>
#include <stdexcept>
#include <string>
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

// proj/include/hps/mesh.hpp:39-61 (uniform trees: build_uniform_tree, mesh.cpp:90-121)
struct DiscretizationTree {
  int dim = 2, p = 0, q = 0, L = 0;
  Box domain;
  long long n_leaves() const { return 1LL << ((dim == 2 ? 2 : 3) * L); }
  long long total_points() const {
    long long per = 1;
    for (int k = 0; k < dim; ++k) per *= p;
    return per * n_leaves();
  }
  int max_depth() const { return L; }
};

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
  t.L = L;
  t.domain = domain;
  return t;
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
};

// proj/include/hps/solver.hpp:30-32
enum class RootBC { dirichlet, radiation };

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
    hpsg_tree t{tree.dim, tree.p, tree.L, tree.domain.lo[0], tree.domain.hi[0]};
    const long long npts = tree.total_points();
    // leaf Chebyshev points, sampled like build_leaf/discretize_operator do on the host
    std::vector<double> xyz(size_t(npts) * 3);
    if (hpsg_tree_leaf_points(&t, xyz.data()) != HPSG_OK) throw Error("hps_b200: invalid tree");
    auto sample = [&](const std::function<Real(const Point&)>& fn) {
      std::vector<double> s(static_cast<size_t>(npts));
      for (long long i = 0; i < npts; ++i) {
        Point x;
        x[0] = xyz[3 * i], x[1] = xyz[3 * i + 1], x[2] = xyz[3 * i + 2];
        s[size_t(i)] = fn(x);
      }
      return s;
    };
    std::vector<hpsg_term> ct;
    for (const CoefficientField& f : terms) {
      samples_.push_back(sample(f.eval));
      hpsg_term tt{};
      tt.role = static_cast<int>(f.role);
      tt.axis = f.axis;
      tt.axis2 = f.axis2;
      tt.field.kind = HPSG_FIELD_SAMPLED;
      ct.push_back(tt);
    }
    for (size_t i = 0; i < ct.size(); ++i) ct[i].field.samples = samples_[i].data();
    hpsg_field src{};
    const hpsg_field* srcp = nullptr;
    if (source) {
      src_samples_ = sample(source);
      src.kind = HPSG_FIELD_SAMPLED;
      src.samples = src_samples_.data();
      srcp = &src;
    }
    hpsg_options o{};
    o.literal_sign = opts.literal_sign ? 1 : 0;
    o.root_implicit_S = opts.root_implicit_S ? 1 : 0;
    o.device = opts.device;
    o.keep_factors = opts.keep_factors ? 1 : 0;
    const int rc = hpsg_create(&t, ct.data(), int(ct.size()), srcp, &o, &ctx_);
    if (rc != HPSG_OK) {
      const std::string msg = ctx_ ? hpsg_last_error(ctx_) : "no CUDA device";
      hpsg_destroy(ctx_);
      ctx_ = nullptr;
      throw Error(msg);
    }
    samples_.clear();  // uploaded
    src_samples_.clear();
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

 private:
  void check(int rc) const {
    if (rc != HPSG_OK) throw Error(hpsg_last_error(ctx_));
  }
  const DiscretizationTree* tree_;
  SolverOptions opts_;
  hpsg_ctx* ctx_ = nullptr;
  std::vector<std::vector<double>> samples_;
  std::vector<double> src_samples_;
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
    hpsg_tree t{tree.dim, tree.p, tree.L, tree.domain.lo[0], tree.domain.hi[0]};
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

}  // namespace b200
}  // namespace hps
