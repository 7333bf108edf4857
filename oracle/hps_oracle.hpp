// hps_oracle.hpp -- TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference HPS hot path (arxiv 2503.17535, reference
// tree /root/reference/proj).  This is the parity CHECKER for the B200 product
// in paper_2503_17535_b200/.  Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load it.  The product
// never links, calls or falls back to it.
//
// Every function cites the reference file:line it restates.  The reference
// itself cannot be compiled here (Eigen3 and vendor/ are absent:
// proj/CMakeLists.txt:13, proj/.gitignore:2), so this is a restatement with a
// small column-major matrix type instead of Eigen, and LAPACK/BLAS (OpenBLAS
// bundled with scipy) in place of Eigen::PartialPivLU and Eigen products.
//
// Parity pinning: the spectral/mesh restatement is pinned by the reference's
// own known-answer tests (proj/tests/test_spectral.cpp, test_mesh.cpp,
// restated in tests/test_oracle_kat.py).  The LU/merge/downward-pass boundary
// has no reference golden vectors (test_local_solve/test_merge/test_solver are
// 4-line stubs), so it is pinned instead by analytic (manufactured) solutions
// and by the monolithic dense collocation system -- see DESIGN.md.
//
// Sign convention: the reference DtN leaf solve sets v_i = -L_ii^-1 f_i
// (proj/src/local_solve.cpp:137,180), i.e. it solves L u = -f.  `literal`
// reproduces that; `corrected` uses +L_ii^-1 f_i.  u_literal(f) == u_corrected(-f).
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace hpso {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
[[noreturn]] inline void fail(const std::string& m) { throw Error(m); }
inline void require(bool ok, const std::string& m) {
  if (!ok) fail(m);
}

using Vec = std::vector<double>;

// Column-major dense matrix (Eigen's default storage, proj/include/hps/core.hpp:17).
struct Mat {
  int r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int rows, int cols) : r(rows), c(cols), a(size_t(rows) * cols, 0.0) {}
  double& operator()(int i, int j) { return a[size_t(j) * r + i]; }
  double operator()(int i, int j) const { return a[size_t(j) * r + i]; }
  double* data() { return a.data(); }
  const double* data() const { return a.data(); }
  bool empty() const { return a.empty(); }
};

struct Point {
  double x[3] = {0, 0, 0};
  double& operator[](int k) { return x[k]; }
  double operator[](int k) const { return x[k]; }
};
struct Box {
  Point lo, hi;
};

// ---- dense kernels (BLAS/LAPACK when available, naive otherwise) ----------
Mat matmul(const Mat& A, const Mat& B);                      // A*B
void gemm(double alpha, const Mat& A, const Mat& B, double beta, Mat& C);
struct LU {
  Mat lu;
  std::vector<int> piv;  // LAPACK 1-based ipiv
  int n = 0;
  void compute(const Mat& A);               // partial pivoting (Eigen PartialPivLU)
  Mat solve(const Mat& B) const;            // A^-1 B
  Vec solve(const Vec& b) const;
};
void set_blas_threads(int n);
int blas_available();

// ---- spectral (proj/src/spectral.cpp) ------------------------------------
Vec cheb_lobatto_1d(int p);
Vec cheb_lobatto_weights(int p);
struct GaussRule {
  Vec nodes, weights;
};
GaussRule gauss_legendre_1d(int q);
Mat cheb_diff_matrix(int p);
Mat barycentric_interp_matrix(const Vec& src, const Vec& dst);
struct IndexSets {
  std::vector<int> interior, exterior;
};
IndexSets leaf_index_sets(int p, int dim);
Mat kron(const Mat& a, const Mat& b);
struct LeafOps {
  int dim = 2, p = 0, q = 0;
  double side = 2.0;
  Mat P, Q;
  IndexSets idx;
};
LeafOps assemble_dtn_ops_2d(int p, int q, double side);
LeafOps assemble_dtn_ops_3d(int p, int q, double side);
struct FaceProjection {
  Mat refine, coarsen;
};
FaceProjection face_projection_ops(int q);
Mat refinement_interpolant(int p);

// ---- mesh (proj/src/mesh.cpp) ---------------------------------------------
extern const int child_offset[8][3];
struct TreeNode {
  Box box;
  int id = -1, parent = -1, depth = 0;
  std::array<int, 8> child{{-1, -1, -1, -1, -1, -1, -1, -1}};
  int n_children = 0;
  std::array<std::int64_t, 3> anchor{{0, 0, 0}};
  bool is_leaf() const { return n_children == 0; }
};
struct Tree {
  int dim = 2, p = 0, q = 0;
  Box domain;
  std::vector<TreeNode> nodes;
  std::vector<int> leaves;
  std::vector<std::vector<int>> levels;
  int n_leaves() const { return int(leaves.size()); }
  long long total_points() const;
  int max_depth() const { return int(levels.size()) - 1; }
  double leaf_side(const TreeNode& n) const {
    return (domain.hi[0] - domain.lo[0]) / double(std::int64_t(1) << n.depth);
  }
  void split(int id);
  void finalize();
};
Tree build_uniform_tree(const Box& domain, int L, int dim, int p);
std::vector<Point> leaf_cheb_points(const Box& box, int p, int dim);
std::vector<Point> leaf_gauss_boundary_points(const Box& box, int q, int dim);

// ---- layout (proj/src/layout.cpp), uniform panels ---------------------------
struct PanelLayout {
  int q = 0, fdim = 1;
  bool split = false;
  std::vector<PanelLayout> sub;
  int panel_pts() const { return fdim == 1 ? q : q * q; }
  int npts() const;
  bool operator==(const PanelLayout& o) const;
  static PanelLayout panel(int q, int fdim) {
    PanelLayout l;
    l.q = q;
    l.fdim = fdim;
    return l;
  }
  static PanelLayout split_of(std::vector<PanelLayout> kids);
};
std::vector<Point> section_points(const Box& box, int dim, int face, const PanelLayout& layout);

// ---- operator terms (proj/include/hps/local_solve.hpp:17-23) ----------------
enum class Role { laplacian = 0, gradient = 1, zeroth = 2, second_order = 3 };
struct Term {
  Role role = Role::laplacian;
  int axis = -1, axis2 = -1;
  // evaluator with access to (leaf ordinal, point index) so sampled fields work
  std::function<double(const Point&, int leaf, int pt)> eval;
};
Mat discretize_operator(const Box& box, int leaf_ord, const std::vector<Term>& terms, int p, int dim);

struct LeafSolution {
  Mat Y, T;
  Vec v, h;
  LU fac;
  double rcond = 1.0;
  bool ill = false;
};
LeafSolution local_solve_dtn(const Mat& lmat, const Vec& f, const LeafOps& ops, bool literal_sign);

// ---- merge (proj/src/merge.cpp) ---------------------------------------------
struct ChildView {
  const Mat* T = nullptr;
  const Vec* h = nullptr;
  const std::vector<PanelLayout>* sections = nullptr;
};
struct FaceMap {
  bool ext = false;
  int offset = 0, src_len = 0, dst_len = 0;
};
struct Artifact {
  int n_ext = 0, n_int = 0;
  bool implicit = false;
  Mat S;       // -D^-1 C
  Vec gtilde;  // -D^-1 h_int
  Vec h_int;
  LU Dfac;
  Mat C;       // kept for implicit apply
  std::vector<std::array<FaceMap, 6>> child_maps;
  std::vector<std::array<int, 7>> child_face_off;
};
struct MergeOut {
  Mat T;
  Vec h;
  std::vector<PanelLayout> sections;
  Artifact art;
};
MergeOut merge_dtn(int dim, const std::vector<ChildView>& ch, bool is_root, bool implicit_S);

// ---- solver (proj/src/solver.cpp) --------------------------------------------
struct SolverOptions {
  bool literal_sign = true;
  bool root_implicit_S = false;
  bool parallel = false;   // OpenMP over leaves / merges in a level ("parallel oracle")
};
class Solver {
 public:
  Solver(const Tree& tree, std::vector<Term> terms,
         std::function<double(const Point&, int leaf, int pt)> source, SolverOptions opts);
  void build();
  void build_leaf(int ord);
  // leaf collocation operator and source samples, exactly as build_leaf forms them
  Mat leaf_operator(int ord, Vec* f) const;
  const LeafOps& ops() const { return ops_; }
  void merge_internal(int id);
  std::vector<Point> root_boundary_points() const;
  std::vector<Vec> solve(const Vec& g_root, std::vector<Vec>* leaf_g = nullptr) const;
  const Tree& tree() const { return *tree_; }
  const LeafSolution& leaf(int ord) const { return leaf_[ord]; }
  const Artifact& artifact(int id) const { return art_[id]; }
  const Mat& node_T(int id) const { return node_T_[id]; }
  const Vec& node_h(int id) const { return node_h_[id]; }
  int top_D_size() const { return art_[0].n_int; }
  double min_rcond() const { return min_rcond_; }
  int leaf_ordinal(int id) const { return leaf_ord_[id]; }
  // per-stage timings of the last build (seconds)
  double t_leaf = 0, t_merge = 0;

 private:
  std::vector<ChildView> child_views(int id) const;
  const Tree* tree_;
  std::vector<Term> terms_;
  std::function<double(const Point&, int, int)> source_;
  SolverOptions opts_;
  LeafOps ops_;
  std::vector<int> leaf_ord_;
  std::vector<LeafSolution> leaf_;
  std::vector<Mat> node_T_;
  std::vector<Vec> node_h_;
  std::vector<std::vector<PanelLayout>> sections_;
  std::vector<Artifact> art_;
  double min_rcond_ = 1.0;
};

}  // namespace hpso
