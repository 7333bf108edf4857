// geometry.hpp -- host-side precompute for the B200 HPS solver (product code).
//
// Everything here is small and computed once per solver on the host, then
// uploaded: the spectral leaf operators (reference: proj/src/spectral.cpp
// cheb_lobatto_1d :14-26, gauss_legendre_1d :51-85, cheb_diff_matrix :87-103,
// barycentric_interp_matrix :105-137, leaf_index_sets :139-160,
// assemble_dtn_ops_2d :260-310, assemble_dtn_ops_3d :370-436), the uniform
// quad/octree in DFS leaf order (proj/src/mesh.cpp:27-121), the index tables of
// the 4->1 / 8->1 merges (proj/src/merge.cpp:20-152, :302-320) and the root
// boundary ordering (proj/src/layout.cpp:89-126).  Matrices are column-major.
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

namespace hpsg {

struct HostMat {
  int r = 0, c = 0;
  std::vector<double> a;
  HostMat() = default;
  HostMat(int rr, int cc) : r(rr), c(cc), a(size_t(rr) * cc, 0.0) {}
  double& operator()(int i, int j) { return a[size_t(j) * r + i]; }
  double operator()(int i, int j) const { return a[size_t(j) * r + i]; }
};

std::vector<double> cheb_nodes(int p);                 // descending from +1
void gauss_rule(int q, std::vector<double>& x, std::vector<double>& w);  // ascending
HostMat cheb_diff(int p);
HostMat bary_interp(const std::vector<double>& src, const std::vector<double>& dst);

struct LeafOperators {
  int dim = 2, p = 0, q = 0;
  int n = 0, ni = 0, ne = 0, nb = 0;  // p^d, (p-2)^d, n-ni, boundary Gauss points
  double side = 0.0;
  std::vector<int> interior, exterior;  // tensor indices, increasing
  HostMat P;   // ne x nb
  HostMat Q;   // nb x n
  HostMat Qi;  // nb x ni  (Q restricted to interior columns)
  HostMat QeP; // nb x nb  (Q restricted to exterior columns, times P)
  HostMat D, D2;  // p x p reference-element first/second derivative
};
LeafOperators make_leaf_operators(int dim, int p, double side);

// 2D: the interior part of Q is separable per side s (geometry.cpp, make_leaf_operators):
//   Qi(s q + i, (i1, i2)) = ds * G(i, m) * d_s(k),  G(i, m) = c2g(i, p-1-(m+1)),  d_s(k) = sgn_s D(fixed_s, k+1)
// with (m, k) = (i1-1, i2-1) on the S/N sides (normal axis 2) and (i2-1, i1-1) on E/W (normal axis 1).
// G: q x (p-2) row-major, d: 4 x (p-2) row-major, ds = 2 / side.  [h|T] = Q_i [v|Y_i] then costs two
// (p-2)-term contractions per boundary point instead of a dense ni-term row.
void q_interior_factors(const LeafOperators& op, std::vector<double>& G, std::vector<double>& d, double& ds);

// A = V diag(lam) V^-1 for a small real matrix with real, distinct eigenvalues (n x n column-major; the
// interior block of the Chebyshev second-derivative matrix for the fast-diagonalisation leaf solve).
// Householder-Hessenberg + Wilkinson-shifted QR for lam, inverse iteration for V, Gauss-Jordan for V^-1.
// Returns false (no decomposition) when an eigenvalue is complex or a residual check fails.
bool real_eigendecomposition(const std::vector<double>& A, int n, std::vector<double>& lam, std::vector<double>& V,
                             std::vector<double>& Vinv);

// Uniform tree of depth L on [lo,hi]^dim.  Node ids follow the reference's
// construction order (breadth-first by level; proj/src/mesh.cpp:113-118); for a
// uniform tree the level order of tree.levels[d] (DFS) coincides with id order,
// and children of level-d node i are level-(d+1) nodes nchild*i + c.
//
// A tree PART (subtree-sharded builds) is the subtree of the full depth-L_full tree
// rooted at node root_index (level order) of depth root_depth, cut at depth root_depth + L:
// part depth d <-> full depth root_depth + d.  cut == false: the part's leaves are real leaves;
// cut == true: they are internal nodes whose [h|T] are inputs.  The full tree is the part
// (0, 0, L_full).
struct UniformTree {
  int dim = 2, p = 0, q = 0, L = 0, nchild = 4, nface = 4;
  double lo = -1, hi = 1;
  int L_full = 0, root_depth = 0;
  long long root_index = 0;
  bool cut = false;
  double rlo[3] = {0, 0, 0}, rhi[3] = {0, 0, 0};  // part root box
  long long level_first_id(int d) const;   // reference id of the first node at part depth d
  long long level_count(int d) const;      // nchild^d
  int face_shift(int d) const { return L_full - 1 - (root_depth + d); }  // child face = q 2^shift sections
  int n_leaves() const { return int(level_count(L)); }
  // leaf lower corners in DFS order (n_leaves x 3) and side length
  std::vector<double> leaf_lo;
  double leaf_side = 0;
};
UniformTree make_uniform_tree(int dim, int p, int L, double lo, double hi);
UniformTree make_part_tree(int dim, int p, int L_full, double lo, double hi, int root_depth, long long root_index,
                           int cut_depth);

// Merge interfaces (proj/src/merge.cpp:20-33): the low child's high face meets the high child's low face.
struct Iface {
  int clo, flo;
  int chi, fhi;
};
const std::vector<Iface>& ifaces(int dim);
// exterior position (quadrant / half of the parent face) of child c's face f, or -1 (merge.cpp:41-56)
int ext_qpos(int dim, int c, int f);
// whether face f of node idx (DFS order) at depth d of a uniform tree lies on the domain boundary
bool face_on_domain_boundary(int dim, int d, long long idx, int f);

// Merge of one level (all nodes at depth d of a uniform tree share it).
// Child boundary layout: faces in reference order, s points per face section.
// Parent exterior: faces in order, each split into nquad child sections
// (qpos order of proj/src/merge.cpp:41-56); interface sections in the order of
// proj/src/merge.cpp:20-33.  All sections hold s points.
struct MergeTables {
  int dim = 2, s = 0, nchild = 4, nface = 4, NI = 4, NE = 8;
  int n_int() const { return NI * s; }
  int n_ext() const { return NE * s; }
  int child_nb() const { return nface * s; }
  // per (child, face): ext section id (>=0) or -(interface id)-1
  std::vector<int> sec;  // nchild*nface
  // gather sources: for each destination block, up to 2 (child, rface, cface);
  // cface == -1 means the outgoing-data (h) column.  Encoded child*64 + rf*8 + (cf+1), -1 = none.
  std::vector<int> md_src;  // NI x (NI + 1 + NE) x 2
  std::vector<int> b_src;   // NE x NI x 2
  std::vector<int> ah_src;  // NE x (1 + NE) x 2
  // downward scatter per (child, face): >=0 : offset into parent g (ext), <0: -(offset into g_int)-1
  std::vector<int> down;    // nchild*nface
};
MergeTables make_merge_tables(int dim, int s);

// ---- ItI (impedance-to-impedance) variant, 2D ------------------------------
// Leaf operators of assemble_iti_ops_2d (proj/src/spectral.cpp:312-368): the 4p-4 boundary walk
// rows G = Ntilde + i eta I_walk, the Gauss interpolation P (walk x 4q) and QH = Q (N - i eta I)
// (4q x p^2).  Complex matrices are held as (re, im) pairs.
struct ItiLeafOperators {
  int p = 0, q = 0, n = 0, ni = 0, nbc = 0, nb = 0;  // p^2, (p-2)^2, 4p-4, 4q
  double eta = 0, side = 0;
  std::vector<int> interior;   // tensor indices, increasing
  HostMat Gr, Gi;              // nbc x n
  HostMat P;                   // nbc x nb
  HostMat QHr, QHi;            // nb x n
};
ItiLeafOperators make_iti_leaf_operators(int p, double eta, double side);

// merge_iti (proj/src/merge.cpp:338-482) as block copies into the REAL-EQUIVALENT merge
// matrices: a complex matrix Z = Zr + i Zi is stored as [[Zr, -Zi], [Zi, Zr]] and a vector as
// [zr; zi], so the DtN LU / GEMM / downward machinery applies unchanged.  Every complex s x s
// block copy becomes the 4 quadrant copies of the child's real-equivalent [h|T].
struct BlockCopy {
  int dst;      // 0: MD = [D | h_int | C], 1: B, 2: AH = [h_ext | A]
  int dr, dc;   // destination offset (real-equivalent rows / columns of that matrix)
  int child;    // source child, or -1: identity block (rows == cols)
  int sr, sc;   // source offset in the child's [h | T] (column 0 = h)
  int rows, cols;
};
struct ItiMergeTables {
  int s = 0;                    // complex points per child face
  int n_int = 0, n_ext = 0;     // real-equivalent sizes (2 x 8s each)
  int child_nb = 0;             // real-equivalent child boundary size (2 x 4s)
  std::vector<BlockCopy> blocks;
  std::vector<int> down;        // 4 children x 8 real-equivalent faces (scatter table of the solve)
};
ItiMergeTables make_iti_merge_tables(int s);

// Root boundary points in the reference's canonical section order
// (HpsSolver::root_boundary_points, proj/src/solver.cpp:159-182).
std::vector<double> root_boundary_points(const UniformTree& t);  // nb_root x 3

// Reference-style problem error string helpers
std::string fmt(const char* f, ...);

}  // namespace hpsg
