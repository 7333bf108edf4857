// tree_general.hpp -- host-side planning of HPS on a GENERAL (adaptive, level-restricted) tree: the
// reference's DiscretizationTree (proj/include/hps/mesh.hpp:28-61) as handed through hpsg_create_tree.
//
// Reference pieces restated here (host precompute, product code):
//   PanelLayout / layout_meet / layout_transfer / section_points  (proj/src/layout.cpp:10-126)
//   face_projection_ops                                          (proj/src/spectral.cpp:454-483)
//   node_section_layout / merge_interior_size                    (proj/src/merge.cpp:751-774)
//   MergeGeom + row_tr / col_tr + child_maps of merge_dtn        (proj/src/merge.cpp:90-152, 183-324)
//
// Device formulation (general.cu): a nonuniform merge projects each child whose interface face is finer
// than the interface ("meet") layout first -- [h|T]' = R [h|T] diag(1, E) with the block-diagonal face
// transfers R (rows) and E (columns) -- after which the merge is the matched-layout merge of the uniform
// path on child faces of unequal sizes.  That is exactly merge_dtn's per-block R * T_blk * E
// (merge.cpp:264-266) and its h_int += R h (:238-243).  Nodes of one depth whose children have identical
// face layouts share every table and size and are merged as one strided batch ("group").
#pragma once

#include <array>
#include <string>
#include <vector>

#include "geometry.hpp"

namespace hpsg {

struct Layout {  // PanelLayout (proj/include/hps/layout.hpp:17-35)
  int q = 0, fdim = 1;
  bool split = false;
  std::vector<Layout> sub;
  int panel_pts() const { return fdim == 1 ? q : q * q; }
  int npts() const;
  int max_level() const;
  bool operator==(const Layout& o) const;
  bool operator!=(const Layout& o) const { return !(*this == o); }
  std::string key() const;  // canonical serialisation (grouping)
  static Layout panel(int q, int fdim);
  static Layout split_of(std::vector<Layout> kids);
};
Layout layout_meet(const Layout& a, const Layout& b);
struct FaceProjection {
  HostMat refine;   // 4q^2 x q^2: coarse panel -> four quadrant panels
  HostMat coarsen;  // q^2 x 4q^2
};
FaceProjection face_projection(int q);
HostMat layout_transfer(const Layout& from, const Layout& to, const FaceProjection& proj);

// the tree as passed through the C-ABI
struct GTree {
  int dim = 3, p = 0, q = 0, nchild = 8, nface = 6;
  std::vector<int> depth, nch, parent;
  std::vector<std::array<int, 8>> child;
  std::vector<double> lo, hi;         // 3 per node
  std::vector<int> leaves;            // depth-first (mesh.cpp:54-71)
  std::vector<int> leaf_ord;          // node -> leaf ordinal, -1 for internal nodes
  std::vector<std::vector<int>> levels;  // node ids per depth, depth-first order
  int max_depth() const { return int(levels.size()) - 1; }
};
// validates (children nest, 2^dim children, DFS leaves) and derives levels / leaf ordinals
void finalize_gtree(GTree& t);

// one merge group: internal nodes of one depth whose children have identical face layouts
struct BlockCopyG {
  int dst;      // 0: MD = [D | h_int | C], 1: B, 2: AH = [h_ext | A]
  int dr, dc;   // destination offset
  int child;    // source child slot
  int sr, sc;   // source offset in the (projected) child [h | T] (column 0 = h)
  int rows, cols;
};
struct DownCopy {   // propagate: child face segment of g (solver.cpp:213-222)
  int child;
  int dst_off, dst_len;   // in the child's own boundary vector
  int src_int;            // 1: from g_int, 0: from the parent's exterior g
  int src_off, src_len;
  int E_off;              // offset of the E matrix (dst_len x src_len, column-major) in Edata, -1: identity
};
struct MergeGroup {
  int depth = 0;
  bool root = false;
  std::vector<int> nodes;           // node ids
  int n_ext = 0, n_int = 0;
  int nchild = 8;
  int child_nb[8] = {};             // child boundary size
  int child_nbp[8] = {};            // projected child boundary size
  bool proj[8] = {};
  HostMat R[8];                     // nbp x nb (row transfers, identity on untouched faces)
  HostMat Ehat[8];                  // (1 + nb) x (1 + nbp): diag(1, E) (column transfers)
  std::vector<BlockCopyG> blocks;   // gather, in two non-overlapping passes (see pass_split)
  int pass_split = 0;               // blocks[0, pass_split) write first, the rest accumulate second
  std::vector<DownCopy> down;
  std::vector<double> Edata;
  std::vector<Layout> sections;     // parent faces (shared by every node of the group)
};

struct LeafGroup {                  // leaves of one depth (one leaf side length, one operator set)
  int depth = 0;
  double side = 0.0;
  std::vector<int> leaves;          // node ids
};

struct GeneralPlan {
  GTree tree;
  std::vector<std::vector<Layout>> sections;  // per node, per face
  std::vector<LeafGroup> leaf_groups;
  std::vector<std::vector<MergeGroup>> merge_groups;  // per depth (deepest last)
  // node -> (kind, group, index): kind 0 leaf group, 1 merge group
  std::vector<std::array<int, 3>> home;
  int root_nb = 0, top_D = 0;
  double build_flops = 0.0;  // counted (SURVEY 8d formulas on the realised sizes)
};
GeneralPlan make_general_plan(GTree tree, bool implicit_root);

// Adaptive 3D refinement (refine_adaptive, proj/src/mesh.cpp:233-318) and the 2:1 level restriction
// (enforce_level_restriction, :141-167): per-field interpolation-error refinement with the parent-to-children
// Chebyshev interpolant (refinement_interpolant, spectral.cpp:438-452), union of the per-field trees, then
// level restriction plus re-verification.  Node order = the reference's construction order.
struct RefineResult {
  GTree tree;                 // depth, nch, child, lo, hi (finalized)
  std::vector<long long> anchor;  // 3 per node
  std::vector<int> unresolved;    // leaves at max_depth that still fail the criterion
  std::vector<double> global_sup;
};
using PointField = double (*)(const void* ctx, const double* x);
RefineResult refine_adaptive(const double* lo, const double* hi, int p, double tol, int max_depth,
                             const std::vector<std::pair<PointField, const void*>>& fields);
void enforce_level_restriction(GTree& t, std::vector<long long>& anchor);

// points of the root boundary in the reference's canonical order (HpsSolver::root_boundary_points)
std::vector<double> general_root_points(const GeneralPlan& g);
// Chebyshev points of every leaf (leaf-major, DFS order)
std::vector<double> general_leaf_points(const GeneralPlan& g);
void general_leaf_points_into(const GeneralPlan& g, double* out);

}  // namespace hpsg
