/* hps_cuda.h -- C-ABI of the B200-native HPS fast direct solver (libhps_b200.so).
 *
 * Drop-in boundary for the reference's HpsSolver<Real> DtN path
 * (/root/reference/proj/include/hps/solver.hpp:40-117).  Plain C types only:
 * host pointers, sizes and int status codes; no CUDA or torch types.  Each entry
 * point names the reference interface it replaces.
 *
 * Conventions (identical to the reference):
 *   - matrices are column-major (proj/include/hps/core.hpp:17);
 *   - leaves are in depth-first order (proj/src/mesh.cpp:54-71), points of a leaf
 *     in tensor order i1*p+i2 (3D (i1*p+i2)*p+i3) with axis node k at
 *     cheb_lobatto_1d(p)[k], descending (proj/include/hps/spectral.hpp:36-37);
 *   - boundary vectors are in the canonical section order of
 *     HpsSolver::root_boundary_points (proj/src/solver.cpp:159-182);
 *   - node ids follow build_uniform_tree's construction order (proj/src/mesh.cpp:113-118).
 *   - solution arrays are leaf-major, point-minor (SPEC.md:438 dump order); with
 *     nrhs > 1 the right-hand side index is outermost.
 */
#ifndef HPS_CUDA_H
#define HPS_CUDA_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (hps::Error in the reference, proj/include/hps/core.hpp:27-35) */
enum {
  HPSG_OK = 0,
  HPSG_ERR_INVALID = 1,        /* bad argument / unsupported configuration (reference: require()) */
  HPSG_ERR_SINGULAR_LEAF = 2,  /* "local_solve_dtn: singular factorization (zero pivot at i)", local_solve.cpp:96-101 */
  HPSG_ERR_SINGULAR_MERGE = 3, /* "merge_dtn: singular interface matrix D (pivot i)", merge.cpp:281-288 */
  HPSG_ERR_NONFINITE = 4,      /* "discretize_operator: non-finite coefficient sample ...", local_solve.cpp:56-61 */
  HPSG_ERR_OOM = 5,
  HPSG_ERR_CUDA = 6,
  HPSG_ERR_STATE = 7,          /* call order (e.g. solve before build) */
  HPSG_ERR_NO_DEVICE = 8       /* no CUDA device: the product never falls back to the CPU */
};

/* coefficient / source field descriptors.  The reference takes
 * std::function<Real(const Point&)> evaluated on the host per point
 * (proj/include/hps/local_solve.hpp:17-23, solver.hpp:43-45); here a field is
 * either a built-in closed form evaluated on the device, or host samples
 * (HPSG_FIELD_SAMPLED, samples[leaf * p^dim + pt]) for arbitrary functions. */
enum {
  HPSG_FIELD_CONST = 0,          /* c0 */
  HPSG_FIELD_BUMPS = 1,          /* c0 + c1 * sum_j exp(-c2 |x - z_j|^2) */
  HPSG_FIELD_PLANE_SIN = 2,      /* c0 * sin(c1 x1 + c2 x2 + c3 x3 + c4) */
  HPSG_FIELD_PLANE_COS = 3,      /* c0 * cos(c1 x1 + c2 x2 + c3 x3 + c4) */
  HPSG_FIELD_BUMPS_SIN = 4,      /* c0 * sum_j exp(-c2 |x-z_j|^2) * sin(c3 x1 + c4 x2 + c5 x3 + c6) */
  HPSG_FIELD_POISSON2D_SRC = 5,  /* source of make_manufactured_2d_dtn, proj/src/problems.cpp:62-66 */
  HPSG_FIELD_SAMPLED = 6,
  HPSG_FIELD_BUMPS_GRAD = 7,     /* d/dx_a of HPSG_FIELD_BUMPS: c1 * sum_j -2 c2 (x_a - z_ja) exp(-c2 |x - z_j|^2), a = c3 */
  HPSG_FIELD_DIVGRAD_SRC = 8,    /* div(eps grad u), eps = BUMPS(c0,c1,c2), u = prod_k sin(c3 x_k + c4) (3D config 4) */
  HPSG_FIELD_WAVEFRONT_SRC = 9,  /* Laplacian of atan(c0 |x - (c1,c2,c3)|^2 - 0.7): make_wavefront_3d, problems.cpp:154-179 */
  HPSG_FIELD_PB_EPS = 10,        /* c0 + (c1 - c0) exp(-c2 rho), rho = sum_j exp(-c3 |x - z_j|^2): PoissonBoltzmannSpec::eps
                                    (smooth), problems.cpp:187-191 */
  HPSG_FIELD_PB_EPS_GRAD = 11    /* d/dx_a of HPSG_FIELD_PB_EPS, a = c4 (PoissonBoltzmannSpec::grad_eps, :200-205) */
};
typedef struct {
  int kind;
  int n_centers;
  double c[8];
  const double* centers; /* n_centers x 3 (host) */
  const double* samples; /* n_leaves x p^dim (host), for HPSG_FIELD_SAMPLED */
} hpsg_field;

/* CoefficientField (proj/include/hps/local_solve.hpp:17-23) */
enum { HPSG_ROLE_LAPLACIAN = 0, HPSG_ROLE_GRADIENT = 1, HPSG_ROLE_ZEROTH = 2, HPSG_ROLE_SECOND_ORDER = 3 };
typedef struct {
  int role;
  int axis, axis2;
  hpsg_field field;
} hpsg_term;

/* uniform quad/octree: build_uniform_tree(domain, L, dim, p), proj/src/mesh.cpp:90-121 */
typedef struct {
  int dim;        /* 2 or 3 */
  int p;          /* Chebyshev points per axis; q = p - 2 Gauss points per panel */
  int L;          /* depth (>= 1) */
  double lo, hi;  /* domain [lo,hi]^dim */
} hpsg_tree;

typedef struct {
  int literal_sign;     /* 1: reference convention v_i = -L_ii^-1 f_i (local_solve.cpp:137); 0: corrected (+) */
  int root_implicit_S;  /* MergeOptions::implicit_S at the root (merge.hpp:104, solver.cpp:104) */
  int device;           /* CUDA device ordinal */
  int keep_factors;     /* keep the leaf LU factors for hpsg_solve_new_source (LeafSolution::fac,
                           local_solve.hpp:36); 2D p=16 L=8: +20 GB, batched leaf path */
  int variant;          /* HPSG_VARIANT_DTN (HpsSolver<Real>) or HPSG_VARIANT_ITI (HpsSolver<Complex>,
                           2D impedance-to-impedance maps, spectral.hpp:87) */
  double eta;           /* ItI impedance parameter (HpsSolver ctor eta, solver.hpp:43) */
  int build_root_T;     /* ItI: form and factor the root T for the radiation closure
                           (SolverOptions::build_root_T, solver.hpp:19; solver.cpp:153-157) */
  const hpsg_field* source_imag;  /* ItI: imaginary part of the complex source (NULL: real source) */
  /* execution choices (zero = the measured default; results agree to roundoff either way) */
  int force_batched_leaf;  /* 1: multi-launch batched leaf path instead of the persistent fused leaf kernel */
  int no_lu_lookahead;     /* 1: plain blocked LU driver instead of the look-ahead driver for n > 512 */
  int force_lu_leaf;       /* 1: LU leaf solve even where the fast-diagonalisation leaf applies (constant
                              Laplacian + zeroth-order terms, uniform 2D tree; leaf_fdm.cu) */
} hpsg_options;
enum { HPSG_VARIANT_DTN = 0, HPSG_VARIANT_ITI = 1 };

typedef struct {
  int n_leaves;
  long long n_points;          /* N = n_leaves * p^dim */
  int root_bsize;              /* length of the root boundary vector */
  int top_D_size;              /* HpsSolver::top_D_size (solver.cpp:321-324) */
  int tree_depth;
  double min_rcond;            /* min over leaves of min|u_ii|/max|u_ii| (local_solve.cpp:103-106); fast-
                                  diagonalisation leaves: min/max |lam_i + lam_j + cbar| of the leaf operator */
  int ill_conditioned;         /* any_ill_conditioned (solver.hpp:92) */
  double t_build_ms, t_leaf_ms, t_merge_ms, t_solve_ms;   /* last build / solve, CUDA events */
  double build_flops;          /* counted algorithmic FLOPs of the build (SURVEY 8d formulas) */
  double solve_bytes;          /* algorithmic HBM bytes of the last solve */
  double device_bytes;         /* device memory held by the context */
  int launches_build, launches_solve; /* kernels launched by the last build / solve */
  int n_levels;                /* = tree depth L */
  double t_level_ms[24];       /* merge time of depth d (CUDA events), d = 0 .. L-1 */
  int leaf_path;               /* last build's leaf stage: 0 fused LU kernel, 1 batched LU, 2 fast
                                  diagonalisation, 3 fast diagonalisation that fell back to the fused LU,
                                  4 ItI by block elimination (fast-diagonalisation interior solve + reduced
                                  boundary LU), 5 ItI block elimination that fell back to the full LU */
  double leaf_exec_flops;      /* fast-diagonalisation leaf stage: FP64 tensor FLOPs it executed (DMMA.8x8x4
                                  instructions x 512, counted on the device); 0 for the LU leaf paths */
} hpsg_stats;

typedef struct hpsg_ctx hpsg_ctx;

/* HpsSolver<Real>(tree, Variant::dtn, eta, terms, source, opts), solver.hpp:43-45 */
int hpsg_create(const hpsg_tree* tree, const hpsg_term* terms, int n_terms, const hpsg_field* source,
                const hpsg_options* opts, hpsg_ctx** out);
/* HpsSolver::build(), solver.hpp:48 / solver.cpp:144-151: leaf stage + all merge levels */
int hpsg_build(hpsg_ctx* ctx);

/* General tree: the reference's DiscretizationTree (proj/include/hps/mesh.hpp:28-61), e.g. an adaptive,
 * level-restricted octree from refine_adaptive (mesh.cpp:233-318).  Node 0 is the root; node i has
 * n_children[i] = 0 (leaf) or 2^dim children in the child_offset slot order (mesh.hpp:24-25), stored in
 * children[8*i .. 8*i+7]; lo/hi (3 per node) are the reference's boxes (children are exact halves).
 * Merges of children with different refinement project the finer interface onto the coarser one
 * (merge.cpp:201-211, 264-266) and undo it in the downward pass.  DtN variant; hpsg_build,
 * hpsg_solve(_device), hpsg_root_boundary_points, hpsg_leaf_points and hpsg_get_stats apply; the
 * uniform-tree entry points (parts, new sources, ItI, getters) return HPSG_ERR_STATE.
 * Replaces HpsSolver(const DiscretizationTree&, ...) (solver.hpp:43-45) for arbitrary trees. */
typedef struct {
  int dim, p;
  int n_nodes;
  const int* depth;       /* n_nodes */
  const int* n_children;  /* n_nodes */
  const int* children;    /* n_nodes x 8 */
  const double* lo;       /* n_nodes x 3 */
  const double* hi;       /* n_nodes x 3 */
} hpsg_tree_desc;
int hpsg_create_tree(const hpsg_tree_desc* tree, const hpsg_term* terms, int n_terms, const hpsg_field* source,
                     const hpsg_options* opts, hpsg_ctx** out);
/* refine_adaptive(domain [lo,hi] (3 each), RefinementCriterion{tol, p, fields}, max_depth, &unresolved)
 * (proj/src/mesh.cpp:233-318, with enforce_level_restriction :141-167): 3D, built-in fields evaluated on the
 * host.  Writes the tree as node arrays in the reference's construction order (n_nodes x {depth, n_children,
 * children[8], lo[3], hi[3]}); returns HPSG_ERR_INVALID with *n_nodes set when cap is too small. */
/* refine_adaptive with caller point functions (the reference's RefinementCriterion::test_fields,
 * std::function<Real(const Point&)>, mesh.hpp:63-68): fns[i](users[i], x[3]). */
typedef double (*hpsg_point_fn)(void* user, const double* x);
int hpsg_refine_adaptive_cb(int p, const double* lo, const double* hi, double tol, int max_depth,
                            hpsg_point_fn const* fns, void* const* users, int n_fields, int cap, int* n_nodes,
                            int* depth, int* n_children, int* children, double* lo_out, double* hi_out,
                            int* n_unresolved);
/* enforce_level_restriction (mesh.cpp:141-167) of a tree: refinement only, node order kept, new nodes
 * appended in the reference's split order. */
int hpsg_enforce_level_restriction(const hpsg_tree_desc* tree, int cap, int* n_nodes, int* depth, int* n_children,
                                   int* children, double* lo, double* hi);
/* leaf_cheb_points of every leaf of a tree (DFS order, leaf-major; mesh.cpp:320-340) */
int hpsg_tree_desc_leaf_points(const hpsg_tree_desc* tree, double* xyz);
/* mesh_to_json (proj/src/mesh.cpp:435-463): the tree as the reference's JSON text (nlohmann dump(1) format,
 * byte-identical).  out == NULL: only *len (without the terminating 0) is set. */
int hpsg_mesh_json(const hpsg_tree_desc* tree, char* out, size_t cap, size_t* len);
/* dump_solution (proj/src/downpass.cpp:108-143): the device-resident solution d_u (n_points
 * doubles, or interleaved complex) to bin_path (raw little-endian FP64, leaf-major / point-minor) and the JSON
 * sidecar json_path {"dtype", "leaf_len", "n_leaves", "tree_ref"}, each written to <path>.tmp and renamed. */
int hpsg_dump_solution(hpsg_ctx* ctx, const double* d_u, int is_complex, const char* json_path, const char* bin_path,
                       const char* tree_ref);
int hpsg_refine_adaptive(int p, const double* lo, const double* hi, double tol, int max_depth,
                         const hpsg_field* fields, int n_fields, int cap, int* n_nodes, int* depth, int* n_children,
                         int* children, double* lo_out, double* hi_out, int* n_unresolved);

/* ---- subtree-sharded builds (the staged build_leaf/merge_internal API of
 * solver.hpp:51-56 at subtree granularity).  A PART is the subtree rooted at node
 * root_index (index within tree.levels[root_depth], = DFS order for uniform trees) cut at
 * depth cut_depth: cut_depth == L -> its leaves are real leaves (leaf stage + merges);
 * cut_depth < L -> its leaves are the depth-cut_depth nodes, whose [h|T] (n x (1+n),
 * column-major, h first) are inputs.  Parts compose: the [h|T] a part produces at its root
 * is exactly the input its parent part expects, and the boundary data a cut part's downward
 * pass produces for its cut nodes is exactly the root data of the parts below. */
typedef struct {
  int root_depth;
  long long root_index;
  int cut_depth;
} hpsg_part;
int hpsg_create_part(const hpsg_tree* tree, const hpsg_part* part, const hpsg_term* terms, int n_terms,
                     const hpsg_field* source, const hpsg_options* opts, hpsg_ctx** out);
/* move a part to another subtree of the same depth (same sizes, new boxes): the device workspace is
 * reused, so subtree recomputation costs no allocation; not for HPSG_FIELD_SAMPLED coefficients */
int hpsg_part_retarget(hpsg_ctx* ctx, long long root_index);
/* n_cut input nodes of cut_nb boundary points each (0 for a part with real leaves); root_nb =
 * boundary points of the part root */
int hpsg_part_sizes(hpsg_ctx* ctx, long long* n_cut, int* cut_nb, int* root_nb);
/* Device footprint of a context (whole tree when part is NULL) without allocating it: the bytes
 * hpsg_create_part would allocate plus, for nrhs > 0, what the first hpsg_solve of nrhs right-hand
 * sides adds (solve workspace and the host-API staging of g and u; 0: build only).
 * The input of the memory-budgeted planner (SPEC.md planner module, make_plan; the reference's
 * proj/src/planner.cpp is a stub). */
int hpsg_estimate_bytes(const hpsg_tree* tree, const hpsg_part* part, const hpsg_term* terms, int n_terms,
                        const hpsg_field* source, const hpsg_options* opts, int nrhs, double* bytes);
/* [h|T] of the part root after hpsg_build (root_depth > 0): device-to-device into d_dst
 * (root_nb x (1+root_nb)); MergeOutput::T/h, merge.hpp:58-66 */
int hpsg_part_root_ht(hpsg_ctx* ctx, double* d_dst);
/* input [h|T] of cut node k (0 <= k < n_cut, level order) from device memory; all must be set
 * before hpsg_build */
int hpsg_part_set_cut_ht(hpsg_ctx* ctx, long long k, const double* d_src);
/* downward pass of a cut part (HpsSolver::propagate, solver.cpp:188-228): root boundary data
 * (device, nrhs x root_nb) -> boundary data of every cut node (device, nrhs x n_cut x cut_nb) */
int hpsg_part_solve_cut(hpsg_ctx* ctx, const double* d_g_root, int nrhs, double* d_g_cut);
/* HpsSolver::solve(g_root, leaf_g_out), solver.hpp:64 / solver.cpp:238-252, for nrhs boundary
 * vectors (g_root: nrhs x root_bsize).  u_out: nrhs x n_leaves x p^dim (host);
 * leaf_g_out (optional): nrhs x n_leaves x (boundary Gauss points of a leaf). */
int hpsg_solve(hpsg_ctx* ctx, const double* g_root, int nrhs, double* u_out, double* leaf_g_out);
/* same with device pointers (no host copies); results are ready when the call returns */
int hpsg_solve_device(hpsg_ctx* ctx, const double* d_g_root, int nrhs, double* d_u_out);
/* ItI variant: HpsSolver<Complex>::solve(g_root) (solver.cpp:238-252) with complex data as
 * interleaved (re, im) doubles: g_root nrhs x root_bsize incoming impedance data at the root
 * boundary Gauss points, u_out nrhs x n_leaves x p^2.  Internally every complex matrix is carried
 * in real-equivalent form [[re, -im], [im, re]]. */
int hpsg_solve_complex(hpsg_ctx* ctx, const double* g_root, int nrhs, double* u_out);
/* HpsSolver::solve_radiation() (solver.cpp:254-259): root data g = -T_root^-1 h_root, then the
 * downward pass; needs build_root_T.  u_out: n_leaves x p^2 interleaved complex; g_out (optional):
 * the closing root data (root_bsize interleaved complex). */
int hpsg_solve_radiation(hpsg_ctx* ctx, double* u_out, double* g_out);
/* ---- output layer, on the device-resident solution of hpsg_solve_device /
 * hpsg_solve_complex's device twin: d_u = n_leaves x p^dim values (is_complex: interleaved).
 * evaluate_at(field, points) (downpass.hpp:19, downpass.cpp:13-95): points_host npts x 3 -> out_host
 * (npts, or 2 npts interleaved); points outside the domain are rejected like the reference. */
int hpsg_evaluate_at(hpsg_ctx* ctx, const double* d_u, int is_complex, const double* points_host, int npts,
                     double* out_host);
/* error_report(field, exact) (problems.hpp:81, problems.cpp:270-293) against a built-in exact
 * field (exact_imag may be NULL): relative L-inf and L2 over every leaf Chebyshev point, reduced on
 * the device (no copy of the solution). */
int hpsg_error_report(hpsg_ctx* ctx, const double* d_u, int is_complex, const hpsg_field* exact,
                      const hpsg_field* exact_imag, double* rel_linf, double* rel_l2);

/* host-only: the ItI leaf operators of assemble_iti_ops_2d (spectral.cpp:312-368), column-major:
 * G = Gr + i Gi ((4p-4) x p^2), P ((4p-4) x 4q), QH = QHr + i QHi (4q x p^2); any pointer may be NULL */
int hpsg_iti_leaf_ops(int p, double eta, double side, double* Gr, double* Gi, double* P, double* QHr, double* QHi);
/* host-only: the operators of the fast-diagonalisation leaf solve for a constant Laplacian coefficient a on leaves
 * of side `side` (2D, p in 4..16, n1 = p-2): A = s^2 (a D2[int, int]) (n1 x n1, s = 2/side, the rounding of the
 * leaf assembly), its eigendecomposition A = V diag(lam) V^-1, and the separable interior Q factors
 * Q_i(s q + i, (i1, i2)) = ds G(i, m) d_s(k) (G: q x n1 row-major, d: 4 x n1 row-major), with (m, k) = (i1-1,
 * i2-1) on the S / N sides and (i2-1, i1-1) on E / W.  Returns
 * HPSG_ERR_INVALID when A has no real eigendecomposition (the solver then keeps the LU leaf).  Any pointer may be
 * NULL. */
int hpsg_fdm_leaf_ops(int p, double side, double a, double* A, double* lam, double* V, double* Vinv, double* G,
                      double* d, double* ds, double* Qi);   /* Qi: the dense interior Q (4q x (p-2)^2, column-major) */
/* HpsSolver::solve_new_source(leaf_f, RootBC::dirichlet, g_root), solver.hpp:71-72 /
 * solver.cpp:285-307 (make_source_state :261-283, leaf_resolve_source local_solve.cpp:174-183,
 * artifact_source_pass merge.cpp:514-567), for nsrc sources at once against the stored build:
 * leaf_f: nsrc x n_leaves x p^dim source samples at the leaf Chebyshev points (only interior
 * points are used), g_root: nsrc x root_bsize, u_out: nsrc x n_leaves x p^dim.  Needs
 * keep_factors = 1 at create time.  The sign convention is the build's (literal_sign). */
int hpsg_solve_new_source(hpsg_ctx* ctx, const double* leaf_f, const double* g_root, int nsrc, double* u_out);
int hpsg_solve_new_source_device(hpsg_ctx* ctx, const double* d_leaf_f, const double* d_g_root, int nsrc,
                                 double* d_u_out);
/* HpsSolver::root_boundary_points(), solver.hpp:60 (root_bsize x 3) */
int hpsg_root_boundary_points(hpsg_ctx* ctx, double* xyz);
/* leaf_cheb_points over all leaves, mesh.hpp:73-74 (n_leaves x p^dim x 3) */
int hpsg_leaf_points(hpsg_ctx* ctx, double* xyz);
/* LeafSolution<Real> of leaf `ord` (local_solve.hpp:30-39): Y (p^d x nb), v (p^d), T (nb x nb), h (nb) */
int hpsg_get_leaf(hpsg_ctx* ctx, int ord, double* Y, double* v, double* T, double* h);
/* MergeArtifact sizes of an internal node (merge.hpp:58-64) */
int hpsg_node_sizes(hpsg_ctx* ctx, int node_id, int* n_ext, int* n_int);
/* MergeArtifact S_mat (n_int x n_ext), gtilde (n_int) and node_T/node_h (n_ext^2, n_ext) of a
 * non-root internal node (solver.hpp:83-85).  Any pointer may be NULL.  The build leaves the rows of T/h on the
 * domain boundary unformed where nothing downstream reads them (a root that forms no T); the first request for
 * T or h forms them (GPU work on the context's stream), with the values an unskipped build stores. */
int hpsg_get_node(hpsg_ctx* ctx, int node_id, double* S, double* gtilde, double* T, double* h);
int hpsg_get_stats(hpsg_ctx* ctx, hpsg_stats* out);
/* run all later work of ctx on a caller-owned cudaStream_t (passed as void*; NULL = legacy
 * default stream) so callers can order and time it with their own events */
int hpsg_set_stream(hpsg_ctx* ctx, void* stream);
const char* hpsg_last_error(hpsg_ctx* ctx);
void hpsg_destroy(hpsg_ctx* ctx);

/* ---- subtree-sharded build/solve over `world` ranks, one GPU each (replaces the
 * single-process HpsSolver(tree, spec, opts) + build() + solve() of solver.cpp:33-252 when the caller
 * runs one process per GPU).  The tree is cut at depth ds (smallest with nchild^ds >= world);
 * depth-ds subtree k belongs to rank k*world/nchild^ds (a contiguous DFS leaf range, mesh.cpp:54-71);
 * nodes above the cut are merged by the owner of their first subtree.  The only transfers are the
 * [h|T] of a child whose owner differs from its parent's (upward, merge.cpp:226-278) and its boundary
 * data (downward, solver.cpp:210-224), sent through the caller's transport on the shard's stream —
 * typically ncclGroupStart / ncclSend / ncclRecv / ncclGroupEnd.  Every call is
 * collective: all ranks call it in the same order.  Real (DtN) uniform trees only. */
typedef struct {
  void* user;
  int (*group_begin)(void* user);                                     /* may be NULL */
  int (*send)(void* user, const void* d_buf, size_t bytes, int peer, void* stream);
  int (*recv)(void* user, void* d_buf, size_t bytes, int peer, void* stream);
  int (*group_end)(void* user, void* stream);                         /* may be NULL */
} hpsg_transport;
typedef struct hpsg_shard hpsg_shard;
/* tr may be NULL for world == 1; opts->device selects this rank's GPU */
int hpsg_shard_create(const hpsg_tree* tree, const hpsg_term* terms, int n_terms, const hpsg_field* source,
                      const hpsg_options* opts, int world, int rank, const hpsg_transport* tr, hpsg_shard** out);
int hpsg_shard_build(hpsg_shard* s);
/* d_g_root (nrhs x root_bsize, device) is read on the root owner (rank 0) only; d_u receives this rank's
 * leaves: nrhs x n_leaves_here x p^dim (device), the leaves [first_leaf, first_leaf + n_leaves_here) of
 * the DFS order */
int hpsg_shard_solve_device(hpsg_shard* s, const double* d_g_root, int nrhs, double* d_u);
int hpsg_shard_info(hpsg_shard* s, int* cut_depth, long long* first_leaf, long long* n_leaves_here);
const char* hpsg_shard_last_error(hpsg_shard* s);
void hpsg_shard_destroy(hpsg_shard* s);

/* centers of the seeded Gaussian-bump fields: std::mt19937_64(seed) with
 * uniform_real_distribution(-0.5, 0.5), as make_scattering / make_pb_spec draw them
 * (proj/src/problems.cpp:126-141, :240-249).  out: n x 3 (z = 0 in 2D). */
void hpsg_bump_centers(unsigned long long seed, int n, int dim, double* out);

/* Host-only geometry (no device, no context): leaf_cheb_points of every leaf of the uniform
 * tree in DFS order (n_leaves x p^dim x 3), so callers can sample std::function fields into
 * HPSG_FIELD_SAMPLED arrays before hpsg_create (mesh.cpp:320-336, solver.cpp:49-57). */
int hpsg_tree_leaf_points(const hpsg_tree* tree, double* xyz);
/* cheb_nodes(p) (proj/src/spectral.cpp:14-26): the p Chebyshev points on [-1, 1], descending from +1; a
 * leaf's points are 0.5 (lo + hi) + 0.5 (hi - lo) t per axis (leaf_cheb_points, mesh.cpp:320-336) */
int hpsg_cheb_nodes(int p, double* t);
/* Host-only: root boundary points in canonical section order (root_bsize x 3), no device needed */
int hpsg_tree_root_points(const hpsg_tree* tree, double* xyz);

/* library-level probes */
int hpsg_device_count(void);
const char* hpsg_build_info(void);

/* Batched primitives on DEVICE pointers (column-major, strided batches; used by the
 * kernel-level parity tests).  They replace the Eigen calls inside the hot path:
 *   hpsg_dev_dgemm     : D = alpha*A*B + beta*C          (Eigen products, merge.cpp:294-295)
 *   hpsg_dev_getrf_aug : PartialPivLU of M[:, :n] and M[:, n:n+m] <- A^-1 M[:, n:n+m]
 *                        (local_solve.cpp:125-137, merge.cpp:280-292); ipiv 0-based,
 *                        stats = (min|u_ii|, max|u_ii|, first zero pivot or -1) per matrix
 *   hpsg_dev_getrs     : R <- A^-1 R with stored factors (MergeArtifact::apply_Dinv, merge.cpp:156-174) */
int hpsg_dev_dgemm(int m, int n, int k, int batch, double alpha, const double* A, long long lda, long long sA,
                   const double* B, long long ldb, long long sB, double beta, const double* C, long long ldc,
                   long long sC, double* D, long long ldd, long long sD);
int hpsg_dev_getrf_aug(int batch, int n, int m, double* M, long long ld, long long stride, int* ipiv,
                       double* stats);
int hpsg_dev_getrs(int batch, int n, int m, const double* LU, long long ld, long long stride, const int* ipiv,
                   double* R, long long ldr, long long strideR);
/* Live timing of the DMMA GEMM inside the hot path (bench roofline of the GEMM): mode 1 starts
 * recording (a CUDA event pair per launch on its own stream, plus 2mnk FLOPs per matrix), mode 0
 * stops, mode 2 synchronises and returns the summed launch time (ms), FLOPs and launch count of the
 * recording.  Instrumentation only: the product path records nothing unless started. */
int hpsg_dev_gemm_timing(int mode, double* ms, double* flops, long long* launches);

#ifdef __cplusplus
}
#endif
#endif /* HPS_CUDA_H */
