// hps_kernels.cuh -- HPS-specific device kernels (leaf assembly, merge gather,
// downward scatter, leaf output).  The dense FP64 work (LU, TRSM, GEMM) lives
// in lu.cu / gemm.cu; these kernels move and build the operands around it.
#pragma once

#include "common.cuh"

namespace hpsk {

constexpr int kMaxTerms = 6;

struct DevField {
  int kind;
  int n_centers;
  double c[8];
  const double* centers;  // device, n_centers x 3
  const double* samples;  // device, n_leaves x npts
};
struct DevTerm {
  int role, axis, axis2;
  DevField f;
};

// ---- stage 1: leaf operator assembly -------------------------------------
// Reference: discretize_operator (proj/src/local_solve.cpp:44-86) restricted to
// the interior rows, plus the source sampling of HpsSolver::build_leaf
// (proj/src/solver.cpp:49-57).  Never materializes the full n x n operator.
struct LeafAsmArgs {
  int dim, p, n, ni, ne, nb, nterms;
  double scale;         // 2/side
  double fsign;         // -1 literal (v = -L^-1 f, local_solve.cpp:137), +1 corrected
  DevTerm terms[kMaxTerms];
  DevField source;
  int has_source;
  const double* leaf_box;  // 6 per leaf (lo[3], hi[3]) in DFS order
  const double* cheb;      // p
  const double* D;         // p x p col-major
  const double* D2;        // p x p col-major
  const int* interior;     // ni tensor indices
  const int* exterior;     // ne
  double* M;               // per leaf: ni x (ni + 1 + nb): [L_ii | sgn*f_i | (filled by GEMM)]
  long long strideM;
  double* E;               // per leaf: ni x ne  (L_ie)
  long long strideE;
  int* bad_point;          // per leaf: first non-finite sample point index (or INT_MAX)
};
void launch_leaf_assemble(const LeafAsmArgs& a, int n_leaves, cudaStream_t st);

// ---- ItI variant (real-equivalent embedding; geometry.hpp ItiLeafOperators / ItiMergeTables) ----
// Leaf system of local_solve_iti (proj/src/local_solve.cpp:145-172) in real-equivalent form:
// M = [B_re | f_re | Prhs_re] with B = [G ; L(I_i, :)] (n x n complex) -> 2n x 2n real, f on the
// interior rows, and the Y right-hand sides [P; 0] and i[P; 0] so that the solve returns the
// real-equivalent Y directly.  M is 2n x (2n + 1 + 2 nb) per leaf, column-major, ld 2n.
struct ItiLeafArgs {
  LeafAsmArgs a;            // coefficient / geometry fields (a.n = p^2, a.ni interior count)
  int nbc, nbq;             // 4p-4 walk rows, 4q Gauss boundary points
  const double* Gr;         // nbc x n
  const double* Gi;         // nbc x n
  const double* P;          // nbc x nbq
  DevField source_im;       // imaginary part of a complex source (has_source_im)
  int has_source_im;
};
void launch_iti_leaf_assemble(const ItiLeafArgs& a, int n_leaves, cudaStream_t st);

// ItI leaf by block elimination of [G; L_int] (local_solve.cpp:145-172): the leaf outputs in the layout of the
// real-equivalent LU path ([v | Y | iY], 2n rows in tensor order) from U_e (exterior) and U_i = W U_e (interior)
struct ItiFdmAssembleArgs {
  const double* Z;      // per leaf: z_re, z_im (nir each) = L_ii^-1 f_i
  const double* Ue;     // per leaf: 2 ne x mrhs (ld 2 ne), stacked re / im
  const double* Ure;    // per leaf: nir x mrhs
  const double* Uim;
  double* M;            // per leaf: [v | Y | iY] (2n x mrhs, ld 2n)
  long long stride;     // per-leaf stride of every array above
  const int* pos;       // tensor index -> interior position (>= 0) or -(exterior position) - 1
  int n, ne, nir, mrhs;
};
void launch_iti_fdm_assemble(const ItiFdmAssembleArgs& a, int n_leaves, cudaStream_t st);
// the real-equivalent columns of imaginary units from those of the real units (i z = (-im, re)), see hps_kernels.cu
void launch_iti_fill_im_half(double* X, long long ld, long long stride, int batch, int nc, int hc, int col_re0,
                             int col_im0, int ncols, cudaStream_t st);

struct DevBlockCopy {
  int dst, dr, dc, child, sr, sc, rows, cols;
};
// Block-list merge gather (ItI): copies every listed block of the children's [h|T] into the
// zero-initialised MD / B / AH of each node (identity blocks when child < 0).
struct BlockGatherArgs {
  const DevBlockCopy* blocks;
  int nblocks, nchild;
  const double* child_HT;
  long long child_ld, child_stride;
  double* dst[3];
  long long ld[3], stride[3];
};
void launch_block_gather(const BlockGatherArgs& a, int n_nodes, cudaStream_t st);
// u (interleaved complex, nrhs x n_leaves x n) from the real-equivalent leaf solution Ui
// (per leaf 2n x nrhs, ld 2n)
// A_b += I (n x n) for a strided batch
void launch_add_identity(double* A, int n, long long ld, long long stride, int batch, cudaStream_t st);
// dst_b[rows x cols] = src_b[rows x cols] for a strided batch of column-major blocks
void launch_copy_batched(double* dst, long long ldd, long long sd, const double* src, long long lds, long long ss,
                         int rows, int cols, int batch, cudaStream_t st);
void launch_iti_leaf_output(double* u, const double* Ui, int n, int nrhs, int n_leaves, cudaStream_t st);
// g_re (planar real-equivalent, nb_re x nrhs) from interleaved complex g (nrhs x nb)
void launch_complex_to_planar(double* g_re, const double* g, int nb, int nrhs, cudaStream_t st);

// ---- output layer on the device -------------------------------------------
// evaluate_at (proj/src/downpass.cpp:13-95): locate_leaf by midpoint descent + tensor barycentric
// interpolation of the leaf's Chebyshev values; u: n_leaves x p^dim (real, or interleaved complex).
struct EvalArgs {
  int dim, p, L, is_complex, npts;
  double lo, hi;
  const double* cheb;   // p nodes, descending
  const double* u;
  const double* x;      // npts x 3
  double* out;          // npts (real) or 2 npts (complex)
};
void launch_evaluate_at(const EvalArgs& a, cudaStream_t st);
// error_report (proj/src/problems.cpp:270-293) partial reductions: per block {max|u-ex|, max|ex|,
// sum|u-ex|^2, sum|ex|^2} over every leaf Chebyshev point; exact = re + i im (im may be kind < 0)
struct ErrArgs {
  int dim, p, npts_leaf, is_complex;
  long long n_leaves;
  const double* leaf_box;
  const double* cheb;
  const double* u;
  DevField ex_re, ex_im;
  int has_im;
  double* partial;      // gridDim x 4
};
int launch_error_partials(const ErrArgs& a, cudaStream_t st);  // returns the number of blocks

// Fused stage 1 (leaf_fused.cu): assembly + -L_ie P + GEPP/solve + [h|T] per leaf in one
// persistent kernel over an L2-resident per-CTA workspace.
struct LeafFusedArgs {
  LeafAsmArgs a;            // M/E fields unused; bad_point used
  const double* P;          // ne x nb
  const double* Qi;         // nb x ni
  const double* ZQeP;       // nb x (1 + nb) = [0 | Q_e P]
  double* scratch;          // per CTA: ni x (ni+1+nb) + ni x ne
  long long scratch_stride;
  double* Yv;               // per leaf: ni x (1 + nb) = [v_i | Y_i]
  long long strideYv;
  double* HT;               // per leaf: nb x (1 + nb) = [h | T]
  long long strideHT;
  double* stats;            // per leaf: min|u_ii|, max|u_ii|, first zero pivot (-1)
  long long* prof;          // optional phase timestamps (clock64) of CTA 0: [leaf_iter][8]
  long long n_leaves;       // leaves to solve: all, or the first n_leaves entries of leaf_list
  const int* leaf_list;     // optional: the leaves to solve (the fast-diagonalisation path's non-converged ones)
};
bool leaf_fused_supported(int n, int p, int ni, int nb, int dim, bool mixed_terms);
int leaf_fused_ctas_per_sm();
long long leaf_fused_scratch_per_cta(int ni, int ne, int nb);
cudaError_t launch_leaf_fused(const LeafFusedArgs& f, int grid, cudaStream_t st);

// Fast-diagonalisation leaf solve (leaf_fdm.cu) for a constant Laplacian plus zeroth-order terms on a
// uniform 2D tree: same outputs as leaf_fused_kernel ([v_i | Y_i], [h | T], statistics), no LU.
struct LeafFdmArgs {
  LeafAsmArgs a;            // fields, geometry, bad_point; M/E unused
  const double* P;          // ne x nb
  const double* Qi;         // nb x ni
  const double* ZQeP;       // nb x (1 + nb)
  const double* V;          // 16 x 16 col-major, zero padded: eigenvectors of the 1D interior operator
  const double* Vinv;       // 16 x 16
  const double* A;          // 16 x 16: the 1D interior operator s^2 (a D2[int, int]), zero padded
  const double* lam;        // 16: its eigenvalues (0 in the padding)
  double lap_coef;          // a (the constant Laplacian coefficient)
  const double* qG;         // separable Q_i (geometry.hpp q_interior_factors): G q x (p-2), d 4 x (p-2), ds
  const double* qd;
  double qds;
  double* Rtab;             // 4(p-2) blocks of 16 x 16: -L_ie P per column (block layout) and R^ = V^-1 R V^-T,
  double* Rhat;             // written by launch_leaf_fdm_prep, read by every leaf
  int iti = 0;              // ItI mode: P = I (ne columns), two source columns, output Z = L_ii^-1 [f_i | -L_ie]
  DevField source_im;       // (Yv = Z, strideYv), no [h|T]
  int has_source_im = 0;
  int src_cols = 0;         // source mode (> 0): src_cols columns per leaf read from Yv and solved in place
  double* Yv;
  long long strideYv;
  double* HT;
  long long strideHT;
  double* stats;            // per leaf: min / max |lam_i + lam_j + cbar|, -1 - (DMMA.8x8x4 issued)
  int* fail_count;          // leaves that did not converge: count and list (the host re-runs them with
  int* fail_list;           // the LU leaf kernel, so every leaf's result is independent of its neighbours)
  long long n_leaves;
};
bool leaf_fdm_shape_ok(int p, int ni, int nb, int dim);
int leaf_fdm_ctas_per_sm(int p);
cudaError_t launch_leaf_fdm_prep(const LeafFdmArgs& f, cudaStream_t st);
cudaError_t launch_leaf_fdm(const LeafFdmArgs& f, int grid, cudaStream_t st);

// ---- stage 2: merge operand gather ------------------------------------------
// Reference block assembly, proj/src/merge.cpp:226-278: child DtN blocks summed
// into [D | h_int | C], B and [h_ext | A] by destination-driven gathers (no atomics).
struct GatherArgs {
  int s, nchild, child_nb;
  const double* child_HT;   // per child: child_nb x (1 + child_nb), [h | T]
  long long child_stride;
  const int* src;           // destination table (2 codes per section block)
  int kind;                 // 0: MD = [D | h_int | C], 1: B, 2: AH = [h_ext | A]
  int NI, NE;
  int nrows, ncols;
  double* dst;
  long long ld, stride;
  // source-pass use (solver.cpp:261-283): logical columns start at col_offset, and nrhs
  // right-hand sides are gathered at once (child source / destination offsets per RHS)
  int col_offset = 0, nrhs = 1;
  long long src_rhs_stride = 0, dst_rhs_stride = 0;
  // rows with no source (structurally zero blocks) are not stored: set when the consumer reads only the
  // nonzero blocks (the block-sparse Schur product's B)
  bool skip_zero = false;
  const int* row_mask = nullptr;  // optional [node][row section]: rows of sections with 0 are not stored
  unsigned smagic = 0;      // set by launch_gather
};
void launch_gather(const GatherArgs& a, int n_nodes, cudaStream_t st);

// ---- stage 3: downward pass scatter ------------------------------------------
// Reference propagate() child gather, proj/src/solver.cpp:210-224: builds each
// child's [1; g] column(s) from the parent's g_ext and the interface values g_int.
struct ScatterArgs {
  int nchild, nface, s, nrhs;
  double lead = 1.0;        // value of the leading row (1: apply the stored gtilde; 0: new-source pass)
  const int* down;          // nchild*nface
  const double* Gp;         // parent: (1 + nbp) x nrhs per node
  long long ldGp, strideGp;
  const double* GI;         // parent interface values: n_int x nrhs per node
  long long ldGI, strideGI;
  double* Gc;               // children: (1 + nchild_b) x nrhs per child
  long long ldGc, strideGc;
};
void launch_scatter(const ScatterArgs& a, int n_parents, cudaStream_t st);

// GI <- -(GI + xh) (implicit root: g_int = -(x_h + D^-1 C g), solver.cpp:204-206)
void launch_neg_add(double* GI, const double* xh, int n, int nrhs, long long ld, cudaStream_t st);

// Leaf output in tensor order: u[rhs][leaf][idx] from the interior block
// Ui (ni x nrhs per leaf) and the exterior block Ue (ne x nrhs per leaf).
struct LeafOutArgs {
  int ni, ne, npts, nrhs, n_leaves;
  const int* interior;
  const int* exterior;
  const double* Ui;
  long long ldUi, strideUi;
  const double* Ue;
  long long ldUe, strideUe;
  double* u;
};
void launch_leaf_output(const LeafOutArgs& a, cudaStream_t st);

// Fill a batch of (1 + nb) x nrhs columns with [1; g]: from a dense g (nb x nrhs, ld nb).
void launch_pack_root(double* G, const double* g, int nb, int nrhs, cudaStream_t st, double lead = 1.0);
// new-source pass helpers: R[leaf][k][r] = sgn * f[k][leaf][interior[r]]; y <- a*y + b*x (n x nrhs blocks)
void launch_pack_source(double* R, const double* f, const int* interior, int ni, int npts, int n_leaves, int nrhs,
                        double sgn, cudaStream_t st);
void launch_axpby(double* y, long long ldy, long long sy, const double* x, long long ldx, long long sx, int n,
                  int nrhs, long long batch, double a, double b, cudaStream_t st);
// Extract leaf boundary data (without the leading 1) for leaf_g_out.
void launch_unpack_leaf_g(double* out, const double* G, int nb, long long ldg, int nrhs, int n_leaves, cudaStream_t st);

}  // namespace hpsk
