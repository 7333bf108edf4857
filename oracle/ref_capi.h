/* ref_capi.h -- TEST INFRASTRUCTURE ONLY.
 *
 * extern "C" face of oracle/_ref/libhps_ref.so: the REFERENCE's own, unmodified hot-path sources
 * (/root/reference/proj/src/{spectral,mesh,layout,local_solve,merge,solver,downpass,problems}.cpp)
 * compiled against the Eigen-API shim in oracle/eigen_shim (Eigen itself is absent from the image),
 * plus this thin wrapper (oracle/ref_capi.cpp), which only calls the reference's public API:
 * hps::build_uniform_tree / refine_adaptive, hps::HpsSolver<Real|Complex> (build, solve,
 * solve_radiation, solve_new_source, leaf_solutions, artifact, node_T/h), hps::problem_by_name,
 * hps::sample_boundary_data, hps::error_report, hps::solve_problem.
 *
 * Used by tests/ to pin the oracle restatement and the B200 product to the reference itself, and by
 * bench.py's reference arm.  Never part of the product.
 *
 * Layouts: matrices column-major; complex data interleaved (re, im) = std::complex<double> memory;
 * solutions leaf-major (tree.leaves order), point-minor (tensor order).  Field descriptors are the
 * oracle's (oracle_capi.h); SAMPLED fields are not supported here (the reference takes point functions).
 */
#ifndef HPS_REF_CAPI_H
#define HPS_REF_CAPI_H

#include "oracle_capi.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* ref_last_error(void);
void ref_set_threads(int n); /* BLAS threads of the shim (Eigen's OpenMP GEMM in the reference build) */

/* uniform tree [lo,hi]^dim, depth L; variant 0 = DtN (HpsSolver<Real>), 1 = ItI (HpsSolver<Complex>).
 * SolverOptions: root_implicit_S, build_root_T (solver.hpp:17-22). */
void* ref_create(int dim, int p, int L, double lo, double hi, const oracle_term* terms, int n_terms,
                 const oracle_field* source, const oracle_field* source_imag, int variant, double eta,
                 int root_implicit, int build_root_T);
/* problem catalog (problems.cpp:255-268) on a uniform (adaptive = 0, depth L) or adaptive tree
 * (refine_adaptive(domain, {tol, p, refinement_fields}, max_depth), mesh.cpp:233), with the solver
 * options solve_problem sets (problems.cpp:383-388); keep_T = 1 drops free_T_after_merge so node T's
 * stay readable. */
void* ref_create_problem(const char* name, double k, unsigned seed, int p, int adaptive, int L, double tol,
                         int max_depth, int keep_T);
void ref_destroy(void* h);

int ref_build(void* h);
int ref_is_complex(void* h);
int ref_n_leaves(void* h);
int ref_n_nodes(void* h);
int ref_dim(void* h);
int ref_p(void* h);
int ref_root_bsize(void* h);
int ref_top_D_size(void* h);
int ref_n_unresolved(void* h);
/* tree export: per node depth, parent, n_children, children[8], box lo[3]/hi[3], anchor[3]; leaves (DFS) */
int ref_tree(void* h, int* depth, int* parent, int* n_children, int* children, double* lo, double* hi,
             long long* anchor, int* leaves);
int ref_root_points(void* h, double* xyz);
int ref_leaf_points(void* h, double* xyz);
/* problem handles: sample_boundary_data(solver, prob) (problems.cpp:328-353) */
int ref_sample_root_data(void* h, double* g);
int ref_solve(void* h, const double* g_root, double* u, double* leaf_g);
int ref_solve_radiation(void* h, double* u);
/* leaf_f: n_leaves x p^dim samples (complex interleaved for ItI); radiation = RootBC::radiation */
int ref_solve_new_source(void* h, const double* leaf_f, int radiation, const double* g_root, double* u);
int ref_get_leaf(void* h, int ord, double* Y, double* v, double* T, double* hh);
int ref_node_sizes(void* h, int id, int* n_ext, int* n_int);
int ref_get_node(void* h, int id, double* S, double* gtilde, double* T, double* hh);
/* problem handles with an exact solution: error_report(field(u), prob.exact) (problems.cpp:270-293) */
int ref_error_report(void* h, const double* u, double* rel_linf, double* rel_l2);
double ref_min_rcond(void* h);
int ref_any_ill_conditioned(void* h);
void ref_times(void* h, double* t_build_s, double* t_solve_s);
/* the reference's end-to-end driver solve_problem (problems.cpp:360-422); out[8] =
 * {rel_linf, rel_l2, n_leaves, N, top_D_size, tree_depth, t_build_s, t_solve_s} */
int ref_solve_problem(const char* name, double k, unsigned seed, int p, int adaptive, int L, double tol,
                      int max_depth, double* out);

/* Bounded, extrapolated sample of the reference's full build + solve of a uniform 2D DtN problem
 * (bench.py's reference arm).  The tree of depth L is split at depth L-m:
 *   - one depth-(L-m) subtree is built and solved end to end by the reference (an HpsSolver over that
 *     subtree's box, m levels, the same operator terms and source); the other 4^(L-m) - 1 subtrees cost the
 *     same (uniform tree, identical shapes);
 *   - for every depth d < L-m, one reference merge_node (merge.cpp:486-494) on four children of the true
 *     size (child T/h synthetic: dense LU / GEMM time does not depend on the values) and the downward
 *     propagate step of that node (solver.cpp:199-212) are timed; there are 4^d such nodes.
 * out[0..3] = {estimated seconds of the full step, t_sub_build, t_sub_solve, leaves in the subtree};
 * out[4 + 2d], out[5 + 2d] = {t_merge(d), t_propagate(d)} for d = 0 .. L-m-1. */
int ref_bench_sample(int p, int L, int m, double lo, double hi, const oracle_term* terms, int n_terms,
                     const oracle_field* source, int root_implicit, double* out);

/* the reference's output formats: mesh_to_json (mesh.cpp:435-463) into buf (returns the length, -1 on error;
 * the text is written only when it fits), dump_solution (downpass.cpp:108-143) of solution u */
long long ref_mesh_json(void* h, char* buf, long long cap);
int ref_dump_solution(void* h, const double* u, const char* json_path, const char* bin_path, const char* tree_ref);

#ifdef __cplusplus
}
#endif
#endif
