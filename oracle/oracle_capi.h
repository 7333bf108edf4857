/* oracle_capi.h -- TEST INFRASTRUCTURE ONLY.
 *
 * ctypes-facing C API of the CPU oracle (hps_oracle.cpp), a restatement of the
 * reference HPS hot path.  Loaded only by tests/, __graft_entry__.smoke() and
 * bench.py's CPU-baseline / --impl reference legs, always as the checker or
 * the timed CPU baseline, never as part of the B200 product.
 *
 * Field descriptors mirror the product's hpsg_field (include/hps_cuda.h) so a
 * test can hand both sides the same problem; they are evaluated here by an
 * independent implementation.
 */
#ifndef HPS_ORACLE_CAPI_H
#define HPS_ORACLE_CAPI_H

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORACLE_FIELD_CONST = 0,           /* c0 */
  ORACLE_FIELD_BUMPS = 1,           /* c0 + c1 * sum_j exp(-c2 |x-z_j|^2) */
  ORACLE_FIELD_PLANE_SIN = 2,       /* c0 * sin(c1 x1 + c2 x2 + c3 x3 + c4) */
  ORACLE_FIELD_PLANE_COS = 3,       /* c0 * cos(c1 x1 + c2 x2 + c3 x3 + c4) */
  ORACLE_FIELD_BUMPS_SIN = 4,       /* c0 * sum_j exp(-c2 |x-z_j|^2) * sin(c3 x1 + c4 x2 + c5 x3 + c6) */
  ORACLE_FIELD_POISSON2D_SRC = 5,   /* manufactured source of proj/src/problems.cpp:62-66 */
  ORACLE_FIELD_SAMPLED = 6,         /* samples[leaf * p^d + pt], leaf order */
  ORACLE_FIELD_BUMPS_GRAD = 7,      /* d/dx_a of BUMPS (a = c3) */
  ORACLE_FIELD_DIVGRAD_SRC = 8      /* div(eps grad u), eps = BUMPS, u = prod sin(c3 x_k + c4) */
};

typedef struct {
  int kind;
  int n_centers;
  double c[8];
  const double* centers; /* n_centers x 3 */
  const double* samples; /* n_leaves x p^dim */
} oracle_field;

typedef struct {
  int role; /* 0 laplacian, 1 gradient, 2 zeroth, 3 second_order (local_solve.hpp:18) */
  int axis, axis2;
  oracle_field field;
} oracle_term;

const char* oracle_last_error(void);
int oracle_blas_available(void);
void oracle_set_threads(int n);

/* std::mt19937_64(seed) + uniform_real_distribution(-0.5,0.5), as in
 * proj/src/problems.cpp:126-141 (2D) / :240-249 (3D). out: n x 3 */
void oracle_bump_centers(unsigned long long seed, int n, int dim, double* out);

/* spectral / mesh known-answer helpers */
void oracle_cheb_lobatto(int p, double* out);
void oracle_cheb_weights(int p, double* out);
int oracle_gauss(int q, double* nodes, double* weights);
void oracle_diff_matrix(int p, double* out); /* p x p col-major */
int oracle_interp_matrix(const double* src, int n, const double* dst, int m, double* out);
int oracle_dtn_ops(int dim, int p, double side, double* P, double* Q, int* P_rows, int* P_cols,
                   int* Q_rows, int* Q_cols); /* pass NULL P/Q to query sizes */
int oracle_index_sets(int p, int dim, int* interior, int* exterior);
void oracle_leaf_cheb_points(const double* lo, const double* hi, int p, int dim, double* out);
void oracle_gauss_boundary_points(const double* lo, const double* hi, int q, int dim, double* out);
int oracle_face_projection(int q, double* refine, double* coarsen);
int oracle_refinement_interpolant(int p, double* out);
int oracle_tree_info(int dim, int L, int p, const double* lo, const double* hi, int* n_nodes, int* n_leaves,
                     long long* total_points, int* leaf_ids, int* node_depth, int* node_parent);

/* solver handle */
void* oracle_create(int dim, int p, int L, double lo, double hi, const oracle_term* terms, int n_terms,
                    const oracle_field* source, int literal_sign, int root_implicit, int parallel);
void oracle_destroy(void* h);
int oracle_build(void* h);
int oracle_n_leaves(void* h);
int oracle_n_nodes(void* h);
int oracle_root_bsize(void* h);
int oracle_root_points(void* h, double* xyz);
int oracle_leaf_points(void* h, double* xyz);
int oracle_discretize(void* h, int ord, double* lmat, double* f);
int oracle_solve(void* h, const double* g_root, double* u, double* leaf_g);
int oracle_get_leaf(void* h, int ord, double* Y, double* v, double* T, double* hh);
int oracle_node_sizes(void* h, int id, int* n_ext, int* n_int);
int oracle_get_node(void* h, int id, double* S, double* gtilde, double* T, double* hh);
int oracle_level_nodes(void* h, int depth, int* ids);
double oracle_min_rcond(void* h);
void oracle_times(void* h, double* t_leaf, double* t_merge);

#ifdef __cplusplus
}
#endif
#endif
