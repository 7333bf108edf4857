// ctx_internal.cuh -- the solver context behind the C-ABI (include/hps_cuda.h), shared by hps_ctx.cu
// (uniform trees, parts, ItI) and general.cu (general / adaptive trees).  Not part of the ABI.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <memory>
#include <string>
#include <vector>

#include "../../include/hps_cuda.h"
#include "gemm.cuh"
#include "geometry.hpp"
#include "hps_kernels.cuh"
#include "lu.cuh"
#include "gemv.cuh"

namespace hpsctx {

struct CudaError {
  cudaError_t e;
  std::string where;
};
struct HpsError {
  int code;
  std::string msg;
};

inline void ck(cudaError_t e, const char* where) {
  if (e != cudaSuccess) throw CudaError{e, where};
}

// Footprint estimation (hpsg_estimate_bytes): while set, DevBuf::alloc and the uploads only count
// bytes -- the context is created through the normal path without touching device memory.
extern thread_local bool g_dry_alloc;

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr, o.bytes = 0; }
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  void alloc(size_t b, size_t* total) {
    if (g_dry_alloc) {
      if (total) *total += b;
      return;
    }
    if (b <= bytes && p) return;
    if (total) *total -= bytes;
    release();
    if (b == 0) return;
    cudaError_t e = cudaMalloc(&p, b);
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw HpsError{HPSG_ERR_OOM, hpsg::fmt("cudaMalloc(%.3f GB) failed: %s", b / 1e9, cudaGetErrorString(e))};
    }
    bytes = b;
    if (total) *total += b;
  }
  double* d() const { return static_cast<double*>(p); }
  int* i() const { return static_cast<int*>(p); }
};

template <class T>
void upload(DevBuf& b, const std::vector<T>& v, size_t* total, cudaStream_t st) {
  b.alloc(v.size() * sizeof(T), total);
  if (!v.empty() && !g_dry_alloc)
    ck(cudaMemcpyAsync(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st), "upload");
}

struct Level {
  int d = 0;
  long long nodes = 0;
  hpsg::MergeTables mt;
  int n_int = 0, n_ext = 0, child_nb = 0;
  DevBuf MD, piv, stats;  // [D | h_int | C] -> [LU | x_h | X]
  DevBuf AH;              // [h | T] of the level's nodes (input of level d-1); unused at the root
  DevBuf md_src, b_src, ah_src, down;
  // block-sparse Schur product: exterior section e only couples to the interfaces of its own
  // child (B_{e,i} = 0 otherwise), as contiguous interface runs {e, first interface, count}
  std::vector<std::array<int, 3>> schur_runs;
  // Schur rows of sections on the domain boundary (skips_boundary_rows): per run, the nodes whose rows are
  // formed in the build (run_off/run_cnt into run_map) and the rest (rest_off/rest_cnt), formed on request;
  // ah_mask[node][section] = 1 on the boundary.  t_partial: those rows not formed yet
  DevBuf run_map, ah_mask;
  std::vector<int> run_off, run_cnt, rest_off, rest_cnt;
  bool t_partial = false;
  hpsg::ItiMergeTables it;  // ItI variant: block copies + real-equivalent scatter table
  DevBuf iblocks;
  int iti_nblocks = 0;
  long long strideMD() const { return (long long)n_int * (n_int + 1 + n_ext); }
  long long strideAH() const { return (long long)n_ext * (1 + n_ext); }
};

struct GenState;  // general-tree plan and buffers (general.cu)
struct GenDeleter {
  void operator()(GenState* g) const;
};

}  // namespace hpsctx

struct hpsg_ctx {
  using DevBuf = hpsctx::DevBuf;
  using Level = hpsctx::Level;
  std::string err;
  int dev = 0;
  cudaStream_t st = nullptr;
  bool own_stream = true;
  cudaEvent_t ev[8] = {};
  cudaEvent_t lev_ev[25] = {};  // merge level boundaries
  cudaStream_t gst = nullptr;   // merge gathers of B and [h_ext | A], overlapped with the level's LU
  cudaEvent_t gev[2] = {};      // [0]: main stream up to the level, [1]: those gathers done
  hpsg_tree tree{};
  hpsg_part part{};  // (0, 0, L) for the whole tree
  bool iti = false;  // ItI variant (real-equivalent complex)
  bool root_T = false;  // ItI radiation closure: the root forms [h|T] and factors T
  DevBuf radM, radPiv, radStats;  // [T_root | -h_root] -> [LU | g_rad]
  DevBuf itiW;                    // ItI merges: [W | X_top - D12 X_bot] of one level
  hpsk::DevField source_im{};
  int has_source_im = 0;
  hpsg::ItiLeafOperators iops;
  DevBuf iGr, iGi, iP, iQHs;
  hpsg_options opts{};
  hpsg::UniformTree T;
  hpsg::LeafOperators ops;
  size_t dev_bytes = 0;
  // problem
  int nterms = 0;
  hpsk::DevTerm terms[hpsk::kMaxTerms]{};
  hpsk::DevField source{};
  int has_source = 0;
  std::vector<std::unique_ptr<DevBuf>> field_bufs;
  // operators
  DevBuf leaf_box, cheb, Dm, D2m, interior, exterior, P, Qi, ZQeP;
  // leaf stage
  DevBuf leafM, leafE, leafPiv, leafStats, leafBad, leafHT;
  DevBuf leafYv, leafScratch;  // fused leaf path
  bool fused = false;
  int fused_grid = 0;
  // fast-diagonalisation leaf path (leaf_fdm.cu): eligible operators, 1D eigendecomposition, fallback flag
  bool fdm = false;
  int fdm_grid = 0;
  double fdm_lap = 0.0, fdm_qds = 0.0;
  DevBuf fdmV, fdmVinv, fdmA, fdmLam, fdmFail, fdmQG, fdmQd, fdmRtab, fdmRhat;
  bool fdm_prepped = false;
  DevBuf itiGire, itiGiim, itiGere, itiGeim, itiGAt, itiGAb, itiPc, fdmPid, itiPos;  // ItI block elimination operands  // fdmFail: count + list of non-converged leaves
  double* yv = nullptr;        // [v_i | Y_i] of leaf 0 (ni x (1+nb), ld ni)
  long long yv_stride = 0;
  // merges
  std::vector<Level> lv;  // index d = 0..L-1
  DevBuf Bscratch;
  // new-source pass (keep_factors): per-leaf RHS -> v, leaf h, per level y = D^-1 h_int and node h
  int src_nrhs = 0;
  DevBuf srcF, srcR, srcH;
  std::vector<std::unique_ptr<DevBuf>> srcY, srcHn;
  // solve workspace
  int ws_nrhs = 0;
  std::vector<std::unique_ptr<DevBuf>> G, GI;
  DevBuf Ui, Ue, g_in, u_out, lg_out, gemv_scratch;
  bool built = false;
  std::vector<char> cut_set;  // cut part: which input [h|T] have been provided
  hpsg_stats stats{};
  int launches = 0;
  hpsk::LuWorkspace luws;  // batched-LU scratch, counted in dev_bytes (lu.cuh)
  std::unique_ptr<hpsctx::GenState, hpsctx::GenDeleter> gen;  // set for general (adaptive) trees

  long long strideLeafM() const { return (long long)ops.ni * (ops.ni + 1 + ops.nb); }
  // [h|T] per part leaf: a real leaf (nb x (1+nb)) or, for a cut part, an input node
  int leaf_nb() const { return T.cut ? lv[T.L - 1].child_nb : ops.nb; }
  // leading dimension of the leaves' [1; g] columns in the solve: 1 + nb rounded up to even for leaf-owning
  // contexts (16-byte aligned columns: the leaf products' B operand is TMA-legal), 1 + nb for cut inputs
  long long ldG_leaf() const { return T.cut ? 1 + leaf_nb() : (2 + (long long)leaf_nb()) & ~1LL; }
  long long strideLeafHT() const { return (long long)leaf_nb() * (1 + leaf_nb()); }
  // the merge at part depth d is the reference's root merge (no T/h, optional implicit S)
  bool global_root(int d) const { return d == 0 && T.root_depth == 0; }
  // the merge at part depth d forms the node's [h|T] (every merge but the root, unless build_root_T)
  bool forms_T(int d) const { return !global_root(d) || root_T; }
};


namespace hpsctx {
// shared helpers (defined in hps_ctx.cu)
void gemm(hpsg_ctx* c, const hpsk::GemmArgs& g);
void matvecs(hpsg_ctx* c, const hpsk::GemmArgs& g);
int lu_launches(int n, int m, bool factor);
hpsk::DevField make_dev_field(hpsg_ctx* c, const hpsg_field& f, bool is_source,
                              std::vector<std::unique_ptr<DevBuf>>* scratch = nullptr);
// general (adaptive) trees (general.cu)
void gen_setup(hpsg_ctx* c, const hpsg_tree_desc* t);  // plan + shared operators
void gen_alloc(hpsg_ctx* c);                            // buffers (after the fields)
long long gen_n_leaves(const hpsg_ctx* c);
std::vector<int> gen_leaf_group_order(const hpsg_ctx* c);  // leaf ordinals, leaf-group-major
void gen_build(hpsg_ctx* c);
void gen_solve(hpsg_ctx* c, const double* d_g, int nrhs, double* d_u, double* d_leaf_g);
std::vector<double> gen_root_points(const hpsg_ctx* c);
std::vector<double> gen_leaf_points(const hpsg_ctx* c);
}  // namespace hpsctx
