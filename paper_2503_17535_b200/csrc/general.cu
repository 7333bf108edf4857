// general.cu -- HPS build + solve on a GENERAL tree (adaptive, level-restricted octrees; any uniform tree)
// behind hpsg_create_tree.  Plan: tree_general.hpp.  Reference path:
//   build_leaf loop           (solver.cpp:44-65, local_solve.cpp:111-143)  -> per leaf-depth group: the
//                              batched leaf path (assembly kernel, R = -L_ie P, batched LU, [h|T] GEMM)
//   merge_internal by depth   (solver.cpp:99-151, merge.cpp:183-324)       -> per (depth, child-layout) group:
//                              child projections [h|T]' = R [h|T] diag(1, E) (two DMMA GEMMs, only children
//                              with a finer interface face), block gather of [D | h_int | C], B, [h_ext | A],
//                              batched LU of [D | h_int | C], Schur GEMM [h|T] = [h_ext|A] - B [x_h|X]
//   propagate / reconstruct   (solver.cpp:188-252)                          -> per group g_int GEMV, scatter with
//                              the undo-projections E (child_maps), per leaf group u = [v|Y][1;g], P g.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstring>

#include "ctx_internal.cuh"
#include "leaf_common.cuh"
#include "tree_general.hpp"

using hpsk::BatchedMat;
using hpsk::GemmArgs;

namespace hpsctx {

namespace {

struct DevBlock {  // hpsg::BlockCopyG on the device
  int dst, dr, dc, child, sr, sc, rows, cols;
};
struct DevDown {   // hpsg::DownCopy on the device
  int child, dst_off, dst_len, src_int, src_off, src_len, E_off;
};

// [D | h_int | C], B, [h_ext | A] += blocks of the (projected) children; one pass never writes an
// entry twice, the second pass adds the other child's contribution of every interface row.
struct GenGatherArgs {
  const DevBlock* blocks;
  int nblocks;
  const double* const* child;  // node * nchild + slot -> the child's (projected) [h | T]
  const int* child_ld;         // per slot
  int nchild;
  double* dst[3];
  long long ld[3], stride[3];
};
__global__ void gen_gather_kernel(const GenGatherArgs a) {
  const long long node = blockIdx.x;
  const DevBlock b = a.blocks[blockIdx.y];
  const double* src = a.child[node * a.nchild + b.child];
  const long long lds = a.child_ld[b.child];
  double* dst = a.dst[b.dst] + node * a.stride[b.dst];
  const long long ldd = a.ld[b.dst];
  for (long long e = threadIdx.x; e < (long long)b.rows * b.cols; e += blockDim.x) {
    const int r = int(e % b.rows), c = int(e / b.rows);
    dst[(long long)(b.dc + c) * ldd + b.dr + r] += src[(long long)(b.sc + c) * lds + b.sr + r];
  }
}

// copy child [h | T] (nb x (1 + nb), contiguous) of every node of a group into a strided staging batch
__global__ void gen_stage_kernel(const double* const* child, int nchild, int slot, long long elems, double* out) {
  const long long node = blockIdx.x;
  const double* src = child[node * nchild + slot];
  double* dst = out + node * elems;
  for (long long e = (long long)blockIdx.y * blockDim.x + threadIdx.x; e < elems; e += (long long)gridDim.y * blockDim.x)
    dst[e] = src[e];
}

// propagate's split into the children (solver.cpp:213-222): child column r of G = [1; g_child]
struct GenScatterArgs {
  const DevDown* down;
  int ndown, nchild, nrhs;
  const double* Gp;        // parent [1; g] columns, ld ldGp, node stride sGp
  long long ldGp, sGp;
  const double* GI;        // g_int, ld ldGI, node stride sGI
  long long ldGI, sGI;
  double* const* childG;   // node * nchild + slot -> child G base (column r at + r * ld)
  const int* childG_ld;    // per slot
  const double* E;         // undo-projection matrices
};
__global__ void gen_scatter_kernel(const GenScatterArgs a) {
  const long long node = blockIdx.x;
  const DevDown d = a.down[blockIdx.y];
  double* cg = a.childG[node * a.nchild + d.child];
  const long long ldc = a.childG_ld[d.child];
  for (int r = 0; r < a.nrhs; ++r) {
    const double* src = d.src_int ? a.GI + node * a.sGI + (long long)r * a.ldGI + d.src_off
                                  : a.Gp + node * a.sGp + (long long)r * a.ldGp + 1 + d.src_off;
    double* dst = cg + (long long)r * ldc + 1 + d.dst_off;
    if (d.dst_off == 0 && threadIdx.x == 0) cg[(long long)r * ldc] = 1.0;  // the leading 1 (applies gtilde)
    for (int t = threadIdx.x; t < d.dst_len; t += blockDim.x) {
      if (d.E_off < 0) {
        dst[t] = src[t];
      } else {
        const double* E = a.E + d.E_off;
        double s = 0.0;
        for (int j = 0; j < d.src_len; ++j) s += E[(long long)j * d.dst_len + t] * src[j];
        dst[t] = s;
      }
    }
  }
}

// u[r][ord[i]] (tensor order) from the interior / exterior pieces of leaf i of a group
__global__ void gen_leaf_output_kernel(double* u, long long n_leaves_total, const int* ord, int nl, int npts, int ni,
                                       int ne, int nrhs, const int* interior, const int* exterior, const double* Ui,
                                       const double* Ue) {
  const long long total = (long long)nl * nrhs * npts;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int k = int(e % (ni + ne));
    const long long lr = e / npts;
    const int i = int(lr % nl), r = int(lr / nl);
    double v;
    int pt;
    if (k < ni) {
      pt = interior[k];
      v = Ui[((long long)i * nrhs + r) * ni + k];
    } else {
      pt = exterior[k - ni];
      v = Ue[((long long)i * nrhs + r) * ne + (k - ni)];
    }
    u[((long long)r * n_leaves_total + ord[i]) * npts + pt] = v;
  }
}

}  // namespace

struct GLeaf {  // one leaf group (leaves of one depth)
  hpsg::LeafGroup g;
  hpsg::LeafOperators ops;
  int n = 0;
  DevBuf box, Qi, ZQeP, ord, M, E, piv, stats, bad, HT, G;
  long long strideM() const { return (long long)ops.ni * (ops.ni + 1 + ops.nb); }
  long long strideHT() const { return (long long)ops.nb * (1 + ops.nb); }
};
struct GMerge {  // one merge group
  hpsg::MergeGroup g;
  int n = 0;
  DevBuf MD, piv, stats, AH, blocks, down, Edata, cptr, cld, hptr, gptr, gld, G, GI;
  DevBuf R[8], Ehat[8];
  long long pproj_off[8] = {};  // offset of slot k's projected children in the shared Pproj scratch
  long long strideMD() const { return (long long)g.n_int * (g.n_int + 1 + g.n_ext); }
  long long strideAH() const { return (long long)g.n_ext * (1 + g.n_ext); }
};
struct GenState {
  hpsg::GeneralPlan plan;
  std::vector<GLeaf> leaves;
  std::vector<std::vector<GMerge>> merges;  // [depth][group]
  DevBuf Bscr, CH, X, Pproj, Ui, Ue;
  int ws_nrhs = 0;
  bool implicit_root = false;
};

void GenDeleter::operator()(GenState* g) const { delete g; }

namespace {

// where a node's [h | T] and G live
const double* home_HT(const GenState& s, int id) {
  const auto& h = s.plan.home[id];
  if (h[0] == 0) return s.leaves[h[1]].HT.d() + h[2] * s.leaves[h[1]].strideHT();
  const GMerge& m = s.merges[s.plan.tree.depth[id]][h[1]];
  return m.AH.d() + h[2] * m.strideAH();
}
double* home_G(const GenState& s, int id, int nrhs) {
  const auto& h = s.plan.home[id];
  if (h[0] == 0) return s.leaves[h[1]].G.d() + (long long)h[2] * (1 + s.leaves[h[1]].ops.nb) * nrhs;
  const GMerge& m = s.merges[s.plan.tree.depth[id]][h[1]];
  return m.G.d() + (long long)h[2] * (1 + m.g.n_ext) * nrhs;
}

template <class T>
void upload_vec(DevBuf& b, const std::vector<T>& v, hpsg_ctx* c) {
  upload(b, v, &c->dev_bytes, c->st);
}

}  // namespace

void gen_setup(hpsg_ctx* c, const hpsg_tree_desc* td) {
  if (!td || td->n_nodes < 1 || !td->depth || !td->n_children || !td->children || !td->lo || !td->hi)
    throw HpsError{HPSG_ERR_INVALID, "hpsg_create_tree: incomplete tree descriptor"};
  if (c->opts.variant != HPSG_VARIANT_DTN)
    throw HpsError{HPSG_ERR_INVALID, "hpsg_create_tree: general trees use the DtN variant (merge_iti is uniform 2D)"};
  if (c->opts.keep_factors) throw HpsError{HPSG_ERR_INVALID, "hpsg_create_tree: keep_factors is not on this path"};
  hpsg::GTree t;
  t.dim = td->dim;
  t.p = td->p;
  const int n = td->n_nodes;
  t.depth.assign(td->depth, td->depth + n);
  t.nch.assign(td->n_children, td->n_children + n);
  t.child.resize(n);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < 8; ++k) t.child[i][k] = td->children[8 * i + k];
  t.lo.assign(td->lo, td->lo + 3 * n);
  t.hi.assign(td->hi, td->hi + 3 * n);
  if (t.p < 4) throw HpsError{HPSG_ERR_INVALID, "build_uniform_tree: p must be >= 4"};
  if ((t.dim == 2 && t.p > 22) || (t.dim == 3 && t.p > 8))
    throw HpsError{HPSG_ERR_INVALID, "hpsg_create_tree: p^dim > 512 not supported by the leaf kernel"};
  auto gs = std::unique_ptr<GenState, GenDeleter>(new GenState);
  gs->implicit_root = c->opts.root_implicit_S != 0;
  try {
    gs->plan = hpsg::make_general_plan(std::move(t), gs->implicit_root);
  } catch (const std::exception& e) {
    throw HpsError{HPSG_ERR_INVALID, e.what()};
  }
  GenState& s = *gs;
  const hpsg::GTree& T = s.plan.tree;
  c->tree.dim = T.dim;
  c->tree.p = T.p;
  c->tree.L = T.max_depth();
  c->tree.lo = T.lo[0];
  c->tree.hi = T.hi[0];
  c->ops = hpsg::make_leaf_operators(T.dim, T.p, T.hi[0] - T.lo[0]);  // shared pieces: D, P, index sets
  const hpsg::LeafOperators& o = c->ops;
  upload(c->cheb, hpsg::cheb_nodes(T.p), &c->dev_bytes, c->st);
  upload(c->Dm, o.D.a, &c->dev_bytes, c->st);
  upload(c->D2m, o.D2.a, &c->dev_bytes, c->st);
  upload(c->interior, o.interior, &c->dev_bytes, c->st);
  upload(c->exterior, o.exterior, &c->dev_bytes, c->st);
  upload(c->P, o.P.a, &c->dev_bytes, c->st);
  // levels of the stats record
  c->stats.n_leaves = int(T.leaves.size());
  c->stats.n_points = (long long)T.leaves.size() * o.n;
  c->stats.root_bsize = s.plan.root_nb;
  c->stats.top_D_size = s.plan.top_D;
  c->stats.tree_depth = T.max_depth();
  c->stats.min_rcond = 1.0;
  c->gen = std::move(gs);
}

// allocation after the fields are known (hpsg_create_tree)
void gen_alloc(hpsg_ctx* c) {
  GenState& s = *c->gen;
  const hpsg::GTree& T = s.plan.tree;
  size_t* tot = &c->dev_bytes;
  // leaf groups
  s.leaves.resize(s.plan.leaf_groups.size());
  for (size_t gi = 0; gi < s.leaves.size(); ++gi) {
    GLeaf& L = s.leaves[gi];
    L.g = s.plan.leaf_groups[gi];
    L.n = int(L.g.leaves.size());
    L.ops = hpsg::make_leaf_operators(T.dim, T.p, L.g.side);
    std::vector<double> box;
    std::vector<int> ord;
    for (int id : L.g.leaves) {
      for (int k = 0; k < 3; ++k) box.push_back(T.lo[3 * id + k]);
      for (int k = 0; k < 3; ++k) box.push_back(T.hi[3 * id + k]);
      ord.push_back(T.leaf_ord[id]);
    }
    upload_vec(L.box, box, c);
    upload_vec(L.ord, ord, c);
    upload(L.Qi, L.ops.Qi.a, tot, c->st);
    std::vector<double> zq(size_t(L.ops.nb) * (1 + L.ops.nb), 0.0);  // [0 | Q_e P]
    for (int j = 0; j < L.ops.nb; ++j)
      for (int i = 0; i < L.ops.nb; ++i) zq[size_t(1 + j) * L.ops.nb + i] = L.ops.QeP(i, j);
    upload(L.ZQeP, zq, tot, c->st);
    L.M.alloc(size_t(L.n) * L.strideM() * 8, tot);
    L.E.alloc(size_t(L.n) * L.ops.ni * L.ops.ne * 8, tot);
    L.piv.alloc(size_t(L.n) * L.ops.ni * 4, tot);
    L.stats.alloc(size_t(L.n) * 3 * 8, tot);
    L.bad.alloc(size_t(L.n) * 4, tot);
    L.HT.alloc(size_t(L.n) * L.strideHT() * 8, tot);
    ck(hpsk::lu_workspace_reserve(c->luws, L.n, L.ops.ni, 1 + L.ops.nb, true, g_dry_alloc), "LU workspace");
  }
  // merge groups
  s.merges.clear();
  s.merges.resize(s.plan.merge_groups.size());
  size_t bmax = 0, chmax = 0, xmax = 0, pmax = 0;
  for (size_t d = 0; d < s.plan.merge_groups.size(); ++d) {
    s.merges[d].reserve(s.plan.merge_groups[d].size());
    for (const hpsg::MergeGroup& mg : s.plan.merge_groups[d]) {
      s.merges[d].emplace_back();
      GMerge& M = s.merges[d].back();
      M.g = mg;
      M.n = int(mg.nodes.size());
      if (mg.n_int > hpsk::bgetrf_max_n())
        throw HpsError{HPSG_ERR_INVALID, hpsg::fmt("interface matrix of size %d exceeds the batched LU limit %d",
                                                   mg.n_int, hpsk::bgetrf_max_n())};
      M.MD.alloc(size_t(M.n) * M.strideMD() * 8, tot);
      M.piv.alloc(size_t(M.n) * mg.n_int * 4, tot);
      M.stats.alloc(size_t(M.n) * 3 * 8, tot);
      if (!mg.root) {
        M.AH.alloc(size_t(M.n) * M.strideAH() * 8, tot);
        bmax = std::max(bmax, size_t(M.n) * mg.n_ext * mg.n_int * 8);
      }
      size_t psum = 0;
      for (int k = 0; k < mg.nchild; ++k) {
        if (!mg.proj[k]) continue;
        upload(M.R[k], mg.R[k].a, tot, c->st);
        upload(M.Ehat[k], mg.Ehat[k].a, tot, c->st);
        const size_t nb = mg.child_nb[k], nbp = mg.child_nbp[k];
        chmax = std::max(chmax, size_t(M.n) * nb * (1 + nb) * 8);
        xmax = std::max(xmax, size_t(M.n) * nb * (1 + nbp) * 8);
        M.pproj_off[k] = (long long)(psum / 8);
        psum += size_t(M.n) * nbp * (1 + nbp) * 8;
      }
      pmax = std::max(pmax, psum);
      std::vector<int> raw;
      for (const auto& b : mg.blocks) raw.insert(raw.end(), {b.dst, b.dr, b.dc, b.child, b.sr, b.sc, b.rows, b.cols});
      upload_vec(M.blocks, raw, c);
      std::vector<int> dw;
      for (const auto& x : mg.down)
        dw.insert(dw.end(), {x.child, x.dst_off, x.dst_len, x.src_int, x.src_off, x.src_len, x.E_off});
      upload_vec(M.down, dw, c);
      upload(M.Edata, mg.Edata.empty() ? std::vector<double>{0.0} : mg.Edata, tot, c->st);
      const int m = (mg.root && s.implicit_root) ? 1 : 1 + mg.n_ext;
      ck(hpsk::lu_workspace_reserve(c->luws, M.n, mg.n_int, m, true, g_dry_alloc), "LU workspace");
    }
  }
  s.Bscr.alloc(bmax, tot);
  s.CH.alloc(chmax, tot);
  s.X.alloc(xmax, tot);
  s.Pproj.alloc(pmax, tot);
  if (g_dry_alloc) return;
  // child [h | T] pointer tables (projected slots point into Pproj)
  for (auto& lvl : s.merges)
    for (GMerge& M : lvl) {
      std::vector<const double*> ptr(size_t(M.n) * M.g.nchild);
      std::vector<int> ld(M.g.nchild);
      for (int k = 0; k < M.g.nchild; ++k) ld[k] = M.g.proj[k] ? M.g.child_nbp[k] : M.g.child_nb[k];
      for (int i = 0; i < M.n; ++i)
        for (int k = 0; k < M.g.nchild; ++k) {
          const int cid = T.child[M.g.nodes[i]][k];
          const long long nbp = M.g.child_nbp[k];
          ptr[size_t(i) * M.g.nchild + k] =
              M.g.proj[k] ? s.Pproj.d() + M.pproj_off[k] + (long long)i * nbp * (1 + nbp) : home_HT(s, cid);
        }
      M.cptr.alloc(ptr.size() * sizeof(void*), tot);
      ck(cudaMemcpyAsync(M.cptr.p, ptr.data(), ptr.size() * sizeof(void*), cudaMemcpyHostToDevice, c->st), "ptr H2D");
      upload_vec(M.cld, ld, c);
      std::vector<const double*> homes(size_t(M.n) * M.g.nchild);  // the children's own [h | T]
      for (int i = 0; i < M.n; ++i)
        for (int k = 0; k < M.g.nchild; ++k) homes[size_t(i) * M.g.nchild + k] = home_HT(s, T.child[M.g.nodes[i]][k]);
      M.hptr.alloc(homes.size() * sizeof(void*), tot);
      ck(cudaMemcpyAsync(M.hptr.p, homes.data(), homes.size() * sizeof(void*), cudaMemcpyHostToDevice, c->st), "ptr");
    }
}

void gen_build(hpsg_ctx* c) {
  GenState& s = *c->gen;
  const hpsg::GTree& T = s.plan.tree;
  const int p = T.p;
  // ---- leaves, one batched pass per leaf depth (local_solve_dtn on every leaf)
  ck(cudaEventRecord(c->ev[0], c->st), "ev");
  for (GLeaf& L : s.leaves) {
    const hpsg::LeafOperators& o = L.ops;
    hpsk::LeafAsmArgs a{};
    a.dim = T.dim;
    a.p = p;
    a.n = o.n;
    a.ni = o.ni;
    a.ne = o.ne;
    a.nb = o.nb;
    a.nterms = c->nterms;
    a.scale = 2.0 / L.g.side;
    a.fsign = c->opts.literal_sign ? -1.0 : 1.0;
    for (int i = 0; i < c->nterms; ++i) a.terms[i] = c->terms[i];
    a.source = c->source;
    a.has_source = c->has_source;
    // sampled fields were uploaded leaf-group-major (hpsg_create_tree): offset to this group's block
    const long long goff = (long long)(&L - s.leaves.data());
    long long lead = 0;
    for (long long gi = 0; gi < goff; ++gi) lead += s.leaves[gi].n;
    for (int i = 0; i < c->nterms; ++i)
      if (a.terms[i].f.kind == HPSG_FIELD_SAMPLED) a.terms[i].f.samples += lead * o.n;
    if (a.has_source && a.source.kind == HPSG_FIELD_SAMPLED) a.source.samples += lead * o.n;
    a.leaf_box = L.box.d();
    a.cheb = c->cheb.d();
    a.D = c->Dm.d();
    a.D2 = c->D2m.d();
    a.interior = c->interior.i();
    a.exterior = c->exterior.i();
    a.M = L.M.d();
    a.strideM = L.strideM();
    a.E = L.E.d();
    a.strideE = (long long)o.ni * o.ne;
    a.bad_point = L.bad.i();
    hpsk::launch_leaf_assemble(a, L.n, c->st);
    ck(cudaGetLastError(), "leaf_assemble");
    GemmArgs g;  // R = -L_ie P
    g.m = o.ni;
    g.n = o.nb;
    g.k = o.ne;
    g.batch = L.n;
    g.A = L.E.d();
    g.lda = o.ni;
    g.sA = (long long)o.ni * o.ne;
    g.B = c->P.d();
    g.ldb = o.ne;
    g.sB = 0;
    g.D = L.M.d() + (long long)(o.ni + 1) * o.ni;
    g.ldd = o.ni;
    g.sD = L.strideM();
    g.alpha = -1.0;
    g.beta = 0.0;
    gemm(c, g);
    ck(hpsk::lu_stats_init(L.stats.d(), L.n, c->st), "stats init");
    ck(hpsk::bgetrf_aug(L.n, o.ni, 1 + o.nb, BatchedMat{L.M.d(), o.ni, L.strideM()}, L.piv.i(), L.stats.d(), c->luws,
                        c->st, false),
       "leaf bgetrf");
    c->launches += 2 + lu_launches(o.ni, 1 + o.nb, true);
    GemmArgs t;  // [h | T] = Q_i [v | Y_i] + [0 | Q_e P]
    t.m = o.nb;
    t.n = 1 + o.nb;
    t.k = o.ni;
    t.batch = L.n;
    t.A = L.Qi.d();
    t.lda = o.nb;
    t.sA = 0;
    t.B = L.M.d() + (long long)o.ni * o.ni;
    t.ldb = o.ni;
    t.sB = L.strideM();
    t.C = L.ZQeP.d();
    t.ldc = o.nb;
    t.sC = 0;
    t.D = L.HT.d();
    t.ldd = o.nb;
    t.sD = L.strideHT();
    t.alpha = 1.0;
    t.beta = 1.0;
    gemm(c, t);
  }
  ck(cudaEventRecord(c->ev[1], c->st), "ev");
  // leaf status words (check_factorization, local_solve.cpp:90-107; non-finite samples, :56-61)
  double mr = 1.0;
  for (GLeaf& L : s.leaves) {
    std::vector<int> bad(L.n);
    std::vector<double> st(size_t(L.n) * 3);
    ck(cudaMemcpyAsync(bad.data(), L.bad.p, bad.size() * 4, cudaMemcpyDeviceToHost, c->st), "bad D2H");
    ck(cudaMemcpyAsync(st.data(), L.stats.p, st.size() * 8, cudaMemcpyDeviceToHost, c->st), "stats D2H");
    ck(cudaStreamSynchronize(c->st), "leaf sync");
    for (int i = 0; i < L.n; ++i) {
      if (bad[i] != INT_MAX)
        throw HpsError{HPSG_ERR_NONFINITE,
                       hpsg::fmt("discretize_operator: non-finite coefficient sample on leaf %d (point %d)",
                                 L.g.leaves[i], bad[i])};
      if (st[3 * i + 2] >= 0)
        throw HpsError{HPSG_ERR_SINGULAR_LEAF, hpsg::fmt("leaf %d: local_solve_dtn: singular factorization (zero pivot "
                                                         "at %d)", L.g.leaves[i], int(st[3 * i + 2]))};
      mr = std::min(mr, st[3 * i] / st[3 * i + 1]);
    }
  }
  c->stats.min_rcond = mr;
  c->stats.ill_conditioned = mr < 1e-12 ? 1 : 0;
  ck(cudaEventRecord(c->ev[2], c->st), "ev");
  // ---- merges, deepest depth first
  for (int d = int(s.merges.size()) - 1; d >= 0; --d) {
    for (GMerge& M : s.merges[d]) {
      const hpsg::MergeGroup& mg = M.g;
      const bool root = mg.root;
      // child projections [h|T]' = R [h|T] diag(1, E)
      for (int k = 0; k < mg.nchild; ++k) {
        if (!mg.proj[k]) continue;
        const long long nb = mg.child_nb[k], nbp = mg.child_nbp[k];
        // staging: the slot-k child [h|T] of every node of the group, as one strided batch
        const long long elems = nb * (1 + nb);
        const int gy = int(std::min<long long>(64, (elems + 255) / 256));
        gen_stage_kernel<<<dim3(M.n, gy), 256, 0, c->st>>>(static_cast<const double* const*>(M.hptr.p), mg.nchild, k,
                                                            elems, s.CH.d());
        ck(cudaGetLastError(), "stage");
        ++c->launches;
        GemmArgs x;  // X = [h|T] diag(1, E)
        x.m = int(nb);
        x.n = int(1 + nbp);
        x.k = int(1 + nb);
        x.batch = M.n;
        x.A = s.CH.d();
        x.lda = nb;
        x.sA = nb * (1 + nb);
        x.B = M.Ehat[k].d();
        x.ldb = 1 + nb;
        x.sB = 0;
        x.D = s.X.d();
        x.ldd = nb;
        x.sD = nb * (1 + nbp);
        gemm(c, x);
        GemmArgs y;  // [h|T]' = R X
        y.m = int(nbp);
        y.n = int(1 + nbp);
        y.k = int(nb);
        y.batch = M.n;
        y.A = M.R[k].d();
        y.lda = nbp;
        y.sA = 0;
        y.B = s.X.d();
        y.ldb = nb;
        y.sB = nb * (1 + nbp);
        y.D = s.Pproj.d() + M.pproj_off[k];
        y.ldd = nbp;
        y.sD = nbp * (1 + nbp);
        gemm(c, y);
      }
      // [D | h_int | C], B, [h_ext | A]
      ck(cudaMemsetAsync(M.MD.p, 0, size_t(M.n) * M.strideMD() * 8, c->st), "MD zero");
      if (!root) {
        ck(cudaMemsetAsync(s.Bscr.p, 0, size_t(M.n) * mg.n_ext * mg.n_int * 8, c->st), "B zero");
        ck(cudaMemsetAsync(M.AH.p, 0, size_t(M.n) * M.strideAH() * 8, c->st), "AH zero");
      }
      GenGatherArgs ga{};
      ga.child = static_cast<const double* const*>(M.cptr.p);
      ga.child_ld = M.cld.i();
      ga.nchild = mg.nchild;
      ga.dst[0] = M.MD.d();
      ga.ld[0] = mg.n_int;
      ga.stride[0] = M.strideMD();
      ga.dst[1] = s.Bscr.d();
      ga.ld[1] = mg.n_ext;
      ga.stride[1] = (long long)mg.n_ext * mg.n_int;
      ga.dst[2] = root ? nullptr : M.AH.d();
      ga.ld[2] = mg.n_ext;
      ga.stride[2] = M.strideAH();
      const DevBlock* blocks = static_cast<const DevBlock*>(M.blocks.p);
      const int nb1 = mg.pass_split, nb2 = int(mg.blocks.size()) - mg.pass_split;
      if (nb1 > 0) {
        ga.blocks = blocks;
        ga.nblocks = nb1;
        gen_gather_kernel<<<dim3(M.n, nb1), 256, 0, c->st>>>(ga);
      }
      if (nb2 > 0) {
        ga.blocks = blocks + nb1;
        ga.nblocks = nb2;
        gen_gather_kernel<<<dim3(M.n, nb2), 256, 0, c->st>>>(ga);
      }
      ck(cudaGetLastError(), "gather");
      c->launches += 2 + (root ? 1 : 3);
      // LU of D with the right-hand sides [h_int | C] (merge.cpp:280-297)
      ck(hpsk::lu_stats_init(M.stats.d(), M.n, c->st), "stats init");
      const int m = (root && s.implicit_root) ? 1 : 1 + mg.n_ext;
      ck(hpsk::bgetrf_aug(M.n, mg.n_int, m, BatchedMat{M.MD.d(), mg.n_int, M.strideMD()}, M.piv.i(), M.stats.d(),
                          c->luws, c->st, root && s.implicit_root),
         "merge bgetrf");
      c->launches += 1 + lu_launches(mg.n_int, m, true);
      if (!root) {  // [h | T] = [h_ext | A] - B [x_h | X]
        GemmArgs g;
        g.m = mg.n_ext;
        g.n = 1 + mg.n_ext;
        g.k = mg.n_int;
        g.batch = M.n;
        g.A = s.Bscr.d();
        g.lda = mg.n_ext;
        g.sA = (long long)mg.n_ext * mg.n_int;
        g.B = M.MD.d() + (long long)mg.n_int * mg.n_int;
        g.ldb = mg.n_int;
        g.sB = M.strideMD();
        g.C = M.AH.d();
        g.ldc = mg.n_ext;
        g.sC = M.strideAH();
        g.D = M.AH.d();
        g.ldd = mg.n_ext;
        g.sD = M.strideAH();
        g.alpha = -1.0;
        g.beta = 1.0;
        gemm(c, g);
      }
    }
  }
  ck(cudaEventRecord(c->ev[3], c->st), "ev");
  ck(cudaStreamSynchronize(c->st), "merge sync");
  for (int d = int(s.merges.size()) - 1; d >= 0; --d)
    for (GMerge& M : s.merges[d]) {
      std::vector<double> st(size_t(M.n) * 3);
      ck(cudaMemcpy(st.data(), M.stats.p, st.size() * 8, cudaMemcpyDeviceToHost), "merge stats D2H");
      for (int i = 0; i < M.n; ++i)
        if (st[3 * i + 2] >= 0)
          throw HpsError{HPSG_ERR_SINGULAR_MERGE, hpsg::fmt("merge_dtn: singular interface matrix D (pivot %d) at node %d",
                                                            int(st[3 * i + 2]), M.g.nodes[i])};
    }
  c->stats.build_flops = s.plan.build_flops;
}

namespace {
void gen_solve_ws(hpsg_ctx* c, int nrhs) {
  GenState& s = *c->gen;
  if (s.ws_nrhs >= nrhs) return;
  size_t* tot = &c->dev_bytes;
  size_t uimax = 0, uemax = 0;
  for (GLeaf& L : s.leaves) {
    L.G.alloc(size_t(L.n) * (1 + L.ops.nb) * nrhs * 8, tot);
    uimax = std::max(uimax, size_t(L.n) * L.ops.ni * nrhs * 8);
    uemax = std::max(uemax, size_t(L.n) * L.ops.ne * nrhs * 8);
  }
  s.Ui.alloc(uimax, tot);
  s.Ue.alloc(uemax, tot);
  for (auto& lvl : s.merges)
    for (GMerge& M : lvl) {
      M.G.alloc(size_t(M.n) * (1 + M.g.n_ext) * nrhs * 8, tot);
      M.GI.alloc(size_t(M.n) * M.g.n_int * nrhs * 8, tot);
    }
  c->gemv_scratch.alloc(size_t(8) << 20, tot);
  if (s.implicit_root)
    ck(hpsk::lu_workspace_reserve(c->luws, 1, s.merges[0][0].g.n_int, nrhs, false, g_dry_alloc), "LU workspace");
  if (!g_dry_alloc) {
    const hpsg::GTree& T = s.plan.tree;
    for (auto& lvl : s.merges)
      for (GMerge& M : lvl) {
        std::vector<double*> ptr(size_t(M.n) * M.g.nchild);
        std::vector<int> ld(M.g.nchild);
        for (int k = 0; k < M.g.nchild; ++k) ld[k] = 1 + M.g.child_nb[k];
        for (int i = 0; i < M.n; ++i)
          for (int k = 0; k < M.g.nchild; ++k) ptr[size_t(i) * M.g.nchild + k] = home_G(s, T.child[M.g.nodes[i]][k], nrhs);
        M.gptr.alloc(ptr.size() * sizeof(void*), tot);
        ck(cudaMemcpyAsync(M.gptr.p, ptr.data(), ptr.size() * sizeof(void*), cudaMemcpyHostToDevice, c->st), "ptr H2D");
        upload(M.gld, ld, tot, c->st);
      }
    ck(cudaStreamSynchronize(c->st), "ws sync");
  }
  s.ws_nrhs = nrhs;
}
}  // namespace

void gen_solve(hpsg_ctx* c, const double* d_g, int nrhs, double* d_u, double* d_leaf_g) {
  GenState& s = *c->gen;
  if (d_leaf_g) throw HpsError{HPSG_ERR_INVALID, "hpsg_solve: leaf boundary data output is uniform-tree only"};
  gen_solve_ws(c, nrhs);
  if (s.ws_nrhs != nrhs) {  // the pointer tables encode the G column count
    s.ws_nrhs = 0;
    gen_solve_ws(c, nrhs);
  }
  const hpsg::GTree& T = s.plan.tree;
  GMerge& R = s.merges[0][0];
  hpsk::launch_pack_root(R.G.d(), d_g, R.g.n_ext, nrhs, c->st, 1.0);
  ++c->launches;
  for (size_t d = 0; d < s.merges.size(); ++d)
    for (GMerge& M : s.merges[d]) {
      const hpsg::MergeGroup& mg = M.g;
      const long long ldG = 1 + mg.n_ext, sG = ldG * nrhs, sGI = (long long)mg.n_int * nrhs;
      if (mg.root && s.implicit_root) {
        // g_int = -(x_h + D^-1 C g)   (solver.cpp:204-206)
        GemmArgs g;
        g.m = mg.n_int;
        g.n = nrhs;
        g.k = mg.n_ext;
        g.A = M.MD.d() + (long long)(mg.n_int + 1) * mg.n_int;
        g.lda = mg.n_int;
        g.B = M.G.d() + 1;
        g.ldb = ldG;
        g.D = M.GI.d();
        g.ldd = mg.n_int;
        g.alpha = 1.0;
        g.beta = 0.0;
        matvecs(c, g);
        ck(hpsk::bgetrs(1, mg.n_int, nrhs, BatchedMat{M.MD.d(), mg.n_int, M.strideMD()}, M.piv.i(),
                        BatchedMat{M.GI.d(), mg.n_int, sGI}, c->luws, c->st),
           "root getrs");
        c->launches += lu_launches(mg.n_int, nrhs, false);
        hpsk::launch_neg_add(M.GI.d(), M.MD.d() + (long long)mg.n_int * mg.n_int, mg.n_int, nrhs, mg.n_int, c->st);
        ++c->launches;
      } else {
        // g_int = S g + gtilde = -[x_h | X] [1; g]   (solver.cpp:207-208)
        GemmArgs g;
        g.m = mg.n_int;
        g.n = nrhs;
        g.k = 1 + mg.n_ext;
        g.batch = M.n;
        g.A = M.MD.d() + (long long)mg.n_int * mg.n_int;
        g.lda = mg.n_int;
        g.sA = M.strideMD();
        g.B = M.G.d();
        g.ldb = ldG;
        g.sB = sG;
        g.D = M.GI.d();
        g.ldd = mg.n_int;
        g.sD = sGI;
        g.alpha = -1.0;
        g.beta = 0.0;
        matvecs(c, g);
      }
      GenScatterArgs sa{};
      sa.down = static_cast<const DevDown*>(M.down.p);
      sa.ndown = int(mg.down.size());
      sa.nchild = mg.nchild;
      sa.nrhs = nrhs;
      sa.Gp = M.G.d();
      sa.ldGp = ldG;
      sa.sGp = sG;
      sa.GI = M.GI.d();
      sa.ldGI = mg.n_int;
      sa.sGI = sGI;
      sa.childG = static_cast<double* const*>(M.gptr.p);
      sa.childG_ld = M.gld.i();
      sa.E = M.Edata.d();
      gen_scatter_kernel<<<dim3(M.n, sa.ndown), 128, 0, c->st>>>(sa);
      ck(cudaGetLastError(), "scatter");
      ++c->launches;
    }
  // leaves: u_i = [v | Y_i][1; g],  u_e = P g   (solver.cpp:230-236)
  for (GLeaf& L : s.leaves) {
    const hpsg::LeafOperators& o = L.ops;
    const long long ldGL = 1 + o.nb, sGL = ldGL * nrhs;
    GemmArgs g;
    g.m = o.ni;
    g.n = nrhs;
    g.k = 1 + o.nb;
    g.batch = L.n;
    g.A = L.M.d() + (long long)o.ni * o.ni;
    g.lda = o.ni;
    g.sA = L.strideM();
    g.B = L.G.d();
    g.ldb = ldGL;
    g.sB = sGL;
    g.D = s.Ui.d();
    g.ldd = o.ni;
    g.sD = (long long)o.ni * nrhs;
    matvecs(c, g);
    GemmArgs e;
    e.m = o.ne;
    e.n = nrhs;
    e.k = o.nb;
    e.batch = L.n;
    e.A = c->P.d();
    e.lda = o.ne;
    e.sA = 0;
    e.B = L.G.d() + 1;
    e.ldb = ldGL;
    e.sB = sGL;
    e.D = s.Ue.d();
    e.ldd = o.ne;
    e.sD = (long long)o.ne * nrhs;
    matvecs(c, e);
    const long long total = (long long)L.n * nrhs * o.n;
    const int blocks = int(std::min<long long>((total + 255) / 256, 148 * 16));
    gen_leaf_output_kernel<<<blocks, 256, 0, c->st>>>(d_u, (long long)T.leaves.size(), L.ord.i(), L.n, o.n, o.ni, o.ne,
                                                      nrhs, c->interior.i(), c->exterior.i(), s.Ui.d(), s.Ue.d());
    ck(cudaGetLastError(), "leaf output");
    ++c->launches;
  }
}

std::vector<double> gen_root_points(const hpsg_ctx* c) { return hpsg::general_root_points(c->gen->plan); }
std::vector<double> gen_leaf_points(const hpsg_ctx* c) { return hpsg::general_leaf_points(c->gen->plan); }
long long gen_n_leaves(const hpsg_ctx* c) { return (long long)c->gen->plan.tree.leaves.size(); }
std::vector<int> gen_leaf_group_order(const hpsg_ctx* c) {
  std::vector<int> out;
  for (const auto& g : c->gen->plan.leaf_groups)
    for (int id : g.leaves) out.push_back(c->gen->plan.tree.leaf_ord[id]);
  return out;
}

}  // namespace hpsctx

// ---------------------------------------------------------------- adaptive refinement (host)
namespace {
double host_field(const void* ctx, const double* x) {
  return hpsk::eval_field_t<3>(*static_cast<const hpsk::DevField*>(ctx), x, 0, 0, 0);
}
}  // namespace

extern "C" int hpsg_refine_adaptive(int p, const double* lo, const double* hi, double tol, int max_depth,
                                    const hpsg_field* fields, int n_fields, int cap, int* n_nodes, int* depth,
                                    int* n_children, int* children, double* lo_out, double* hi_out,
                                    int* n_unresolved) {
  if (!lo || !hi || !fields || n_fields < 1 || !n_nodes || p < 4) return HPSG_ERR_INVALID;
  try {
    std::vector<hpsk::DevField> f(n_fields);
    for (int i = 0; i < n_fields; ++i) {
      if (fields[i].kind == HPSG_FIELD_SAMPLED || fields[i].kind < 0 || fields[i].kind > HPSG_FIELD_PB_EPS_GRAD)
        return HPSG_ERR_INVALID;
      f[i].kind = fields[i].kind;
      f[i].n_centers = fields[i].n_centers;
      for (int k = 0; k < 8; ++k) f[i].c[k] = fields[i].c[k];
      f[i].centers = fields[i].centers;  // host pointer: evaluated on the host
      f[i].samples = nullptr;
    }
    std::vector<std::pair<hpsg::PointField, const void*>> pf;
    for (const auto& x : f) pf.push_back({host_field, &x});
    const hpsg::RefineResult r = hpsg::refine_adaptive(lo, hi, p, tol, max_depth, pf);
    const int n = int(r.tree.depth.size());
    *n_nodes = n;
    if (n_unresolved) *n_unresolved = int(r.unresolved.size());
    if (n > cap) return HPSG_ERR_INVALID;  // *n_nodes tells the caller the capacity needed
    for (int i = 0; i < n; ++i) {
      if (depth) depth[i] = r.tree.depth[i];
      if (n_children) n_children[i] = r.tree.nch[i];
      for (int k = 0; k < 8; ++k)
        if (children) children[8 * i + k] = r.tree.child[i][k];
      for (int k = 0; k < 3; ++k) {
        if (lo_out) lo_out[3 * i + k] = r.tree.lo[3 * i + k];
        if (hi_out) hi_out[3 * i + k] = r.tree.hi[3 * i + k];
      }
    }
    return HPSG_OK;
  } catch (const std::exception&) {
    return HPSG_ERR_INVALID;
  }
}

namespace {
struct CbField {
  hpsg_point_fn fn;
  void* user;
};
double cb_field(const void* ctx, const double* x) {
  const CbField* f = static_cast<const CbField*>(ctx);
  return f->fn(f->user, x);
}
int write_tree(const hpsg::GTree& t, int cap, int* n_nodes, int* depth, int* n_children, int* children, double* lo,
               double* hi) {
  const int n = int(t.depth.size());
  *n_nodes = n;
  if (n > cap) return HPSG_ERR_INVALID;
  for (int i = 0; i < n; ++i) {
    if (depth) depth[i] = t.depth[i];
    if (n_children) n_children[i] = t.nch[i];
    for (int k = 0; k < 8; ++k)
      if (children) children[8 * i + k] = t.child[i][k];
    for (int k = 0; k < 3; ++k) {
      if (lo) lo[3 * i + k] = t.lo[3 * i + k];
      if (hi) hi[3 * i + k] = t.hi[3 * i + k];
    }
  }
  return HPSG_OK;
}
hpsg::GTree read_tree(const hpsg_tree_desc* d) {
  hpsg::GTree t;
  t.dim = d->dim;
  t.p = d->p;
  const int n = d->n_nodes;
  t.depth.assign(d->depth, d->depth + n);
  t.nch.assign(d->n_children, d->n_children + n);
  t.child.resize(n);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < 8; ++k) t.child[i][k] = d->children[8 * i + k];
  t.lo.assign(d->lo, d->lo + 3 * n);
  t.hi.assign(d->hi, d->hi + 3 * n);
  return t;
}
}  // namespace

extern "C" int hpsg_refine_adaptive_cb(int p, const double* lo, const double* hi, double tol, int max_depth,
                                       hpsg_point_fn const* fns, void* const* users, int n_fields, int cap,
                                       int* n_nodes, int* depth, int* n_children, int* children, double* lo_out,
                                       double* hi_out, int* n_unresolved) {
  if (!lo || !hi || !fns || n_fields < 1 || !n_nodes || p < 4) return HPSG_ERR_INVALID;
  try {
    std::vector<CbField> f(n_fields);
    std::vector<std::pair<hpsg::PointField, const void*>> pf;
    for (int i = 0; i < n_fields; ++i) {
      f[i] = {fns[i], users ? users[i] : nullptr};
      pf.push_back({cb_field, &f[i]});
    }
    const hpsg::RefineResult r = hpsg::refine_adaptive(lo, hi, p, tol, max_depth, pf);
    if (n_unresolved) *n_unresolved = int(r.unresolved.size());
    return write_tree(r.tree, cap, n_nodes, depth, n_children, children, lo_out, hi_out);
  } catch (const std::exception&) {
    return HPSG_ERR_INVALID;
  }
}

extern "C" int hpsg_enforce_level_restriction(const hpsg_tree_desc* in, int cap, int* n_nodes, int* depth,
                                              int* n_children, int* children, double* lo, double* hi) {
  if (!in || !n_nodes) return HPSG_ERR_INVALID;
  try {
    hpsg::GTree t = read_tree(in);
    hpsg::finalize_gtree(t);
    std::vector<long long> anchor(3 * t.depth.size(), 0);  // integer coordinates (TreeNode::anchor)
    for (int d = 0; d <= t.max_depth(); ++d)
      for (int id : t.levels[d])
        for (int c = 0; c < t.nch[id]; ++c)
          for (int k = 0; k < 3; ++k) {
            static const int off[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                                          {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};
            anchor[3 * t.child[id][c] + k] = k < t.dim ? 2 * anchor[3 * id + k] + off[c][k] : 0;
          }
    hpsg::enforce_level_restriction(t, anchor);
    return write_tree(t, cap, n_nodes, depth, n_children, children, lo, hi);
  } catch (const std::exception&) {
    return HPSG_ERR_INVALID;
  }
}

extern "C" int hpsg_tree_desc_leaf_points(const hpsg_tree_desc* d, double* xyz) {
  if (!d || !xyz) return HPSG_ERR_INVALID;
  try {
    hpsg::GeneralPlan g;
    g.tree = read_tree(d);
    hpsg::finalize_gtree(g.tree);
    hpsg::general_leaf_points_into(g, xyz);
    return HPSG_OK;
  } catch (const std::exception&) {
    return HPSG_ERR_INVALID;
  }
}
