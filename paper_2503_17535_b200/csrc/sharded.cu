// sharded.cu -- the subtree-sharded multi-GPU build/solve behind the C-ABI, for C/C++ hosts.
//
// Same plan as paper_2503_17535_b200/sharded.py: the tree is cut at depth ds (smallest with
// nchild^ds >= world); subtree k of depth ds is owned by rank floor(k * world / nchild^ds) (a contiguous
// range of the DFS leaf order, mesh.cpp:54-71); every node above the cut is merged by the owner of its
// first subtree.  The only data-path exchanges are the algorithm's own: the [h|T] of a child whose owner
// differs from its parent's (merge.cpp:226-278 consumes it) travels up, its boundary data g
// (solver.cpp:210-224) travels down.  Every rank's numerical work runs through C-ABI parts
// (hpsg_create_part) on one stream; the transfers go through the caller's transport (NCCL send/recv in a
// group on that stream, or any other device-to-device mechanism).
#include <cuda_runtime.h>

#include <algorithm>
#include <iterator>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/hps_cuda.h"

namespace {

struct DBuf {  // device buffer owned by the shard
  double* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  explicit DBuf(size_t count) : n(count) {
    if (count && cudaMalloc(&p, count * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      throw std::runtime_error("hpsg_shard: cudaMalloc failed");
    }
  }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr, o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    std::swap(p, o.p);
    std::swap(n, o.n);
    return *this;
  }
  ~DBuf() {
    if (p) cudaFree(p);
  }
};

struct Plan {
  int L = 0, nchild = 4, world = 1, ds = 0;
  std::vector<int> sub_owner;
  long long n_sub() const { return (long long)sub_owner.size(); }
  int owner(int depth, long long index) const {
    long long f = 1;
    if (depth >= ds) {
      for (int k = 0; k < depth - ds; ++k) f *= nchild;
      return sub_owner[size_t(index / f)];
    }
    for (int k = 0; k < ds - depth; ++k) f *= nchild;
    return sub_owner[size_t(index * f)];
  }
};

}  // namespace

struct hpsg_shard {
  std::string err;
  Plan plan;
  int rank = 0;
  hpsg_transport tr{};
  hpsg_tree tree{};
  cudaStream_t st = nullptr;
  int device = 0;
  std::map<long long, hpsg_ctx*> sub;                    // owned subtrees (depth ds)
  std::map<std::pair<int, long long>, hpsg_ctx*> top;    // owned nodes above the cut
  std::map<std::pair<int, long long>, DBuf> ht, g;       // [h|T] / boundary data of held nodes
  std::map<std::pair<int, long long>, int> nb;           // boundary size of a node held here
  ~hpsg_shard() {
    for (auto& kv : sub) hpsg_destroy(kv.second);
    for (auto& kv : top) hpsg_destroy(kv.second);
    if (st) cudaStreamDestroy(st);
  }
};

namespace {

int fail(hpsg_shard* s, int code, const std::string& m) {
  if (s) s->err = m;
  return code;
}

int node_nb(const hpsg_tree& t, int depth) {  // boundary points of a node at `depth` of a uniform tree
  const int q = t.p - 2;
  long long f = 1;
  for (int k = 0; k < t.L - depth; ++k) f *= 2;
  return t.dim == 2 ? int(4 * q * f) : int(6LL * q * q * f * f);
}

void check(hpsg_shard*, int rc, hpsg_ctx* c, const char* what) {
  if (rc != HPSG_OK) throw std::runtime_error(std::string(what) + ": " + (c ? hpsg_last_error(c) : "error"));
}

struct Msg {
  int peer;
  std::pair<int, long long> key;
  double* buf;
  size_t bytes;
  bool send;
};

void exchange(hpsg_shard* s, std::vector<Msg>& msgs) {
  if (msgs.empty()) return;
  // deterministic order on both sides: by (peer, key), sends and receives interleaved as posted
  std::sort(msgs.begin(), msgs.end(), [](const Msg& a, const Msg& b) {
    return a.peer != b.peer ? a.peer < b.peer : a.key < b.key;
  });
  if (s->tr.group_begin && s->tr.group_begin(s->tr.user) != 0) throw std::runtime_error("transport group_begin");
  for (const Msg& m : msgs) {
    const int rc = m.send ? s->tr.send(s->tr.user, m.buf, m.bytes, m.peer, s->st)
                          : s->tr.recv(s->tr.user, m.buf, m.bytes, m.peer, s->st);
    if (rc != 0) throw std::runtime_error("transport send/recv");
  }
  if (s->tr.group_end && s->tr.group_end(s->tr.user, s->st) != 0) throw std::runtime_error("transport group_end");
}

}  // namespace

extern "C" {

int hpsg_shard_create(const hpsg_tree* tree, const hpsg_term* terms, int n_terms, const hpsg_field* source,
                      const hpsg_options* opts, int world, int rank, const hpsg_transport* tr, hpsg_shard** out) {
  if (!tree || !out || world < 1 || rank < 0 || rank >= world) return HPSG_ERR_INVALID;
  if (world > 1 && (!tr || !tr->send || !tr->recv)) return HPSG_ERR_INVALID;
  *out = nullptr;
  auto s = std::make_unique<hpsg_shard>();
  s->tree = *tree;
  s->rank = rank;
  if (tr) s->tr = *tr;
  s->device = opts ? opts->device : 0;
  Plan& p = s->plan;
  p.L = tree->L;
  p.nchild = tree->dim == 2 ? 4 : 8;
  p.world = world;
  long long n = 1;
  while (n < world) n *= p.nchild, ++p.ds;
  if (world > 1 && p.ds > p.L - 1) {
    *out = s.release();
    return fail(*out, HPSG_ERR_INVALID, "hpsg_shard_create: tree too shallow to shard over this many ranks");
  }
  for (long long k = 0; k < n; ++k) p.sub_owner.push_back(int(k * world / n));
  try {
    if (cudaSetDevice(s->device) != cudaSuccess || cudaStreamCreateWithFlags(&s->st, cudaStreamNonBlocking) != cudaSuccess)
      throw std::runtime_error("hpsg_shard_create: CUDA device/stream");
    auto make = [&](int root_depth, long long root_index, int cut_depth) {
      hpsg_part part{root_depth, root_index, cut_depth};
      hpsg_ctx* c = nullptr;
      const int rc = hpsg_create_part(tree, &part, terms, n_terms, source, opts, &c);
      if (rc != HPSG_OK) {
        const std::string m = c ? hpsg_last_error(c) : "no CUDA device";
        hpsg_destroy(c);
        throw std::runtime_error("hpsg_create_part: " + m);
      }
      std::unique_ptr<hpsg_ctx, void (*)(hpsg_ctx*)> guard(c, hpsg_destroy);
      check(s.get(), hpsg_set_stream(c, s->st), c, "hpsg_set_stream");
      long long n_cut = 0;
      int cut_nb = 0, root_nb = 0;
      check(s.get(), hpsg_part_sizes(c, &n_cut, &cut_nb, &root_nb), c, "hpsg_part_sizes");
      if (root_nb != node_nb(*tree, root_depth) || (cut_depth < tree->L && cut_nb != node_nb(*tree, cut_depth)))
        throw std::runtime_error("hpsg_shard_create: only real (DtN) uniform trees shard");
      return guard.release();
    };
    for (long long k = 0; k < p.n_sub(); ++k)
      if (p.sub_owner[size_t(k)] == rank) s->sub[k] = make(p.ds, k, p.L);
    long long cnt = 1;
    for (int d = 0; d < p.ds; ++d, cnt *= p.nchild)
      for (long long i = 0; i < cnt; ++i)
        if (p.owner(d, i) == rank) s->top[{d, i}] = make(d, i, d + 1);
  } catch (const std::exception& e) {
    *out = s.release();
    return fail(*out, HPSG_ERR_INVALID, e.what());
  }
  *out = s.release();
  return HPSG_OK;
}

int hpsg_shard_build(hpsg_shard* s) {
  if (!s) return HPSG_ERR_INVALID;
  try {
    const Plan& p = s->plan;
    s->ht.clear();
    for (auto& kv : s->sub) {  // leaves + merges of every owned subtree
      check(s, hpsg_build(kv.second), kv.second, "hpsg_build");
      if (p.ds > 0) {
        const int nb = node_nb(s->tree, p.ds);
        DBuf b(size_t(nb) * (1 + nb));
        check(s, hpsg_part_root_ht(kv.second, b.p), kv.second, "hpsg_part_root_ht");
        s->ht[{p.ds, kv.first}] = std::move(b);
      }
    }
    long long cnt = 1;
    for (int d = 0; d < p.ds - 1; ++d) cnt *= p.nchild;
    for (int depth = p.ds - 1; depth >= 0; --depth, cnt /= p.nchild) {
      // upward [h|T] of children whose owner differs from the parent's
      std::vector<Msg> msgs;
      const int cnb = node_nb(s->tree, depth + 1);
      for (long long i = 0; i < cnt; ++i) {
        const int dst = p.owner(depth, i);
        for (int c = 0; c < p.nchild; ++c) {
          const std::pair<int, long long> key{depth + 1, p.nchild * i + c};
          const int src = p.owner(key.first, key.second);
          if (src == dst) continue;
          const size_t bytes = size_t(cnb) * (1 + cnb) * sizeof(double);
          if (src == s->rank) msgs.push_back({dst, key, s->ht[key].p, bytes, true});
          if (dst == s->rank) {
            s->ht[key] = DBuf(size_t(cnb) * (1 + cnb));
            msgs.push_back({src, key, s->ht[key].p, bytes, false});
          }
        }
      }
      exchange(s, msgs);
      for (auto& kv : s->top) {
        if (kv.first.first != depth) continue;
        const long long i = kv.first.second;
        for (int c = 0; c < p.nchild; ++c)
          check(s, hpsg_part_set_cut_ht(kv.second, c, s->ht[{depth + 1, p.nchild * i + c}].p), kv.second,
                "hpsg_part_set_cut_ht");
        check(s, hpsg_build(kv.second), kv.second, "hpsg_build");
        if (depth > 0) {
          const int nb = node_nb(s->tree, depth);
          DBuf b(size_t(nb) * (1 + nb));
          check(s, hpsg_part_root_ht(kv.second, b.p), kv.second, "hpsg_part_root_ht");
          s->ht[kv.first] = std::move(b);
        }
      }
      for (auto it = s->ht.begin(); it != s->ht.end();)  // consumed children
        it = it->first.first == depth + 1 ? s->ht.erase(it) : std::next(it);
    }
    if (cudaStreamSynchronize(s->st) != cudaSuccess) throw std::runtime_error("hpsg_shard_build: stream");
  } catch (const std::exception& e) {
    return fail(s, HPSG_ERR_INVALID, e.what());
  }
  return HPSG_OK;
}

int hpsg_shard_solve_device(hpsg_shard* s, const double* d_g_root, int nrhs, double* d_u) {
  if (!s || nrhs < 1 || !d_u) return HPSG_ERR_INVALID;
  try {
    const Plan& p = s->plan;
    s->g.clear();
    const int nb0 = node_nb(s->tree, 0);
    if (s->rank == p.owner(0, 0)) {
      if (!d_g_root) throw std::runtime_error("hpsg_shard_solve_device: the root owner needs the root data");
      DBuf g(size_t(nb0) * nrhs);
      if (cudaMemcpyAsync(g.p, d_g_root, g.n * sizeof(double), cudaMemcpyDeviceToDevice, s->st) != cudaSuccess)
        throw std::runtime_error("root data copy");
      s->g[{0, 0}] = std::move(g);
    }
    long long cnt = 1;
    for (int depth = 0; depth < p.ds; ++depth, cnt *= p.nchild) {
      const int cnb = node_nb(s->tree, depth + 1);
      for (auto& kv : s->top) {  // downward pass of the owned top nodes: children boundary data
        if (kv.first.first != depth) continue;
        DBuf out(size_t(nrhs) * p.nchild * cnb);
        check(s, hpsg_part_solve_cut(kv.second, s->g[kv.first].p, nrhs, out.p), kv.second, "hpsg_part_solve_cut");
        for (int c = 0; c < p.nchild; ++c) {  // child c of rhs r: out[(r * nchild + c) * cnb ...]
          DBuf gc(size_t(nrhs) * cnb);
          if (cudaMemcpy2DAsync(gc.p, size_t(cnb) * 8, out.p + size_t(c) * cnb, size_t(p.nchild) * cnb * 8,
                                size_t(cnb) * 8, size_t(nrhs), cudaMemcpyDeviceToDevice, s->st) != cudaSuccess)
            throw std::runtime_error("child data copy");
          s->g[{depth + 1, p.nchild * kv.first.second + c}] = std::move(gc);
        }
        if (cudaStreamSynchronize(s->st) != cudaSuccess) throw std::runtime_error("stream");
        s->g.erase(kv.first);
      }
      std::vector<Msg> msgs;
      for (long long i = 0; i < cnt; ++i) {
        const int src = p.owner(depth, i);
        for (int c = 0; c < p.nchild; ++c) {
          const std::pair<int, long long> key{depth + 1, p.nchild * i + c};
          const int dst = p.owner(key.first, key.second);
          if (src == dst) continue;
          const size_t bytes = size_t(nrhs) * cnb * sizeof(double);
          if (src == s->rank) msgs.push_back({dst, key, s->g[key].p, bytes, true});
          if (dst == s->rank) {
            s->g[key] = DBuf(size_t(nrhs) * cnb);
            msgs.push_back({src, key, s->g[key].p, bytes, false});
          }
        }
      }
      exchange(s, msgs);
    }
    // leaves of the owned subtrees, in subtree (= DFS) order: u[r][local leaf][pt]
    std::vector<long long> np;
    long long n_total = 0;
    for (auto& kv : s->sub) {
      hpsg_stats st{};
      check(s, hpsg_get_stats(kv.second, &st), kv.second, "hpsg_get_stats");
      np.push_back(st.n_points);
      n_total += st.n_points;
    }
    long long off = 0;
    size_t j = 0;
    for (auto& kv : s->sub) {
      const double* g = p.ds > 0 ? s->g[{p.ds, kv.first}].p : d_g_root;
      DBuf u(size_t(nrhs) * np[j]);
      check(s, hpsg_solve_device(kv.second, g, nrhs, u.p), kv.second, "hpsg_solve_device");
      if (cudaMemcpy2DAsync(d_u + off, size_t(n_total) * 8, u.p, size_t(np[j]) * 8, size_t(np[j]) * 8,
                            size_t(nrhs), cudaMemcpyDeviceToDevice, s->st) != cudaSuccess)
        throw std::runtime_error("u copy");
      off += np[j++];
      if (cudaStreamSynchronize(s->st) != cudaSuccess) throw std::runtime_error("stream");
    }
  } catch (const std::exception& e) {
    return fail(s, HPSG_ERR_INVALID, e.what());
  }
  return HPSG_OK;
}

int hpsg_shard_info(hpsg_shard* s, int* cut_depth, long long* first_leaf, long long* n_leaves) {
  if (!s) return HPSG_ERR_INVALID;
  const Plan& p = s->plan;
  long long per = 1;  // leaves per depth-ds subtree
  for (int k = 0; k < p.L - p.ds; ++k) per *= p.nchild;
  long long first = -1, count = 0;
  for (auto& kv : s->sub) {
    if (first < 0) first = kv.first * per;
    count += per;
  }
  if (cut_depth) *cut_depth = p.ds;
  if (first_leaf) *first_leaf = first < 0 ? 0 : first;
  if (n_leaves) *n_leaves = count;
  return HPSG_OK;
}

const char* hpsg_shard_last_error(hpsg_shard* s) { return s ? s->err.c_str() : "null shard"; }

void hpsg_shard_destroy(hpsg_shard* s) {
  if (s && s->st) cudaStreamSynchronize(s->st);
  delete s;
}

}  // extern "C"
