// sharded_emulate_b200.cpp -- the subtree-sharded C-ABI (hpsg_shard_*) driven by `world` rank threads that
// share one GPU, with an in-process mailbox transport standing in for NCCL send/recv.  Each rank builds and
// solves its share; the gathered solution is compared with one single-context hpsg_create/hpsg_build/
// hpsg_solve_device of the same problem.  This checks the plan, the exchange schedule and the layout of
// every message without a second GPU (each rank's kernels run to completion before its messages are sent,
// so nothing waits on another rank's kernel).  Prints one JSON line.
//   usage: sharded_emulate_b200 [world=4] [L=5] [p=16] [dim=2] [nrhs=2]
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <deque>
#include <map>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "hps_cuda.h"

namespace {

struct Mailbox {
  std::mutex m;
  std::condition_variable cv;
  std::map<std::pair<int, int>, std::deque<std::vector<char>>> q;  // (src, dst) -> FIFO
  long long bytes = 0, messages = 0;
};

struct RankTransport {
  Mailbox* mb;
  int rank;
  struct Pending {
    void* d;
    size_t bytes;
    int peer;
  };
  std::vector<Pending> pend;
};

int tr_send(void* user, const void* d_buf, size_t bytes, int peer, void* stream) {
  auto* t = static_cast<RankTransport*>(user);
  if (cudaStreamSynchronize(static_cast<cudaStream_t>(stream)) != cudaSuccess) return 1;
  std::vector<char> h(bytes);
  if (cudaMemcpy(h.data(), d_buf, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
  std::lock_guard<std::mutex> lk(t->mb->m);
  t->mb->q[{t->rank, peer}].push_back(std::move(h));
  t->mb->bytes += (long long)bytes;
  t->mb->messages += 1;
  t->mb->cv.notify_all();
  return 0;
}

int tr_recv(void* user, void* d_buf, size_t bytes, int peer, void*) {
  static_cast<RankTransport*>(user)->pend.push_back({d_buf, bytes, peer});
  return 0;
}

int tr_group_end(void* user, void*) {  // receives complete here, after every send of the group was posted
  auto* t = static_cast<RankTransport*>(user);
  for (const auto& r : t->pend) {
    std::vector<char> h;
    {
      std::unique_lock<std::mutex> lk(t->mb->m);
      auto& fifo = t->mb->q[{r.peer, t->rank}];
      t->mb->cv.wait(lk, [&] { return !fifo.empty(); });
      h = std::move(fifo.front());
      fifo.pop_front();
    }
    if (h.size() != r.bytes) return 1;
    if (cudaMemcpy(r.d, h.data(), r.bytes, cudaMemcpyHostToDevice) != cudaSuccess) return 1;
  }
  t->pend.clear();
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  const int world = argc > 1 ? std::atoi(argv[1]) : 4;
  const int L = argc > 2 ? std::atoi(argv[2]) : 5;
  const int p = argc > 3 ? std::atoi(argv[3]) : 16;
  const int dim = argc > 4 ? std::atoi(argv[4]) : 2;
  const int nrhs = argc > 5 ? std::atoi(argv[5]) : 2;

  const hpsg_tree tree{dim, p, L, 0.0, 1.0};
  std::vector<double> centers(8 * 3);
  hpsg_bump_centers(20260810ULL, 8, dim, centers.data());
  hpsg_term terms[2] = {};
  terms[0].role = HPSG_ROLE_LAPLACIAN;
  terms[0].field.kind = HPSG_FIELD_CONST;
  terms[0].field.c[0] = 1.0;
  terms[1].role = HPSG_ROLE_ZEROTH;  // Helmholtz-type: -k^2 (1 + 0.5 sum of bumps), k = 20
  terms[1].field.kind = HPSG_FIELD_BUMPS;
  terms[1].field.n_centers = 8;
  terms[1].field.c[0] = -400.0;
  terms[1].field.c[1] = -200.0;
  terms[1].field.c[2] = 60.0;
  terms[1].field.centers = centers.data();
  hpsg_field source{};
  source.kind = HPSG_FIELD_BUMPS;
  source.n_centers = 8;
  source.c[0] = 0.0;
  source.c[1] = 1.0;
  source.c[2] = 80.0;
  source.centers = centers.data();
  hpsg_options opts{};
  opts.literal_sign = 1;

  // single-context baseline
  hpsg_ctx* one = nullptr;
  if (hpsg_create(&tree, terms, 2, &source, &opts, &one) != HPSG_OK || hpsg_build(one) != HPSG_OK) {
    std::fprintf(stderr, "single context: %s\n", one ? hpsg_last_error(one) : "create failed");
    return 1;
  }
  hpsg_stats st{};
  hpsg_get_stats(one, &st);
  const long long npts = st.n_points;
  std::vector<double> g(size_t(nrhs) * st.root_bsize);
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  for (double& x : g) x = U(rng);
  double *d_g = nullptr, *d_u1 = nullptr;
  cudaMalloc(&d_g, g.size() * 8);
  cudaMalloc(&d_u1, size_t(nrhs) * npts * 8);
  cudaMemcpy(d_g, g.data(), g.size() * 8, cudaMemcpyHostToDevice);
  if (hpsg_solve_device(one, d_g, nrhs, d_u1) != HPSG_OK) {
    std::fprintf(stderr, "single solve: %s\n", hpsg_last_error(one));
    return 1;
  }
  std::vector<double> u1(size_t(nrhs) * npts), u(size_t(nrhs) * npts, NAN);
  cudaMemcpy(u1.data(), d_u1, u1.size() * 8, cudaMemcpyDeviceToHost);
  hpsg_destroy(one);
  cudaFree(d_u1);

  // world rank threads
  Mailbox mb;
  std::vector<std::thread> th;
  std::vector<int> rc(static_cast<size_t>(world), 0);
  std::vector<std::string> err(static_cast<size_t>(world));
  std::vector<int> cut(static_cast<size_t>(world));
  std::vector<double> t_build(static_cast<size_t>(world)), t_solve(static_cast<size_t>(world));
  std::mutex umx;
  for (int r = 0; r < world; ++r)
    th.emplace_back([&, r] {
      cudaSetDevice(0);
      RankTransport rt{&mb, r, {}};
      hpsg_transport tr{&rt, nullptr, tr_send, tr_recv, tr_group_end};
      hpsg_shard* s = nullptr;
      int e = hpsg_shard_create(&tree, terms, 2, &source, &opts, world, r, &tr, &s);
      const auto t0 = std::chrono::steady_clock::now();
      if (e == HPSG_OK) e = hpsg_shard_build(s);
      const auto t1 = std::chrono::steady_clock::now();
      long long first = 0, nl = 0;
      double* d_u = nullptr;
      if (e == HPSG_OK) e = hpsg_shard_info(s, &cut[size_t(r)], &first, &nl);
      const long long np = nl * (dim == 2 ? p * p : p * p * p);
      if (e == HPSG_OK && cudaMalloc(&d_u, size_t(nrhs) * np * 8 + 8) != cudaSuccess) e = HPSG_ERR_OOM;
      if (e == HPSG_OK) e = hpsg_shard_solve_device(s, r == 0 ? d_g : nullptr, nrhs, d_u);
      const auto t2 = std::chrono::steady_clock::now();
      if (e == HPSG_OK) {
        std::vector<double> h(size_t(nrhs) * np);
        cudaMemcpy(h.data(), d_u, h.size() * 8, cudaMemcpyDeviceToHost);
        const long long off = first * (dim == 2 ? p * p : p * p * p);
        std::lock_guard<std::mutex> lk(umx);
        for (int k = 0; k < nrhs; ++k)
          for (long long i = 0; i < np; ++i) u[size_t(k) * npts + size_t(off + i)] = h[size_t(k) * np + size_t(i)];
      } else {
        err[size_t(r)] = s ? hpsg_shard_last_error(s) : "create failed";
      }
      rc[size_t(r)] = e;
      t_build[size_t(r)] = std::chrono::duration<double>(t1 - t0).count();
      t_solve[size_t(r)] = std::chrono::duration<double>(t2 - t1).count();
      if (d_u) cudaFree(d_u);
      hpsg_shard_destroy(s);
    });
  for (auto& t : th) t.join();
  for (int r = 0; r < world; ++r)
    if (rc[size_t(r)] != HPSG_OK) {
      std::fprintf(stderr, "rank %d: error %d: %s\n", r, rc[size_t(r)], err[size_t(r)].c_str());
      return 1;
    }
  double num = 0, den = 0;
  bool missing = false;  // a leaf value no rank wrote stays NaN
  for (size_t i = 0; i < u.size(); ++i) {
    missing = missing || std::isnan(u[i]);
    num = std::fmax(num, std::fabs(u[i] - u1[i]));
    den = std::fmax(den, std::fabs(u1[i]));
  }
  if (missing) num = NAN;
  cudaFree(d_g);
  double tb = 0, ts = 0;
  for (int r = 0; r < world; ++r) tb = std::fmax(tb, t_build[size_t(r)]), ts = std::fmax(ts, t_solve[size_t(r)]);
  std::printf("{\"world\": %d, \"L\": %d, \"p\": %d, \"dim\": %d, \"nrhs\": %d, \"cut_depth\": %d, \"messages\": %lld, "
              "\"bytes\": %lld, \"rel_diff\": %.3e, \"t_build_s\": %.3f, \"t_solve_s\": %.3f}\n",
              world, L, p, dim, nrhs, cut[0], mb.messages, mb.bytes, num / den, tb, ts);
  return std::isfinite(num / den) && num / den < 1e-10 ? 0 : 2;
}
