// adapter_e2e_b200.cpp -- the headline workload (BASELINE configs[1]: 2D variable-coefficient Helmholtz,
// p=16, L=8) end to end through the reference-facing C++ drop-in, as a caller of hps::HpsSolver<Real>
// writes it: std::function coefficient/source fields sampled on the host at every leaf Chebyshev point
// (16.8 M points x 3 fields at L=8) and uploaded, build(), sample_root_data(), solve() into the
// reference's per-leaf SolutionField.  Times every stage with the host clock; prints one JSON line per rep.
//   usage: adapter_e2e_b200 [L=8] [reps=2] [host_threads=0 (every core)]
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "hps/hps_b200.hpp"

using namespace hps::b200;

int main(int argc, char** argv) {
  const int L = argc > 1 ? std::atoi(argv[1]) : 8;
  const int reps = argc > 2 ? std::atoi(argv[2]) : 2;
  const int host_threads = argc > 3 ? std::atoi(argv[3]) : 0;
  const int p = 16;
  const double k = 30.0, alpha = 50.0, phase = 0.3;  // problems.py helmholtz_bumps (make_scattering's bumps)
  std::vector<double> z(10 * 3);
  hpsg_bump_centers(7ULL, 10, 2, z.data());
  auto q = [&](const Point& x) {
    double s = 0;
    for (int j = 0; j < 10; ++j) {
      const double d0 = x[0] - z[3 * j], d1 = x[1] - z[3 * j + 1];
      s += std::exp(-alpha * (d0 * d0 + d1 * d1));
    }
    return s;
  };
  auto u = [&](const Point& x) { return std::sin(k * x[0] + phase); };
  try {
    for (int rep = 0; rep < reps; ++rep) {
      Box dom;
      dom.lo[0] = dom.lo[1] = -1.0;
      dom.hi[0] = dom.hi[1] = 1.0;
      const auto t0 = std::chrono::steady_clock::now();
      DiscretizationTree tree = build_uniform_tree(dom, L, 2, p);
      std::vector<CoefficientField> terms;
      terms.push_back({CoefficientField::Role::laplacian, -1, -1, [](const Point&) { return 1.0; }});
      terms.push_back({CoefficientField::Role::zeroth, -1, -1, [&](const Point& x) { return k * k * (1.0 + q(x)); }});
      SolverOptions opts;
      opts.literal_sign = false;
      opts.root_implicit_S = true;
      opts.host_threads = host_threads;
      HpsSolver solver(tree, Variant::dtn, 1.0, terms,
                       [&](const Point& x) { return k * k * q(x) * std::sin(k * x[0] + phase); }, opts);
      const auto t1 = std::chrono::steady_clock::now();
      solver.build();
      const auto t2 = std::chrono::steady_clock::now();
      const std::vector<Real> g = solver.sample_root_data(u);
      const SolutionField field = solver.solve(g);
      const auto t3 = std::chrono::steady_clock::now();
      double num = 0, den = 0;  // error against the plane wave (outside the timed stages)
      const std::vector<Point> pts = leaf_cheb_points(tree);
      const int np = p * p;
      for (long long l = 0; l < tree.n_leaves(); ++l)
        for (int i = 0; i < np; ++i) {
          const double e = u(pts[size_t(l * np + i)]);
          num = std::fmax(num, std::fabs(field.u[size_t(l)][size_t(i)] - e));
          den = std::fmax(den, std::fabs(e));
        }
      auto s = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
      const double N = double(tree.total_points());
      std::printf("{\"rep\": %d, \"L\": %d, \"N\": %.0f, \"host_threads\": %d, \"t_setup_s\": %.4f, \"t_build_s\": %.4f, "
                  "\"t_solve_s\": %.4f, \"t_total_s\": %.4f, \"dof_per_s_build_solve\": %.4e, \"dof_per_s_total\": %.4e, "
                  "\"rel_linf\": %.3e}\n",
                  rep, L, N, host_threads, s(t0, t1), s(t1, t2), s(t2, t3), s(t0, t3), N / s(t1, t3), N / s(t0, t3),
                  num / den);
      std::fflush(stdout);
    }
    return 0;
  } catch (const Error& e) {
    std::fprintf(stderr, "hps::b200::Error: %s\n", e.what());
    return 1;
  }
}
