// solve_problem_b200.cpp -- the reference's solve_problem() flow (proj/src/problems.cpp:360-422)
// for the poisson2d manufactured problem (proj/src/problems.cpp:40-74), written against the
// C++ drop-in include/hps/hps_b200.hpp.  Only the include and namespace differ from a caller of
// hps::HpsSolver<Real>.
//
//   g++ -std=c++17 -O2 -Iinclude examples/solve_problem_b200.cpp -Lpaper_2503_17535_b200
//       -lhps_b200 -Wl,-rpath,$PWD/paper_2503_17535_b200 -o solve_problem_b200
//   ./solve_problem_b200 [L] [p] [literal_sign]
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "hps/hps_b200.hpp"

using namespace hps::b200;

int main(int argc, char** argv) {
  const int L = argc > 1 ? std::atoi(argv[1]) : 3;
  const int p = argc > 2 ? std::atoi(argv[2]) : 16;
  const bool literal = argc > 3 ? std::atoi(argv[3]) != 0 : false;
  // 4th argument 1: build WITHOUT the source, then solve through solve_new_source (the
  // repeated-source path, solver.cpp:285-307) with the manufactured source sampled per leaf
  const bool new_source = argc > 4 ? std::atoi(argv[4]) != 0 : false;
  try {
    Box dom;
    dom.lo[0] = dom.lo[1] = -1.0;
    dom.hi[0] = dom.hi[1] = 1.0;
    const auto t0 = std::chrono::steady_clock::now();
    DiscretizationTree tree = build_uniform_tree(dom, L, 2, p);
    // operator and manufactured solution of make_manufactured_2d_dtn
    std::vector<CoefficientField> terms;
    terms.push_back({CoefficientField::Role::laplacian, -1, -1, [](const Point&) { return 1.0; }});
    terms.push_back({CoefficientField::Role::gradient, 0, -1, [](const Point& x) { return -std::cos(5.0 * x[1]); }});
    terms.push_back({CoefficientField::Role::gradient, 1, -1, [](const Point& x) { return std::sin(5.0 * x[1]); }});
    auto u = [](const Point& x) {
      return std::exp(5.0 * x[0]) * std::sin(5.0 * x[1]) + std::sin(10.0 * M_PI * x[0]) * std::sin(M_PI * x[1]);
    };
    auto f = [](const Point& x) {
      const double X = x[0], Y = x[1];
      const double ux = 5.0 * std::exp(5.0 * X) * std::sin(5.0 * Y) +
                        10.0 * M_PI * std::cos(10.0 * M_PI * X) * std::sin(M_PI * Y);
      const double uy = 5.0 * std::exp(5.0 * X) * std::cos(5.0 * Y) + M_PI * std::sin(10.0 * M_PI * X) * std::cos(M_PI * Y);
      const double lap = -101.0 * M_PI * M_PI * std::sin(10.0 * M_PI * X) * std::sin(M_PI * Y);
      return lap - std::cos(5.0 * Y) * ux + std::sin(5.0 * Y) * uy;
    };
    SolverOptions opts;
    opts.literal_sign = literal;
    opts.keep_factors = new_source;
    HpsSolver solver(tree, Variant::dtn, 1.0, terms, new_source ? std::function<Real(const Point&)>() : f, opts);
    const auto t1 = std::chrono::steady_clock::now();
    solver.build();
    const auto t2 = std::chrono::steady_clock::now();
    const std::vector<Real> g = solver.sample_root_data(u);
    const std::vector<Point> pts = leaf_cheb_points(tree);
    SolutionField field;
    if (new_source) {
      const int np = p * p;
      std::vector<std::vector<Real>> leaf_f(size_t(tree.n_leaves()), std::vector<Real>(size_t(np)));
      for (long long l = 0; l < tree.n_leaves(); ++l)
        for (int i = 0; i < np; ++i) {
          leaf_f[size_t(l)][size_t(i)] = f(pts[size_t(l * np + i)]);
        }
      field = solver.solve_new_source(leaf_f, RootBC::dirichlet, &g);
    } else {
      field = solver.solve(g);
    }
    const auto t3 = std::chrono::steady_clock::now();
    // error_report (proj/src/problems.cpp:270-293) at the leaf Chebyshev points
    double num = 0, den = 0;
    const int npts = p * p;
    for (long long l = 0; l < tree.n_leaves(); ++l)
      for (int i = 0; i < npts; ++i) {
        const Point& x = pts[size_t(l * npts + i)];
        num = std::fmax(num, std::fabs(field.u[size_t(l)][size_t(i)] - u(x)));
        den = std::fmax(den, std::fabs(u(x)));
      }
    auto s = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
    std::printf("{\"L\": %d, \"p\": %d, \"N\": %lld, \"top_D\": %d, \"rel_linf\": %.3e, \"t_setup_s\": %.4f, "
                "\"t_build_s\": %.4f, \"t_solve_s\": %.4f}\n",
                L, p, tree.total_points(), solver.top_D_size(), num / den, s(t0, t1), s(t1, t2), s(t2, t3));
    return 0;
  } catch (const Error& e) {
    std::fprintf(stderr, "hps::b200::Error: %s\n", e.what());
    return 1;
  }
}
