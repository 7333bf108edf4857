// iti_robin_b200.cpp -- the reference's ItI problem (make_manufactured_2d_iti, proj/src/problems.cpp:76-107)
// through the C++ drop-in header: complex source, impedance root data, SPEC.md:545 gate (< 1e-6 at L=4).
//   make -C paper_2503_17535_b200 example  (builds examples/iti_robin_b200 too)
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "hps/hps_b200.hpp"

using namespace hps::b200;

int main(int argc, char** argv) {
  const int L = argc > 1 ? std::atoi(argv[1]) : 4;
  const int p = argc > 2 ? std::atoi(argv[2]) : 16;
  try {
    Box dom;
    dom.lo[0] = dom.lo[1] = -1.0;
    dom.hi[0] = dom.hi[1] = 1.0;
    DiscretizationTree tree = build_uniform_tree(dom, L, 2, p);
    const Complex I(0.0, 1.0);
    auto q = [](const Point& x) { return 1.0 + std::exp(-50.0 * (x[0] * x[0] + x[1] * x[1])); };
    std::vector<CoefficientField> terms;
    terms.push_back({CoefficientField::Role::laplacian, -1, -1, [](const Point&) { return 1.0; }});
    terms.push_back({CoefficientField::Role::zeroth, -1, -1, q});
    auto u = [&](const Point& x) { return std::exp(I * 20.0 * x[0]) + std::exp(I * 30.0 * x[1]); };
    auto f = [&](const Point& x) {
      return -400.0 * std::exp(I * 20.0 * x[0]) - 900.0 * std::exp(I * 30.0 * x[1]) + q(x) * u(x);
    };
    HpsSolverComplex solver(tree, Variant::iti, 1.0, terms, f);
    solver.build();
    const auto pts = solver.root_boundary_points();
    std::vector<Complex> g(pts.size());
    const size_t per = pts.size() / 4;
    const double nx[4] = {0, 1, 0, -1}, ny[4] = {-1, 0, 1, 0};
    for (size_t i = 0; i < pts.size(); ++i) {
      const int s = int(i / per);
      const Point& x = pts[i];
      const Complex gx = 20.0 * I * std::exp(I * 20.0 * x[0]), gy = 30.0 * I * std::exp(I * 30.0 * x[1]);
      g[i] = nx[s] * gx + ny[s] * gy + I * u(x);   // eta = 1
    }
    SolutionFieldC field = solver.solve(g);
    hpsg_tree t{2, p, L, -1.0, 1.0};
    std::vector<double> xyz(size_t(tree.total_points()) * 3);
    hpsg_tree_leaf_points(&t, xyz.data());
    double num = 0, den = 0;
    for (long long l = 0; l < tree.n_leaves(); ++l)
      for (int i = 0; i < p * p; ++i) {
        Point x;
        const size_t k = size_t(l * p * p + i);
        x[0] = xyz[3 * k], x[1] = xyz[3 * k + 1];
        num = std::fmax(num, std::abs(field.u[size_t(l)][size_t(i)] - u(x)));
        den = std::fmax(den, std::abs(u(x)));
      }
    std::printf("{\"L\": %d, \"p\": %d, \"rel_linf\": %.3e}\n", L, p, num / den);
    return 0;
  } catch (const Error& e) {
    std::fprintf(stderr, "hps::b200::Error: %s\n", e.what());
    return 1;
  }
}
