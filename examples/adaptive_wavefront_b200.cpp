// adaptive_wavefront_b200.cpp -- the reference's adaptive 3D flow (solve_problem with Discretization::adaptive,
// proj/src/problems.cpp:360-392) through the C++ drop-in: refine_adaptive on the wavefront source
// (make_wavefront_3d, problems.cpp:154-179), an HpsSolver on the resulting level-restricted octree (nonuniform
// merges on the B200), Dirichlet data from the exact front, error against it.  Prints one JSON line.
//   usage: adaptive_wavefront_b200 [p=8] [tol=3e-4] [max_depth=5]
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "hps/hps_b200.hpp"

using namespace hps::b200;

int main(int argc, char** argv) {
  const int p = argc > 1 ? std::atoi(argv[1]) : 8;
  const double tol = argc > 2 ? std::atof(argv[2]) : 3e-4;
  const int max_depth = argc > 3 ? std::atoi(argv[3]) : 5;
  try {
    const double a = 30.0;  // kWavefrontAlpha (problems.cpp:34)
    auto rho2 = [](const Point& x) {
      const double d0 = x[0] - 0.5, d1 = x[1] - 0.5, d2 = x[2] - 0.5;
      return d0 * d0 + d1 * d1 + d2 * d2;
    };
    auto u = [&](const Point& x) { return std::atan(a * rho2(x) - 0.7); };
    auto lap = [&](const Point& x) {
      const double w = a * rho2(x) - 0.7, s = 1.0 + w * w;
      return -2.0 * w / (s * s) * 4.0 * a * a * rho2(x) + 6.0 * a / s;
    };
    Box dom;
    dom.lo[0] = dom.lo[1] = dom.lo[2] = 0.0;
    dom.hi[0] = dom.hi[1] = dom.hi[2] = 1.0;
    const auto t0 = std::chrono::steady_clock::now();
    RefinementCriterion crit;
    crit.tol = tol;
    crit.p = p;
    crit.test_fields.push_back(lap);
    std::vector<int> unresolved;
    DiscretizationTree tree = refine_adaptive(dom, crit, max_depth, &unresolved);
    const auto t1 = std::chrono::steady_clock::now();
    std::vector<CoefficientField> terms{{CoefficientField::Role::laplacian, -1, -1, [](const Point&) { return 1.0; }}};
    SolverOptions opts;
    opts.literal_sign = false;    // corrected DtN sign (the reference's literal sign solves L u = -f)
    opts.root_implicit_S = true;  // solve_problem's 3D setting (problems.cpp:383-386)
    HpsSolver solver(tree, Variant::dtn, 1.0, terms, lap, opts);
    solver.build();
    const auto t2 = std::chrono::steady_clock::now();
    const SolutionField field = solver.solve(solver.sample_root_data(u));
    const auto t3 = std::chrono::steady_clock::now();
    const std::vector<Point> pts = leaf_cheb_points(tree);
    const int np = p * p * p;
    double num = 0, den = 0;
    for (int l = 0; l < tree.n_leaves(); ++l)
      for (int i = 0; i < np; ++i) {
        const Point& x = pts[size_t(l) * np + size_t(i)];
        num = std::fmax(num, std::fabs(field.u[size_t(l)][size_t(i)] - u(x)));
        den = std::fmax(den, std::fabs(u(x)));
      }
    int maxd = 0;
    for (int id : tree.leaves) maxd = std::max(maxd, tree.nodes[size_t(id)].depth);
    auto s = [](auto x, auto y) { return std::chrono::duration<double>(y - x).count(); };
    std::printf("{\"p\": %d, \"tol\": %g, \"n_leaves\": %d, \"N\": %lld, \"max_leaf_depth\": %d, \"top_D\": %d, "
                "\"unresolved\": %d, \"rel_linf\": %.3e, \"t_mesh_s\": %.3f, \"t_build_s\": %.4f, \"t_solve_s\": %.4f, "
                "\"mesh_json_bytes\": %zu}\n",
                p, tol, tree.n_leaves(), tree.total_points(), maxd, solver.top_D_size(), int(unresolved.size()),
                num / den, s(t0, t1), s(t1, t2), s(t2, t3), mesh_to_json(tree).size());
    return 0;
  } catch (const Error& e) {
    std::fprintf(stderr, "hps::b200::Error: %s\n", e.what());
    return 1;
  }
}
