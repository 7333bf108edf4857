// field_eval.hpp -- TEST INFRASTRUCTURE ONLY: closed-form coefficient/source fields of the oracle_field
// descriptors (oracle_capi.h), shared by the restatement (oracle_capi.cpp) and the reference build's
// std::function closures (ref_capi.cpp).  Same formulas as the product's device fields (hpsg_field).
#ifndef HPS_ORACLE_FIELD_EVAL_HPP
#define HPS_ORACLE_FIELD_EVAL_HPP

#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "oracle_capi.h"

namespace hpso_fields {

struct FieldEval {
  oracle_field f{};
  std::vector<double> centers, samples;
  int dim = 2, npts = 0;
  template <class P>
  double bumps(const P& x) const {
    double s = 0.0;
    for (int j = 0; j < f.n_centers; ++j) {
      double r2 = 0.0;
      for (int k = 0; k < dim; ++k) {
        const double d = x[k] - centers[3 * j + k];
        r2 += d * d;
      }
      s += std::exp(-f.c[2] * r2);
    }
    return s;
  }
  template <class P>
  double operator()(const P& x, int leaf, int pt) const {
    const double* c = f.c;
    switch (f.kind) {
      case ORACLE_FIELD_CONST: return c[0];
      case ORACLE_FIELD_BUMPS: return c[0] + c[1] * bumps(x);
      case ORACLE_FIELD_PLANE_SIN: return c[0] * std::sin(c[1] * x[0] + c[2] * x[1] + c[3] * x[2] + c[4]);
      case ORACLE_FIELD_PLANE_COS: return c[0] * std::cos(c[1] * x[0] + c[2] * x[1] + c[3] * x[2] + c[4]);
      case ORACLE_FIELD_BUMPS_SIN:
        return c[0] * bumps(x) * std::sin(c[3] * x[0] + c[4] * x[1] + c[5] * x[2] + c[6]);
      case ORACLE_FIELD_POISSON2D_SRC: {
        // proj/src/problems.cpp:50-66
        const double X = x[0], Y = x[1];
        const double ux = 5.0 * std::exp(5.0 * X) * std::sin(5.0 * Y) +
                          10.0 * M_PI * std::cos(10.0 * M_PI * X) * std::sin(M_PI * Y);
        const double uy = 5.0 * std::exp(5.0 * X) * std::cos(5.0 * Y) +
                          M_PI * std::sin(10.0 * M_PI * X) * std::cos(M_PI * Y);
        const double lap = -101.0 * M_PI * M_PI * std::sin(10.0 * M_PI * X) * std::sin(M_PI * Y);
        return lap - std::cos(5.0 * Y) * ux + std::sin(5.0 * Y) * uy;
      }
      case ORACLE_FIELD_SAMPLED: return samples[size_t(leaf) * npts + pt];
      case ORACLE_FIELD_BUMPS_GRAD: {
        const int a = int(c[3]);
        double s = 0.0;
        for (int j = 0; j < f.n_centers; ++j) {
          double r2 = 0.0;
          for (int k = 0; k < dim; ++k) {
            const double d = x[k] - centers[3 * j + k];
            r2 += d * d;
          }
          s += -2.0 * c[2] * (x[a] - centers[3 * j + a]) * std::exp(-c[2] * r2);
        }
        return c[1] * s;
      }
      case ORACLE_FIELD_DIVGRAD_SRC: {
        double sn[3], cs[3], u = 1.0;
        for (int k = 0; k < dim; ++k) sn[k] = std::sin(c[3] * x[k] + c[4]), cs[k] = std::cos(c[3] * x[k] + c[4]), u *= sn[k];
        double eps = c[0], geps[3] = {0.0, 0.0, 0.0};
        for (int j = 0; j < f.n_centers; ++j) {
          double r2 = 0.0;
          for (int k = 0; k < dim; ++k) {
            const double d = x[k] - centers[3 * j + k];
            r2 += d * d;
          }
          const double e = std::exp(-c[2] * r2);
          eps += c[1] * e;
          for (int k = 0; k < dim; ++k) geps[k] += c[1] * -2.0 * c[2] * (x[k] - centers[3 * j + k]) * e;
        }
        double f2 = -dim * c[3] * c[3] * u * eps;
        for (int k = 0; k < dim; ++k) {
          double du = c[3] * cs[k];
          for (int l = 0; l < dim; ++l)
            if (l != k) du *= sn[l];
          f2 += geps[k] * du;
        }
        return f2;
      }
      default: throw std::runtime_error("oracle: unknown field kind " + std::to_string(f.kind));
    }
  }
};

}  // namespace hpso_fields

#endif
