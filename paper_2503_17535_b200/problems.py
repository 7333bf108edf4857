"""Problem catalog for the B200 HPS solver (mirrors proj/src/problems.cpp).

Each problem is a ProblemSpec-like record: operator terms and source as device
field descriptors (hps.Field), Dirichlet boundary data and, where manufactured,
the exact solution as numpy callables on (..., 3) point arrays.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

from .hps import (FIELD_BUMPS, FIELD_BUMPS_GRAD, FIELD_BUMPS_SIN, FIELD_CONST, FIELD_DIVGRAD_SRC, FIELD_PB_EPS,
                  FIELD_PB_EPS_GRAD, FIELD_PLANE_COS, FIELD_PLANE_SIN, FIELD_POISSON2D_SRC, FIELD_WAVEFRONT_SRC,
                  ROLE_GRADIENT, ROLE_LAPLACIAN, ROLE_ZEROTH, Field, Term)
from .seeded import bump_centers  # pure Python: defining a problem never loads a shared object


@dataclass
class Problem:
    name: str
    dim: int
    lo: float
    hi: float
    terms: list
    source: Field | None
    boundary: Callable  # x (...,3) -> values
    exact: Callable | None = None


def poisson2d() -> Problem:
    """make_manufactured_2d_dtn, proj/src/problems.cpp:40-74:
    Delta u - cos(5 x2) d1 u + sin(5 x2) d2 u = f, u = e^{5x1} sin 5x2 + sin(10 pi x1) sin(pi x2)."""
    def u(x):
        return np.exp(5 * x[..., 0]) * np.sin(5 * x[..., 1]) + np.sin(10 * np.pi * x[..., 0]) * np.sin(np.pi * x[..., 1])

    terms = [Term(ROLE_LAPLACIAN, Field(FIELD_CONST, (1.0,))),
             Term(ROLE_GRADIENT, Field(FIELD_PLANE_COS, (-1.0, 0.0, 5.0, 0.0, 0.0)), axis=0),
             Term(ROLE_GRADIENT, Field(FIELD_PLANE_SIN, (1.0, 0.0, 5.0, 0.0, 0.0)), axis=1)]
    return Problem("poisson2d", 2, -1.0, 1.0, terms, Field(FIELD_POISSON2D_SRC), u, u)


def helmholtz_bumps(k=30.0, seed=7, n_bumps=10, alpha=50.0, phase=0.3) -> Problem:
    """Headline config 2 (BASELINE.json configs[1]): variable-coefficient Helmholtz on [-1,1]^2,

        Delta u + k^2 (1 + q(x)) u = f,   q = sum_j exp(-alpha |x - z_j|^2),

    q is the seeded random-bump potential of make_scattering (proj/src/problems.cpp:126-141,
    centers from std::mt19937_64(seed)).  Manufactured from the plane wave
    u = sin(k x1 + phase): f = k^2 q u, Dirichlet data u on the boundary.

    k = 30 is chosen away from Dirichlet resonances of the node boxes: the roundoff floor of
    the exact-solution error grows ~4x per level for every k, and is ~20x higher at k = 20
    (oracle, p=16: 1.2e-9 at L=6 for k=20 vs 1.9e-11 for k=30).
    """
    z = bump_centers(seed, n_bumps, 2)
    k2 = k * k
    terms = [Term(ROLE_LAPLACIAN, Field(FIELD_CONST, (1.0,))),
             Term(ROLE_ZEROTH, Field(FIELD_BUMPS, (k2, k2, alpha), centers=z))]
    src = Field(FIELD_BUMPS_SIN, (k2, 0.0, alpha, k, 0.0, 0.0, phase), centers=z)

    def u(x):
        return np.sin(k * x[..., 0] + phase)

    return Problem(f"helmholtz_bumps(k={k:g},seed={seed})", 2, -1.0, 1.0, terms, src, u, u)


def laplace_poly2d() -> Problem:
    """Harmonic polynomial u = x^3 - 3 x y^2 + x y (f = 0): HPS is exact up to roundoff."""
    def u(x):
        return x[..., 0] ** 3 - 3 * x[..., 0] * x[..., 1] ** 2 + x[..., 0] * x[..., 1]

    return Problem("laplace_poly2d", 2, -1.0, 1.0, [Term(ROLE_LAPLACIAN, Field(FIELD_CONST, (1.0,)))], None, u, u)


def poisson3d_const() -> Problem:
    """3D Laplace with the harmonic cubic u = x^3 - 3 x y^2 + z^2 - x^2 + x y z on [0,1]^3 (exact for q >= 4)."""
    def u(x):
        X, Y, Z = x[..., 0], x[..., 1], x[..., 2]
        return X ** 3 - 3 * X * Y ** 2 + Z ** 2 - X ** 2 + X * Y * Z

    return Problem("laplace3d", 3, 0.0, 1.0, [Term(ROLE_LAPLACIAN, Field(FIELD_CONST, (1.0,)))], None, u, u)


def poisson3d_var(seed=11, n_bumps=5, amp=0.5, alpha=4.0, omega=2.0, phase=0.5) -> Problem:
    """BASELINE.json configs[3]: 3D variable-coefficient Poisson div(eps grad u) = f on [-1,1]^3
    (roles laplacian = eps, gradient_a = d_a eps), eps = 1 + amp * sum_j exp(-alpha |x - z_j|^2)
    with seeded centers (std::mt19937_64, proj/src/problems.cpp:126-141), manufactured
    u = prod_k sin(omega x_k + phase)."""
    z = bump_centers(seed, n_bumps, 3)
    terms = [Term(ROLE_LAPLACIAN, Field(FIELD_BUMPS, (1.0, amp, alpha), centers=z))]
    terms += [Term(ROLE_GRADIENT, Field(FIELD_BUMPS_GRAD, (0.0, amp, alpha, float(a)), centers=z), axis=a)
              for a in range(3)]
    src = Field(FIELD_DIVGRAD_SRC, (1.0, amp, alpha, omega, phase), centers=z)

    def u(x):
        return np.sin(omega * x[..., 0] + phase) * np.sin(omega * x[..., 1] + phase) * np.sin(omega * x[..., 2] + phase)

    return Problem("poisson3d_var", 3, -1.0, 1.0, terms, src, u, u)


def wavefront3d(alpha=30.0) -> Problem:
    """make_wavefront_3d (proj/src/problems.cpp:154-179): Laplace(u) = f on [0,1]^3 with the spherical front
    u = atan(alpha |x - c|^2 - 0.7), c = (1/2, 1/2, 1/2), Dirichlet data from u.  The paper's Table 1 problem
    (adaptive octrees); its refinement field is the source."""
    def u(x):
        r2 = ((x[..., :3] - 0.5) ** 2).sum(axis=-1)
        return np.arctan(alpha * r2 - 0.7)

    src = Field(FIELD_WAVEFRONT_SRC, (alpha, 0.5, 0.5, 0.5))
    return Problem("wavefront3d", 3, 0.0, 1.0, [Term(ROLE_LAPLACIAN, Field(FIELD_CONST, (1.0,)))], src, u, u)


def poisson_boltzmann3d(seed=20260810, n_centers=50, delta=45.0, eps0=16.0, eps_inf=100.0, amp=10.0) -> Problem:
    """make_poisson_boltzmann with the smooth permittivity (proj/src/problems.cpp:181-253):
    eps Lap(u) + grad(eps).grad(u) = -rho on [-1,1]^3, u = 0 on the boundary, rho = sum_j exp(-delta |x - z_j|^2)
    over 50 seeded centers (make_pb_spec: std::mt19937_64, U(-1/2, 1/2)), eps = eps0 + (eps_inf - eps0) exp(-amp rho).
    No closed-form solution (accuracy is judged by self-convergence)."""
    z = bump_centers(seed, n_centers, 3)
    c = (eps0, eps_inf, amp, delta)
    terms = [Term(ROLE_LAPLACIAN, Field(FIELD_PB_EPS, c, centers=z))]
    terms += [Term(ROLE_GRADIENT, Field(FIELD_PB_EPS_GRAD, c + (float(a),), centers=z), axis=a) for a in range(3)]
    src = Field(FIELD_BUMPS, (0.0, -1.0, delta), centers=z)
    return Problem("poisson_boltzmann3d", 3, -1.0, 1.0, terms, src, lambda x: np.zeros(x.shape[:-1]), None)


CATALOG = {"poisson2d": poisson2d, "helmholtz_bumps": helmholtz_bumps, "laplace_poly2d": laplace_poly2d,
           "laplace3d": poisson3d_const, "poisson3d_var": poisson3d_var, "wavefront3d": wavefront3d,
           "poisson_boltzmann3d": poisson_boltzmann3d}


def rel_linf(u, ref):
    """error_report rel L-inf (proj/src/problems.cpp:270-293)."""
    return float(np.abs(u - ref).max() / np.abs(ref).max())


# ---- ItI problems (proj/src/problems.cpp:76-152) -------------------------------------------------
@dataclass
class ItiProblem:
    name: str
    eta: float
    terms: list
    source_re: Field | None
    source_im: Field | None
    impedance: Callable | None   # (points) -> incoming impedance data du/dn + i eta u (None: radiation)
    exact: Callable | None = None
    lo: float = -1.0
    hi: float = 1.0
    dim: int = 2


def _impedance(x, u, grad, eta):
    """du/dn + i eta u on the root boundary points (faces S, E, N, W of the square)."""
    nb = len(x)
    side = np.repeat(np.arange(4), nb // 4)
    nrm = np.array([[0, -1], [1, 0], [0, 1], [-1, 0]], dtype=float)[side]
    gx, gy = grad(x)
    return nrm[:, 0] * gx + nrm[:, 1] * gy + 1j * eta * u(x)


def helmholtz_robin2d(tree) -> ItiProblem:
    """make_manufactured_2d_iti (problems.cpp:76-107): Delta u + (1 + exp(-50|x|^2)) u = f with
    u = e^{20 i x1} + e^{30 i x2}, impedance data (eta = 1).  The complex source is sampled at the
    leaf points of `tree` (SPEC.md:545 gate: p=16 L=4 rel Linf < 1e-6)."""
    from .hps import FIELD_SAMPLED, tree_leaf_points_of
    q = Field(FIELD_BUMPS, (1.0, 1.0, 50.0), centers=np.zeros((1, 3)))
    terms = [Term(ROLE_LAPLACIAN, Field(FIELD_CONST, (1.0,))), Term(ROLE_ZEROTH, q)]

    def u(x):
        return np.exp(20j * x[..., 0]) + np.exp(30j * x[..., 1])

    def grad(x):
        return 20j * np.exp(20j * x[..., 0]), 30j * np.exp(30j * x[..., 1])

    pts = tree_leaf_points_of(tree)
    qv = 1.0 + np.exp(-50.0 * (pts[..., 0] ** 2 + pts[..., 1] ** 2))
    f = -400.0 * np.exp(20j * pts[..., 0]) - 900.0 * np.exp(30j * pts[..., 1]) + qv * u(pts)
    return ItiProblem("helmholtz_robin2d", 1.0, terms, Field(FIELD_SAMPLED, samples=np.ascontiguousarray(f.real)),
                      Field(FIELD_SAMPLED, samples=np.ascontiguousarray(f.imag)),
                      lambda x: _impedance(x, u, grad, 1.0), u)


def scatter2d(k=20.0, seed=7) -> ItiProblem:
    """make_scattering (problems.cpp:109-152): Delta u + k^2 (1 + q) u = -k^2 q e^{i k x1}, q = ten seeded
    Gaussian bumps exp(-50 |x - z|^2), radiation closure at the root (eta = k)."""
    z = bump_centers(seed, 10, 2)
    k2 = k * k
    terms = [Term(ROLE_LAPLACIAN, Field(FIELD_CONST, (1.0,))),
             Term(ROLE_ZEROTH, Field(FIELD_BUMPS, (k2, k2, 50.0), centers=z))]
    # -k^2 q (cos k x1 + i sin k x1): BUMPS_SIN with phases pi/2 (cos) and 0 (sin)
    src_re = Field(FIELD_BUMPS_SIN, (-k2, 0.0, 50.0, k, 0.0, 0.0, np.pi / 2), centers=z)
    src_im = Field(FIELD_BUMPS_SIN, (-k2, 0.0, 50.0, k, 0.0, 0.0, 0.0), centers=z)
    return ItiProblem(f"scatter2d(k={k:g},seed={seed})", k, terms, src_re, src_im, None)
