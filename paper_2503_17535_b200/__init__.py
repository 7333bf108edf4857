"""B200-native HPS fast direct solver (arxiv 2503.17535), drop-in for the
reference HpsSolver<Real> DtN build/solve path.

Product code: hand-written sm_100a CUDA (csrc/) behind the C-ABI in
include/hps_cuda.h, compiled to libhps_b200.so; this package is the Python
host mirror of the reference API (hps.py) plus the problem catalog
(problems.py).
"""
from .hps import (FIELD_BUMPS, FIELD_BUMPS_SIN, FIELD_CONST, FIELD_PLANE_COS, FIELD_PLANE_SIN,  # noqa: F401
                  FIELD_POISSON2D_SRC, FIELD_SAMPLED, ROLE_GRADIENT, ROLE_LAPLACIAN, ROLE_SECOND_ORDER, ROLE_ZEROTH,
                  Field, HpsError, HpsSolver, Term, UniformTree, build_library, build_uniform_tree, bump_centers,
                  estimate_bytes, lib,
                  tree_root_points)
from . import problems  # noqa: F401
