"""ctypes wrapper of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Loaded by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs as
the parity checker / timed CPU baseline.  The B200 product
(paper_2503_17535_b200) never imports this module.

The oracle is a C++ restatement of the reference HPS hot path (see
oracle/hps_oracle.hpp for the file:line citations and the parity-pinning
statement).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

FIELD_CONST, FIELD_BUMPS, FIELD_PLANE_SIN, FIELD_PLANE_COS, FIELD_BUMPS_SIN, FIELD_POISSON2D_SRC, FIELD_SAMPLED, \
    FIELD_BUMPS_GRAD, FIELD_DIVGRAD_SRC = range(9)
ROLE_LAPLACIAN, ROLE_GRADIENT, ROLE_ZEROTH, ROLE_SECOND_ORDER = range(4)


class Field(C.Structure):
    _fields_ = [("kind", C.c_int), ("n_centers", C.c_int), ("c", C.c_double * 8),
                ("centers", C.POINTER(C.c_double)), ("samples", C.POINTER(C.c_double))]


class Term(C.Structure):
    _fields_ = [("role", C.c_int), ("axis", C.c_int), ("axis2", C.c_int), ("field", Field)]


_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int)
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_create.restype = C.c_void_p
        L.oracle_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.POINTER(Term), C.c_int,
                                    C.POINTER(Field), C.c_int, C.c_int, C.c_int]
        for name in ["oracle_destroy", "oracle_build", "oracle_n_leaves", "oracle_n_nodes", "oracle_root_bsize"]:
            getattr(L, name).argtypes = [C.c_void_p]
        L.oracle_root_points.argtypes = [C.c_void_p, dp]
        L.oracle_leaf_points.argtypes = [C.c_void_p, dp]
        L.oracle_discretize.argtypes = [C.c_void_p, C.c_int, dp, dp]
        L.oracle_solve.argtypes = [C.c_void_p, dp, dp, dp]
        L.oracle_get_leaf.argtypes = [C.c_void_p, C.c_int, dp, dp, dp, dp]
        L.oracle_node_sizes.argtypes = [C.c_void_p, C.c_int, ip, ip]
        L.oracle_get_node.argtypes = [C.c_void_p, C.c_int, dp, dp, dp, dp]
        L.oracle_level_nodes.argtypes = [C.c_void_p, C.c_int, ip]
        L.oracle_min_rcond.restype = C.c_double
        L.oracle_min_rcond.argtypes = [C.c_void_p]
        L.oracle_times.argtypes = [C.c_void_p, dp, dp]
        L.oracle_bump_centers.argtypes = [C.c_ulonglong, C.c_int, C.c_int, dp]
        L.oracle_cheb_lobatto.argtypes = [C.c_int, dp]
        L.oracle_cheb_weights.argtypes = [C.c_int, dp]
        L.oracle_gauss.argtypes = [C.c_int, dp, dp]
        L.oracle_diff_matrix.argtypes = [C.c_int, dp]
        L.oracle_interp_matrix.argtypes = [dp, C.c_int, dp, C.c_int, dp]
        L.oracle_dtn_ops.argtypes = [C.c_int, C.c_int, C.c_double, dp, dp, ip, ip, ip, ip]
        L.oracle_index_sets.argtypes = [C.c_int, C.c_int, ip, ip]
        L.oracle_leaf_cheb_points.argtypes = [dp, dp, C.c_int, C.c_int, dp]
        L.oracle_gauss_boundary_points.argtypes = [dp, dp, C.c_int, C.c_int, dp]
        L.oracle_face_projection.argtypes = [C.c_int, dp, dp]
        L.oracle_refinement_interpolant.argtypes = [C.c_int, dp]
        L.oracle_tree_info.argtypes = [C.c_int, C.c_int, C.c_int, dp, dp, ip, ip, C.POINTER(C.c_longlong), ip, ip, ip]
        L.oracle_set_threads.argtypes = [C.c_int]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int)) if a is not None else None


def err():
    return lib().oracle_last_error().decode()


def check(rc):
    if rc != 0:
        raise RuntimeError("oracle: " + err())


# ---------------------------------------------------------------- KAT helpers
def cheb_lobatto(p):
    out = np.zeros(p)
    lib().oracle_cheb_lobatto(p, _dp(out))
    return out


def cheb_weights(p):
    out = np.zeros(p)
    lib().oracle_cheb_weights(p, _dp(out))
    return out


def gauss(q):
    n, w = np.zeros(q), np.zeros(q)
    check(lib().oracle_gauss(q, _dp(n), _dp(w)))
    return n, w


def diff_matrix(p):
    out = np.zeros(p * p)
    lib().oracle_diff_matrix(p, _dp(out))
    return out.reshape(p, p, order="F")


def interp_matrix(src, dst):
    src = np.ascontiguousarray(src, dtype=np.float64)
    dst = np.ascontiguousarray(dst, dtype=np.float64)
    out = np.zeros(len(src) * len(dst))
    check(lib().oracle_interp_matrix(_dp(src), len(src), _dp(dst), len(dst), _dp(out)))
    return out.reshape(len(dst), len(src), order="F")


def dtn_ops(dim, p, side=2.0):
    pr, pc, qr, qc = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    check(lib().oracle_dtn_ops(dim, p, side, None, None, C.byref(pr), C.byref(pc), C.byref(qr), C.byref(qc)))
    P, Q = np.zeros(pr.value * pc.value), np.zeros(qr.value * qc.value)
    check(lib().oracle_dtn_ops(dim, p, side, _dp(P), _dp(Q), C.byref(pr), C.byref(pc), C.byref(qr), C.byref(qc)))
    return P.reshape(pr.value, pc.value, order="F"), Q.reshape(qr.value, qc.value, order="F")


def index_sets(p, dim):
    n = p ** dim
    ni = (p - 2) ** dim
    ii, ie = np.zeros(ni, np.int32), np.zeros(n - ni, np.int32)
    check(lib().oracle_index_sets(p, dim, _ip(ii), _ip(ie)))
    return ii, ie


def leaf_cheb_points(lo, hi, p, dim):
    lo, hi = np.asarray(lo, np.float64), np.asarray(hi, np.float64)
    out = np.zeros(p ** dim * 3)
    lib().oracle_leaf_cheb_points(_dp(lo), _dp(hi), p, dim, _dp(out))
    return out.reshape(-1, 3)


def gauss_boundary_points(lo, hi, q, dim):
    lo, hi = np.asarray(lo, np.float64), np.asarray(hi, np.float64)
    out = np.zeros(2 * dim * q ** (dim - 1) * 3)
    lib().oracle_gauss_boundary_points(_dp(lo), _dp(hi), q, dim, _dp(out))
    return out.reshape(-1, 3)


def face_projection(q):
    r, c = np.zeros(4 * q ** 4), np.zeros(4 * q ** 4)
    check(lib().oracle_face_projection(q, _dp(r), _dp(c)))
    return r.reshape(4 * q * q, q * q, order="F"), c.reshape(q * q, 4 * q * q, order="F")


def refinement_interpolant(p):
    pc = p ** 3
    out = np.zeros(8 * pc * pc)
    check(lib().oracle_refinement_interpolant(p, _dp(out)))
    return out.reshape(8 * pc, pc, order="F")


def tree_info(dim, L, p, lo, hi):
    lo, hi = np.asarray(lo, np.float64), np.asarray(hi, np.float64)
    nn, nl, tp = C.c_int(), C.c_int(), C.c_longlong()
    check(lib().oracle_tree_info(dim, L, p, _dp(lo), _dp(hi), C.byref(nn), C.byref(nl), C.byref(tp), None, None, None))
    leaves = np.zeros(nl.value, np.int32)
    depth, parent = np.zeros(nn.value, np.int32), np.zeros(nn.value, np.int32)
    check(lib().oracle_tree_info(dim, L, p, _dp(lo), _dp(hi), C.byref(nn), C.byref(nl), C.byref(tp), _ip(leaves),
                                 _ip(depth), _ip(parent)))
    return dict(n_nodes=nn.value, n_leaves=nl.value, total_points=tp.value, leaves=leaves, depth=depth, parent=parent)


def bump_centers(seed, n=10, dim=2):
    out = np.zeros(3 * n)
    lib().oracle_bump_centers(seed, n, dim, _dp(out))
    return out.reshape(n, 3)


def set_threads(n):
    lib().oracle_set_threads(n)


# ---------------------------------------------------------------- problems
def make_field(kind, c=(), centers=None, samples=None):
    """Returns (Field, keepalive list)."""
    f = Field()
    f.kind = kind
    for i, v in enumerate(c):
        f.c[i] = v
    keep = []
    if centers is not None:
        centers = np.ascontiguousarray(centers, dtype=np.float64).reshape(-1, 3)
        f.n_centers = centers.shape[0]
        f.centers = _dp(centers)
        keep.append(centers)
    if samples is not None:
        samples = np.ascontiguousarray(samples, dtype=np.float64)
        f.samples = _dp(samples)
        keep.append(samples)
    return f, keep


class Solver:
    """Oracle HpsSolver<Real> (DtN) over a uniform tree on [lo,hi]^dim.

    terms: list of (role, axis, axis2, Field) ; source: Field or None.
    """

    def __init__(self, dim, p, L, lo, hi, terms, source, literal_sign=True, root_implicit=False, parallel=False,
                 keep=()):
        self.keep = list(keep)
        arr = (Term * len(terms))()
        for i, (role, axis, axis2, fld) in enumerate(terms):
            arr[i].role, arr[i].axis, arr[i].axis2, arr[i].field = role, axis, axis2, fld
        self._terms = arr
        self._src = source
        self.dim, self.p, self.L = dim, p, L
        self.h = lib().oracle_create(dim, p, L, lo, hi, arr, len(terms), C.byref(source) if source is not None else None,
                                     int(literal_sign), int(root_implicit), int(parallel))
        if not self.h:
            raise RuntimeError("oracle_create: " + err())
        self.n_leaves = lib().oracle_n_leaves(self.h)
        self.n_nodes = lib().oracle_n_nodes(self.h)
        self.npts = p ** dim
        self.nb = lib().oracle_root_bsize(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().oracle_destroy(self.h)
            self.h = None

    def build(self):
        check(lib().oracle_build(self.h))

    def times(self):
        a, b = C.c_double(), C.c_double()
        lib().oracle_times(self.h, C.byref(a), C.byref(b))
        return a.value, b.value

    def min_rcond(self):
        return lib().oracle_min_rcond(self.h)

    def root_points(self):
        out = np.zeros(self.nb * 3)
        check(lib().oracle_root_points(self.h, _dp(out)))
        return out.reshape(-1, 3)

    def leaf_points(self):
        out = np.zeros(self.n_leaves * self.npts * 3)
        check(lib().oracle_leaf_points(self.h, _dp(out)))
        return out.reshape(self.n_leaves, self.npts, 3)

    def discretize(self, ord_):
        lm, f = np.zeros(self.npts * self.npts), np.zeros(self.npts)
        check(lib().oracle_discretize(self.h, ord_, _dp(lm), _dp(f)))
        return lm.reshape(self.npts, self.npts, order="F"), f

    def solve(self, g, want_leaf_g=False):
        g = np.ascontiguousarray(g, dtype=np.float64)
        assert g.shape == (self.nb,)
        u = np.zeros(self.n_leaves * self.npts)
        nbl = 2 * self.dim * (self.p - 2) ** (self.dim - 1)
        lg = np.zeros(self.n_leaves * nbl) if want_leaf_g else None
        check(lib().oracle_solve(self.h, _dp(g), _dp(u), _dp(lg)))
        u = u.reshape(self.n_leaves, self.npts)
        return (u, lg.reshape(self.n_leaves, nbl)) if want_leaf_g else u

    def get_leaf(self, ord_):
        q = self.p - 2
        nbl = 2 * self.dim * q ** (self.dim - 1)
        Y, v, T, h = np.zeros(self.npts * nbl), np.zeros(self.npts), np.zeros(nbl * nbl), np.zeros(nbl)
        check(lib().oracle_get_leaf(self.h, ord_, _dp(Y), _dp(v), _dp(T), _dp(h)))
        return Y.reshape(self.npts, nbl, order="F"), v, T.reshape(nbl, nbl, order="F"), h

    def node_sizes(self, nid):
        a, b = C.c_int(), C.c_int()
        check(lib().oracle_node_sizes(self.h, nid, C.byref(a), C.byref(b)))
        return a.value, b.value

    def get_node(self, nid, root_implicit=False):
        ne, ni = self.node_sizes(nid)
        S = np.zeros(ni * ne) if not (nid == 0 and root_implicit) else None
        gt = np.zeros(ni)
        T = np.zeros(ne * ne) if nid != 0 else None
        h = np.zeros(ne) if nid != 0 else None
        check(lib().oracle_get_node(self.h, nid, _dp(S), _dp(gt), _dp(T), _dp(h)))
        return (S.reshape(ni, ne, order="F") if S is not None else None, gt,
                T.reshape(ne, ne, order="F") if T is not None else None, h)

    def level_nodes(self, depth):
        n = lib().oracle_level_nodes(self.h, depth, None)
        ids = np.zeros(n, np.int32)
        lib().oracle_level_nodes(self.h, depth, _ip(ids))
        return ids
