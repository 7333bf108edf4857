"""ctypes wrapper of oracle/_ref/libhps_ref.so -- TEST INFRASTRUCTURE ONLY.

libhps_ref.so is the reference's own hot path (/root/reference/proj/src, unmodified) compiled against
the Eigen-API shim (oracle/eigen_shim) by oracle/Makefile.ref, behind the marshalling wrapper
oracle/ref_capi.cpp.  Loaded only by tests/ and bench.py's reference arm, as the checker / the timed
reference.  The B200 product (paper_2503_17535_b200) never imports this module.

The library is built in the development container (where /root/reference exists) and travels to the
GPU box as a file; `available()` is False where neither the library nor the sources exist.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from oracle.oracle import Field, Term, make_field  # noqa: F401  (same descriptors as the oracle)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libhps_ref.so")
REF_SRC = "/root/reference/proj/src"

_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE, "-f", "Makefile.ref", "-j", str(min(8, os.cpu_count() or 1))],
                   check=True)


def available():
    return os.path.exists(LIB_PATH) or os.path.isdir(REF_SRC)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        dp, ip, vp = C.POINTER(C.c_double), C.POINTER(C.c_int), C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_set_threads.argtypes = [C.c_int]
        L.ref_create.restype = vp
        L.ref_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.POINTER(Term), C.c_int,
                                 C.POINTER(Field), C.POINTER(Field), C.c_int, C.c_double, C.c_int, C.c_int]
        L.ref_create_problem.restype = vp
        L.ref_create_problem.argtypes = [C.c_char_p, C.c_double, C.c_uint, C.c_int, C.c_int, C.c_int, C.c_double,
                                         C.c_int, C.c_int]
        for name in ["ref_destroy", "ref_build", "ref_is_complex", "ref_n_leaves", "ref_n_nodes", "ref_dim", "ref_p",
                     "ref_root_bsize", "ref_top_D_size", "ref_n_unresolved", "ref_any_ill_conditioned"]:
            getattr(L, name).argtypes = [vp]
        L.ref_tree.argtypes = [vp, ip, ip, ip, ip, dp, dp, C.POINTER(C.c_longlong), ip]
        L.ref_root_points.argtypes = [vp, dp]
        L.ref_leaf_points.argtypes = [vp, dp]
        L.ref_sample_root_data.argtypes = [vp, dp]
        L.ref_solve.argtypes = [vp, dp, dp, dp]
        L.ref_solve_radiation.argtypes = [vp, dp]
        L.ref_solve_new_source.argtypes = [vp, dp, C.c_int, dp, dp]
        L.ref_get_leaf.argtypes = [vp, C.c_int, dp, dp, dp, dp]
        L.ref_node_sizes.argtypes = [vp, C.c_int, ip, ip]
        L.ref_get_node.argtypes = [vp, C.c_int, dp, dp, dp, dp]
        L.ref_error_report.argtypes = [vp, dp, dp, dp]
        L.ref_min_rcond.restype = C.c_double
        L.ref_min_rcond.argtypes = [vp]
        L.ref_times.argtypes = [vp, dp, dp]
        L.ref_solve_problem.argtypes = [C.c_char_p, C.c_double, C.c_uint, C.c_int, C.c_int, C.c_int, C.c_double,
                                        C.c_int, dp]
        L.ref_bench_sample.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.POINTER(Term), C.c_int,
                                       C.POINTER(Field), C.c_int, dp]
        L.ref_mesh_json.restype = C.c_longlong
        L.ref_mesh_json.argtypes = [vp, C.c_char_p, C.c_longlong]
        L.ref_dump_solution.argtypes = [vp, dp, C.c_char_p, C.c_char_p, C.c_char_p]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int)) if a is not None else None


def check(rc):
    if rc != 0:
        raise RuntimeError("reference: " + lib().ref_last_error().decode())


def set_threads(n):
    lib().ref_set_threads(n)


def _as_doubles(x, cplx):
    x = np.ascontiguousarray(x, dtype=np.complex128 if cplx else np.float64)
    return x.view(np.float64) if cplx else x


def solve_problem(name, p, L=3, adaptive=False, tol=1e-3, max_depth=10, k=0.0, seed=7):
    """The reference's end-to-end driver solve_problem (problems.cpp:360-422)."""
    out = np.zeros(8)
    check(lib().ref_solve_problem(name.encode(), k, seed, p, int(adaptive), L, tol, max_depth, _dp(out)))
    keys = ["rel_linf", "rel_l2", "n_leaves", "N", "top_D_size", "tree_depth", "t_build_s", "t_solve_s"]
    return dict(zip(keys, out.tolist()))


def bench_sample(p, L, m, lo, hi, terms, source, root_implicit=True):
    """ref_bench_sample (ref_capi.h): the reference's full 2D build + solve time, estimated from one
    depth-(L-m) subtree solved end to end plus one merge_node + propagate step per top depth."""
    arr = (Term * max(1, len(terms)))()
    for i, (role, axis, axis2, fld) in enumerate(terms):
        arr[i].role, arr[i].axis, arr[i].axis2, arr[i].field = role, axis, axis2, fld
    top = L - m
    out = np.zeros(4 + 2 * max(top, 0))
    check(lib().ref_bench_sample(p, L, m, lo, hi, arr, len(terms), C.byref(source) if source is not None else None,
                                 int(root_implicit), _dp(out)))
    return dict(est_s=out[0], sub_build_s=out[1], sub_solve_s=out[2], sub_leaves=int(out[3]),
                merge_s=[out[4 + 2 * d] for d in range(top)], propagate_s=[out[5 + 2 * d] for d in range(top)])


class RefSolver:
    """The reference's hps::HpsSolver<Real> (variant 0) / <Complex> (variant 1).

    Either a uniform tree with field descriptors (like oracle.Solver) or, with `problem=name`, the
    reference's problem catalog on a uniform or adaptive tree.
    """

    def __init__(self, dim=2, p=16, L=3, lo=-1.0, hi=1.0, terms=(), source=None, source_imag=None, variant=0,
                 eta=1.0, root_implicit=False, build_root_T=False, keep=(), problem=None, k=0.0, seed=7,
                 adaptive=False, tol=1e-3, max_depth=10, keep_T=True):
        self.keep = list(keep)
        if problem is not None:
            self.h = lib().ref_create_problem(problem.encode(), k, seed, p, int(adaptive), L, tol, max_depth,
                                              int(keep_T))
        else:
            arr = (Term * max(1, len(terms)))()
            for i, (role, axis, axis2, fld) in enumerate(terms):
                arr[i].role, arr[i].axis, arr[i].axis2, arr[i].field = role, axis, axis2, fld
            self._terms = arr
            self.h = lib().ref_create(dim, p, L, lo, hi, arr, len(terms),
                                      C.byref(source) if source is not None else None,
                                      C.byref(source_imag) if source_imag is not None else None, variant, eta,
                                      int(root_implicit), int(build_root_T))
        if not self.h:
            raise RuntimeError("ref_create: " + lib().ref_last_error().decode())
        Lb = lib()
        self.cplx = bool(Lb.ref_is_complex(self.h))
        self.dim, self.p = Lb.ref_dim(self.h), Lb.ref_p(self.h)
        self.q = self.p - 2
        self.n_leaves, self.n_nodes = Lb.ref_n_leaves(self.h), Lb.ref_n_nodes(self.h)
        self.npts = self.p ** self.dim
        self.nb = Lb.ref_root_bsize(self.h)
        self.nbl = 2 * self.dim * self.q ** (self.dim - 1)
        self.dtype = np.complex128 if self.cplx else np.float64

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_destroy(self.h)
            self.h = None

    def build(self):
        check(lib().ref_build(self.h))

    def times(self):
        a, b = C.c_double(), C.c_double()
        lib().ref_times(self.h, C.byref(a), C.byref(b))
        return a.value, b.value

    def top_D_size(self):
        return lib().ref_top_D_size(self.h)

    def n_unresolved(self):
        return lib().ref_n_unresolved(self.h)

    def min_rcond(self):
        return lib().ref_min_rcond(self.h)

    def tree(self):
        n = self.n_nodes
        depth, parent, nch = (np.zeros(n, np.int32) for _ in range(3))
        children = np.zeros(8 * n, np.int32)
        lo, hi = np.zeros(3 * n), np.zeros(3 * n)
        anchor = np.zeros(3 * n, np.int64)
        leaves = np.zeros(self.n_leaves, np.int32)
        check(lib().ref_tree(self.h, _ip(depth), _ip(parent), _ip(nch), _ip(children), _dp(lo), _dp(hi),
                             anchor.ctypes.data_as(C.POINTER(C.c_longlong)), _ip(leaves)))
        return dict(depth=depth, parent=parent, n_children=nch, children=children.reshape(n, 8),
                    lo=lo.reshape(n, 3), hi=hi.reshape(n, 3), anchor=anchor.reshape(n, 3), leaves=leaves)

    def root_points(self):
        out = np.zeros(self.nb * 3)
        check(lib().ref_root_points(self.h, _dp(out)))
        return out.reshape(-1, 3)

    def leaf_points(self):
        out = np.zeros(self.n_leaves * self.npts * 3)
        check(lib().ref_leaf_points(self.h, _dp(out)))
        return out.reshape(self.n_leaves, self.npts, 3)

    def sample_root_data(self):
        g = np.zeros(self.nb, self.dtype)
        check(lib().ref_sample_root_data(self.h, _dp(g.view(np.float64))))
        return g

    def solve(self, g, want_leaf_g=False):
        g = _as_doubles(g, self.cplx)
        assert g.size == self.nb * (2 if self.cplx else 1)
        u = np.zeros(self.n_leaves * self.npts, self.dtype)
        lg = np.zeros(self.n_leaves * self.nbl, self.dtype) if want_leaf_g else None
        check(lib().ref_solve(self.h, _dp(g), _dp(u.view(np.float64)),
                              _dp(lg.view(np.float64)) if lg is not None else None))
        u = u.reshape(self.n_leaves, self.npts)
        return (u, lg.reshape(self.n_leaves, self.nbl)) if want_leaf_g else u

    def solve_radiation(self):
        u = np.zeros(self.n_leaves * self.npts, self.dtype)
        check(lib().ref_solve_radiation(self.h, _dp(u.view(np.float64))))
        return u.reshape(self.n_leaves, self.npts)

    def solve_new_source(self, leaf_f, g=None, radiation=False):
        f = _as_doubles(leaf_f, self.cplx)
        gd = _as_doubles(g, self.cplx) if g is not None else None
        u = np.zeros(self.n_leaves * self.npts, self.dtype)
        check(lib().ref_solve_new_source(self.h, _dp(f), int(radiation), _dp(gd), _dp(u.view(np.float64))))
        return u.reshape(self.n_leaves, self.npts)

    def get_leaf(self, ord_):
        dt, n, nb = self.dtype, self.npts, self.nbl
        Y, v, T, h = np.zeros(n * nb, dt), np.zeros(n, dt), np.zeros(nb * nb, dt), np.zeros(nb, dt)
        f = lambda a: _dp(a.view(np.float64))  # noqa: E731
        check(lib().ref_get_leaf(self.h, ord_, f(Y), f(v), f(T), f(h)))
        return Y.reshape(n, nb, order="F"), v, T.reshape(nb, nb, order="F"), h

    def node_sizes(self, nid):
        a, b = C.c_int(), C.c_int()
        check(lib().ref_node_sizes(self.h, nid, C.byref(a), C.byref(b)))
        return a.value, b.value

    def get_node(self, nid, want_S=True, want_T=True):
        """(S, gtilde, T, h) of MergeArtifact/node_T/node_h; S None for an implicit root, T/h None at the
        root unless build_root_T."""
        ne, ni = self.node_sizes(nid)
        dt = self.dtype
        S = np.zeros(ni * ne, dt) if want_S else None
        gt = np.zeros(ni, dt)
        T = np.zeros(ne * ne, dt) if want_T else None
        h = np.zeros(ne, dt) if want_T else None
        f = lambda a: _dp(a.view(np.float64)) if a is not None else None  # noqa: E731
        check(lib().ref_get_node(self.h, nid, f(S), f(gt), f(T), f(h)))
        return (S.reshape(ni, ne, order="F") if S is not None else None, gt,
                T.reshape(ne, ne, order="F") if T is not None else None, h)

    def mesh_json(self):
        n = lib().ref_mesh_json(self.h, None, 0)
        buf = C.create_string_buffer(n + 1)
        lib().ref_mesh_json(self.h, buf, n + 1)
        return buf.value.decode()

    def dump_solution(self, u, json_path, bin_path, tree_ref):
        u = _as_doubles(u, self.cplx)
        check(lib().ref_dump_solution(self.h, _dp(u), json_path.encode(), bin_path.encode(), tree_ref.encode()))

    def error_report(self, u):
        u = _as_doubles(u, self.cplx)
        a, b = C.c_double(), C.c_double()
        check(lib().ref_error_report(self.h, _dp(u), C.byref(a), C.byref(b)))
        return a.value, b.value
