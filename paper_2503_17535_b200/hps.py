"""Python host mirror of the reference HpsSolver<Real> API over the B200 C-ABI.

The reference API (/root/reference/proj/include/hps/solver.hpp:40-117) is C++:
HpsSolver(tree, variant, eta, terms, source, opts); build(); solve(g_root).
This module binds the same surface to libhps_b200.so (include/hps_cuda.h)
with ctypes, so tests and bench.py drive exactly the entry points a C/C++
caller would.  There is no CPU fallback: without the shared library or a
CUDA device every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HPS_B200_LIB") or os.path.join(HERE, "libhps_b200.so")  # env: developer A/B builds

# status codes (include/hps_cuda.h)
HPSG_OK, HPSG_ERR_INVALID, HPSG_ERR_SINGULAR_LEAF, HPSG_ERR_SINGULAR_MERGE, HPSG_ERR_NONFINITE, HPSG_ERR_OOM, \
    HPSG_ERR_CUDA, HPSG_ERR_STATE, HPSG_ERR_NO_DEVICE = range(9)

FIELD_CONST, FIELD_BUMPS, FIELD_PLANE_SIN, FIELD_PLANE_COS, FIELD_BUMPS_SIN, FIELD_POISSON2D_SRC, FIELD_SAMPLED, \
    FIELD_BUMPS_GRAD, FIELD_DIVGRAD_SRC, FIELD_WAVEFRONT_SRC, FIELD_PB_EPS, FIELD_PB_EPS_GRAD = range(12)
ROLE_LAPLACIAN, ROLE_GRADIENT, ROLE_ZEROTH, ROLE_SECOND_ORDER = range(4)


class HpsError(RuntimeError):
    """hps::Error (proj/include/hps/core.hpp:27-29) raised from a C-ABI status."""

    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class _Field(C.Structure):
    _fields_ = [("kind", C.c_int), ("n_centers", C.c_int), ("c", C.c_double * 8),
                ("centers", C.POINTER(C.c_double)), ("samples", C.POINTER(C.c_double))]


class _Term(C.Structure):
    _fields_ = [("role", C.c_int), ("axis", C.c_int), ("axis2", C.c_int), ("field", _Field)]


class _Tree(C.Structure):
    _fields_ = [("dim", C.c_int), ("p", C.c_int), ("L", C.c_int), ("lo", C.c_double), ("hi", C.c_double)]


class _Part(C.Structure):
    _fields_ = [("root_depth", C.c_int), ("root_index", C.c_longlong), ("cut_depth", C.c_int)]


class _Options(C.Structure):
    _fields_ = [("literal_sign", C.c_int), ("root_implicit_S", C.c_int), ("device", C.c_int), ("keep_factors", C.c_int),
                ("variant", C.c_int), ("eta", C.c_double), ("build_root_T", C.c_int),
                ("source_imag", C.POINTER(_Field)), ("force_batched_leaf", C.c_int), ("no_lu_lookahead", C.c_int),
                ("force_lu_leaf", C.c_int)]


class _Stats(C.Structure):
    _fields_ = [("n_leaves", C.c_int), ("n_points", C.c_longlong), ("root_bsize", C.c_int), ("top_D_size", C.c_int),
                ("tree_depth", C.c_int), ("min_rcond", C.c_double), ("ill_conditioned", C.c_int),
                ("t_build_ms", C.c_double), ("t_leaf_ms", C.c_double), ("t_merge_ms", C.c_double),
                ("t_solve_ms", C.c_double), ("build_flops", C.c_double), ("solve_bytes", C.c_double),
                ("device_bytes", C.c_double), ("launches_build", C.c_int), ("launches_solve", C.c_int),
                ("n_levels", C.c_int), ("t_level_ms", C.c_double * 24), ("leaf_path", C.c_int),
                ("leaf_exec_flops", C.c_double)]


_lib = None


def build_library():
    subprocess.run(["make", "-s", "-C", HERE, "-j8"], check=True)


def lib():
    """Load libhps_b200.so (fails loudly; the product has no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise HpsError(HPSG_ERR_STATE, f"{LIB_PATH} not built: run __graft_entry__.build() or make -C {HERE}")
        L = C.CDLL(LIB_PATH)
        vp, dp = C.c_void_p, C.POINTER(C.c_double)
        L.hpsg_create.argtypes = [C.POINTER(_Tree), C.POINTER(_Term), C.c_int, C.POINTER(_Field), C.POINTER(_Options),
                                  C.POINTER(vp)]
        L.hpsg_create_part.argtypes = [C.POINTER(_Tree), C.POINTER(_Part), C.POINTER(_Term), C.c_int,
                                       C.POINTER(_Field), C.POINTER(_Options), C.POINTER(vp)]
        L.hpsg_create_tree.argtypes = [C.POINTER(_TreeDesc), C.POINTER(_Term), C.c_int, C.POINTER(_Field),
                                       C.POINTER(_Options), C.POINTER(vp)]
        L.hpsg_part_sizes.argtypes = [vp, C.POINTER(C.c_longlong), C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.hpsg_estimate_bytes.argtypes = [C.POINTER(_Tree), C.POINTER(_Part), C.POINTER(_Term), C.c_int,
                                          C.POINTER(_Field), C.POINTER(_Options), C.c_int, dp]
        L.hpsg_part_root_ht.argtypes = [vp, C.c_void_p]
        L.hpsg_part_retarget.argtypes = [vp, C.c_longlong]
        L.hpsg_part_set_cut_ht.argtypes = [vp, C.c_longlong, C.c_void_p]
        L.hpsg_part_solve_cut.argtypes = [vp, C.c_void_p, C.c_int, C.c_void_p]
        L.hpsg_solve_new_source.argtypes = [vp, dp, dp, C.c_int, dp]
        L.hpsg_solve_complex.argtypes = [vp, dp, C.c_int, dp]
        L.hpsg_solve_radiation.argtypes = [vp, dp, dp]
        L.hpsg_evaluate_at.argtypes = [vp, C.c_void_p, C.c_int, dp, C.c_int, dp]
        L.hpsg_error_report.argtypes = [vp, C.c_void_p, C.c_int, C.POINTER(_Field), C.POINTER(_Field),
                                        C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.hpsg_solve_new_source_device.argtypes = [vp, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
        L.hpsg_build.argtypes = [vp]
        L.hpsg_solve.argtypes = [vp, dp, C.c_int, dp, dp]
        L.hpsg_solve_device.argtypes = [vp, C.c_void_p, C.c_int, C.c_void_p]
        L.hpsg_root_boundary_points.argtypes = [vp, dp]
        L.hpsg_leaf_points.argtypes = [vp, dp]
        L.hpsg_get_leaf.argtypes = [vp, C.c_int, dp, dp, dp, dp]
        L.hpsg_node_sizes.argtypes = [vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.hpsg_get_node.argtypes = [vp, C.c_int, dp, dp, dp, dp]
        L.hpsg_get_stats.argtypes = [vp, C.POINTER(_Stats)]
        L.hpsg_set_stream.argtypes = [vp, C.c_void_p]
        L.hpsg_last_error.argtypes = [vp]
        L.hpsg_last_error.restype = C.c_char_p
        L.hpsg_destroy.argtypes = [vp]
        L.hpsg_build_info.restype = C.c_char_p
        L.hpsg_bump_centers.argtypes = [C.c_ulonglong, C.c_int, C.c_int, dp]
        L.hpsg_tree_root_points.argtypes = [C.POINTER(_Tree), dp]
        L.hpsg_tree_leaf_points.argtypes = [C.POINTER(_Tree), dp]
        _lib = L
    return _lib


def _dp(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


# ----------------------------------------------------------------------------- problem description
@dataclass
class Field:
    """Coefficient/source field: a device-evaluated closed form or host samples.

    Mirrors the reference's std::function<Real(const Point&)> fields
    (proj/include/hps/local_solve.hpp:17-23) -- see include/hps_cuda.h HPSG_FIELD_*.
    """
    kind: int
    c: tuple = ()
    centers: np.ndarray | None = None
    samples: np.ndarray | None = None

    def to_c(self, keep):
        f = _Field()
        f.kind = self.kind
        for i, v in enumerate(self.c):
            f.c[i] = float(v)
        if self.centers is not None:
            cen = np.ascontiguousarray(self.centers, dtype=np.float64).reshape(-1, 3)
            keep.append(cen)
            f.n_centers = cen.shape[0]
            f.centers = _dp(cen)
        if self.samples is not None:
            smp = np.ascontiguousarray(self.samples, dtype=np.float64)
            keep.append(smp)
            f.samples = _dp(smp)
        return f

    @staticmethod
    def const(v):
        return Field(FIELD_CONST, (v,))


@dataclass
class Term:
    """CoefficientField (role, axis, axis2, field), proj/include/hps/local_solve.hpp:17-23."""
    role: int
    field: Field
    axis: int = -1
    axis2: int = -1


@dataclass
class UniformTree:
    """build_uniform_tree(domain=[lo,hi]^dim, L, dim, p), proj/src/mesh.cpp:90-121."""
    dim: int
    p: int
    L: int
    lo: float = -1.0
    hi: float = 1.0

    @property
    def q(self):
        return self.p - 2

    @property
    def n_leaves(self):
        return (4 if self.dim == 2 else 8) ** self.L

    @property
    def total_points(self):
        return self.n_leaves * self.p ** self.dim

    @property
    def leaf_boundary_size(self):
        return 2 * self.dim * self.q ** (self.dim - 1)

    @property
    def root_boundary_size(self):
        return 4 * self.q * 2 ** self.L if self.dim == 2 else 6 * self.q ** 2 * 4 ** self.L


def build_uniform_tree(lo, hi, L, dim, p):
    return UniformTree(dim=dim, p=p, L=L, lo=lo, hi=hi)


class _TreeDesc(C.Structure):
    _fields_ = [("dim", C.c_int), ("p", C.c_int), ("n_nodes", C.c_int), ("depth", C.POINTER(C.c_int)),
                ("n_children", C.POINTER(C.c_int)), ("children", C.POINTER(C.c_int)),
                ("lo", C.POINTER(C.c_double)), ("hi", C.POINTER(C.c_double))]


class GeneralTree:
    """The reference's DiscretizationTree (proj/include/hps/mesh.hpp:28-61) as node arrays: any tree --
    adaptive, level-restricted octrees from refine_adaptive (mesh.cpp:233-318) or uniform ones.
    depth (n,), n_children (n,), children (n, 8), lo / hi (n, 3); node 0 is the root; leaves are
    enumerated depth-first (DiscretizationTree::finalize, mesh.cpp:54-71)."""

    def __init__(self, dim, p, depth, n_children, children, lo, hi):
        self.dim, self.p = int(dim), int(p)
        self.depth = np.ascontiguousarray(depth, dtype=np.int32)
        self.n_children = np.ascontiguousarray(n_children, dtype=np.int32)
        self.children = np.ascontiguousarray(np.asarray(children).reshape(-1, 8), dtype=np.int32)
        self.lo = np.ascontiguousarray(np.asarray(lo, dtype=np.float64).reshape(-1, 3))
        self.hi = np.ascontiguousarray(np.asarray(hi, dtype=np.float64).reshape(-1, 3))
        self.n_nodes = len(self.depth)
        nc = 4 if self.dim == 2 else 8
        leaves, stack = [], [0]
        while stack:
            i = stack.pop()
            if self.n_children[i] == 0:
                leaves.append(i)
            else:
                stack.extend(int(c) for c in self.children[i, :nc][::-1])
        self.leaves = np.array(leaves, dtype=np.int32)

    @classmethod
    def from_arrays(cls, d, dim, p):
        """From a dict with keys depth, n_children, children, lo, hi (e.g. oracle.ref.RefSolver.tree())."""
        return cls(dim, p, d["depth"], d["n_children"], d["children"], d["lo"], d["hi"])

    @property
    def q(self):
        return self.p - 2

    @property
    def n_leaves(self):
        return len(self.leaves)

    @property
    def total_points(self):
        return self.n_leaves * self.p ** self.dim

    @property
    def leaf_boundary_size(self):
        return 2 * self.dim * self.q ** (self.dim - 1)

    def total_nodes(self):
        return self.n_nodes

    def desc(self):
        return _TreeDesc(self.dim, self.p, self.n_nodes, self.depth.ctypes.data_as(C.POINTER(C.c_int)),
                         self.n_children.ctypes.data_as(C.POINTER(C.c_int)),
                         self.children.ctypes.data_as(C.POINTER(C.c_int)), _dp(self.lo), _dp(self.hi))


def tree_root_points(tree: UniformTree):
    """Root boundary points of a tree without a solver (hpsg_tree_root_points; solver.cpp:159-182)."""
    out = np.zeros((tree.root_boundary_size, 3))
    tr = _Tree(tree.dim, tree.p, tree.L, tree.lo, tree.hi)
    rc = lib().hpsg_tree_root_points(C.byref(tr), _dp(out))
    if rc != HPSG_OK:
        raise HpsError(rc, "hpsg_tree_root_points: invalid tree")
    return out


def tree_leaf_points_of(tree: UniformTree):
    """leaf_cheb_points over the whole tree without a solver (n_leaves, p^d, 3)."""
    out = np.zeros((tree.n_leaves, tree.p ** tree.dim, 3))
    tr = _Tree(tree.dim, tree.p, tree.L, tree.lo, tree.hi)
    rc = lib().hpsg_tree_leaf_points(C.byref(tr), _dp(out))
    if rc != HPSG_OK:
        raise HpsError(rc, "hpsg_tree_leaf_points: invalid tree")
    return out


def bump_centers(seed, n=10, dim=2):
    """std::mt19937_64(seed) + uniform_real_distribution(-0.5,0.5) (proj/src/problems.cpp:126-141)."""
    out = np.zeros(3 * n)
    lib().hpsg_bump_centers(seed, n, dim, _dp(out))
    return out.reshape(n, 3)


def mesh_json(tree: GeneralTree) -> str:
    """mesh_to_json (proj/src/mesh.cpp:435-463), byte-identical to the reference's output."""
    L = lib()
    L.hpsg_mesh_json.argtypes = [C.POINTER(_TreeDesc), C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]
    d = tree.desc()
    n = C.c_size_t()
    if L.hpsg_mesh_json(C.byref(d), None, 0, C.byref(n)) != HPSG_OK:
        raise HpsError(HPSG_ERR_INVALID, "hpsg_mesh_json failed")
    buf = C.create_string_buffer(n.value + 1)
    if L.hpsg_mesh_json(C.byref(d), buf, n.value + 1, C.byref(n)) != HPSG_OK:
        raise HpsError(HPSG_ERR_INVALID, "hpsg_mesh_json failed")
    return buf.value.decode()


def refine_adaptive(lo, hi, p, fields, tol=1e-3, max_depth=10, cap=1 << 20):
    """refine_adaptive(domain, RefinementCriterion{tol, p, test_fields}, max_depth) (proj/src/mesh.cpp:233-318)
    in 3D on [lo,hi]^3 with built-in fields -> (GeneralTree, n_unresolved)."""
    keep = []
    arr = (_Field * len(fields))()
    for i, f in enumerate(fields):
        arr[i] = f.to_c(keep)
    lo3, hi3 = np.full(3, float(lo)), np.full(3, float(hi))
    n, nu = C.c_int(), C.c_int()
    L = lib()
    ip = C.POINTER(C.c_int)
    L.hpsg_refine_adaptive.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_double, C.c_int,
                                       C.POINTER(_Field), C.c_int, C.c_int, ip, ip, ip, ip, C.POINTER(C.c_double),
                                       C.POINTER(C.c_double), ip]
    rc = L.hpsg_refine_adaptive(p, _dp(lo3), _dp(hi3), tol, max_depth, arr, len(fields), 0, C.byref(n), None, None,
                                None, None, None, C.byref(nu))
    if rc != HPSG_OK and n.value == 0:
        raise HpsError(rc, "hpsg_refine_adaptive failed")
    nn = n.value
    depth, nch = np.zeros(nn, np.int32), np.zeros(nn, np.int32)
    ch = np.zeros((nn, 8), np.int32)
    tlo, thi = np.zeros((nn, 3)), np.zeros((nn, 3))
    ipn = lambda a: a.ctypes.data_as(ip)  # noqa: E731
    rc = L.hpsg_refine_adaptive(p, _dp(lo3), _dp(hi3), tol, max_depth, arr, len(fields), nn, C.byref(n), ipn(depth),
                                ipn(nch), ipn(ch), _dp(tlo), _dp(thi), C.byref(nu))
    if rc != HPSG_OK:
        raise HpsError(rc, "hpsg_refine_adaptive failed")
    return GeneralTree(3, p, depth, nch, ch, tlo, thi), nu.value


# ----------------------------------------------------------------------------- footprint
def estimate_bytes(tree: UniformTree, terms, source: Field | None = None, part=None, nrhs=1, literal_sign=True,
                   root_implicit_S=False, device=0, keep_factors=False) -> float:
    """Device bytes an HpsSolver(tree, terms, source, part=..., ...) would hold after its build and a
    solve of nrhs right-hand sides, computed by the library's own allocation path without allocating
    (include/hps_cuda.h hpsg_estimate_bytes).  DtN variant."""
    L = lib()
    keep = []
    arr = (_Term * max(1, len(terms)))()
    for i, t in enumerate(terms):
        arr[i].role, arr[i].axis, arr[i].axis2 = t.role, t.axis, t.axis2
        arr[i].field = t.field.to_c(keep)
    src = source.to_c(keep) if source is not None else None
    tr = _Tree(tree.dim, tree.p, tree.L, tree.lo, tree.hi)
    op = _Options(int(literal_sign), int(root_implicit_S), device, int(keep_factors), 0, 1.0, 0)
    pt = _Part(*(tuple(part) if part is not None else (0, 0, tree.L)))
    out = np.zeros(1)
    rc = L.hpsg_estimate_bytes(C.byref(tr), C.byref(pt), arr, len(terms), C.byref(src) if src is not None else None,
                               C.byref(op), int(nrhs), _dp(out))
    if rc != HPSG_OK:
        raise HpsError(rc, "hpsg_estimate_bytes failed (invalid tree/part or no CUDA device)")
    return float(out[0])


# ----------------------------------------------------------------------------- solver
class HpsSolver:
    """HpsSolver<Real> (DtN variant) on one B200, via libhps_b200.so.

    literal_sign=True reproduces the reference's v_i = -L_ii^-1 f_i
    (proj/src/local_solve.cpp:137); False uses the corrected +L_ii^-1 f_i.

    part=(root_depth, root_index, cut_depth) restricts the solver to a subtree PART of the tree
    (include/hps_cuda.h hpsg_create_part; the subtree-sharded build of SURVEY 8e): its leaves are
    the real leaves below the part root (cut_depth == L) or the depth-cut_depth nodes whose [h|T]
    are inputs (cut_depth < L).
    """

    def __init__(self, tree: UniformTree, terms, source: Field | None = None, literal_sign=True,
                 root_implicit_S=False, device=0, part=None, keep_factors=False, variant="dtn", eta=1.0,
                 build_root_T=False, source_imag: Field | None = None, force_batched_leaf=False,
                 lu_lookahead=True, fdm_leaf=True):
        L = lib()
        self.tree = tree
        keep = []
        arr = (_Term * max(1, len(terms)))()
        for i, t in enumerate(terms):
            arr[i].role, arr[i].axis, arr[i].axis2 = t.role, t.axis, t.axis2
            arr[i].field = t.field.to_c(keep)
        src = source.to_c(keep) if source is not None else None
        tr = _Tree(tree.dim, tree.p, tree.L, tree.lo, tree.hi) if isinstance(tree, UniformTree) else None
        if variant not in ("dtn", "iti"):
            raise HpsError(HPSG_ERR_INVALID, f"unknown variant {variant!r}")
        self.variant = variant
        op = _Options(int(literal_sign), int(root_implicit_S), device, int(keep_factors), 1 if variant == "iti" else 0,
                      float(eta), int(build_root_T))
        if source_imag is not None:
            self._src_im = source_imag.to_c(keep)
            op.source_imag = C.pointer(self._src_im)
        op.force_batched_leaf = int(force_batched_leaf)
        op.no_lu_lookahead = int(not lu_lookahead)
        op.force_lu_leaf = int(not fdm_leaf)
        h = C.c_void_p()
        if isinstance(tree, GeneralTree):  # hpsg_create_tree: adaptive / arbitrary trees
            if part is not None:
                raise HpsError(HPSG_ERR_INVALID, "parts are uniform-tree only")
            self.part = None
            self._desc = tree.desc()
            rc = L.hpsg_create_tree(C.byref(self._desc), arr, len(terms), C.byref(src) if src is not None else None,
                                    C.byref(op), C.byref(h))
        else:
            self.part = tuple(part) if part is not None else (0, 0, tree.L)
            pt = _Part(*self.part)
            rc = L.hpsg_create_part(C.byref(tr), C.byref(pt), arr, len(terms),
                                    C.byref(src) if src is not None else None, C.byref(op), C.byref(h))
        self._h = h
        if rc != HPSG_OK:
            msg = L.hpsg_last_error(h).decode() if h.value else "no CUDA device"
            self.close()
            raise HpsError(rc, f"hpsg_create: {msg}")
        self.root_implicit_S = root_implicit_S
        self.npts = tree.p ** tree.dim
        if self.part is None:
            st = self.stats()
            self.n_cut, self.cut_nb, self.nb_root = 0, 0, st["root_bsize"]
            self.n_leaves = tree.n_leaves
            return
        nc, cnb, rnb = C.c_longlong(), C.c_int(), C.c_int()
        self._check(L.hpsg_part_sizes(h, C.byref(nc), C.byref(cnb), C.byref(rnb)), "part_sizes")
        self.n_cut, self.cut_nb, self.nb_root = nc.value, cnb.value, rnb.value
        nchild = 4 if tree.dim == 2 else 8
        self.n_leaves = 0 if self.n_cut else nchild ** (self.part[2] - self.part[0])

    def _check(self, rc, what):
        if rc != HPSG_OK:
            raise HpsError(rc, f"{what}: {lib().hpsg_last_error(self._h).decode()}")

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().hpsg_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def build(self):
        self._check(lib().hpsg_build(self._h), "build")

    def root_boundary_points(self):
        out = np.zeros((self.nb_root, 3))
        self._check(lib().hpsg_root_boundary_points(self._h, _dp(out)), "root_boundary_points")
        return out

    def leaf_points(self):
        out = np.zeros((self.n_leaves, self.npts, 3))
        self._check(lib().hpsg_leaf_points(self._h, _dp(out)), "leaf_points")
        return out

    def solve(self, g_root, want_leaf_g=False):
        """g_root: (nb,) or (nrhs, nb) host array -> u: (n_leaves, p^d) or (nrhs, n_leaves, p^d)."""
        g = np.ascontiguousarray(g_root, dtype=np.float64)
        single = g.ndim == 1
        g2 = g.reshape(1, -1) if single else g
        nrhs = g2.shape[0]
        assert g2.shape[1] == self.nb_root
        u = np.empty((nrhs, self.n_leaves, self.npts))
        lg = np.empty((nrhs, self.n_leaves, self.tree.leaf_boundary_size)) if want_leaf_g else None
        self._check(lib().hpsg_solve(self._h, _dp(g2), nrhs, _dp(u), _dp(lg)), "solve")
        if single:
            u = u[0]
            lg = lg[0] if lg is not None else None
        return (u, lg) if want_leaf_g else u

    def solve_device(self, d_g_ptr, nrhs, d_u_ptr):
        """Zero-copy solve on device pointers (e.g. torch.Tensor.data_ptr())."""
        self._check(lib().hpsg_solve_device(self._h, C.c_void_p(d_g_ptr), nrhs, C.c_void_p(d_u_ptr)), "solve")

    def solve_complex(self, g_root):
        """ItI variant (HpsSolver<Complex>::solve): g_root (nb,) or (nrhs, nb) complex incoming impedance
        data at the root boundary points -> u (n_leaves, p^2) or (nrhs, n_leaves, p^2) complex."""
        g = np.ascontiguousarray(g_root, dtype=np.complex128)
        single = g.ndim == 1
        g2 = g.reshape(1, -1) if single else g
        nrhs = g2.shape[0]
        assert g2.shape[1] == self.nb_root
        u = np.empty((nrhs, self.n_leaves, self.npts), dtype=np.complex128)
        self._check(lib().hpsg_solve_complex(self._h, g2.ctypes.data_as(C.POINTER(C.c_double)), nrhs,
                                             u.ctypes.data_as(C.POINTER(C.c_double))), "solve")
        return u[0] if single else u

    def evaluate_at(self, d_u_ptr, points, is_complex=False):
        """evaluate_at(field, points) (downpass.cpp:13-95) on a device-resident solution (pointer to
        n_leaves x p^d values, interleaved complex when is_complex) at host points (npts, 3)."""
        x = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        out = np.empty(len(x), dtype=np.complex128 if is_complex else np.float64)
        self._check(lib().hpsg_evaluate_at(self._h, C.c_void_p(d_u_ptr), int(is_complex), _dp(x), len(x),
                                           out.ctypes.data_as(C.POINTER(C.c_double))), "evaluate_at")
        return out

    def error_report(self, d_u_ptr, exact: Field, exact_imag: Field | None = None, is_complex=False):
        """error_report (problems.cpp:270-293) on the device: (rel L-inf, rel L2) vs a built-in field."""
        keep = []
        fe = exact.to_c(keep)
        fi = exact_imag.to_c(keep) if exact_imag is not None else None
        li, l2 = C.c_double(), C.c_double()
        self._check(lib().hpsg_error_report(self._h, C.c_void_p(d_u_ptr), int(is_complex), C.byref(fe),
                                            C.byref(fi) if fi is not None else None, C.byref(li), C.byref(l2)),
                    "error_report")
        return li.value, l2.value

    def solve_radiation(self, want_g=False):
        """HpsSolver::solve_radiation() (solver.cpp:254-259): root data closing T g = -h (ItI,
        build_root_T=True) -> u (n_leaves, p^2) complex [, g (nb,) complex]."""
        u = np.empty((self.n_leaves, self.npts), dtype=np.complex128)
        g = np.empty(self.nb_root, dtype=np.complex128)
        self._check(lib().hpsg_solve_radiation(self._h, u.ctypes.data_as(C.POINTER(C.c_double)),
                                               g.ctypes.data_as(C.POINTER(C.c_double))), "solve_radiation")
        return (u, g) if want_g else u

    def solve_new_source(self, leaf_f, g_root):
        """HpsSolver::solve_new_source(leaf_f, RootBC::dirichlet, g_root) (solver.cpp:285-307) for
        one or several sources: leaf_f (n_leaves, p^d) or (nsrc, n_leaves, p^d) samples at the leaf
        points, g_root (nb,) or (nsrc, nb).  Needs keep_factors=True."""
        f = np.ascontiguousarray(leaf_f, dtype=np.float64)
        g = np.ascontiguousarray(g_root, dtype=np.float64)
        single = f.ndim == 2
        f3 = f.reshape(1, *f.shape) if single else f
        g2 = g.reshape(1, -1) if g.ndim == 1 else g
        nsrc = f3.shape[0]
        assert f3.shape[1:] == (self.n_leaves, self.npts) and g2.shape == (nsrc, self.nb_root)
        u = np.empty((nsrc, self.n_leaves, self.npts))
        self._check(lib().hpsg_solve_new_source(self._h, _dp(f3), _dp(g2), nsrc, _dp(u)), "solve_new_source")
        return u[0] if single else u

    def solve_new_source_device(self, d_f_ptr, d_g_ptr, nsrc, d_u_ptr):
        self._check(lib().hpsg_solve_new_source_device(self._h, C.c_void_p(d_f_ptr), C.c_void_p(d_g_ptr), nsrc,
                                                       C.c_void_p(d_u_ptr)), "solve_new_source")

    # ---- subtree parts (include/hps_cuda.h hpsg_part_*)
    def root_ht_device(self, d_dst_ptr):
        """[h|T] of the part root (nb_root x (1+nb_root), column-major) -> device buffer."""
        self._check(lib().hpsg_part_root_ht(self._h, C.c_void_p(d_dst_ptr)), "part_root_ht")

    def retarget(self, root_index):
        """Move this subtree part to sibling subtree `root_index` of the same depth (workspace reused)."""
        self._check(lib().hpsg_part_retarget(self._h, root_index), "part_retarget")
        self.part = (self.part[0], root_index, self.part[2])

    def set_cut_ht_device(self, k, d_src_ptr):
        """Input [h|T] (cut_nb x (1+cut_nb)) of cut node k from a device buffer."""
        self._check(lib().hpsg_part_set_cut_ht(self._h, k, C.c_void_p(d_src_ptr)), "part_set_cut_ht")

    def solve_cut_device(self, d_g_ptr, nrhs, d_out_ptr):
        """Downward pass of a cut part: root data (nrhs x nb_root) -> cut-node data (nrhs x n_cut x cut_nb)."""
        self._check(lib().hpsg_part_solve_cut(self._h, C.c_void_p(d_g_ptr), nrhs, C.c_void_p(d_out_ptr)),
                    "part_solve_cut")

    def get_leaf(self, ord_):
        n, nb = self.npts, self.tree.leaf_boundary_size
        Y, v, T, h = np.zeros(n * nb), np.zeros(n), np.zeros(nb * nb), np.zeros(nb)
        self._check(lib().hpsg_get_leaf(self._h, ord_, _dp(Y), _dp(v), _dp(T), _dp(h)), "get_leaf")
        return Y.reshape(n, nb, order="F"), v, T.reshape(nb, nb, order="F"), h

    def node_sizes(self, node_id):
        a, b = C.c_int(), C.c_int()
        self._check(lib().hpsg_node_sizes(self._h, node_id, C.byref(a), C.byref(b)), "node_sizes")
        return a.value, b.value

    def get_node(self, node_id):
        ne, ni = self.node_sizes(node_id)
        want_S = not (node_id == 0 and self.root_implicit_S)
        S = np.zeros(ni * ne) if want_S else None
        gt = np.zeros(ni)
        T = np.zeros(ne * ne) if node_id != 0 else None
        h = np.zeros(ne) if node_id != 0 else None
        self._check(lib().hpsg_get_node(self._h, node_id, _dp(S), _dp(gt), _dp(T), _dp(h)), "get_node")
        return (S.reshape(ni, ne, order="F") if S is not None else None, gt,
                T.reshape(ne, ne, order="F") if T is not None else None, h)

    def dump_solution(self, d_u_ptr, json_path, bin_path, tree_ref, is_complex=False):
        """dump_solution (proj/src/downpass.cpp:108-143) of a device-resident solution."""
        lib().hpsg_dump_solution.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_char_p, C.c_char_p, C.c_char_p]
        self._check(lib().hpsg_dump_solution(self._h, C.c_void_p(d_u_ptr), int(is_complex), json_path.encode(),
                                             bin_path.encode(), tree_ref.encode()), "dump_solution")

    def set_stream(self, stream_handle):
        """Run on a caller-owned cudaStream_t (int handle, e.g. torch.cuda.current_stream().cuda_stream)."""
        self._check(lib().hpsg_set_stream(self._h, C.c_void_p(stream_handle)), "set_stream")

    def stats(self):
        s = _Stats()
        self._check(lib().hpsg_get_stats(self._h, C.byref(s)), "stats")
        out = {k: getattr(s, k) for k, _ in _Stats._fields_}
        out["t_level_ms"] = list(s.t_level_ms)[:s.n_levels]
        return out
