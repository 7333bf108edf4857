"""Subtree-sharded build/solve (paper_2503_17535_b200/sharded.py).

CPU (no GPU): the ownership plan, and the routing of [h|T] up / g down through
torch.distributed point-to-point ops (gloo, world_size 2 and 4) with MOCK parts whose
"merge" and "propagate" are exact, composable functions of the tree path -- so the sharded
result must equal the same computation done on the whole tree in one part, and any
misrouted, misordered or missing message changes it.
GPU: the same phases with the real C-ABI parts (libhps_b200), all ranks emulated in one
process (one GPU), against the unsharded solver on identical inputs.
"""
import os

import numpy as np
import pytest
import torch

from paper_2503_17535_b200 import sharded as SH


# ----------------------------------------------------------------------------- plan
@pytest.mark.parametrize("world,ds,owners", [(1, 0, (0,)), (2, 1, (0, 0, 1, 1)), (3, 1, (0, 0, 1, 2)),
                                             (4, 1, (0, 1, 2, 3)), (8, 2, tuple(k // 2 for k in range(16)))])
def test_plan_2d(world, ds, owners):
    p = SH.make_plan(8, 2, world)
    assert p.ds == ds and p.sub_owner == owners
    # every subtree owned once; every rank owns >= 1 subtree; parents merged by their first child's owner
    assert sorted(k for r in range(world) for k in p.subtrees(r)) == list(range(p.n_sub))
    assert all(p.subtrees(r) for r in range(world))
    assert p.owner(0, 0) == 0
    for d in range(ds):
        for i in range(4 ** d):
            assert p.owner(d, i) == p.owner(d + 1, 4 * i)
    if world == 8:
        assert [p.owner(1, i) for i in range(4)] == [0, 2, 4, 6]  # depth-1 merges on four ranks at once


def test_plan_3d_and_limits():
    p = SH.make_plan(4, 3, 8)
    assert p.ds == 1 and p.sub_owner == tuple(range(8))
    with pytest.raises(ValueError):
        SH.make_plan(1, 2, 2)   # no merge below the root to shard
    with pytest.raises(ValueError):
        SH.make_plan(2, 2, 8)   # 8 ranks need 16 subtrees below the root merge
    with pytest.raises(ValueError):
        SH.make_plan(3, 2, 0)


# ----------------------------------------------------------------------------- mock parts
W = [0.0, 1.0, 0.37, 0.051, 0.0077, 0.00113, 0.000171, 2.3e-5, 3.1e-6, 4.7e-7]


class MockParts:
    """Exact composable stand-ins for the C-ABI parts: node [h|T][0,0] = sum over the leaves
    below of leaf_value(leaf); g(child c of a depth-d node) = g + (c+1) * W[d+1];
    u(leaf) = g(leaf) + leaf_value(leaf)."""

    def __init__(self, L, nchild, dev="cpu"):
        self.L, self.nchild, self.dev = L, nchild, torch.device(dev)

    def make(self, rd, ri, cd):
        return MockPart(self, rd, ri, cd)


def leaf_value(L, nchild, leaf):
    return float((leaf * 7919) % 1009) + 0.25 * leaf


class MockPart:
    def __init__(self, f, rd, ri, cd):
        self.f, self.rd, self.ri, self.cd = f, rd, ri, cd
        self.nb_root = 2 + f.L - rd
        self.cut = cd < f.L
        self.n_cut = f.nchild ** (cd - rd) if self.cut else 0
        self.cut_nb = 2 + f.L - cd if self.cut else 0
        self.n_leaves = 0 if self.cut else f.nchild ** (f.L - rd)
        self.npts = 3
        self.inp = {}
        self.built = None

    def set_cut_ht(self, k, t):
        assert t.shape == (1 + self.cut_nb, self.cut_nb)
        self.inp[k] = float(t[0, 0])

    def build(self):
        if self.cut:
            assert sorted(self.inp) == list(range(self.n_cut)), "missing cut input"
            self.built = sum(self.inp[k] for k in range(self.n_cut))
        else:
            first = self.ri * self.n_leaves
            self.built = sum(leaf_value(self.f.L, self.f.nchild, first + j) for j in range(self.n_leaves))

    def root_ht(self):
        t = torch.zeros((1 + self.nb_root, self.nb_root), dtype=torch.float64, device=self.f.dev)
        t[0, 0] = self.built
        return t

    def solve_cut(self, g):
        assert g.shape[1] == self.nb_root
        n = self.f.nchild
        out = torch.empty((g.shape[0], n ** (self.cd - self.rd), self.cut_nb), dtype=torch.float64, device=self.f.dev)
        for k in range(out.shape[1]):
            add, kk = 0.0, k
            for lev in range(self.cd, self.rd, -1):
                add += (kk % n + 1) * W[lev]
                kk //= n
            out[:, k, :] = g[:, :1] + add
        return out

    def solve_leaves(self, g):
        assert g.shape[1] == self.nb_root
        n, L = self.f.nchild, self.f.L
        u = torch.empty((g.shape[0], self.n_leaves, self.npts), dtype=torch.float64, device=self.f.dev)
        first = self.ri * self.n_leaves
        for j in range(self.n_leaves):
            add, kk = 0.0, j
            for lev in range(L, self.rd, -1):
                add += (kk % n + 1) * W[lev]
                kk //= n
            u[:, j, :] = g[:, :1] + add + leaf_value(L, n, first + j)
        return u


def direct_mock(L, nchild, g_root):
    """The same mock computation on the whole tree as one part."""
    f = MockParts(L, nchild)
    whole = f.make(0, 0, L)
    whole.build()
    return whole.built, whole.solve_leaves(g_root)


@pytest.mark.parametrize("L,dim,world", [(3, 2, 2), (3, 2, 4), (4, 2, 8), (3, 2, 3), (2, 3, 8)])
def test_emulate_mock_matches_direct(L, dim, world):
    nchild = 4 if dim == 2 else 8
    plan = SH.make_plan(L, dim, world)
    f = MockParts(L, nchild)
    shards = [SH.ShardedHps(plan, r, f) for r in range(world)]
    g_root = torch.tensor([[1.5] * (2 + L), [-0.25] * (2 + L)], dtype=torch.float64)
    u = SH.assemble_u(SH.emulate(shards, g_root), plan)
    root_sum, u_ref = direct_mock(L, nchild, g_root)
    assert torch.allclose(u, u_ref, rtol=0, atol=1e-12)
    # the root merge saw every leaf exactly once
    assert shards[0].top[(0, 0)].built == root_sum


def _dist_worker(rank, world, L, dim, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        nchild = 4 if dim == 2 else 8
        plan = SH.make_plan(L, dim, world)
        shard = SH.ShardedHps(plan, rank, MockParts(L, nchild))
        g_root = torch.tensor([[0.75] * (2 + L)], dtype=torch.float64)
        u = SH.run_dist(shard, g_root if rank == 0 else None, nrhs=1)
        _, u_ref = direct_mock(L, nchild, g_root)
        per = nchild ** (L - plan.ds)
        ok = all(torch.allclose(u[k], u_ref[:, k * per:(k + 1) * per], rtol=0, atol=1e-12) for k in plan.subtrees(rank))
        ok = ok and sorted(u) == plan.subtrees(rank)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, ok, ""))
    except Exception as e:  # report to the parent instead of hanging it
        q.put((rank, False, repr(e)))


@pytest.mark.parametrize("world,L", [(2, 3), (4, 3)])
def test_run_dist_gloo(world, L):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 2000) + world
    procs = [ctx.Process(target=_dist_worker, args=(r, world, L, 2, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res


# ----------------------------------------------------------------------------- GPU: real parts
@pytest.mark.gpu
@pytest.mark.parametrize("name,p,L,world,literal,implicit", [
    ("poisson2d", 16, 3, 2, True, False), ("poisson2d", 16, 3, 4, False, True),
    ("helmholtz_bumps", 16, 4, 8, False, True), ("helmholtz_bumps", 12, 4, 3, True, False),
    ("laplace3d", 6, 2, 8, False, True)])
def test_sharded_matches_unsharded(name, p, L, world, literal, implicit):
    import paper_2503_17535_b200 as H
    from paper_2503_17535_b200 import problems as PR
    prob = PR.CATALOG[name]()
    tree = H.build_uniform_tree(prob.lo, prob.hi, L, prob.dim, p)
    ref = H.HpsSolver(tree, prob.terms, prob.source, literal_sign=literal, root_implicit_S=implicit)
    ref.build()
    g = prob.boundary(ref.root_boundary_points())
    u_ref = ref.solve(np.stack([g, 0.5 * g]))
    plan = SH.make_plan(L, prob.dim, world)
    parts = SH.CudaParts(tree, prob.terms, prob.source, literal_sign=literal, root_implicit_S=implicit)
    shards = [SH.ShardedHps(plan, r, parts) for r in range(world)]
    g_dev = torch.tensor(np.stack([g, 0.5 * g]), device="cuda")
    u = SH.assemble_u(SH.emulate(shards, g_dev), plan).cpu().numpy()
    err = np.abs(u - u_ref).max() / np.abs(u_ref).max()
    assert err < 1e-12, err
    # subtree root [h|T] equals the unsharded node T/h (same kernels, same per-node arithmetic)
    k = plan.subtrees(world - 1)[-1]
    node_id = sum(plan.nchild ** d for d in range(plan.ds)) + k
    _, _, T_ref, h_ref = ref.get_node(node_id)
    ht = shards[world - 1].sub[k].root_ht().cpu().numpy()   # (1+nb, nb) row-major = column-major [h|T]
    assert np.abs(ht[0] - h_ref).max() <= 1e-12 * max(1.0, np.abs(h_ref).max())
    assert np.abs(ht[1:].T - T_ref).max() <= 1e-12 * max(1.0, np.abs(T_ref).max())
