"""Subtree-sharded HPS build/solve across ranks (north star: "each GPU owns whole
subtrees, runs their leaves and lower merges locally, then ships only its top-level DtN matrices
over NVLink with NCCL for the few remaining top merges").

The tree is cut at depth ``ds`` (smallest depth with nchild**ds >= world).  Subtree k of that
depth (a contiguous range of the DFS leaf order, proj/src/mesh.cpp:54-71) is owned by rank
``k * world // nchild**ds``.  Every node above the cut is merged by the owner of its first
subtree, so the depth-1 merges of an 8-rank 2D run proceed on four ranks at once and only the
root merge is serial.  The only data-path exchanges are the real ones of the algorithm:

* upward, the [h|T] of each child whose owner differs from its parent's owner
  (merge.cpp:226-278 consumes the child T/h; 2D L=8: 103 MB per depth-2 child, 411 MB per
  depth-1 child);
* downward, the boundary data g of those same children (solver.cpp:210-224; a few hundred KB).

Each rank's numerical work goes through C-ABI tree parts (include/hps_cuda.h hpsg_create_part),
one per owned subtree (cut_depth = L: leaves + merges) and one per owned top node (one merge
level, inputs = its children's [h|T]).  Transport is torch.distributed point-to-point (NCCL
between GPUs; gloo for the CPU tests of this module's routing) or, in one process, the
``emulate`` runner that plays every rank in turn (used by the single-GPU parity tests).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class Plan:
    """Ownership of subtree parts and top merges for ``world`` ranks."""
    L: int
    nchild: int
    world: int
    ds: int                  # cut depth (0: no sharding)
    sub_owner: tuple         # owner rank of each depth-ds subtree

    @property
    def n_sub(self):
        return self.nchild ** self.ds

    def owner(self, depth, index):
        """Rank that holds node (depth, index): its subtree's owner, or the owner of its first subtree."""
        if depth >= self.ds:
            return self.sub_owner[index // self.nchild ** (depth - self.ds)]
        return self.sub_owner[index * self.nchild ** (self.ds - depth)]

    def top_nodes(self, rank, depth):
        """Nodes above the cut at ``depth`` merged by ``rank``."""
        return [i for i in range(self.nchild ** depth) if self.owner(depth, i) == rank]

    def subtrees(self, rank):
        return [k for k in range(self.n_sub) if self.sub_owner[k] == rank]


def make_plan(L, dim, world):
    nchild = 4 if dim == 2 else 8
    if world < 1:
        raise ValueError("world size must be >= 1")
    ds = 0
    while nchild ** ds < world:
        ds += 1
    if world > 1 and ds > L - 1:
        raise ValueError(f"a depth-{L} tree has only {nchild ** (L - 1)} subtrees below the root merge; "
                         f"cannot shard over {world} ranks")
    n_sub = nchild ** ds
    return Plan(L=L, nchild=nchild, world=world, ds=ds, sub_owner=tuple(k * world // n_sub for k in range(n_sub)))


class CudaParts:
    """Part factory over libhps_b200 (the product path: every part is a C-ABI context)."""

    def __init__(self, tree, terms, source, literal_sign=True, root_implicit_S=False, device=0):
        from . import hps as H
        self.H = H
        self.tree, self.terms, self.source = tree, terms, source
        self.literal_sign, self.root_implicit_S, self.device = literal_sign, root_implicit_S, device
        self.dev = torch.device("cuda", device)

    def make(self, root_depth, root_index, cut_depth):
        part = _CudaPart(self, root_depth, root_index, cut_depth)
        # one stream per rank: parts, torch collectives and CUDA-event timing share torch's stream
        part.s.set_stream(torch.cuda.current_stream(self.dev).cuda_stream)
        return part


class _CudaPart:
    def __init__(self, f, root_depth, root_index, cut_depth):
        self.s = f.H.HpsSolver(f.tree, f.terms, f.source, literal_sign=f.literal_sign,
                               root_implicit_S=f.root_implicit_S, device=f.device,
                               part=(root_depth, root_index, cut_depth))
        self.dev = f.dev
        self.nb_root, self.n_cut, self.cut_nb = self.s.nb_root, self.s.n_cut, self.s.cut_nb
        self.n_leaves, self.npts = self.s.n_leaves, self.s.npts

    def set_cut_ht(self, k, t):
        self.s.set_cut_ht_device(k, t.data_ptr())

    def build(self):
        self.s.build()

    def root_ht(self):
        out = torch.empty((1 + self.nb_root, self.nb_root), dtype=torch.float64, device=self.dev)
        self.s.root_ht_device(out.data_ptr())
        return out

    def solve_cut(self, g):
        nrhs = g.shape[0]
        out = torch.empty((nrhs, self.n_cut, self.cut_nb), dtype=torch.float64, device=self.dev)
        self.s.solve_cut_device(g.contiguous().data_ptr(), nrhs, out.data_ptr())
        return out

    def solve_leaves(self, g):
        nrhs = g.shape[0]
        u = torch.empty((nrhs, self.n_leaves, self.npts), dtype=torch.float64, device=self.dev)
        self.s.solve_device(g.contiguous().data_ptr(), nrhs, u.data_ptr())
        return u

    def stats(self):
        return self.s.stats()


class ShardedHps:
    """One rank's share of a subtree-sharded build/solve.

    Phases (all ranks run them in the same order; ``runner`` moves the tensors):
      build:  build_local()  then for depth = ds-1 .. 0: up_messages(depth) -> merge_level(depth)
      solve:  set_root_data(g) then for depth = 0 .. ds-1: down_level(depth) -> down_messages(depth),
              then solve_local()
    """

    def __init__(self, plan: Plan, rank: int, parts):
        self.plan, self.rank, self.parts = plan, rank, parts
        p = plan
        if p.ds == 0:
            self.sub = {0: parts.make(0, 0, p.L)}
            self.top = {}
        else:
            self.sub = {k: parts.make(p.ds, k, p.L) for k in p.subtrees(rank)}
            self.top = {(d, i): parts.make(d, i, d + 1) for d in range(p.ds) for i in p.top_nodes(rank, d)}
        self.ht = {}    # (depth, index) -> [h|T] tensor of nodes this rank holds
        self.g = {}     # (depth, index) -> boundary data (nrhs x nb) of nodes this rank holds
        self.u = {}     # subtree k -> u (nrhs x leaves x p^d)

    # ---- build
    def build_local(self):
        for k, part in self.sub.items():
            part.build()
            if self.plan.ds > 0:
                self.ht[(self.plan.ds, k)] = part.root_ht()

    def up_messages(self, depth):
        """(sends, recvs) of children [h|T] for the merges at ``depth``: lists of (peer, key, tensor)."""
        p, sends, recvs = self.plan, [], []
        for i in range(p.nchild ** depth):
            dst = p.owner(depth, i)
            for c in range(p.nchild):
                key = (depth + 1, p.nchild * i + c)
                src = p.owner(*key)
                if src == dst:
                    continue
                if src == self.rank:
                    sends.append((dst, key, self.ht[key]))
                elif dst == self.rank:
                    part = self.top[(depth, i)]
                    buf = torch.empty((1 + part.cut_nb, part.cut_nb), dtype=torch.float64,
                                      device=self.parts.dev)
                    recvs.append((src, key, buf))
        return sends, recvs

    def accept(self, recvs, store):
        for _, key, t in recvs:
            store[key] = t

    def merge_level(self, depth):
        p = self.plan
        for i in p.top_nodes(self.rank, depth):
            part = self.top[(depth, i)]
            for c in range(p.nchild):
                part.set_cut_ht(c, self.ht[(depth + 1, p.nchild * i + c)])
            part.build()
            if depth > 0:
                self.ht[(depth, i)] = part.root_ht()
        # children [h|T] are consumed; release what this rank no longer needs
        for key in [k for k in self.ht if k[0] == depth + 1]:
            del self.ht[key]

    # ---- solve
    def set_root_data(self, g_root):
        """Root boundary data (nrhs x nb_root), on the owner of the root (rank 0)."""
        if self.rank == self.plan.owner(0, 0):
            self.g[(0, 0)] = g_root

    def down_level(self, depth):
        p = self.plan
        for i in p.top_nodes(self.rank, depth):
            gc = self.top[(depth, i)].solve_cut(self.g.pop((depth, i)))
            for c in range(p.nchild):
                self.g[(depth + 1, p.nchild * i + c)] = gc[:, c, :].contiguous()

    def down_messages(self, depth):
        """(sends, recvs) of the children boundary data produced at ``depth``."""
        p, sends, recvs = self.plan, [], []
        for i in range(p.nchild ** depth):
            src = p.owner(depth, i)
            for c in range(p.nchild):
                key = (depth + 1, p.nchild * i + c)
                dst = p.owner(*key)
                if src == dst:
                    continue
                if src == self.rank:
                    sends.append((dst, key, self.g.pop(key)))
                elif dst == self.rank:
                    recvs.append((src, key, None))
        return sends, recvs

    def solve_local(self):
        for k, part in self.sub.items():
            self.u[k] = part.solve_leaves(self.g.pop((self.plan.ds, k)))
        return self.u


# ----------------------------------------------------------------------------- runners
def _nb_of(shard, key, nrhs):
    """Shape of the boundary data a rank receives for node ``key``."""
    p = shard.plan
    if key[0] == p.ds:
        return (nrhs, shard.sub[key[1]].nb_root)
    return (nrhs, shard.top[key].nb_root)


def run_dist(shard: ShardedHps, g_root=None, nrhs=1, build=True, solve=True):
    """Drive one rank with torch.distributed point-to-point ops (NCCL or gloo)."""
    import torch.distributed as dist
    p = shard.plan

    # gloo has no device-memory point-to-point: stage through the host (CPU tests, one-GPU runs)
    stage = dist.get_backend() == "gloo"

    def exchange(sends, recvs):
        ops, staged = [], []
        for peer, key, t in sorted(sends, key=lambda x: (x[0], x[1])):
            t = t.contiguous()
            ops.append(dist.P2POp(dist.isend, t.cpu() if stage and t.is_cuda else t, peer))
        for peer, key, t in sorted(recvs, key=lambda x: (x[0], x[1])):
            if stage and t.is_cuda:
                h = torch.empty(t.shape, dtype=t.dtype)
                staged.append((h, t))
                t = h
            ops.append(dist.P2POp(dist.irecv, t, peer))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
            for h, t in staged:
                t.copy_(h)
            # no host synchronisation: with NCCL, wait() orders the transfers before later work on
            # torch's current stream, which is the stream every part of this rank runs on
            # (CudaParts.make -> set_stream), so the merges that read the received buffers through
            # plain device pointers queue behind them on the device

    if build:
        shard.build_local()
        for depth in range(p.ds - 1, -1, -1):
            sends, recvs = shard.up_messages(depth)
            exchange(sends, recvs)
            shard.accept(recvs, shard.ht)
            shard.merge_level(depth)
    if solve:
        shard.set_root_data(g_root)
        for depth in range(p.ds):
            shard.down_level(depth)
            sends, recvs = shard.down_messages(depth)
            recvs = [(src, key, torch.empty(_nb_of(shard, key, nrhs), dtype=torch.float64, device=shard.parts.dev))
                     for src, key, _ in recvs]
            exchange(sends, recvs)
            shard.accept(recvs, shard.g)
        return shard.solve_local()
    return None


def emulate(shards, g_root=None, build=True, solve=True):
    """Play every rank of ``shards`` in one process (same phases, tensors handed over directly)."""
    p = shards[0].plan

    def exchange(msgs):
        box = {}
        for s, (sends, _) in zip(shards, msgs):
            for peer, key, t in sends:
                box[(s.rank, peer, key)] = t
        return box

    if build:
        for s in shards:
            s.build_local()
        for depth in range(p.ds - 1, -1, -1):
            msgs = [s.up_messages(depth) for s in shards]
            box = exchange(msgs)
            for s, (_, recvs) in zip(shards, msgs):
                s.accept([(src, key, box[(src, s.rank, key)]) for src, key, _ in recvs], s.ht)
            for s in shards:
                s.merge_level(depth)
    if solve:
        for s in shards:
            s.set_root_data(g_root)
        for depth in range(p.ds):
            for s in shards:
                s.down_level(depth)
            msgs = [s.down_messages(depth) for s in shards]
            box = exchange(msgs)
            for s, (_, recvs) in zip(shards, msgs):
                s.accept([(src, key, box[(src, s.rank, key)]) for src, key, _ in recvs], s.g)
        out = {}
        for s in shards:
            out.update(s.solve_local())
        return out
    return None


def assemble_u(u_by_subtree, plan):
    """Concatenate per-subtree solutions into the DFS leaf order of the whole tree."""
    return torch.cat([u_by_subtree[k] for k in range(plan.n_sub)], dim=1)
