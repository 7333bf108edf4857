"""Subtree recomputation on one GPU (the paper's memory strategy; SURVEY 8e "Recompute vs store").

The north star asks that "solutions across the whole solve are recomputed on-device rather than
stored": after the build only the [h|T] of the depth-`ds` subtree roots and the merges above them are
kept; the solve re-runs each subtree's build (leaves + lower merges) right before its downward pass
in one reused workspace.  Peak memory is one subtree's workspace plus the top part instead of the whole
tree, at the price of building every subtree twice -- the trade the paper measures as "subtree
recomputation (depth d)" (the BASELINE.md headline: 4.02 s at p=16 L=8 on an H100).

Every step goes through the C-ABI tree parts (include/hps_cuda.h hpsg_create_part), so the numbers
are the store-mode kernels' numbers.  In recompute mode ONE subtree part is created and moved from
subtree to subtree (hpsg_part_retarget: same sizes, new boxes), so recomputation allocates nothing;
`recompute=False` keeps one part per subtree alive between build and solve (store mode at subtree
granularity).
"""
from __future__ import annotations

import torch

from . import hps as H


class SubtreeRecomputeSolver:
    """HpsSolver-like driver: build(), solve_device(g) -> u (n_leaves x p^d, DFS leaf order)."""

    def __init__(self, tree: H.UniformTree, terms, source=None, depth=2, literal_sign=True, root_implicit_S=False,
                 device=0, recompute=True):
        if not 1 <= depth <= tree.L - 1:
            raise ValueError("subtree depth must satisfy 1 <= depth <= L - 1")
        self.tree, self.terms, self.source = tree, terms, source
        self.ds, self.recompute = depth, recompute
        self.kw = dict(literal_sign=literal_sign, root_implicit_S=root_implicit_S, device=device)
        self.dev = torch.device("cuda", device)
        self.nchild = 4 if tree.dim == 2 else 8
        self.n_sub = self.nchild ** depth
        self.top = H.HpsSolver(tree, terms, source, part=(0, 0, depth), **self.kw)
        self.sub = {}                 # kept subtree parts (store mode)
        self.stream = torch.cuda.current_stream(self.dev)
        self.top.set_stream(self.stream.cuda_stream)
        self.work = None              # the one retargeted part (recompute mode)

    def _part(self, k):
        if self.recompute:
            if self.work is None:
                self.work = H.HpsSolver(self.tree, self.terms, self.source, part=(self.ds, k, self.tree.L), **self.kw)
                self.work.set_stream(self.stream.cuda_stream)
            elif self.work.part[1] != k:
                self.work.retarget(k)
            return self.work
        s = H.HpsSolver(self.tree, self.terms, self.source, part=(self.ds, k, self.tree.L), **self.kw)
        s.set_stream(self.stream.cuda_stream)
        return s

    def build(self):
        ht = None
        for k in range(self.n_sub):
            part = self.sub.get(k) or self._part(k)
            part.build()
            if ht is None:
                nb = part.nb_root
                ht = torch.empty((1 + nb, nb), dtype=torch.float64, device=self.dev)
            part.root_ht_device(ht.data_ptr())
            self.top.set_cut_ht_device(k, ht.data_ptr())
            if not self.recompute:
                self.sub[k] = part
        self.top.build()
        self.nb_sub = self.top.cut_nb

    def solve_device(self, g_root: torch.Tensor, u_out: torch.Tensor | None = None) -> torch.Tensor:
        """g_root (nrhs, nb_root) or (nb_root,) on the device -> u (nrhs, n_leaves, p^d)."""
        g = g_root.reshape(-1, g_root.shape[-1]).contiguous()
        nrhs = g.shape[0]
        gc = torch.empty((nrhs, self.n_sub, self.nb_sub), dtype=torch.float64, device=self.dev)
        self.top.solve_cut_device(g.data_ptr(), nrhs, gc.data_ptr())
        per = self.nchild ** (self.tree.L - self.ds)
        npts = self.tree.p ** self.tree.dim
        if u_out is None:
            u_out = torch.empty((nrhs, self.tree.n_leaves, npts), dtype=torch.float64, device=self.dev)
        tmp = torch.empty((nrhs, per, npts), dtype=torch.float64, device=self.dev)
        for k in range(self.n_sub):
            part = self.sub.get(k)
            if part is None:      # recompute: rebuild the subtree for its downward pass
                part = self._part(k)
                part.build()
            gk = gc[:, k, :].contiguous()
            part.solve_device(gk.data_ptr(), nrhs, tmp.data_ptr())
            u_out[:, k * per:(k + 1) * per] = tmp
        return u_out

    def root_boundary_points(self):
        return self.top.root_boundary_points()

    def close(self):
        for p in self.sub.values():
            p.close()
        self.sub.clear()
        if self.work is not None:
            self.work.close()
        self.top.close()
