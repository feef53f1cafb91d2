"""TEST INFRASTRUCTURE: a CPU engine for ``paper_2602_19873_b200.distributed`` over the
oracle restatement, so the domain-decomposition orchestration (exact split, payload
all-to-all, global octree, node-geometry all-reduce, halo exchange, range build and
pass) runs and is checked with gloo on CPU ("union of per-rank stores
must equal the single-domain oracle store").

Particles absent from a rank are NaN: a build or pass that read a particle the halo
did not deliver produces different masks/outputs, which the tests catch.
"""
from __future__ import annotations

import numpy as np
import torch

from oracle.oracle import Oracle, Particles, Store
from paper_2602_19873_b200.api import NeighborStore, ReduceResult

KNAMES = {0: "count", 1: "density", 2: "lj", 3: "lj_coulomb"}
COLS = ("x", "y", "z", "h", "m", "q")


class OracleEngine:
    def __init__(self, oracle: Oracle, box6, periodic, bits=21):
        self.o = oracle
        self.box6 = np.asarray(box6, np.float64)
        self.periodic = tuple(periodic)
        self.bits = bits
        self.device = torch.device("cpu")

    def upload(self, ps: Particles):
        self.local = ps
        self.n_local = ps.n

    def local_sort(self):
        keys, perm = self.o.sort_by_sfc(self.local, self.bits)
        self.sl = self.local.permuted(perm)
        return torch.from_numpy(keys.view(np.int64).copy())

    def payload(self):
        return torch.from_numpy(np.stack([getattr(self.sl, c) for c in COLS], 1))

    def own(self, recv, n_total, p0, runs=None):
        a = recv.numpy()
        ps = Particles(*[np.ascontiguousarray(a[:, k]) for k in range(6)], self.box6.copy(), self.periodic)
        keys, perm = self.o.sort_by_sfc(ps, self.bits)
        sp = ps.permuted(perm)
        self.g = Particles(*[np.full(n_total, np.nan) for _ in COLS], self.box6.copy(), self.periodic)
        for c in COLS:
            getattr(self.g, c)[p0: p0 + sp.n] = getattr(sp, c)
        self.n_total = n_total
        return torch.from_numpy(keys.view(np.int64).copy())

    def octree(self, gkeys, bucket):
        self.tree = self.o.tree(gkeys.numpy().view(np.uint64), self.bits, bucket)
        return len(self.tree.pend)

    def node_geometry_partial(self, p0, p1):
        lo, hi, mh = self.o.node_geometry_range(self.tree, self.g, p0, p1)
        geo = np.zeros((len(mh), 8))
        geo[:, 0:3], geo[:, 3:6], geo[:, 6] = lo, hi, mh
        return torch.from_numpy(geo)

    def set_node_geometry(self, geo):
        g = geo.numpy()
        self.geo = (g[:, 0:3].copy(), g[:, 3:6].copy(), g[:, 6].copy())

    def _bp(self, bp):
        c = bp.params
        return dict(ci=c.ci, cj=c.cj, mode=int(bp.mode), scale=bp.build_radius_scale)

    def halo_flags(self, bp, sc0, sc1, max_h):
        return torch.from_numpy(self.o.halo_mark(self.g, self.tree, self.geo, sc0, sc1, max_h, **self._bp(bp)))

    def gather_rows(self, idx):
        i = idx.numpy()
        return torch.from_numpy(np.stack([getattr(self.g, c)[i] for c in COLS], 1))

    def scatter_rows(self, idx, rows):
        i, r = idx.numpy(), rows.numpy()
        for k, c in enumerate(COLS):
            getattr(self.g, c)[i] = r[:, k]

    def build_range(self, bp, sc0, sc1, max_h, download):
        c = bp.params
        self.store = self.o.build_store_range(self.g, self.tree, self.geo, sc0, sc1, max_h, c.ci, c.cj, c.w,
                                              int(bp.mode), int(bool(bp.compress)), bp.build_radius_scale)
        self.sc0 = sc0
        s = self.store
        return NeighborStore(bp, self.n_total, s.counts, s.offsets, s.blob)

    def reduce(self, kernel, cfg, nloc, download):
        outs, cnt = self.o.reduce_range(KNAMES[kernel.kind], self.g, self.store, self.sc0, cfg.query_scale,
                                        kernel.epsilon, kernel.sigma, kernel.coulomb_k)
        return ReduceResult(list(kernel.names), outs, cnt)
