"""TEST INFRASTRUCTURE: a CPU engine for ``paper_2602_19873_b200.distributed`` over the
oracle restatement, so the domain-decomposition orchestration (exact split, payload
all-to-all, global octree, node-geometry all-reduce, halo exchange, range build and
pass) runs and is checked with gloo on CPU ("union of per-rank stores
must equal the single-domain oracle store").

Particles absent from a rank are NaN: a build or pass that read a particle the halo
did not deliver produces different masks/outputs, which the tests catch.

The engine implements both orchestrations of DomainDecomposition: the O(owned + halo)
one for gather stores (radix-select splitter, distributed octree from all-reduced level
bounds, owner-side halo selection against the ranks' chunk boxes, node geometry from the
present particles only) and the legacy one (symmetric stores). It keeps global-index
arrays (memory is not the point on CPU), so "local" positions equal global ones.
"""
from __future__ import annotations

import numpy as np
import torch

from oracle.oracle import Oracle, Particles, Store, Tree
from paper_2602_19873_b200.api import NeighborStore, ReduceResult

KNAMES = {0: "count", 1: "density", 2: "lj", 3: "lj_coulomb"}
COLS = ("x", "y", "z", "h", "m", "q")


U64 = np.uint64


class OracleEngine:
    supports_local = True

    def __init__(self, oracle: Oracle, box6, periodic, bits=21):
        self.o = oracle
        self.box6 = np.asarray(box6, np.float64)
        self.periodic = tuple(periodic)
        self.bits = bits
        self.fields = ["m", "q"]
        self.device = torch.device("cpu")

    def upload(self, ps: Particles):
        self.local = ps
        self.n_local = ps.n

    def local_sort(self):
        keys, perm = self.o.sort_by_sfc(self.local, self.bits)
        self.sl = self.local.permuted(perm)
        self.keys_local = keys
        return torch.from_numpy(keys.view(np.int64).copy())

    def payload(self):
        return [torch.from_numpy(getattr(self.sl, c).copy()) for c in COLS] + \
            [torch.from_numpy(self.keys_local.view(np.float64).copy())]

    # ---- O(owned + halo) orchestration (DomainDecomposition._run_local)
    def key_hist(self, prefix, shift):
        keys, n = self.keys_local, len(self.keys_local)
        out = np.zeros((prefix.numel(), 65536), np.int64)
        for q, base in enumerate(prefix.tolist()):
            bnd = [base + (b << shift) for b in range(65537)]
            pos = np.array([n if v >= 1 << 64 else int(np.searchsorted(keys, U64(v), "left")) for v in bnd])
            out[q] = np.diff(pos)
        return torch.from_numpy(out)

    def merge_owned(self, moved, runs):
        a = [c.numpy() for c in moved[:6]]
        ps = Particles(*[np.ascontiguousarray(v) for v in a], self.box6.copy(), self.periodic)
        keys, perm = self.o.sort_by_sfc(ps, self.bits)  # stable: (key, source rank, position)
        self.owned = ps.permuted(perm)
        self.n_owned = ps.n

    def max_h(self):
        return torch.tensor([float(self.owned.h.max()) if self.n_owned else 0.0], dtype=torch.float64)

    def octree_dist(self, bucket, n_global, comm):
        """build_octree (octree.cpp:9-59) of the global key multiset: per level the local
        lower bounds of the children are summed over ranks; then the reference's DFS
        allocation order numbers the nodes."""
        keys, bits = self.keys_local, self.bits
        levels = [dict(kf=np.zeros(1, np.uint64), gpb=np.array([0]), gpe=np.array([n_global]))]
        d = 0
        while True:
            L = levels[d]
            split = ((L["gpe"] - L["gpb"]) > bucket) & (d < bits)
            L["split"] = split
            if not split.any():
                break
            span = U64(1) << U64(3 * (bits - d - 1))
            ckf = (L["kf"][split][:, None] + span * np.arange(8, dtype=np.uint64)[None, :]).ravel()
            lpb = np.searchsorted(keys, ckf, "left").astype(np.int64)
            lpe = np.searchsorted(keys, ckf + span, "left").astype(np.int64)
            g = torch.from_numpy(np.concatenate([lpb, lpe]))
            comm.allreduce_(g, "sum")
            g = g.numpy()
            levels.append(dict(kf=ckf, gpb=g[: len(ckf)], gpe=g[len(ckf):]))
            d += 1
        for L in levels:
            L["rank"] = np.cumsum(L["split"]) - 1  # index among the level's split nodes
        recs = [[0, 0, 0, 0, -1, 0]]

        def rec(d, i, idx):
            L = levels[d]
            kf = int(L["kf"][i])
            recs[idx][:4] = [kf, kf + (1 << (3 * (bits - d))), int(L["gpb"][i]), int(L["gpe"][i])]
            recs[idx][5] = d
            if not L["split"][i]:
                return
            first = len(recs)
            recs[idx][4] = first
            recs.extend([[0, 0, 0, 0, -1, 0] for _ in range(8)])
            j = int(L["rank"][i])
            for c in range(8):
                rec(d + 1, 8 * j + c, first + c)

        rec(0, 0, 0)
        r = np.array(recs, dtype=object)
        self.tree = Tree(r[:, 0].astype(np.uint64), r[:, 1].astype(np.uint64), r[:, 2].astype(np.uint32),
                         r[:, 3].astype(np.uint32), r[:, 4].astype(np.int32), r[:, 5].astype(np.uint8), bits)
        return len(recs)

    def straddling_leaves(self, bounds):
        t = self.tree
        b = np.array(list(bounds), np.int64)[None, :]
        hit = ((t.pbegin.astype(np.int64)[:, None] < b) & (t.pend.astype(np.int64)[:, None] > b)).any(1)
        return torch.from_numpy(np.nonzero(hit & (t.first_child < 0))[0])

    def leaf_boxes(self, p0, p1):
        t, o = self.tree, self.owned
        lb = np.empty((len(t.pend), 6))
        lb[:, :3], lb[:, 3:] = np.inf, -np.inf
        for k in np.nonzero(t.first_child < 0)[0]:
            b, e = max(int(t.pbegin[k]), p0), min(int(t.pend[k]), p1)
            if b < e:
                pts = np.stack([o.x[b - p0:e - p0], o.y[b - p0:e - p0], o.z[b - p0:e - p0]], 1)
                lb[k, :3], lb[k, 3:] = pts.min(0), pts.max(0)
        return torch.from_numpy(lb)

    def domain_boxes(self, k):
        o = self.owned
        db = np.empty((k, 6))
        db[:, :3], db[:, 3:] = np.inf, -np.inf
        m = (-(-o.n // k) + 63) // 64 * 64 if o.n else 0  # whole super-clusters per chunk
        for c in range(k):
            b, e = c * m, min(c * m + m, o.n)
            if b < e:
                pts = np.stack([o.x[b:e], o.y[b:e], o.z[b:e]], 1)
                db[c, :3], db[c, 3:] = pts.min(0), pts.max(0)
        return torch.from_numpy(db)

    def _box_d2(self, a, b):
        """aabb_dist_sq (core.hpp:152-165) between box a and boxes b [m, 6] (3 images)."""
        L = self.box6[3:] - self.box6[:3]
        s = np.zeros(len(b))
        for d in range(3):
            def gap(lo, hi):
                return np.maximum(np.maximum(a[d], lo) - np.minimum(a[3 + d], hi), 0.0)
            g = gap(b[:, d], b[:, 3 + d])
            if self.periodic[d]:
                g = np.minimum(g, gap(b[:, d] - L[d], b[:, 3 + d] - L[d]))
                g = np.minimum(g, gap(b[:, d] + L[d], b[:, 3 + d] + L[d]))
            s += g * g
        empty = (b[:, 0] > b[:, 3]) | (a[0] > a[3])
        return np.where(empty, np.inf, s)

    def halo_select(self, p0, p1, cj, lb, boxes, rank, reach):
        t, lb, boxes = self.tree, lb.numpy(), boxes.numpy()
        P = boxes.shape[0]
        ncl = -(-(p1 - p0) // cj)
        flags = np.zeros((P, ncl), np.uint8)
        for k in np.nonzero(t.first_child < 0)[0]:
            b, e = max(int(t.pbegin[k]), p0), min(int(t.pend[k]), p1)
            if b >= e:
                continue
            for q in range(P):
                if q != rank and (self._box_d2(lb[k], boxes[q]) <= reach * reach).any():
                    flags[q, b // cj - p0 // cj:(e - 1) // cj - p0 // cj + 1] = 1
        return torch.from_numpy(flags)

    def pack_clusters(self, p0, p1, cj, ids):
        o = self.owned
        g = (ids.numpy().astype(np.int64)[:, None] * cj + np.arange(cj)[None, :]).ravel()
        ok = (g >= p0) & (g < p1)
        rows = np.full((len(g), 6), np.nan)
        for k, c in enumerate(COLS):
            rows[ok, k] = getattr(o, c)[g[ok] - p0]
        return torch.from_numpy(rows)

    def place_local(self, n_global, p0, p1, cj, halo_ids, halo_rows):
        self.g = Particles(*[np.full(n_global, np.nan) for _ in COLS], self.box6.copy(), self.periodic)
        for c in COLS:
            getattr(self.g, c)[p0:p1] = getattr(self.owned, c)
        ids = halo_ids.numpy().astype(np.int64)
        rows = halo_rows.numpy()
        g = (ids[:, None] * cj + np.arange(cj)[None, :]).ravel()
        ok = g < n_global
        for k, c in enumerate(COLS):
            getattr(self.g, c)[g[ok]] = rows[ok, k]
        lo, hi, mh = self.o.node_geometry_range(self.tree, self.g, 0, n_global)  # NaN (absent) loses
        self.geo = (lo, hi, mh)
        self.n_total = n_global
        return p0  # global index space

    def own(self, recv, n_total, p0, runs=None):
        a = torch.stack(list(recv)[:6], 1).numpy() if isinstance(recv, (list, tuple)) else recv.numpy()
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
