"""SFC key-range domain decomposition over ranks.

The reference is single-process (``parallel_for`` over super-clusters,
neighbor_build.cpp:109 / reduce.hpp:217-220). Super-clusters are independent, so the
path shards: rank r owns a contiguous range of the GLOBAL SFC order, snapped to
super-cluster (64-particle) boundaries, and builds + queries only its super-clusters.
The union of the per-rank stores is byte-identical to the single-domain store and the
union of the per-rank pass outputs is identical to the single-domain outputs.

Gather stores (``DomainDecomposition.run``, one process per GPU) keep per-rank memory
O(owned + halo): no array of the global particle count is allocated.

1. local SFC sort of the rank's input particles (K1-K3, own kernels);
2. exact global split of the (key, global id) order at the super-cluster bounds: a
   radix select over the 63-bit keys, 4 rounds of 16 bits, each one histogram kernel
   (sfcnl_cu_key_hist) + one all-reduce of (P-1) x 65536 counts; ties split in rank
   order (= global id order);
3. all-to-all of the particle payload (x, y, z, h, fields, key bits) to the owners;
4. owner: the P received runs (each in (key, global id) order) are merged by a kernel
   (sfcnl_cu_merge_runs: binary searches, (key, source rank) order = the global stable
   order, no re-sort);
5. distributed octree (sfcnl_cu_build_octree_dist): every rank runs the reference's
   build_octree over the GLOBAL key multiset of which its step-1 keys are a part; per
   level the child particle bounds (local lower bounds) are summed over ranks by one
   all-reduce, so every rank holds the identical single-domain node array (reference
   numbering) without ever seeing another rank's keys;
6. exact boxes of the leaves overlapping the owned range (sfcnl_cu_leaf_boxes); the
   handful of leaves that straddle a rank boundary are combined by one MIN/MAX
   all-reduce of (P-1) boxes;
7. halo, owner side (sfcnl_cu_halo_select): each rank all-gathers K chunk boxes of every
   rank's owned particles; an owner sends rank q every owned cluster of every leaf whose
   box is within scale * max h of one of q's boxes. This is a superset of the clusters
   q's traversal can accept (acceptance needs the leaf's box within scale * h of one of
   q's super-cluster boxes, each inside one of q's chunk boxes), so q has every
   particle of every leaf it may accept;
8. local index space (sfcnl_cu_dd_place / dd_localize): owned + halo particles in
   ascending global order ([halo below][NaN padding to 64][owned][halo above]); the
   global octree's particle ranges are mapped into it, node and cluster geometry are
   computed from the local particles (partial boxes of nodes whose particles are not all
   present only ever contain the boxes of present leaves, so no leaf the reference
   accepts is pruned and none it rejects is accepted);
9. range build (global cluster ids written by the encoder) and range passes (stored
   global ids mapped back to local clusters by the decoders).

Symmetric stores use ``_run_legacy`` (global-index arrays, traversal-marked halo, node
geometry all-reduce) because their reverse halo reduction ships per-entry j-side sums
keyed by global cluster ids (pass_sym.cuh).

Collectives go through ``Comm`` (torch.distributed: NCCL on device tensors; other
backends, e.g. gloo for CPU tests or several ranks sharing one GPU, are staged through
host memory). The engine does the per-rank work: ``CudaEngine`` (this module) drives
the C-ABI context; the parity tests plug in a CPU engine over the oracle.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence

import ctypes as C
import os

import numpy as np

from .api import (BuildParams, Context, Kernel, NeighborStore, ParticleSet, PassConfig, ReduceResult,
                  SimulationBox, kDefaultSfcBits)

SC = 64  # super-cluster size (cluster.hpp:9)
KEY_SPAN = 1 << 63  # keys are < 2^(3*21)


def _torch():
    import torch
    return torch


def sc_partition(n_total: int, world: int):
    """Super-cluster bounds and particle bounds of each rank (balanced SC counts)."""
    total_sc = (n_total + SC - 1) // SC
    scb = [(q * total_sc) // world for q in range(world + 1)]
    pb = [min(SC * s, n_total) for s in scb]
    return scb, pb


class Comm:
    """Collectives over a torch.distributed process group on the engine's tensors."""

    def __init__(self, group=None, always: bool = False):
        """always (or SFCNL_COMM_ALWAYS=1): issue the collectives at world size 1 too
        instead of short-circuiting them (exercises the NCCL path on one GPU)."""
        import os
        dist = _torch().distributed
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.staged = dist.get_backend(group) != "nccl"
        self.alone = self.world == 1 and not (always or os.environ.get("SFCNL_COMM_ALWAYS") == "1")

    def _in(self, t):
        return t.cpu() if (self.staged and t.is_cuda) else t

    def allreduce_(self, t, op="sum"):
        dist = _torch().distributed
        o = {"sum": dist.ReduceOp.SUM, "min": dist.ReduceOp.MIN, "max": dist.ReduceOp.MAX}[op]
        if self.alone:
            return t
        c = self._in(t)
        dist.all_reduce(c, op=o, group=self.group)
        if c is not t:
            t.copy_(c)
        return t

    def all_gather(self, t):
        """Equal-size all-gather along dim 0 -> [world, *t.shape]."""
        torch = _torch()
        if self.alone:
            return t.unsqueeze(0).clone()
        c = self._in(t.contiguous())
        out = torch.empty((self.world * c.shape[0],) + tuple(c.shape[1:]), dtype=c.dtype, device=c.device)
        torch.distributed.all_gather_into_tensor(out, c, group=self.group)
        return out.view((self.world,) + tuple(c.shape)).to(t.device)

    def all_gather_v(self, t, counts: Sequence[int]):
        """Concatenation over ranks of t (dim 0), rank q contributing counts[q] rows."""
        torch = _torch()
        if self.alone:
            return t.clone()
        m = max(max(counts), 1)
        pad = torch.zeros((m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        g = self.all_gather(pad)
        return torch.cat([g[q, : counts[q]] for q in range(self.world)])

    def all_to_all_v(self, t, send: Sequence[int], recv: Sequence[int]):
        torch = _torch()
        if self.alone:
            return t.clone()
        c = self._in(t.contiguous())
        out = torch.empty((int(sum(recv)),) + tuple(c.shape[1:]), dtype=c.dtype, device=c.device)
        torch.distributed.all_to_all_single(out, c, output_split_sizes=[int(v) for v in recv],
                                            input_split_sizes=[int(v) for v in send], group=self.group)
        return out.to(t.device)


@dataclass
class RankResult:
    rank: int
    n_total: int
    p_begin: int
    p_end: int
    sc_begin: int
    sc_end: int
    num_nodes: int
    halo_particles: int
    store: Optional[NeighborStore]
    results: List[Optional[ReduceResult]]


def _ptr(t):
    return C.c_void_p(int(t.data_ptr()))


def _ptr_array(ts):
    return (C.c_void_p * len(ts))(*[int(t.data_ptr()) for t in ts])


class _CudaEngineLocal:
    """O(owned + halo) steps of CudaEngine (include/sfcnl_cu.h section (6b), dd.cu)."""

    supports_local = True

    def key_hist(self, prefix, shift):
        torch = _torch()
        nq = int(prefix.numel())
        h = torch.zeros((nq, 65536), dtype=torch.int64, device=self.device)
        self.ctx.check(self.ctx.L.sfcnl_cu_key_hist(self.ctx.h, nq, _ptr(prefix), int(shift), _ptr(h)))
        return h

    def merge_owned(self, moved, runs):
        """Step 4: the received runs merged (dd.cu k_merge_runs) into owned columns."""
        torch = _torch()
        nf = 4 + len(self.fields)
        n = int(moved[0].shape[0])
        self.owned = [torch.empty(n, dtype=torch.float64, device=self.device) for _ in range(nf)]
        cols = [c.contiguous() for c in moved[:nf]]
        keys = moved[nf].contiguous()
        bnd = (C.c_uint64 * (len(runs) + 1))(*np.concatenate([[0], np.cumsum(runs)]).astype(np.uint64).tolist())
        self.ctx.check(self.ctx.L.sfcnl_cu_merge_runs(self.ctx.h, n, nf, _ptr_array(cols), _ptr(keys), len(runs), bnd,
                                                      _ptr_array(self.owned)))
        self.n_owned = n

    def max_h(self):
        torch = _torch()
        if self.n_owned == 0:
            return torch.zeros(1, dtype=torch.float64, device=self.device)
        return self.owned[3].max().view(1).clone()

    def octree_dist(self, bucket, n_global, comm):
        """Step 5: the single-domain octree from the step-1 local keys (octree.cu with a
        DistTree); the per-level all-reduce runs on the context's stream."""
        torch = _torch()
        dev = self.device

        def cb(user, ptr, count):
            try:
                class _V:
                    __cuda_array_interface__ = {"shape": (int(count),), "typestr": "<i4", "data": (int(ptr), False),
                                                "version": 3, "strides": None}
                comm.allreduce_(torch.as_tensor(_V(), device=dev), "sum")
                return 0
            except Exception:  # reported as a CUDA-class error by the context
                return 1

        from . import _native as N
        self._cb = N.ALLREDUCE_U32(cb)  # keep alive for the call
        nn = C.c_uint64()
        self.ctx.check(self.ctx.L.sfcnl_cu_build_octree_dist(self.ctx.h, int(bucket), int(n_global), self._cb, None,
                                                             C.byref(nn)))
        self.num_nodes = nn.value
        return nn.value

    def nodes_i32(self):
        torch = _torch()
        return self.ctx.device_array("nodes", torch.int32, self.num_nodes * 8).view(self.num_nodes, 8)

    def straddling_leaves(self, bounds):
        """Leaves whose global particle range contains an interior rank boundary."""
        torch = _torch()
        nd = self.nodes_i32()
        pb, pe, fc = nd[:, 4].to(torch.int64), nd[:, 5].to(torch.int64), nd[:, 6]
        b = torch.tensor(list(bounds), dtype=torch.int64, device=self.device).view(1, -1)
        hit = ((pb.view(-1, 1) < b) & (pe.view(-1, 1) > b)).any(1) & (fc < 0)
        return torch.nonzero(hit).view(-1)

    def leaf_boxes(self, p0, p1):
        torch = _torch()
        lb = torch.empty((self.num_nodes, 6), dtype=torch.float64, device=self.device)
        x, y, z = self.owned[0], self.owned[1], self.owned[2]
        self.ctx.check(self.ctx.L.sfcnl_cu_leaf_boxes(self.ctx.h, int(p0), int(p1), _ptr(x), _ptr(y), _ptr(z), _ptr(lb)))
        return lb

    def domain_boxes(self, k):
        torch = _torch()
        db = torch.empty((k, 6), dtype=torch.float64, device=self.device)
        if self.n_owned == 0:
            db[:, :3], db[:, 3:] = float("inf"), float("-inf")
            return db
        x, y, z = self.owned[0], self.owned[1], self.owned[2]
        self.ctx.check(self.ctx.L.sfcnl_cu_domain_boxes(self.ctx.h, self.n_owned, _ptr(x), _ptr(y), _ptr(z), k, _ptr(db)))
        return db

    def halo_select(self, p0, p1, cj, lb, boxes, rank, reach):
        torch = _torch()
        P, K = int(boxes.shape[0]), int(boxes.shape[1])
        ncl = (p1 - p0 + cj - 1) // cj
        flags = torch.zeros((P, max(ncl, 1)), dtype=torch.uint8, device=self.device)
        bx = boxes.contiguous()
        self.ctx.check(self.ctx.L.sfcnl_cu_halo_select(self.ctx.h, int(p0), int(p1), int(cj), _ptr(lb), P, int(rank), K,
                                                       _ptr(bx), float(reach), _ptr(flags)))
        return flags[:, :ncl]

    def pack_clusters(self, p0, p1, cj, ids):
        torch = _torch()
        nf = 4 + len(self.fields)
        ids32 = ids.to(torch.int32).contiguous()
        rows = torch.empty((int(ids.numel()) * cj, nf), dtype=torch.float64, device=self.device)
        self.ctx.check(self.ctx.L.sfcnl_cu_pack_clusters(self.ctx.h, int(p0), int(p1), int(cj), _ptr(ids32),
                                                         int(ids.numel()), nf, _ptr_array(self.owned), _ptr(rows)))
        return rows

    def place_local(self, n_global, p0, p1, cj, halo_ids, halo_rows):
        """Step 8: local index space (dd.cu); returns the local offset of the owned block."""
        torch = _torch()
        dev = self.device
        ngc = (n_global + cj - 1) // cj
        c0, c1 = p0 // cj, (p1 + cj - 1) // cj
        present = torch.zeros(ngc, dtype=torch.uint8, device=dev)
        present[c0:c1] = 1
        hid = halo_ids.to(torch.int64)
        if hid.numel():
            present[hid] = 1
        below = int(present[:c0].sum().item())
        o_own = ((below * cj + SC - 1) // SC) * SC
        pad_cl = (o_own - below * cj) // cj
        cs = torch.cumsum(present.to(torch.int64), 0)
        lpos64 = torch.zeros(ngc + 1, dtype=torch.int64, device=dev)
        lpos64[1:] = cs
        lpos64[c0:] += pad_cl
        nlc = int(lpos64[ngc].item())
        last_partial = n_global % cj
        n_local = nlc * cj
        if last_partial and bool(present[ngc - 1].item()):
            n_local -= cj - last_partial
        lpos = lpos64.to(torch.int32).contiguous()
        self.ctx.alloc_sorted(n_local, self.box, self.fields)
        lc2g = torch.empty(max(nlc, 1), dtype=torch.int32, device=dev)
        L, h = self.ctx.L, self.ctx.h
        self.ctx.check(L.sfcnl_cu_dd_lc2g(h, ngc, _ptr(lpos), _ptr(present), _ptr(lc2g), nlc))
        hid32 = hid.to(torch.int32).contiguous()
        rows = halo_rows.contiguous()
        self.ctx.check(L.sfcnl_cu_dd_place(h, int(n_global), int(p0), int(p1), int(cj), _ptr(lpos), n_local,
                                           4 + len(self.fields), _ptr_array(self.owned), _ptr(hid32),
                                           int(hid.numel()), _ptr(rows), _ptr(lc2g)))
        self.ctx.check(L.sfcnl_cu_dd_localize(h, int(cj), _ptr(lpos), _ptr(present), ngc, _ptr(lc2g)))
        if o_own == 0 and n_local == n_global:  # one rank: the local space is the global one
            self.ctx.check(L.sfcnl_cu_dd_clear(h))
        self._maps = (lpos, present, lc2g)  # the context keeps raw pointers to lpos / lc2g
        self.owned = None  # placed: the staging columns are released
        self.n_local = n_local
        self.n_total = n_global
        return o_own

    def memory_bytes(self):
        v = C.c_uint64()
        self.ctx.check(self.ctx.L.sfcnl_cu_memory_bytes(self.ctx.h, C.byref(v)))
        return v.value


class CudaEngine(_CudaEngineLocal):
    """Per-rank work on one GPU through the C-ABI context (device-resident)."""

    def __init__(self, ctx: Context, box: SimulationBox, field_names: Sequence[str], bits=kDefaultSfcBits):
        self.cj = 8
        self.ctx, self.box, self.fields = ctx, box, list(field_names)
        self.bits = bits
        torch = _torch()
        self.device = torch.device(f"cuda:{ctx.device}")
        self.stream = torch.cuda.ExternalStream(ctx.stream(), device=self.device)
        self.n_total = 0
        self.num_nodes = 0

    # -- inputs: the rank's particles stay resident (device copies) across steps
    def upload(self, ps: ParticleSet):
        """The rank's input particles into the context's input slot (device copies that stay
        resident across steps; the staging tensors are released)."""
        torch = _torch()
        cols = [ps.x, ps.y, ps.z, ps.h] + [ps.field(k) for k in self.fields]
        with torch.cuda.stream(self.stream):
            inp = [torch.from_numpy(np.ascontiguousarray(c)).to(self.device, non_blocking=True) for c in cols]
            self.ctx.set_particles_device(ps.size(), inp, self.fields, self.box)
            self.ctx.synchronize()
        self.n_in = ps.size()

    def _cols(self, n):
        torch = _torch()
        return [self.ctx.device_array(a, torch.float64, n) for a in ["x", "y", "z", "h"] + self.fields]

    # -- (1) local sort; returns sorted keys (int64)
    def local_sort(self):
        torch = _torch()
        self.ctx.sort(self.bits)
        self.ctx.apply_order()
        return self.ctx.device_array("keys", torch.int64, self.n_in)

    def payload(self):
        """Columns in local key order: x, y, z, h, fields, and the key's bits as a float64
        (one all-to-all per contiguous column: no row packing)."""
        torch = _torch()
        keys = self.ctx.device_array("keys", torch.int64, self.n_in)
        return self._cols(self.n_in) + [keys.view(torch.float64)]

    # -- (4) owner placement; returns the owned sorted keys
    def own(self, recv, n_total, p0, runs=None):
        """The received rows are P runs (one per source rank, source order), each sorted
        by (key, global id); their merge in (key, source rank) order is the global
        (key, global id) order. Position of a row of run s = its index in s + the
        number of rows of runs q < s with key <= its key + of runs q > s with key < its
        key (binary searches, no re-sort). The rows are written straight into the
        global-index arrays at [p0, p0 + n)."""
        torch = _torch()
        nf = 4 + len(self.fields)
        cols_in = list(recv) if isinstance(recv, (list, tuple)) else [recv[:, f] for f in range(nf + 1)]
        n = cols_in[0].shape[0]
        keys = cols_in[nf].contiguous().view(torch.int64)
        runs = [n] if runs is None else [int(v) for v in runs]
        bnd = np.concatenate([[0], np.cumsum(runs)]).astype(np.int64)
        nonempty = [q for q in range(len(runs)) if runs[q]]
        if len(nonempty) <= 1:
            dest = None
        else:
            dest = torch.empty(n, dtype=torch.int64, device=keys.device)
            for s_ in nonempty:
                seg = keys[bnd[s_]:bnd[s_ + 1]]
                acc = torch.arange(seg.numel(), dtype=torch.int64, device=keys.device)
                for q in nonempty:
                    if q != s_:
                        acc += torch.searchsorted(keys[bnd[q]:bnd[q + 1]], seg, right=q < s_)
                dest[bnd[s_]:bnd[s_ + 1]] = acc
        self.ctx.alloc_sorted(n_total, self.box, self.fields)
        cols = self._cols(n_total)
        for f in range(nf):
            dst = cols[f].narrow(0, p0, n)
            if dest is None:
                dst.copy_(cols_in[f])
            else:
                dst.index_copy_(0, dest, cols_in[f].contiguous())
        self.n_total = n_total
        if dest is None:
            return keys.clone()
        out = torch.empty_like(keys)
        out.index_copy_(0, dest, keys)
        return out

    # -- (5) global octree
    def octree(self, gkeys, bucket):
        self.ctx.set_keys_device(gkeys, self.bits)
        self.num_nodes = self.ctx.octree(bucket)
        return self.num_nodes

    # -- (6) partial node geometry: [num_nodes, 8] view (lo3, hi3, maxh, pad), combined in place
    def node_geometry_partial(self, p0, p1):
        torch = _torch()
        self.ctx.node_geometry_range(p0, p1)
        return self.ctx.device_array("node_geo", torch.float64, self.num_nodes * 8).view(self.num_nodes, 8)

    def set_node_geometry(self, geo):
        pass  # combined in place in the context's array

    # -- (7) halo
    def halo_flags(self, bp: BuildParams, sc0, sc1, max_h):
        torch = _torch()
        nj = self.ctx.halo_mark(bp, sc0, sc1)
        return self.ctx.device_array("halo_flags", torch.uint8, nj)

    def gather_rows(self, idx):
        torch = _torch()
        return torch.stack([c[idx] for c in self._cols(self.n_total)], dim=1)

    def scatter_rows(self, idx, rows):
        for f, c in enumerate(self._cols(self.n_total)):
            c[idx] = rows[:, f]

    # -- (8) build + pass
    def build_range(self, bp: BuildParams, sc0, sc1, max_h, download):
        nsc, nb = self.ctx.build_store_range(bp, sc0, sc1, max_h)
        if not download:
            return None
        return self.ctx.get_store(bp, self.n_total, nsc, nb)

    def reduce(self, kernel: Kernel, cfg: PassConfig, nloc, download):
        return self.ctx.reduce(kernel, cfg, nloc, download=download)

    # symmetric stores: entries -> (ship to owners) -> ordered fold (pass_sym.cuh)
    def sym_entries(self, kernel: Kernel, cfg: PassConfig):
        """-> (jacc [E, outputs*cj] f64, jcnt [E, cj] i32, ejcl [E] i32, esc [E] i32) device views."""
        torch = _torch()
        ne = self.ctx.sym_range_entries(kernel, cfg)
        cj, no = self.cj, len(kernel.names)
        if ne == 0:
            z = torch.zeros(0, dtype=torch.int32, device=self.device)
            return torch.zeros((0, no * cj), dtype=torch.float64, device=self.device), z.view(0, 1).expand(0, cj), z, z
        jacc = self.ctx.device_array("sym.jacc", torch.float64, ne * no * cj).view(ne, no * cj)
        jcnt = self.ctx.device_array("sym.jcnt", torch.int32, ne * cj).view(ne, cj)
        ejcl = self.ctx.device_array("sym.ejcl", torch.int32, ne)
        esc = self.ctx.device_array("sym.esc", torch.int32, ne)
        return jacc, jcnt, ejcl, esc

    def sym_final(self, kernel: Kernel, cfg: PassConfig, remote, nloc, download):
        return self.ctx.sym_range_final(kernel, cfg, nloc, remote, download)


class DomainDecomposition:
    """The distributed build-and-query step (module docstring)."""

    def __init__(self, engine, comm: Comm, bp: BuildParams, kernels: Sequence[Kernel], cfg: PassConfig,
                 bucket=64, nbox=32):
        self.E, self.comm, self.bp = engine, comm, bp
        self.nbox = nbox  # chunk boxes per rank for the owner-side halo selection
        self.kernels = list(kernels)
        self.cfg = cfg
        self.bucket = bucket

    def _ctx_stream(self):
        s = getattr(self.E, "stream", None)
        if s is None:
            import contextlib
            return contextlib.nullcontext()
        return _torch().cuda.stream(s)

    def run(self, download=True) -> RankResult:
        with self._ctx_stream():
            local = getattr(self.E, "supports_local", False) and self.bp.mode == 0 and \
                not os.environ.get("SFCNL_DD_LEGACY")
            return self._run_local(download) if local else self._run_legacy(download)

    # ---------------------------------------------------------------- common steps
    def _split(self, keys, counts, pb):
        """Step 2: cut[s, q] = number of rank s's (sorted) keys that go to ranks < q, so that
        rank q receives the global (key, global id) positions [pb[q], pb[q + 1])."""
        torch = _torch()
        E, comm = self.E, self.comm
        P = comm.world
        dev = E.device
        cut = torch.zeros((P, P + 1), dtype=torch.int64, device=dev)
        if P > 1:
            tgt = torch.tensor(pb[1:-1], dtype=torch.int64, device=dev)
            if hasattr(E, "key_hist"):
                # radix select: 4 rounds of 16 key bits; below = #keys < prefix (global)
                prefix = torch.zeros(P - 1, dtype=torch.int64, device=dev)
                below = torch.zeros(P - 1, dtype=torch.int64, device=dev)
                for shift in (48, 32, 16, 0):
                    h = E.key_hist(prefix, shift)
                    comm.allreduce_(h, "sum")
                    cum = torch.cumsum(h, 1)
                    b = torch.searchsorted(cum, (tgt - below).view(-1, 1), right=True).view(-1)
                    prev = torch.gather(cum, 1, (b - 1).clamp(min=0).view(-1, 1)).view(-1)
                    below = below + torch.where(b > 0, prev, torch.zeros_like(prev))
                    prefix = prefix + (b << shift)
                lo = prefix  # the key at global position tgt
            else:
                lo = torch.zeros(P - 1, dtype=torch.int64, device=dev)
                hi = torch.full((P - 1,), KEY_SPAN - 1, dtype=torch.int64, device=dev)
                for _ in range(64):  # smallest K with #(key <= K) > t
                    mid = lo + (hi - lo) // 2
                    c = torch.searchsorted(keys, mid, right=True)
                    comm.allreduce_(c, "sum")
                    ok = c > tgt
                    hi = torch.where(ok, mid, hi)
                    lo = torch.where(ok, lo, mid + 1)
            less = torch.searchsorted(keys, lo, right=False)
            eq = torch.searchsorted(keys, lo, right=True) - less
            less_all = comm.all_gather(less)  # [P, P-1]
            eq_all = comm.all_gather(eq)
            need = tgt - less_all.sum(0)
            eq_before = torch.cumsum(eq_all, 0) - eq_all
            take = torch.minimum(torch.clamp(need.unsqueeze(0) - eq_before, min=0), eq_all)
            cut[:, 1:P] = less_all + take
        cut[:, P] = torch.tensor(counts, dtype=torch.int64, device=dev)
        return cut

    def _run_local(self, download):
        """Gather stores, O(owned + halo) per rank: module docstring steps 1-9."""
        torch = _torch()
        E, comm = self.E, self.comm
        P, r = comm.world, comm.rank
        dev = E.device
        prof = os.environ.get("SFCNL_DD_PROF") is not None and dev.type == "cuda"
        marks = []

        def mark(name):
            if prof:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record()
                marks.append((name, ev))

        mark("start")
        keys = E.local_sort()  # (1)
        mark("local_sort")
        n_l = int(keys.numel())
        counts = comm.all_gather(torch.tensor([n_l], dtype=torch.int64, device=dev)).view(-1).tolist()
        N = int(sum(counts))
        scb, pb = sc_partition(N, P)
        p0, p1 = pb[r], pb[r + 1]
        sc0, sc1 = scb[r], scb[r + 1]
        cut = self._split(keys, counts, pb)  # (2)
        mark("split")
        cut_h = cut.cpu().numpy()
        send = np.diff(cut_h[r]).tolist()
        recv = [int(cut_h[s, r + 1] - cut_h[s, r]) for s in range(P)]
        moved = [comm.all_to_all_v(col, send, recv) for col in E.payload()]  # (3)
        mark("payload_a2a")
        assert int(moved[0].shape[0]) == p1 - p0, "distributed split lost particles"
        E.merge_owned(moved, recv)  # (4)
        del moved
        hmax = float(comm.allreduce_(E.max_h(), "max").item())
        mark("merge")
        nn = E.octree_dist(self.bucket, N, comm)  # (5)
        mark("octree")
        lb = E.leaf_boxes(p0, p1)  # (6)
        strad = E.straddling_leaves(pb[1:-1]) if P > 1 else None
        if strad is not None and strad.numel():
            part = lb[strad]
            lo, hi = part[:, :3].contiguous(), part[:, 3:].contiguous()
            comm.allreduce_(lo, "min")
            comm.allreduce_(hi, "max")
            lb[strad] = torch.cat([lo, hi], 1)
        mark("leaf_boxes")
        cj = self.bp.params.cj
        halo = 0
        hids = torch.zeros(0, dtype=torch.int64, device=dev)
        hrows = torch.zeros((0, 4 + len(getattr(E, "fields", []))), dtype=torch.float64, device=dev)
        if P > 1:  # (7)
            boxes = comm.all_gather(E.domain_boxes(self.nbox))  # [P, K, 6]
            reach = self.bp.build_radius_scale * hmax
            flags = E.halo_select(p0, p1, cj, lb, boxes, r, reach)
            c0 = p0 // cj
            ids = [torch.nonzero(flags[q]).view(-1) + c0 for q in range(P)]
            nsend = torch.tensor([int(t.numel()) for t in ids], dtype=torch.int64, device=dev)
            mat = comm.all_gather(nsend).cpu().numpy()  # mat[s, q] = clusters s sends to q
            sendc, recvc = mat[r].tolist(), mat[:, r].tolist()
            allids = torch.cat(ids)
            hids = comm.all_to_all_v(allids, sendc, recvc)
            rows = E.pack_clusters(p0, p1, cj, allids)
            hrows = comm.all_to_all_v(rows, [v * cj for v in sendc], [v * cj for v in recvc])
            halo = int(hids.numel()) * cj
        mark("halo")
        o_own = E.place_local(N, p0, p1, cj, hids, hrows)  # (8)
        lsc0 = o_own // SC
        lsc1 = lsc0 + (sc1 - sc0)
        mark("local_space")
        store = E.build_range(self.bp, lsc0, lsc1, hmax, download)  # (9)
        mark("build")
        results = [E.reduce(k, self.cfg, p1 - p0, download) for k in self.kernels]
        mark("passes")
        if prof:
            marks[-1][1].synchronize()
            print("dd phases ms:", {b[0]: round(a[1].elapsed_time(b[1]), 2) for a, b in zip(marks, marks[1:])},
                  flush=True)
        return RankResult(r, N, p0, p1, sc0, sc1, nn, halo, store, results)

    def _run_legacy(self, download):
        torch = _torch()
        E, comm = self.E, self.comm
        P, r = comm.world, comm.rank
        dev = E.device
        prof = os.environ.get("SFCNL_DD_PROF") is not None and dev.type == "cuda"
        marks = []

        def mark(name):
            if prof:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record()
                marks.append((name, ev))

        mark("start")
        # (1) local keys
        keys = E.local_sort()
        mark("local_sort")
        n_l = int(keys.numel())
        counts = comm.all_gather(torch.tensor([n_l], dtype=torch.int64, device=dev)).view(-1).tolist()
        N = int(sum(counts))
        scb, pb = sc_partition(N, P)
        cut = self._split(keys, counts, pb)  # (2) exact split at the interior bounds
        mark("split")
        cut_h = cut.cpu().numpy()
        send = np.diff(cut_h[r]).tolist()
        recv = [int(cut_h[s, r + 1] - cut_h[s, r]) for s in range(P)]
        # (3) payload to owners
        pay = E.payload()
        if isinstance(pay, (list, tuple)):
            moved = [comm.all_to_all_v(col, send, recv) for col in pay]
            n_moved = int(moved[0].shape[0])
        else:
            moved = comm.all_to_all_v(pay, send, recv)
            n_moved = int(moved.shape[0])
        mark("payload_a2a")
        # (4) owners place their particles at global positions [p0, p1)
        p0, p1 = pb[r], pb[r + 1]
        assert n_moved == p1 - p0, "distributed split lost particles"
        own_keys = E.own(moved, N, p0, recv)
        mark("own_sort_place")
        # (5) global keys -> global octree
        gkeys = comm.all_gather_v(own_keys, [pb[q + 1] - pb[q] for q in range(P)])
        mark("gather_keys")
        nn = E.octree(gkeys, self.bucket)
        mark("octree")
        # (6) node geometry: partial over owned particles, exact MIN all-reduce
        geo = E.node_geometry_partial(p0, p1)
        geo[:, 3:7].neg_()
        comm.allreduce_(geo, "min")
        geo[:, 3:7].neg_()
        E.set_node_geometry(geo)
        max_h = float(geo[0, 6]) if nn else 0.0  # root max h = max over all particles
        mark("node_geometry")
        # (7) halo exchange
        sc0, sc1 = scb[r], scb[r + 1]
        halo = 0
        if P > 1:
            cj = self.bp.params.cj
            flags = E.halo_flags(self.bp, sc0, sc1, max_h)
            jc = torch.nonzero(flags).view(-1).to(torch.int64)
            first = jc * cj
            jc = jc[(first < p0) | (first >= p1)]
            bounds = torch.tensor(pb[1:], dtype=torch.int64, device=dev)
            owner = torch.searchsorted(bounds, jc * cj, right=True)
            req = torch.bincount(owner, minlength=P)
            req_all = comm.all_gather(req).cpu().numpy()  # [P, P]: req_all[s, q] = s asks q
            send_req = req_all[r].tolist()
            recv_req = req_all[:, r].tolist()
            asked = comm.all_to_all_v(jc, send_req, recv_req)
            lane = torch.arange(cj, dtype=torch.int64, device=dev)
            aidx = (asked.unsqueeze(1) * cj + lane).view(-1).clamp_(max=N - 1)
            rows = E.gather_rows(aidx)
            back = comm.all_to_all_v(rows, [v * cj for v in recv_req], [v * cj for v in send_req])
            widx = (jc.unsqueeze(1) * cj + lane).view(-1)
            keep = widx < N
            E.scatter_rows(widx[keep], back[keep])
            halo = int(keep.sum())
        mark("halo")
        # (8) range build + pass
        store = E.build_range(self.bp, sc0, sc1, max_h, download)
        mark("build")
        if self.bp.mode != 0:  # symmetric: entries shipped to the owners of their j-clusters
            results = [self._sym_reduce(k, pb, p1 - p0, download) for k in self.kernels]
        else:
            results = [E.reduce(k, self.cfg, p1 - p0, download) for k in self.kernels]
        mark("passes")
        if prof:
            marks[-1][1].synchronize()
            print("dd phases ms:", {b[0]: round(a[1].elapsed_time(b[1]), 2) for a, b in zip(marks, marks[1:])},
                  flush=True)
        return RankResult(r, N, p0, p1, sc0, sc1, nn, halo, store, results)


def _sym_reduce_impl(self, kernel, pb, nloc, download):
    """Symmetric pass over the rank's range (sfcnl_cu_sym_range_*): every entry's j-side
    accumulators go to the rank owning its j-cluster (a later rank or this one), which
    folds the received ones (earlier ranks, rank order = global entry order) before its
    own in the reference order."""
    torch = _torch()
    E, comm = self.E, self.comm
    P, r = comm.world, comm.rank
    dev = E.device
    E.cj = self.bp.params.cj
    jacc, jcnt, ejcl, esc = E.sym_entries(kernel, self.cfg)
    cj, no = self.bp.params.cj, len(kernel.names)
    remote = None
    if P > 1:
        bounds = torch.tensor(pb[1:], dtype=torch.int64, device=dev)
        owner = torch.searchsorted(bounds, ejcl.to(torch.int64) * cj, right=True)
        sel = torch.nonzero(owner != r).view(-1)
        order = torch.argsort(owner[sel], stable=True)
        sel = sel[order]
        rows = torch.cat([jacc[sel], jcnt[sel].to(torch.float64), ejcl[sel].to(torch.float64).unsqueeze(1),
                          esc[sel].to(torch.float64).unsqueeze(1)], dim=1)
        send = torch.bincount(owner[sel], minlength=P)
        mat = comm.all_gather(send).cpu().numpy()  # mat[s, q]: s sends q
        got = comm.all_to_all_v(rows, mat[r].tolist(), mat[:, r].tolist())
        if got.shape[0]:
            remote = (got[:, :no * cj].contiguous(), got[:, no * cj:no * cj + cj].to(torch.int32).contiguous(),
                      got[:, no * cj + cj].to(torch.int32).contiguous(), got[:, no * cj + cj + 1].to(torch.int32).contiguous())
    return E.sym_final(kernel, self.cfg, remote, nloc, download)


DomainDecomposition._sym_reduce = _sym_reduce_impl


def merge_stores(parts: Sequence[NeighborStore]) -> NeighborStore:
    """Concatenate per-rank range stores (rank order) into the single-domain layout."""
    counts = np.concatenate([p.counts for p in parts])
    blobs, offs, base = [], [], 0
    for p in parts:
        offs.append(np.asarray(p.offsets[:-1], np.uint64) + np.uint64(base))
        blobs.append(np.asarray(p.blob, np.uint8))
        base += len(p.blob)
    offs.append(np.array([base], np.uint64))
    return NeighborStore(parts[0].build, parts[0].n, counts, np.concatenate(offs), np.concatenate(blobs))
