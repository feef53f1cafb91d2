"""Python mirror of the reference's public C++ API (``/root/reference/proj/include/sfcnl``)
over the B200 C-ABI. Names, argument meaning and error types follow the
reference so the parity tests read like the reference's own tests:

=============================  ===========================================
reference (C++)                here
=============================  ===========================================
``sort_by_sfc`` hilbert.hpp:126        :func:`sort_by_sfc` (GPU K1+K2)
``apply_sfc_order`` hilbert.hpp:129    :func:`apply_sfc_order` (GPU K3)
``build_octree`` octree.hpp:51         :func:`build_octree` (GPU K5)
``compute_node_aabbs`` octree.hpp:57   :func:`compute_node_aabbs` (GPU)
``build_neighbor_store`` neighbor_build.hpp:18  :func:`build_neighbor_store` (GPU K4,K6,K7)
``reduce<Real,K>`` reduce.hpp:38       :func:`reduce` (GPU K8)
``codec::*`` nibble_codec.hpp          :mod:`codec` functions (host)
``make_uniform/make_evrard``           :func:`make_uniform` / :func:`make_evrard` (host)
=============================  ===========================================

``threads`` arguments are accepted and ignored (the GPU grid replaces
parallel_for, parallel.hpp:22). Every free function runs on a per-process default
:class:`Context` (device = LOCAL_RANK or 0) unless one is passed.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import struct
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N
from ._native import BuildError, DecodeError, InputError  # noqa: F401  (re-exported)

kDefaultSfcBits = 21
kSuperClusterSize = 64


def _ptr(a):
    return C.c_void_p(a.ctypes.data) if a is not None and a.size else C.c_void_p(0)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ----------------------------------------------------------------- value types
@dataclass
class SimulationBox:
    """core.hpp:50-74."""
    lo: Tuple[float, float, float] = (0.0, 0.0, 0.0)
    hi: Tuple[float, float, float] = (1.0, 1.0, 1.0)
    periodic: Tuple[bool, bool, bool] = (False, False, False)

    def __post_init__(self):
        self.lo = tuple(float(v) for v in self.lo)
        self.hi = tuple(float(v) for v in self.hi)
        self.periodic = tuple(bool(v) for v in self.periodic)
        for d in range(3):
            if not (self.hi[d] > self.lo[d]):
                raise InputError("SimulationBox: hi must exceed lo on every axis")

    def length(self, d):
        return self.hi[d] - self.lo[d]

    def c(self):
        b = N.Box()
        for d in range(3):
            b.lo[d], b.hi[d], b.periodic[d] = self.lo[d], self.hi[d], int(self.periodic[d])
        return b


@dataclass
class ParticleSet:
    """core.hpp:168-198 (SoA positions, radii and named fields)."""
    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    h: np.ndarray
    fields: Dict[str, np.ndarray] = field(default_factory=dict)

    def __post_init__(self):
        self.x, self.y, self.z, self.h = (_f64(v) for v in (self.x, self.y, self.z, self.h))
        self.fields = {k: _f64(v) for k, v in self.fields.items()}

    def size(self):
        return len(self.x)

    def field(self, name):
        if name not in self.fields:
            raise InputError("ParticleSet: no such field: " + name)
        return self.fields[name]

    def check(self):
        n = len(self.x)
        if len(self.y) != n or len(self.z) != n or len(self.h) != n:
            raise InputError("ParticleSet: array length mismatch")
        for k, v in self.fields.items():
            if len(v) != n:
                raise InputError("ParticleSet: field length mismatch: " + k)


@dataclass
class SfcOrder:
    """hilbert.hpp:116-122."""
    keys: np.ndarray
    perm: np.ndarray
    bits: int = kDefaultSfcBits

    def size(self):
        return len(self.keys)


NODE_DTYPE = np.dtype([("key_first", "<u8"), ("key_last", "<u8"), ("particle_begin", "<u4"),
                       ("particle_end", "<u4"), ("first_child", "<i4"), ("depth", "u1"),
                       ("pad_", "u1", (3,))])
assert NODE_DTYPE.itemsize == 32


@dataclass
class Octree:
    """octree.hpp:11-46; ``nodes`` is a structured array in OctreeNode layout."""
    nodes: np.ndarray
    bits: int = kDefaultSfcBits
    n: int = 0


@dataclass
class ClusterParams:
    """cluster.hpp:12-29."""
    ci: int = 8
    cj: int = 8
    w: int = 32
    sc_size: int = kSuperClusterSize

    def __post_init__(self):
        if self.ci == 0 or self.cj == 0:
            raise InputError("ClusterParams: cluster sizes must be positive")
        if self.sc_size % self.ci or self.sc_size % self.cj:
            raise InputError("ClusterParams: cluster sizes must divide the super-cluster size")
        if self.ci % self.cj:
            raise InputError("ClusterParams: cj must divide ci")
        if self.w not in (32, 64):
            raise InputError("ClusterParams: block width must be 32 or 64")

    def iclusters_per_sc(self):
        return self.sc_size // self.ci

    def mask_bytes_per_entry(self):
        return (self.iclusters_per_sc() + 7) // 8


GATHER, SYMMETRIC = 0, 1


@dataclass
class BuildParams:
    """neighbor_store.hpp:18-29."""
    params: ClusterParams = field(default_factory=ClusterParams)
    mode: int = GATHER
    compress: bool = True
    build_radius_scale: float = 1.0

    def __post_init__(self):
        if not (self.build_radius_scale >= 1.0):
            raise InputError("BuildParams: build_radius_scale must be >= 1")

    def c(self):
        return N.BuildParamsC(self.params.ci, self.params.cj, self.params.w, int(self.mode),
                              int(bool(self.compress)), float(self.build_radius_scale))


@dataclass
class NeighborStore:
    """neighbor_store.hpp:44-59."""
    build: BuildParams
    n: int
    counts: np.ndarray
    offsets: np.ndarray
    blob: np.ndarray

    def num_superclusters(self):
        return len(self.counts)

    def header_bytes(self):
        return 4 * len(self.counts) + 8 * len(self.offsets)

    def total_bytes(self):
        return self.header_bytes() + len(self.blob)


@dataclass
class FullVerletList:
    """baselines.hpp:27-38: classic per-particle Verlet list in CSR form, neighbors ascending."""
    mode: int = GATHER
    build_scale: float = 1.0
    offsets: np.ndarray = field(default_factory=lambda: np.zeros(1, np.uint64))
    neighbors: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))

    def memory_bytes(self):
        return 8 * len(self.offsets) + 4 * len(self.neighbors)


@dataclass
class MemoryFootprint:
    total_bytes: int
    bytes_per_particle: float


_STORE_MAGIC = b"SFNLSTOR"
_STORE_HEAD = struct.Struct("<8sIBBHIIIIdQQQ")  # magic, version, mode, compress, reserved, ci, cj, sc, w, scale, n, nsc, nb


def write_store(store: NeighborStore, path_or_file) -> None:
    """write_store (neighbor_store.hpp:79-82, neighbor_store.cpp:84-103): the
    "SFNLSTOR" v1 little-endian dump -- header, counts (u32), offsets (u64), blob."""
    p = store.build.params
    head = _STORE_HEAD.pack(_STORE_MAGIC, 1, int(store.build.mode), 1 if store.build.compress else 0, 0,
                            p.ci, p.cj, p.sc_size, p.w, float(store.build.build_radius_scale), int(store.n),
                            len(store.counts), len(store.blob))
    body = [np.ascontiguousarray(store.counts, "<u4").tobytes(), np.ascontiguousarray(store.offsets, "<u8").tobytes(),
            np.ascontiguousarray(store.blob, np.uint8).tobytes()]
    if isinstance(path_or_file, (str, bytes, os.PathLike)):
        with open(path_or_file, "wb") as f:
            f.write(head), [f.write(b) for b in body]
    else:
        path_or_file.write(head), [path_or_file.write(b) for b in body]


def read_store(path_or_file) -> NeighborStore:
    """read_store (neighbor_store.hpp:83-86, neighbor_store.cpp:110-146), same errors:
    DecodeError("bad store magic", 0), ("unsupported store version", 8),
    ("unsupported super-cluster size", 0), ("store file truncated", offset)."""
    if isinstance(path_or_file, (str, bytes, os.PathLike)):
        with open(path_or_file, "rb") as f:
            data = f.read()
    else:
        data = path_or_file.read()
    if len(data) < 8 or data[:8] != _STORE_MAGIC:
        raise DecodeError("bad store magic", 0)
    if len(data) < 12:
        raise DecodeError("store file truncated", len(data))
    if struct.unpack_from("<I", data, 8)[0] != 1:
        raise DecodeError("unsupported store version", 8)
    if len(data) < _STORE_HEAD.size:
        raise DecodeError("store file truncated", len(data))
    _, _, mode, comp, _, ci, cj, sc, w, scale, n, nsc, nb = _STORE_HEAD.unpack_from(data, 0)
    if sc != kSuperClusterSize:
        raise DecodeError("unsupported super-cluster size", 0)
    o = _STORE_HEAD.size
    need = o + 4 * nsc + 8 * (nsc + 1) + nb
    if len(data) < need:
        raise DecodeError("store file truncated", len(data))
    counts = np.frombuffer(data, "<u4", nsc, o).astype(np.uint32)
    offsets = np.frombuffer(data, "<u8", nsc + 1, o + 4 * nsc).astype(np.uint64)
    blob = np.frombuffer(data, np.uint8, nb, o + 4 * nsc + 8 * (nsc + 1)).copy()
    bp = BuildParams(ClusterParams(ci, cj, w), GATHER if mode == 0 else SYMMETRIC, comp != 0, scale)
    return NeighborStore(bp, n, counts, offsets, blob)


def memory_footprint(store: NeighborStore) -> MemoryFootprint:
    """neighbor_store.cpp:56-61."""
    t = store.total_bytes()
    return MemoryFootprint(t, t / store.n if store.n else 0.0)


# ----------------------------------------------------------------- kernels
@dataclass
class Kernel:
    """The built-in pair kernels (builtin_kernels.hpp:24-122)."""
    kind: int
    names: Tuple[str, ...]
    epsilon: float = 1.0
    sigma: float = 1.0
    coulomb_k: float = 0.0


def count_kernel():
    return Kernel(0, ("count",))


def sph_density_kernel():
    return Kernel(1, ("rho",))


def lj_kernel(epsilon, sigma):
    return Kernel(2, ("fx", "fy", "fz", "energy"), float(epsilon), float(sigma))


def lj_coulomb_kernel(epsilon, sigma, coulomb_k):
    return Kernel(3, ("fx", "fy", "fz", "energy"), float(epsilon), float(sigma), float(coulomb_k))


F64, MIXED = 0, 1


@dataclass
class PassConfig:
    """pair_kernel.hpp:95-105. ``precision``: F64 (bitwise reduce<double>) or MIXED
    (reduce<float> slot; exact pair set, values within 1e-5 of fp64)."""
    query_scale: float = 1.0
    precision: int = F64
    threads: int = 1

    def __post_init__(self):
        if not (self.query_scale >= 0):
            raise InputError("PassConfig: query_scale must be >= 0")


@dataclass
class ReduceResult:
    """pair_kernel.hpp:109-120."""
    names: List[str]
    outputs: List[np.ndarray]
    neighbor_count: np.ndarray

    def output(self, name):
        for k, nm in enumerate(self.names):
            if nm == name:
                return self.outputs[k]
        raise InputError("ReduceResult: no such output: " + name)


# ----------------------------------------------------------------- context
class Context:
    """One CUDA stream + device-resident state on one GPU (``sfcnl_cu_ctx``)."""

    def __init__(self, device: Optional[int] = None):
        L = N.lib()
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", "0"))
        h = C.c_void_p()
        rc = L.sfcnl_cu_ctx_create(int(device), C.byref(h))
        if rc:
            N.raise_for(rc, L.sfcnl_cu_last_error(None, None).decode())
        self.h = h
        self.device = device
        self.L = L

    def close(self):
        if getattr(self, "h", None):
            self.L.sfcnl_cu_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc):
        if rc:
            off = C.c_uint64(0)
            msg = self.L.sfcnl_cu_last_error(self.h, C.byref(off)).decode()
            N.raise_for(rc, msg, off.value)

    # raw C-ABI wrappers --------------------------------------------------
    def set_particles(self, ps: ParticleSet, box: SimulationBox, sorted_slot=False):
        ps.check()
        b = box.c()
        f = self.L.sfcnl_cu_set_sorted_particles if sorted_slot else self.L.sfcnl_cu_set_particles
        self.check(f(self.h, ps.size(), _ptr(ps.x), _ptr(ps.y), _ptr(ps.z), _ptr(ps.h), C.byref(b)))
        g = self.L.sfcnl_cu_set_sorted_field if sorted_slot else self.L.sfcnl_cu_set_field
        for name, v in ps.fields.items():
            self.check(g(self.h, name.encode(), _ptr(v)))

    def sort(self, bits=kDefaultSfcBits):
        self.check(self.L.sfcnl_cu_sort_by_sfc(self.h, int(bits)))

    def get_order(self, n):
        keys = np.empty(n, np.uint64)
        perm = np.empty(n, np.uint32)
        self.check(self.L.sfcnl_cu_get_order(self.h, _ptr(keys), _ptr(perm)))
        return keys, perm

    def set_order(self, order: SfcOrder):
        keys = np.ascontiguousarray(order.keys, np.uint64)
        perm = np.ascontiguousarray(order.perm, np.uint32)
        self.check(self.L.sfcnl_cu_set_order(self.h, len(keys), _ptr(keys), _ptr(perm), int(order.bits)))

    def apply_order(self):
        self.check(self.L.sfcnl_cu_apply_order(self.h))

    def get_sorted(self, name, n):
        out = np.empty(n)
        self.check(self.L.sfcnl_cu_get_sorted(self.h, name.encode(), _ptr(out)))
        return out

    def octree(self, bucket=64):
        nn = C.c_uint64()
        self.check(self.L.sfcnl_cu_build_octree(self.h, int(bucket), C.byref(nn)))
        return nn.value

    def get_octree(self, num_nodes):
        nodes = np.zeros(num_nodes, NODE_DTYPE)
        self.check(self.L.sfcnl_cu_get_octree(self.h, _ptr(nodes)))
        return nodes

    def set_octree(self, tree: Octree):
        nodes = np.ascontiguousarray(tree.nodes, NODE_DTYPE)
        self.check(self.L.sfcnl_cu_set_octree(self.h, len(nodes), _ptr(nodes), int(tree.bits), int(tree.n)))

    def node_geometry(self, num_nodes):
        lo = np.empty((num_nodes, 3))
        hi = np.empty((num_nodes, 3))
        rad = np.empty(num_nodes)
        self.check(self.L.sfcnl_cu_node_geometry(self.h, _ptr(lo), _ptr(hi), _ptr(rad)))
        return lo, hi, rad

    def build_store(self, bp: BuildParams):
        nsc, nb = C.c_uint64(), C.c_uint64()
        p = bp.c()
        self.check(self.L.sfcnl_cu_build_store(self.h, C.byref(p), C.byref(nsc), C.byref(nb)))
        return nsc.value, nb.value

    def get_store(self, bp: BuildParams, n, nsc, nb, into=None) -> NeighborStore:
        """Downloads the store; `into` = (counts, offsets, blob) host arrays to fill
        (e.g. pinned buffers reused across steps), large enough for nsc / nb."""
        if into is not None:
            counts, offsets, blob = into[0][:nsc], into[1][:nsc + 1], into[2][:max(nb, 1)]
        else:
            counts = np.empty(nsc, np.uint32)
            offsets = np.empty(nsc + 1, np.uint64)
            blob = np.empty(max(nb, 1), np.uint8)
        self.check(self.L.sfcnl_cu_get_store(self.h, _ptr(counts), _ptr(offsets), _ptr(blob)))
        return NeighborStore(bp, n, counts, offsets, blob[:nb])

    def set_store(self, store: NeighborStore):
        p = store.build.c()
        counts = np.ascontiguousarray(store.counts, np.uint32)
        offsets = np.ascontiguousarray(store.offsets, np.uint64)
        blob = np.ascontiguousarray(store.blob, np.uint8)
        buf = blob if blob.size else np.zeros(1, np.uint8)
        self.check(self.L.sfcnl_cu_set_store(self.h, C.byref(p), int(store.n), len(counts), _ptr(counts),
                                             _ptr(offsets), _ptr(buf), len(blob)))

    def reduce(self, kernel: Kernel, cfg: PassConfig, n, download=True, into=None):
        """`into` = (list of output arrays, count array) host buffers to fill."""
        pp = N.PassParamsC(kernel.kind, int(cfg.precision), float(cfg.query_scale), kernel.epsilon,
                           kernel.sigma, kernel.coulomb_k)
        nout = len(kernel.names)
        if not download:
            self.check(self.L.sfcnl_cu_reduce(self.h, C.byref(pp), None, None))
            return None
        if into is not None:
            outs, cnt = [o[:n] for o in into[0][:nout]], into[1][:n]
        else:
            outs = [np.empty(n) for _ in range(nout)]
            cnt = np.empty(n, np.uint32)
        arr = (C.c_void_p * 4)(*([o.ctypes.data for o in outs] + [None] * (4 - nout)))
        self.check(self.L.sfcnl_cu_reduce(self.h, C.byref(pp), arr, _ptr(cnt)))
        return ReduceResult(list(kernel.names), outs, cnt)

    # full Verlet list baseline (include/sfcnl_cu.h section (5b)) ----------
    def build_full_list(self, build_scale):
        """Full list of the current whole-range gather store's pairs; returns num_pairs."""
        npairs = C.c_uint64()
        self.check(self.L.sfcnl_cu_build_full_list(self.h, float(build_scale), C.byref(npairs)))
        return npairs.value

    def get_full_list(self, n, num_pairs, build_scale, mode=GATHER) -> FullVerletList:
        offsets = np.empty(n + 1, np.uint64)
        nbrs = np.empty(max(num_pairs, 1), np.uint32)
        self.check(self.L.sfcnl_cu_get_full_list(self.h, _ptr(offsets), _ptr(nbrs)))
        return FullVerletList(mode, float(build_scale), offsets, nbrs[:num_pairs])

    def set_full_list(self, fl: FullVerletList):
        offsets = np.ascontiguousarray(fl.offsets, np.uint64)
        nbrs = np.ascontiguousarray(fl.neighbors, np.uint32)
        if len(offsets) < 1:
            raise InputError("reduce_full: list/particle-set mismatch")
        buf = nbrs if nbrs.size else np.zeros(1, np.uint32)
        self.check(self.L.sfcnl_cu_set_full_list(self.h, len(offsets) - 1, int(fl.mode), float(fl.build_scale),
                                                 _ptr(offsets), _ptr(buf), len(nbrs)))

    def reduce_full(self, kernel: Kernel, cfg: PassConfig, n, download=True):
        pp = N.PassParamsC(kernel.kind, int(cfg.precision), float(cfg.query_scale), kernel.epsilon,
                           kernel.sigma, kernel.coulomb_k)
        nout = len(kernel.names)
        if not download:
            self.check(self.L.sfcnl_cu_reduce_full(self.h, C.byref(pp), None, None))
            return None
        outs = [np.empty(n) for _ in range(nout)]
        cnt = np.empty(n, np.uint32)
        arr = (C.c_void_p * 4)(*([o.ctypes.data for o in outs] + [None] * (4 - nout)))
        self.check(self.L.sfcnl_cu_reduce_full(self.h, C.byref(pp), arr, _ptr(cnt)))
        return ReduceResult(list(kernel.names), outs, cnt)

    def sym_range_entries(self, kernel: Kernel, cfg: PassConfig):
        """Symmetric range store: j-side accumulators of the range's entries (device arrays
        "sym.jacc", "sym.jcnt", "sym.ejcl", "sym.esc"); returns the entry count."""
        pp = N.PassParamsC(kernel.kind, int(cfg.precision), float(cfg.query_scale), kernel.epsilon,
                           kernel.sigma, kernel.coulomb_k)
        ne = C.c_uint64()
        self.check(self.L.sfcnl_cu_sym_range_entries(self.h, C.byref(pp), C.byref(ne)))
        return ne.value

    def sym_range_final(self, kernel: Kernel, cfg: PassConfig, n, remote, download=True):
        """remote = (jacc, jcnt, ejcl, esc) device tensors of the entries received from
        earlier ranks (or None); returns the range particles' ReduceResult."""
        pp = N.PassParamsC(kernel.kind, int(cfg.precision), float(cfg.query_scale), kernel.epsilon,
                           kernel.sigma, kernel.coulomb_k)
        nr = 0 if remote is None else int(remote[3].numel())
        ptrs = [None] * 4 if not nr else [int(t.data_ptr()) for t in remote]
        nout = len(kernel.names)
        if not download:
            self.check(self.L.sfcnl_cu_sym_range_final(self.h, C.byref(pp), nr, *ptrs, None, None))
            return None
        outs = [np.empty(n) for _ in range(nout)]
        cnt = np.empty(n, np.uint32)
        arr = (C.c_void_p * 4)(*([o.ctypes.data for o in outs] + [None] * (4 - nout)))
        self.check(self.L.sfcnl_cu_sym_range_final(self.h, C.byref(pp), nr, *ptrs, arr, _ptr(cnt)))
        return ReduceResult(list(kernel.names), outs, cnt)

    def cluster_slots(self):
        """Pair slots of the current gather store (cluster_overhead numerator)."""
        v = C.c_uint64()
        self.check(self.L.sfcnl_cu_cluster_slots(self.h, C.byref(v)))
        return v.value

    # domain decomposition (include/sfcnl_cu.h section (6)) ----------------
    def set_particles_device(self, n, cols, names, box: SimulationBox):
        """Orig slot from device arrays: cols = [x, y, z, h, *fields] (torch CUDA tensors)."""
        b = box.c()
        ptr = [int(c.data_ptr()) for c in cols]
        self.check(self.L.sfcnl_cu_set_particles(self.h, int(n), *ptr[:4], C.byref(b)))
        for name, p in zip(names, ptr[4:]):
            self.check(self.L.sfcnl_cu_set_field(self.h, name.encode(), p))

    def set_particle_records(self, n, rec, names, box: SimulationBox):
        """Orig slot from a device row-major [n, 4 + len(names)] float64 tensor."""
        b = box.c()
        arr = (C.c_char_p * max(len(names), 1))(*[f.encode() for f in names])
        self.check(self.L.sfcnl_cu_set_particle_records(self.h, int(n), int(rec.data_ptr()), int(rec.shape[1]), arr,
                                                        C.byref(b)))

    def alloc_sorted(self, n, box: SimulationBox, fields):
        b = box.c()
        arr = (C.c_char_p * max(len(fields), 1))(*[f.encode() for f in fields])
        self.check(self.L.sfcnl_cu_alloc_sorted(self.h, int(n), C.byref(b), arr, len(fields)))

    def apply_order_into(self, offset):
        self.check(self.L.sfcnl_cu_apply_order_into(self.h, int(offset)))

    def set_keys_device(self, keys_tensor, bits=kDefaultSfcBits):
        self.check(self.L.sfcnl_cu_set_keys(self.h, int(keys_tensor.numel()), int(keys_tensor.data_ptr()), 1,
                                            int(bits)))

    def node_geometry_range(self, p0, p1):
        self.check(self.L.sfcnl_cu_node_geometry_range(self.h, int(p0), int(p1)))

    def halo_mark(self, bp: BuildParams, sc0, sc1):
        p = bp.c()
        nj = C.c_uint64()
        self.check(self.L.sfcnl_cu_halo_mark(self.h, C.byref(p), int(sc0), int(sc1), C.byref(nj)))
        return nj.value

    def build_store_range(self, bp: BuildParams, sc0, sc1, max_h=0.0):
        nsc, nb = C.c_uint64(), C.c_uint64()
        p = bp.c()
        self.check(self.L.sfcnl_cu_build_store_range(self.h, C.byref(p), int(sc0), int(sc1), float(max_h),
                                                     C.byref(nsc), C.byref(nb)))
        return nsc.value, nb.value

    def device_array(self, name, dtype, count=None):
        """Zero-copy torch view of an internal device array (see sfcnl_cu_device_array)."""
        import torch  # plumbing only: views for collectives
        ptr, nbytes = C.c_void_p(), C.c_uint64()
        self.check(self.L.sfcnl_cu_device_array(self.h, name.encode(), C.byref(ptr), C.byref(nbytes)))
        item = torch.empty((), dtype=dtype).element_size()
        n = nbytes.value // item if count is None else int(count)
        if n * item > nbytes.value:
            raise InputError(f"device_array {name}: {n} elements exceed {nbytes.value} bytes")
        typestr = {torch.float64: "<f8", torch.int64: "<i8", torch.uint8: "|u1", torch.int32: "<i4",
                   torch.uint32: "<u4", torch.float32: "<f4"}[dtype]

        class _View:
            __cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr.value or 0, False),
                                        "version": 3, "strides": None}

        return torch.as_tensor(_View(), device=f"cuda:{self.device}")

    def stream(self):
        return self.L.sfcnl_cu_stream(self.h)

    def synchronize(self):
        self.check(self.L.sfcnl_cu_synchronize(self.h))

    def launch_count(self):
        return int(self.L.sfcnl_cu_launch_count(self.h))

    def set_timing(self, on=True):
        self.L.sfcnl_cu_set_timing(self.h, int(bool(on)))

    STAGES = ("keygen", "sort", "permute", "octree", "node_geometry", "cluster_geometry", "build",
              "encode", "pass")

    def stage_times(self):
        ms = (C.c_double * 16)()
        k = self.L.sfcnl_cu_stage_times(self.h, ms, 16)
        return {self.STAGES[i]: ms[i] for i in range(k)}


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context()
    return _default_ctx


# ----------------------------------------------------------------- reference API
def sort_by_sfc(ps: ParticleSet, box: SimulationBox, bits: int = kDefaultSfcBits, ctx=None) -> SfcOrder:
    """hilbert.cpp:8-26 on the GPU (K1 keygen + K2 onesweep radix sort)."""
    if bits < 1 or bits > 21:
        raise InputError("bits per dimension must be in [1, 21]")
    ctx = ctx or default_context()
    ctx.set_particles(ParticleSet(ps.x, ps.y, ps.z, ps.h), box)
    ctx.sort(bits)
    keys, perm = ctx.get_order(ps.size())
    return SfcOrder(keys, perm, bits)


def apply_sfc_order(ps: ParticleSet, order: SfcOrder, ctx=None) -> ParticleSet:
    """hilbert.cpp:28-44 on the GPU (K3 gather)."""
    n = ps.size()
    if len(order.perm) != n:
        raise InputError("apply_sfc_order: permutation size mismatch")
    ctx = ctx or default_context()
    ctx.set_particles(ps, SimulationBox((0, 0, 0), (1, 1, 1)))
    ctx.set_order(order)
    ctx.apply_order()
    out = ParticleSet(ctx.get_sorted("x", n), ctx.get_sorted("y", n), ctx.get_sorted("z", n),
                      ctx.get_sorted("h", n))
    for name in ps.fields:
        out.fields[name] = ctx.get_sorted(name, n)
    return out


def build_octree(order: SfcOrder, bucket_size: int = 64, ctx=None) -> Octree:
    """octree.cpp:43-59 on the GPU, identical node array."""
    if bucket_size < 1:
        raise InputError("build_octree: bucket_size must be >= 1")
    ctx = ctx or default_context()
    ctx.set_order(SfcOrder(order.keys, np.zeros(0, np.uint32) if False else order.perm, order.bits))
    nn = ctx.octree(bucket_size)
    return Octree(ctx.get_octree(nn), order.bits, order.size())


def _tree_arrays(ps, tree, ctx):
    ctx.set_particles(ps, SimulationBox((-1e300,) * 3, (1e300,) * 3), sorted_slot=True)
    ctx.set_octree(tree)
    return ctx.node_geometry(len(tree.nodes))


def compute_node_aabbs(tree: Octree, ps: ParticleSet, ctx=None):
    """octree.cpp:68-81: (lo[nodes,3], hi[nodes,3]); empty nodes are (+inf, -inf)."""
    lo, hi, _ = _tree_arrays(ps, tree, ctx or default_context())
    return lo, hi


def compute_node_max_radius(tree: Octree, ps: ParticleSet, ctx=None):
    """octree.cpp:83-96."""
    return _tree_arrays(ps, tree, ctx or default_context())[2]


def build_neighbor_store(ps: ParticleSet, box: SimulationBox, tree: Octree, bp: BuildParams,
                         threads: int = 1, ctx=None) -> NeighborStore:
    """neighbor_build.cpp:74-184 on the GPU; byte-identical NeighborStore."""
    ctx = ctx or default_context()
    ctx.set_particles(ps, box, sorted_slot=True)
    if tree.n != ps.size():
        raise BuildError("build_neighbor_store: octree/particle-set mismatch")
    ctx.set_octree(tree)
    nsc, nb = ctx.build_store(bp)
    return ctx.get_store(bp, ps.size(), nsc, nb)


def reduce(ps: ParticleSet, box: SimulationBox, store: NeighborStore, kernel: Kernel,
           cfg: PassConfig = None, ctx=None) -> ReduceResult:
    """reduce.hpp:38-231 on the GPU for the built-in kernels."""
    cfg = cfg or PassConfig()
    ctx = ctx or default_context()
    if store.n != ps.size():
        raise InputError("reduce: store/particle-set size mismatch")
    ctx.set_particles(ps, box, sorted_slot=True)
    ctx.set_store(store)
    return ctx.reduce(kernel, cfg, ps.size())


def build_full_list(ps: ParticleSet, box: SimulationBox, build_scale: float, mode: int = GATHER,
                    ctx=None) -> FullVerletList:
    """build_full_list (baselines.hpp:42-44, baselines.cpp:39-131) on the GPU.

    The list is derived from a compressed gather store built at `build_scale` over the
    SFC-sorted copy of `ps` (K1-K4 of the hot path + pass_full.cuh). When `ps` is not
    in SFC order, the sorted-index list is mapped back to `ps`'s numbering on the host
    (rows by the permutation, each row re-sorted ascending). Gather mode only: a
    symmetric full list (d <= scale max(h_i, h_j)) is not derivable from a gather
    store at the same scale."""
    if mode != GATHER:
        raise InputError("build_full_list: only gather lists are built on the GPU")
    if not (build_scale >= 0):
        raise InputError("build_full_list: build_scale must be >= 0")
    ctx = ctx or default_context()
    n = ps.size()
    ctx.set_particles(ParticleSet(ps.x, ps.y, ps.z, ps.h), box)
    ctx.sort()
    ctx.apply_order()
    ctx.octree(64)
    ctx.build_store(BuildParams(ClusterParams(8, 8, 32), GATHER, True, float(build_scale)))
    pairs = ctx.build_full_list(build_scale)
    fl = ctx.get_full_list(n, pairs, build_scale)
    _, perm = ctx.get_order(n)
    if n and not np.array_equal(perm, np.arange(n, dtype=np.uint32)):
        cnt = np.diff(fl.offsets).astype(np.int64)
        rows = np.repeat(perm.astype(np.int64), cnt)
        cols = perm[fl.neighbors.astype(np.int64)].astype(np.int64)
        o = np.lexsort((cols, rows))
        per_row = np.bincount(rows, minlength=n)
        offsets = np.zeros(n + 1, np.uint64)
        np.cumsum(per_row, out=offsets[1:])
        fl = FullVerletList(GATHER, float(build_scale), offsets, cols[o].astype(np.uint32))
    return fl


def reduce_full(ps: ParticleSet, box: SimulationBox, fl: FullVerletList, kernel: Kernel,
                cfg: PassConfig = None, ctx=None) -> ReduceResult:
    """reduce_full<Real,K> (baselines.hpp:47-129) on the GPU: precision F64 is
    bit-equal to reduce_full<double>."""
    cfg = cfg or PassConfig()
    ctx = ctx or default_context()
    if len(fl.offsets) != ps.size() + 1:
        raise InputError("reduce_full: list/particle-set mismatch")
    if cfg.query_scale > fl.build_scale:
        raise InputError("reduce_full: query_scale exceeds the list's build scale")
    ctx.set_particles(ps, box, sorted_slot=True)
    ctx.set_full_list(fl)
    return ctx.reduce_full(kernel, cfg, ps.size())


def cluster_overhead(store: NeighborStore, true_directed_pairs: int, ctx=None) -> float:
    """bench::cluster_overhead (bench.cpp:93-122): evaluated pair slots / true directed
    pairs; the slot count is a device pass over the store (k_cluster_slots)."""
    if store.build.mode != GATHER:
        raise InputError("cluster_overhead: requires a gather-mode store")
    if true_directed_pairs == 0:
        raise InputError("cluster_overhead: no in-range pairs")
    ctx = ctx or default_context()
    ctx.set_store(store)
    return ctx.cluster_slots() / float(true_directed_pairs)


# ----------------------------------------------------------------- store helpers (host)
def entry_mask(records: np.ndarray, entry: int, mask_bytes: int) -> int:
    """neighbor_store.cpp:10-16."""
    v = 0
    for b in range(mask_bytes):
        v |= int(records[entry * mask_bytes + b]) << (8 * b)
    return v


def decode_entry_indices(store: NeighborStore, sc: int):
    """neighbor_store.cpp:18-42: (indices, mask records) of one super-cluster."""
    if sc >= store.num_superclusters():
        raise InputError("decode_entry_indices: super-cluster out of range")
    count = int(store.counts[sc])
    begin, end = int(store.offsets[sc]), int(store.offsets[sc + 1])
    mb = count * store.build.params.mask_bytes_per_entry()
    if begin + mb > end:
        raise DecodeError("blob slice too short for bitmasks", begin)
    rec = store.blob[begin:begin + mb]
    data = store.blob[begin + mb:end]
    if store.build.compress:
        idx, used = decode_into(data, count, store.build.params.w)
        if used != len(data):
            raise DecodeError("trailing bytes in index blob", used)
    else:
        if len(data) != 4 * count:
            raise DecodeError("raw index blob length mismatch", len(data))
        idx = np.frombuffer(data.tobytes(), "<u4").copy()
    return idx, rec


def neighbor_clusters(store: NeighborStore, sc: int):
    """neighbor_store.cpp:44-54: [(jcluster, mask)]."""
    idx, rec = decode_entry_indices(store, sc)
    mb = store.build.params.mask_bytes_per_entry()
    return [(int(j), entry_mask(rec, e, mb)) for e, j in enumerate(idx)]


# ----------------------------------------------------------------- codec (host)
def delta_encode(indices: Sequence[int]):
    """nibble_codec.cpp:56-70."""
    out = []
    prev = 0
    for k, cur in enumerate(indices):
        cur = int(cur)
        if k == 0:
            out.append(cur + 1)
        else:
            if cur <= prev:
                raise InputError("delta_encode: input not strictly increasing")
            out.append(cur - prev)
        prev = cur
    return out


def encoded_size_bits(v: int) -> int:
    """nibble_codec.cpp:188-194."""
    if v == 0:
        raise InputError("encoded_size_bits: zero difference")
    if v > 0xFFFFFFFF:
        raise InputError("encoded_size_bits: difference exceeds 2^32 - 1")
    if v == 1:
        return 1
    if v <= 9:
        return 5
    return 5 + 4 * ((v.bit_length() + 3) // 4)


def encode(indices, w=32) -> np.ndarray:
    """codec::encode (nibble_codec.cpp:117-134) -> bytes."""
    idx = np.ascontiguousarray(indices, np.uint32)
    cap = 64 + 8 * len(idx) * 2
    out = np.empty(cap, np.uint8)
    ln = C.c_uint64()
    N.host_check(N.lib().sfcnl_codec_encode(_ptr(idx), len(idx), int(w), _ptr(out), cap, C.byref(ln)))
    return out[: ln.value].copy()


def decode_into(data, count, w=32):
    """codec::decode_into (nibble_codec.cpp:136-178) -> (indices, bytes consumed)."""
    data = np.ascontiguousarray(data, np.uint8)
    buf = data if data.size else np.zeros(1, np.uint8)
    out = np.empty(max(int(count), 1), np.uint32)
    used = C.c_uint64()
    N.host_check(N.lib().sfcnl_codec_decode_into(_ptr(buf), len(data), int(count), int(w), _ptr(out),
                                                 C.byref(used)))
    return out[:count], used.value


def decode(data, count, w=32):
    """codec::decode (nibble_codec.cpp:180-186)."""
    idx, used = decode_into(data, count, w)
    if used != len(data):
        raise DecodeError("trailing bytes after encoded list", used)
    return idx


def hilbert_encode(ix, iy, iz, bits):
    k = C.c_uint64()
    N.host_check(N.lib().sfcnl_hilbert_encode(int(ix), int(iy), int(iz), int(bits), C.byref(k)))
    return k.value


def hilbert_decode(key, bits):
    out = (C.c_uint32 * 3)()
    N.host_check(N.lib().sfcnl_hilbert_decode(int(key), int(bits), out))
    return tuple(out)


# ----------------------------------------------------------------- generators (host)
@dataclass
class UniformSpec:
    """generators.hpp:14-21."""
    n: int = 1000
    density: float = 100.0
    target_neighbors: float = 50.0
    periodic: Tuple[bool, bool, bool] = (True, True, True)
    h_jitter: float = 0.0
    seed: int = 42


@dataclass
class EvrardSpec:
    """generators.hpp:26-32."""
    n: int = 1000
    target_neighbors: float = 50.0
    constant_h: bool = False
    periodic: Tuple[bool, bool, bool] = (False, False, False)
    seed: int = 42


def _gen_arrays(n):
    return [np.empty(n) for _ in range(6)], np.empty(6)


def make_uniform(spec: UniformSpec):
    """generators.cpp:21-45 -> (ParticleSet, SimulationBox)."""
    a, box6 = _gen_arrays(spec.n)
    per = (C.c_int32 * 3)(*[int(p) for p in spec.periodic])
    N.host_check(N.lib().sfcnl_make_uniform(spec.n, spec.density, spec.target_neighbors, per, spec.h_jitter,
                                            spec.seed, *[_ptr(v) for v in a], _ptr(box6)))
    ps = ParticleSet(a[0], a[1], a[2], a[3], {"m": a[4], "q": a[5]})
    return ps, SimulationBox(tuple(box6[:3]), tuple(box6[3:]), spec.periodic)


def make_evrard(spec: EvrardSpec):
    """generators.cpp:47-82 -> (ParticleSet, SimulationBox)."""
    a, box6 = _gen_arrays(spec.n)
    per = (C.c_int32 * 3)(*[int(p) for p in spec.periodic])
    N.host_check(N.lib().sfcnl_make_evrard(spec.n, spec.target_neighbors, int(spec.constant_h), per, spec.seed,
                                           *[_ptr(v) for v in a], _ptr(box6)))
    ps = ParticleSet(a[0], a[1], a[2], a[3], {"m": a[4], "q": a[5]})
    return ps, SimulationBox(tuple(box6[:3]), tuple(box6[3:]), spec.periodic)


def uniform_h_for_target(target, rho):
    """generators.cpp:14-19."""
    if not (target > 0) or not (rho > 0):
        raise InputError("uniform_h_for_target: positive inputs required")
    return math.pow(3.0 * target / (4.0 * math.pi * rho), 1.0 / 3.0)
