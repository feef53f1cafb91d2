"""TEST INFRASTRUCTURE ONLY — numpy front-end for the two CPU checkers.

* ``Oracle("port")``      — the plain-C restatement ``oracle/liboracle.so``
  (``sfcnl_oracle.c``; each function cites the reference file:line it follows).
* ``Oracle("reference")`` — the UNMODIFIED reference library compiled from
  ``/root/reference/proj/src`` into ``oracle/_ref/libsfcnl_ref.so`` (``ref_shim.cpp``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module, and only as the checker. The
product (``paper_2602_19873_b200``) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libsfcnl_ref.so")

KERNELS = {"count": 0, "density": 1, "lj": 2, "lj_coulomb": 3}


class OracleError(RuntimeError):
    def __init__(self, code, msg, offset):
        super().__init__(f"[{code}] {msg}")
        self.code, self.msg, self.offset = code, msg, offset


def _p(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype)) if a is not None else None


D, U8, U32, U64, I32 = C.c_double, C.c_uint8, C.c_uint32, C.c_uint64, C.c_int32


@dataclass
class Particles:
    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    h: np.ndarray
    m: np.ndarray
    q: np.ndarray
    box6: np.ndarray
    periodic: tuple

    @property
    def n(self):
        return len(self.x)

    def permuted(self, perm):
        return Particles(self.x[perm], self.y[perm], self.z[perm], self.h[perm],
                         self.m[perm], self.q[perm], self.box6.copy(), self.periodic)


@dataclass
class Tree:
    key_first: np.ndarray
    key_last: np.ndarray
    pbegin: np.ndarray
    pend: np.ndarray
    first_child: np.ndarray
    depth: np.ndarray
    bits: int


@dataclass
class Store:
    n: int
    ci: int
    cj: int
    w: int
    mode: int
    compress: int
    scale: float
    counts: np.ndarray
    offsets: np.ndarray
    blob: np.ndarray


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_LIB if kind == "port" else REF_LIB
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run `make -C oracle`)")
        self.lib = C.CDLL(path)
        self.p = "orc_" if kind == "port" else "ref_"
        getattr(self.lib, self.p + "last_error").restype = C.c_char_p
        for name in ("octree_size",):
            getattr(self.lib, self.p + name).restype = C.c_uint64

    def _f(self, name):
        return getattr(self.lib, self.p + name)

    def _check(self, rc):
        if rc:
            off = C.c_uint64(0)
            msg = self._f("last_error")(C.byref(off))
            raise OracleError(rc, msg.decode(), off.value)

    # ---- generators
    def make_uniform(self, n, density, target, periodic=(1, 1, 1), h_jitter=0.0, seed=42):
        a = [np.empty(n) for _ in range(6)]
        box6 = np.empty(6)
        per = (C.c_int * 3)(*periodic)
        self._check(self._f("make_uniform")(U64(n), D(density), D(target), per, D(h_jitter),
                                            U64(seed), *[_p(v, D) for v in a], _p(box6, D)))
        return Particles(*a, box6, tuple(periodic))

    def make_evrard(self, n, target, constant_h=False, periodic=(0, 0, 0), seed=42):
        a = [np.empty(n) for _ in range(6)]
        box6 = np.empty(6)
        per = (C.c_int * 3)(*periodic)
        self._check(self._f("make_evrard")(U64(n), D(target), C.c_int(int(constant_h)), per,
                                           U64(seed), *[_p(v, D) for v in a], _p(box6, D)))
        return Particles(*a, box6, tuple(periodic))

    # ---- SFC
    def hilbert_encode(self, ix, iy, iz, bits):
        k = C.c_uint64()
        self._check(self._f("hilbert_encode")(U32(ix), U32(iy), U32(iz), C.c_int(bits), C.byref(k)))
        return k.value

    def hilbert_decode(self, key, bits):
        out = (C.c_uint32 * 3)()
        self._check(self._f("hilbert_decode")(U64(key), C.c_int(bits), out))
        return tuple(out)

    def sort_by_sfc(self, ps: Particles, bits=21):
        n = ps.n
        keys = np.empty(n, np.uint64)
        perm = np.empty(n, np.uint32)
        per = (C.c_int * 3)(*ps.periodic)
        if self.kind == "port":
            rc = self._f("sort_by_sfc")(U64(n), _p(ps.x, D), _p(ps.y, D), _p(ps.z, D),
                                        _p(ps.box6, D), per, C.c_int(bits), _p(keys, U64), _p(perm, U32))
        else:
            rc = self._f("sort_by_sfc")(U64(n), _p(ps.x, D), _p(ps.y, D), _p(ps.z, D), _p(ps.h, D),
                                        _p(ps.box6, D), per, C.c_int(bits), _p(keys, U64), _p(perm, U32))
        self._check(rc)
        return keys, perm

    # ---- octree
    def build_octree(self, keys, bits=21, bucket=64):
        keys = np.ascontiguousarray(keys, np.uint64)
        h = C.c_void_p()
        self._check(self._f("build_octree")(U64(len(keys)), _p(keys, U64), C.c_int(bits),
                                            U32(bucket), C.byref(h)))
        try:
            nn = self._f("octree_size")(h)
            t = Tree(np.empty(nn, np.uint64), np.empty(nn, np.uint64), np.empty(nn, np.uint32),
                     np.empty(nn, np.uint32), np.empty(nn, np.int32), np.empty(nn, np.uint8), bits)
            self._f("octree_nodes")(h, _p(t.key_first, U64), _p(t.key_last, U64), _p(t.pbegin, U32),
                                    _p(t.pend, U32), _p(t.first_child, I32), _p(t.depth, U8))
            return t, h
        except Exception:
            self._f("octree_free")(h)
            raise

    def tree(self, keys, bits=21, bucket=64):
        t, h = self.build_octree(keys, bits, bucket)
        self._f("octree_free")(h)
        return t

    def node_geometry(self, keys, ps: Particles, bits=21, bucket=64):
        t, h = self.build_octree(keys, bits, bucket)
        try:
            nn = len(t.pend)
            lo = np.empty((nn, 3))
            hi = np.empty((nn, 3))
            rad = np.empty(nn)
            self._check(self._f("node_geometry")(h, *self._node_geom_args(ps), _p(lo, D), _p(hi, D), _p(rad, D)))
            return t, lo, hi, rad
        finally:
            self._f("octree_free")(h)

    def _node_geom_args(self, ps):
        if self.kind == "port":
            return (_p(ps.x, D), _p(ps.y, D), _p(ps.z, D), _p(ps.h, D))
        return (U64(ps.n), _p(ps.x, D), _p(ps.y, D), _p(ps.z, D), _p(ps.h, D))

    # ---- store
    def build_store(self, ps: Particles, tree: Tree, ci=8, cj=8, w=32, mode=0, compress=1,
                    scale=1.0, threads=1, write_path=None) -> Store:
        per = (C.c_int * 3)(*ps.periodic)
        h = C.c_void_p()
        common = (U64(ps.n), _p(ps.x, D), _p(ps.y, D), _p(ps.z, D), _p(ps.h, D), _p(ps.box6, D), per,
                  C.c_int(tree.bits), U64(len(tree.pend)), _p(tree.key_first, U64), _p(tree.key_last, U64),
                  _p(tree.pbegin, U32), _p(tree.pend, U32), _p(tree.first_child, I32))
        if self.kind == "port":
            rc = self._f("build_store")(*common, U32(ci), U32(cj), C.c_int(w), C.c_int(mode),
                                        C.c_int(compress), D(scale), C.byref(h))
        else:
            rc = self._f("build_store_nodes")(*common, _p(tree.depth, U8), U32(ci), U32(cj), C.c_int(w),
                                              C.c_int(mode), C.c_int(compress), D(scale),
                                              C.c_int(threads), C.byref(h))
        self._check(rc)
        try:
            nsc, nb = C.c_uint64(), C.c_uint64()
            self._f("store_info")(h, C.byref(nsc), C.byref(nb))
            counts = np.empty(nsc.value, np.uint32)
            offsets = np.empty(nsc.value + 1, np.uint64)
            blob = np.empty(max(nb.value, 1), np.uint8)
            self._f("store_copy")(h, _p(counts, U32), _p(offsets, U64), _p(blob, U8))
            if write_path is not None:  # the reference's own SFNLSTOR writer (reference kind only)
                self._check(self._f("store_write")(h, write_path.encode()))
            return Store(ps.n, ci, cj, w, mode, compress, scale, counts, offsets, blob[: nb.value])
        finally:
            self._f("store_free")(h)

    # ---- pass
    def reduce(self, kernel, ps: Particles, store: Store, query_scale=1.0, eps=1.0, sigma=1.0,
               ck=0.0, real="double", isa=0, threads=1):
        kid = KERNELS[kernel]
        nout = 4 if kid >= 2 else 1
        n = ps.n
        outs = [np.zeros(n) for _ in range(nout)]
        optr = (C.POINTER(C.c_double) * 4)(*[_p(o, D) for o in outs])
        cnt = np.zeros(n, np.uint32)
        per = (C.c_int * 3)(*ps.periodic)
        blob = store.blob if len(store.blob) else np.zeros(1, np.uint8)
        common_a = (C.c_int(kid),)
        common_b = (U64(n), _p(ps.x, D), _p(ps.y, D), _p(ps.z, D), _p(ps.h, D), _p(ps.m, D), _p(ps.q, D),
                    _p(ps.box6, D), per, U32(store.ci), U32(store.cj), C.c_int(store.w),
                    C.c_int(store.mode), C.c_int(store.compress), D(store.scale),
                    U64(len(store.counts)), _p(store.counts, U32), _p(store.offsets, U64),
                    _p(blob, U8), U64(len(store.blob)), D(query_scale))
        if self.kind == "port":
            rc = self._f("reduce")(*common_a, *common_b, D(eps), D(sigma), D(ck), optr, _p(cnt, U32))
        else:
            rc = self._f("reduce")(*common_a, C.c_int(1 if real == "float" else 0), *common_b,
                                   C.c_int(isa), C.c_int(threads), D(eps), D(sigma), D(ck), optr,
                                   _p(cnt, U32))
        self._check(rc)
        return outs, cnt

    # ---- domain-decomposition helpers (port only; SURVEY §8(e) parity checks)
    def _store_from(self, h, n, ci, cj, w, mode, compress, scale):
        try:
            nsc, nb = C.c_uint64(), C.c_uint64()
            self._f("store_info")(h, C.byref(nsc), C.byref(nb))
            counts = np.empty(nsc.value, np.uint32)
            offsets = np.empty(nsc.value + 1, np.uint64)
            blob = np.empty(max(nb.value, 1), np.uint8)
            self._f("store_copy")(h, _p(counts, U32), _p(offsets, U64), _p(blob, U8))
            return Store(n, ci, cj, w, mode, compress, scale, counts, offsets, blob[: nb.value])
        finally:
            self._f("store_free")(h)

    def node_geometry_range(self, tree: Tree, ps: Particles, p0, p1):
        """Partial node geometry from particles [p0, p1): (lo (nn,3), hi (nn,3), maxh (nn,))."""
        assert self.kind == "port"
        nn = len(tree.pend)
        lo, hi, mh = np.empty((nn, 3)), np.empty((nn, 3)), np.empty(nn)
        self._check(self._f("node_geometry_range")(
            U64(nn), _p(tree.pbegin, U32), _p(tree.pend, U32), _p(tree.first_child, I32), _p(ps.x, D),
            _p(ps.y, D), _p(ps.z, D), _p(ps.h, D), U64(p0), U64(p1), _p(lo, D), _p(hi, D), _p(mh, D)))
        return lo, hi, mh

    def _range_common(self, ps, tree, geo):
        lo, hi, mh = (np.ascontiguousarray(a, np.float64) for a in geo)
        per = (C.c_int * 3)(*ps.periodic)
        return (U64(ps.n), _p(ps.x, D), _p(ps.y, D), _p(ps.z, D), _p(ps.h, D), _p(ps.box6, D), per,
                U64(len(tree.pend)), _p(tree.pbegin, U32), _p(tree.pend, U32), _p(tree.first_child, I32),
                _p(lo, D), _p(hi, D), _p(mh, D)), (lo, hi, mh)

    def halo_mark(self, ps: Particles, tree: Tree, geo, sc0, sc1, max_h, ci=8, cj=8, mode=0, scale=1.0):
        assert self.kind == "port"
        flags = np.zeros(max((ps.n + cj - 1) // cj, 1), np.uint8)
        common, keep = self._range_common(ps, tree, geo)
        self._check(self._f("halo_mark")(*common, U32(ci), U32(cj), C.c_int(mode), D(scale), U64(sc0),
                                         U64(sc1), D(max_h), _p(flags, U8)))
        return flags[: (ps.n + cj - 1) // cj]

    def build_store_range(self, ps: Particles, tree: Tree, geo, sc0, sc1, max_h, ci=8, cj=8, w=32, mode=0,
                          compress=1, scale=1.0) -> Store:
        assert self.kind == "port"
        h = C.c_void_p()
        common, keep = self._range_common(ps, tree, geo)
        self._check(self._f("build_store_range")(*common, U32(ci), U32(cj), C.c_int(w), C.c_int(mode),
                                                 C.c_int(compress), D(scale), U64(sc0), U64(sc1), D(max_h),
                                                 C.byref(h)))
        return self._store_from(h, ps.n, ci, cj, w, mode, compress, scale)

    def reduce_range(self, kernel, ps: Particles, store: Store, sc_base, query_scale=1.0, eps=1.0, sigma=1.0,
                     ck=0.0):
        """Gather-mode pass over a range store; outputs for particles [64*sc_base, ...)."""
        assert self.kind == "port"
        kid = KERNELS[kernel]
        nout = 4 if kid >= 2 else 1
        nsc = len(store.counts)
        nloc = max(0, min(ps.n, 64 * (sc_base + nsc)) - 64 * sc_base)
        outs = [np.zeros(max(nloc, 1)) for _ in range(nout)]
        optr = (C.POINTER(C.c_double) * 4)(*[_p(o, D) for o in outs])
        cnt = np.zeros(max(nloc, 1), np.uint32)
        per = (C.c_int * 3)(*ps.periodic)
        blob = store.blob if len(store.blob) else np.zeros(1, np.uint8)
        self._check(self._f("reduce_range")(
            C.c_int(kid), U64(ps.n), _p(ps.x, D), _p(ps.y, D), _p(ps.z, D), _p(ps.h, D), _p(ps.m, D),
            _p(ps.q, D), _p(ps.box6, D), per, U32(store.ci), U32(store.cj), C.c_int(store.w),
            C.c_int(store.compress), D(store.scale), U64(sc_base), U64(nsc), _p(store.counts, U32),
            _p(store.offsets, U64), _p(blob, U8), D(query_scale), D(eps), D(sigma), D(ck), optr, _p(cnt, U32)))
        return [o[:nloc] for o in outs], cnt[:nloc]

    # ---- reference-only checkers for the full-size parity tests
    def cluster_geometry(self, ps: Particles, width):
        """compute_cluster_geometry (neighbor_build.cpp:19-38) via cluster_aabb /
        cluster_max_radius (cluster.hpp:77-90): (lo (ncl,3), hi (ncl,3), maxh (ncl,))."""
        assert self.kind == "reference"
        ncl = (ps.n + width - 1) // width
        lo, hi, mh = np.empty((max(ncl, 1), 3)), np.empty((max(ncl, 1), 3)), np.empty(max(ncl, 1))
        self._check(self._f("cluster_geometry")(U64(ps.n), _p(ps.x, D), _p(ps.y, D), _p(ps.z, D), _p(ps.h, D),
                                                U32(width), _p(lo, D), _p(hi, D), _p(mh, D)))
        return lo[:ncl], hi[:ncl], mh[:ncl]

    def lj_abs_sums(self, ps: Particles, store: Store, query_scale=1.0, eps=1.0, sigma=1.0, threads=1):
        """sum_j |F_ij| and sum_j |E_ij| per particle through the reference's reduce<double>
        with a make_pair_kernel user kernel (the LJ normwise tolerance denominators)."""
        assert self.kind == "reference"
        n = ps.n
        absf, abse = np.zeros(n), np.zeros(n)
        per = (C.c_int * 3)(*ps.periodic)
        blob = store.blob if len(store.blob) else np.zeros(1, np.uint8)
        self._check(self._f("lj_abs_sums")(
            U64(n), _p(ps.x, D), _p(ps.y, D), _p(ps.z, D), _p(ps.h, D), _p(ps.box6, D), per, U32(store.ci),
            U32(store.cj), C.c_int(store.w), C.c_int(store.mode), C.c_int(store.compress), D(store.scale),
            U64(len(store.counts)), _p(store.counts, U32), _p(store.offsets, U64), _p(blob, U8),
            U64(len(store.blob)), D(query_scale), C.c_int(threads), D(eps), D(sigma), _p(absf, D), _p(abse, D)))
        return absf, abse

    # ---- full Verlet list baseline (reference only: baselines.hpp:39-131)
    def full_list(self, ps: Particles, build_scale=1.0, kernels=(), query_scale=1.0, eps=1.0, sigma=1.0, mode=0):
        """build_full_list (cell grid, baselines.cpp:39-131) -> (offsets u64[n+1],
        neighbors u32[]), plus reduce_full<double> (baselines.hpp:47-129) outputs for
        each kernel name in `kernels`. mode 0 gather, 1 symmetric."""
        assert self.kind == "reference"
        per = (C.c_int * 3)(*ps.periodic)
        h, npairs = C.c_void_p(), C.c_uint64()
        self._check(self._f("full_list")(U64(ps.n), _p(ps.x, D), _p(ps.y, D), _p(ps.z, D), _p(ps.h, D),
                                         _p(ps.box6, D), per, D(build_scale), C.c_int(mode), C.c_int(2),
                                         C.byref(h), C.byref(npairs)))
        try:
            offsets = np.empty(ps.n + 1, np.uint64)
            nbrs = np.empty(max(npairs.value, 1), np.uint32)
            self._f("full_copy")(h, _p(offsets, U64), _p(nbrs, U32))
            res = {}
            for kern in kernels:
                kid = KERNELS[kern]
                nout = 4 if kid >= 2 else 1
                outs = [np.zeros(ps.n) for _ in range(nout)]
                optr = (C.POINTER(C.c_double) * 4)(*[_p(o, D) for o in outs])
                cnt = np.zeros(ps.n, np.uint32)
                self._check(self._f("reduce_full")(h, C.c_int(kid), U64(ps.n), _p(ps.x, D), _p(ps.y, D), _p(ps.z, D),
                                                   _p(ps.h, D), _p(ps.m, D), _p(ps.q, D), _p(ps.box6, D), per,
                                                   D(query_scale), D(eps), D(sigma), D(0.0), optr, _p(cnt, U32)))
                res[kern] = (outs, cnt)
            return offsets, nbrs[: npairs.value], res
        finally:
            self._f("full_free")(h)

    def cluster_overhead(self, st: Store, true_pairs):
        """bench::cluster_overhead (bench.cpp:93-122) of a gather store."""
        assert self.kind == "reference"
        out = D()
        blob = st.blob if len(st.blob) else np.zeros(1, np.uint8)
        self._check(self._f("cluster_overhead")(U64(st.n), U32(st.ci), U32(st.cj), C.c_int(st.w), C.c_int(st.compress),
                                                U64(len(st.counts)), _p(st.counts, U32), _p(st.offsets, U64),
                                                _p(blob, U8), U64(len(st.blob)), U64(int(true_pairs)), C.byref(out)))
        return out.value

    # ---- codec
    def encode(self, idx, w=32):
        idx = np.ascontiguousarray(idx, np.uint32)
        cap = 16 + 8 * len(idx) * 2
        out = np.empty(cap, np.uint8)
        ln = C.c_uint64()
        self._check(self._f("codec_encode")(_p(idx, U32), U64(len(idx)), C.c_int(w), _p(out, U8),
                                            U64(cap), C.byref(ln)))
        return out[: ln.value].copy()

    def decode(self, data, count, w=32):
        data = np.ascontiguousarray(data, np.uint8)
        buf = data if len(data) else np.zeros(1, np.uint8)
        out = np.empty(max(count, 1), np.uint32)
        used = C.c_uint64()
        self._check(self._f("codec_decode_into")(_p(buf, U8), U64(len(data)), U32(count), C.c_int(w),
                                                 _p(out, U32), C.byref(used)))
        return out[:count], used.value

    # ---- whole pipeline
    def pipeline(self, ps: Particles, sorted_ps=None, ci=8, cj=8, w=32, mode=0, compress=1,
                 scale=1.0, bits=21, bucket=64):
        keys, perm = self.sort_by_sfc(ps, bits)
        sp = ps.permuted(perm)
        tree = self.tree(keys, bits, bucket)
        store = self.build_store(sp, tree, ci, cj, w, mode, compress, scale)
        return keys, perm, sp, tree, store


def available(kind):
    return os.path.exists(PORT_LIB if kind == "port" else REF_LIB)
