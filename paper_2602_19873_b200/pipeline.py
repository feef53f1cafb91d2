"""Device-resident build-and-query step: the sequence the reference's bench runs
(bench.cpp:147-186) — sort_by_sfc -> apply_sfc_order -> build_octree ->
build_neighbor_store -> reduce — with every intermediate kept in HBM.

``Pipeline.run()`` launches only GPU work (inputs already resident);
``Pipeline.run_e2e()`` is the same step through the C-ABI with host buffers: it
uploads the particle arrays, runs, and downloads the results the reference API
would return (store + pass outputs).
"""
from __future__ import annotations

import numpy as np

from .api import (BuildParams, Context, Kernel, NeighborStore, ParticleSet, PassConfig,
                  SimulationBox, kDefaultSfcBits)


class Pipeline:
    def __init__(self, ctx: Context, ps: ParticleSet, box: SimulationBox, bp: BuildParams,
                 kernels, cfg: PassConfig, bits=kDefaultSfcBits, bucket=64):
        self.ctx, self.ps, self.box, self.bp = ctx, ps, box, bp
        self.kernels = list(kernels)
        self.cfg = cfg
        self.bits, self.bucket = bits, bucket
        self.n = ps.size()
        self.num_nodes = 0
        self.num_sc = 0
        self.blob_bytes = 0

    def upload(self):
        self.ctx.set_particles(self.ps, self.box)

    def run(self):
        """One full step on resident inputs; no host transfers of particle data."""
        c = self.ctx
        c.sort(self.bits)
        c.apply_order()
        self.num_nodes = c.octree(self.bucket)
        self.num_sc, self.blob_bytes = c.build_store(self.bp)
        for k in self.kernels:
            c.reduce(k, self.cfg, self.n, download=False)

    def host_buffers(self, alloc=np.empty):
        """Reusable host result buffers for run_e2e (pass e.g. a pinned allocator):
        store arrays sized for the worst case (w/8 + 10 bytes per possible entry is
        never reached; blob capacity grows on demand) and per-kernel outputs."""
        nsc = (self.n + 63) // 64
        self._out = {
            "store": [alloc(nsc, np.uint32), alloc(nsc + 1, np.uint64), alloc(max(16 * self.n // 4, 16), np.uint8)],
            "pass": [([alloc(self.n, np.float64) for _ in k.names], alloc(self.n, np.uint32)) for k in self.kernels],
        }
        self._alloc = alloc
        return self._out

    def run_e2e(self):
        """Upload -> step -> download (store + every kernel's outputs) into the host
        buffers of host_buffers() when set (fresh arrays otherwise)."""
        self.upload()
        c = self.ctx
        c.sort(self.bits)
        c.apply_order()
        self.num_nodes = c.octree(self.bucket)
        self.num_sc, self.blob_bytes = c.build_store(self.bp)
        out = getattr(self, "_out", None)
        if out is not None and len(out["store"][2]) < self.blob_bytes:
            out["store"][2] = self._alloc(self.blob_bytes, np.uint8)
        store = c.get_store(self.bp, self.n, self.num_sc, self.blob_bytes, into=out["store"] if out else None)
        results = [c.reduce(k, self.cfg, self.n, download=True, into=out["pass"][i] if out else None)
                   for i, k in enumerate(self.kernels)]
        return store, results

    def h2d_bytes(self):
        return 8 * self.n * (4 + len(self.ps.fields))

    def d2h_bytes(self):
        store = 4 * self.num_sc + 8 * (self.num_sc + 1) + self.blob_bytes
        outs = sum(len(k.names) * 8 * self.n + 4 * self.n for k in self.kernels)
        return store + outs
