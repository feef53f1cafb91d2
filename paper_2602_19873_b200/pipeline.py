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


class StreamedPipeline(Pipeline):
    """End-to-end steps with the host transfers overlapped with the device work of
    the neighbouring steps (a serving loop): every step still uploads its own
    inputs from pinned host memory and downloads its store and every pass's
    outputs to pinned host memory, but on a copy stream --

      * step k+1's inputs are uploaded into the input slot as soon as step k's
        apply_sfc_order has consumed it (the slot is not read again in step k);
      * the store and the last pass's outputs are downloaded straight from the
        context's arrays while the following stages run (the stage that would
        overwrite them waits for the download's event); the outputs of earlier
        passes are first copied device-to-device (a kernel, not a copy engine)
        into a side buffer, because the next pass reuses the arrays.

    The C-ABI calls stay synchronous on the context stream; only torch copies on a
    second stream and events are added (plumbing). The pinned host buffers of
    host_buffers() are reused by every step (a consumer reads them between steps)."""

    def run_stream(self, steps: int):
        import torch
        c = self.ctx
        dev = torch.device("cuda", c.device)
        S = torch.cuda.ExternalStream(c.stream(), device=dev)
        C = torch.cuda.Stream(device=dev)
        out = getattr(self, "_out", None)
        if out is None:
            raise RuntimeError("run_stream: call host_buffers(pinned allocator) first")
        npdt = {torch.int32: np.int32, torch.int64: np.int64, torch.uint8: np.uint8, torch.float64: np.float64}
        names = ["x", "y", "z", "h"] + list(self.ps.fields)
        host_in = [torch.from_numpy(getattr(self.ps, k) if k in "xyzh" else self.ps.fields[k]) for k in names]
        n, nk = self.n, len(self.kernels)
        if not hasattr(self, "_side"):
            self._side = {}
        side = self._side

        def d2h(pairs):
            C.wait_stream(S)
            with torch.cuda.stream(C):
                for src, host in pairs:
                    torch.from_numpy(host.view(npdt[src.dtype])).copy_(src, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(C)
            return ev

        ev_in = ev_store = ev_last = None
        for k in range(steps):
            if k == 0:
                self.upload()
            else:
                S.wait_event(ev_in)
            c.sort(self.bits)
            c.apply_order()
            if k + 1 < steps:  # next step's inputs into the (now free) input slot
                C.wait_stream(S)
                with torch.cuda.stream(C):
                    for name, h in zip(names, host_in):
                        c.device_array("orig." + name, torch.float64, n).copy_(h, non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(C)
            self.num_nodes = c.octree(self.bucket)
            if ev_store is not None:
                S.wait_event(ev_store)  # the previous store has left the device
            self.num_sc, self.blob_bytes = c.build_store(self.bp)
            nsc, nb = self.num_sc, self.blob_bytes
            if len(out["store"][2]) < nb:
                out["store"][2] = self._alloc(nb, np.uint8)
            ev_store = d2h([(c.device_array("store.counts", torch.int32, nsc), out["store"][0][:nsc]),
                            (c.device_array("store.offsets", torch.int64, nsc + 1), out["store"][1][:nsc + 1]),
                            (c.device_array("store.blob", torch.uint8, nb), out["store"][2][:nb])])
            for ki, kern in enumerate(self.kernels):
                if ki == 0 and ev_last is not None:
                    S.wait_event(ev_last)  # the previous step's last outputs have left the device
                c.reduce(kern, self.cfg, n, download=False)
                arrs = [(c.device_array(f"out{o}", torch.float64, n), out["pass"][ki][0][o][:n])
                        for o in range(len(kern.names))]
                arrs.append((c.device_array("count", torch.int32, n), out["pass"][ki][1][:n]))
                if ki + 1 < nk:  # the next pass reuses the arrays: kernel copy into a side buffer
                    pairs = []
                    with torch.cuda.stream(S):
                        for o, (src, host) in enumerate(arrs):
                            key = (ki, o)
                            buf = side.get(key)
                            if buf is None or buf.numel() != n or buf.dtype != src.dtype:
                                buf = side[key] = torch.empty(n, dtype=src.dtype, device=dev)
                            torch.add(src, 0, out=buf)
                            pairs.append((buf, host))
                    d2h(pairs)
                else:
                    ev_last = d2h(arrs)
        C.synchronize()
        S.synchronize()
