import numpy as np
def run_stream_traced(self, steps, trace):
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

    def d2h(pairs, tag="d2h"):
        C.wait_stream(S)
        e0 = torch.cuda.Event(enable_timing=True); e0.record(C)
        with torch.cuda.stream(C):
            for src, host in pairs:
                torch.from_numpy(host.view(npdt[src.dtype])).copy_(src, non_blocking=True)
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(C)
        trace.append((tag, e0, ev))
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
            h0 = torch.cuda.Event(enable_timing=True); h0.record(C)
            with torch.cuda.stream(C):
                for name, h in zip(names, host_in):
                    c.device_array("orig." + name, torch.float64, n).copy_(h, non_blocking=True)
            ev_in = torch.cuda.Event(enable_timing=True)
            ev_in.record(C)
            trace.append(("h2d", h0, ev_in))
        self.num_nodes = c.octree(self.bucket)
        if ev_store is not None:
            S.wait_event(ev_store)  # the previous store has left the device
        self.num_sc, self.blob_bytes = c.build_store(self.bp)
        nsc, nb = self.num_sc, self.blob_bytes
        if len(out["store"][2]) < nb:
            out["store"][2] = self._alloc(nb, np.uint8)
        ev_store = d2h(tag="store_d2h", pairs=[(c.device_array("store.counts", torch.int32, nsc), out["store"][0][:nsc]),
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
                d2h(pairs, 'rho_d2h')
            else:
                ev_last = d2h(arrs, 'lj_d2h')
    C.synchronize()
    S.synchronize()

