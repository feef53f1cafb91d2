# Host-side timeline of StreamedPipeline.run_stream: which calls block, and for how long
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2602_19873_b200 as S
import paper_2602_19873_b200.pipeline as PL
n = 1 << 26
ctx = S.Context(0)
ps0, box = S.make_uniform(S.UniformSpec(n=n, density=float(n), target_neighbors=200.0, seed=42))
pin = {}
for name, v in (("x", ps0.x), ("y", ps0.y), ("z", ps0.z), ("h", ps0.h), ("m", ps0.fields["m"])):
    t = torch.empty(n, dtype=torch.float64, pin_memory=True)
    t.numpy()[:] = v
    pin[name] = t
ps = S.ParticleSet(pin["x"].numpy(), pin["y"].numpy(), pin["z"].numpy(), pin["h"].numpy(), {"m": pin["m"].numpy()})
sigma = 0.5 * (1.0 / n) ** (1 / 3)
pipe = S.StreamedPipeline(ctx, ps, box, S.BuildParams(), [S.sph_density_kernel(), S.lj_kernel(1.0, sigma)],
                          S.PassConfig(1.0, S.MIXED))
TD = {np.dtype(np.float64): torch.float64, np.dtype(np.uint8): torch.uint8, np.dtype(np.uint32): torch.int32,
      np.dtype(np.uint64): torch.int64}
pipe.host_buffers(lambda k, dt: torch.empty(int(k), dtype=TD[np.dtype(dt)], pin_memory=True).numpy().view(dt))
pipe.upload(); pipe.run(); ctx.synchronize()
pipe.run_stream(2); ctx.synchronize()
# wrap the context's methods with host timers
log = []
for name in ("sort", "apply_order", "octree", "build_store", "reduce", "device_array"):
    f = getattr(ctx, name)
    def wrap(*a, _f=f, _n=name, **k):
        t0 = time.perf_counter(); r = _f(*a, **k); log.append((_n, (time.perf_counter() - t0) * 1e3)); return r
    setattr(ctx, name, wrap)
t0 = time.perf_counter(); pipe.run_stream(4); ctx.synchronize(); T = (time.perf_counter() - t0) * 1e3 / 4
agg = {}
for nme, ms in log:
    a = agg.setdefault(nme, [0, 0.0, 0.0]); a[0] += 1; a[1] += ms; a[2] = max(a[2], ms)
print("ms/step", round(T, 1))
for nme, (c, tot, mx) in agg.items():
    print(f"{nme:14s} calls/step {c / 4:5.1f}  ms/step {tot / 4:8.2f}  max {mx:7.2f}")
# device-side copy timeline (events on the copy stream)
sys.path.insert(0, 'scripts')
from _rs_traced import run_stream_traced
trace = []
torch.cuda.synchronize()
base = torch.cuda.Event(enable_timing=True); base.record()
run_stream_traced(pipe, 3, trace)
torch.cuda.synchronize()
for tag, a, b in trace:
    print(f"{tag:10s} start {base.elapsed_time(a):8.1f}  dur {a.elapsed_time(b):7.1f} ms")
