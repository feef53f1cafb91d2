# Stage times of the device step while the StreamedPipeline's transfers run (vs device-only)
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2602_19873_b200 as S
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
ctx.set_timing(True)
pipe.run(); ctx.synchronize()
print("device-only", {k: round(v, 2) for k, v in ctx.stage_times().items()})
pipe.run_stream(2); ctx.synchronize()
t0 = time.perf_counter(); pipe.run_stream(8); ctx.synchronize(); t1 = time.perf_counter()
print("streamed ms/step", round((t1 - t0) * 1e3 / 8, 2), {k: round(v, 2) for k, v in ctx.stage_times().items()})
