import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_2602_19873_b200 as S
ctx = S.Context(0)
ctx.set_timing(True)
for n in [1<<20, 1<<23]:
    ps, box = S.make_uniform(S.UniformSpec(n=n, density=float(n), target_neighbors=200.0))
    sigma = 0.5 * (1.0/n) ** (1/3)
    pipe = S.Pipeline(ctx, ps, box, S.BuildParams(), [S.sph_density_kernel(), S.lj_kernel(1.0, sigma)], S.PassConfig(1.0, S.MIXED))
    pipe.upload()
    for it in range(3):
        ctx.synchronize(); t = time.perf_counter(); pipe.run(); ctx.synchronize(); dt = time.perf_counter() - t
        print(n, f"step {dt*1e3:.2f} ms  {dt*1e9/n:.2f} ns/particle", {k: round(v, 3) for k, v in ctx.stage_times().items()}, "B/p", (pipe.blob_bytes + 12*pipe.num_sc + 8)/n, flush=True)
    for prec in (S.F64,):
        ctx.synchronize(); t = time.perf_counter(); ctx.reduce(S.sph_density_kernel(), S.PassConfig(1.0, prec), n, download=False); ctx.synchronize()
        print("fp64 density pass", (time.perf_counter()-t)*1e3, "ms")
