# Per-stage timing of StreamedPipeline.run_stream on 2^26 (S-stream events + host wall)
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2602_19873_b200 as S
n = 1 << 26
ctx = S.Context(0)
ps, box = S.make_uniform(S.UniformSpec(n=n, density=float(n), target_neighbors=200.0, seed=42))
pinned = {}
for name in ("x", "y", "z", "h"):
    t = torch.empty(n, dtype=torch.float64, pin_memory=True); t.numpy()[:] = getattr(ps, name); pinned[name] = t
t = torch.empty(n, dtype=torch.float64, pin_memory=True); t.numpy()[:] = ps.fields["m"]; pinned["m"] = t
pps = S.ParticleSet(*(pinned[k].numpy() for k in "xyzh"), {"m": pinned["m"].numpy()})
dt = {np.dtype(np.uint32): torch.int32, np.dtype(np.uint64): torch.int64, np.dtype(np.uint8): torch.uint8, np.dtype(np.float64): torch.float64}
pipe = S.StreamedPipeline(ctx, pps, box, S.BuildParams(S.ClusterParams(8, 8, 32), S.GATHER, True, 1.0),
                          [S.sph_density_kernel(), S.lj_kernel(1.0, 0.5 * (1.0 / n) ** (1 / 3))], S.PassConfig(1.0, S.MIXED))
pipe.upload()
pipe.host_buffers(lambda cnt, d: torch.empty(int(cnt), dtype=dt[np.dtype(d)], pin_memory=True).numpy().view(d))
pipe.run_stream(2)
for K in (1, 4, 8):
    torch.cuda.synchronize(); t0 = time.perf_counter(); pipe.run_stream(K); print("K", K, "ms/step", round((time.perf_counter() - t0) * 1e3 / K, 1), flush=True)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(4): pipe.run()
ctx.synchronize(); print("device-only ms/step", round((time.perf_counter() - t0) * 1e3 / 4, 1))
# device-only steps while a second stream keeps PCIe busy (both directions)
Cs = torch.cuda.Stream()
hb = torch.empty(1 << 27, dtype=torch.float64, pin_memory=True); db = torch.empty(1 << 27, dtype=torch.float64, device="cuda")
hb2 = torch.empty(1 << 27, dtype=torch.float64, pin_memory=True); db2 = torch.empty(1 << 27, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
with torch.cuda.stream(Cs):
    for _ in range(40):
        hb.copy_(db, non_blocking=True); db2.copy_(hb2, non_blocking=True)
t0 = time.perf_counter()
for _ in range(4): pipe.run()
ctx.synchronize(); print("device-only with concurrent PCIe copies ms/step", round((time.perf_counter() - t0) * 1e3 / 4, 1))
torch.cuda.synchronize()
