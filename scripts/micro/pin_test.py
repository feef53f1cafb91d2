import torch, numpy as np, time
a = torch.empty(1 << 26, dtype=torch.float64, pin_memory=True)
v = a.numpy().view(np.float64)
t = torch.from_numpy(v)
print("pinned via from_numpy:", t.is_pinned(), a.is_pinned())
d = torch.empty(1 << 26, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
for name, dst, src in (("D2H pinned", a, d), ("D2H from_numpy", t, d), ("H2D pinned", d, a)):
    t0 = time.perf_counter(); dst.copy_(src, non_blocking=True); torch.cuda.synchronize()
    t0 = time.perf_counter(); dst.copy_(src, non_blocking=True); torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(name, round(dt * 1e3, 2), "ms", round(a.numel() * 8 / dt / 1e9, 1), "GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
b = torch.empty(1 << 26, dtype=torch.float64, pin_memory=True)
d2 = torch.empty(1 << 26, dtype=torch.float64, device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter()
with torch.cuda.stream(s1): a.copy_(d, non_blocking=True)
with torch.cuda.stream(s2): d2.copy_(b, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
print("duplex 2x512MB", round(dt * 1e3, 2), "ms")
