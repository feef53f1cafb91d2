# H2D / D2H bandwidth through the paths the StreamedPipeline uses (pinned numpy views)
import time, torch, numpy as np
n = 1 << 26
dev = torch.device("cuda", 0)
C = torch.cuda.Stream(device=dev)
host = [torch.empty(n, dtype=torch.float64, pin_memory=True) for _ in range(5)]
hostnp = [h.numpy() for h in host]
dst = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(5)]
for label, srcs in (("pinned tensors", host), ("from_numpy(pinned numpy)", [torch.from_numpy(a) for a in hostnp])):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(C):
        for s, d in zip(srcs, dst):
            d.copy_(s, non_blocking=True)
    C.synchronize()
    t = time.perf_counter() - t0
    print(f"H2D {label}: {5 * n * 8 / t / 1e9:.1f} GB/s ({t * 1e3:.1f} ms)", flush=True)
    t0 = time.perf_counter()
    with torch.cuda.stream(C):
        for s, d in zip(srcs, dst):
            s.copy_(d, non_blocking=True)
    C.synchronize()
    t = time.perf_counter() - t0
    print(f"D2H {label}: {5 * n * 8 / t / 1e9:.1f} GB/s ({t * 1e3:.1f} ms)", flush=True)
print("is_pinned from_numpy:", torch.from_numpy(hostnp[0]).is_pinned())
