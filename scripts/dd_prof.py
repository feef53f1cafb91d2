# Wall-clock + GPU phase profile of one rank of the domain decomposition (world 1).
import os, sys, time
sys.path.insert(0, '.')
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29519")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
import numpy as np, torch, torch.distributed as dist
import paper_2602_19873_b200 as S
from paper_2602_19873_b200.distributed import Comm, CudaEngine, DomainDecomposition
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
ctx = S.Context(0)
ps, _ = S.make_uniform(S.UniformSpec(n=n, density=float(n), target_neighbors=200.0, seed=42))
box = S.SimulationBox((0.0, 0.0, 0.0), (1.0, 1.0, 1.0), (True, True, True))
E = CudaEngine(ctx, box, ["m"]); E.upload(ps)
dd = DomainDecomposition(E, Comm(), S.BuildParams(S.ClusterParams(8, 8, 32), S.GATHER, True, 1.0),
                         [S.sph_density_kernel(), S.lj_kernel(1.0, 0.5 * (1.0 / n) ** (1 / 3))], S.PassConfig(1.0, S.MIXED))
for it in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    dd.run(download=False)
    torch.cuda.synchronize(); print("step wall ms", round((time.perf_counter() - t0) * 1e3, 1), flush=True)
import cProfile, pstats
pr = cProfile.Profile(); pr.enable(); dd.run(download=False); torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
dist.destroy_process_group()
