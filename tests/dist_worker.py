"""TEST INFRASTRUCTURE: one rank of a domain-decomposed step (launched by
tests/test_distributed.py as P processes; RANK/WORLD_SIZE/MASTER_* from the env).

usage: dist_worker.py OUT_DIR CONFIG_JSON
Every rank generates the same global particle set, keeps an (uneven) contiguous
share of global ids as its input, runs DomainDecomposition.run() and writes its
store slice and pass outputs to OUT_DIR/rank{r}.npz.
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2602_19873_b200 as sfcnl  # noqa: E402
from paper_2602_19873_b200.distributed import Comm, CudaEngine, DomainDecomposition  # noqa: E402

KERNELS = {"count": lambda: sfcnl.count_kernel(), "density": lambda: sfcnl.sph_density_kernel(),
           "lj": lambda: sfcnl.lj_kernel(1.0, 0.05), "lj_coulomb": lambda: sfcnl.lj_coulomb_kernel(1.0, 0.05, 0.3)}


def shares(n, world):
    # deliberately uneven contiguous shares of the global ids
    b = [int(round(n * (q / world) ** 1.3)) for q in range(world + 1)]
    b[-1] = n
    return b


def main():
    out_dir, cfg = sys.argv[1], json.loads(sys.argv[2])
    if cfg.get("backend", "gloo") == "nccl":
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    from oracle.oracle import Oracle
    o = Oracle("port")
    if cfg.get("dist", "uniform") == "uniform":
        gp = o.make_uniform(cfg["n"], float(cfg["n"]), cfg["target"], tuple(cfg["periodic"]),
                            cfg.get("h_jitter", 0.0), cfg["seed"])
    else:
        gp = o.make_evrard(cfg["n"], cfg["target"], False, tuple(cfg["periodic"]), cfg["seed"])
    b = [gp.n * q // world for q in range(world + 1)] if cfg.get("even_shares") else shares(gp.n, world)
    idx = np.arange(b[rank], b[rank + 1])
    bp = sfcnl.BuildParams(sfcnl.ClusterParams(cfg["ci"], cfg["cj"], cfg["w"]), cfg.get("mode", sfcnl.GATHER),
                           bool(cfg.get("compress", 1)), cfg.get("scale", 1.0))
    kernels = [KERNELS[k]() for k in cfg["kernels"]]
    pcfg = sfcnl.PassConfig(cfg.get("query_scale", 1.0), cfg.get("precision", sfcnl.F64))
    box = sfcnl.SimulationBox(tuple(gp.box6[:3]), tuple(gp.box6[3:]), tuple(bool(p) for p in gp.periodic))
    if cfg["engine"] == "oracle":
        from dist_engines import OracleEngine
        E = OracleEngine(o, gp.box6, gp.periodic)
        E.upload(gp.permuted(idx))
    else:
        ctx = sfcnl.Context(int(os.environ.get("LOCAL_RANK", "0")))
        E = CudaEngine(ctx, box, ["m", "q"])
        E.upload(sfcnl.ParticleSet(gp.x[idx], gp.y[idx], gp.z[idx], gp.h[idx], {"m": gp.m[idx], "q": gp.q[idx]}))
    mem = {}
    if cfg.get("measure_memory"):
        # single-GPU footprint of the same step on the rank's own particles (own context)
        c1 = sfcnl.Context(int(os.environ.get("LOCAL_RANK", "0")))
        ps1 = sfcnl.ParticleSet(gp.x[idx], gp.y[idx], gp.z[idx], gp.h[idx], {"m": gp.m[idx], "q": gp.q[idx]})
        pipe = sfcnl.Pipeline(c1, ps1, box, bp, kernels, pcfg)
        pipe.upload()
        pipe.run()
        c1.synchronize()
        mem["single"] = E.memory_bytes()  # every DBuf of the process: c1 (E's context is still empty)
        c1.close()
        del pipe, c1
        mem["base"] = E.memory_bytes()
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
    dd = DomainDecomposition(E, Comm(), bp, kernels, pcfg)
    res = dd.run(download=not cfg.get("measure_memory"))
    if cfg.get("measure_memory"):
        torch.cuda.synchronize()
        mem["dd_ctx"] = E.memory_bytes() - mem["base"]
        mem["dd_torch"] = torch.cuda.memory_allocated()
        mem["dd_torch_peak"] = torch.cuda.max_memory_allocated()
        mem["n_in"] = len(idx)
        mem["n_local"] = E.n_local
        mem["halo"] = res.halo_particles
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **{k: np.array(v) for k, v in mem.items()})
        dist.barrier()
        dist.destroy_process_group()
        return
    rec = dict(p0=res.p_begin, p1=res.p_end, sc0=res.sc_begin, sc1=res.sc_end, n=res.n_total,
               num_nodes=res.num_nodes, halo=res.halo_particles, counts=res.store.counts,
               offsets=res.store.offsets, blob=res.store.blob)
    t = getattr(E, "tree", None)
    if t is not None:  # the rank's copy of the (distributed) global octree
        rec.update(t_kf=t.key_first, t_kl=t.key_last, t_pb=t.pbegin, t_pe=t.pend, t_fc=t.first_child, t_d=t.depth)
    for k, rr in enumerate(res.results):
        for j, v in enumerate(rr.outputs):
            rec[f"k{k}_o{j}"] = v
        rec[f"k{k}_cnt"] = rr.neighbor_count
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **rec)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
