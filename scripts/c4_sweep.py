"""C4 cluster-geometry study (bench.cpp:124-210 run_bench):
LJ fluid, 4M particles at density 100, build_radius_scale 1.100642, sigma 0.2, for
8x8 (w32), 8x4 (w64) and 1x1 over a target-neighbour sweep. Per row: device build and
LJ-pass times (stage events, min of reps), bytes/particle, mean neighbours, and
bench::cluster_overhead (device slot count / directed pairs at query scale 1).
Writes gpurun_out/c4_sweep.jsonl."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2602_19873_b200 as S  # noqa: E402

n = int(os.environ.get("SFCNL_C4_N", "4000000"))
targets = [float(t) for t in os.environ.get("SFCNL_C4_TARGETS", "25,50,100,150,200,300,500").split(",")]
geoms = os.environ.get("SFCNL_C4_GEOMS", "8x8,8x4,1x1").split(",")
reps = 3
ctx = S.Context(0)
ctx.set_timing(True)
os.makedirs("gpurun_out", exist_ok=True)
f = open("gpurun_out/c4_sweep.jsonl", "w")
for t in targets:
    ps, box = S.make_uniform(S.UniformSpec(n=n, density=100.0, target_neighbors=t, seed=42))
    ctx.set_particles(ps, box)
    ctx.sort(); ctx.apply_order(); ctx.octree(64)
    for gname in geoms:
        cp = {"8x8": S.ClusterParams(8, 8, 32), "8x4": S.ClusterParams(8, 4, 64), "1x1": S.ClusterParams(1, 1, 32)}[gname]
        bp = S.BuildParams(cp, S.GATHER, True, 1.100642)
        bt, pt = [], []
        for _ in range(reps):
            nsc, nb = ctx.build_store(bp)
            ctx.synchronize()
            st = ctx.stage_times()
            bt.append(st.get("cluster_geometry", 0) + st.get("build", 0) + st.get("encode", 0))
        for _ in range(reps):
            ctx.reduce(S.lj_kernel(1.0, 0.2), S.PassConfig(1.0, S.MIXED), n, download=False)
            ctx.synchronize()
            pt.append(ctx.stage_times().get("pass", 0))
        cnt = ctx.reduce(S.count_kernel(), S.PassConfig(1.0, S.MIXED), n).neighbor_count
        pairs = int(cnt.astype(np.int64).sum())
        row = dict(config_id=f"uniform-n{n}-t{t:g}-{gname}-comp-gather-lj-mixed-seed42", n=n, target=t,
                   geometry=gname, mean_neighbors=pairs / n, build_ms=min(bt), pass_ms=min(pt),
                   bytes_per_particle=(4 * nsc + 8 * (nsc + 1) + nb) / n,
                   overhead_ratio=ctx.cluster_slots() / pairs, pass_precision="mixed" if cp.ci == 8 else "f64")
        print(json.dumps(row), flush=True)
        f.write(json.dumps(row) + "\n")
        f.flush()
