"""Symmetric (half-list) mode at scale: device build and pass times of a
symmetric store vs the gather store on the C2 workload (SFCNL_SYM_N particles, default
2^24), and the pair-set witness (sum of neighbor counts equal). Stage-event timing.
Writes gpurun_out/sym_bench.json."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2602_19873_b200 as S  # noqa: E402

n = int(os.environ.get("SFCNL_SYM_N", str(1 << 24)))
ctx = S.Context(0)
ctx.set_timing(True)
ps, box = S.make_uniform(S.UniformSpec(n=n, density=float(n), target_neighbors=200.0, seed=42))
ctx.set_particles(ps, box)
ctx.sort(); ctx.apply_order(); ctx.octree(64)
sigma = 0.5 * (1.0 / n) ** (1.0 / 3.0)
out = dict(n=n)
for mode, name in ((S.GATHER, "gather"), (S.SYMMETRIC, "symmetric")):
    bp = S.BuildParams(S.ClusterParams(8, 8, 32), mode, True, 1.0)
    bt = []
    for _ in range(3):
        nsc, nb = ctx.build_store(bp)
        ctx.synchronize()
        st = ctx.stage_times()
        bt.append(st.get("cluster_geometry", 0) + st.get("build", 0) + st.get("encode", 0))
    out[f"{name}_build_ms"] = min(bt)
    out[f"{name}_bytes_per_particle"] = (4 * nsc + 8 * (nsc + 1) + nb) / n
    for kn, k in (("density", S.sph_density_kernel()), ("lj", S.lj_kernel(1.0, sigma))):
        for prec, pn in ((S.F64, "f64"), (S.MIXED, "mixed")):
            pt = []
            for _ in range(3):
                ctx.reduce(k, S.PassConfig(1.0, prec), n, download=False)
                ctx.synchronize()
                pt.append(ctx.stage_times().get("pass", 0))
            out[f"{name}_{kn}_{pn}_ms"] = min(pt)
    cnt = ctx.reduce(S.count_kernel(), S.PassConfig(1.0, S.F64), n).neighbor_count
    out[f"{name}_pairs"] = int(cnt.astype(np.int64).sum())
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/sym_bench.json", "w"), indent=1)
print(json.dumps(out))
