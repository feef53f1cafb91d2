"""Compressed clustered list vs the full per-particle Verlet list on
one B200: memory and device time of the build and of the density / LJ passes at the
C2 configuration (SFCNL_FL_N particles, default 2^26, 200 neighbours, 8x8 clusters).
Device times from the context's stage events (kPass covers the list build / pass).
Writes gpurun_out/full_list_bench.json."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2602_19873_b200 as S  # noqa: E402

n = int(os.environ.get("SFCNL_FL_N", str(1 << 26)))
reps = 3
ctx = S.Context(0)
ps, box = S.make_uniform(S.UniformSpec(n=n, density=float(n), target_neighbors=200.0, seed=42))
bp = S.BuildParams(S.ClusterParams(8, 8, 32), S.GATHER, True, 1.0)
sigma = 0.5 * (1.0 / n) ** (1.0 / 3.0)
ctx.set_particles(ps, box)
ctx.set_timing(True)


def timed(fn, stages):
    best = []
    for _ in range(reps):
        fn()
        ctx.synchronize()
        t = ctx.stage_times()
        best.append(sum(t.get(s, 0.0) for s in stages))
    return min(best), float(np.median(best))


out = dict(n=n, config="C2 uniform periodic, 200 neighbours, 8x8 gather compressed")
ctx.sort(); ctx.apply_order(); nn = ctx.octree(64)
nsc, nb = ctx.build_store(bp)
out["store_bytes"] = 4 * nsc + 8 * (nsc + 1) + nb
out["store_build_ms"] = timed(lambda: ctx.build_store(bp), ("cluster_geometry", "build", "encode"))
for name, k in (("density", S.sph_density_kernel()), ("lj", S.lj_kernel(1.0, sigma))):
    for prec, pn in ((S.MIXED, "mixed"), (S.F64, "f64")):
        out[f"compressed_{name}_{pn}_ms"] = timed(lambda: ctx.reduce(k, S.PassConfig(1.0, prec), n, download=False),
                                                  ("pass",))
rho = ctx.reduce(S.count_kernel(), S.PassConfig(1.0, S.MIXED), n)
pairs_store = int(rho.neighbor_count.astype(np.int64).sum())
pairs = ctx.build_full_list(1.0)
out["full_pairs"] = pairs
assert pairs == pairs_store, (pairs, pairs_store)
out["full_list_bytes"] = 8 * (n + 1) + 4 * pairs
out["full_build_from_store_ms"] = timed(lambda: ctx.build_full_list(1.0), ("pass",))
for name, k in (("density", S.sph_density_kernel()), ("lj", S.lj_kernel(1.0, sigma))):
    for prec, pn in ((S.MIXED, "warp_f64"), (S.F64, "f64")):
        out[f"full_{name}_{pn}_ms"] = timed(lambda: ctx.reduce_full(k, S.PassConfig(1.0, prec), n, download=False),
                                            ("pass",))
# cross-check: the two passes see the same pair set
a = ctx.reduce(S.sph_density_kernel(), S.PassConfig(1.0, S.MIXED), n)
b = ctx.reduce_full(S.sph_density_kernel(), S.PassConfig(1.0, S.MIXED), n)
assert np.array_equal(a.neighbor_count, b.neighbor_count)
out["density_max_rel_diff_compressed_vs_full"] = float(np.max(np.abs(a.outputs[0] - b.outputs[0]) / b.outputs[0]))
out["bytes_per_particle"] = dict(compressed=out["store_bytes"] / n, full=out["full_list_bytes"] / n)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/full_list_bench.json", "w"), indent=1)
print(json.dumps(out))
