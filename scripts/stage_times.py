"""Per-stage device times of the bench step (median of R instrumented steps).
usage: stage_times.py [--n N] [--evrard] [--reps R] [--label L] [--f64]"""
import argparse, json, sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_19873_b200 as S

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 26)
ap.add_argument("--evrard", action="store_true")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--label", default=os.environ.get("SFCNL_LIB", "default"))
ap.add_argument("--f64", action="store_true")
a = ap.parse_args()
n = a.n
ctx = S.Context(0)
if a.evrard:
    ps, box = S.make_evrard(S.EvrardSpec(n=n, target_neighbors=200.0, seed=42))
else:
    ps, box = S.make_uniform(S.UniformSpec(n=n, density=float(n), target_neighbors=200.0, seed=42))
sigma = 0.5 * (1.0 / n) ** (1.0 / 3.0)
kernels = [S.sph_density_kernel(), S.lj_kernel(1.0, sigma)]
bp = S.BuildParams(S.ClusterParams(8, 8, 32), S.GATHER, True, 1.0)
precs = [S.MIXED] + ([S.F64] if a.f64 else [])
ctx.set_particles(ps, box)
rows = []
for r in range(a.reps + 1):
    ctx.set_timing(True)
    ctx.sort(21); ctx.apply_order(); ctx.octree(64); ctx.build_store(bp)
    st = {k: v for k, v in ctx.stage_times().items() if k != "pass"}
    for p in precs:
        for k in kernels:
            ctx.reduce(k, S.PassConfig(1.0, p), n, download=False)
            st[("pass_" if p == S.MIXED else "f64_") + k.names[0]] = ctx.stage_times()["pass"]
    ctx.set_timing(False)
    if r:
        rows.append(st)
med = {k: round(float(np.median([r[k] for r in rows])), 3) for k in rows[0]}
med["total"] = round(sum(v for k, v in med.items() if not k.startswith("f64_")), 3)
print(json.dumps({"label": a.label, "n": n, "evrard": a.evrard, "stages_ms": med}), flush=True)
