# symmetric mixed density on Evrard (checks the a-posteriori bound does not send it to fp64)
import sys, time
sys.path.insert(0, '.')
import paper_2602_19873_b200 as S
n = 1 << 22
ctx = S.Context(0)
ps, box = S.make_evrard(S.EvrardSpec(n=n, target_neighbors=200.0, seed=42))
ctx.set_particles(ps, box); ctx.sort(); ctx.apply_order(); ctx.octree(64)
for mode in (S.GATHER, S.SYMMETRIC):
    ctx.build_store(S.BuildParams(S.ClusterParams(8, 8, 32), mode, True, 1.0))
    ctx.set_timing(True)
    for prec in (S.MIXED, S.F64):
        ctx.reduce(S.sph_density_kernel(), S.PassConfig(1.0, prec), n, download=False)
        ctx.synchronize()
        print("mode", mode, "prec", prec, "density pass ms", round(ctx.stage_times()["pass"], 2), flush=True)
