# how many SCs the density fast pass hands to fp64 (error bound), per config
import sys, ctypes as C
sys.path.insert(0, '.')
import paper_2602_19873_b200 as S
for name, gen, n, kw in (("C2", "uniform", 1 << 26, dict(density=float(1 << 26), target_neighbors=200.0)),
                         ("C3", "evrard", 1 << 24, dict(target_neighbors=200.0)),
                         ("C4", "uniform", 4_000_000, dict(density=100.0, target_neighbors=150.0))):
    ctx = S.Context(0)
    ps, box = (S.make_uniform(S.UniformSpec(n=n, seed=42, **kw)) if gen == "uniform" else S.make_evrard(S.EvrardSpec(n=n, seed=42, **kw)))
    ctx.set_particles(ps, box); ctx.sort(); ctx.apply_order(); ctx.octree(64)
    ctx.build_store(S.BuildParams(S.ClusterParams(8, 8, 32), S.GATHER, True, 1.100642 if name == "C4" else 1.0))
    ctx.set_timing(True)
    ctx.reduce(S.sph_density_kernel(), S.PassConfig(1.0, S.MIXED), n, download=False)
    ctx.synchronize()
    t = ctx.stage_times()["pass"]
    p, nb = C.c_void_p(), C.c_uint64()
    print(name, "density pass ms", round(t, 2), flush=True)
    del ctx
