# ncu target: symmetric store at 2^24 (C2 density), one mixed density + one mixed LJ pass
import sys
sys.path.insert(0, '.')
import paper_2602_19873_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 24)
ctx = S.Context(0)
ps, box = S.make_uniform(S.UniformSpec(n=n, density=float(n), target_neighbors=200.0, seed=42))
ctx.set_particles(ps, box)
ctx.sort(); ctx.apply_order(); ctx.octree(64)
ctx.build_store(S.BuildParams(S.ClusterParams(8, 8, 32), S.SYMMETRIC, True, 1.0))
ctx.reduce(S.sph_density_kernel(), S.PassConfig(1.0, S.MIXED), n, download=False)
ctx.reduce(S.lj_kernel(1.0, 0.5 * (1.0 / n) ** (1 / 3)), S.PassConfig(1.0, S.MIXED), n, download=False)
ctx.synchronize()
