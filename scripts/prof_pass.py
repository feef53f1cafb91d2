# ncu target: one uniform step (build + density + LJ mixed passes)
import sys
sys.path.insert(0, '.')
import paper_2602_19873_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 21)
ctx = S.Context(0)
ps, box = S.make_uniform(S.UniformSpec(n=n, density=float(n), target_neighbors=200.0))
sigma = 0.5 * (1.0 / n) ** (1 / 3)
pipe = S.Pipeline(ctx, ps, box, S.BuildParams(), [S.sph_density_kernel(), S.lj_kernel(1.0, sigma)], S.PassConfig(1.0, S.MIXED))
pipe.upload()
pipe.run()
ctx.synchronize()
