import sys; sys.path.insert(0, '.')
import paper_2602_19873_b200 as S
n = 1 << 24
ctx = S.Context(0)
ps, box = S.make_evrard(S.EvrardSpec(n=n, target_neighbors=200.0, seed=42))
bp = S.BuildParams(S.ClusterParams(8, 8, 32), S.GATHER, True, 1.0)
pipe = S.Pipeline(ctx, ps, box, bp, [S.sph_density_kernel()], S.PassConfig(1.0, S.MIXED))
pipe.upload(); pipe.run(); ctx.synchronize()
