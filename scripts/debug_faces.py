import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
import paper_2602_19873_b200 as S
from test_gpu_edge import _case, P
op = _case("faces")
ctx = S.Context(0)
for mode in (0, 1):
    keys, perm, sp, tree, st = P.pipeline(op, mode=mode)
    ps = S.ParticleSet(op.x, op.y, op.z, op.h, {"m": op.m, "q": op.q})
    box = S.SimulationBox(tuple(op.box6[:3]), tuple(op.box6[3:]), tuple(bool(v) for v in op.periodic))
    order = S.sort_by_sfc(ps, box, ctx=ctx)
    gtree = S.build_octree(order, 64, ctx=ctx)
    sps = S.apply_sfc_order(ps, order, ctx=ctx)
    store = S.build_neighbor_store(sps, box, gtree, S.BuildParams(S.ClusterParams(8, 8, 32), mode, True, 1.0), ctx=ctx)
    outs, cnt = P.reduce("density", sp, st)
    r32 = S.reduce(sps, box, store, S.sph_density_kernel(), S.PassConfig(1.0, S.MIXED), ctx=ctx)
    rel = np.abs(r32.outputs[0] - outs[0]) / np.abs(outs[0])
    k = np.argsort(rel)[-5:]
    print("mode", mode, "max rel", rel.max(), "worst i", k, rel[k], "cnt", cnt[k], "h", sp.h[k])
    for i in k[-2:]:
        print("  i", i, "sc", i // 64, "x", sp.x[i], sp.y[i], sp.z[i], "rho ref", outs[0][i], "gpu", r32.outputs[0][i])
