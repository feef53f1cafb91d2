# overflow counts of the warp build's tiers at C2 (reads build_ctl through device_array-free path: stderr print needs PHASE_PROF)
import sys, ctypes as C
sys.path.insert(0, '.')
import paper_2602_19873_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 26)
ctx = S.Context(0)
ps, box = S.make_uniform(S.UniformSpec(n=n, density=float(n), target_neighbors=200.0, seed=42))
ctx.set_particles(ps, box); ctx.sort(); ctx.apply_order(); ctx.octree(64)
ctx.set_timing(True)
ctx.build_store(S.BuildParams())
ctx.synchronize()
print(ctx.stage_times())
