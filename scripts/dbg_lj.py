# LJ mixed-pass error per golden fixture (force normwise vs sum_j|F_ij|, energy vs sum_j|E_ij|)
import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2602_19873_b200 as S
from conftest import golden_names, load_golden, golden_particles, oracle_particles, oracle_store
import test_gpu_parity as T
ctx = S.Context(0)
for name in golden_names():
    g = load_golden(name)
    if int(g["params"][3]) != 0: continue
    sp, box = golden_particles(g, sorted_=True)
    store = S.NeighborStore(T._bp(g), len(g["x"]), g["counts"], g["offsets"], g["blob"])
    qs, sigma = float(g["scale"][1]), float(g["scale"][2])
    res = S.reduce(sp, box, store, S.lj_kernel(1.0, sigma), S.PassConfig(qs, S.MIXED), ctx=ctx)
    ref = [g[f"lj_double_{k}"] for k in range(4)]
    absf, abse = T._sum_abs_pair_forces(oracle_particles(g, True), oracle_store(g), qs, sigma)
    err = np.sqrt(sum((res.outputs[k] - ref[k]) ** 2 for k in range(3)))
    rel = err / np.maximum(absf, 1e-300)
    erel = np.abs(res.outputs[3] - ref[3]) / np.maximum(abse, 1e-300)
    w = int(np.argmax(erel))
    print(name, "F err", rel.max(), "E err", erel.max(), "at", w, "E", res.outputs[3][w], ref[3][w], "abse", abse[w], "cnt ok", np.array_equal(res.neighbor_count, g["lj_double_count"]))
