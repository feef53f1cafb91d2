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
    absf = T._sum_abs_pair_forces(oracle_particles(g, True), oracle_store(g), qs, sigma)
    err = np.sqrt(sum((res.outputs[k] - ref[k]) ** 2 for k in range(3)))
    rel = err / np.maximum(absf, 1e-300)
    w = int(np.argmax(rel))
    refn = np.sqrt(sum(ref[k] ** 2 for k in range(3)))
    print(name, "max norm err", rel.max(), "at", w, "absf", absf[w], "err", err[w], "|F|", refn[w], "cnt", res.neighbor_count[w],
          "E rel", np.max(np.abs(res.outputs[3] - ref[3]) / np.maximum(np.abs(ref[3]), 1e-300)))
    print("   F gpu", [res.outputs[k][w] for k in range(4)], "ref", [ref[k][w] for k in range(4)])
