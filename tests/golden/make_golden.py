"""Generates the golden fixtures in tests/golden/*.npz by running the UNMODIFIED
reference (oracle/_ref/libsfcnl_ref.so, compiled from /root/reference/proj/src by
oracle/Makefile) on small seeded inputs. Run in the build container:

    make -C oracle ref && python tests/golden/make_golden.py

Each fixture pins, for one configuration: the inputs, sort_by_sfc (keys, perm),
build_octree (node arrays), compute_node_aabbs/max_radius, the NeighborStore
bytes, and reduce<double>/reduce<float> outputs of the count, SPH-density and LJ
kernels. The GPU tests and the oracle tests both check against these files.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import Oracle  # noqa: E402

CONFIGS = {
    # name: (generator, gen args, ci, cj, w, mode, compress, build scale, query scale)
    "uniform_8x8": ("uniform", dict(n=3000, density=3000.0, target=60.0, periodic=(1, 1, 1)), 8, 8, 32, 0, 1, 1.0, 1.0),
    "evrard_8x8": ("evrard", dict(n=3000, target=60.0, periodic=(0, 0, 0)), 8, 8, 32, 0, 1, 1.0, 1.0),
    "uniform_8x4_w64_raw": ("uniform", dict(n=2500, density=2500.0, target=50.0, periodic=(1, 0, 1)), 8, 4, 64, 0, 0, 1.0, 1.0),
    "uniform_symmetric": ("uniform", dict(n=2000, density=2000.0, target=40.0, periodic=(1, 1, 1), h_jitter=0.3), 8, 8, 32, 1, 1, 1.0, 1.0),
    "jitter_skin": ("uniform", dict(n=2777, density=2777.0, target=50.0, periodic=(1, 1, 1), h_jitter=0.25), 8, 8, 32, 0, 1, 1.2, 1.0),
    "uniform_1x1": ("uniform", dict(n=700, density=700.0, target=30.0, periodic=(1, 1, 1)), 1, 1, 32, 0, 1, 1.0, 1.0),
}


def make(name, spec, R):
    gen, ga, ci, cj, w, mode, comp, scale, qs = spec
    if gen == "uniform":
        ps = R.make_uniform(ga["n"], ga["density"], ga["target"], ga["periodic"], ga.get("h_jitter", 0.0), 42)
    else:
        ps = R.make_evrard(ga["n"], ga["target"], False, ga["periodic"], 42)
    keys, perm = R.sort_by_sfc(ps)
    sp = ps.permuted(perm)
    tree, lo, hi, rad = R.node_geometry(keys, sp)
    # the reference's own SFNLSTOR v1 writer (neighbor_store.cpp:84-103) -> <name>.sfnl
    store = R.build_store(sp, tree, ci, cj, w, mode, comp, scale, threads=1,
                          write_path=os.path.join(HERE, name + ".sfnl"))
    sigma = 0.5 * (1.0 / (ga["density"] if gen == "uniform" else ga["n"])) ** (1.0 / 3.0)
    out = dict(x=ps.x, y=ps.y, z=ps.z, h=ps.h, m=ps.m, q=ps.q, box6=ps.box6,
               periodic=np.array(ps.periodic, np.int32), keys=keys, perm=perm,
               key_first=tree.key_first, key_last=tree.key_last, pbegin=tree.pbegin, pend=tree.pend,
               first_child=tree.first_child, depth=tree.depth, node_lo=lo, node_hi=hi, node_radius=rad,
               counts=store.counts, offsets=store.offsets, blob=store.blob,
               params=np.array([ci, cj, w, mode, comp], np.int64), scale=np.array([scale, qs, sigma]))
    for kern in ("count", "density", "lj"):
        for real in ("double", "float"):
            o, c = R.reduce(kern, sp, store, query_scale=qs, eps=1.0, sigma=sigma, real=real, threads=1)
            for k, arr in enumerate(o):
                out[f"{kern}_{real}_{k}"] = arr
            out[f"{kern}_{real}_count"] = c
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, "n", ps.n, "nodes", len(tree.pend), "blob", len(store.blob))


if __name__ == "__main__":
    R = Oracle("reference")
    for name, spec in CONFIGS.items():
        make(name, spec, R)
