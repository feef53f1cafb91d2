"""Golden vectors for the full Verlet list baseline: runs the
UNMODIFIED reference's build_full_list (cell grid, baselines.cpp:39-131) and
reduce_full<double> (baselines.hpp:47-129) through oracle/_ref on the particles of
every tests/golden/*.npz fixture (SFC order and original order) and writes
tests/golden/full_lists.npz: per case and order the pair count, the SHA-256 of
offsets||neighbors, the reduce_full<double> outputs of count / density / LJ, and
(gather stores) bench::cluster_overhead of the fixture's store against the
in-range pair count of the full list at query scale.
Run in the build container:

    make -C oracle ref && python tests/golden/make_full_golden.py
"""
import glob
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))
from conftest import oracle_particles  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402


def digest(offsets, nbrs):
    return hashlib.sha256(np.ascontiguousarray(offsets, np.uint64).tobytes()
                          + np.ascontiguousarray(nbrs, np.uint32).tobytes()).hexdigest()


def main():
    R = Oracle("reference")
    out = {}
    for path in sorted(glob.glob(os.path.join(HERE, "*.npz"))):
        name = os.path.basename(path)[:-4]
        if name == "full_lists":
            continue
        g = dict(np.load(path))
        scale, qs, sigma = (float(v) for v in g["scale"])
        mode = int(g["params"][3])
        for order in ("sorted", "orig"):
            ps = oracle_particles(g, sorted_=order == "sorted")
            off, nb, res = R.full_list(ps, scale, ("count", "density", "lj"), qs, 1.0, sigma, mode=mode)
            key = f"{name}.{order}"
            out[key + ".pairs"] = np.array([len(nb)], np.uint64)
            out[key + ".sha"] = np.frombuffer(bytes.fromhex(digest(off, nb)), np.uint8)
            for kern, (outs, cnt) in res.items():
                out[f"{key}.{kern}.count"] = cnt
                for o, v in enumerate(outs):
                    out[f"{key}.{kern}.{o}"] = v
            if order == "sorted" and mode == 0:
                # reduce_full<double> over the gather full list == reduce<double> over the store
                # (same pair set, same ascending-j order): pins both against each other
                for kern in ("count", "density", "lj"):
                    assert np.array_equal(res[kern][1], g[f"{kern}_double_count"]), (name, kern)
                    for o in range(len(res[kern][0])):
                        assert np.array_equal(res[kern][0][o], g[f"{kern}_double_{o}"]), (name, kern, o)
            if order == "sorted" and mode == 0:
                from conftest import oracle_store
                pairs_q = int(res["count"][1].astype(np.int64).sum())
                out[name + ".overhead"] = np.array([R.cluster_overhead(oracle_store(g), pairs_q)])
            print(name, order, len(nb))
    np.savez_compressed(os.path.join(HERE, "full_lists.npz"), **out)


if __name__ == "__main__":
    main()
