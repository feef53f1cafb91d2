"""Golden vectors for the LJ + Coulomb kernel (builtin_kernels.hpp:41-77 with
Coulomb = true, lj_coulomb_kernel): reduce<double> of the UNMODIFIED reference
(oracle/_ref) over every tests/golden/*.npz store, eps = 1, the fixture's sigma,
coulomb_k = 0.3. Writes tests/golden/lj_coulomb.npz. Run in the build container:

    make -C oracle ref && python tests/golden/make_coulomb_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))
from conftest import golden_names, load_golden, oracle_particles, oracle_store  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402

CK = 0.3


def main():
    R = Oracle("reference")
    out = {}
    for name in golden_names():
        g = load_golden(name)
        qs, sigma = float(g["scale"][1]), float(g["scale"][2])
        outs, cnt = R.reduce("lj_coulomb", oracle_particles(g, sorted_=True), oracle_store(g), query_scale=qs,
                             eps=1.0, sigma=sigma, ck=CK)
        out[name + ".count"] = cnt
        for k in range(4):
            out[f"{name}.{k}"] = outs[k]
        print(name, int(cnt.sum()))
    np.savez_compressed(os.path.join(HERE, "lj_coulomb.npz"), **out)


if __name__ == "__main__":
    main()
