import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs via gpurun)")


def golden_names():
    names = (os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))
    return sorted(n for n in names if n not in ("full_lists", "lj_coulomb"))  # make_full/coulomb_golden.py


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


@pytest.fixture(params=golden_names())
def golden(request):
    g = load_golden(request.param)
    g["name"] = request.param
    return g


def golden_particles(g, sorted_=False):
    """ParticleSet + box from a fixture (original order, or SFC order)."""
    from paper_2602_19873_b200 import ParticleSet, SimulationBox
    idx = g["perm"] if sorted_ else slice(None)
    ps = ParticleSet(g["x"][idx], g["y"][idx], g["z"][idx], g["h"][idx],
                     {"m": g["m"][idx], "q": g["q"][idx]})
    box = SimulationBox(tuple(g["box6"][:3]), tuple(g["box6"][3:]), tuple(bool(v) for v in g["periodic"]))
    return ps, box


def oracle_particles(g, sorted_=False):
    from oracle.oracle import Particles
    idx = g["perm"] if sorted_ else slice(None)
    return Particles(g["x"][idx].copy(), g["y"][idx].copy(), g["z"][idx].copy(), g["h"][idx].copy(),
                     g["m"][idx].copy(), g["q"][idx].copy(), g["box6"].copy(),
                     tuple(int(v) for v in g["periodic"]))


def oracle_tree(g):
    from oracle.oracle import Tree
    return Tree(g["key_first"], g["key_last"], g["pbegin"], g["pend"], g["first_child"], g["depth"], 21)


def oracle_store(g):
    from oracle.oracle import Store
    ci, cj, w, mode, comp = (int(v) for v in g["params"])
    return Store(len(g["x"]), ci, cj, w, mode, comp, float(g["scale"][0]), g["counts"], g["offsets"], g["blob"])
