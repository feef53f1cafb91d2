"""LJ + Coulomb kernel (builtin_kernels.hpp:41-77, Coulomb = true) against the
reference's reduce<double> (tests/golden/lj_coulomb.npz, make_coulomb_golden.py).

CPU: the plain-C restatement reproduces the golden outputs bit for bit.
GPU: the fp64 pass is bit-equal (gather and symmetric stores); the mixed pass has the
exact pair set and force / energy errors <= 1e-5 x sum_j |term_ij| (LJ + Coulomb terms,
brute force over the same neighbourhood)."""
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_names, golden_particles, load_golden, oracle_particles, oracle_store
from oracle.oracle import Oracle

CK = 0.3
GOLD = dict(np.load(os.path.join(GOLDEN, "lj_coulomb.npz")))


@pytest.mark.parametrize("name", golden_names())
def test_restatement_matches_reference(name):
    g = load_golden(name)
    qs, sigma = float(g["scale"][1]), float(g["scale"][2])
    outs, cnt = Oracle("port").reduce("lj_coulomb", oracle_particles(g, sorted_=True), oracle_store(g), query_scale=qs,
                                      eps=1.0, sigma=sigma, ck=CK)
    assert np.array_equal(cnt, GOLD[name + ".count"])
    for k in range(4):
        assert np.array_equal(outs[k], GOLD[f"{name}.{k}"]), k


def _abs_terms(g, qs, sigma, mode):
    idx = g["perm"]
    pos = np.stack([g["x"][idx], g["y"][idx], g["z"][idx]], 1)
    h, q = g["h"][idx], g["q"][idx]
    L = g["box6"][3:] - g["box6"][:3]
    per = np.array(g["periodic"], bool)
    absf, abse = np.zeros(len(h)), np.zeros(len(h))
    for i in range(len(h)):
        d = pos[i] - pos
        d[:, per] -= L[per] * np.rint(d[:, per] / L[per])
        d2 = (d * d).sum(1)
        r = qs * (np.maximum(h[i], h) if mode else h[i])
        ok = d2 <= r * r
        ok[i] = False
        d2o = d2[ok]
        inv2 = 1.0 / d2o
        s6 = (sigma * sigma * inv2) ** 3
        qq = CK * q[i] * q[ok]
        ir = np.sqrt(inv2)
        absf[i] = np.sum((np.abs(24.0 * inv2 * (2 * s6 * s6 - s6)) + np.abs(qq * ir * inv2)) * np.sqrt(d2o))
        abse[i] = np.sum(np.abs(4.0 * (s6 * s6 - s6)) + np.abs(qq * ir))
    return absf, abse


@pytest.mark.gpu
@pytest.mark.parametrize("name", golden_names())
def test_gpu_lj_coulomb(name):
    import paper_2602_19873_b200 as S
    g = load_golden(name)
    ci, cj, w, mode, comp = (int(v) for v in g["params"])
    qs, sigma = float(g["scale"][1]), float(g["scale"][2])
    sp, box = golden_particles(g, sorted_=True)
    store = S.NeighborStore(S.BuildParams(S.ClusterParams(ci, cj, w), mode, bool(comp), float(g["scale"][0])),
                            len(g["x"]), g["counts"], g["offsets"], g["blob"])
    kern = S.lj_coulomb_kernel(1.0, sigma, CK)
    ctx = S.Context(0)
    res = S.reduce(sp, box, store, kern, S.PassConfig(qs, S.F64), ctx=ctx)
    assert np.array_equal(res.neighbor_count, GOLD[name + ".count"])
    for k in range(4):
        assert np.array_equal(res.outputs[k], GOLD[f"{name}.{k}"]), k
    res = S.reduce(sp, box, store, kern, S.PassConfig(qs, S.MIXED), ctx=ctx)
    assert np.array_equal(res.neighbor_count, GOLD[name + ".count"])
    absf, abse = _abs_terms(g, qs, sigma, mode)
    err = np.sqrt(sum((res.outputs[k] - GOLD[f"{name}.{k}"]) ** 2 for k in range(3)))
    assert np.max(err / np.maximum(absf, 1e-300)) <= 1e-5
    assert np.max(np.abs(res.outputs[3] - GOLD[f"{name}.3"]) / np.maximum(abse, 1e-300)) <= 1e-5
