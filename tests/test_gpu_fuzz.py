"""Randomised configurations against the plain-C restatement (pinned to the reference by
tests/test_oracle_golden.py): particle count, distribution (uniform with h jitter /
Evrard), periodicity per axis, cluster geometry, list mode, compression, build radius
scale (Verlet skin) and query scale are drawn from a seeded generator. Checks: SFC order
and store bytes bit-exact; fp64 density and LJ bit-exact; mixed pass exact counts,
density within 1e-5 relative, LJ within 1e-5 normwise."""
import os

import numpy as np
import pytest

from oracle.oracle import Oracle

pytestmark = pytest.mark.gpu
P = Oracle("port")
GEOMS = [(8, 8, 32), (8, 4, 64), (1, 1, 32), (8, 8, 64), (8, 4, 32)]


def _draw(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.choice([int(rng.integers(1, 300)), int(rng.integers(300, 6000))]))
    ci, cj, w = GEOMS[int(rng.integers(0, len(GEOMS)))]
    mode = int(rng.random() < 0.35)
    comp = int(rng.random() < 0.8)
    per = tuple(int(v) for v in rng.random(3) < 0.6)
    target = float(rng.uniform(5, 60))
    scale = float(rng.choice([1.0, rng.uniform(1.0, 1.3)]))
    qs = float(min(scale, rng.uniform(0.7, 1.3)))
    evrard = rng.random() < 0.25
    jitter = float(rng.choice([0.0, rng.uniform(0.05, 0.4)]))
    return dict(n=n, ci=ci, cj=cj, w=w, mode=mode, comp=comp, per=per, target=target, scale=scale, qs=qs,
                evrard=evrard, jitter=jitter, seed=seed)


def _abs_lj(sp, sigma, qs, mode):
    pos = np.stack([sp.x, sp.y, sp.z], 1)
    L = sp.box6[3:] - sp.box6[:3]
    per = np.array(sp.periodic, bool)
    absf, abse = np.zeros(sp.n), np.zeros(sp.n)
    for i in range(sp.n):
        d = pos[i] - pos
        d[:, per] -= L[per] * np.rint(d[:, per] / L[per])
        d2 = (d * d).sum(1)
        r = qs * (np.maximum(sp.h[i], sp.h) if mode else sp.h[i])
        ok = d2 <= r * r
        ok[i] = False
        inv2 = 1.0 / d2[ok]
        s6 = (sigma * sigma * inv2) ** 3
        absf[i] = np.sum(np.abs(24.0 * inv2 * (2 * s6 * s6 - s6)) * np.sqrt(d2[ok]))
        abse[i] = np.sum(np.abs(4.0 * (s6 * s6 - s6)))
    return absf, abse


@pytest.fixture(scope="module")
def ctx():
    import paper_2602_19873_b200 as S
    return S.Context(0)


@pytest.mark.parametrize("seed", range(int(os.environ.get("SFCNL_FUZZ_N", "40"))))
def test_random_configuration(ctx, seed):
    import paper_2602_19873_b200 as S
    c = _draw(seed)
    if c["evrard"]:
        op = P.make_evrard(c["n"], c["target"], False, c["per"], 7 + seed)
    else:
        op = P.make_uniform(c["n"], float(c["n"]), c["target"], c["per"], c["jitter"], 7 + seed)
    # a periodic axis must span twice the largest cutoff (neighbor_build.cpp:83-87)
    L = op.box6[3:] - op.box6[:3]
    if any(p and L[d] < 2.0 * c["scale"] * op.h.max() for d, p in enumerate(op.periodic)):
        pytest.skip("periodic box below twice the cutoff for this draw")
    keys, perm, sp, tree, st = P.pipeline(op, ci=c["ci"], cj=c["cj"], w=c["w"], mode=c["mode"], compress=c["comp"],
                                          scale=c["scale"])
    ps = S.ParticleSet(op.x, op.y, op.z, op.h, {"m": op.m, "q": op.q})
    box = S.SimulationBox(tuple(op.box6[:3]), tuple(op.box6[3:]), tuple(bool(v) for v in op.periodic))
    order = S.sort_by_sfc(ps, box, ctx=ctx)
    assert np.array_equal(order.keys, keys) and np.array_equal(order.perm, perm), c
    gtree = S.build_octree(order, 64, ctx=ctx)
    sps = S.apply_sfc_order(ps, order, ctx=ctx)
    bp = S.BuildParams(S.ClusterParams(c["ci"], c["cj"], c["w"]), c["mode"], bool(c["comp"]), c["scale"])
    store = S.build_neighbor_store(sps, box, gtree, bp, ctx=ctx)
    assert np.array_equal(store.counts, st.counts) and np.array_equal(store.blob, st.blob), c
    sigma = 0.4 * (float(np.prod(L)) / max(op.n, 1)) ** (1.0 / 3.0)
    outs, cnt = P.reduce("density", sp, st, query_scale=c["qs"])
    lo, lcnt = P.reduce("lj", sp, st, query_scale=c["qs"], eps=1.0, sigma=sigma)
    d64 = S.reduce(sps, box, store, S.sph_density_kernel(), S.PassConfig(c["qs"], S.F64), ctx=ctx)
    assert np.array_equal(d64.neighbor_count, cnt) and np.array_equal(d64.outputs[0], outs[0]), c
    l64 = S.reduce(sps, box, store, S.lj_kernel(1.0, sigma), S.PassConfig(c["qs"], S.F64), ctx=ctx)
    assert np.array_equal(l64.neighbor_count, lcnt), c
    for k in range(4):
        assert np.array_equal(l64.outputs[k], lo[k]), (c, k)
    d32 = S.reduce(sps, box, store, S.sph_density_kernel(), S.PassConfig(c["qs"], S.MIXED), ctx=ctx)
    assert np.array_equal(d32.neighbor_count, cnt), c
    nz = outs[0] != 0
    assert np.all(d32.outputs[0][~nz] == 0), c
    if nz.any():
        assert np.max(np.abs(d32.outputs[0][nz] - outs[0][nz]) / np.abs(outs[0][nz])) <= 1e-5, c
    l32 = S.reduce(sps, box, store, S.lj_kernel(1.0, sigma), S.PassConfig(c["qs"], S.MIXED), ctx=ctx)
    assert np.array_equal(l32.neighbor_count, lcnt), c
    absf, abse = _abs_lj(sp, sigma, c["qs"], c["mode"])
    err = np.sqrt(sum((l32.outputs[k] - lo[k]) ** 2 for k in range(3)))
    assert np.max(err / np.maximum(absf, 1e-300)) <= 1e-5, c
    assert np.max(np.abs(l32.outputs[3] - lo[3]) / np.maximum(abse, 1e-300)) <= 1e-5, c
