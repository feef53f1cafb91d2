"""The restructured fp64 pass (pass_x64.cuh: fp32 classification with a guard band,
then lane-parallel fp64 evaluation of the marked slots in the reference order) is
bit-equal to reduce<double> (reduce.hpp:151-197) -- checked against the plain-C
restatement and against the thread-per-target kernel it replaces (k_pass_exact,
SFCNL_PASS_EXACT_V1=1), for every built-in kernel, both j-cluster widths, open and
periodic boxes, per-particle h (Evrard), a query scale below the build scale (skin),
raw and w = 64 stores and a periodic box close to twice the cutoff."""
import os

import numpy as np
import pytest

import paper_2602_19873_b200 as S
from oracle.oracle import Oracle

pytestmark = pytest.mark.gpu
P = Oracle("port")


@pytest.fixture(scope="module")
def ctx():
    return S.Context(0)


def _run(ctx, sps, box, store, kern, qs, v1=False):
    if v1:
        os.environ["SFCNL_PASS_EXACT_V1"] = "1"
    try:
        return S.reduce(sps, box, store, kern, S.PassConfig(qs, S.F64), ctx=ctx)
    finally:
        os.environ.pop("SFCNL_PASS_EXACT_V1", None)


CASES = [
    ("uniform", 30000, (8, 8, 32, 1, 1.0), 1.0, (1, 1, 1)),
    ("evrard", 30000, (8, 8, 32, 1, 1.0), 1.0, (0, 0, 0)),
    ("uniform", 20011, (8, 4, 64, 1, 1.0), 1.0, (1, 1, 1)),
    ("uniform", 25000, (8, 8, 32, 0, 1.15), 1.0, (1, 0, 1)),  # raw store, skin
    ("uniform", 25000, (8, 8, 32, 1, 1.2), 0.9, (1, 1, 1)),   # query scale below the build scale
    ("uniform", 3000, (8, 4, 32, 1, 1.0), 1.0, (1, 1, 1)),    # small periodic box: unsafe SCs
]


@pytest.mark.parametrize("gen,n,cfg,qs,per", CASES)
def test_x64_bit_equal(ctx, gen, n, cfg, qs, per):
    ci, cj, w, comp, scale = cfg
    if gen == "uniform":
        op = P.make_uniform(n, float(n), 150.0 if n > 5000 else 400.0, per, 0.3, 11)
    else:
        op = P.make_evrard(n, 120.0, False, per, 11)
    op.q = np.random.default_rng(5).uniform(-1.0, 1.0, n)
    ps = S.ParticleSet(op.x, op.y, op.z, op.h, {"m": op.m, "q": op.q})
    box = S.SimulationBox(tuple(op.box6[:3]), tuple(op.box6[3:]), tuple(bool(v) for v in op.periodic))
    order = S.sort_by_sfc(ps, box, ctx=ctx)
    tree = S.build_octree(order, 64, ctx=ctx)
    sps = S.apply_sfc_order(ps, order, ctx=ctx)
    store = S.build_neighbor_store(sps, box, tree, S.BuildParams(S.ClusterParams(ci, cj, w), 0, bool(comp), scale),
                                   ctx=ctx)
    keys, perm, sp, otree, ost = P.pipeline(op, ci=ci, cj=cj, w=w, mode=0, compress=comp, scale=scale)
    assert np.array_equal(store.blob, ost.blob)
    sigma = 0.5 * (1.0 / n) ** (1.0 / 3.0)
    kernels = [("count", S.count_kernel(), {}), ("density", S.sph_density_kernel(), {}),
               ("lj", S.lj_kernel(1.0, sigma), dict(eps=1.0, sigma=sigma)),
               ("lj_coulomb", S.lj_coulomb_kernel(1.0, sigma, 0.7), dict(eps=1.0, sigma=sigma, ck=0.7))]
    for name, kern, kw in kernels:
        res = _run(ctx, sps, box, store, kern, qs)
        ref = _run(ctx, sps, box, store, kern, qs, v1=True)
        outs, cnt = P.reduce(name, sp, ost, query_scale=qs, **kw)
        assert np.array_equal(res.neighbor_count, cnt), name
        assert np.array_equal(ref.neighbor_count, cnt), name
        for o in range(len(outs)):
            assert np.array_equal(res.outputs[o], outs[o]), (name, o)
            assert np.array_equal(res.outputs[o], ref.outputs[o]), (name, o)


def test_x64_coincident_particles_raise(ctx):
    op = P.make_uniform(4000, 4000.0, 100.0, (1, 1, 1), 0.0, 3)
    op.x[7], op.y[7], op.z[7] = op.x[8], op.y[8], op.z[8]
    ps = S.ParticleSet(op.x, op.y, op.z, op.h, {"m": op.m})
    box = S.SimulationBox(tuple(op.box6[:3]), tuple(op.box6[3:]), (True, True, True))
    order = S.sort_by_sfc(ps, box, ctx=ctx)
    tree = S.build_octree(order, 64, ctx=ctx)
    sps = S.apply_sfc_order(ps, order, ctx=ctx)
    store = S.build_neighbor_store(sps, box, tree, S.BuildParams(), ctx=ctx)
    with pytest.raises(S.InputError, match="coincident"):
        S.reduce(sps, box, store, S.lj_kernel(1.0, 0.01), S.PassConfig(1.0, S.F64), ctx=ctx)
