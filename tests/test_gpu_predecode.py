"""The decoded-list cache (pass.cu ensure_decoded / k_decode_store): the gather passes
read the store's index lists decoded once per store generation instead of decoding
the codec in each pass.  Results must not depend on it (bit-equal to the in-pass
decode, SFCNL_NO_PREDECODE=1, for the mixed and the fp64 pass), and the cache must
follow the store: several stores reduced in turn on one context each give the
oracle's answer (reduce.hpp:151-197), including a store rebuilt with other
parameters and a re-uploaded blob."""
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


def _setup(ctx, n, seed):
    op = P.make_uniform(n, float(n), 150.0, (1, 1, 1), 0.3, seed)
    ps = S.ParticleSet(op.x, op.y, op.z, op.h, {"m": op.m})
    box = S.SimulationBox(tuple(op.box6[:3]), tuple(op.box6[3:]), (True, True, True))
    order = S.sort_by_sfc(ps, box, ctx=ctx)
    tree = S.build_octree(order, 64, ctx=ctx)
    sps = S.apply_sfc_order(ps, order, ctx=ctx)
    return op, box, tree, sps


def _reduce(ctx, sps, box, store, kern, prec, predecode=True):
    if not predecode:
        os.environ["SFCNL_NO_PREDECODE"] = "1"
    try:
        return S.reduce(sps, box, store, kern, S.PassConfig(1.0, prec), ctx=ctx)
    finally:
        os.environ.pop("SFCNL_NO_PREDECODE", None)


@pytest.mark.parametrize("cj,comp", [(8, 1), (4, 1), (8, 0)])
def test_predecode_equals_in_pass_decode(ctx, cj, comp):
    n = 40000
    op, box, tree, sps = _setup(ctx, n, 21)
    store = S.build_neighbor_store(sps, box, tree, S.BuildParams(S.ClusterParams(8, cj, 32), 0, bool(comp), 1.0),
                                   ctx=ctx)
    sigma = 0.5 * (1.0 / n) ** (1.0 / 3.0)
    for kern in (S.count_kernel(), S.sph_density_kernel(), S.lj_kernel(1.0, sigma)):
        for prec in (S.MIXED, S.F64):
            a = _reduce(ctx, sps, box, store, kern, prec, True)
            b = _reduce(ctx, sps, box, store, kern, prec, False)
            assert np.array_equal(a.neighbor_count, b.neighbor_count)
            for o in range(len(a.outputs)):
                assert np.array_equal(a.outputs[o], b.outputs[o]), (prec, o)


def test_cache_follows_the_store(ctx):
    n = 30000
    op, box, tree, sps = _setup(ctx, n, 33)
    stores = [S.build_neighbor_store(sps, box, tree, S.BuildParams(S.ClusterParams(8, cj, 32), 0, True, sc),
                                     ctx=ctx) for cj, sc in ((8, 1.0), (4, 1.0), (8, 1.25))]
    expect = []
    for cj, sc in ((8, 1.0), (4, 1.0), (8, 1.25)):
        _, _, sp, _, ost = P.pipeline(op, ci=8, cj=cj, w=32, mode=0, compress=1, scale=sc)
        outs, cnt = P.reduce("density", sp, ost, query_scale=1.0)
        expect.append((outs, cnt))
    for i in (0, 1, 2, 1, 0, 2, 2):
        res = _reduce(ctx, sps, box, stores[i], S.sph_density_kernel(), S.F64)
        outs, cnt = expect[i]
        assert np.array_equal(res.neighbor_count, cnt), i
        assert np.array_equal(res.outputs[0], outs[0]), i
