"""Edge cases of the GPU path against the plain-C restatement (pinned to the reference's
golden fixtures by tests/test_oracle_golden.py): tiny and ragged particle counts (partial
i-/j-clusters and super-clusters), duplicated positions (stable-sort ties, d = 0 pairs,
the LJ coincidence error), a periodic box barely twice the cutoff (every SC takes the
exact "unsafe" paths), positions exactly on the box faces (wrap), and a strongly
clustered set (deep octree, per-particle h over two decades). For each: SFC keys/perm,
store bytes bit-exact; fp64 density bit-exact; mixed density exact counts and within
1e-5; for 8x8 / 8x4 gather, 8x8 symmetric and 1x1 geometries."""
import zlib

import numpy as np
import pytest

from oracle.oracle import Oracle, Particles

pytestmark = pytest.mark.gpu
P = Oracle("port")
GEOMS = [(8, 8, 32, 0, 1), (8, 4, 64, 0, 0), (8, 8, 32, 1, 1), (1, 1, 32, 0, 1)]


def _particles(x, y, z, h, box6, periodic, seed=0):
    rng = np.random.default_rng(seed)
    n = len(x)
    return Particles(np.ascontiguousarray(x, float), np.ascontiguousarray(y, float), np.ascontiguousarray(z, float),
                     np.ascontiguousarray(h, float), rng.uniform(0.5, 1.5, n), np.where(rng.random(n) < 0.5, -1.0, 1.0),
                     np.array(box6, float), tuple(periodic))


def _case(name):
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    if name.startswith("tiny"):
        n = int(name.split("-")[1])
        p = rng.random((n, 3))
        return _particles(p[:, 0], p[:, 1], p[:, 2], np.full(n, 0.3), [0, 0, 0, 1, 1, 1], (0, 0, 0))
    if name == "duplicates":
        base = rng.random((100, 3))
        p = np.repeat(base, 5, axis=0)
        return _particles(p[:, 0], p[:, 1], p[:, 2], np.full(500, 0.2), [0, 0, 0, 1, 1, 1], (0, 0, 0))
    if name == "tight-periodic":
        p = rng.random((4000, 3))
        return _particles(p[:, 0], p[:, 1], p[:, 2], np.full(4000, 0.495), [0, 0, 0, 1, 1, 1], (1, 1, 1))
    if name == "faces":
        p = rng.random((3000, 3))
        k = rng.integers(0, 3000, 600)
        p[k[:300], 0] = 1.0  # exactly on hi (inside: c <= hi)
        p[k[300:], 1] = 0.0
        p[k[::7], 2] = 1.0
        return _particles(p[:, 0], p[:, 1], p[:, 2], np.full(3000, 0.09), [0, 0, 0, 1, 1, 1], (1, 1, 0))
    if name == "clustered":
        a = 0.5 + 1e-4 * rng.standard_normal((2900, 3))
        b = rng.random((100, 3))
        p = np.clip(np.vstack([a, b]), 0, 1)
        h = np.exp(rng.uniform(np.log(1e-3), np.log(0.05), 3000))
        return _particles(p[:, 0], p[:, 1], p[:, 2], h, [0, 0, 0, 1, 1, 1], (0, 0, 0))
    raise KeyError(name)


CASES = [f"tiny-{n}" for n in (1, 2, 7, 8, 9, 63, 64, 65, 127, 129, 700)] + ["duplicates", "tight-periodic", "faces",
                                                                               "clustered"]


@pytest.fixture(scope="module")
def ctx():
    import paper_2602_19873_b200 as S
    return S.Context(0)


@pytest.mark.parametrize("geom", GEOMS, ids=lambda g: f"{g[0]}x{g[1]}w{g[2]}{'s' if g[3] else 'g'}{'c' if g[4] else 'r'}")
@pytest.mark.parametrize("name", CASES)
def test_edge_case(ctx, name, geom):
    import paper_2602_19873_b200 as S
    ci, cj, w, mode, comp = geom
    op = _case(name)
    keys, perm, sp, tree, st = P.pipeline(op, ci=ci, cj=cj, w=w, mode=mode, compress=comp)
    ps = S.ParticleSet(op.x, op.y, op.z, op.h, {"m": op.m, "q": op.q})
    box = S.SimulationBox(tuple(op.box6[:3]), tuple(op.box6[3:]), tuple(bool(v) for v in op.periodic))
    order = S.sort_by_sfc(ps, box, ctx=ctx)
    assert np.array_equal(order.keys, keys) and np.array_equal(order.perm, perm)
    gtree = S.build_octree(order, 64, ctx=ctx)
    sps = S.apply_sfc_order(ps, order, ctx=ctx)
    store = S.build_neighbor_store(sps, box, gtree, S.BuildParams(S.ClusterParams(ci, cj, w), mode, bool(comp), 1.0),
                                   ctx=ctx)
    assert np.array_equal(store.counts, st.counts)
    assert np.array_equal(store.offsets, st.offsets)
    assert np.array_equal(store.blob, st.blob)
    outs, cnt = P.reduce("density", sp, st)
    r64 = S.reduce(sps, box, store, S.sph_density_kernel(), S.PassConfig(1.0, S.F64), ctx=ctx)
    assert np.array_equal(r64.neighbor_count, cnt)
    assert np.array_equal(r64.outputs[0], outs[0])
    r32 = S.reduce(sps, box, store, S.sph_density_kernel(), S.PassConfig(1.0, S.MIXED), ctx=ctx)
    assert np.array_equal(r32.neighbor_count, cnt)
    ref = outs[0]
    nz = ref != 0
    assert np.all(r32.outputs[0][~nz] == 0)
    if nz.any():
        assert np.max(np.abs(r32.outputs[0][nz] - ref[nz]) / np.abs(ref[nz])) <= 1e-5
    if name == "duplicates":  # coincident particles: LJ raises InputError on both paths
        with pytest.raises(Exception):
            P.reduce("lj", sp, st, eps=1.0, sigma=0.01)
        for prec in (S.F64, S.MIXED):
            with pytest.raises(S.InputError, match="coincident"):
                S.reduce(sps, box, store, S.lj_kernel(1.0, 0.01), S.PassConfig(1.0, prec), ctx=ctx)
