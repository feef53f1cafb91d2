"""Edge cases of the GPU path against the plain-C restatement (pinned to the reference's
golden fixtures by tests/test_oracle_golden.py): tiny and ragged particle counts (partial
i-/j-clusters and super-clusters), duplicated positions (stable-sort ties, d = 0 pairs,
the LJ coincidence error), a periodic box barely twice the cutoff (every SC takes the
exact "unsafe" paths), positions exactly on the box faces (wrap), and a strongly
clustered set (deep octree, per-particle h over two decades). For each: SFC keys/perm,
store bytes bit-exact; fp64 density and LJ bit-exact; mixed density exact counts and
within 1e-5; mixed LJ exact counts, force / energy error <= 1e-5 x sum_j |term_ij|; for
8x8 / 8x4 gather, 8x8 symmetric and 1x1 geometries."""
import zlib

import numpy as np
import pytest

from oracle.oracle import Oracle, OracleError, Particles

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


def _abs_lj(sp, sigma, mode):
    """sum_j |F_ij| and sum_j |E_ij| over the neighbourhood (gather: d <= h_i; symmetric:
    d <= max(h_i, h_j)), brute force."""
    pos = np.stack([sp.x, sp.y, sp.z], 1)
    L = sp.box6[3:] - sp.box6[:3]
    per = np.array(sp.periodic, bool)
    absf, abse = np.zeros(sp.n), np.zeros(sp.n)
    for i in range(sp.n):
        d = pos[i] - pos
        d[:, per] -= L[per] * np.rint(d[:, per] / L[per])
        d2 = (d * d).sum(1)
        r = np.maximum(sp.h[i], sp.h) if mode else sp.h[i]
        ok = d2 <= r * r
        ok[i] = False
        inv2 = 1.0 / d2[ok]
        s6 = (sigma * sigma * inv2) ** 3
        absf[i] = np.sum(np.abs(24.0 * inv2 * (2 * s6 * s6 - s6)) * np.sqrt(d2[ok]))
        abse[i] = np.sum(np.abs(4.0 * (s6 * s6 - s6)))
    return absf, abse


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
    sigma = 0.3 * (1.0 / op.n) ** (1.0 / 3.0)
    try:
        lo, lcnt = P.reduce("lj", sp, st, eps=1.0, sigma=sigma)
    except OracleError as e:  # coincident pair in range (d2 == 0, e.g. across a periodic face)
        assert "coincident" in str(e)
        for prec in (S.F64, S.MIXED):
            with pytest.raises(S.InputError, match="coincident"):
                S.reduce(sps, box, store, S.lj_kernel(1.0, sigma), S.PassConfig(1.0, prec), ctx=ctx)
        lo = None
    if lo is not None:
        l64 = S.reduce(sps, box, store, S.lj_kernel(1.0, sigma), S.PassConfig(1.0, S.F64), ctx=ctx)
        assert np.array_equal(l64.neighbor_count, lcnt)
        for k in range(4):
            assert np.array_equal(l64.outputs[k], lo[k]), k
        l32 = S.reduce(sps, box, store, S.lj_kernel(1.0, sigma), S.PassConfig(1.0, S.MIXED), ctx=ctx)
        assert np.array_equal(l32.neighbor_count, lcnt)
        absf, abse = _abs_lj(sp, sigma, mode)
        err = np.sqrt(sum((l32.outputs[k] - lo[k]) ** 2 for k in range(3)))
        assert np.max(err / np.maximum(absf, 1e-300)) <= 1e-5
        assert np.max(np.abs(l32.outputs[3] - lo[3]) / np.maximum(abse, 1e-300)) <= 1e-5
    if name == "duplicates":  # coincident particles must take the error branch above
        assert lo is None


@pytest.mark.parametrize("mode", [0, 1])
def test_empty_particle_set(ctx, mode):
    """n = 0 through every stage (the reference returns a one-node octree, an empty
    store with offsets [0], empty outputs; the full list has offsets [0])."""
    import paper_2602_19873_b200 as S
    e = np.zeros(0)
    ps = S.ParticleSet(e, e, e, e, {"m": e, "q": e})
    box = S.SimulationBox((0, 0, 0), (1, 1, 1), (True, True, True))
    order = S.sort_by_sfc(ps, box, ctx=ctx)
    assert len(order.keys) == 0 and len(order.perm) == 0
    tree = S.build_octree(order, ctx=ctx)
    op = _particles(e, e, e, e, [0, 0, 0, 1, 1, 1], (1, 1, 1))
    keys, perm, sp, otree, st = P.pipeline(op, mode=mode)
    assert np.array_equal(tree.nodes["particle_end"], otree.pend)
    assert np.array_equal(tree.nodes["first_child"], otree.first_child)
    sps = S.apply_sfc_order(ps, order, ctx=ctx)
    store = S.build_neighbor_store(sps, box, tree, S.BuildParams(S.ClusterParams(8, 8, 32), mode, True, 1.0), ctx=ctx)
    assert len(store.counts) == 0 and np.array_equal(store.offsets, st.offsets) and len(store.blob) == 0
    for prec in (S.F64, S.MIXED):
        for k in (S.count_kernel(), S.sph_density_kernel(), S.lj_kernel(1.0, 0.1)):
            res = S.reduce(sps, box, store, k, S.PassConfig(1.0, prec), ctx=ctx)
            assert len(res.neighbor_count) == 0 and all(len(o) == 0 for o in res.outputs)
    if mode == 0:
        fl = S.build_full_list(ps, box, 1.0, ctx=ctx)
        assert np.array_equal(fl.offsets, np.zeros(1, np.uint64)) and len(fl.neighbors) == 0
        res = S.reduce_full(ps, box, fl, S.sph_density_kernel(), ctx=ctx)
        assert len(res.outputs[0]) == 0
