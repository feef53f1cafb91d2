"""Full Verlet list baseline: the classic per-particle CSR list and
its pass (baselines.hpp:27-129), pinned to the reference's build_full_list /
reduce_full<double> outputs in tests/golden/full_lists.npz (make_full_golden.py).

CPU: an independent numpy restatement of build_full_list (periodic_delta,
d2 <= (scale h_i)^2, gather; d2 <= (scale max(h_i, h_j))^2, symmetric) reproduces
the golden list digests.
GPU: the list derived from the compressed store (pass_full.cuh) is byte-identical to
the reference's (SHA-256 of offsets||neighbors), in SFC order and through the
unsorted-input wrapper; reduce_full precision F64 is bit-equal to reduce_full<double>
(gather and an uploaded symmetric list); precision MIXED (warp per i, tree sum) within
1e-12 relative; the reference's InputErrors are raised."""
import hashlib
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_names, golden_particles, load_golden

FULL = dict(np.load(os.path.join(GOLDEN, "full_lists.npz")))


def _digest(offsets, nbrs):
    return hashlib.sha256(np.ascontiguousarray(offsets, np.uint64).tobytes()
                          + np.ascontiguousarray(nbrs, np.uint32).tobytes()).digest()


def numpy_full_list(g, sorted_, scale, mode):
    """baselines.cpp:39-131 restated: for each i every j != i with
    |periodic_delta(x_i, x_j)|^2 <= r^2, ascending j (test infrastructure)."""
    idx = g["perm"] if sorted_ else slice(None)
    pos = np.stack([g["x"][idx], g["y"][idx], g["z"][idx]], 1)
    h = g["h"][idx]
    L = g["box6"][3:] - g["box6"][:3]
    per = np.array(g["periodic"], bool)
    n = len(h)
    offsets = np.zeros(n + 1, np.uint64)
    rows = []
    for i in range(n):
        d = pos[i] - pos
        d[:, per] -= L[per] * np.rint(d[:, per] / L[per])
        d2 = d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1] + d[:, 2] * d[:, 2]
        r = scale * (np.maximum(h[i], h) if mode else h[i])
        ok = d2 <= r * r
        ok[i] = False
        js = np.nonzero(ok)[0].astype(np.uint32)
        rows.append(js)
        offsets[i + 1] = offsets[i] + len(js)
    return offsets, np.concatenate(rows) if rows else np.zeros(0, np.uint32)


@pytest.mark.parametrize("name", ["uniform_1x1", "uniform_symmetric", "uniform_8x4_w64_raw"])
def test_numpy_restatement_matches_reference_digest(name):
    g = load_golden(name)
    scale, mode = float(g["scale"][0]), int(g["params"][3])
    for order in ("sorted", "orig"):
        off, nb = numpy_full_list(g, order == "sorted", scale, mode)
        assert len(nb) == int(FULL[f"{name}.{order}.pairs"][0])
        assert _digest(off, nb) == FULL[f"{name}.{order}.sha"].tobytes(), (name, order)


# ------------------------------------------------------------------------ GPU
GATHER_CASES = [n for n in golden_names() if n != "uniform_symmetric"]


@pytest.fixture(scope="module")
def ctx():
    import paper_2602_19873_b200 as S
    return S.Context(0)


def _kernels(S, sigma):
    return (("count", S.count_kernel()), ("density", S.sph_density_kernel()), ("lj", S.lj_kernel(1.0, sigma)))


@pytest.mark.gpu
@pytest.mark.parametrize("name", GATHER_CASES)
def test_gpu_full_list_matches_reference(ctx, name):
    import paper_2602_19873_b200 as S
    g = load_golden(name)
    scale, qs, sigma = (float(v) for v in g["scale"])
    for order in ("sorted", "orig"):
        ps, box = golden_particles(g, sorted_=order == "sorted")
        key = f"{name}.{order}"
        fl = S.build_full_list(ps, box, scale, ctx=ctx)
        assert len(fl.neighbors) == int(FULL[key + ".pairs"][0])
        assert _digest(fl.offsets, fl.neighbors) == FULL[key + ".sha"].tobytes(), key
        assert fl.memory_bytes() == 8 * (len(g["x"]) + 1) + 4 * len(fl.neighbors)
        for kern, k in _kernels(S, sigma):
            res = S.reduce_full(ps, box, fl, k, S.PassConfig(qs, S.F64), ctx=ctx)
            assert np.array_equal(res.neighbor_count, FULL[f"{key}.{kern}.count"]), (key, kern)
            for o in range(len(k.names)):
                assert np.array_equal(res.outputs[o], FULL[f"{key}.{kern}.{o}"]), (key, kern, o)
            res = S.reduce_full(ps, box, fl, k, S.PassConfig(qs, S.MIXED), ctx=ctx)
            assert np.array_equal(res.neighbor_count, FULL[f"{key}.{kern}.count"]), (key, kern)
            for o in range(len(k.names)):
                ref = FULL[f"{key}.{kern}.{o}"]
                np.testing.assert_allclose(res.outputs[o], ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


@pytest.mark.gpu
def test_gpu_full_list_device_path_and_query_scale(ctx):
    """Context-level path on the sorted slot (store -> list stays on the device), a
    build scale below the store's, and a query scale below the list's."""
    import paper_2602_19873_b200 as S
    g = load_golden("jitter_skin")  # store build scale 1.2
    ps, box = golden_particles(g, sorted_=True)
    n = len(ps.x)
    ctx.set_particles(ps, box)  # already in SFC order: the sort is the identity
    ctx.sort()
    ctx.apply_order()
    ctx.octree(64)
    ctx.build_store(S.BuildParams(S.ClusterParams(8, 8, 32), S.GATHER, True, 1.2))
    for scale in (1.2, 1.0):
        pairs = ctx.build_full_list(scale)
        fl = ctx.get_full_list(n, pairs, scale)
        off, nb = numpy_full_list(g, True, scale, 0)
        assert np.array_equal(fl.offsets, off) and np.array_equal(fl.neighbors, nb), scale
    res = ctx.reduce_full(S.count_kernel(), S.PassConfig(1.0, S.F64), n)
    assert np.array_equal(res.neighbor_count, FULL["jitter_skin.sorted.count.count"])
    with pytest.raises(S.InputError, match="query_scale exceeds the list's build scale"):
        ctx.reduce_full(S.count_kernel(), S.PassConfig(1.1, S.F64), n)
    with pytest.raises(S.InputError, match="build_scale exceeds"):
        ctx.build_full_list(1.3)


@pytest.mark.gpu
def test_gpu_reduce_full_symmetric_uploaded_list(ctx):
    import paper_2602_19873_b200 as S
    g = load_golden("uniform_symmetric")
    scale, qs, sigma = (float(v) for v in g["scale"])
    ps, box = golden_particles(g, sorted_=True)
    off, nb = numpy_full_list(g, True, scale, 1)
    assert _digest(off, nb) == FULL["uniform_symmetric.sorted.sha"].tobytes()
    fl = S.FullVerletList(S.SYMMETRIC, scale, off, nb)
    for kern, k in _kernels(S, sigma):
        res = S.reduce_full(ps, box, fl, k, S.PassConfig(qs, S.F64), ctx=ctx)
        assert np.array_equal(res.neighbor_count, FULL[f"uniform_symmetric.sorted.{kern}.count"])
        for o in range(len(k.names)):
            assert np.array_equal(res.outputs[o], FULL[f"uniform_symmetric.sorted.{kern}.{o}"]), (kern, o)
    bad = S.FullVerletList(S.GATHER, scale, off[:-1], nb)
    with pytest.raises(S.InputError, match="list/particle-set mismatch"):
        S.reduce_full(ps, box, bad, S.count_kernel(), ctx=ctx)


@pytest.mark.gpu
@pytest.mark.parametrize("name", GATHER_CASES)
def test_gpu_cluster_overhead_matches_reference(ctx, name):
    """bench::cluster_overhead (bench.cpp:93-122) from the device slot count."""
    import paper_2602_19873_b200 as S
    g = load_golden(name)
    ci, cj, w, mode, comp = (int(v) for v in g["params"])
    store = S.NeighborStore(S.BuildParams(S.ClusterParams(ci, cj, w), mode, bool(comp), float(g["scale"][0])),
                            len(g["x"]), g["counts"], g["offsets"], g["blob"])
    pairs = int(FULL[f"{name}.sorted.count.count"].astype(np.int64).sum())
    assert S.cluster_overhead(store, pairs, ctx=ctx) == float(FULL[name + ".overhead"][0])
    with pytest.raises(S.InputError, match="no in-range pairs"):
        S.cluster_overhead(store, 0, ctx=ctx)


def test_cluster_overhead_rejects_symmetric_store():
    import paper_2602_19873_b200 as S
    g = load_golden("uniform_symmetric")
    store = S.NeighborStore(S.BuildParams(S.ClusterParams(8, 8, 32), S.SYMMETRIC, True, 1.0), len(g["x"]),
                            g["counts"], g["offsets"], g["blob"])
    with pytest.raises(S.InputError, match="requires a gather-mode store"):
        S.cluster_overhead(store, 1)
