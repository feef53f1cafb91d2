"""Malformed stores on every pass path: the GPU raises DecodeError with the same
message kind and byte offset as the compiled reference (DecodeError{byte_offset},
core.hpp:28-33; decode_entry_indices neighbor_store.cpp:18-42, codec::decode_into
nibble_codec.cpp:136-178). Corruptions: an index stream cut short, trailing bytes in a
super-cluster's slice, a slice too short for its mask records. Paths: fp64 and mixed
precision, 8x8 / 8x4 gather, 8x8 symmetric, 1x1."""
import numpy as np
import pytest

from oracle.oracle import Oracle, OracleError, available

pytestmark = pytest.mark.gpu
GEOMS = [(8, 8, 32, 0, 1), (8, 4, 64, 0, 1), (8, 8, 32, 1, 1), (1, 1, 32, 0, 1), (8, 8, 32, 0, 0)]


def _setup(ctx, geom):
    import paper_2602_19873_b200 as S
    ci, cj, w, mode, comp = geom
    ps, box = S.make_uniform(S.UniformSpec(n=5000, density=5000.0, target_neighbors=60.0, seed=13))
    order = S.sort_by_sfc(ps, box, ctx=ctx)
    tree = S.build_octree(order, ctx=ctx)
    sps = S.apply_sfc_order(ps, order, ctx=ctx)
    bp = S.BuildParams(S.ClusterParams(ci, cj, w), mode, bool(comp), 1.0)
    return sps, box, S.build_neighbor_store(sps, box, tree, bp, ctx=ctx)


def _corrupt(store, how):
    import paper_2602_19873_b200 as S
    sc = int(np.argmax(store.counts))
    offs, blob = store.offsets.copy(), store.blob.copy()
    e = int(offs[sc + 1])
    if how == "truncated":  # the SC's index stream loses its last 3 bytes
        blob = np.delete(blob, slice(e - 3, e))
        offs[sc + 1:] -= 3
    elif how == "trailing":  # two extra bytes after the SC's index stream
        blob = np.insert(blob, e, np.array([0x55, 0xAA], np.uint8))
        offs[sc + 1:] += 2
    elif how == "masks":  # the slice cannot hold its mask records
        counts = store.counts.copy()
        counts[sc] = np.uint32(int(offs[sc + 1] - offs[sc]) + 5)
        return S.NeighborStore(store.build, store.n, counts, offs, blob), sc
    return S.NeighborStore(store.build, store.n, store.counts, offs, blob), sc


def _ref_error(sps, box, store, kern):
    from oracle.oracle import Particles
    R = Oracle("reference")
    b = store.build
    st = type("St", (), {})()
    from oracle.oracle import Store
    st = Store(store.n, b.params.ci, b.params.cj, b.params.w, int(b.mode), int(b.compress), b.build_radius_scale,
               np.ascontiguousarray(store.counts, np.uint32), np.ascontiguousarray(store.offsets, np.uint64),
               np.ascontiguousarray(store.blob, np.uint8))
    p = Particles(sps.x, sps.y, sps.z, sps.h, sps.fields["m"], sps.fields["q"],
                  np.array(list(box.lo) + list(box.hi)), tuple(int(v) for v in box.periodic))
    with pytest.raises(OracleError) as ei:
        R.reduce(kern, p, st, eps=1.0, sigma=0.01)
    return ei.value


@pytest.mark.skipif(not available("reference"), reason="oracle/_ref not built")
@pytest.mark.parametrize("how", ["truncated", "trailing", "masks"])
@pytest.mark.parametrize("geom", GEOMS, ids=lambda g: f"{g[0]}x{g[1]}w{g[2]}{'s' if g[3] else 'g'}{'c' if g[4] else 'r'}")
def test_decode_errors_match_reference(geom, how):
    import paper_2602_19873_b200 as S
    ctx = S.Context(0)
    sps, box, store = _setup(ctx, geom)
    bad, sc = _corrupt(store, how)
    for kname, kern in (("count", S.count_kernel()), ("density", S.sph_density_kernel()), ("lj", S.lj_kernel(1.0, 0.01))):
        ref = _ref_error(sps, box, bad, kname)
        for prec in (S.F64, S.MIXED):
            with pytest.raises(S.DecodeError) as ei:
                S.reduce(sps, box, bad, kern, S.PassConfig(1.0, prec), ctx=ctx)
            assert ei.value.byte_offset == ref.offset, (kname, prec, str(ei.value), ref.msg)
