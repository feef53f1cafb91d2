"""SFNLSTOR v1 store files (neighbor_store.hpp:79-86, neighbor_store.cpp:63-152):
the Python mirror's write_store/read_store against files written by the compiled
reference's own write_store (tests/golden/*.sfnl, made by tests/golden/make_golden.py),
the reference's error behaviour, and a GPU round trip (build -> file -> set_store ->
pass)."""
import io
import os

import numpy as np
import pytest

import paper_2602_19873_b200 as S
from conftest import golden_names, load_golden

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _bp(g):
    ci, cj, w, mode, comp = (int(v) for v in g["params"])
    return S.BuildParams(S.ClusterParams(ci, cj, w), mode, bool(comp), float(g["scale"][0]))


@pytest.mark.parametrize("name", golden_names())
def test_read_reference_file(name):
    g = load_golden(name)
    st = S.read_store(os.path.join(HERE, name + ".sfnl"))
    assert st.n == len(g["x"])
    assert st.build == _bp(g)
    assert np.array_equal(st.counts, g["counts"]) and np.array_equal(st.offsets, g["offsets"])
    assert np.array_equal(st.blob, g["blob"])


@pytest.mark.parametrize("name", golden_names())
def test_write_matches_reference_bytes(name):
    g = load_golden(name)
    st = S.NeighborStore(_bp(g), len(g["x"]), g["counts"], g["offsets"], g["blob"])
    buf = io.BytesIO()
    S.write_store(st, buf)
    with open(os.path.join(HERE, name + ".sfnl"), "rb") as f:
        assert buf.getvalue() == f.read()


def test_errors_follow_reference():
    with open(os.path.join(HERE, "uniform_8x8.sfnl"), "rb") as f:
        data = f.read()
    with pytest.raises(S.DecodeError) as e:
        S.read_store(io.BytesIO(b"SFNLSTOX" + data[8:]))
    assert e.value.byte_offset == 0
    with pytest.raises(S.DecodeError) as e:
        S.read_store(io.BytesIO(data[:8] + b"\x02\x00\x00\x00" + data[12:]))
    assert e.value.byte_offset == 8
    with pytest.raises(S.DecodeError):
        S.read_store(io.BytesIO(data[:-1]))


@pytest.mark.gpu
def test_gpu_store_file_round_trip(tmp_path):
    ctx = S.Context(0)
    ps, box = S.make_uniform(S.UniformSpec(n=50000, density=50000.0, target_neighbors=120.0, seed=9))
    order = S.sort_by_sfc(ps, box, ctx=ctx)
    tree = S.build_octree(order, 64, ctx=ctx)
    sps = S.apply_sfc_order(ps, order, ctx=ctx)
    store = S.build_neighbor_store(sps, box, tree, S.BuildParams(), ctx=ctx)
    path = tmp_path / "list.sfnl"
    S.write_store(store, str(path))
    back = S.read_store(str(path))
    assert np.array_equal(back.blob, store.blob) and np.array_equal(back.offsets, store.offsets)
    a = S.reduce(sps, box, store, S.sph_density_kernel(), S.PassConfig(1.0, S.F64), ctx=ctx)
    b = S.reduce(sps, box, back, S.sph_density_kernel(), S.PassConfig(1.0, S.F64), ctx=ctx)
    assert np.array_equal(a.outputs[0], b.outputs[0]) and np.array_equal(a.neighbor_count, b.neighbor_count)
