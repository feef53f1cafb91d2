"""SFC keys at the edges of the key generator's arithmetic (grid_coords(box.wrap(p)),
core.hpp:65-73 / hilbert.hpp:94-107): the CUDA key generator skips the periodic wrap's
division for in-box positions and computes the cell through a reciprocal with a guarded
fallback to the exact division near cell boundaries (csrc/sfc_sort.cu grid_axis). Keys
and the stable order must equal the restatement's bit for bit for positions on and next
to every boundary: the box faces, outside the box (periodic wrap), cell boundaries
k L / 2^bits and their neighbouring doubles, in boxes with non-power-of-two lengths."""
import numpy as np
import pytest

import paper_2602_19873_b200 as S
from oracle.oracle import Oracle, Particles

pytestmark = pytest.mark.gpu
P = Oracle("port")


@pytest.fixture(scope="module")
def ctx():
    return S.Context(0)


def _edge_positions(lo, hi, rng, n_random=4000, bits=21):
    L = hi - lo
    cells = 2 ** bits
    k = rng.integers(0, cells + 1, 3000)
    b = lo + k * (L / cells)
    pts = [lo, hi, np.nextafter(hi, -np.inf), np.nextafter(lo, np.inf), lo - 0.25 * L, hi + 0.3 * L,
           lo - L, hi + L, np.nextafter(lo, -np.inf), np.nextafter(hi, np.inf)]
    pts += list(b) + list(np.nextafter(b, np.inf)) + list(np.nextafter(b, -np.inf))
    pts += list(rng.uniform(lo - 0.5 * L, hi + 0.5 * L, n_random))
    return np.array(pts, dtype=np.float64)


@pytest.mark.parametrize("box6,periodic", [
    ((0.0, 0.0, 0.0, 1.0, 1.0, 1.0), (1, 1, 1)),
    ((-0.3, 0.1, 2.0, 0.7000000000000001, 1.3, 5.123), (1, 1, 1)),
    ((-1.7, -2.2, 0.0, 3.1, 0.9, 0.37), (1, 0, 1)),
    ((0.0, 0.0, 0.0, 3.0, 7.0, 11.0), (0, 0, 0)),
])
def test_keys_at_cell_and_box_boundaries(ctx, box6, periodic):
    rng = np.random.default_rng(17)
    lo, hi = np.array(box6[:3]), np.array(box6[3:])
    cols = []
    for d in range(3):
        v = _edge_positions(lo[d], hi[d], rng)
        if not periodic[d]:  # open axes: inside [lo, hi] (clamped by the reference's grid)
            v = np.clip(v, lo[d], hi[d])
        cols.append(v)
    n = min(len(c) for c in cols)
    x, y, z = (rng.permutation(c)[:n] for c in cols)
    h = np.full(n, 0.01)
    op = Particles(x, y, z, h, np.ones(n), np.zeros(n), np.array(box6, dtype=np.float64), tuple(periodic))
    keys, perm = P.sort_by_sfc(op)
    ps = S.ParticleSet(x, y, z, h, {})
    box = S.SimulationBox(tuple(box6[:3]), tuple(box6[3:]), tuple(bool(p) for p in periodic))
    order = S.sort_by_sfc(ps, box, ctx=ctx)
    assert np.array_equal(order.keys, keys)
    assert np.array_equal(order.perm, perm)


@pytest.mark.parametrize("nf", [0, 1, 2, 3, 5])
@pytest.mark.parametrize("n", [1, 255, 256, 257, 100003])
def test_apply_order_record_widths(ctx, nf, n):
    """apply_sfc_order (hilbert.cpp:28-44) is a gather by perm for every record width:
    4 + nf doubles per particle (the 4- and 6-wide records take the staged pack and the
    16-byte gather, the others the per-double kernels), ragged tails of the 256-particle
    pack blocks included."""
    rng = np.random.default_rng(n + nf)
    x, y, z, h = (rng.uniform(-1, 1, n) for _ in range(4))
    fields = {f"f{k}": rng.standard_normal(n) for k in range(nf)}
    perm = rng.permutation(n).astype(np.uint32)
    keys = np.arange(n, dtype=np.uint64)
    out = S.apply_sfc_order(S.ParticleSet(x, y, z, h, fields), S.SfcOrder(keys, perm, 21), ctx=ctx)
    for a, b in ((out.x, x), (out.y, y), (out.z, z), (out.h, h)):
        assert np.array_equal(a, b[perm])
    for k in range(nf):
        assert np.array_equal(out.fields[f"f{k}"], fields[f"f{k}"][perm])
