"""CPU: pin the plain-C restatement (oracle/liboracle.so) against
 (a) the reference's own known-answer tests (test_codec.cpp, test_hilbert.cpp), and
 (b) the golden fixtures produced by the compiled, unmodified reference."""
import random

import numpy as np
import pytest

from conftest import oracle_particles, oracle_store, oracle_tree
from oracle.oracle import Oracle, OracleError

P = Oracle("port")


# ---- test_codec.cpp known answers ---------------------------------------------
def test_codec_table1_golden_blocks():
    # test_codec.cpp:33-58 (logical blocks, width 6) -> serialized bytes of the same
    # sequences as index lists: indices = running sum - 1 of the differences.
    for diffs, mask, info, data in [
        ([1, 1, 1, 1, 1, 1], 0b000000, [], []),
        ([1, 2, 9, 7, 1, 1], 0b001110, [0x8, 0xF, 0xD], []),
        ([234, 1, 1, 56789, 1, 1], 0b001001, [0x1, 0x3], [0xE, 0xA, 0xD, 0xD, 0xD, 0x5]),
    ]:
        idx = np.cumsum(diffs) - 1
        enc = P.encode(idx.astype(np.uint32), 32)
        assert int.from_bytes(bytes(enc[:4]), "little") == mask
        nib = info + data
        packed = [(nib[i] | ((nib[i + 1] if i + 1 < len(nib) else 0) << 4)) for i in range(0, len(nib), 2)]
        assert list(enc[4:]) == packed
        dec, used = P.decode(enc, len(idx), 32)
        assert np.array_equal(dec, idx) and used == len(enc)


def _expected_bytes(idx, w):
    # test_codec.cpp:107-120
    diffs = [idx[0] + 1] + [int(idx[k]) - int(idx[k - 1]) for k in range(1, len(idx))] if len(idx) else []

    def bits(v):
        return 1 if v == 1 else 5 if v <= 9 else 5 + 4 * ((int(v).bit_length() + 3) // 4)
    total = 0
    for b in range(0, len(diffs), w):
        nib = sum((bits(v) - 1) // 4 for v in diffs[b:b + w])
        total += w // 8 + (nib + 1) // 2
    return total


def _random_increasing(rng, length):
    # test_codec.cpp:122-138
    v, cur = [], rng.getrandbits(64) % 1024
    for _ in range(length):
        v.append(cur)
        kind = rng.getrandbits(64) % 10
        if kind < 6:
            gap = 1
        elif kind < 8:
            gap = 2 + rng.getrandbits(64) % 8
        elif kind < 9:
            gap = 10 + rng.getrandbits(64) % 1000
        else:
            gap = 1 + rng.getrandbits(64) % 0xFFFFF
        cur += gap
        if cur > 0xFFFFFFFF:
            break
    return np.array(v, np.uint32)


@pytest.mark.parametrize("w", [32, 64])
def test_codec_roundtrip_and_size_law(w):
    rng = random.Random(123)
    cases = [np.array([0], np.uint32), np.array([0xFFFFFFFE], np.uint32), np.array([0, 0xFFFFFFFF], np.uint32),
             np.arange(w, dtype=np.uint32), (3 * np.arange(w + 1)).astype(np.uint32)]
    cases += [_random_increasing(rng, rng.getrandbits(64) % 300) for _ in range(500)]
    for v in cases:
        enc = P.encode(v, w)
        dec, used = P.decode(enc, len(v), w)
        assert np.array_equal(dec, v)
        assert used == len(enc) == _expected_bytes(v, w)


def test_codec_all_ones_and_errors():
    run = np.arange(1000, dtype=np.uint32)
    for w in (32, 64):
        assert len(P.encode(run, w)) == ((1000 + w - 1) // w) * w // 8  # test_codec.cpp:188-198
    with pytest.raises(OracleError) as e:  # first-element overflow, test_codec.cpp:210-215
        P.encode(np.array([0xFFFFFFFF], np.uint32), 32)
    assert e.value.code == 1
    v = (np.arange(40) * 1000).astype(np.uint32)  # truncation, test_codec.cpp:217-240
    enc = P.encode(v, 32)
    for keep in (0, 2, len(enc) - 1):
        with pytest.raises(OracleError) as e:
            P.decode(enc[:keep], 40, 32)
        assert e.value.code == 3
    with pytest.raises(OracleError) as e:
        P.decode(enc[:1], 40, 32)
    assert e.value.offset <= 1


# ---- test_hilbert.cpp known answers -------------------------------------------
def test_hilbert_bijection_adjacency_small_bits():
    for bits in (1, 2, 3):
        side = 1 << bits
        seen = set()
        for x in range(side):
            for y in range(side):
                for z in range(side):
                    k = P.hilbert_encode(x, y, z, bits)
                    assert k < (1 << (3 * bits))
                    seen.add(k)
                    assert P.hilbert_decode(k, bits) == (x, y, z)
        assert len(seen) == side ** 3
        prev = P.hilbert_decode(0, bits)
        for k in range(1, side ** 3):
            cur = P.hilbert_decode(k, bits)
            moved = [abs(a - b) for a, b in zip(cur, prev) if a != b]
            assert moved == [1]
            prev = cur


def test_hilbert_origin_and_random_roundtrip():
    for bits in range(1, 22):
        assert P.hilbert_encode(0, 0, 0, bits) == 0
    rng = random.Random(7)
    for _ in range(2000):
        x, y, z = (rng.getrandbits(21) for _ in range(3))
        assert P.hilbert_decode(P.hilbert_encode(x, y, z, 21), 21) == (x, y, z)


# ---- golden fixtures from the compiled reference ------------------------------
def test_port_matches_reference_fixtures(golden):
    g = golden
    ps = oracle_particles(g)
    keys, perm = P.sort_by_sfc(ps)
    assert np.array_equal(keys, g["keys"]) and np.array_equal(perm, g["perm"])
    t = P.tree(keys)
    for f in ("key_first", "key_last", "pbegin", "pend", "first_child", "depth"):
        assert np.array_equal(getattr(t, f), g[f]), f
    sp = oracle_particles(g, sorted_=True)
    ci, cj, w, mode, comp = (int(v) for v in g["params"])
    s = P.build_store(sp, oracle_tree(g), ci, cj, w, mode, comp, float(g["scale"][0]))
    assert np.array_equal(s.counts, g["counts"])
    assert np.array_equal(s.offsets, g["offsets"])
    assert np.array_equal(s.blob, g["blob"])
    st = oracle_store(g)
    for kern, nout in (("count", 1), ("density", 1), ("lj", 4)):
        outs, cnt = P.reduce(kern, sp, st, query_scale=float(g["scale"][1]), eps=1.0, sigma=float(g["scale"][2]))
        assert np.array_equal(cnt, g[f"{kern}_double_count"])
        for k in range(nout):
            # bitwise, same summation order (symmetric: the ordered j-side commit)
            assert np.array_equal(outs[k], g[f"{kern}_double_{k}"]), (kern, k, mode)
