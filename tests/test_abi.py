"""CPU: the C-ABI library loads and exports every symbol include/sfcnl_cu.h declares,
and its host-side functions (codec, Hilbert keys, generators) agree bit for bit with
the oracle (which itself is pinned to the reference, tests/test_oracle_golden.py)."""
import os
import random
import re
import subprocess

import numpy as np
import pytest

import paper_2602_19873_b200 as S
from paper_2602_19873_b200 import _native
from oracle.oracle import Oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = Oracle("port")


def _declared():
    hdr = open(os.path.join(ROOT, "include", "sfcnl_cu.h")).read()
    return sorted(set(re.findall(r"\b(sfcnl_(?:cu_)?[a-z_0-9]+)\s*\(", hdr)))


def test_header_matches_binding_list():
    assert _declared() == sorted(_native.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = _native.lib()
    for name in _declared():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [s for s in _declared() if s not in exported]
    assert not missing, missing


def test_dropin_library_exports_reference_api():
    lib = os.path.join(ROOT, "paper_2602_19873_b200", "libsfcnl.so")
    if not os.path.exists(lib):
        pytest.skip("libsfcnl.so not built")
    out = subprocess.run(["nm", "-DC", "--defined-only", lib], capture_output=True, text=True).stdout
    for sym in ["sfcnl::sort_by_sfc(", "sfcnl::apply_sfc_order(", "sfcnl::build_octree(",
                "sfcnl::compute_node_aabbs(", "sfcnl::build_neighbor_store(", "sfcnl::gpu::run_pass(",
                "sfcnl::codec::encode(", "sfcnl::codec::decode_into(", "sfcnl::read_store(",
                "sfcnl::write_store(", "sfcnl::make_uniform(", "sfcnl::make_evrard("]:
        assert sym in out, sym


def test_no_gpu_means_loud_failure():
    """The product path has no CPU fallback: without a B200, creating a context fails."""
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("GPU present")
    with pytest.raises(_native.CudaError):
        S.Context(0)


@pytest.mark.parametrize("w", [32, 64])
def test_host_codec_matches_oracle(w):
    rng = np.random.default_rng(5)
    for _ in range(300):
        v = np.unique(rng.integers(0, 1 << 20, rng.integers(0, 400))).astype(np.uint32)
        enc = S.encode(v, w)
        assert np.array_equal(enc, P.encode(v, w))
        assert np.array_equal(S.decode(enc, len(v), w), v)
    with pytest.raises(S.InputError):
        S.encode(np.array([5, 3], np.uint32), w)
    v = (np.arange(50) * 7).astype(np.uint32)
    enc = S.encode(v, w)
    for keep in range(0, len(enc) - 1, 3):  # truncation -> DecodeError with the oracle's offset
        with pytest.raises(S.DecodeError) as e:
            S.decode(enc[:keep], len(v), w)
        try:
            P.decode(enc[:keep], len(v), w)
        except Exception as oe:  # noqa: BLE001
            assert e.value.byte_offset == oe.offset


def test_host_hilbert_matches_oracle():
    for bits in (1, 2, 3):
        for x in range(1 << bits):
            for y in range(1 << bits):
                for z in range(1 << bits):
                    k = S.hilbert_encode(x, y, z, bits)
                    assert k == P.hilbert_encode(x, y, z, bits)
                    assert S.hilbert_decode(k, bits) == (x, y, z)
    r = random.Random(7)
    for _ in range(5000):
        x, y, z = (r.getrandbits(21) for _ in range(3))
        k = S.hilbert_encode(x, y, z, 21)
        assert k == P.hilbert_encode(x, y, z, 21)
        assert S.hilbert_decode(k, 21) == (x, y, z)
    with pytest.raises(S.InputError):
        S.hilbert_encode(8, 0, 0, 3)


def test_generators_match_oracle():
    ps, box = S.make_uniform(S.UniformSpec(n=4000, density=4000.0, target_neighbors=80.0, h_jitter=0.2, seed=9))
    q = P.make_uniform(4000, 4000.0, 80.0, (1, 1, 1), 0.2, 9)
    for f in "xyzh":
        assert np.array_equal(getattr(ps, f), getattr(q, f))
    assert np.array_equal(ps.fields["q"], q.q)
    ps, box = S.make_evrard(S.EvrardSpec(n=3000, target_neighbors=70.0, seed=4))
    q = P.make_evrard(3000, 70.0, False, (0, 0, 0), 4)
    for f in "xyzh":
        assert np.array_equal(getattr(ps, f), getattr(q, f))
    assert np.array_equal(ps.fields["m"], q.m)
    assert box.lo == (-1.1, -1.1, -1.1)


def test_python_mirror_validation_errors():
    with pytest.raises(S.InputError):
        S.ClusterParams(8, 3)
    with pytest.raises(S.InputError):
        S.ClusterParams(4, 8)
    with pytest.raises(S.InputError):
        S.ClusterParams(8, 8, 16)
    with pytest.raises(S.InputError):
        S.BuildParams(S.ClusterParams(), S.GATHER, True, 0.5)
    with pytest.raises(S.InputError):
        S.SimulationBox((0, 0, 0), (1, 0, 1))
    assert S.ClusterParams(1, 1).mask_bytes_per_entry() == 8
