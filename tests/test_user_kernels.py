"""User pair kernels (make_pair_kernel / BasicPairKernel, pair_kernel.hpp:60-91) on the
B200: reduce<Real, K> with a kernel that is not built in runs the generic device pass
(include/sfcnl/gpu_pair_kernel.cuh) instantiated in the caller's CUDA translation unit.
tests/cpp/user_kernel_run.cpp (compiled by nvcc with -fmad=false against the drop-in)
runs three kernels -- a weighted sum over an input field, min / max reductions, a
postamble -- in double and float on five stores (8x8, 8x4 w64 with a skin and a query
scale below it, Evrard in an open box, 1x1, raw), and every output and neighbour count
must equal, bit for bit, what the unmodified reference's reduce<Real> computes with the
same kernels (SHA-256 per section, tests/golden/user_kernels.json from
tests/golden/make_user_kernel_golden.py)."""
import hashlib
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "bin", "test_dropin_user_kernels")
CASES = [("uniform8x8", 20000), ("uniform8x4_skin", 20011), ("evrard8x8", 12000), ("uniform1x1", 3001),
         ("uniform8x8_raw", 9000)]
KERNELS = [("weighted", 2), ("minmax", 2), ("post", 1)]


def sections():
    """(name, begin, end) of every (case, Real, kernel) block of the runner's output."""
    out, at = [], 0
    for case, n in CASES:
        for real, size in (("double", 8), ("float", 4)):
            for k, no in KERNELS:
                nb = no * n * size + 4 * n
                out.append((f"{case}/{real}/{k}", at, at + nb))
                at += nb
    return out


@pytest.mark.gpu
def test_user_kernels_bit_equal_to_reference(tmp_path):
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "user_kernels.json")))
    out = tmp_path / "uk.bin"
    r = subprocess.run([BIN, str(out)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    data = out.read_bytes()
    assert len(data) == gold["bytes"]
    bad = [name for name, a, b in sections() if hashlib.sha256(data[a:b]).hexdigest() != gold["sha256"][name]]
    assert not bad, bad


def test_user_kernel_runner_built():
    assert os.path.exists(BIN), "tests/cpp/bin/test_dropin_user_kernels not built (make -C paper_2602_19873_b200)"
