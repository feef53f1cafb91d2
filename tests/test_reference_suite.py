"""The reference's own unit tests (proj/tests/test_*.cpp, doctest) compiled unchanged
against the B200 drop-in (include/sfcnl + libsfcnl.so) with tests/cpp/doctest.h.
Built by __graft_entry__.build() in the build container (it reads the test sources
from /root/reference); the binaries travel with the tree.

test_cluster / test_codec exercise host-side API only and run on CPU;
test_hilbert / test_octree call sort_by_sfc / build_octree / compute_node_aabbs,
which run on the GPU. test_dropin_baselines (tests/cpp, built by `make all`) checks the
drop-in's full-list / reduce_full / cluster_overhead C++ API on the GPU."""
import os
import subprocess

import pytest

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "bin")


def _run(name):
    exe = os.path.join(BIN, name)
    if not os.path.exists(exe):
        pytest.skip(f"{name} not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed checks" in r.stdout


@pytest.mark.parametrize("name", ["test_cluster", "test_codec"])
def test_reference_host_suites(name):
    _run(name)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["test_hilbert", "test_octree", "test_dropin_baselines"])
def test_reference_gpu_suites(name):
    _run(name)
