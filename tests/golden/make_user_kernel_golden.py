"""Golden hashes for the user-pair-kernel device pass (tests/test_user_kernels.py).

Compiles tests/cpp/user_kernel_run.cpp against the UNMODIFIED reference
(/root/reference/proj/include + the reference objects oracle/Makefile builds into
oracle/_ref, namespace renamed) with g++ -ffp-contract=off, runs it, and stores the
SHA-256 of every (case, Real, kernel) section of its output: the reference's own
reduce<Real> with make_pair_kernel kernels (reduce.hpp:38-231). Needs the reference
tree, so it runs in the build container; the hashes travel with the repository."""
import glob
import hashlib
import json
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_user_kernels import sections  # noqa: E402


def main():
    objs = [o for o in sorted(glob.glob(os.path.join(ROOT, "oracle", "_ref", "*.o"))) if not o.endswith("ref_shim.o")]
    with tempfile.TemporaryDirectory() as td:
        exe, out = os.path.join(td, "uk_ref"), os.path.join(td, "uk_ref.bin")
        subprocess.run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-Dsfcnl=sfcnl_ref",
                        "-I/root/reference/proj/include", "-I" + os.path.join(ROOT, "tests", "cpp"),
                        os.path.join(ROOT, "tests", "cpp", "user_kernel_run.cpp"), *objs, "-lpthread", "-o", exe],
                       check=True)
        subprocess.run([exe, out], check=True)
        data = open(out, "rb").read()
    hashes = {name: hashlib.sha256(data[a:b]).hexdigest() for name, a, b in sections()}
    assert sections()[-1][2] == len(data), (sections()[-1][2], len(data))
    with open(os.path.join(HERE, "user_kernels.json"), "w") as f:
        json.dump({"bytes": len(data), "sha256": hashes}, f, indent=1)
    print(f"{len(hashes)} sections, {len(data)} bytes")


if __name__ == "__main__":
    main()
