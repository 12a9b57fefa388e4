"""The C++ drop-in (include/trigrid_b200.hpp) compiles with g++ against the
C-ABI library, its host API behaves like the reference's, and (GPU) its
launch_edm output is bit-exact with the oracle."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "shim_demo")


@pytest.fixture(scope="module")
def shim_bin(tg):
    from paper_1308_1419_b200 import _lib
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    libdir = os.path.dirname(_lib.LIB_PATH)
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "shim_demo.cpp"), "-o", BIN,
                    "-L", libdir, "-ltrigrid_b200", f"-Wl,-rpath,{libdir}"], check=True)
    return BIN


def test_shim_host(shim_bin):
    r = subprocess.run([shim_bin, "host"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "host checks ok" in r.stdout


@pytest.mark.gpu
def test_shim_launch_edm(shim_bin, orc, tmp_path):
    out = tmp_path / "edm.bin"
    r = subprocess.run([shim_bin, "edm", "2048", "3", str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    got = np.fromfile(out, dtype=np.float32)
    want = orc.edm_reference(orc.gen_points(2048, 3, 42))
    assert got.tobytes() == want.tobytes()
    assert "coverage 1" in r.stdout
