"""The reference's OWN C++ callers, compiled UNMODIFIED against the drop-in.

/root/reference/proj/src/bench.cpp (run_suite, emit_csv) and
/root/reference/proj/src/checks.cpp (verify_strategies, check_cell_coverage,
ltm_exactness_sweep) are compiled with -I include/trigrid_compat, whose
trigrid/{tri,fastmath,strategies,edm,engine}.hpp put include/trigrid_b200.hpp
into namespace trigrid, and linked with libtrigrid_b200.so
(tests/cpp/ref_callers_main.cpp drives them).  The build needs
/root/reference, so it happens here (CPU container); the binary travels to
the GPU box, where the -m gpu tests run it.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "ref_callers")
REF = "/root/reference/proj"


def build_ref_callers() -> str:
    from paper_1308_1419_b200 import _lib, build
    build.build()
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    libdir = os.path.dirname(_lib.LIB_PATH)
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include", "trigrid_compat"),
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(REF, "include"),
           os.path.join(ROOT, "tests", "cpp", "ref_callers_main.cpp"),
           os.path.join(REF, "src", "bench.cpp"), os.path.join(REF, "src", "checks.cpp"),
           "-o", BIN + ".tmp", "-L", libdir, "-ltrigrid_b200",
           "-Wl,-rpath,$ORIGIN/../../../paper_1308_1419_b200"]
    subprocess.run(cmd, check=True)
    os.replace(BIN + ".tmp", BIN)
    return BIN


@pytest.fixture(scope="module")
def ref_callers():
    if os.path.isdir(REF):
        return build_ref_callers()
    if not os.path.exists(BIN):
        pytest.skip("reference sources absent and no prebuilt tests/cpp/_build/ref_callers")
    return BIN


def test_reference_callers_compile_unmodified(ref_callers):
    assert os.path.exists(ref_callers)


@pytest.mark.gpu
def test_verify_strategies_all(ref_callers):
    """checks.cpp verify_strategies("all", 256, 16): 18 lines, all ok
    (coverage sweeps of every strategy at rho 16 and 1 on the GPU, every REC
    (m, k) schedule, g(lambda) block bijections per engine)."""
    r = subprocess.run([ref_callers, "verify", "all", "256", "16"], capture_output=True, text=True, timeout=1200)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith(("ok ", "FAIL"))]
    assert r.returncode == 0, r.stdout + r.stderr
    assert len(lines) == 18 and all(ln.startswith("ok ") for ln in lines), r.stdout


@pytest.mark.gpu
def test_run_suite_edm(ref_callers, tmp_path):
    """bench.cpp run_suite over all seven strategies, EDM d=3, N in
    {1024, 2048, 4096}: every strategy verified against edm_reference before
    timing (bench.cpp:80-108), CSV in the reference schema."""
    csv = tmp_path / "suite.csv"
    r = subprocess.run([ref_callers, "suite", "edm", str(csv), "1024", "2048", "4096"], capture_output=True,
                       text=True, timeout=1200)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all_verified 1" in r.stdout
    rows = csv.read_text().splitlines()
    assert rows[0].startswith("strategy,N,rho,d,kernel,repetition,wall_time_ns")
    body = [x.split(",") for x in rows[1:]]
    assert {b[0] for b in body} == {"bb", "ltm-x", "ltm-n", "ltm-r", "utm", "rb", "rec"}
    assert all(b[11] == "passed" for b in body)  # N <= verify_cap: every row oracle-checked


@pytest.mark.gpu
def test_run_suite_dummy(ref_callers, tmp_path):
    csv = tmp_path / "dummy.csv"
    r = subprocess.run([ref_callers, "suite", "dummy", str(csv), "1024", "65536"], capture_output=True, text=True,
                       timeout=1200)
    assert r.returncode == 0, r.stdout + r.stderr
    assert len(csv.read_text().splitlines()) == 1 + 2 * 7 * 3


@pytest.mark.gpu
def test_rec_per_pass_through_launch_count(ref_callers):
    r = subprocess.run([ref_callers, "perpass", "65536", "16"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    passes = [ln.split() for ln in r.stdout.splitlines() if ln.startswith("pass ")]
    assert len(passes) == 13  # (m, k) = (16, 12): 12 square levels + the diagonal pass
    assert all(int(p[4]) > 0 for p in passes)
    assert "bad 0" in r.stdout


def test_exactness_sweep_host(ref_callers, golden):
    """ltm_exactness_sweep (checks.cpp:81-95) through the drop-in's host
    ltm_map(RepairPolicy::Off): identical counts to the reference's own run."""
    r = subprocess.run([ref_callers, "sweep", "2048"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    names = {"native-single": "native", "newton-raphson": "newton", "reciprocal": "reciprocal",
             "exact-integer": "exact"}
    for ln in r.stdout.splitlines():
        v, diag, checked, mism, first = ln.split()
        want = golden["exactness"][f"2048|{names[v]}|{diag}"]
        assert [int(checked), int(mism), int(first)] == want, ln
