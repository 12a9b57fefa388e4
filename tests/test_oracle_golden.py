"""Pin the oracle restatement (oracle/trigrid_oracle.c) against golden vectors
produced by the UNMODIFIED reference (tests/golden/make_golden.py).  Runs on
CPU everywhere (also where /root/reference is absent)."""
import hashlib

import numpy as np
import pytest

ENG = ["native", "newton", "reciprocal", "exact"]


@pytest.mark.parametrize("eng", ENG)
@pytest.mark.parametrize("diag", [True, False])
@pytest.mark.parametrize("rep", ["auto", "off"])
def test_ltm_map_golden(orc, golden, eng, diag, rep):
    lams = golden["ltm_lams"]
    want = golden["ltm"][f"{eng}|{int(diag)}|{rep}"]
    got = [orc.ltm_map(l, eng, diag, rep) for l in lams]
    bad = [(l, g, tuple(w)) for l, g, w in zip(lams, got, want) if g != tuple(w)]
    assert not bad, bad[:5]


def test_exactness_golden(orc, golden):
    import ctypes as C
    for key, want in golden["exactness"].items():
        n, e, diag = key.split("|")
        c, m, f = C.c_uint64(), C.c_uint64(), C.c_uint64()
        orc.lib().or_ltm_exactness_sweep(int(n), orc.ENGINES[e], int(diag), C.byref(c), C.byref(m), C.byref(f))
        assert [c.value, m.value, f.value] == want, key


def test_exactness_known_breakpoints(golden):
    # float-only ltm-r breaks first at 2,110,485 (n=4096 sweep)
    ex = golden["exactness"]
    assert ex["1920|reciprocal|1"][1] == 0 and ex["1920|newton|1"][1] == 0
    assert ex["4096|reciprocal|1"][2] == 2110485
    assert ex["4096|newton|1"][2] == 1884711


def test_utm_golden(orc, golden):
    for n, e, ks, want in golden["utm"]:
        got = [list(orc.utm_map(k, n, e)) for k in ks]
        assert got == want, (n, e)


def test_rb_golden(orc, golden):
    for n, wh, cells in golden["rb"]:
        for tx, ty, want in cells:
            got = orc.rb_map(tx, ty, n)
            assert (list(got) if got else None) == want, (n, tx, ty)


def test_rec_decompose_golden(orc, golden):
    for n, rho, want in golden["rec_decompose"]:
        got = orc.rec_decompose(n, rho)
        assert (list(got) if got else None) == want


def test_scalars_golden(orc, golden):
    L = orc.lib()
    for v, want in golden["isqrt"]:
        assert L.or_isqrt(v) == want
    for n, want in golden["grid_side_balanced"]:
        assert L.or_grid_side_balanced(n) == want
    for x, it, want in golden["fast_inv_sqrt"]:
        assert np.float32(L.or_fast_inv_sqrt(x, it)) == np.float32(want)
    for x, want in golden["rsqrt_single"]:
        assert np.float32(L.or_rsqrt_single(x)) == np.float32(want)
    import ctypes as C
    ok = C.c_int()
    for e, x, want in golden["sqrt_via"]:
        assert L.or_sqrt_via(orc.ENGINES[e], x, C.byref(ok)) == want and ok.value
    for s, n, want in golden["count_wasted"]:
        assert L.or_count_wasted(int(s != "bb"), n) == want
    for b, t, n, want in golden["improvement_model"]:
        assert L.or_improvement_model(b, t, n) == pytest.approx(want, rel=0, abs=0)


def test_stats_golden(orc, golden):
    for s, n, rho, want in golden["stats"]:
        try:
            _, st = orc.run_strategy(s, n, rho, mode="none")
        except ValueError:
            st = None
        assert (list(st) if st else None) == want, (s, n, rho)


def test_coverage_golden(orc, golden):
    for s, n, rho, want in golden["coverage_ok"]:
        cnt, _ = orc.run_strategy(s, n, rho, mode="count")
        T = np.repeat(np.arange(n), np.arange(1, n + 1))
        jj = np.arange(cnt.size) - np.repeat(np.arange(n) * (np.arange(n) + 1) // 2, np.arange(1, n + 1))
        expect = np.where((jj == T) & (s == "utm"), 0, 1)
        assert bool((cnt == expect).all()) == want, (s, n, rho)


def test_gen_points_golden(orc, golden):
    for key, head in golden["gen_points_head"].items():
        n, d = map(int, key.split("|"))
        assert orc.gen_points(n, d, 42).ravel()[:16].tolist() == head


@pytest.mark.parametrize("n", [1, 2, 3, 17, 64, 256, 1024, 4096])
@pytest.mark.parametrize("d", [1, 2, 3, 4])
def test_edm_reference_sha(orc, golden, n, d):
    e = orc.edm_reference(orc.gen_points(n, d, 42))
    assert hashlib.sha256(e.tobytes()).hexdigest() == golden["edm_sha256"][f"{n}|{d}"]


def test_edm_d64_and_kat(orc, golden):
    pts64 = orc.gen_points(16 * 128, 4, 42).reshape(128, 64)
    assert np.array_equal(pts64, orc.gen_points(128, 64, 42))  # shape-invariant stream
    e = orc.edm_reference(pts64)
    assert hashlib.sha256(e.tobytes()).hexdigest() == golden["edm_sha256"]["128|64"]
    kat = orc.edm_reference(np.array([[0.0], [1.0], [2.0]], np.float32))
    assert kat.tolist() == golden["edm_kat"] == [0, 1, 0, 2, 1, 0]


def test_edm_rows_match_reference(orc):
    pts = orc.gen_points(300, 3, 7)
    full = orc.edm_reference(pts)
    T = lambda i: i * (i + 1) // 2  # noqa: E731
    assert np.array_equal(orc.edm_rows(pts, 100, 180), full[T(100):T(180)])
    ci = np.array([5, 299, 150], np.uint64)
    cj = np.array([0, 299, 17], np.uint64)
    assert np.array_equal(orc.edm_cells(pts, ci, cj), full[(ci * (ci + 1) // 2 + cj).astype(np.int64)])


def test_edm_strategy_stats_golden(orc, golden):
    for s, want in golden["edm_strategy_stats"].items():
        _, st = orc.run_strategy(s, 4096, 16, mode="none")
        assert list(st) == [want["blocks_launched"], want["blocks_discarded"], want["threads_discarded"]]
    assert golden["edm_strategy_stats"]["ltm-r"] == {"blocks_launched": 33124, "blocks_discarded": 228,
                                                    "threads_discarded": 30720}


def test_write_reference(orc):
    for n in (1, 5, 64, 100):
        w, _ = orc.run_strategy("ltm-r", n, 4, mode="write")
        assert np.array_equal(w, orc.write_reference(n))


def test_collide_reference_semantics(orc):
    # brute-force restatement in numpy float32 (no FMA: numpy ops round per op)
    sph = orc.gen_points(200, 4, 42)
    r_max = np.float32(0.0625)
    bits, hits = orc.collide_reference(sph, float(r_max))
    x = sph
    want = []
    for i in range(1, 200):
        for j in range(i):
            d = x[i, :3] - x[j, :3]
            s = np.float32(np.float32(d[0] * d[0] + d[1] * d[1]) + d[2] * d[2])
            rr = np.float32(x[i, 3] * r_max + x[j, 3] * r_max)
            want.append(s <= np.float32(rr * rr))
    want = np.array(want)
    got = np.unpackbits(bits, bitorder="little")[: want.size].astype(bool)
    assert np.array_equal(got, want) and hits == int(want.sum())
    u8, h2 = orc.collide_rows_u8(sph, float(r_max), 50, 120)
    off = 50 * 49 // 2
    assert h2 == int(u8.sum()) and np.array_equal(u8.astype(bool), want[off: off + u8.size])
