"""CPU tests of the product's host side: the C-ABI library loads and exports
every symbol include/trigrid_b200.h declares; the host mapping functions,
closed-form DispatchStats and shard geometry match the reference's golden
vectors and the oracle; errors map to the reference's exception classes.
No compute kernel is launched (no GPU here)."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_symbols_exported(tg):
    from paper_1308_1419_b200 import _lib
    hdr = open(os.path.join(ROOT, "include", "trigrid_b200.h")).read()
    decl = set(re.findall(r"\b(tg_[a-z0-9_]+)\s*\(", hdr))
    decl -= {"tg_status", "tg_strategy", "tg_kernel", "tg_mode"}
    assert len(decl) >= 30
    L = _lib.load()
    for name in sorted(decl):
        assert hasattr(L, name), f"{name} declared in trigrid_b200.h but not exported"
    assert decl <= set(_lib.EXPORTED), decl - set(_lib.EXPORTED)
    assert L.tg_api_version() == 2


def test_sm100a_cubin_present(tg):
    import subprocess
    from paper_1308_1419_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_reference_names_mirrored(tg):
    ref_names = ["__version__", "bb_map", "count_wasted", "coverage_ok", "edm_reference", "edm_strategy",
                 "enumerate_lower", "fast_inv_sqrt", "gen_points", "grid_side_balanced", "improvement_model",
                 "isqrt", "ltm_map", "rb_map", "rb_rect", "rec_decompose", "rsqrt_single", "sqrt_via",
                 "tri_count", "tri_linear_index", "utm_map"]
    assert sorted(tg.__all__) == sorted(ref_names)
    for n in ref_names:
        assert hasattr(tg, n)


@pytest.mark.parametrize("eng", ["native", "newton", "reciprocal", "exact"])
@pytest.mark.parametrize("diag", [True, False])
def test_ltm_map_golden(tg, golden, eng, diag):
    want = golden["ltm"][f"{eng}|{int(diag)}|auto"]
    for lam, w in zip(golden["ltm_lams"], want):
        assert tg.ltm_map(lam, eng, diag) == tuple(w), lam


def test_ltm_map_exact_everywhere(tg, orc):
    # the product's g(lambda) is exact for every lambda (float guess + integer fix-up)
    rng = np.random.default_rng(0)
    for lam in [int(x) for x in rng.integers(0, 2**40, 2000)] + [2**32 - 1, 2**32, 5 * 10**11]:
        i, j = tg.ltm_map(lam, "reciprocal")
        assert i * (i + 1) // 2 + j == lam and j <= i
        i2, j2 = tg.ltm_map(lam, "reciprocal", False)
        assert i2 * (i2 - 1) // 2 + j2 == lam and j2 < i2


def test_mappers_golden(tg, golden):
    for n, e, ks, want in golden["utm"]:
        assert [list(tg.utm_map(k, n, e)) for k in ks] == want
    for n, wh, cells in golden["rb"]:
        assert list(tg.rb_rect(n)) == wh
        for tx, ty, w in cells:
            got = tg.rb_map(tx, ty, n)
            assert (list(got) if got else None) == w
    for n, rho, w in golden["rec_decompose"]:
        got = tg.rec_decompose(n, rho)
        assert (list(got) if got else None) == w
    assert tg.bb_map(3, 2) is None and tg.bb_map(2, 3) == (3, 2)


def test_scalars_golden(tg, golden):
    for v, w in golden["isqrt"]:
        assert tg.isqrt(v) == w
    for n, w in golden["grid_side_balanced"]:
        assert tg.grid_side_balanced(n) == w
    for x, it, w in golden["fast_inv_sqrt"]:
        assert np.float32(tg.fast_inv_sqrt(x, it)) == np.float32(w)
    for x, w in golden["rsqrt_single"]:
        assert np.float32(tg.rsqrt_single(x)) == np.float32(w)
    for e, x, w in golden["sqrt_via"]:
        assert tg.sqrt_via(e, x) == w
    for s, n, w in golden["count_wasted"]:
        assert tg.count_wasted(s, n) == w
    # ltm_diag_waste_blocks (engine.cpp:219-221): n / 2 as a double
    for n in (1, 2, 3, 1920, 4097, 1 << 20):
        assert tg.ltm_diag_waste_blocks(n) == n / 2.0
    for b, t, n, w in golden["improvement_model"]:
        assert tg.improvement_model(b, t, n) == w
    assert tg.tri_count(4) == 10 and tg.tri_count(1920) == 1844160 and tg.tri_count(5, False) == 10
    assert tg.tri_linear_index(2, 1) == 4
    assert tg.enumerate_lower(3) == [(0, 0), (1, 0), (1, 1), (2, 0), (2, 1), (2, 2)]
    assert tg.enumerate_lower(3, False) == [(1, 0), (2, 0), (2, 1)]


def test_dispatch_stats_golden(tg, golden):
    for s, n, rho, want in golden["stats"]:
        if want is None:
            with pytest.raises(ValueError):
                tg.dispatch_stats(s, n, rho)
            continue
        st = tg.dispatch_stats(s, n, rho)
        assert [st["blocks_launched"], st["blocks_discarded"], st["threads_discarded"]] == want, (s, n, rho)
    for s, want in golden["edm_strategy_stats"].items():
        st = tg.dispatch_stats(s, 4096, 16)
        st.pop("wall_time_ns")
        assert st == want


def test_dispatch_stats_vs_oracle_dense(tg, orc):
    for s in ("bb", "ltm-r", "utm", "rb", "rec"):
        for n in list(range(1, 70)) + [127, 128, 129, 1000]:
            for rho in (1, 3, 4, 8, 16, 32, 40):
                try:
                    _, want = orc.run_strategy(s, n, rho, mode="none")
                except ValueError:
                    with pytest.raises(ValueError):
                        tg.dispatch_stats(s, n, rho)
                    continue
                st = tg.dispatch_stats(s, n, rho)
                assert (st["blocks_launched"], st["blocks_discarded"], st["threads_discarded"]) == want, (s, n, rho)


def test_shard_geometry(tg):
    assert tg.shard_rows(65536, 16, 8) == [0, 1448, 2048, 2508, 2896, 3238, 3547, 3831, 4096]
    assert tg.shard_rows(131072, 16, 8) == [0, 2896, 4096, 5016, 5792, 6476, 7094, 7663, 8192]
    for n, rho, G in ((65536, 16, 8), (131072, 16, 4), (1000, 16, 3), (17, 4, 8), (5, 16, 2), (4096, 16, 1)):
        for diag in (True, False):
            prev = 0
            for g in range(G):
                b, e = tg.shard_elems(n, rho, g, G, diag)
                assert b == prev and e >= b
                prev = e
            assert prev == tg.tri_count(n, diag)
        # balanced within one block row of elements
        if G > 1 and n >= 65536:
            sizes = [tg.shard_elems(n, rho, g, G)[1] - tg.shard_elems(n, rho, g, G)[0] for g in range(G)]
            assert max(sizes) / min(sizes) < 1.01


def test_shard_stats_sum(tg):
    for s in ("bb", "ltm-r", "rec"):
        for n, G in ((65536, 8), (1024, 3), (4096, 2), (3072, 5)):
            tot = [0, 0, 0]
            for g in range(G):
                st = tg.dispatch_stats(s, n, 16, (g, G))
                tot = [a + st[k] for a, k in zip(tot, ("blocks_launched", "blocks_discarded", "threads_discarded"))]
            whole = tg.dispatch_stats(s, n, 16)
            # surviving tiles and filtered threads are partitioned exactly
            assert tot[0] - tot[1] == whole["blocks_launched"] - whole["blocks_discarded"]
            assert tot[2] == whole["threads_discarded"]
    # REC shards partition every pass exactly (blocks, discards, filtered threads)
    for n, G in ((65536, 8), (3072, 5)):
        whole = tg.dispatch_stats("rec", n, 16, per_pass=True)
        parts = [tg.dispatch_stats("rec", n, 16, (g, G), per_pass=True) for g in range(G)]
        for p, wp in enumerate(whole["per_pass"]):
            for k in ("blocks_launched", "blocks_discarded", "threads_discarded"):
                assert sum(q["per_pass"][p][k] for q in parts) == wp[k]
    # rb / utm shards: the span walk's own tile counts (no reference counterpart), >= 1 per non-empty shard
    for s in ("rb", "utm"):
        assert all(tg.dispatch_stats(s, 4096, 16, (g, 4))["blocks_launched"] > 0 for g in range(4))


def test_errors_mirror_reference(tg):
    with pytest.raises(TypeError):
        tg.ltm_map(-1)
    with pytest.raises(TypeError):
        tg.ltm_map(1.5)
    with pytest.raises(ValueError, match="unknown engine 'foo'"):
        tg.ltm_map(3, "foo")
    with pytest.raises(IndexError):
        tg.tri_linear_index(1, 2)
    with pytest.raises(IndexError):
        tg.utm_map(10, 4)
    with pytest.raises(IndexError):
        tg.utm_map(0, 1)
    with pytest.raises(ValueError):
        tg.rb_rect(1)
    with pytest.raises(ValueError):
        tg.count_wasted("utm", 4)
    with pytest.raises(ValueError):
        tg.count_wasted("bb", 0)
    with pytest.raises(ValueError):
        tg.improvement_model(0, 1, 1)
    with pytest.raises(ValueError):
        tg.sqrt_via("newton", 0.0)
    with pytest.raises(ValueError):
        tg.sqrt_via("exact", 2.5)
    with pytest.raises(ValueError, match="too large"):
        tg.enumerate_lower(6000)
    with pytest.raises(ValueError):
        tg.grid_side_balanced(0)
    with pytest.raises(ValueError, match="unknown strategy 'zz'"):
        tg.count_wasted("zz", 3)
    assert tg.rec_decompose(100) is None
    assert tg.rec_decompose(64, 0) is None  # the reference divides by zero here


def test_points_conversion_mirrors_pybind(tg):
    # pybind array_t<float, c_style> without forcecast: float64/int32 -> TypeError;
    # safe casts and lists convert; 1-D -> ValueError (module.cpp:29-36)
    for bad in (np.zeros((4, 2)), np.zeros((4, 2), np.int32)):
        with pytest.raises(TypeError):
            tg._points(bad)
    for ok in (np.zeros((4, 2), np.int16), np.zeros((4, 2), np.uint8), np.zeros((4, 2), np.float16),
               [[0.0, 1.0], [1.0, 2.0]], [[0, 1], [1, 2]], np.zeros((4, 4), np.float32)[:, ::2]):
        a = tg._points(ok)
        assert a.dtype == np.float32 and a.flags.c_contiguous
    with pytest.raises(ValueError, match="2-D"):
        tg._points(np.zeros(4, np.float32))
