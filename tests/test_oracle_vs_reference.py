"""Pin the oracle restatement against the reference itself, compiled from its
own sources (oracle/_ref).  Skipped where the reference was not built (the
GPU box); tests/test_oracle_golden.py covers that case with fixtures."""
import ctypes as C

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def _p(a, t=C.c_uint64):
    return a.ctypes.data_as(C.POINTER(t))


@pytest.mark.parametrize("eng", ["native", "newton", "reciprocal", "exact"])
@pytest.mark.parametrize("diag", [1, 0])
@pytest.mark.parametrize("rep", ["auto", "off"])
def test_ltm_map_bulk(orc, eng, diag, rep):
    R = oracle.ref()
    for l0, cnt in ((0, 2_200_000), (33_000_000, 200_000), (2**31, 50_000)):
        a = orc.ltm_map_range(l0, cnt, eng, bool(diag), rep)
        bi, bj = np.empty(cnt, np.uint64), np.empty(cnt, np.uint64)
        R.ref_ltm_map_range(l0, cnt, oracle.ENGINES[eng], diag, oracle.REPAIR[rep], _p(bi), _p(bj))
        assert np.array_equal(a[0], bi) and np.array_equal(a[1], bj)


@pytest.mark.parametrize("strat", ["bb", "ltm-x", "ltm-n", "ltm-r", "utm", "rb", "rec"])
def test_engine_counts_and_stats(orc, strat):
    R = oracle.ref()
    for n in (1, 2, 3, 15, 16, 17, 31, 64, 100, 256, 300, 512):
        for rho in (16, 1, 4, 5):
            try:
                cnt, st = orc.run_strategy(strat, n, rho)
            except ValueError:
                st = None
            c = np.zeros(orc.tri_count(n), np.uint32)
            s = np.zeros(4, np.uint64)
            rc = R.ref_launch_count(strat.encode(), n, rho, 1, _p(c, C.c_uint32), _p(s))
            if rc:
                assert st is None
                continue
            assert tuple(int(x) for x in s[:3]) == st
            assert np.array_equal(c, cnt)


def test_gen_points_and_edm(orc):
    R = oracle.ref()
    for n, d in ((1000, 3), (333, 4), (2048, 1), (777, 2)):
        a = orc.gen_points(n, d, 99)
        b = np.empty((n, d), np.float32)
        R.ref_gen_points(n, d, 99, _p(b, C.c_float))
        assert np.array_equal(a, b)
        ea = orc.edm_reference(a)
        eb = np.empty_like(ea)
        R.ref_edm_reference(_p(b, C.c_float), n, d, _p(eb, C.c_float))
        assert ea.tobytes() == eb.tobytes()


def test_verify_strategies_reference_green():
    # the reference's own self-check (checks.cpp:177-206) passes on its build
    assert oracle.ref().ref_verify_strategies(b"all", 64, 16) == 1


def test_utm_bulk(orc):
    R = oracle.ref()
    for n in (2, 7, 64, 1000):
        cnt = n * (n - 1) // 2
        a, b = np.empty(cnt, np.uint64), np.empty(cnt, np.uint64)
        assert R.ref_utm_map_range(0, cnt, n, 1, _p(a), _p(b)) == 0
        got = np.array([orc.utm_map(k, n) for k in range(cnt)], np.uint64)
        assert np.array_equal(got[:, 0], a) and np.array_equal(got[:, 1], b)
