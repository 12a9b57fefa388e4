"""GPU tests of the span (B200) forms of every mapping: exactly-once
coverage of the owned-chunk rule, explicit REC schedules, per-pass device
timing (LaunchOptions::per_pass), UTM engines, sharded count tables.

Reference semantics: process_block / run_strategy (engine.cpp:17-136), the
strategy classes (strategies.hpp:247-391), rec_schedule (strategies.cpp:
116-140)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SPAN7 = ("bb", "ltm-x", "ltm-n", "ltm-r", "ltm-exact", "rec", "rb", "utm")


def _rec_ok(orc, n, rho):
    return orc.rec_decompose(n, rho) is not None


def test_utm_superblock_widths(tg, cuda):
    """The UTM super-block side scales with N (16..64 run widths, about 4
    super-block rows): exactly-once coverage around the sizes where it
    changes (16 -> 32 -> 64) and at odd N (ragged last super-block)."""
    for n in (16383, 16385, 20000, 32768, 40000, 65535):
        r = tg.coverage("utm", n, 16, mode="span")
        assert r["ok"], (n, r)


@pytest.mark.parametrize("strat", SPAN7)
def test_span_coverage_exactly_once(tg, orc, cuda, strat):
    """COUNT in span form adds 1 to every cell of every owned chunk: each cell
    must end at exactly 1 (0 on the diagonal for UTM's no-diagonal domain)."""
    for n in (1, 2, 3, 4, 5, 7, 15, 16, 17, 31, 33, 100, 255, 256, 257, 1000, 1024, 3000, 4096):
        for rho in (16, 4, 8, 32, 64):
            if strat == "rec" and not _rec_ok(orc, n, rho):
                continue
            if strat == "rb" and n < 2:
                continue
            r = tg.coverage(strat, n, rho, mode="span")
            assert r["ok"], (strat, n, rho, r)


def test_rec_explicit_schedules(tg, orc, cuda):
    """Every (m, k) with m a multiple of rho and N = m 2^k <= 512 (the sweep of
    verify_rec, checks.cpp:167-190): span coverage, span / grid EDM parity."""
    import torch
    for rho in (16, 4):
        k = 1
        while (1 << k) <= 512:
            m = rho
            while (m << k) <= 512:
                n = m << k
                assert tg.coverage("rec", n, rho, mode="span", rec=(m, k))["ok"], (m, k, rho)
                assert tg.coverage("rec", n, rho, mode="grid", rec=(m, k))["ok"], (m, k, rho)
                if (m + k) % 3 == 0:
                    pts_np = orc.gen_points(n, 3, m + k)
                    pts = torch.from_numpy(pts_np).to(cuda)
                    want = orc.edm_reference(pts_np)
                    for mode in ("span", "grid"):
                        out = torch.empty(n * (n + 1) // 2, dtype=torch.float32, device=cuda)
                        tg.launch("edm", "rec", n, points=pts, out=out, rho=rho, mode=mode, rec=(m, k))
                        assert out.cpu().numpy().tobytes() == want.tobytes(), (m, k, rho, mode)
                m += rho
            k += 1
    with pytest.raises(ValueError):
        tg.coverage("rec", 96, 16, rec=(16, 2))  # 16 * 2^2 != 96
    with pytest.raises(ValueError):
        tg.coverage("rec", 96, 16, rec=(24, 2))  # 24 % 16 != 0


def test_rec_per_pass(tg, orc, cuda):
    """LaunchOptions::per_pass: one entry per grid pass in rec_schedule order
    (levels 1..k, then the diagonal pass), closed-form counts equal to the
    reference's per-pass tallies, device time per pass."""
    import torch
    n = 4096
    gs = tg.grid_spec("rec", n, 16)
    m, k = orc.rec_decompose(n, 16)
    assert len(gs) == k + 1 and gs[-1]["level"]["level"] == 0
    assert [g["level"]["level"] for g in gs[:-1]] == list(range(1, k + 1))
    out = torch.empty(n * (n + 1) // 2, dtype=torch.int32, device=cuda)
    for mode in ("span", "grid"):
        st = tg.launch("write", "rec", n, out=out, rho=16, mode=mode, per_pass=True)
        pp = st["per_pass"]
        assert len(pp) == k + 1
        for key in ("blocks_launched", "blocks_discarded", "threads_discarded"):
            assert sum(p[key] for p in pp) == st[key]
        for p, g in zip(pp, gs):
            assert p["blocks_launched"] == g["blocks_x"] * g["blocks_y"]
            assert p["wall_time_ns"] > 0
        assert np.array_equal(out.cpu().numpy().view(np.uint32), orc.write_reference(n)), mode
    # single-pass strategies: per_pass[0] is the whole launch
    st = tg.launch("write", "ltm-r", n, out=out, rho=16, per_pass=True)
    assert len(st["per_pass"]) == 1 and st["per_pass"][0]["blocks_launched"] == st["blocks_launched"]


@pytest.mark.parametrize("engine", ["native", "newton", "reciprocal", "exact"])
def test_utm_engines(tg, orc, cuda, engine):
    """StrategyId{UpperTri, engine}: every engine maps exactly (the walk
    repairs the float row), in span and grid form."""
    import torch
    for n in (2, 17, 1000, 2048):
        pts_np = orc.gen_points(n, 2, n)
        pts = torch.from_numpy(pts_np).to(cuda)
        want = orc.edm_reference(pts_np)
        for mode in ("span", "grid"):
            out = torch.empty(n * (n + 1) // 2, dtype=torch.float32, device=cuda)
            tg.launch("edm", "utm", n, points=pts, out=out, rho=16, mode=mode, engine=engine)
            assert out.cpu().numpy().tobytes() == want.tobytes(), (n, mode)
        assert tg.coverage("utm", n, 16, mode="span", engine=engine)["ok"]


def test_count_shards(tg, orc, cuda):
    """Sharded COUNT: each shard's table (its packed slice) is all ones
    (diagonal 0 for UTM) -- the shard windows partition the cells exactly."""
    import torch
    for strat in ("ltm-r", "bb", "rec", "rb", "utm"):
        for n, G in ((1024, 3), (3000, 8), (4096, 2)):
            if strat == "rec" and not _rec_ok(orc, n, 16):
                continue
            total = 0
            for g in range(G):
                b, e = tg.shard_elems(n, 16, g, G)
                cnt = torch.zeros(max(e - b, 1), dtype=torch.int32, device=cuda)
                tg.launch("count", strat, n, out=cnt, rho=16, mode="span", shard=(g, G))
                got = cnt.cpu().numpy()[: e - b]
                want = np.ones(e - b, np.int32)
                if strat == "utm":  # diagonal cells T(i+1) - 1 stay 0
                    i = np.arange(n)
                    diag = i * (i + 1) // 2 + i
                    sel = diag[(diag >= b) & (diag < e)] - b
                    want[sel] = 0
                assert np.array_equal(got, want), (strat, n, G, g)
                total += e - b
            assert total == n * (n + 1) // 2


def test_rb_span_odd_even(tg, orc, cuda):
    """RB's fold differs for odd and even N (strategies.hpp:182-193): both
    parities, every rho, EDM and write tables bit-exact."""
    import torch
    for n in range(2, 70):
        for rho in (4, 8, 16):
            pts_np = orc.gen_points(n, 3, n)
            out = torch.empty(n * (n + 1) // 2, dtype=torch.float32, device=cuda)
            tg.launch("edm", "rb", n, points=torch.from_numpy(pts_np).to(cuda), out=out, rho=rho, mode="span")
            assert out.cpu().numpy().tobytes() == orc.edm_reference(pts_np).tobytes(), (n, rho)


def test_multi_device_host_dropin(tg, orc, cuda):
    """edm_strategy(devices=[...]): the lambda range split over several GPUs of
    one process (here the same GPU twice), each slice copied out on its own."""
    import torch
    n = 3000
    pts = orc.gen_points(n, 3, 5)
    want = orc.edm_reference(pts)
    for s in ("ltm-r", "rb", "utm", "bb"):
        got, st = tg.edm_strategy(s, pts, 16, devices=[0, 0])
        assert got.tobytes() == want.tobytes(), s
    got, _ = tg.edm_strategy("rec", orc.gen_points(4096, 3, 5), 16, devices=[0, 0, 0])
    assert got.tobytes() == orc.edm_reference(orc.gen_points(4096, 3, 5)).tobytes()
    assert torch.cuda.current_device() == 0


def test_device_selection_follows_tensors(tg, orc, cuda):
    """launch() runs on the device of its tensors and leaves the caller's
    current device unchanged."""
    import torch
    before = torch.cuda.current_device()
    pts_np = orc.gen_points(500, 3, 1)
    out = tg.edm(torch.from_numpy(pts_np).to(cuda), strategy="ltm-r")
    assert out.cpu().numpy().tobytes() == orc.edm_reference(pts_np).tobytes()
    tg.gen_values(100, 1, cuda)
    tg.collide(torch.from_numpy(orc.gen_points(100, 4, 1)).to(cuda), 0.1)
    assert torch.cuda.current_device() == before
