"""Randomised parity sweep (fixed seed): random N, d, rho, mapping, execution
shape, shard and persistence, every result compared byte for byte with the
oracle (oracle/trigrid_oracle.c).  Complements the structured grids of
test_gpu_parity.py with combinations nobody picked by hand (odd N with RB's
fold, REC schedules at rho 4/8/32, shards of UTM / RB, d > 4 windows, ...)."""
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

STRATS = ["bb", "ltm-x", "ltm-n", "ltm-r", "ltm-exact", "utm", "rb", "rec"]


def _cases(count, seed):
    rng = random.Random(seed)
    for _ in range(count):
        yield (rng.choice(STRATS), rng.randint(1, 2500), rng.choice([4, 8, 12, 16, 16, 16, 32]),
               rng.choice(["span", "span", "grid"]), rng.randint(1, 3), rng.random() < 0.2, rng.randint(0, 1 << 30))


def _valid(orc, strat, n, rho):
    if strat == "rec" and orc.rec_decompose(n, rho) is None:
        return False
    return not (strat == "rb" and n < 2)


def test_fuzz_edm(tg, orc, cuda):
    import torch
    done = 0
    for strat, n, rho, mode, shards, persistent, seed in _cases(80, 20261017):
        if not _valid(orc, strat, n, rho):
            continue
        d = 1 + seed % 4
        pts_np = orc.gen_points(n, d, seed)
        want = orc.edm_reference(pts_np)
        pts = torch.from_numpy(pts_np).to(cuda)
        if mode == "span" and shards > 1:
            for g in range(shards):
                b, e = tg.shard_elems(n, rho, g, shards)
                if e == b:
                    continue
                got = tg.edm(pts, strategy=strat, rho=rho, mode="span", shard=(g, shards)).cpu().numpy()
                assert got.tobytes() == want[b:e].tobytes(), (strat, n, rho, d, g, shards)
        else:
            got = tg.edm(pts, strategy=strat, rho=rho, mode=mode, persistent=persistent and mode == "span")
            assert got.cpu().numpy().tobytes() == want.tobytes(), (strat, n, rho, d, mode, persistent)
        done += 1
    assert done >= 50


def test_fuzz_edm_wide(tg, orc, cuda):
    """d > 4: the 512-column pipelined direct kernel (span, rho = 16) and the
    grid kernel, random d in 5..70."""
    import torch
    rng = random.Random(7)
    for _ in range(12):
        strat = rng.choice(["bb", "ltm-r", "ltm-n", "rec"])
        n, d = rng.randint(1, 1800), rng.randint(5, 70)
        if not _valid(orc, strat, n, 16):
            continue
        pts_np = orc.gen_points(n * d, 1, rng.randint(0, 1 << 30)).reshape(n, d)
        want = orc.edm_reference(pts_np)
        mode = rng.choice(["span", "grid"])
        got = tg.edm(torch.from_numpy(pts_np).to(cuda), strategy=strat, rho=16, mode=mode).cpu().numpy()
        assert got.tobytes() == want.tobytes(), (strat, n, d, mode)


def test_fuzz_write_and_collide(tg, orc, cuda):
    import torch
    for strat, n, rho, mode, shards, _, seed in _cases(40, 99):
        if not _valid(orc, strat, n, rho):
            continue
        out = torch.empty(n * (n + 1) // 2, dtype=torch.int32, device=cuda)
        tg.launch("write", strat, n, out=out, rho=rho, mode=mode)
        assert np.array_equal(out.cpu().numpy().view(np.uint32), orc.write_reference(n)), (strat, n, rho, mode)
        if n < 2:
            continue
        cmode = "grid" if strat == "utm" else mode  # the span collision kernel: square tiles and RB
        r_max = 0.05 + (seed % 100) / 500.0
        sph_np = orc.gen_points(n, 4, seed)
        want_bits, want_hits = orc.collide_reference(sph_np, r_max)
        bits, hits = tg.collide(torch.from_numpy(sph_np).to(cuda), r_max, strategy=strat, rho=rho, mode=cmode)
        assert int(hits.item()) == int(want_hits), (strat, n, rho, cmode)
        got = bits.cpu().numpy().view(np.uint8)[: want_bits.size]
        assert np.array_equal(got, want_bits), (strat, n, rho, cmode)
