"""GPU parity at BASELINE.json's full sizes, pinned to the reference.

Every full-size output is compared by sha256 with tests/golden/
golden_large.json, which make_golden_large.py generated HERE from the
unmodified reference (oracle/_ref: launch_edm through every strategy, which
all agree; edm_reference for d=64) and, for the collision table (no reference
implementation exists), from the repo's C restatement.  Output buffers are
poisoned (0xFF bytes) before every launch, so a cell a kernel forgets cannot
match.  Exactly-once coverage of all 2.1e9 cells is checked for every
strategy in both execution shapes (span: the owned-chunk rule of the product
kernels; grid: the paper-faithful kernel), and UTM at N=131072 (k >= 2^33).
"""
import numpy as np
import pytest

from conftest import dev_sha256, poison_

pytestmark = pytest.mark.gpu

N = 65536
ALL7 = ("bb", "ltm-x", "ltm-n", "ltm-r", "utm", "rb", "rec")


def _tri(n):
    return n * (n + 1) // 2


@pytest.fixture(scope="module")
def edm_buf(cuda):
    import torch
    buf = torch.empty(_tri(N), dtype=torch.float32, device=cuda)
    yield buf
    del buf
    torch.cuda.empty_cache()


@pytest.fixture(scope="module")
def pts65536(orc, cuda):
    import torch
    return torch.from_numpy(orc.gen_points(N, 3, 42)).to(cuda)


@pytest.mark.parametrize("mode", ["span", "grid"])
@pytest.mark.parametrize("strat", ALL7)
def test_coverage_full_n65536(tg, cuda, strat, mode):
    r = tg.coverage(strat, N, 16, mode=mode)
    assert r["ok"], r


@pytest.mark.parametrize("mode", ["span", "grid"])
def test_coverage_utm_n131072(tg, cuda, mode):
    # UTM thread index k up to 8.6e9 (u64, float-discriminant walk at 2^33)
    r = tg.coverage("utm", 131072, 16, mode=mode)
    assert r["ok"], r


def test_edm_full_sha_span_all_strategies(tg, golden_large, cuda, pts65536, edm_buf):
    """Packed EDM N=65536 d=3 (the metric workload): sha256 of the whole 8.59 GB
    output == the reference's launch_edm, for every mapping in span form."""
    want = golden_large["edm"]["65536|3"]["sha256"]
    for s in ("ltm-r", "bb", "rec", "rb", "utm", "ltm-x", "ltm-n", "ltm-exact"):
        poison_(edm_buf)
        tg.edm(pts65536, strategy=s, mode="span", out=edm_buf)
        assert dev_sha256(edm_buf) == want, s
    poison_(edm_buf)
    tg.edm(pts65536, strategy="ltm-r", mode="span", out=edm_buf, persistent=True)
    assert dev_sha256(edm_buf) == want, "persistent"


@pytest.mark.parametrize("strat", ["utm", "rb", "ltm-r", "rec"])
def test_edm_full_sha_grid(tg, golden_large, cuda, pts65536, edm_buf, strat):
    """The paper-faithful one-thread-per-cell kernels at full size, same bytes."""
    poison_(edm_buf)
    tg.edm(pts65536, strategy=strat, mode="grid", out=edm_buf)
    assert dev_sha256(edm_buf) == golden_large["edm"]["65536|3"]["sha256"], strat


@pytest.mark.parametrize("G", [2, 4, 8])
def test_edm_full_shards_sha(tg, golden_large, cuda, pts65536, G):
    """lambda-range shards (the 2/4/8-GPU layout): bounds and per-shard sha256
    equal the reference's slices, for every shardable mapping."""
    import torch
    info = golden_large["edm_shards"]["65536|3"][str(G)]
    assert tg.shard_rows(N, 16, G) == info["rows"]
    strats = ("ltm-r", "bb", "rec", "rb", "utm") if G == 8 else ("ltm-r", "rec")
    for s in strats:
        for g in range(G):
            b, e = tg.shard_elems(N, 16, g, G)
            part = poison_(torch.empty(e - b, dtype=torch.float32, device=cuda))
            tg.edm(pts65536, strategy=s, shard=(g, G), out=part)
            assert dev_sha256(part) == info["sha256"][g], (s, g)
            del part


def test_write_full_n65536_sha(tg, golden_large, cuda, edm_buf):
    import torch
    out = edm_buf.view(torch.int32)
    want = golden_large["write"]["65536"]
    for s, mode in (("ltm-r", "span"), ("bb", "span"), ("rec", "span"), ("rb", "span"), ("utm", "span"),
                    ("utm", "grid"), ("rb", "grid")):
        poison_(out)
        st = tg.launch("write", s, N, out=out, rho=16, mode=mode)
        assert dev_sha256(out) == want, (s, mode)
        if s in ("ltm-r", "bb"):
            assert st["blocks_launched"] == {"ltm-r": 2897 ** 2, "bb": 4096 ** 2}[s]
            assert st["blocks_discarded"] == {"ltm-r": 1953, "bb": 8386560}[s]


def test_edm_strategy_host_full_sha(tg, golden_large, orc, cuda):
    """The drop-in host path (tg_edm_strategy_host: H2D, pipelined pieces,
    D2H into pinned memory) at full size."""
    import hashlib

    import torch
    pts = orc.gen_points(N, 3, 42)
    out = torch.empty(_tri(N), dtype=torch.float32).pin_memory().numpy()
    for s in ("ltm-r", "rb"):
        out.view(np.uint32)[:] = 0xFFFFFFFF
        tg.edm_strategy(s, pts, 16, out=out)
        h = hashlib.sha256()
        for a in range(0, out.size, 1 << 27):
            h.update(memoryview(out[a:a + (1 << 27)]))
        assert h.hexdigest() == golden_large["edm"]["65536|3"]["sha256"], s


def test_collide_full_n32768_sha(tg, golden_large, orc, cuda):
    """C3: bit-packed no-diagonal collision table N=32768, r_max=0.0625: sha256
    of the table words and the hit count pinned (750,603 hits), whole table and
    the 8 lambda-range shards, LTM / BB / REC / RB."""
    import torch
    n, r_max = 32768, 0.0625
    ref = golden_large["collide"][f"{n}|{r_max}"]
    sph = torch.from_numpy(orc.gen_points(n, 4, 42)).to(cuda)
    for s in ("ltm-r", "bb", "rec", "rb"):
        bits, hits = tg.collide(sph, r_max, strategy=s)
        assert bits.numel() == ref["words"]
        assert dev_sha256(bits) == ref["sha256"], s
        assert int(hits.item()) == ref["hits"] == 750603
    info = ref["shards"]["8"]
    for g in range(8):
        bits, hits = tg.collide(sph, r_max, strategy="ltm-r", shard=(g, 8))
        assert dev_sha256(bits) == info["sha256"][g], g
        assert int(hits.item()) == info["hits"][g]


def test_edm_direct_d64_full_sha(tg, golden_large, orc, cuda, edm_buf):
    """C4 direct path (bit-exact d > 4 kernel) at N=65536, d=64 == the
    reference's edm_reference, whole output."""
    import torch
    pts = torch.from_numpy(orc.gen_points(N, 64, 42)).to(cuda)
    for s in ("ltm-r", "bb"):
        poison_(edm_buf)
        tg.edm(pts, strategy=s, out=edm_buf)
        assert dev_sha256(edm_buf) == golden_large["edm"]["65536|64"]["sha256"], s
    info = golden_large["edm_shards"]["65536|64"]["8"]
    b, e = tg.shard_elems(N, 16, 3, 8)
    part = poison_(torch.empty(e - b, dtype=torch.float32, device=cuda))
    tg.edm(pts, strategy="ltm-r", shard=(3, 8), out=part)
    assert dev_sha256(part) == info["sha256"][3]


def test_edm_c5_n131072_sha(tg, golden_large, orc, cuda, edm_buf):
    """C5: N=131072, d=3 (34.4 GB packed): the whole output on one B200 and the
    8 lambda-range shards, sha256 == the reference's launch_edm."""
    import torch
    n = 131072
    pts = torch.from_numpy(orc.gen_points(n, 3, 42)).to(cuda)
    info = golden_large["edm_shards"][f"{n}|3"]["8"]
    assert tg.shard_rows(n, 16, 8) == info["rows"]
    for g in range(8):
        b, e = tg.shard_elems(n, 16, g, 8)
        part = poison_(torch.empty(e - b, dtype=torch.float32, device=cuda))
        tg.edm(pts, strategy="ltm-r" if g % 2 else "rec", shard=(g, 8), out=part)
        assert dev_sha256(part) == info["sha256"][g], g
        del part
    torch.cuda.empty_cache()
    whole = poison_(torch.empty(_tri(n), dtype=torch.float32, device=cuda))
    tg.edm(pts, strategy="ltm-r", out=whole)
    assert dev_sha256(whole) == golden_large["edm"][f"{n}|3"]["sha256"]
    del whole
    torch.cuda.empty_cache()


@pytest.mark.parametrize("d", [1, 2, 4])
def test_edm_n16384_other_d_sha(tg, golden_large, orc, cuda, d):
    import torch
    pts = torch.from_numpy(orc.gen_points(16384, d, 42)).to(cuda)
    for s in ("ltm-r", "utm", "rb"):
        out = poison_(torch.empty(_tri(16384), dtype=torch.float32, device=cuda))
        tg.edm(pts, strategy=s, out=out)
        assert dev_sha256(out) == golden_large["edm"][f"16384|{d}"]["sha256"], (s, d)
