"""Gram-trick EDM on tcgen05 (mode="gram"): NOT bit-exact by design.  Stated
tolerance (tg_gram.cuh):
    |d_gram^2 - d_exact^2| <= 2^-17 * (|x_i|^2 + |x_j|^2),   d_gram(i, i) == 0
checked against the exact oracle on every packed cell."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
TOL = 2.0 ** -17


def _gram(tg, cuda, pts_np, shard=None, strategy="ltm-r"):
    import torch
    pts = torch.from_numpy(pts_np).to(cuda)
    return tg.edm(pts, strategy=strategy, mode="gram", shard=shard).cpu().numpy()


def _check(orc, pts, got):
    n = pts.shape[0]
    want = orc.edm_reference(pts).astype(np.float64)
    i = np.repeat(np.arange(n), np.arange(1, n + 1))
    j = np.arange(want.size) - np.repeat(np.arange(n) * (np.arange(n) + 1) // 2, np.arange(1, n + 1))
    nrm = (pts.astype(np.float64) ** 2).sum(1)
    err = np.abs(got.astype(np.float64) ** 2 - want ** 2)
    bound = TOL * (nrm[i] + nrm[j])
    assert np.all(got[i == j] == 0.0)
    worst = float(np.max(err / np.maximum(bound, 1e-30)))
    assert np.all(err <= bound), f"max err/bound = {worst}"
    return worst


@pytest.mark.parametrize("n,d", [(1, 8), (100, 8), (128, 64), (200, 64), (1000, 64), (777, 100), (4096, 64), (300, 3), (300, 200), (513, 128), (130, 65), (260, 256), (200, 300), (2000, 128), (1100, 37), (300, 512), (1500, 192)])
def test_gram_tolerance(tg, orc, cuda, n, d):
    pts = orc.gen_points(n, d, 11 + d)
    _check(orc, pts, _gram(tg, cuda, pts))


def test_gram_shards_and_bb(tg, orc, cuda):
    pts = orc.gen_points(1500, 64, 5)
    whole = _gram(tg, cuda, pts)
    parts = [_gram(tg, cuda, pts, shard=(g, 4)) for g in range(4)]
    assert np.concatenate(parts).tobytes() == whole.tobytes()
    assert _gram(tg, cuda, pts, strategy="bb").tobytes() == whole.tobytes()


def test_gram_c4_full_size_sampled(tg, orc, cuda):
    import torch
    n, d = 65536, 64
    pts_np = orc.gen_points(n, d, 42)
    out = tg.edm(torch.from_numpy(pts_np).to(cuda), strategy="ltm-r", mode="gram")
    rng = np.random.default_rng(3)
    nrm = (pts_np.astype(np.float64) ** 2).sum(1)
    for r in [0, 127, 128, 4095, 65535] + [int(x) for x in rng.integers(0, n, 12)]:
        got = out[r * (r + 1) // 2: (r + 1) * (r + 2) // 2].cpu().numpy().astype(np.float64)
        want = orc.edm_rows(pts_np, r, r + 1).astype(np.float64)
        assert got[r] == 0.0
        assert np.all(np.abs(got ** 2 - want ** 2) <= TOL * (nrm[r] + nrm[: r + 1])), r


@pytest.mark.parametrize("kind", ["offset", "mixed_scale", "duplicates", "negative"])
def test_gram_tolerance_adversarial(tg, orc, cuda, kind):
    """The stated tolerance on data that stresses the Gram formula: a large
    common offset (cancellation), points of very different magnitudes (the
    global fp16 scale), exact duplicates (d = 0 off the diagonal), signs."""
    n, d = 700, 64
    pts = orc.gen_points(n, d, 99).astype(np.float64)
    if kind == "offset":
        pts = pts + 1000.0
    elif kind == "mixed_scale":
        pts[::2] *= 1e3
        pts[1::2] *= 1e-3
    elif kind == "duplicates":
        pts[1::3] = pts[0::3][: pts[1::3].shape[0]]
    else:
        pts = pts - 0.5
    pts = pts.astype(np.float32)
    _check(orc, pts, _gram(tg, cuda, pts))


@pytest.mark.parametrize("ratio,d", [(1e-5, 64), (1e-8, 64), (1e-11, 64), (1e-8, 200), (1e-9, 3), (1e-20, 64)])
def test_gram_tolerance_wide_range(tg, orc, cuda, ratio, d):
    """Per-point magnitudes spread over more than 2^20: with one
    global fp16 scale the small points fall to fp16's subnormal floor; the
    kernel switches to per-point scales and the stated bound holds for every
    pair -- small vs small (incl. exact duplicates and all-zero points), small
    vs large, large vs large."""
    n = 600
    pts = orc.gen_points(n, d, 5).astype(np.float64) - 0.5
    small = np.arange(n) % 3 != 0
    pts[~small] *= 1e3
    pts[small] *= 1e3 * ratio
    pts[4::9] = pts[1::9][: pts[4::9].shape[0]]  # duplicates among the small points
    pts[7] = 0.0
    pts = pts.astype(np.float32)
    _check(orc, pts, _gram(tg, cuda, pts))


def test_gram_concurrent_streams(tg, orc, cuda):
    """Two host threads, two streams, different inputs: the per-launch device
    scratch (operands, norms) is private, so each result equals its serial run."""
    import threading

    import torch
    pa = torch.from_numpy(orc.gen_points(3000, 64, 1)).to(cuda)
    pb = torch.from_numpy(orc.gen_points(3000, 100, 2)).to(cuda)
    want_a = tg.edm(pa, mode="gram").cpu()
    want_b = tg.edm(pb, mode="gram").cpu()
    got = {}

    def run(key, pts):
        s = torch.cuda.Stream()
        outs = []
        for _ in range(4):
            outs.append(tg.edm(pts, mode="gram", stream=s))
        s.synchronize()
        got[key] = [o.cpu() for o in outs]

    ts = [threading.Thread(target=run, args=("a", pa)), threading.Thread(target=run, args=("b", pb))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert all(torch.equal(o, want_a) for o in got["a"])
    assert all(torch.equal(o, want_b) for o in got["b"])
