"""The reference's output formats and CLI on the GPU path: run_suite CSV
(byte-identical to the reference's emit_csv after a reference parse/emit
round trip), PEDM dump/load interchangeable with the reference's
save/load_packed_edm, improvement-model fit, and the CLI's exit codes."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle
from paper_1308_1419_b200 import pedm, suite

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def _records():
    return [suite.BenchRecord("ltm-r", 1024, 16, 0, "dummy", r, 12345 + r, 2145, 65, 1920, 1.0 / 3.0 + r, "skipped")
            for r in range(3)] + \
           [suite.BenchRecord("rec", 30720, 16, 3, "edm", 0, 99, 1, 0, 0, 1.0512345678901234, "passed")]


def test_csv_roundtrip_python(tmp_path):
    p = tmp_path / "r.csv"
    recs = _records()
    suite.emit_csv(recs, str(p))
    back = suite.parse_csv(str(p))
    assert [vars(r) for r in back] == [vars(r) for r in recs]
    (tmp_path / "bad.csv").write_text("nope\n")
    with pytest.raises(RuntimeError):
        suite.parse_csv(str(tmp_path / "bad.csv"))


@needs_ref
def test_csv_bytes_match_reference(tmp_path):
    R = oracle.ref()
    R.ref_csv_roundtrip.argtypes = [C.c_char_p, C.c_char_p]
    ours = tmp_path / "ours.csv"
    theirs = tmp_path / "theirs.csv"
    suite.emit_csv(_records(), str(ours))
    assert R.ref_csv_roundtrip(str(ours).encode(), str(theirs).encode()) == 0
    assert ours.read_bytes() == theirs.read_bytes()


@needs_ref
def test_pedm_interchange_with_reference(tmp_path, orc):
    R = oracle.ref()
    R.ref_save_pedm.argtypes = [C.POINTER(C.c_float), C.c_uint64, C.c_uint32, C.c_char_p]
    R.ref_load_pedm.argtypes = [C.c_char_p, C.POINTER(C.c_float), C.c_uint64, C.POINTER(C.c_uint64),
                                C.POINTER(C.c_uint32)]
    n, d = 300, 3
    vals = orc.edm_reference(orc.gen_points(n, d, 5))
    ours = tmp_path / "ours.pedm"
    theirs = tmp_path / "theirs.pedm"
    pedm.save_packed_edm(vals, n, d, str(ours))
    assert R.ref_save_pedm(vals.ctypes.data_as(C.POINTER(C.c_float)), n, d, str(theirs).encode()) == 0
    assert ours.read_bytes() == theirs.read_bytes()
    out = np.empty_like(vals)
    nn, dd = C.c_uint64(), C.c_uint32()
    assert R.ref_load_pedm(str(ours).encode(), out.ctypes.data_as(C.POINTER(C.c_float)), out.size,
                           C.byref(nn), C.byref(dd)) == 0
    assert nn.value == n and dd.value == d and out.tobytes() == vals.tobytes()
    back, n2, d2 = pedm.load_packed_edm(str(theirs))
    assert (n2, d2) == (n, d) and back.tobytes() == vals.tobytes()
    (tmp_path / "x").write_bytes(b"NOPE" + bytes(12))
    with pytest.raises(RuntimeError):
        pedm.load_packed_edm(str(tmp_path / "x"))


def test_improvement_model_fit(tg):
    recs = []
    for n in (1024, 4096, 16384):
        nb = n // 16
        I = tg.improvement_model(0.6, 1.0, nb)  # = 1.2 * nb^2/(nb^2+nb)
        recs.append(suite.BenchRecord("ltm-r", n, 16, 0, "dummy", 0, 1, 1, 0, 0, I, "skipped"))
    fit = suite.fit_improvement_model(recs)
    assert fit["ltm-r"]["two_beta_over_tau"] == pytest.approx(1.2, rel=1e-12)


def test_cli_config_errors_exit_2(tg):
    from paper_1308_1419_b200 import cli
    assert cli.main(["bench", "--strategies", "zz"]) == 2
    assert cli.main(["bench", "--kernel", "foo"]) == 2
    assert cli.main(["exactness", "--engine", "bb"]) == 2
    with pytest.raises(SystemExit) as e:
        cli.main(["nosuchcmd"])
    assert e.value.code == 2


@pytest.mark.gpu
def test_cli_gpu_commands(tg, tmp_path, orc, capsys):
    from paper_1308_1419_b200 import cli
    assert cli.main(["verify", "--n-max", "40"]) == 0
    assert "verify: all checks passed" in capsys.readouterr().out
    assert cli.main(["exactness", "--engine", "ltm-n", "--n", "30720"]) == 0
    # float-only Newton rows break first at lambda 1,884,711 (> T(1920)): same as the reference
    assert cli.main(["exactness", "--engine", "ltm-n", "--n", "65536"]) == 1
    assert "first at lambda=1884711" in capsys.readouterr().out
    out = tmp_path / "e.pedm"
    assert cli.main(["edm", "--n", "500", "--features", "3", "--strategy", "ltm-r", "--out", str(out), "--check"]) == 0
    vals, n, d = pedm.load_packed_edm(str(out))
    assert (n, d) == (500, 3) and vals.tobytes() == orc.edm_reference(orc.gen_points(500, 3, 42)).tobytes()
    csv = tmp_path / "b.csv"
    assert cli.main(["bench", "--kernel", "edm", "--features", "2", "--n-start", "256", "--n-end", "1024",
                     "--n-step", "256", "--reps", "3", "--out", str(csv)]) == 0
    recs = suite.parse_csv(str(csv))
    assert recs and all(r.verified == "passed" for r in recs)
    assert {r.strategy for r in recs} == {"bb", "ltm-x", "ltm-n", "ltm-r", "utm", "rb", "rec"}
    assert os.path.exists(str(csv) + ".fit.json")
    # Gram mode: the check is the stated tolerance, reported as max err / bound
    assert cli.main(["edm", "--n", "700", "--features", "40", "--strategy", "ltm-r", "--mode", "gram", "--check"]) == 0
    assert "within tolerance" in capsys.readouterr().out


@pytest.mark.gpu
def test_pedm_device_writer_large(tg, orc, tmp_path, cuda):
    import torch
    n = 8192
    pts = torch.from_numpy(orc.gen_points(n, 3, 1)).to(cuda)
    dev = tg.edm(pts)
    p = tmp_path / "big.pedm"
    old = pedm._CHUNK
    pedm._CHUNK = 1 << 20  # force several staging chunks
    try:
        pedm.save_packed_edm(dev, n, 3, str(p))
    finally:
        pedm._CHUNK = old
    vals, nn, dd = pedm.load_packed_edm(str(p))
    assert (nn, dd) == (n, 3) and vals.tobytes() == dev.cpu().numpy().tobytes()


def test_pedm_shard_writer_host(tmp_path, orc):
    """Lambda-range shards written in any order into one PEDM file (per-shard
    save_packed_edm, edm.cpp:65-77) are byte-identical to the whole-matrix dump
    and load back equal to the oracle."""
    import hashlib
    n, d = 300, 3
    pts = orc.gen_points(n, d, 7)
    want = orc.edm_reference(pts)
    whole = tmp_path / "whole.pedm"
    pedm.save_packed_edm(want, n, d, str(whole))
    rows = [0, 5, 9, 13, 16, 19]  # block rows at rho = 16 (last = ceil(300 / 16))
    p = tmp_path / "sharded.pedm"
    for g in (3, 0, 4, 1, 2):  # any order
        b, e = rows[g] * 16, min(n, rows[g + 1] * 16)
        e0, e1 = b * (b + 1) // 2, e * (e + 1) // 2
        pedm.save_packed_edm_shard(want[e0:e1].copy(), n, d, str(p), e0)
    assert hashlib.sha256(p.read_bytes()).digest() == hashlib.sha256(whole.read_bytes()).digest()
    vals, nn, dd = pedm.load_packed_edm(str(p))
    assert (nn, dd) == (n, d) and vals.tobytes() == want.tobytes()
    with pytest.raises(ValueError):
        pedm.save_packed_edm_shard(want[:10].copy(), n, d, str(p), n * (n + 1) // 2 - 5)


@pytest.mark.gpu
def test_pedm_shard_writer_device(tg, orc, tmp_path, cuda):
    """C5 layout: every lambda-range shard computed on device and written at its
    offset of one shared PEDM file; the reassembled file equals the oracle."""
    import torch
    n, G = 4096, 8
    pts_np = orc.gen_points(n, 3, 42)
    pts = torch.from_numpy(pts_np).to(cuda)
    p = tmp_path / "c5.pedm"
    old = pedm._CHUNK
    pedm._CHUNK = 1 << 18
    try:
        for g in reversed(range(G)):
            b, e = tg.shard_elems(n, 16, g, G)
            part = tg.edm(pts, shard=(g, G))
            assert part.numel() == e - b
            pedm.save_packed_edm_shard(part, n, 3, str(p), b)
    finally:
        pedm._CHUNK = old
    vals, nn, dd = pedm.load_packed_edm(str(p))
    assert (nn, dd) == (n, 3) and vals.tobytes() == orc.edm_reference(pts_np).tobytes()
