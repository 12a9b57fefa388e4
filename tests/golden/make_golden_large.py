"""Full-size golden fixtures (tests/golden/golden_large.json) for the metric
configs, generated HERE from the UNMODIFIED reference (oracle/_ref, compiled
from /root/reference/proj/src) -- the GPU box has no /root/reference, so these
hashes are what the full-size GPU parity tests and bench.py's verify compare
against.

    python tests/golden/make_golden_large.py            (~10 min, ~45 GB RAM)

Recorded:
  edm|N|d          sha256 of the whole packed fp32 EDM of gen_points(N, d, 42)
                   (launch_edm, engine.cpp:157-175, through every strategy the
                   reference can schedule -- all must agree; d > 4 via
                   edm_reference, edm.cpp:53-63, which has no d cap)
  edm_shards|N|d   per-shard sha256 of the lambda-range shards G = 2, 4, 8
                   (block-row bounds recorded next to them)
  write|N          sha256 of the u32 i+j table (enumerate_lower order)
  collide|N|r_max  sha256 of the bit-packed no-diagonal collision table
                   (uint32 words, LSB first) + hit count, and per-shard shas;
                   from the repo's C restatement (the reference has no
                   collision kernel: PAPER.md, SURVEY 8c -- parity unpinned
                   w.r.t. the reference, pinned to trigrid_oracle.c)
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

RHO, SEED = 16, 42
OUT = os.path.join(HERE, "golden_large.json")


def tri(n: int) -> int:
    return n * (n + 1) // 2


def shard_rows(n: int, rho: int, G: int) -> list[int]:
    """Block-row bounds nearest to g*T(nb)/G, exact integers."""
    nb = -(-n // rho)
    total = tri(nb)
    rows = [0] * (G + 1)
    rows[G] = nb
    for g in range(1, G):
        t = total * g // G
        r = (math.isqrt(8 * t + 1) - 1) // 2  # T(r) <= t < T(r+1)
        b = r if t - tri(r) <= tri(r + 1) - t else r + 1
        rows[g] = min(max(b, rows[g - 1]), nb)
    return rows


def sha_chunks(buf: np.ndarray, lo: int = 0, hi: int | None = None, chunk: int = 1 << 28) -> str:
    h = hashlib.sha256()
    hi = buf.size if hi is None else hi
    for a in range(lo, hi, chunk):
        h.update(memoryview(buf[a:min(hi, a + chunk)]).cast("B"))
    return h.hexdigest()


def ref_edm(strategy: str, pts: np.ndarray):
    """launch_edm of the reference into its own PackedEdm; returns (session, view)."""
    R = oracle.ref()
    n, d = pts.shape
    sess = R.ref_edm_session_create(strategy.encode(), pts.ctypes.data_as(C.POINTER(C.c_float)), n, d, RHO)
    if not sess:
        raise RuntimeError(R.ref_last_error().decode())
    st = np.zeros(4, np.uint64)
    rc = R.ref_edm_session_run(sess, 0, st.ctypes.data_as(C.POINTER(C.c_uint64)))
    if rc:
        raise RuntimeError(R.ref_last_error().decode())
    ptr = R.ref_edm_session_data(sess)
    view = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_float)), shape=(tri(n),))
    return sess, view


def edm_entry(g: dict, n: int, d: int, strategies) -> None:
    pts = oracle.gen_points(n, d, SEED)
    R = oracle.ref()
    shas = {}
    shard_info = None
    for s in strategies:
        t0 = time.time()
        sess, view = ref_edm(s, pts)
        shas[s] = sha_chunks(view)
        if shard_info is None:
            shard_info = {}
            for G in (2, 4, 8):
                rows = shard_rows(n, RHO, G)
                bounds = [tri(min(n, RHO * r)) for r in rows]
                shard_info[str(G)] = {"rows": rows,
                                      "sha256": [sha_chunks(view, bounds[k], bounds[k + 1]) for k in range(G)]}
        R.ref_edm_session_destroy(sess)
        print(f"  edm N={n} d={d} {s}: {shas[s][:16]}  ({time.time() - t0:.1f} s)", flush=True)
    assert len(set(shas.values())) == 1, f"reference strategies disagree at N={n}: {shas}"
    g["edm"][f"{n}|{d}"] = {"sha256": next(iter(shas.values())), "strategies": sorted(shas),
                            "source": "reference launch_edm (oracle/_ref), workers=0"}
    g["edm_shards"][f"{n}|{d}"] = shard_info


def edm_wide_entry(g: dict, n: int, d: int) -> None:
    """d > 4: the reference's edm_reference (no d cap); points = the shape-invariant stream."""
    t0 = time.time()
    pts = oracle.gen_points(n * d // 4, 4, SEED).reshape(n, d)
    out = np.empty(tri(n), np.float32)
    oracle.ref().ref_edm_reference(pts.ctypes.data_as(C.POINTER(C.c_float)), n, d,
                                   out.ctypes.data_as(C.POINTER(C.c_float)))
    sha = sha_chunks(out)
    shard_info = {}
    for G in (2, 4, 8):
        rows = shard_rows(n, RHO, G)
        bounds = [tri(min(n, RHO * r)) for r in rows]
        shard_info[str(G)] = {"rows": rows, "sha256": [sha_chunks(out, bounds[k], bounds[k + 1]) for k in range(G)]}
    g["edm"][f"{n}|{d}"] = {"sha256": sha, "strategies": ["edm_reference"],
                            "source": "reference edm_reference (oracle/_ref), sequential"}
    g["edm_shards"][f"{n}|{d}"] = shard_info
    print(f"  edm N={n} d={d} edm_reference: {sha[:16]}  ({time.time() - t0:.1f} s)", flush=True)


def write_entry(g: dict, n: int) -> None:
    h = hashlib.sha256()
    step = 4096
    for r0 in range(0, n, step):
        r1 = min(n, r0 + step)
        i = np.repeat(np.arange(r0, r1, dtype=np.uint64), np.arange(r0 + 1, r1 + 1))
        starts = np.repeat(np.arange(r0, r1, dtype=np.uint64) * np.arange(r0 + 1, r1 + 1, dtype=np.uint64) // 2,
                           np.arange(r0 + 1, r1 + 1))
        j = np.arange(tri(r0), tri(r1), dtype=np.uint64) - starts
        h.update((i + j).astype(np.uint32).tobytes())
    g["write"][str(n)] = h.hexdigest()
    print(f"  write N={n}: {g['write'][str(n)][:16]}", flush=True)


def pack_words(bits_u8: np.ndarray, npairs: int) -> np.ndarray:
    """LSB-first byte table -> uint32 words (zero past the end)."""
    words = (npairs + 31) // 32
    buf = np.zeros(4 * max(words, 1), np.uint8)
    buf[:bits_u8.size] = bits_u8
    return buf.view(np.uint32)[:max(words, 1)]


def collide_entry(g: dict, n: int, r_max: float) -> None:
    t0 = time.time()
    sph = oracle.gen_points(n, 4, SEED)
    bits_u8, hits = oracle.collide_reference(sph, r_max)
    npairs = n * (n - 1) // 2
    words = pack_words(bits_u8, npairs)
    entry = {"sha256": hashlib.sha256(words.tobytes()).hexdigest(), "hits": hits, "pairs": npairs,
             "words": int(words.size), "source": "oracle/trigrid_oracle.c or_collide_reference "
             "(no reference implementation exists; semantics in DESIGN.md)", "shards": {}}
    flat = np.unpackbits(bits_u8, bitorder="little")[:npairs]
    for G in (2, 4, 8):
        rows = shard_rows(n, RHO, G)
        b = [min(n, RHO * r) * (min(n, RHO * r) - 1) // 2 for r in rows]
        sh, hs = [], []
        for k in range(G):
            seg = flat[b[k]:b[k + 1]]
            packed = np.packbits(seg, bitorder="little")
            w = pack_words(packed, seg.size)
            sh.append(hashlib.sha256(w.tobytes()).hexdigest())
            hs.append(int(seg.sum(dtype=np.uint64)))
        entry["shards"][str(G)] = {"rows": rows, "sha256": sh, "hits": hs}
    g["collide"][f"{n}|{r_max}"] = entry
    print(f"  collide N={n} r_max={r_max}: hits {hits} sha {entry['sha256'][:16]} ({time.time() - t0:.1f} s)",
          flush=True)


def main():
    oracle.build()
    only = set(sys.argv[1:])
    g = {"edm": {}, "edm_shards": {}, "write": {}, "collide": {}}
    if os.path.exists(OUT):
        with open(OUT) as f:
            g.update(json.load(f))

    def want(key):
        return not only or key in only

    if want("collide"):
        collide_entry(g, 32768, 0.0625)
        collide_entry(g, 4096, 0.0625)
    if want("write"):
        for n in (65536,):
            write_entry(g, n)
    if want("edm65536"):
        edm_entry(g, 65536, 3, ("ltm-r", "bb", "rec", "rb", "ltm-x", "ltm-n", "utm"))
    if want("edm16384"):
        for d in (1, 2, 4):
            edm_entry(g, 16384, d, ("ltm-r",))
    if want("edm131072"):
        edm_entry(g, 131072, 3, ("ltm-r",))
    if want("edm_d64"):
        edm_wide_entry(g, 65536, 64)
    with open(OUT, "w") as f:
        json.dump(g, f, indent=1, sort_keys=True)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
