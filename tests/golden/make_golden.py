"""Generate tests/golden/* from the UNMODIFIED reference.

Runs here (where /root/reference exists): builds oracle/_ref (the reference
compiled from its own sources plus its own pybind module) and records its
outputs.  The GPU box has no /root/reference, so the committed fixtures are
what pins the oracle and the product there.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

oracle.build()
sys.path.insert(0, oracle.REF_DIR)
import _trigrid as T  # noqa: E402  (the reference's own module)

R = oracle.ref()
ENG = ["native", "newton", "reciprocal", "exact"]


def ref_ltm_range(l0, cnt, eng, diag, repair):
    oi = np.empty(cnt, np.uint64)
    oj = np.empty(cnt, np.uint64)
    R.ref_ltm_map_range(l0, cnt, oracle.ENGINES[eng], int(diag), oracle.REPAIR[repair],
                        oi.ctypes.data_as(C.POINTER(C.c_uint64)), oj.ctypes.data_as(C.POINTER(C.c_uint64)))
    return oi, oj


def main():
    g = {}
    rng = np.random.default_rng(1308)
    # ---- g(lambda): sampled lambdas incl. the float-path break points
    lams = sorted(set(list(range(0, 4096)) + [1844159, 1844160, 1884711, 2110485, 10619135]
                      + [int(x) for x in rng.integers(0, 33_558_528, 3000)]
                      + [int(x) for x in rng.integers(0, 2**31, 1000)]))
    g["ltm_lams"] = lams
    g["ltm"] = {}
    for e in ENG:
        for diag in (True, False):
            for rep in ("auto", "off"):
                if rep == "auto":  # the module's own ltm_map (module.cpp:90-96)
                    out = [T.ltm_map(l, e, diag) for l in lams]
                else:              # RepairPolicy::Off through the C++ API
                    out = []
                    for l in lams:
                        i, j = ref_ltm_range(l, 1, e, diag, "off")
                        out.append((int(i[0]), int(j[0])))
                g["ltm"][f"{e}|{int(diag)}|{rep}"] = [list(map(int, c)) for c in out]
    # ---- exactness sweeps (float row, repair off) -- checks.cpp:81-95
    g["exactness"] = {}
    for n in (256, 1920, 2048, 4096):
        for e in ENG:
            for diag in (True, False):
                r3 = np.zeros(3, np.uint64)
                R.ref_ltm_exactness_sweep(n, oracle.ENGINES[e], int(diag), r3.ctypes.data_as(C.POINTER(C.c_uint64)))
                g["exactness"][f"{n}|{e}|{int(diag)}"] = [int(x) for x in r3]
    # ---- utm / rb / rec
    g["utm"] = []
    for n in (2, 3, 4, 5, 17, 100, 1000, 65536, 131072):
        pairs = n * (n - 1) // 2
        ks = sorted(set([0, pairs - 1, pairs // 2] + [int(x) for x in rng.integers(0, pairs, 200)]))
        for e in ("newton", "native", "reciprocal", "exact"):
            g["utm"].append([n, e, ks, [list(T.utm_map(k, n, e)) for k in ks]])
    g["rb"] = []
    for n in (2, 3, 6, 7, 16, 33):
        w, h = T.rb_rect(n)
        g["rb"].append([n, [w, h], [[tx, ty, T.rb_map(tx, ty, n)] for tx in range(w + 1) for ty in range(h + 1)]])
    g["rec_decompose"] = [[n, rho, T.rec_decompose(n, rho)] for n in (16, 32, 48, 100, 1024, 3072, 30720, 65536, 131072, 7)
                          for rho in (1, 4, 16)]
    # ---- scalar helpers
    g["isqrt"] = [[v, T.isqrt(v)] for v in [0, 1, 2, 3, 4, 15, 16, 17, 14753281, 2**32 - 1, 2**32, 2**52 + 1,
                                            2**63, 2**64 - 1, 10**18]]
    g["grid_side_balanced"] = [[n, T.grid_side_balanced(n)] for n in (1, 2, 3, 16, 256, 1920, 2048, 4096, 8192)]
    xs = [0.25, 1.0, 2.0, 3.5, 100.0, 12345.678, 1e-3, 1e10, 16777217.0]
    g["fast_inv_sqrt"] = [[x, it, T.fast_inv_sqrt(x, it)] for x in xs for it in (0, 1, 3)]
    g["rsqrt_single"] = [[x, T.rsqrt_single(x)] for x in xs]
    g["sqrt_via"] = [[e, x, T.sqrt_via(e, x)] for e in ("native", "newton", "reciprocal") for x in xs] + \
                    [["exact", x, T.sqrt_via("exact", x)] for x in (0.0, 1.0, 15.0, 16.0, 1e15)]
    g["count_wasted"] = [[s, n, T.count_wasted(s, n)] for s in ("bb", "ltm-r") for n in (1, 2, 16, 1920, 4096, 8192)]
    g["improvement_model"] = [[b, t, n, T.improvement_model(b, t, n)] for b, t, n in
                              [(1, 1.74, 1920), (1, 1.0, 1), (2, 3, 100)]]
    # ---- dispatch stats per strategy (launch_dummy through the reference engine)
    g["stats"] = []
    for s in ("bb", "ltm-x", "ltm-n", "ltm-r", "utm", "rb", "rec"):
        for n in (1, 2, 15, 16, 17, 100, 256, 1000, 1024, 3072, 4096):
            for rho in (16, 4, 1, 5, 32):
                st = np.zeros(4, np.uint64)
                rc = R.ref_launch_dummy(s.encode(), n, rho, 1, st.ctypes.data_as(C.POINTER(C.c_uint64)))
                g["stats"].append([s, n, rho, None if rc else [int(x) for x in st[:3]]])
    # ---- coverage_ok via the reference's own module
    g["coverage_ok"] = [[s, n, rho, T.coverage_ok(s, n, rho)] for s in ("bb", "ltm-r", "utm", "rb", "rec")
                        for n in (2, 16, 17, 64, 96) for rho in (16, 4) if not (s == "rec" and T.rec_decompose(n, rho) is None)]
    # ---- points and EDM
    g["gen_points_head"] = {f"{n}|{d}": T.gen_points(n, d, 42).ravel()[:16].tolist() for n, d in ((4, 1), (8, 3), (16, 4))}
    g["edm_sha256"] = {}
    for n in (1, 2, 3, 17, 64, 256, 1024, 4096):
        for d in (1, 2, 3, 4):
            e = T.edm_reference(T.gen_points(n, d, 42))
            g["edm_sha256"][f"{n}|{d}"] = hashlib.sha256(e.tobytes()).hexdigest()
    # d=64 set (shape-invariant stream) -- small N only
    pts64 = T.gen_points(16 * 128, 4, 42).reshape(128, 64)
    g["edm_sha256"]["128|64"] = hashlib.sha256(T.edm_reference(pts64).tobytes()).hexdigest()
    # known-answer from SPEC: edm_reference([0,1,2]) = [0,1,0,2,1,0]
    g["edm_kat"] = T.edm_reference(np.array([[0.0], [1.0], [2.0]], np.float32)).tolist()
    np.save(os.path.join(HERE, "edm_n64_d3.npy"), T.edm_reference(T.gen_points(64, 3, 42)))
    # edm_strategy stats (the module's own dispatch path) at the SURVEY N=4096 anchor
    g["edm_strategy_stats"] = {}
    pts = T.gen_points(4096, 3, 42)
    for s in ("bb", "ltm-r", "rec", "rb", "utm"):
        _, st = T.edm_strategy(s, pts, 16, 0)
        st.pop("wall_time_ns")
        g["edm_strategy_stats"][s] = st
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(g, f, separators=(",", ":"))
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
