"""The reference's verification suite on the GPU (checks.cpp:115-206):
exhaustive cell coverage per strategy (COUNT kernel on device, exactly-once,
diagonal untouched for utm), g(lambda) block bijection per engine (device
lambda sweep with the integer fix-up), and the float-only exactness sweep
(checks.cpp:81-95) on device for any N.

Difference: the reference's REC sweep enumerates every (m, k) with
N = m*2^k (checks.cpp:151-173); the drop-in REC strategy always uses the
largest-k decomposition (make_strategy, strategies.cpp:200-206), so the GPU
sweep covers every decomposable N <= 2*n_max with that schedule.
"""
from __future__ import annotations

from . import trigrid as tg


def _note(lines, ok, text, detail=""):
    lines.append(("ok   " if ok else "FAIL ") + text + ("" if ok or not detail else " -- " + detail))
    return ok


def _coverage_sweep(lines, strat, n_min, n_max, rho):
    ok_all = True
    for r in (rho, 1):
        first = ""
        fails = 0
        for n in range(n_min, n_max + 1):
            if not tg.coverage_ok(strat, n, r):
                fails += 1
                first = first or f"N={n}"
        ok_all &= _note(lines, fails == 0, f"{strat} cell coverage, N in [{n_min}, {n_max}], rho={r}", first)
    return ok_all


def verify_strategies(which: str = "all", n_max: int = 256, rho: int = 16):
    lines: list[str] = []
    ok = True
    every = which == "all"
    if every or which == "bb":
        ok &= _coverage_sweep(lines, "bb", 1, n_max, rho)
    if every or which in ("ltm", "ltm-x", "ltm-n", "ltm-r"):
        all_eng = every or which == "ltm"
        engines = {"ltm-x": "native", "ltm-n": "newton", "ltm-r": "reciprocal"}
        sel = ["native", "newton", "reciprocal", "exact"] if all_eng else [engines[which]]
        for e in sel:
            for diag in (True, False):
                total = tg.tri_count(n_max, diag)
                m, first = tg.lambda_sweep(e, 0, total, with_diag=diag, fixup=True)
                ok &= _note(lines, m == 0, f"ltm block bijection, {e}, "
                            f"{'with diagonal' if diag else 'no diagonal'} (lambda < {total})",
                            f"first bad lambda {first}")
        ok &= _coverage_sweep(lines, "ltm-r" if all_eng else which, 1, n_max, rho)
    if every or which == "utm":
        ok &= _coverage_sweep(lines, "utm", 1, n_max, rho)
    if every or which == "rb":
        ok &= _coverage_sweep(lines, "rb", 2, n_max, rho)
    if every or which == "rec":
        for r in (rho, 1):
            cfgs = fails = 0
            first = ""
            for n in range(1, 2 * n_max + 1):
                if tg.rec_decompose(n, r) is None:
                    continue
                cfgs += 1
                if not tg.coverage_ok("rec", n, r):
                    fails += 1
                    first = first or f"N={n}"
            ok &= _note(lines, fails == 0, f"rec cell coverage, {cfgs} N values, N <= {2 * n_max}, rho={r}", first)
    if not lines:
        return False, [f"FAIL unknown strategy selector '{which}'"]
    return ok, lines


def exactness(engine: str, n_elems: int, rho: int = 16):
    """ltm_exactness_sweep (checks.cpp:81-95) on device: float row only
    (no fix-up) over every lambda of the n-block grid, both diagonal modes.
    Returns [(with_diag, checked, mismatches, first)]."""
    nb = (n_elems + rho - 1) // rho
    out = []
    for diag in (True, False):
        total = tg.tri_count(nb, diag)
        m, first = tg.lambda_sweep(engine, 0, total, with_diag=diag, fixup=False)
        out.append((diag, total, m, first))
    return out
