"""trigrid command line on the B200 (mirrors tools/trigrid_main.cpp:1-258).

    python -m paper_1308_1419_b200.cli bench     [--strategies ...] [--kernel dummy|edm|write] ...
    python -m paper_1308_1419_b200.cli verify    [--strategy all] [--n-max 256] [--rho 16]
    python -m paper_1308_1419_b200.cli exactness [--engine ltm-r] [--n 30720] [--rho 16] [--device-fixup]
    python -m paper_1308_1419_b200.cli edm       [--n 1024] [--features 1] [--strategy reference] [--out f.pedm] [--check]

Same subcommands, options, defaults and exit codes (0 success, 1
verification failure, 2 configuration error) as the reference CLI.
Additions: --mode (grid | span | auto) and --kernel write for bench; the
GPU-only columns go to <out>.gpu.csv and the improvement-model fit to
<out>.fit.json.
"""
from __future__ import annotations

import argparse
import json
import sys

CHECK_HOST_CAP = 8192  # --check: points up to which the sequential host edm_reference is the checker


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # configuration errors exit 2 like CLI11's
        self.print_usage(sys.stderr)
        sys.stderr.write(f"error: {message}\n")
        raise SystemExit(2)


def _strategy_list(csv: str):
    from . import trigrid as tg
    names = [s for s in csv.split(",") if s]
    for s in names:
        if s not in ("bb", "ltm-x", "ltm-n", "ltm-r", "utm", "rb", "rec", "ltm-exact"):
            raise ValueError(f"--strategies: unknown strategy '{s}'")
    if not names:
        raise ValueError("--strategies: no strategies selected")
    del tg
    return names


def run_bench(a) -> int:
    from . import suite
    if a.kernel not in ("dummy", "edm", "write"):
        raise ValueError("--kernel: expected dummy, edm or write")
    n_end = a.n_end or (8192 if a.kernel == "edm" else 30720)
    if a.n_start == 0 or a.n_step == 0 or n_end < a.n_start:
        raise ValueError("--n-start/--n-end/--n-step: bad sweep range")
    cfg = suite.BenchConfig(strategies=_strategy_list(a.strategies), n_values=list(range(a.n_start, n_end + 1, a.n_step)),
                            rho=a.rho, kernel=a.kernel, features=a.features, repetitions=a.reps,
                            seed=a.seed, verify_cap=a.verify_cap, mode=a.mode)
    res = suite.run_suite(cfg)
    for s in res.skipped:
        sys.stderr.write(f"skipped: {s}\n")
    suite.emit_csv(res.records, a.out)
    if res.gpu_rows:
        suite.emit_gpu_csv(res.gpu_rows, a.out + ".gpu.csv")
    with open(a.out + ".fit.json", "w") as f:
        json.dump(suite.fit_improvement_model(res.records), f, indent=1)
    print(f"wrote {len(res.records)} records to {a.out} ({len(res.skipped)} skipped)")
    if not res.all_verified:
        sys.stderr.write("EDM verification FAILED for at least one row group\n")
        return 1
    return 0


def run_verify(a) -> int:
    from . import checks
    ok, lines = checks.verify_strategies(a.strategy, a.n_max, a.rho)
    for ln in lines:
        print(ln)
    print("verify: all checks passed" if ok else "verify: FAILED")
    return 0 if ok else 1


def run_exactness(a) -> int:
    from . import checks
    engines = {"ltm-x": "native", "ltm-n": "newton", "ltm-r": "reciprocal"}
    if a.engine not in engines:
        raise ValueError("--engine: expected ltm-x, ltm-n or ltm-r")
    ok = True
    for diag, checked, mism, first in checks.exactness(engines[a.engine], a.n, a.rho):
        line = f"{a.engine}, {'with' if diag else 'no'} diagonal: {checked} lambdas checked, {mism} mismatches"
        if mism:
            line += f" (first at lambda={first})"
            ok = False
        print(line)
    print("exactness: " + ("exact over the full range" if ok else "FAILED"))
    return 0 if ok else 1


def run_edm(a) -> int:
    import torch

    from . import pedm
    from . import trigrid as tg
    pts = tg.gen_values(a.n * a.features, a.seed).view(a.n, a.features)
    if a.strategy == "reference":
        out = tg.edm(pts, strategy="ltm-exact", rho=a.rho, mode="grid")
    else:
        if a.strategy not in ("bb", "ltm-x", "ltm-n", "ltm-r", "utm", "rb", "rec"):
            raise ValueError(f"--strategy: unknown strategy '{a.strategy}'")
        out = torch.empty(tg.tri_count(a.n), dtype=torch.float32, device=pts.device)
        st = tg.launch("edm", a.strategy, a.n, points=pts, out=out, d=a.features, rho=a.rho, mode=a.mode)
        print(f"{a.strategy}: {st['blocks_launched']} blocks launched, {st['blocks_discarded']} discarded, "
              f"{st['wall_time_ns'] / 1e6:.3f} ms")
    if a.out:
        pedm.save_packed_edm(out, a.n, a.features, a.out)
        print(f"wrote {out.numel()} packed cells to {a.out}")
    if a.check:
        # sequential host edm_reference (edm.cpp:53-63) up to CHECK_HOST_CAP points (independent of
        # every device kernel); above it a GPU self-consistency check against the grid ltm-exact kernel
        host_check = a.n <= CHECK_HOST_CAP
        if host_check:
            ref = torch.from_numpy(tg.edm_reference(pts.cpu().numpy())).to(pts.device)
        else:
            ref = tg.edm(pts, strategy="ltm-exact", rho=a.rho, mode="grid")
        what = "host edm_reference check" if host_check else "GPU self-check (grid ltm-exact kernel, not an oracle)"
        if a.mode == "gram":  # stated tolerance, not bit-exact
            nrm = (pts.double() ** 2).sum(1)
            ok, worst = True, 0.0
            for r0 in range(0, a.n, 1024):  # row blocks of the packed layout
                r1 = min(a.n, r0 + 1024)
                e0, e1 = r0 * (r0 + 1) // 2, r1 * (r1 + 1) // 2
                i = torch.repeat_interleave(torch.arange(r0, r1, device=pts.device),
                                            torch.arange(r0 + 1, r1 + 1, device=pts.device))
                j = torch.arange(e0, e1, device=pts.device) - i * (i + 1) // 2
                err = (out[e0:e1].double() ** 2 - ref[e0:e1].double() ** 2).abs()
                ratio = err / (2.0 ** -17 * (nrm[i] + nrm[j])).clamp_min(1e-300)
                worst = max(worst, float(ratio.max()))
                ok = ok and bool((out[e0:e1][i == j] == 0).all())
            ok = ok and worst <= 1.0
            print(f"{what} (gram tolerance |d^2 - d_exact^2| <= 2^-17 (|x_i|^2 + |x_j|^2)): "
                  f"max err/bound = {worst:.3g} -> " + ("within tolerance" if ok else "OUT OF TOLERANCE"))
            return 0 if ok else 1
        same = bool(torch.equal(out.view(torch.int32), ref.view(torch.int32)))
        print(f"{what}: " + ("bitwise identical" if same else "MISMATCH"))
        if not same:
            return 1
    return 0


def main(argv=None) -> int:
    p = _Parser(prog="trigrid", description="Grid-to-triangular-domain mapping strategies on B200")
    sub = p.add_subparsers(dest="cmd", required=True, parser_class=_Parser)
    b = sub.add_parser("bench", help="Sweep N and emit benchmark CSV")
    b.add_argument("--strategies", default="bb,ltm-x,ltm-n,ltm-r,utm,rb,rec")
    b.add_argument("--kernel", default="dummy")
    b.add_argument("--features", type=int, default=1)
    b.add_argument("--n-start", type=int, default=1024)
    b.add_argument("--n-end", type=int, default=0)
    b.add_argument("--n-step", type=int, default=1024)
    b.add_argument("--rho", type=int, default=16)
    b.add_argument("--reps", type=int, default=5)
    b.add_argument("--workers", default="AUTO")
    b.add_argument("--seed", type=int, default=42)
    b.add_argument("--verify-cap", type=int, default=1024)
    b.add_argument("--out", default="results.csv")
    b.add_argument("--mode", default="auto", choices=["auto", "grid", "span"])
    v = sub.add_parser("verify", help="Exhaustive bijection oracle")
    v.add_argument("--strategy", default="all")
    v.add_argument("--n-max", type=int, default=256)
    v.add_argument("--rho", type=int, default=16)
    v.add_argument("--workers", default="AUTO")
    e = sub.add_parser("exactness", help="Row-exactness lambda sweep")
    e.add_argument("--engine", default="ltm-r")
    e.add_argument("--n", type=int, default=30720)
    e.add_argument("--rho", type=int, default=16)
    m = sub.add_parser("edm", help="Compute a packed distance matrix")
    m.add_argument("--n", type=int, default=1024)
    m.add_argument("--features", type=int, default=1)
    m.add_argument("--seed", type=int, default=42)
    m.add_argument("--strategy", default="reference")
    m.add_argument("--rho", type=int, default=16)
    m.add_argument("--workers", default="AUTO")
    m.add_argument("--out", default="")
    m.add_argument("--check", action="store_true")
    m.add_argument("--mode", default="auto", choices=["auto", "grid", "span", "gram"])
    a = p.parse_args(argv)
    try:
        return {"bench": run_bench, "verify": run_verify, "exactness": run_exactness, "edm": run_edm}[a.cmd](a)
    except ValueError as exc:
        sys.stderr.write(f"error: {exc}\n")
        return 2


if __name__ == "__main__":
    sys.exit(main())
