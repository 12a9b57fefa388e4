"""Summarise ncu captures into profiles/ (tracked).

    python scripts/ncu_summary.py <tag> gpurun_out/prof_span_edm.ncu-rep [...] \
        [--launches gpurun_out/launches.csv] [--traffic-key edm_ltm-r_n65536_d3_g1]

Writes profiles/<tag>_<kernel>.md with the metrics the roofline needs
(duration, DRAM bytes read/written, DRAM %, issue %, pipe utilisation,
registers, occupancy, top stall reasons) and, for --launches, a per-kernel
share table of the launch list.  --traffic-key records dram read+write bytes
of the first report into profiles/traffic.json for bench.py's roofline.traffic.
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM bandwidth % of peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__inst_executed.sum", "instructions executed"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid size"),
    ("launch__block_size", "block size"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__cycles_elapsed.avg.per_second", "DRAM clock"),
]


def _page(rep: str, page: str) -> str:
    """A report page as CSV text: from the .ncu-rep, or from the <prefix>.<page>.csv
    export gpu_round.sh writes on the GPU box (reports are too big to bring back)."""
    if rep.endswith(".ncu-rep"):
        extra = ["--print-source=sass"] if page == "source" else []
        return subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True,
                              text=True).stdout
    path = f"{rep}.{page}.csv"
    return open(path).read() if os.path.exists(path) else ""


def raw(rep: str):
    out = _page(rep, "raw")
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return None
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        kernels.append({h: (v, u) for h, v, u in zip(hdr, vals, units)})
    return kernels


def stalls(rep: str):
    out = _page(rep, "details")
    res = []
    for r in csv.reader(io.StringIO(out)):
        if len(r) > 14 and r[11] in ("Warp State Statistics", "Scheduler Statistics", "Compute Workload Analysis",
                                     "Memory Workload Analysis", "Occupancy", "GPU Speed Of Light Throughput"):
            res.append((r[11], r[12], r[13], r[14]))
    return res


def summarise(tag: str, rep: str) -> tuple[str, dict]:
    ks = raw(rep)
    if not ks:
        return "", {}
    k = ks[0]
    name = k.get("Kernel Name", ("?", ""))[0]
    short = name.split("(")[0].replace("void ", "").replace("tg::", "")
    lines = [f"# {tag}: `{name}`", "", f"source: `{os.path.relpath(rep, ROOT)}` (ncu --set full, --clock-control none)", "",
             "| metric | value | unit |", "|---|---|---|"]
    vals = {}
    for m, label in METRICS:
        if m in k:
            v, u = k[m]
            vals[m] = (v, u)
            lines.append(f"| {label} (`{m}`) | {v} | {u} |")
    lines += ["", "## scheduler / warp state / workload", "", "| section | metric | unit | value |", "|---|---|---|---|"]
    for sec, met, unit, val in stalls(rep):
        if met:
            lines.append(f"| {sec} | {met} | {unit} | {val} |")
    stall_cols = [m for m in k if m.startswith("smsp__pcsamp_warps_issue_stalled_") and not m.endswith("not_issued")]
    samp = []
    for m in stall_cols:
        try:
            samp.append((float(k[m][0].replace(",", "")), m.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
    tot = sum(v for v, _ in samp) or 1.0
    if samp:
        lines += ["", "## warp stall samples (all warps)", "", "| reason | samples | share |", "|---|---|---|"]
        for v, nm in sorted(samp, reverse=True)[:10]:
            lines.append(f"| {nm} | {v:.0f} | {100 * v / tot:.1f}% |")
    src = _page(rep, "source")
    if src:
        rows = list(csv.reader(io.StringIO(src)))
        hi = next((i for i, r in enumerate(rows) if "Instructions Executed" in r), None)
        if hi is not None:
            hdr = rows[hi]
            ia, ss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
            agg, tot_i = defaultdict(lambda: [0, 0]), 0
            for r in rows[hi + 1:]:
                if len(r) <= max(ia, ss) or not r[ia].isdigit():
                    continue
                toks = r[1].strip().split()
                op = (toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "?"))
                op = op.split(".")[0]
                agg[op][0] += int(r[ia])
                agg[op][1] += int(r[ss] or 0) if r[ss].isdigit() else 0
                tot_i += int(r[ia])
            lines += ["", f"## SASS instruction mix ({tot_i} warp instructions executed)", "",
                      "| opcode | executed | share | stall samples |", "|---|---|---|---|"]
            for op, (c, st) in sorted(agg.items(), key=lambda x: -x[1][0])[:16]:
                lines.append(f"| {op} | {c} | {100 * c / max(tot_i, 1):.1f}% | {st} |")
    return "\n".join(lines) + "\n", {"kernel": name, "short": short, **{m: v for m, (v, _) in vals.items()}}


def launches_table(path: str) -> str:
    text = open(path).read().splitlines()
    start = next(i for i, ln in enumerate(text) if ln.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(text[start:]))))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        v_us = v / 1e3 if unit in ("nsecond", "ns") else (v * 1e3 if unit in ("msecond", "ms") else v)
        agg[name][0] += 1
        agg[name][1] += v_us
    tot = sum(t for _, t in agg.values()) or 1.0
    lines = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for name, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{name}` | {c} | {t:.1f} | {100 * t / tot:.1f}% |")
    return "\n".join(lines) + "\n"


def to_bytes(v: str, unit: str) -> float:
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def main():
    args = sys.argv[1:]
    tag = args.pop(0)
    launches = traffic_key = None
    if "--launches" in args:
        k = args.index("--launches")
        launches = args[k + 1]
        del args[k:k + 2]
    if "--traffic-key" in args:
        k = args.index("--traffic-key")
        traffic_key = args[k + 1]
        del args[k:k + 2]
    os.makedirs(PROF, exist_ok=True)
    first = None
    for rep in args:
        md, vals = summarise(tag, rep)
        if not md:
            continue
        out = os.path.join(PROF, f"{tag}_{vals['short'].split('<')[0]}.md")
        open(out, "w").write(md)
        print("wrote", out)
        first = first or (rep, vals)
    if launches:
        out = os.path.join(PROF, f"{tag}_launches.md")
        open(out, "w").write(f"# {tag}: launch list (ncu gpu__time_duration.sum, cold-cache, serialised)\n\n"
                             f"source: `{os.path.relpath(launches, ROOT)}`\n\n" + launches_table(launches))
        print("wrote", out)
    if traffic_key and first:
        rep, _ = first
        k = raw(rep)[0]
        rd = to_bytes(*k["dram__bytes_read.sum"])
        wr = to_bytes(*k["dram__bytes_write.sum"])
        tp = os.path.join(PROF, "traffic.json")
        d = json.load(open(tp)) if os.path.exists(tp) else {}
        d[traffic_key] = rd + wr
        json.dump(d, open(tp, "w"), indent=1)
        print("traffic", traffic_key, rd + wr)


if __name__ == "__main__":
    main()
