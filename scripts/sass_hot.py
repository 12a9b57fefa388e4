"""Per-instruction SASS listing of an ncu source-page export with stall samples.

    python scripts/sass_hot.py gpurun_out/prof_X.source.csv [--min 50] [--top 40]
"""
import csv
import sys


def main():
    path = sys.argv[1]
    mn = int(sys.argv[sys.argv.index("--min") + 1]) if "--min" in sys.argv else 0
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 0
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    recs = []
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        try:
            smp = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
            ex = int(r[ix["Instructions Executed"]] or 0)
        except ValueError:
            continue
        st = sorted(((int(r[ix[h]] or 0), h[6:]) for h in stall_cols), reverse=True)[:3]
        recs.append((r[ix["Address"]], r[ix["Source"]], smp, ex, st))
    total = sum(x[2] for x in recs) or 1
    if top:
        for a, s, smp, ex, st in sorted(recs, key=lambda x: -x[2])[:top]:
            print(f"{a:>6} {smp:7d} {100*smp/total:5.1f}% ex={ex:10d} {s[:60]:60s} {' '.join(f'{n}:{v}' for v, n in st if v)}")
        return
    for a, s, smp, ex, st in recs:
        if smp >= mn:
            print(f"{a:>6} {smp:7d} {100*smp/total:5.1f}% ex={ex:10d} {s[:60]:60s} {' '.join(f'{n}:{v}' for v, n in st if v)}")


if __name__ == "__main__":
    main()
