"""Print per-launch kernel name / grid / duration from an ncu --csv metrics log on stdin."""
import csv
import sys

rows = list(csv.reader(l for l in sys.stdin if l.startswith('"')))
hdr = rows[0]
ik, ig, im, iu, iv = (hdr.index(h) for h in ("Kernel Name", "Grid Size", "Metric Name", "Metric Unit", "Metric Value"))
for r in rows[1:]:
    if r[im] == "gpu__time_duration.sum":
        print(r[ik].split("(")[0][:40], r[ig], r[iv], r[iu])
