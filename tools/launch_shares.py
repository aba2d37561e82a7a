"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel share."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[hi]
idx = {h: j for j, h in enumerate(hdr)}
agg = defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) < len(hdr) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[idx["Kernel Name"]].split("(")[0].split("::")[-1]
    v = float(r[idx["Metric Value"]].replace(",", ""))
    unit = r[idx["Metric Unit"]]
    v = v * 1e3 if unit == "ms" else v / 1e3 if unit == "ns" else v
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(t for _, t in agg.values())
print(f"{'kernel':34s} {'launches':>8s} {'total_us':>12s} {'share':>7s} {'avg_us':>11s}")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:34s} {n:8d} {t:12.1f} {100 * t / tot:6.1f}% {t / n:11.1f}")
