"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per-kernel
launch count, total and mean device time, and share of the captured window."""
import csv
import gzip
import re
import sys
from collections import defaultdict

rows = []
with (gzip.open(sys.argv[1], "rt") if sys.argv[1].endswith(".gz") else open(sys.argv[1])) as f:
    lines = [ln for ln in f if ln.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "")
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    us = v / 1000.0 if unit == "ns" else (v * 1000.0 if unit == "ms" else v)
    rows.append((name, us))
agg = defaultdict(lambda: [0, 0.0])
for n, us in rows:
    agg[n][0] += 1
    agg[n][1] += us
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':45s} {'launches':>8s} {'total_ms':>9s} {'mean_us':>8s} {'share':>6s}")
for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n[:45]:45s} {c:8d} {t/1e3:9.3f} {t/c:8.2f} {100*t/tot:5.1f}%")
print(f"{'TOTAL':45s} {sum(v[0] for v in agg.values()):8d} {tot/1e3:9.3f}")
