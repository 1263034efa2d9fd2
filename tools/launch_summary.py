"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) by kernel."""
import collections
import csv
import io
import re
import sys

text = open(sys.argv[1]).read()
start = text.index('"ID"')
rows = list(csv.DictReader(io.StringIO(text[start:])))
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    m = re.search(r"sb::(\w+)<", name)
    key = name if not m else m.group(1) + name[name.index("<"):name.index("<") + 90]
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3}.get(r["Metric Unit"], 1e-3)
    agg[key][0] += 1
    agg[key][1] += float(r["Metric Value"]) * scale
tot = sum(v[1] for v in agg.values())
print(f"{'launches':>8} {'total_us':>10} {'share':>6} {'avg_us':>8}  kernel")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{v[0]:8d} {v[1]:10.1f} {100 * v[1] / tot:5.1f}% {v[1] / v[0]:8.2f}  {k}")
print(f"{sum(v[0] for v in agg.values()):8d} {tot:10.1f} total")
