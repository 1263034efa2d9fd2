"""Per-kernel averages of an ncu --csv launch list with several metrics per launch."""
import collections
import csv
import io
import re
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
         "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
text = open(sys.argv[1]).read()
rows = list(csv.DictReader(io.StringIO(text[text.index('"ID"'):])))
agg = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
for r in rows:
    name = r["Kernel Name"]
    m = re.search(r"sb::(\w+)<", name)
    key = (m.group(1) if m else name)[:28] + name[name.find("<"):name.find("<") + 56]
    v = float(r["Metric Value"].replace(",", "")) * SCALE.get(r["Metric Unit"], 1.0)
    if r["Metric Name"] == "gpu__time_duration.sum":
        cnt[key] += 1
    agg[key][r["Metric Name"]] += v
tot = sum(d["gpu__time_duration.sum"] for d in agg.values())
for k, d in sorted(agg.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"])[:8]:
    n = max(cnt[k], 1)
    extra = " ".join(f"{m.split('__')[-1][:22]}={v / n:.1f}" for m, v in d.items()
                     if m not in ("gpu__time_duration.sum",))
    print(f"{n:5d} {d['gpu__time_duration.sum'] / n:8.2f}us {100 * d['gpu__time_duration.sum'] / tot:5.1f}%  {k}\n        {extra}")
