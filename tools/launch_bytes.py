"""Per-kernel launch totals from an ncu --csv launch list that carries
gpu__time_duration.sum, dram__bytes_read.sum and dram__bytes_write.sum: launches,
average duration, average DRAM bytes and the DRAM GB/s they imply (cold-cache,
serialised launches: compare with the live CUDA-event timings, not as absolutes)."""
import csv
import re
import sys
from collections import OrderedDict

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
         "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
iK, iN, iU, iV, iID = (h.index(c) for c in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
launch = OrderedDict()
for r in rows[1:]:
    d = launch.setdefault(r[iID], {"k": r[iK]})
    d[r[iN]] = float(r[iV].replace(",", "")) * SCALE.get(r[iU], 1.0)
# host-polled solver loops launch whole chunks, and the launches after the stop are
# no-ops: per kernel, only launches longer than 10% of its longest one are counted
per = OrderedDict()
for d in launch.values():
    k = re.sub(r"\(.*$", "", d["k"].replace("void ", "")).replace("sb::", "")[:70]
    per.setdefault(k, []).append(d)
agg = OrderedDict()
for k, ds in per.items():
    tmax = max(d.get("gpu__time_duration.sum", 0.0) for d in ds)
    a = agg.setdefault(k, [0, 0.0, 0.0])
    for d in ds:
        if d.get("gpu__time_duration.sum", 0.0) < 0.1 * tmax:
            continue
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
print(f"{'active':>8s} {'share':>6s} {'avg_us':>9s} {'avg_MB':>9s} {'GB/s':>7s}  kernel")
for k, (n, us, mb) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n:8d} {100 * us / tot:5.1f}% {us / n:9.2f} {mb / n:9.2f} {mb / us * 1e3 if us else 0:7.0f}  {k}")
