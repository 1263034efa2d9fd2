"""DRAM traffic JSON (profiles/r2_*_traffic.json) from an ncu --set full report of one
launch: python tools/traffic_json.py REPORT KERNEL_REGEX OUT [iterations] [alg_bytes]"""
import csv
import io
import json
import re
import subprocess
import sys

rep, pat, out = sys.argv[1], sys.argv[2], sys.argv[3]
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 1
alg = int(sys.argv[5]) if len(sys.argv) > 5 else None
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3,
        "ns": 1e-3, "nsecond": 1e-3}
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h, u = rows[0], rows[1]
row = next(r for r in rows[2:] if re.search(pat, r[h.index("Kernel Name")]))
val = lambda m: float(row[h.index(m)].replace(",", "")) * UNIT.get(u[h.index(m)], 1)
rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
rec = {"kernel": re.sub(r"\(.*$", "", row[h.index("Kernel Name")]).replace("void ", ""), "source": f"ncu --set full --clock-control none ({rep.split('/')[-1]})",
       "dram_bytes_read": int(rd), "dram_bytes_write": int(wr), "ncu_duration_us": val("gpu__time_duration.sum")}
if iters > 1:
    rec.update({"iterations": iters, "traffic_per_iteration": int((rd + wr) / iters),
                "algorithmic_bytes_per_iteration": alg})
else:
    rec.update({"traffic": int(rd + wr), "algorithmic_bytes": alg})
json.dump(rec, open(out, "w"), indent=1)
print(json.dumps(rec))
