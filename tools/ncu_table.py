"""One line per profiled launch of an ncu report: kernel, grid, duration, DRAM bytes,
DRAM throughput, achieved occupancy, L2 hit rate (ncu -i REPORT --page raw --csv)."""
import csv
import io
import re
import subprocess
import sys

COLS = [("gpu__time_duration.sum", "us", 1e-3), ("dram__bytes_read.sum", "MB_rd", 1e-6),
        ("dram__bytes_write.sum", "MB_wr", 1e-6),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%", 1),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%", 1),
        ("lts__t_sector_hit_rate.pct", "L2hit%", 1), ("launch__registers_per_thread", "regs", 1)]
UNIT = {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9, "s": 1e9, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
        "Gbyte": 1e9, "%": 1, "register/thread": 1, "": 1}

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
print(f"{'kernel':58s} {'grid':>6s} " + " ".join(f"{c[1]:>8s}" for c in COLS))
for v in rows[2:]:
    name = v[hdr.index("Kernel Name")]
    name = re.sub(r"\(.*$", "", name.replace("void ", ""))
    name = re.sub(r"sb::", "", name)[:58]
    grid = v[hdr.index("launch__grid_size")] if "launch__grid_size" in hdr else ""
    cells = []
    for m, short, scale in COLS:
        if m not in hdr:
            cells.append(f"{'-':>8s}")
            continue
        i = hdr.index(m)
        try:
            x = float(v[i].replace(",", "")) * UNIT.get(units[i], 1) * scale
            if m.startswith("gpu__time"):
                x = float(v[i].replace(",", "")) * UNIT.get(units[i], 1) * 1e-3
            cells.append(f"{x:8.1f}")
        except ValueError:
            cells.append(f"{v[i]:>8s}")
    print(f"{name:58s} {grid:>6s} " + " ".join(cells))
