"""Summarise scripts/sweep_step.sh output: per (doubling, occupancy) the mean ncu launch time,
DRAM GB per launch, grid, and the timed probe-steps/s of prof_step.py."""
import csv
import glob
import io
import os
import re
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
for f in sorted(glob.glob(os.path.join(d, "sweep_*.csv"))):
    tag = os.path.basename(f)[6:-4]
    txt = open(f).read()
    i = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[i:]))) if i >= 0 else []
    m = {}
    for r in rows:
        try:
            v = float(r["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        m.setdefault(r["Metric Name"], []).append((v, r["Metric Unit"]))
    def avg(k, scale=1.0):
        xs = m.get(k, [])
        return sum(x for x, _ in xs) / len(xs) * scale if xs else float("nan")
    units = {k: v[0][1] for k, v in m.items() if v}
    tu = units.get("gpu__time_duration.sum", "")
    t = avg("gpu__time_duration.sum", {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3}.get(tu, 1.0))
    gb = sum(avg(k, 1.0 if units.get(k) == "Gbyte" else 1e-3 if units.get(k) == "Mbyte" else 1e-9)
             for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    txt = f.replace("sweep_", "var_")[:-4] + ".txt"
    if not os.path.exists(txt):
        txt = f[:-4] + ".txt"
    ps = re.findall(r"([\d.]+) probe-steps/s", open(txt).read()) if os.path.exists(txt) else []
    inst = avg("smsp__inst_executed.sum") / 1e9
    print(f"{tag:10s} launch {t:7.3f} ms  dram {gb:6.2f} GB  grid {avg('launch__grid_size'):5.0f}  inst {inst:5.2f}e9  "
          f"timed probe-steps/s {ps[-1] if ps else '-'}")
