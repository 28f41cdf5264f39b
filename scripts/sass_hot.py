"""Hottest SASS lines (warp stall samples) of an ncu source-page CSV (gz ok).

    python scripts/sass_hot.py gpurun_out/x_sass.csv.gz [N]
"""
import csv
import gzip
import io
import sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
f = io.TextIOWrapper(gzip.open(path)) if path.endswith(".gz") else open(path)
rows = list(csv.reader(f))
h = rows[1]
ia, isrc, iss, iex = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
body = [r for r in rows[2:] if len(r) > iss and r[iss].strip().isdigit()]
tot = sum(int(r[iss]) for r in body)
print("total samples", tot, "instructions", len(body))
for idx, r in sorted(enumerate(body), key=lambda t: -int(t[1][iss]))[:n]:
    print(f"{idx:5d} {int(r[iss]):7d} {100 * int(r[iss]) / tot:5.1f}%  ex={r[iex]:>8s}  {r[isrc].strip()}")
