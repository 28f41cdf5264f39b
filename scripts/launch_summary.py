"""Per-kernel shares of an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv
--log-file X`): writes a JSON summary next to it.

    python scripts/launch_summary.py profiles/r01_launches.csv profiles/r01_launches_summary.json "source text"
"""
import csv
import io
import json
import sys
from collections import OrderedDict


def main(src, dst, source):
    txt = open(src).read()
    i = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[i:])))
    k = OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r["Metric Unit"], 1.0)
        e = k.setdefault(r["Kernel Name"], [0, 0.0])
        e[0] += 1
        e[1] += v * scale
    tot = sum(e[1] for e in k.values())
    out = {"source": source, "kernels": {n: {"launches": e[0], "total_us": round(e[1], 1),
                                              "mean_us": round(e[1] / e[0], 2), "share": round(e[1] / tot, 4)}
                                          for n, e in sorted(k.items(), key=lambda x: -x[1][1])}}
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out, indent=1)[:1500])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
