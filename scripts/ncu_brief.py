"""Print the handful of ncu metrics we track for a step-kernel capture (.ncu-rep).

    python scripts/ncu_brief.py gpurun_out/step_d0.ncu-rep [...]
"""
import csv
import io
import subprocess
import sys
from collections import Counter

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum", "launch__grid_size",
       "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
       "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "dram__throughput.avg.pct_of_peak_sustained_elapsed",
       "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sector_hit_rate.pct",
       "l1tex__t_sector_hit_rate.pct"]


def ncu(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True)
    return list(csv.reader(io.StringIO(out.stdout)))


def brief(rep):
    rows = ncu(rep, "raw")
    h, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(h, vals))
    u = dict(zip(h, units))
    print(f"== {rep}: {d.get('Kernel Name', '')[:80]}")
    for k in RAW:
        if k in d:
            print(f"  {k:75s} {d[k]:>18s} {u.get(k, '')}")
    src = ncu(rep, "source", ["--print-source", "sass"])
    hh = src[1]
    ie, si = hh.index("Instructions Executed"), hh.index("Source")
    c, tot = Counter(), 0
    for r in src[2:]:
        if len(r) <= ie or not r[ie]:
            continue
        n = int(r[ie])
        tot += n
        toks = r[si].split()
        op = toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")
        c[op.split(".")[0]] += n
    print(f"  warp instructions {tot}; top opcodes: " +
          ", ".join(f"{k} {v / tot:.3f}" for k, v in c.most_common(12)))


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        brief(rep)
