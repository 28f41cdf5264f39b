"""Shared-memory-resident kernel vs the L2-resident persistent kernel vs per-step launches:
per-estimate time (CUDA events, min over reps) and the largest moment difference between the
schedules (w_j is bit-identical; the dot products differ only in summation order).

    python scripts/exp_resident.py [--cases torus256,gmrf32] [--ks 16,32,64] [--reps 5]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_1503_06394_b200 as P  # noqa: E402


def t_est(est, reps, flush):
    est.run(check=True)
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        est.run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    est.run(check=True)
    return min(ts), est.mu.cpu().numpy().copy()


SCHED = {"resident": (1, 1), "persistent": (2, 0), "per_step": (0, 0)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--cases", default="torus256,gmrf32")
    ap.add_argument("--ks", default="16,32,64")
    ap.add_argument("--scheds", default="resident,persistent,per_step")
    ap.add_argument("--doubling", action="store_true", help="also time moment doubling (G25) on each schedule")
    args = ap.parse_args()
    flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
    for name in args.cases.split(","):
        wl = W.get_workload(name)
        A, _ = wl.matrices()
        dA = P.DeviceCSR.from_host(A)
        op = P.Operator(wl.mode, dA, None, wl.r1_c)
        for k in [int(x) for x in args.ks.split(",")]:
            mus = {}
            for sname, dbl in [(x, d) for d in ([False, True] if args.doubling else [False])
                               for x in args.scheds.split(",")]:
                pers, res = SCHED[sname]
                P.set_persistent(pers)
                P.set_resident(res)
                P.set_doubling(dbl)
                est = P.Estimator(op, wl.a, wl.b, wl.degree, wl.num_probes, k, seed=wl.seed)
                ms, mu = t_est(est, args.reps, flush)
                P.set_doubling(False)
                mus[sname] = mu
                ref = mus[args.scheds.split(",")[0]]
                diff = float(np.abs(mu - ref).max() / max(1.0, np.abs(ref).max()))
                print(json.dumps({"workload": name, "k": k, "schedule": sname + ("+doubling" if dbl else ""), "m": wl.num_probes, "n": wl.degree,
                                  "ms": round(ms, 4), "us_per_step": round(1e3 * ms / wl.degree / -(-wl.num_probes // k), 3),
                                  "probe_steps_per_s": wl.num_probes * wl.degree / ms * 1e3,
                                  "max_rel_diff_vs_first": diff}), flush=True)
    P.set_persistent(1)
    P.set_resident(1)


if __name__ == "__main__":
    main()
