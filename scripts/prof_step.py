"""Small driver for ncu captures of the step kernel: one workload, a few estimates.

    python scripts/prof_step.py --workload gmrf1000 --k 64 --reps 2
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_1503_06394_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="gmrf1000")
    ap.add_argument("--k", type=int, default=64)
    ap.add_argument("--probes", type=int, default=0)
    ap.add_argument("--degree", type=int, default=0)
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    wl = W.get_workload(args.workload)
    A, At = wl.matrices()
    op = P.Operator(wl.mode, P.DeviceCSR.from_host(A), P.DeviceCSR.from_host(At) if At is not None else None,
                    wl.r1_c)
    a, b = (wl.a, wl.b) if wl.a is not None else P.bounds_btb(op)
    m = args.probes or wl.num_probes
    k = args.k or next((kk for kk in (8, 16, 32, 64) if kk >= m), 64)  # 0: the bench's choice
    est = P.Estimator(op, a, b, args.degree or wl.degree, m, k, seed=wl.seed)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for r in range(args.reps):
        ev0.record()
        gp, st = est.run()
        ev1.record()
        torch.cuda.synchronize()
        n = (args.degree or wl.degree) * m
        print(f"rep {r}: {ev0.elapsed_time(ev1):.2f} ms  {n / ev0.elapsed_time(ev1) * 1e3:.1f} probe-steps/s "
              f"gamma={st[0].item():.6f}", flush=True)


if __name__ == "__main__":
    main()
