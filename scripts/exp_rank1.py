"""Where does a configs[1] step go?  Times the torus256 estimate (k = 32, n = 1000, m = 32) as
rank-1 and as plain csr (same matrix, same tiles; csr has no u^T w reduction, so the difference
is the cost of the rank-1 synchronisation), persistent and per-step, plus gmrf32 (configs[0]).

    python scripts/exp_rank1.py [--reps 5]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

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
    return min(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--cases", default="torus256,gmrf32")
    args = ap.parse_args()
    flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
    for name in args.cases.split(","):
        wl = W.get_workload(name)
        A, _ = wl.matrices()
        dA = P.DeviceCSR.from_host(A)
        k = next(kk for kk in (8, 16, 32, 64) if kk >= wl.num_probes)
        kinds = [("rank1", wl.a, wl.b), ("csr", 1e-9, 8.0)] if wl.mode == "rank1" else [("csr", wl.a, wl.b)]
        for kind, a, b in kinds:
            op = P.Operator(kind, dA, None, wl.r1_c)
            for persist in (2, 0):
                P.set_persistent(persist)
                est = P.Estimator(op, a, b, wl.degree, wl.num_probes, k, seed=wl.seed)
                ms = t_est(est, args.reps, flush)
                print(json.dumps({"workload": name, "kind": kind, "persistent": persist, "k": k,
                                  "ms": ms, "us_per_step": 1e3 * ms / wl.degree}), flush=True)
    P.set_persistent(1)


if __name__ == "__main__":
    main()
