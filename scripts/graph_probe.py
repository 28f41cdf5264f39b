"""Does one whole estimate (prep, init, n fused steps per block, finalize) capture into a CUDA graph
through the C ABI, and what does replay save?  python scripts/graph_probe.py --workload gmrf1000"""
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
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    wl = W.get_workload(args.workload)
    A, At = wl.matrices()
    op = P.Operator(wl.mode, P.DeviceCSR.from_host(A), P.DeviceCSR.from_host(At) if At is not None else None, wl.r1_c)
    a, b = (wl.a, wl.b) if wl.a is not None else P.bounds_btb(op)
    m = wl.num_probes
    k = next((kk for kk in (8, 16, 32, 64) if kk >= m), 64)
    est = P.Estimator(op, a, b, wl.degree, m, k, seed=wl.seed)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        gp, st = est.run()
    torch.cuda.synchronize()
    ref = st.clone()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        ev0.record(s)
        for _ in range(args.reps):
            gp, st = est.run()
        ev1.record(s)
    torch.cuda.synchronize()
    t_eager = ev0.elapsed_time(ev1) / args.reps
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        gp_g, st_g = est.run()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        g.replay()
        ev0.record(s)
        for _ in range(args.reps):
            g.replay()
        ev1.record(s)
    torch.cuda.synchronize()
    t_graph = ev0.elapsed_time(ev1) / args.reps
    same = bool(torch.equal(st_g, ref))
    print(f"{args.workload}: eager {t_eager:.3f} ms, graph replay {t_graph:.3f} ms, identical stats {same}")


if __name__ == "__main__":
    main()
