"""Measurements for the SURVEY §8(f) rows (one JSON line each; device time via CUDA events):

  f1  paper §5.1 scaling sweep: Algorithm 2 (B^T B, m=10, n=15) on the paper's random SPD
      generator for d = 1e3 .. 3e7 (Fig. 1(a) analogue; the paper: 500 s at d = 3e7)
  f2  GMRF rho-likelihood scan at 5000 x 5000 (BASELINE configs[3] matrix): 8 thetas x 64 probes,
      batched (one pass serves all thetas) vs separate estimates
  f3  Taylor baseline on configs[3] (power recurrence on the same kernels)
  f4  spectral-bound estimate (block power iteration) on configs[3]

    python scripts/bench_extras.py [f1 f2 f3 f4]
"""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_1503_06394_b200 as P  # noqa: E402


def timed(fn, reps=3, warm=1):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return float(np.median(ts))


def f1():
    for d in (1_000, 10_000, 100_000, 1_000_000, 3_000_000, 10_000_000, 30_000_000):
        t0 = time.perf_counter()
        C = W.random_spd(d, 1, device="cuda")
        gen = time.perf_counter() - t0
        dC = P.DeviceCSR.from_host(C)
        op = P.Operator("btb", dC, dC)
        a, b = P.bounds_btb(op)
        est = P.Estimator(op, a, b, 15, 10, 16, seed=1)
        t = timed(lambda: est.run(), reps=3)
        st = est.run()[1].cpu().numpy()
        print(json.dumps({"row": "f1", "what": "paper §5.1 Alg. 2 (m=10, n=15)", "d": d, "nnz": int(C.nnz),
                          "seconds": t, "probe_steps_per_s": 150 / t, "generate_s": gen,
                          "log_abs_det_C": 0.5 * float(st[0]),
                          "paper": "500 s at d=3e7 on a 3.40 GHz i7 (P:601-606)"}), flush=True)
        del est, op, dC, C
        torch.cuda.empty_cache()


def _gmrf5000():
    wl = W.get_workload("gmrf5000")
    A, _ = wl.matrices()
    return wl, A


def f2():
    """5000 x 5000 GMRF likelihood scan, 8 thetas, n = 100: members batched in the columns of each
    probe block (cheb_family_moments) vs one estimate per member (shared workspace), at 64 and at
    16 probes per member."""
    import paper_1503_06394_b200.gmrf as G
    base = W.grid_gmrf(5000, 1.0)
    fam = G.PrecisionFamily(P.DeviceCSR.from_host(base))
    x = torch.randn(base.n_rows, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(0))
    thetas = np.linspace(-0.24, -0.20, 8)
    for m in (64, 16):
        out = {"row": "f2", "what": f"rho-likelihood scan, 5000x5000 GMRF, 8 thetas x {m} probes, n=100"}
        for batched in (True, False):
            t = timed(lambda: G.likelihood_scan(fam, thetas, [x], 100, m, seed=1, batched=batched), reps=2, warm=1)
            key = "batched" if batched else "separate"
            out[f"{key}_scan_seconds"] = t
            out[f"{key}_probe_steps_per_s"] = 8 * m * 100 / t
        out["batched_probe_block"] = G.scan_probe_block(8, m)
        print(json.dumps(out), flush=True)


def f3():
    wl, A = _gmrf5000()
    op = P.Operator("csr", P.DeviceCSR.from_host(A))
    est = P.Estimator(op, wl.a, wl.b, 100, 128, 64, seed=1, basis="taylor")
    P.profile_begin()
    t = timed(lambda: est.run(), reps=2)
    prof = P.profile_end()
    ms, nl = prof["single"]
    d, nnz, k = wl.d, A.nnz, 64
    bytes_launch = 12 * nnz + 8 * (d + 1) + 16 * d * k + d * 8
    print(json.dumps({"row": "f3", "what": "Taylor baseline on configs[3] (power recurrence), n=100, m=128",
                      "seconds": t, "probe_steps_per_s": 128 * 100 / t,
                      "step_kernel_GBps": bytes_launch / (ms / nl / 1e3) / 1e9}), flush=True)


def f4():
    """Lanczos spectral interval of configs[3] (cheb_spectrum_bounds), and the estimate on it vs the
    closed-form interval (same probes)."""
    wl, A = _gmrf5000()
    op = P.Operator("csr", P.DeviceCSR.from_host(A))
    lam_max = 1 + 4 * 0.24 * math.cos(math.pi / 5001)
    for steps in (50, 100):
        res = {}
        t = timed(lambda: res.update(P.spectrum_bounds(op, steps, 8, seed=77)), reps=1)
        ra = P.logdet(op, res["a"], res["b"], wl.degree, wl.num_probes, seed=wl.seed, k=64)
        rc = P.logdet(op, wl.a, wl.b, wl.degree, wl.num_probes, seed=wl.seed, k=64)
        print(json.dumps({"row": "f4", "what": f"Lanczos bounds on configs[3], {steps} steps x 8 probes",
                          "seconds": t, **res, "closed_form_lambda_max": lam_max,
                          "closed_form_lambda_min": 2 - lam_max, "gamma_on_lanczos_interval": ra.logdet,
                          "gamma_on_closed_form_interval": rc.logdet, "stderr": rc.stderr}), flush=True)


if __name__ == "__main__":
    rows = sys.argv[1:] or ["f1", "f2", "f3", "f4"]
    for r in rows:
        globals()[r]()
