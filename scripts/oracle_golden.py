#!/usr/bin/env python
"""Write the oracle's full moment tables for BASELINE.json configs[0..4] to tests/golden/oracle_mu/.

TEST INFRASTRUCTURE.  Calls only oracle/ (the pinned CPU implementation) and workloads/ (input
generators).  Nothing here touches the CUDA path.  The GPU parity tests
(tests/test_parity_full_gpu.py) compare every probe's moments mu_{p,j}, every Gamma_p and Gamma
of the CUDA path, in the bench launch configuration, against these tables (compute
the oracle once with all host cores, cache it keyed by (config, seed, probe, n)).

Each file <name>.npz holds
  mu[m][n+1]   oracle moments v_p^T T_j(Ã) v_p of global probes 0..m-1 (Algorithm 1)
  c[n+1]       oracle coefficients
  gamma_p[m], gamma, stderr     oracle accumulation (reading G7)
  a, b, degree, seed, d, nnz    the problem
  matrix_sha256                 hash of the generated CSR arrays (the test regenerates the matrix
                                and refuses a stale table)
  oracle_sha256                 hash of oracle/cheb_oracle.c at generation time

    python scripts/oracle_golden.py gmrf5000 [--workers 8]
"""
import argparse
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import workloads as W  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "oracle_mu")


def matrix_sha(A, At=None):
    h = hashlib.sha256()
    for M in (A, At):
        if M is None:
            continue
        for arr in (M.row_ptr, M.col_idx, M.val):
            h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()


def oracle_sha():
    with open(os.path.join(ROOT, "oracle", "cheb_oracle.c"), "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="+")
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    for name in args.names:
        wl = W.get_workload(name)
        A, At = wl.matrices()
        a, b = (wl.a, wl.b) if wl.a is not None else oracle.bounds_btb(A)
        op = oracle.Op(wl.mode, A, wl.r1_c)
        t0 = time.perf_counter()
        mu = oracle.moments(op, a, b, wl.degree, wl.seed, range(wl.num_probes), workers=args.workers)
        dt = time.perf_counter() - t0
        c = oracle.coeffs_log(a, b, wl.degree)
        gamma, gp, se = oracle.gamma_from_moments(c, mu)
        path = os.path.join(OUT, name + ".npz")
        np.savez_compressed(path, mu=mu, c=c, gamma_p=gp, gamma=gamma, stderr=se, a=a, b=b,
                            degree=wl.degree, seed=wl.seed, d=wl.d, nnz=A.nnz, r1_c=wl.r1_c,
                            mode=wl.mode, matrix_sha256=matrix_sha(A, At), oracle_sha256=oracle_sha(),
                            oracle_seconds=dt, workers=args.workers)
        print(f"{name}: m={wl.num_probes} n={wl.degree} d={wl.d} gamma={gamma!r} stderr={se:.6g} "
              f"({dt:.1f} s on {args.workers} workers) -> {path}", flush=True)


if __name__ == "__main__":
    main()
