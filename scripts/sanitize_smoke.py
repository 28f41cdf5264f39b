"""Tiny invocation of every kernel variant, for compute-sanitizer (one tool per run) or the
CHEB_CHECKS=1 build (device asserts on every gather index, staging offset and tile bound):

    CHEB_LIB=build_variants/libchebld_checked.so python scripts/sanitize_smoke.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_1503_06394_b200 as P  # noqa: E402


def dev(A):
    return P.DeviceCSR.from_host(A)


def main():
    G = W.grid_gmrf(23, 0.2)
    T = W.torus_laplacian(11)
    B = W.random_nonsingular(777, 2)
    op_g = P.Operator("csr", dev(G))
    op_t = P.Operator("rank1", dev(T), None, 0.01, torch.from_numpy(np.linspace(0.5, 1.5, T.n_rows)).cuda())
    op_b = P.Operator("btb", dev(B), dev(W.transpose(B)))
    a, b = P.bounds_btb(op_b)
    P.probes(1000, 3, 5, 16)
    for small in (1, 0):  # 16-row tiles for L2-resident operators (default) and the standard geometry
        P.set_small_tiles(small)
        for persist in (0, 2):
            P.set_persistent(persist)
            for k in (8, 64):
                P.logdet(op_g, 0.2, 1.8, 7, 11, seed=1, k=k)
                P.logdet(op_t, 0.01, 8.5, 7, 11, seed=1, k=k)
                P.taylor_logdet(op_g, 2.0, 5, 9, 1, k)
    P.set_small_tiles(1)
    P.set_persistent(1)
    P.logdet(op_b, a, b, 5, 9, seed=1, k=16)
    P.set_doubling(True)  # moment-doubling kernels, per step and persistent
    for persist in (0, 2):
        P.set_persistent(persist)
        P.logdet(op_g, 0.2, 1.8, 7, 11, seed=1, k=16)
        P.logdet(op_t, 0.01, 8.5, 7, 11, seed=1, k=16)
    P.set_persistent(1)
    P.logdet(op_b, a, b, 5, 9, seed=1, k=16)
    P.set_doubling(False)
    # shared-memory-resident kernel: one cluster and the flat grid, Algorithm 1 and doubling
    for single in ("8192", "0"):
        os.environ["CHEB_RES_SINGLE_MAX"] = single
        for k in (8, 16, 64):
            P.logdet(op_g, 0.2, 1.8, 7, 11, seed=1, k=k)
            P.logdet(op_t, 0.01, 8.5, 7, 11, seed=1, k=k)
        P.set_doubling(True)
        P.logdet(op_t, 0.01, 8.5, 7, 11, seed=1, k=16)
        P.set_doubling(False)
    os.environ.pop("CHEB_RES_SINGLE_MAX", None)
    torch.cuda.synchronize()
    print("sanitize smoke ok")


if __name__ == "__main__":
    main()
