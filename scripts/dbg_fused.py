import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W, paper_1503_06394_b200 as P
for (name, A, k, n) in [("spd20000", W.random_spd(20000, 6), 16, 7), ("grid61", W.grid_gmrf(61, 0.24), 16, 7),
                        ("spd4000", W.random_spd(4000, 6), 16, 5), ("grid300", W.grid_gmrf(300, 0.24), 64, 6)]:
    op = P.Operator("csr", P.DeviceCSR.from_host(A))
    lam = 1.0 + 2.0 * np.abs(A.val).max() * 12
    res = {}
    for mode in (1, 3):
        P.set_fusion(mode)
        res[mode] = P.moments(op, 0.01, lam, n, 0, 16, 3, k).cpu().numpy()
    d = np.abs(res[1] - res[3])
    print(name, "maxdiff per column", d.max(axis=0), "rel", (d / (np.abs(res[1]) + 1)).max())
