import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W, paper_1503_06394_b200 as P
T = W.torus_laplacian(256)
dT = P.DeviceCSR.from_host(T)
lam2 = 2 - 2 * np.cos(2 * np.pi / 256)
for name, op, a, b in [("rank1", P.Operator("rank1", dT, None, lam2 / 65536), lam2, 8.0),
                       ("csr", P.Operator("csr", dT), 1e-3, 8.0)]:
    for k in (32,):
        for persist in (1, 0):
            P.set_persistent(persist)
            est = P.Estimator(op, a, b, 1000, 32, k, seed=1)
            est.run(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); est.run(); e1.record(); torch.cuda.synchronize()
            print(name, "k", k, "persist", persist, f"{e0.elapsed_time(e1):.2f} ms")
for mt in ("1",):
    pass
