"""One estimate on the resident schedule (for ncu): python scripts/prof_res.py WORKLOAD K [M]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_1503_06394_b200 as P  # noqa: E402

name, k = sys.argv[1], int(sys.argv[2])
wl = W.get_workload(name)
m = int(sys.argv[3]) if len(sys.argv) > 3 else k
A, _ = wl.matrices()
op = P.Operator(wl.mode, P.DeviceCSR.from_host(A), None, wl.r1_c)
est = P.Estimator(op, wl.a, wl.b, wl.degree, m, k, seed=wl.seed)
for _ in range(2):
    est.run(check=True)
torch.cuda.synchronize()
print(name, k, P.last_schedule())
