import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W, paper_1503_06394_b200 as P, oracle as orc
B = W.random_nonsingular(300, 3)
Bt = W.transpose(B)
op = P.Operator("btb", P.DeviceCSR.from_host(B), P.DeviceCSR.from_host(Bt))
a, b = P.bounds_btb(op)
s = a + b
D = W.to_dense(B); M = D.T @ D; A = np.eye(300) - M / s
for n in (1, 2, 3):
    for k in (8, 16):
        mu = P.power_moments(op, s, n, 0, 8, 1, k).cpu().numpy()
        v = orc.rademacher(1, 0, 300)
        want = [v @ np.linalg.matrix_power(A, j) @ v for j in range(n + 1)]
        print(n, k, mu[0], np.round(want, 6))
# also csr with the same M materialised
from workloads.csr import from_coo
r, c = np.nonzero(M)
Mc = from_coo(300, 300, r, c, M[r, c])
opm = P.Operator("csr", P.DeviceCSR.from_host(Mc))
print("csr", P.power_moments(opm, s, 3, 0, 8, 1, 8).cpu().numpy()[0])
