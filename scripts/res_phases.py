"""Phase breakdown of the shared-memory-resident kernel (needs the "resprof" build):

    CHEB_LIB=build_variants/libchebld_resprof.so python scripts/res_phases.py torus256 16

Phases per step, thread 0 of each CTA, SM cycles: rows (gathers + compute, up to the CTA
barrier after the warp partials), cpart (per-CTA partial), csync (cluster barrier), gwait (group
sums + grid counter wait; multi-cluster only), fin (second-level sums), tail (mu / s_j writes).
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
import paper_1503_06394_b200 as P  # noqa: E402
from paper_1503_06394_b200 import _lib  # noqa: E402

name, k = sys.argv[1], int(sys.argv[2])
wl = W.get_workload(name)
A, _ = wl.matrices()
op = P.Operator(wl.mode, P.DeviceCSR.from_host(A), None, wl.r1_c)
est = P.Estimator(op, wl.a, wl.b, wl.degree, k, k, seed=wl.seed)
est.run(check=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
est.run(check=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
lib = _lib.load()
buf = (ctypes.c_longlong * (1024 * 8))()
assert lib.cheb_res_prof_read(buf, 1024 * 8) == 0
a = np.frombuffer(buf, dtype=np.int64).reshape(1024, 8)
g = int(np.nonzero(a.sum(axis=1))[0].max()) + 1
a = a[:g, :6] / wl.degree
names = ["rows", "cpart", "csync", "fin", "tail", "gwait"]
print(json.dumps({"workload": name, "k": k, "schedule": P.last_schedule(), "grid": g, "ms": ms,
                  "us_per_step": 1e3 * ms / wl.degree,
                  "cycles_per_step_mean": {n: round(float(a[:, i].mean()), 1) for i, n in enumerate(names)},
                  "cycles_per_step_max": {n: round(float(a[:, i].max()), 1) for i, n in enumerate(names)}}))
