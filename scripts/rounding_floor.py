"""Oracle rounding floor per BASELINE config: Gamma_p of probe 0 from the problem
as given and from its row-reversed permutation; writes profiles/r01_rounding_floor.json.
Calls only oracle/ and workloads/ (CPU)."""
import json
import os
import sys
from concurrent.futures import ProcessPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from test_rounding_floor import _gamma  # noqa: E402

if __name__ == "__main__":
    names = sys.argv[1:] or ["gmrf32", "torus256", "gmrf1000", "gmrf5000", "btb4m"]
    out = {}
    with ProcessPoolExecutor(max_workers=4) as ex:
        futs = {(n, r): ex.submit(_gamma, n, r, 0) for n in names for r in (False, True)}
        for n in names:
            g0, g1 = futs[(n, False)].result(), futs[(n, True)].result()
            out[n] = {"gamma_p0": g0, "gamma_p0_reversed": g1, "rel_diff": abs(g0 - g1) / abs(g0)}
            print(n, out[n], flush=True)
    with open(os.path.join(ROOT, "profiles", "r01_rounding_floor.json"), "w") as f:
        json.dump(out, f, indent=1)
