"""Registry of the BASELINE.json workloads (configs[0..4]) plus scaled-down
variants for parity tests.  Inputs only: matrices, operator mode, spectral
interval where it is a closed-form property of the generated matrix, degree n,
probe count m.  Config 4's interval is *computed by the path* (a0, Johnson /
norm bounds), so it is None here.
"""
import math
from dataclasses import dataclass, field
from typing import Callable, Optional

from .csr import CSR, transpose
from .generators import grid_gmrf, torus_laplacian, random_nonsingular, random_spd


@dataclass
class Workload:
    name: str
    mode: str                 # "csr" | "rank1" | "btb"
    build: Callable[[], CSR]  # builds A (csr/rank1) or B (btb)
    d: int
    a: Optional[float]        # spectral interval of the applied operator M
    b: Optional[float]        # (None: computed from the matrix)
    degree: int
    num_probes: int
    r1_c: float = 0.0         # rank-1 weight c (u = all-ones)
    seed: int = 1
    notes: str = ""
    extra: dict = field(default_factory=dict)
    symmetric: bool = False   # btb with symmetric B: B^T is B itself
    paper_probe_steps_per_s: Optional[float] = None  # BASELINE.md number for this exact workload

    def matrices(self):
        """Return (A, At) -- At is the exact transpose for btb, else None."""
        A = self.build()
        if self.mode != "btb":
            return A, None
        return A, (A if self.symmetric else transpose(A))


def _gmrf(name, N, theta, degree, m, notes):
    return Workload(name, "csr", lambda: grid_gmrf(N, theta), N * N,
                    1.0 - 4.0 * theta, 1.0 + 4.0 * theta, degree, m,
                    notes=notes, extra={"grid_N": N, "theta": theta})


def _torus(name, N, degree, m, notes):
    d = N * N
    lam2 = 2.0 - 2.0 * math.cos(2.0 * math.pi / N)
    return Workload(name, "rank1", lambda: torus_laplacian(N), d, lam2, 8.0,
                    degree, m, r1_c=lam2 / d, notes=notes,
                    extra={"torus_N": N, "lambda2": lam2})


def _btb(name, d, degree, m, seed, notes):
    return Workload(name, "btb", lambda: random_nonsingular(d, seed), d, None, None,
                    degree, m, notes=notes, extra={"matrix_seed": seed})


def _gpu_or_cpu():
    try:
        import torch
        return "cuda" if torch.cuda.is_available() else "cpu"
    except Exception:  # pragma: no cover
        return "cpu"


def _spd_paper(name, d, notes, paper=None):
    """Paper §5.1: Algorithm 2 on a random sparse SPD C with m = 10,
    n = 15, sigma_min = 1e-3, sigma_max = ||C||_1 -- in [a,b] form the B^T B
    interval [sigma_min^2, ||C||_1 ||C||_inf], which the path's bounds kernel
    computes from the matrix (Johnson's bound equals 1e-3 exactly for this C)."""
    return Workload(name, "btb", lambda: random_spd(d, 1, device=_gpu_or_cpu()), d, None, None,
                    15, 10, notes=notes, symmetric=True, paper_probe_steps_per_s=paper,
                    extra={"matrix_seed": 1, "paper_seconds": 500.0 if paper else None})


CONFIGS = {
    # BASELINE.json configs[0..4]
    "gmrf32": _gmrf("gmrf32", 32, 0.2, 30, 64, "BJ.configs[0]"),
    "torus256": _torus("torus256", 256, 1000, 32, "BJ.configs[1]"),
    "gmrf1000": _gmrf("gmrf1000", 1000, 0.24, 100, 64, "BJ.configs[2]"),
    "gmrf5000": _gmrf("gmrf5000", 5000, 0.24, 100, 128, "BJ.configs[3] (headline)"),
    "btb4m": _btb("btb4m", 4_000_000, 50, 64, 1, "BJ.configs[4]"),
    # scaled-down parity cases (several tiles + ragged tails)
    "gmrf_s": _gmrf("gmrf_s", 61, 0.24, 40, 20, "parity: ragged grid"),
    "torus_s": _torus("torus_s", 37, 120, 12, "parity: small torus + rank-1"),
    "btb_s": _btb("btb_s", 5003, 20, 12, 3, "parity: small random B"),
    # the paper's own timed workload (Fig. 1(a); 500 s at d = 3e7 on a
    # 3.40 GHz i7, i.e. 10 probes x 15 steps / 500 s = 0.30 probe-steps/s)
    "spd30m": _spd_paper("spd30m", 30_000_000, "paper §5.1 Fig. 1(a), d = 3e7", paper=0.30),
    "spd1m": _spd_paper("spd1m", 1_000_000, "paper §5.1 Fig. 1(a), d = 1e6"),
    "spd_s": _spd_paper("spd_s", 4099, "parity: paper §5.1 generator, small"),
}

BASELINE_ORDER = ["gmrf32", "torus256", "gmrf1000", "gmrf5000", "btb4m"]


def get_workload(name: str) -> Workload:
    try:
        return CONFIGS[name]
    except KeyError:
        raise KeyError(f"unknown workload {name!r}; have {sorted(CONFIGS)}")
