"""Multi-GPU probe sharding ("very easy to parallelize").

One process per GPU (torchrun).  Every rank holds the full operator; rank g of G
computes the moments of global probes [g*m//G, (g+1)*m//G) into its rows of a
zero-initialised mu[m][n+1]; one all_reduce(SUM) over NCCL/NVLink combines them.
Adding zeros is exact, so the combined mu -- hence Gamma -- is bit-identical for
every G at a fixed probe block k.  This is the only inter-GPU traffic.

Command line (one estimate, rank 0 prints one JSON line):

    torchrun --nproc-per-node G --master-addr 127.0.0.1 -m paper_1503_06394_b200.dist \\
        --workload gmrf5000 [--k 16] [--probes 128] [--degree 100] [--seed 1]
    torchrun ... -m paper_1503_06394_b200.dist --csr A.npz --a 0.04 --b 1.96 ...

`--workload` names a synthetic input of the repo's `workloads` package (BASELINE configs);
`--csr` loads row_ptr / col_idx / val arrays (and At_* for --mode btb) from an .npz file.
"""
import argparse
import json
import math
import os
import sys
import time
from typing import Optional, Tuple

import torch
import torch.distributed as dist


def shard_range(m: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous global probe range of `rank` (empty ranges allowed when m < world)."""
    if m < 0 or world < 1 or not (0 <= rank < world):
        raise ValueError("bad shard arguments")
    return rank * m // world, (rank + 1) * m // world


def combine_moments(mu: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the zero-padded per-rank moment tables in place (NCCL on GPU, gloo on CPU)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(mu, op=dist.ReduceOp.SUM, group=group)
    return mu


def init_from_env(backend: Optional[str] = None):
    """Initialise the default process group from torchrun's environment; returns
    (rank, world, local_rank).  Single-process runs skip initialisation."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group(backend, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local


class ShardedEstimator:
    """Estimator over this rank's probe shard; `run()` enqueues moments, the
    all-reduce and the device finalisation on the current stream."""

    def __init__(self, op, a, b, degree, num_probes, k, seed=1, group=None, basis="chebyshev"):
        from .api import Estimator
        self.group = group
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.begin, self.end = shard_range(num_probes, world, rank)
        self.est = Estimator(op, a, b, degree, num_probes, k, seed, self.begin, self.end, basis=basis)

    def run(self, check: bool = True):
        """One estimate over all ranks; returns device (gamma_p, stats).  check=True (default)
        synchronises and raises ChebError on any rank whose estimate is invalid: a timed-out spin
        wait on this rank (its moments are NaN, so after the all-reduce every rank's estimate is
        non-finite) or a non-finite moment anywhere.  Timed loops pass check=False and call
        check() on the stats afterwards."""
        self.est.mu.zero_()
        self.est.enqueue_moments()
        combine_moments(self.est.mu, self.group)
        gp, stats = self.est.enqueue_finalize()
        if check:
            self.check(stats)
        return gp, stats

    def check(self, stats):
        self.est.check(stats)


def _load_operator(args, dev):
    """(Operator, a, b, degree, m, seed, description) from --workload or --csr."""
    from .api import DeviceCSR, Operator, bounds_btb
    if args.workload:
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        if root not in sys.path:
            sys.path.insert(0, root)
        import workloads as W  # seeded synthetic inputs (no method arithmetic)
        wl = W.get_workload(args.workload)
        A, At = wl.matrices()
        op = Operator(wl.mode, DeviceCSR.from_host(A, dev), DeviceCSR.from_host(At, dev) if At is not None else None,
                      wl.r1_c)
        a, b = (wl.a, wl.b) if wl.a is not None else bounds_btb(op)
        return (op, a, b, args.degree or wl.degree, args.probes or wl.num_probes,
                wl.seed if args.seed is None else args.seed, wl.name)
    import numpy as np

    class _H:
        pass

    z = np.load(args.csr)

    def csr(prefix):
        h = _H()
        h.row_ptr, h.col_idx, h.val = z[prefix + "row_ptr"], z[prefix + "col_idx"], z[prefix + "val"]
        h.n_rows = h.row_ptr.size - 1
        h.n_cols = int(z[prefix + "n_cols"]) if prefix + "n_cols" in z else h.n_rows
        return DeviceCSR.from_host(h, dev)
    At = csr("At_") if args.mode == "btb" else None
    op = Operator(args.mode, csr(""), At, args.c)
    if args.a is None or args.b is None:
        if args.mode != "btb":
            raise SystemExit("--a and --b are required for csr / rank1 operators")
        a, b = bounds_btb(op)
    else:
        a, b = args.a, args.b
    return op, a, b, args.degree or 15, args.probes or 30, 1 if args.seed is None else args.seed, args.csr


def main(argv=None):
    ap = argparse.ArgumentParser(description="Chebyshev-Hutchinson log det, probes sharded over GPUs")
    src = ap.add_mutually_exclusive_group(required=True)
    src.add_argument("--workload", help="synthetic BASELINE workload name (workloads package)")
    src.add_argument("--csr", help=".npz with row_ptr, col_idx, val [, At_row_ptr, At_col_idx, At_val]")
    ap.add_argument("--mode", choices=["csr", "rank1", "btb"], default="csr")
    ap.add_argument("--c", type=float, default=0.0, help="rank-1 weight (u = ones)")
    ap.add_argument("--a", type=float)
    ap.add_argument("--b", type=float)
    ap.add_argument("--degree", type=int, default=0)
    ap.add_argument("--probes", type=int, default=0, help="total probes m over all ranks")
    ap.add_argument("--seed", type=int)
    ap.add_argument("--k", type=int, default=16, help="probe block per launch (8..128)")
    args = ap.parse_args(argv)

    from .api import log_abs_det_from_btb
    rank, world, local = init_from_env()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    op, a, b, n, m, seed, what = _load_operator(args, dev)
    sh = ShardedEstimator(op, a, b, n, m, args.k, seed)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    gp, stats = sh.run(check=True)
    st = stats.cpu().numpy()
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    if rank == 0:
        out = {"input": what, "mode": op.kind, "d": op.d, "a": a, "b": b, "degree": n, "num_probes": m,
               "probe_block": args.k, "world": world, "logdet": float(st[0]), "stderr": float(st[1]),
               "seconds": float(dt.item()), "probe_steps_per_s": m * n / float(dt.item())}
        if op.kind == "btb":
            out["log_abs_det_B"] = log_abs_det_from_btb(float(st[0]))
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
