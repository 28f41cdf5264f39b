"""Multi-GPU probe sharding ("very easy to parallelize").

One process per GPU (torchrun).  Every rank holds the full operator; rank g of G
computes the moments of global probes [g*m//G, (g+1)*m//G) into its rows of a
zero-initialised mu[m][n+1]; one all_reduce(SUM) over NCCL/NVLink combines them.
Adding zeros is exact, so the combined mu -- hence Gamma -- is bit-identical for
every G at a fixed probe block k.  This is the only inter-GPU traffic.
"""
import os
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

    def run(self):
        self.est.mu.zero_()
        self.est.enqueue_moments()
        combine_moments(self.est.mu, self.group)
        return self.est.enqueue_finalize()
