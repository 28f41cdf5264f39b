"""Multi-process (world_size 2, gloo on CPU) coverage of the probe-sharding logic
of paper_1503_06394_b200/dist.py: shard ranges, zero-padded moment tables and the
all-reduce reproduce the single-process moments exactly.  The per-shard moments
come from the oracle (the CPU stand-in for cheb_moments on a GPU-less box)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

from paper_1503_06394_b200.dist import shard_range, combine_moments


def test_shard_ranges_partition():
    for m in (0, 1, 5, 64, 127, 128):
        for world in (1, 2, 3, 4, 8):
            got = [shard_range(m, world, r) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == m
            assert all(got[i][1] == got[i + 1][0] for i in range(world - 1))
            sizes = [e - b for b, e in got]
            assert max(sizes) - min(sizes) <= 1
    assert shard_range(128, 8, 3) == (48, 64)  # 16 probes per GPU at m = 128, G = 8
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import workloads as W
    wl = W.get_workload("gmrf_s")
    A, _ = wl.matrices()
    m, n = 13, 9
    b0, b1 = shard_range(m, world, rank)
    mu = torch.zeros((m, n + 1), dtype=torch.float64)
    if b1 > b0:
        mu[b0:b1] = torch.from_numpy(oracle.moments(oracle.Op("csr", A), wl.a, wl.b, n, wl.seed,
                                                    range(b0, b1)))
    combine_moments(mu)
    np.save(os.path.join(out_dir, f"mu{rank}.npy"), mu.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_combine_equals_single_process(tmp_path, orc):
    import workloads as W
    world, port = 2, _free_port()
    tmp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    wl = W.get_workload("gmrf_s")
    A, _ = wl.matrices()
    full = orc.moments(orc.Op("csr", A), wl.a, wl.b, 9, wl.seed, range(13))
    for r in range(world):
        got = np.load(tmp_path / f"mu{r}.npy")
        assert np.array_equal(got, full)  # zero padding + sum is exact


def _worker_poison(rank, world, port, out_dir):
    """Rank 1's shard comes back poisoned (NaN rows: what cheb_moments' status epilogue writes
    after a timed-out spin wait); after the all-reduce EVERY rank holds non-finite moments, so
    every rank's finalize flags the estimate and ShardedEstimator.check raises on all of them."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import workloads as W
    from paper_1503_06394_b200.api import check_estimate
    from paper_1503_06394_b200._lib import ChebError
    wl = W.get_workload("gmrf_s")
    A, _ = wl.matrices()
    m, n = 10, 6
    b0, b1 = shard_range(m, world, rank)
    mu = torch.zeros((m, n + 1), dtype=torch.float64)
    mu[b0:b1] = torch.from_numpy(oracle.moments(oracle.Op("csr", A), wl.a, wl.b, n, wl.seed, range(b0, b1)))
    if rank == 1:
        mu[b0:b1] = float("nan")
    combine_moments(mu)
    g, gp, se = oracle.gamma_from_moments(oracle.coeffs_log(wl.a, wl.b, n), mu.numpy())
    stats = torch.tensor([g, se, 1.0 if np.all(np.isfinite(gp)) else 0.0], dtype=torch.float64)
    try:
        check_estimate(stats)
        raised = 0
    except ChebError as e:
        raised = e.code
    np.save(os.path.join(out_dir, f"raised{rank}.npy"), np.array([raised]))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_error_reaches_every_rank(tmp_path):
    world, port = 2, _free_port()
    tmp.spawn(_worker_poison, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert int(np.load(tmp_path / f"raised{r}.npy")[0]) == -5
