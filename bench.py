#!/usr/bin/env python
"""Benchmark of the Chebyshev-Hutchinson log-det hot path (BASELINE.json metric:
probe*Chebyshev-steps/sec, HBM GB/s vs peak, log-det wall time at 25M vars).

One bench "step" = one whole estimate: probe initialisation, `degree` fused Chebyshev steps per
probe block, reductions, the moment all-reduce (N > 1) and the device accumulation of Gamma.

Headline (default): BASELINE configs[3] as the config states it -- gmrf5000 (d = 2.5e7, n = 100),
m = 128 probes IN TOTAL sharded across the N GPUs (strong scaling), probe block k = 16 at every N
("scaling curves use fixed k = 16, so per-GPU bytes per probe-step are identical
across G"; 16 probes per GPU at N = 8).  Beside it, in the same JSON line, `weak_scaling`: m = 128
probes PER GPU at the best single-GPU block size k = 64.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--k K] [--scaling weak]
    python bench.py --impl reference ...    # the CPU oracle as the reference arm

Under torchrun each rank drives one GPU; rank 0 prints ONE JSON line.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402

METRIC = "probe*Chebyshev-steps/sec"
UNIT = "probe-steps/s"
FALLBACK_HBM_GBS = 6650.0


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured"
    return FALLBACK_HBM_GBS, "fallback"


def _traffic_per_launch(workload, k, kernel="step", cv=False):
    """dram read+write bytes per launch from the committed ncu --set full summaries (key suffix
    /cv: measured with the compressed matrix copy)."""
    p = os.path.join(ROOT, "profiles", "ncu_step_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        j = json.load(f)
    e = j.get(f"{workload}/k{k}" + ("" if kernel == "step" else f"/{kernel}") + ("/cv" if cv else ""))
    return float(e["dram_bytes_per_launch"]) if e else None


CV_U = 5  # entries per row of the compressed matrix copy (CHEB_NNZ_UNROLL)


def step_bytes(d, nnz, k, first=False, mode="csr", doubling=False, cv=False):
    """Algorithmic HBM bytes of one cheb_step_kernel launch over a block of k probes
    (SURVEY §8(d)): gather matrix (val 8 + col 4 per nnz, row_ptr 8 per
    row; the compressed copy when the library used it: 3 bytes per entry of U = 5 per row, no
    row pointer, a 2 KB value table) once per block; per row and probe 8 B each for the gather
    source read, W_prev read and W_next write (no W_prev on the first step) -- plus, for B^T B,
    the W_cur read of the -beta*w term; sign bits (4 B per row per 32 probes, >= 4; the
    moment-doubling schedule reads none: its dots are w_j.w_j and w_j.w_{j-1})."""
    vec = (16 if first else 24) * d * k
    if mode == "btb":
        vec += 8 * d * k
    mat = 3 * CV_U * d + 2048 if cv else 12 * nnz + 8 * (d + 1)
    return mat + vec + (0 if doubling else d * max(4, k // 8))


def spmm_bytes(d, nnz_b, k):
    """Algorithmic HBM bytes of one spmm_kernel launch (B^T B: Y = B w): B once, w read, Y written."""
    return 12 * nnz_b + 8 * (d + 1) + 16 * d * k


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, bus_id=None):
        self.rows, self.proc, self.bus_id = [], None, bus_id

    def start(self):
        cmd = ["nvidia-smi", f"--query-gpu=pci.bus_id,{self.FIELDS}", "--format=csv,noheader,nounits",
               "-lms", "200"]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        rows = self.rows
        if self.bus_id is not None:
            mine = [r for r in rows if r and self.bus_id.lower() in r[0].lower()]
            rows = mine or rows
        sm = [float(r[1]) for r in rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) > 8 for i in range(4)
                          if r[5 + i].lower() == "active"})
        if not sm:
            return None
        pw = []
        for r in rows:
            try:
                pw.append(float(r[3]))
            except (IndexError, ValueError):
                pass
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(smax) if smax else None,
                "power_w_median": float(np.median(pw)) if pw else None, "samples": len(sm),
                "reasons": reasons}


def build_workload(name):
    wl = W.get_workload(name)
    t0 = time.perf_counter()
    A, At = wl.matrices()
    build_workload.gen_s = time.perf_counter() - t0  # host generation time of the operator
    return wl, A, At


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def plan(args, wl, world):
    """(m_total, k, scaling) of the headline line."""
    if args.scaling == "strong":
        m_total = args.probes or wl.num_probes
        k = args.k or 16
    else:
        m_total = (args.probes or wl.num_probes) * world
        k = args.k or next((kk for kk in (8, 16, 32, 64) if kk >= m_total // world), 64)
    return m_total, k


# ------------------------------------------------------------------------- oracle (CPU) arm
def oracle_sample(wl, A, steps_per_probe, probes, workers):
    """Time the oracle AS IT STANDS on a bounded sample: `probes` probes x
    `steps_per_probe` Chebyshev steps of the same workload, one probe per worker."""
    import oracle
    a, b = wl.a, wl.b
    if a is None:
        a, b = oracle.bounds_btb(A)
    op = oracle.Op(wl.mode, A, wl.r1_c)
    oracle.lib()
    t0 = time.perf_counter()
    oracle.moments(op, a, b, steps_per_probe, wl.seed, range(probes), workers=workers)
    dt = time.perf_counter() - t0
    return probes * steps_per_probe / dt, dt


def _oracle_plan(wl, budget_s=20.0):
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except (ValueError, OSError):
        avail = 16 << 30
    per_worker = 6 * 8 * wl.d  # probe + 3 work vectors (+ scratch) of d doubles
    workers = max(1, min(cores, 64, int(0.5 * avail // max(per_worker, 1))))
    nnz_per_row = 5 if wl.mode != "btb" else 18
    est_step_s = wl.d * nnz_per_row * 2.5e-9 + wl.d * 3e-9  # ~single-core C loop
    steps = int(max(1, min(wl.degree, budget_s / max(est_step_s, 1e-9))))
    return workers, steps


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    wl, A, At = build_workload(args.workload)
    m_total, k = plan(args, wl, world)
    workers, steps = _oracle_plan(wl, budget_s=args.ref_budget)
    for _ in range(args.warmup):
        oracle_sample(wl, A, 1, workers, workers)
    vals, times = [], []
    for _ in range(args.steps):
        v, dt = oracle_sample(wl, A, steps, workers, workers)
        vals.append(v)
        times.append(dt)
    value = float(np.median(vals))
    sample = (f"{workers} probes x {steps} Chebyshev steps of {wl.name} (d={wl.d}) per bench step, "
              f"one single-threaded oracle process per probe")
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(times)),
           "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": {"workload": wl.name, "d": wl.d, "degree": wl.degree,
                                            "num_probes": m_total, "probe_block": k,
                                            "num_probes_per_step": workers, "steps_per_probe": steps},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "oracle", "cpu_model": cpu_model(),
                            "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


# ------------------------------------------------------------------------- GPU arm
def timed_region(sh, steps, flush_buf, P, torch, dist, world, dev):
    """Time `steps` whole estimates on the device (events on the launching stream; max over
    ranks).  With flush_buf, a 2x-L2 write precedes each estimate outside its event pair.
    Returns (ms, profile, launches, [stats])."""
    stream = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps if flush_buf is not None else 1)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    n_launch0 = P.launch_count()
    P.profile_begin()
    all_stats = []
    if flush_buf is not None:
        for i in range(steps):
            flush_buf.fill_(i)
            evs[i][0].record(stream)
            all_stats.append(sh.run(check=False)[1])
            evs[i][1].record(stream)
    else:
        evs[0][0].record(stream)
        for _ in range(steps):
            all_stats.append(sh.run(check=False)[1])
        evs[0][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    prof = P.profile_end()
    launches = P.launch_count() - n_launch0
    elapsed = torch.tensor([sum(e0.elapsed_time(e1) for e0, e1 in evs)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(elapsed, op=dist.ReduceOp.MAX)
    for s in all_stats:  # every timed estimate must be valid (raises ChebError otherwise)
        sh.check(s)
    return float(elapsed.item()), prof, launches, all_stats


def roofline(wl, A, At, k, blocks, steps, t_ms, prof, args, hbm, peak_kind, sched="per_step", cv=False):
    """Roofline of the dominant kernel from its measured launch times and algorithmic bytes."""
    d = wl.d
    gnnz = A.nnz if wl.mode != "btb" else At.nnz  # gather matrix of the step kernel
    (s_ms, s_n), (b_ms, b_n), (p_ms, p_n) = prof["single"], prof["spmm"], prof["persistent"]
    dbl = bool(args.doubling)
    gather_aware = None
    if p_ms > s_ms:  # persistent multi-step kernel: one launch = all steps of a block
        kern = (f"cheb_resident_kernel<{k},{wl.mode}>" if sched == "resident" else
                f"cheb_persist_kernel<{k},{wl.mode}>")
        apps = (wl.degree + 1) // 2 if dbl else wl.degree  # applications of A~ per launch
        bytes_per_launch = (step_bytes(d, gnnz, k, True, wl.mode, dbl)
                            + (apps - 1) * step_bytes(d, gnnz, k, args.basis == "taylor", wl.mode, dbl))
        avg_launch_ms, dom_ms, nl = p_ms / max(p_n, 1), p_ms, p_n
    else:
        kern = f"cheb_step_kernel<{k},{wl.mode}>"
        per_block = s_n / max(blocks * steps, 1)
        if args.basis == "taylor":  # power recurrence: every launch reads w_{j-1}, writes w_j
            tot = s_n * step_bytes(d, gnnz, k, True, wl.mode, cv=cv)
        else:
            tot = blocks * steps * (step_bytes(d, gnnz, k, True, wl.mode, dbl, cv)
                                    + (per_block - 1) * step_bytes(d, gnnz, k, False, wl.mode, dbl, cv))
        nl = s_n
        if wl.mode == "btb" and b_n:
            # one B^T B application = spmm (Y = B w) + step (B^T Y, recurrence, dots): both halves
            kern += f" + spmm_kernel<{k}>"
            tot += b_n * spmm_bytes(d, A.nnz, k)
            # random columns: every gathered row of w (spmm) and of Y (step) is an HBM access
            # (8k bytes per nonzero) rather than an L2 hit
            ga = tot - 8 * d * k * (s_n + b_n) + 8 * k * (gnnz * s_n + A.nnz * b_n)
            gather_aware = {"bytes_per_application": ga / nl,
                            "achieved": ga / ((s_ms + b_ms) / 1e3) / 1e9,
                            "frac": ga / ((s_ms + b_ms) / 1e3) / 1e9 / hbm}
            s_ms += b_ms
        bytes_per_launch = tot / max(nl, 1)
        avg_launch_ms, dom_ms = s_ms / max(nl, 1), s_ms
    achieved = bytes_per_launch / (avg_launch_ms / 1e3) / 1e9
    return {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
            "peak_kind": peak_kind, "frac_vs_nominal_8000": achieved / 8000.0, "kernel": kern,
            "bytes_per_launch": bytes_per_launch, "avg_launch_ms": avg_launch_ms,
            "launches": int(nl), "step_kernel_share": dom_ms / t_ms,
            "matrix_format": "compressed (3 B per entry, DESIGN.md §6)" if cv else "csr (12 B per nonzero)",
            "traffic": _traffic_per_launch(wl.name, k, cv=cv), "gather_aware": gather_aware,
            "note": ("shared-memory-resident kernel: the vectors never reach HBM; achieved = the HBM step "
                     "model's bytes / time (equivalent bandwidth)" if sched == "resident" else
                     "L2-resident persistent kernel: HBM step-model bytes / time (equivalent bandwidth)"
                     if p_ms > s_ms else None)}


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1503_06394_b200 import dist as pdist
    import paper_1503_06394_b200 as P

    # BENCH_SHARE_GPU=1: functional check of the N > 1 code path on a one-GPU box (every rank on
    # cuda:0, gloo instead of NCCL); the line is flagged and is never a measurement
    share = os.environ.get("BENCH_SHARE_GPU") == "1"
    rank, world, local = pdist.init_from_env("gloo" if share else "nccl")
    if share:
        local = 0
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    wl, A, At = build_workload(args.workload)
    m_total, k = plan(args, wl, world)
    p0, p1 = pdist.shard_range(m_total, world, rank)
    m_mine = p1 - p0

    # CPU baseline first (fork-based pool before any CUDA context exists)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        workers, steps = _oracle_plan(wl, budget_s=args.ref_budget)
        v, dt = oracle_sample(wl, A, steps, workers, workers)
        cpu = {"value": v, "unit": UNIT, "cores": workers, "kind": "oracle", "cpu_model": cpu_model(),
               "sample": f"{workers} probes x {steps} Chebyshev steps of {wl.name} (d={wl.d}), "
                         f"one single-threaded oracle process per probe, {dt:.1f} s"}

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    torch.cuda.synchronize()
    t_up = time.perf_counter()
    dA = P.DeviceCSR.from_host(A, dev)
    dAt = P.DeviceCSR.from_host(At, dev) if At is not None else None
    op = P.Operator(wl.mode, dA, dAt, wl.r1_c)
    a, b = (wl.a, wl.b) if wl.a is not None else P.bounds_btb(op)
    torch.cuda.synchronize()
    upload_s = time.perf_counter() - t_up
    if args.doubling:
        P.set_doubling(True)
    sh = pdist.ShardedEstimator(op, a, b, wl.degree, m_total, k, seed=wl.seed, basis=args.basis)

    for _ in range(args.warmup):
        sh.run(check=True)
    torch.cuda.synchronize()

    # L2 between timed iterations: a working set (two probe blocks + matrix) larger than L2 needs
    # no flush; a smaller one gets a 2x-L2 buffer write between iterations, outside the per-
    # iteration event pairs (one pair per iteration, times summed)
    l2_bytes = int(getattr(torch.cuda.get_device_properties(dev), "L2_cache_size", 0) or 0)
    wset = 2 * wl.d * k * 8 + 12 * int(A.nnz + (At.nnz if At is not None else 0)) + 8 * wl.d
    flush = l2_bytes > 0 and wset < l2_bytes
    flush_buf = torch.empty(2 * l2_bytes // 4, dtype=torch.int32, device=dev) if flush else None

    # ---- timed region (device events on the launching stream; max over ranks)
    clocks = ClockSampler(None)
    if rank == 0:
        props = torch.cuda.get_device_properties(dev)
        bus = getattr(props, "pci_bus_id", None)
        clocks.bus_id = None if bus is None else f":{int(bus):02X}:00."
        clocks.start()
    t_ms, prof, launches, all_stats = timed_region(sh, args.steps, flush_buf, P, torch, dist, world, dev)
    clk = clocks.stop() if rank == 0 else None
    sched = P.last_schedule()
    cv = bool(P.workspace_status(sh.est.workspace) & 0x100)  # the per-step kernels read the compressed copy
    st = all_stats[-1].cpu().numpy()

    # ---- weak scaling beside the headline: m per GPU fixed, best single-GPU block size
    weak = None
    if args.scaling == "strong" and not args.no_weak:
        m_w = (args.probes or wl.num_probes) * world
        k_w = next((kk for kk in (8, 16, 32, 64) if kk >= m_w // world), 64)
        sw = pdist.ShardedEstimator(op, a, b, wl.degree, m_w, k_w, seed=wl.seed, basis=args.basis)
        sw.run(check=True)
        reps = max(1, min(args.steps, 3))
        tw, profw, _, stw = timed_region(sw, reps, flush_buf, P, torch, dist, world, dev)
        sched_w = P.last_schedule()
        cv_w = bool(P.workspace_status(sw.est.workspace) & 0x100)
        hbm, peak_kind = _peaks()
        rw = roofline(wl, A, At, k_w, math.ceil((m_w // world) / k_w), reps, tw, profw, args, hbm, peak_kind,
                      sched_w, cv_w)
        weak = {"scaling": "weak", "num_probes": m_w, "probes_per_gpu": m_w // world, "probe_block": k_w,
                "value": m_w * wl.degree * reps / (tw / 1e3), "unit": UNIT, "ms_per_step": tw / reps,
                "steps": reps, "logdet_wall_s": tw / reps / 1e3, "gamma": float(stw[-1].cpu().numpy()[0]),
                "roofline_frac": rw["frac"], "roofline_achieved_gbs": rw["achieved"], "kernel_schedule": sched_w}
        del sw

    # ---- the other schedule on the same operator (Algorithm 1 <-> moment doubling)
    alt = None
    if not args.no_alt and args.basis == "chebyshev":
        alt = run_alt_schedule(args, sh, P, torch, dist, world, dev, float(st[0]))

    # ---- end-to-end through the public C ABI with HOST buffers (pinned)
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, wl, A, At, a, b, m_total, k, rank, world, dev, P, pdist, torch, dist)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    units = m_total * wl.degree * args.steps  # degree-n Chebyshev moments delivered per probe
    value = units / (t_ms / 1e3)
    hbm, peak_kind = _peaks()
    nnz = A.nnz + (At.nnz if At is not None else 0)
    blocks = math.ceil(m_mine / k)
    roof = roofline(wl, A, At, k, blocks, args.steps, t_ms, prof, args, hbm, peak_kind, sched, cv)
    cfg = {"workload": wl.name, "baseline_config": wl.notes, "mode": wl.mode, "d": wl.d,
           "nnz": int(nnz), "degree": wl.degree, "num_probes": m_total, "probes_per_gpu": m_mine,
           "probe_block": k, "a": a, "b": b, "basis": args.basis,
           "schedule": ("moment doubling: ceil(n/2) applications of A~ per probe, value counts "
                        "the n Chebyshev steps delivered" if args.doubling else
                        "Algorithm 1: n applications of A~ per probe"),
           "applications_per_probe": (wl.degree + 1) // 2 if args.doubling else wl.degree,
           "kernel_schedule": sched,
           "parallelism": f"probe-dp{world}",
           "l2": (f"L2 flushed between timed iterations ({2 * l2_bytes / 1e6:.0f} MB write outside the "
                  f"per-iteration events; working set {wset / 1e6:.1f} MB < L2 {l2_bytes / 1e6:.0f} MB)"
                  if flush else f"inputs larger than L2 (working set {wset / 1e9:.1f} GB/GPU > L2), "
                  "no flush needed"),
           "logdet_wall_s": t_ms / args.steps / 1e3,
           "logdet_wall_incl_generation_upload_s": build_workload.gen_s + upload_s + t_ms / args.steps / 1e3,
           "generation_s": build_workload.gen_s, "upload_s": upload_s, "gamma": float(st[0]),
           "stderr": float(st[1])}
    if wl.mode == "btb":
        cfg["log_abs_det_B"] = P.log_abs_det_from_btb(float(st[0]))  # Alg. 2's output
        cfg["log_abs_det_B_stderr"] = 0.5 * float(st[1])
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
           "scaling": args.scaling,
           "vs_baseline": (value / wl.paper_probe_steps_per_s) if wl.paper_probe_steps_per_s else None,
           "dtype": "f64", "data": "synthetic", "config": cfg,
           **({"functional_check_shared_gpu": "all ranks on cuda:0 over gloo: not a measurement"} if share else {}),
           "roofline": roof, "gpu_launches": int(launches),
           "gpu_launches_per_step": launches / args.steps, "clocks": clk, "cpu_baseline": cpu,
           "e2e": e2e, "weak_scaling": weak, "alt_schedule": alt}
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_alt_schedule(args, sh, P, torch, dist, world, dev, gamma_main):
    """Time the other moment schedule on the same sharded estimator (device events, max over
    ranks), reported beside the headline, never instead of it: moment doubling (G25) when the
    headline is Algorithm 1, and vice versa."""
    n = sh.est.degree
    if not args.doubling:
        name, apps, switch = "moment doubling", (n + 1) // 2, (lambda on: P.set_doubling(on))
    else:
        name, apps, switch = "Algorithm 1 recurrence", n, (lambda on: P.set_doubling(not on))
    switch(True)
    try:
        sh.run(check=True)
        torch.cuda.synchronize()
        reps = max(1, min(args.steps, 3))
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        ev0.record()
        for _ in range(reps):
            gp, stats = sh.run(check=False)
        ev1.record()
        torch.cuda.synchronize()
        sh.check(stats)
        el = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        g = float(stats.cpu().numpy()[0])
    finally:
        switch(False)
    wall = float(el.item()) / reps / 1e3
    return [{"schedule": name, "applications_per_probe": apps, "logdet_wall_s": wall,
             "chebyshev_steps_per_s": sh.est.m * n / wall, "gamma": g,
             "rel_diff_gamma_vs_headline": abs(g - gamma_main) / abs(gamma_main), "reps": reps}]


def run_e2e(args, wl, A, At, a, b, m_total, k, rank, world, dev, P, pdist, torch, dist):
    """Same metric end to end through the C ABI with HOST buffers: every step copies the operator
    from pinned host memory to the device, runs the estimate and reads the result back.
    N = 1: cheb_logdet_host.  N > 1: every rank calls cheb_moments_host for its probe shard (H2D
    of the CSR, moments, D2H of its moment rows), the zero-padded tables are summed with one NCCL
    all_reduce and cheb_finalize accumulates Gamma (device), read back to the host."""
    def pin(x):
        return torch.from_numpy(np.ascontiguousarray(x)).pin_memory()

    class HostCSR:
        pass

    def host_csr(M):
        h = HostCSR()
        h.n_rows, h.n_cols = M.n_rows, M.n_cols
        h.row_ptr, h.col_idx, h.val = pin(M.row_ptr), pin(M.col_idx), pin(M.val)
        return h

    hA = host_csr(A)
    hAt = host_csr(At) if At is not None else None
    h2d = sum(t.numel() * t.element_size() for h in (hA, hAt) if h is not None
              for t in (h.row_ptr, h.col_idx, h.val))
    steps = max(1, min(args.steps, args.e2e_steps))
    n = wl.degree
    if world == 1:
        def one():
            return P.logdet_host(wl.mode, hA, a, b, n, m_total, seed=wl.seed, k=k, At=hAt, c=wl.r1_c)
        one()  # warm
        t0 = time.perf_counter()
        for _ in range(steps):
            one()
        dt = time.perf_counter() - t0
        d2h = 8 * (3 + m_total)
        h2d_mu = 0
    else:
        p0, p1 = pdist.shard_range(m_total, world, rank)
        c = torch.from_numpy(P.coeffs_log(a, b, n)).to(dev)
        mu_h = torch.zeros((m_total, n + 1), dtype=torch.float64).pin_memory()

        def one():
            if p1 > p0:
                P.moments_host(wl.mode, hA, a, b, n, p0, p1, wl.seed, k, At=hAt, c=wl.r1_c,
                               out=mu_h[p0:p1].numpy())
            mu = mu_h.to(dev, non_blocking=True)
            pdist.combine_moments(mu)
            gp, stats = P.finalize(mu, c)
            s = stats.cpu()
            if s[2].item() != 1.0:
                raise P.ChebError(-5, "non-finite estimate on the e2e path")
            return s
        one()
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            one()
        torch.cuda.synchronize()
        dist.barrier()
        dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        dt = float(dt.item())
        d2h = 8 * (n + 1) * (p1 - p0) + 8 * 3
        h2d_mu = 8 * (n + 1) * m_total
    return {"value": m_total * n * steps / dt, "unit": UNIT, "h2d_bytes_per_step": int(h2d + h2d_mu),
            "d2h_bytes_per_step": int(d2h), "steps": steps, "wall_s_per_step": dt / steps,
            "api": "cheb_logdet_host (C ABI, pinned host CSR)" if world == 1 else
                   "cheb_moments_host per rank (C ABI, pinned host CSR) + NCCL all_reduce + cheb_finalize",
            "includes": ("H2D copy of the CSR from pinned host memory, operator prep, all steps, D2H "
                         "of the result; device workspace from the library's per-thread arena "
                         "(allocated by the warm-up call)")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="gmrf5000")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="strong (default): the config's m probes in total over all GPUs, k = 16; "
                         "weak: m probes per GPU at the best single-GPU block size")
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--basis", choices=["chebyshev", "taylor"], default="chebyshev",
                    help="taylor: the Fig. 1(d) power-series baseline on the same kernels")
    ap.add_argument("--probes", type=int, default=0,
                    help="probes (total for strong scaling, per GPU for weak; default: the config's m)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--ref-budget", type=float, default=15.0, help="seconds of oracle work per sample")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--doubling", action="store_true",
                    help="moment-doubling schedule (ceil(n/2) applications of A~) for the timed region")
    ap.add_argument("--no-alt", action="store_true", help="skip timing the other moment schedule")
    ap.add_argument("--no-weak", action="store_true", help="skip the weak-scaling line")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
