#!/usr/bin/env python
"""Planning-cycle benchmark (BASELINE.json metric: candidate-steps/s and
planning-cycle latency) on 1..8 B200s, plus the reference CPU arm.

  python bench.py [--gpus N --steps K --warmup W --config c2 --precision fp32]
  python bench.py --impl reference ...       # reference CPU planner arm

A "step" is one planning cycle: every candidate of the workload rolled out
over the full horizon (N ZOH steps x S=10 Euler substeps), scored, and the
arg-min selected (per GPU, then across GPUs with one NCCL MIN).  One
candidate-step = one 0.05 s ZOH step of one candidate.

Default workload at N=1 is BASELINE configs[1] (c2: K=16384, N=100, 512^2
fractal, 20 obstacles, 10 m/s, random-walk controls); for N>1 the same
per-GPU shard (K=16384 per GPU, weak scaling).  --config c4 runs the
K=262,144 sharded cycle (strong scaling).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# Algorithmic fp32 work of one candidate-substep, counted by the op-counting
# oracle run (oracle variant 4; FMA = 2 flops, divides counted, the 12
# sin/cos, 4 atan and 4 sqrt not counted) — DESIGN.md §6.
ALGO_FLOPS_PER_SUBSTEP = {"c1": 548.1, "c2": 628.0, "c3": 547.2, "c4": 628.0, "c5": 548.0}
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, help="c1..c5 (default c2)")
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.samples, self.stop = device, [], threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)

    def run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device),
                                      f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.1)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def workload_for(args, world):
    from paper_2603_20525_b200 import workloads as W
    name = args.config or "c2"
    w = W.make_workload(name)
    if name == "c2" and world > 1:  # weak scaling: the c2 shard on every GPU
        w = w.with_(n_samples=w.cfg.n_samples * world)
    return name, w


def cpu_reference_rate(w, n_cand, threads, kind="reference"):
    """Reference CPU planner (oracle/_ref, else the restatement) on the first
    n_cand candidates of the workload: candidate-steps/s, wall seconds."""
    from oracle.oracle import Oracle
    from paper_2603_20525_b200 import planner as PL
    if kind == "reference" and not Oracle.available("reference"):
        kind = "port"
    orc = Oracle(kind)
    ws = w.with_(n_samples=n_cand)
    p = ws.params()
    smp, _k = PL.make_sampling(ws.cfg)
    sd = None if ws.sdist is None else PL.SignedDistanceMap(ws.grid, ws.sdist, True)
    terr, _t = PL.make_terrain(PL.Heightmap(ws.grid, ws.heights), sd)
    t0 = time.perf_counter()
    rc, res, *_ = orc.solve(p, smp, terr, ws.s0, threads=threads)
    dt = time.perf_counter() - t0
    return n_cand * p.n_steps / dt, dt, kind, int(res.substeps_executed)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return  # rank 0 alone times the CPU reference
    name, w = workload_for(args, 1)
    threads = os.cpu_count() or 1
    n_cand = int(os.environ.get("TMPC_REF_SAMPLE", "2048"))
    for _ in range(args.warmup):
        cpu_reference_rate(w, min(n_cand, 256), threads)
    rates, times = [], []
    kind = "reference"
    for _ in range(args.steps):
        r, dt, kind, _sub = cpu_reference_rate(w, n_cand, threads)
        rates.append(r)
        times.append(dt)
    value = statistics.median(rates)
    cycle_ms = w.cfg.n_samples * w.cfg.n_steps / value * 1e3
    line = {
        "metric": "candidate-steps/s", "value": value, "unit": "candidate-steps/s",
        "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.median(times) * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{name}: K={w.cfg.n_samples} N={w.cfg.n_steps} S=10 "
                   f"grid={w.grid.nx}^2 obstacles={0 if w.polys is None else len(w.polys[0]) - 1}",
                   "planning_cycle_ms_extrapolated": cycle_ms},
        "cpu_baseline": {"value": value, "unit": "candidate-steps/s", "cores": threads,
                         "kind": kind, "sample": f"first {n_cand} of {w.cfg.n_samples} "
                         f"candidates, full horizon, per step"},
        "e2e": {"value": value, "unit": "candidate-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    from paper_2603_20525_b200 import _abi, planner as PL
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    name, w = workload_for(args, world)
    prec = _abi.PRECISION_FP64 if args.precision == "fp64" else _abi.PRECISION_FP32
    K_total, N = w.cfg.n_samples, w.cfg.n_steps
    k0, kc = PL.shard_range(K_total, rank, world)
    nccl_id = None
    if world > 1:
        buf = [None]
        if rank == 0:
            idb = C.create_string_buffer(128)
            assert _abi.load().tmpc_nccl_unique_id(idb) == 0
            buf[0] = idb.raw
        dist.broadcast_object_list(buf, src=0)
        nccl_id = buf[0]
    pl = PL.Planner(device=local, rank=rank, world_size=world, k_max=kc, n_steps_max=N,
                    nccl_id=nccl_id, precision=prec)
    p = w.params()
    pl.set_params(p)
    pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
    smp, _keep = PL.make_sampling(w.cfg, k0, kc)
    lib = pl.lib
    stream = torch.cuda.ExternalStream(lib.tmpc_get_stream(pl.ctx), device=local)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=f"cuda:{local}")
    s0 = np.ascontiguousarray(w.s0)
    res = _abi.tmpc_result()

    def cycle_device():
        assert lib.tmpc_stage_cycle(pl.ctx, _abi.dptr(s0), C.byref(smp)) == 0
        assert lib.tmpc_launch_cycle(pl.ctx) == 0, pl._err()

    def finish():
        rc = lib.tmpc_finish_cycle(pl.ctx, C.byref(res))
        assert rc == 0, pl._err()

    # ---- warm-up
    for _ in range(args.warmup):
        cycle_device()
        finish()

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident timing: events on the context stream around each
    # cycle; L2 flushed (256 MB write) between timed cycles, outside the events
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    kern_ms, substeps = [], []
    barrier()
    with ClockSampler(local) as clocks:
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
                ev[i][0].record(stream)
            cycle_device()
            ev[i][1].record(stream)
            finish()
            kern_ms.append(res.kernel_ms)
            substeps.append(res.substeps_executed)
        barrier()
    cyc_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(cyc_ms)
    if dist:
        t = torch.tensor([total_ms], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = K_total * N / (ms_per_step * 1e-3)

    # ---- end to end through the public API: host s0 in, winner controls out
    barrier()
    e2e_ms = []
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r, ctrl = pl.solve_raw(s0, smp)
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_mean = statistics.mean(e2e_ms)
    if dist:
        t = torch.tensor([e2e_mean], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_mean = float(t.item())
    e2e_value = K_total * N / (e2e_mean * 1e-3)

    # ---- roofline of the rollout kernel (FP32 SIMT bound)
    kmean = statistics.mean(kern_ms)
    sub_mean = statistics.mean(substeps) / world if world > 1 else statistics.mean(substeps)
    flops = ALGO_FLOPS_PER_SUBSTEP.get(name, 600.0) * sub_mean
    achieved = flops / (kmean * 1e-3) / 1e12
    peak = C.c_double(0.0)
    lib.tmpc_fp32_peak(local, C.byref(peak))
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        pl.close()
        return
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        n_cand = int(os.environ.get("TMPC_REF_SAMPLE", "2048"))
        rate, dt, kind, _ = cpu_reference_rate(w, n_cand, os.cpu_count() or 1)
        cpu = {"value": rate, "unit": "candidate-steps/s", "cores": os.cpu_count() or 1,
               "kind": kind, "sample": f"first {n_cand} of {K_total} candidates, full "
               f"horizon ({dt:.1f} s wall, all host threads)"}
    clk = clocks.summary()
    line = {
        "metric": "candidate-steps/s", "value": value, "unit": "candidate-steps/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak" if (name == "c2" and world > 1) or world == 1 else "strong",
        "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
        "config": {"workload": f"{name}: K={K_total} N={N} S=10 grid={w.grid.nx}^2 "
                   f"obstacles={0 if w.polys is None else len(w.polys[0]) - 1} v0={w.v0} m/s",
                   "planning_cycle_ms": ms_per_step, "parallelism": f"candidates sharded over {world} GPU",
                   "l2": "flushed (256 MB write) between timed cycles",
                   "substeps_per_s": statistics.mean(substeps) / (ms_per_step * 1e-3),
                   "executed_fraction": statistics.mean(substeps) / (K_total * N * 10) * (world if world > 1 else 1),
                   "precision": args.precision},
        "e2e": {"value": e2e_value, "unit": "candidate-steps/s", "h2d_bytes_per_step": 13 * 8,
                "d2h_bytes_per_step": 88, "cycle_ms": e2e_mean,
                "api": "tmpc_solve (host s0 -> device, result + winner controls -> host)"},
        "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak.value,
                     "unit": "TFLOP/s", "frac": achieved / peak.value if peak.value else None,
                     "traffic": None,
                     "peak_source": "FFMA probe on this GPU (MEASURED_PEAKS.json has no FP32 entry)",
                     "algo_flops_per_substep": ALGO_FLOPS_PER_SUBSTEP.get(name),
                     "kernel_ms": kmean},
        "cpu_baseline": cpu,
        "clocks": clk,
        "gpu_launches": int(lib.tmpc_kernels_per_cycle(pl.ctx)) * args.steps,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    pl.close()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
