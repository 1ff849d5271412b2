#!/usr/bin/env python
"""Planning-cycle benchmark (BASELINE.json metric: candidate-steps/s and
planning-cycle latency) on 1..8 B200s, plus the reference CPU arm.

  python bench.py [--gpus N --steps K --warmup W --config c2 --precision fp32]
  python bench.py --impl reference ...       # reference CPU planner arm

A "step" is one planning cycle: every candidate of the workload rolled out
over the full horizon (N ZOH steps x S=10 Euler substeps of 5 ms), scored,
and the arg-min selected (per GPU, then across GPUs with one NCCL MIN).  One
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
# oracle run (oracle variant 4 over the device algorithm: FMA = 2 flops,
# divides counted as 1; the 12 sin/cos, 4 atan and 4 sqrt not counted), with
# / without the 4 planar-footprint SDF lookups — DESIGN.md §6.
ALGO_FLOPS_PER_SUBSTEP = {"c1": 548.1, "c2": 628.0, "c3": 547.2, "c4": 628.0, "c5": 548.0}
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2
NCU_SUMMARY = ROOT / "profiles" / "ncu_summary.json"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, help="c1..c5 (default c2)")
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="minimum CPU work of the cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """`nvidia-smi -lms 50` clocks + throttle reasons, timestamped so the
    samples inside the timed window can be told apart."""

    Q = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device, self.rows, self.proc = device, [], None
        self.windows = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [v.strip() for v in line.split(",")]))

    def mark(self, name):
        self.windows.append((name, time.time()))

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t0=None, t1=None):
        rows = [r for ts, r in self.rows if (t0 is None or ts >= t0) and (t1 is None or ts <= t1)]
        if not rows:
            rows = [r for _, r in self.rows]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}

        def num(v):
            try:
                return float(v)
            except ValueError:
                return None
        sm = [num(r[1]) for r in rows if len(r) > 2 and num(r[1]) is not None]
        mx = [num(r[2]) for r in rows if len(r) > 2 and num(r[2]) is not None]
        reasons = sorted({self.NAMES[i] for r in rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def workload_for(args, world):
    from paper_2603_20525_b200 import workloads as W
    name = args.config or "c2"
    w = W.make_workload(name)
    if name == "c2" and world > 1:  # weak scaling: the c2 shard on every GPU
        w = w.with_(n_samples=w.cfg.n_samples * world)
    return name, w


def cpu_cycle(w, n_cand, threads, kind="reference"):
    """The reference CPU planner (oracle/_ref: the unmodified reference headers
    + the SPEC planner loop; the restatement if _ref is absent) on the first
    n_cand candidates of the workload.  Returns (candidate-steps, seconds, kind)."""
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
    return n_cand * p.n_steps, time.perf_counter() - t0, kind


def cpu_baseline(w, name, min_seconds):
    """All host threads on the first n_cand candidates (>= min_seconds of CPU
    work), plus a single-thread rate on a 1/16 sample (SURVEY §8(d) asks for
    both)."""
    threads = os.cpu_count() or 1
    n_cand = min(w.cfg.n_samples, int(os.environ.get("TMPC_REF_SAMPLE", "16384")))
    done, secs, reps, kind = 0, 0.0, 0, "reference"
    while secs < min_seconds or reps == 0:
        cs, dt, kind = cpu_cycle(w, n_cand, threads)
        done, secs, reps = done + cs, secs + dt, reps + 1
    n1 = max(1, n_cand // 16)
    cs1, dt1, _ = cpu_cycle(w, n1, 1)
    return {"value": done / secs, "unit": "candidate-steps/s", "cores": threads, "kind": kind,
            "sample": f"{reps} x first {n_cand} of {w.cfg.n_samples} {name} candidates, full "
                      f"horizon, {secs:.1f} s of CPU work on {threads} host threads",
            "value_1_thread": cs1 / dt1,
            "sample_1_thread": f"first {n1} candidates, full horizon, {dt1:.1f} s on 1 thread",
            "cycle_ms_all_threads": w.cfg.n_samples * w.cfg.n_steps / (done / secs) * 1e3}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return  # rank 0 alone times the CPU reference
    # the same workload (config) as our arm at this N; each step times a
    # bounded candidate sample of it on all host threads (rate-based)
    name, w = workload_for(args, world)
    threads = os.cpu_count() or 1
    n_cand = min(w.cfg.n_samples, int(os.environ.get("TMPC_REF_SAMPLE", "16384")))
    for _ in range(args.warmup):
        cpu_cycle(w, min(n_cand, 512), threads)
    rates, times = [], []
    kind = "reference"
    for _ in range(args.steps):
        cs, dt, kind = cpu_cycle(w, n_cand, threads)
        rates.append(cs / dt)
        times.append(dt * w.cfg.n_samples / n_cand)  # full-cycle latency
    value = statistics.median(rates)
    line = {
        "metric": "candidate-steps/s", "value": value, "unit": "candidate-steps/s",
        "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.median(times) * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{name}: K={w.cfg.n_samples} N={w.cfg.n_steps} S=10 "
                   f"grid={w.grid.nx}^2 obstacles={0 if w.polys is None else len(w.polys[0]) - 1}",
                   "planning_cycle_ms": statistics.median(times) * 1e3},
        "cpu_baseline": {"value": value, "unit": "candidate-steps/s", "cores": threads,
                         "kind": kind, "sample": f"per step the first {n_cand} of "
                         f"{w.cfg.n_samples} candidates, full horizon"},
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

    def launch():
        assert lib.tmpc_stage_cycle(pl.ctx, _abi.dptr(s0), C.byref(smp)) == 0
        assert lib.tmpc_launch_cycle(pl.ctx) == 0, pl._err()

    def finish():
        assert lib.tmpc_finish_cycle(pl.ctx, C.byref(res)) == 0, pl._err()

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    with ClockSampler(local) as clocks:
        for _ in range(args.warmup):
            launch()
            finish()
        # ---- device-resident timing: events on the context stream around each
        # cycle; L2 flushed (256 MB write) between timed cycles, outside the events
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        kern_ms, substeps = [], []
        barrier()
        t_start = time.time()
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
                ev[i][0].record(stream)
            launch()
            ev[i][1].record(stream)
            finish()
            kern_ms.append(res.kernel_ms)
            substeps.append(res.substeps_executed)
        barrier()
        t_end = time.time()
        cyc_ms = [a.elapsed_time(b) for a, b in ev]
        total_ms = sum(cyc_ms)
        if dist:
            t = torch.tensor([total_ms], device=f"cuda:{local}", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            total_ms = float(t.item())
        ms_per_step = total_ms / args.steps
        value = K_total * N / (ms_per_step * 1e-3)

        # ---- end to end through the public API: host s0 in (tmpc_solve), the
        # result block and the regenerated winner controls out
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
    sub_local = statistics.mean(substeps) / world
    flops = ALGO_FLOPS_PER_SUBSTEP.get(name, 600.0) * sub_local
    achieved = flops / (kmean * 1e-3) / 1e12
    peak = C.c_double(0.0)
    lib.tmpc_fp32_peak(local, C.byref(peak))
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        pl.close()
        return
    ncu = json.loads(NCU_SUMMARY.read_text()) if NCU_SUMMARY.exists() else {}
    ncu_cfg = ncu.get(name, {})
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = cpu_baseline(w, name, args.cpu_seconds)
    line = {
        "metric": "candidate-steps/s", "value": value, "unit": "candidate-steps/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak" if (name == "c2" or world == 1) else "strong",
        "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
        "config": {"workload": f"{name}: K={K_total} N={N} S=10 grid={w.grid.nx}^2 "
                   f"obstacles={0 if w.polys is None else len(w.polys[0]) - 1} v0={w.v0} m/s",
                   "planning_cycle_ms": ms_per_step,
                   "planning_cycle_ms_p50": statistics.median(cyc_ms),
                   "planning_cycle_ms_p99": float(np.percentile(cyc_ms, 99)),
                   "parallelism": f"candidates sharded over {world} GPU(s)",
                   "l2": "flushed (256 MB write) between timed cycles",
                   "substeps_per_s": K_total * N * 10 / (ms_per_step * 1e-3),
                   # the paper's unit: 800-substep (4 s at 5 ms) rollouts per second
                   "paper_samples_per_s_800_substeps": K_total * N * 10 / (ms_per_step * 1e-3) / 800,
                   "executed_substep_fraction": statistics.mean(substeps) / (K_total * N * 10),
                   "lanes_per_candidate": "auto", "precision": args.precision},
        "e2e": {"value": e2e_value, "unit": "candidate-steps/s", "h2d_bytes_per_step": 13 * 8,
                "d2h_bytes_per_step": 88, "cycle_ms": e2e_mean,
                "api": "tmpc_solve: host s0 (104 B) in, result block (88 B) out, winner "
                       "controls regenerated on the host from (seed, index)"},
        "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak.value,
                     "unit": "TFLOP/s", "frac": achieved / peak.value if peak.value else None,
                     "traffic": ncu_cfg.get("dram_bytes_per_launch"),
                     "peak_source": "FFMA probe on this GPU (tmpc_fp32_peak; "
                                    "MEASURED_PEAKS.json has HBM and bf16 only)",
                     "algo_flops_per_substep": ALGO_FLOPS_PER_SUBSTEP.get(name),
                     "kernel_ms": kmean,
                     "ncu_fma_pipe_pct": ncu_cfg.get("fma_pipe_pct"),
                     "ncu_issue_active_pct": ncu_cfg.get("issue_active_pct"),
                     "ncu_l1_sectors_per_request": ncu_cfg.get("l1_sectors_per_request"),
                     "ncu_source": ncu_cfg.get("source"),
                     # the same kernel where the batch gives >= 2 warps per scheduler
                     "ncu_fma_pipe_pct_by_config": {c: v.get("fma_pipe_pct") for c, v in ncu.items()
                                                    if c in ("c2", "c3", "c4")},
                     "note": "latency-bound at c2: 512 warps = 0.86 per scheduler, the cycle is "
                             "within 2% of one warp's in-order substep chain (DESIGN.md section 7)"},
        "cpu_baseline": cpu,
        "clocks": dict(clocks.summary(t_start, t_end), window="timed region (+-50 ms)"),
        "gpu_launches": int(lib.tmpc_kernels_per_cycle(pl.ctx)) * args.steps,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    pl.close()


def run_closed_loop(args):
    """BASELINE c5: `--steps` consecutive receding-horizon cycles (warm-started
    Gaussian candidates around the shifted previous winner, RK4 1 ms plant
    between cycles).  A step = one planning cycle through tmpc_solve (host
    state in, winner out) followed by the plant; p50/p99 cycle latency."""
    import torch
    from paper_2603_20525_b200 import _abi, closed_loop as CL, workloads as W
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = W.make_workload("c5")
    nccl_id = None
    if world > 1:
        buf = [None]
        if rank == 0:
            idb = C.create_string_buffer(128)
            assert _abi.load().tmpc_nccl_unique_id(idb) == 0
            buf[0] = idb.raw
        dist.broadcast_object_list(buf, src=0)
        nccl_id = buf[0]
    prec = _abi.PRECISION_FP64 if args.precision == "fp64" else _abi.PRECISION_FP32
    loop = CL.ClosedLoop(w.heights, w.grid, w.sdist, w.goal, w.cfg)
    plan = loop.device_planner(device=local, precision=prec, rank=rank, world_size=world,
                               nccl_id=nccl_id)
    loop.run(plan, w.s0, cycles=args.warmup)  # warm-up trial
    if dist:
        dist.barrier()
    with ClockSampler(local) as clocks:
        t0 = time.time()
        rec = loop.run(plan, w.s0, cycles=args.steps)
        t1 = time.time()
    lat = rec.latencies()
    kern = np.array([c.kernel_ms for c in rec.cycles])
    if dist:
        t = torch.tensor([lat.mean(), kern.mean()], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        lat_mean, kern_mean = t.tolist()
    else:
        lat_mean, kern_mean = float(lat.mean()), float(kern.mean())
    if rank == 0:
        K, N = w.cfg.n_samples, w.cfg.n_steps
        p50, p99 = rec.p50_p99()
        line = {
            "metric": "candidate-steps/s", "value": K * N / (kern_mean * 1e-3),
            "unit": "candidate-steps/s", "n_gpus": world, "steps": len(rec.cycles),
            "warmup": args.warmup, "ms_per_step": kern_mean, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
            "config": {"workload": f"c5 closed loop: K={K} N={N} S=10 grid={w.grid.nx}^2, "
                       "warm-started Gaussian (sigma 10% range), RK4 1 ms plant",
                       "planning_cycle_ms_p50": p50, "planning_cycle_ms_p99": p99,
                       "outcome": rec.outcome, "cycles": len(rec.cycles)},
            "e2e": {"value": K * N / (lat_mean * 1e-3), "unit": "candidate-steps/s",
                    "h2d_bytes_per_step": 13 * 8 + N * 2 * 8, "d2h_bytes_per_step": 88,
                    "cycle_ms": lat_mean},
            "clocks": dict(clocks.summary(t0, t1), window="closed loop"),
            "gpu_launches": int(plan.planner.lib.tmpc_kernels_per_cycle(plan.planner.ctx))
                            * len(rec.cycles),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.config == "c5":
        run_closed_loop(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
