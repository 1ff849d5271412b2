#!/usr/bin/env python
"""Planning-cycle benchmark (BASELINE.json metric: candidate-steps/s and
planning-cycle latency) on 1..8 B200s, plus the reference CPU arm.

  python bench.py [--gpus N --steps K --warmup W --config cN --precision fp32]
  python bench.py --impl reference ...       # reference CPU planner arm

A "step" is one planning cycle: every candidate of the workload rolled out
over the full horizon (N ZOH steps x S=10 Euler substeps of 5 ms), scored,
and the arg-min selected (per GPU, then across GPUs).  One candidate-step =
one 0.05 s ZOH step of one candidate.

Workload: N=1 -> BASELINE configs[1] (c2: K=16384, N=100, 512^2 fractal, 20
obstacles, 10 m/s, random-walk controls), with c3 and c4 timed beside it in
config.rows; N>1 -> BASELINE configs[3] (c4: K=262,144 sharded over the N
GPUs, strong scaling); --weak runs c2 with K=16384 per GPU instead.

GPUs: under torchrun (WORLD_SIZE set) one process per GPU, the cross-GPU
arg-min through the library's NCCL all-gather; without torchrun, --gpus N
drives N GPUs from this one process (the library's device list) and fails
loudly when fewer than N are visible.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import platform
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
# / without the 4 planar-footprint SDF lookups -- DESIGN.md §7.
ALGO_FLOPS_PER_SUBSTEP = {"c1": 548.1, "c2": 628.0, "c3": 547.2, "c4": 628.0, "c5": 548.0}
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2
NCU_SUMMARY = ROOT / "profiles" / "ncu_summary.json"
WEAK_K_PER_GPU = 16384


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, help="c1..c5 (default: c2 at N=1, c4 at N>1)")
    ap.add_argument("--weak", action="store_true", help="N>1: c2 with K=16384 per GPU")
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="minimum CPU work of the cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-rows", action="store_true", help="N=1: skip the c3 / c4 rows")
    ap.add_argument("--row-steps", type=int, default=10)
    ap.add_argument("--shadow-stride", type=int, default=64,
                    help="c5: oracle re-evaluates every n-th candidate of every cycle")
    ap.add_argument("--dry-run", action="store_true",
                    help="no GPU: the multi-rank plumbing (topology, shards, record gather + "
                         "fold, max over ranks) over gloo with synthetic per-candidate outputs")
    return ap.parse_args(argv)


# ----------------------------------------------------------------- topology
def resolve_world(args, need_gpus=True):
    """Who am I and which GPUs do I drive.

    torchrun (WORLD_SIZE set, also 1): one process per GPU, mode "ranks".  Otherwise
    one process driving --gpus N devices, mode "devices" (N = 1: "single").
    Fails loudly (SystemExit) when the GPUs asked for are not there."""
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is not None:  # torchrun, any N (N = 1: a 1-rank communicator)
        world = int(env_world)
        if args.gpus is not None and args.gpus != world:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but torchrun started {world} ranks")
        rank = int(os.environ.get("RANK", "0"))
        local = int(os.environ.get("LOCAL_RANK", str(rank)))
        topo = dict(mode="ranks", rank=rank, world=world, local=local, n_gpus=world,
                    devices=[local])
    else:
        n = args.gpus or 1
        if n < 1:
            raise SystemExit("bench.py: --gpus must be >= 1")
        topo = dict(mode="single" if n == 1 else "devices", rank=0, world=1, local=0, n_gpus=n,
                    devices=list(range(n)))
    if need_gpus:
        import torch
        have = torch.cuda.device_count()
        want = max(topo["devices"]) + 1
        if have < want:
            raise SystemExit(f"bench.py --gpus {topo['n_gpus']}: needs {want} CUDA device(s), "
                             f"{have} visible")
    return topo


def workload_name(args, n_gpus):
    if args.config:
        return args.config
    return "c2" if (n_gpus == 1 or args.weak) else "c4"


def make_workload(args, n_gpus, lib=None):
    from paper_2603_20525_b200 import workloads as W
    name = workload_name(args, n_gpus)
    w = W.make_workload(name, lib=lib)
    if args.weak and name == "c2" and n_gpus > 1:
        w = w.with_(n_samples=WEAK_K_PER_GPU * n_gpus)
    scaling = "weak" if (n_gpus == 1 or args.weak) else "strong"
    return name, w, scaling


def warm_seq_for(w):
    """c5 samples around a warm-start sequence: straight ahead for one cycle."""
    from paper_2603_20525_b200 import planner as PL
    return np.zeros((w.cfg.n_steps, 2)) if w.cfg.sampler == PL.SAMPLE_WARM_GAUSS else None


def native_libs():
    """Shared objects of this repo mapped into the process (evidence of which
    native code ran)."""
    out = set()
    try:
        for line in open("/proc/self/maps"):
            p = line.split()[-1] if line.strip() else ""
            if p.endswith(".so") and str(ROOT) in os.path.realpath(p):
                out.add(os.path.relpath(os.path.realpath(p), ROOT))
    except OSError:
        pass
    return sorted(out)


class ClockSampler:
    """`nvidia-smi -lms 50` clocks + throttle reasons, timestamped so the
    samples inside the timed window can be told apart."""

    Q = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, devices):
        self.devices, self.rows, self.proc = devices, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", ",".join(str(d) for d in self.devices), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi takes a few hundred ms to print its first line: wait
            # for it, so a short timed region still has samples around it
            deadline = time.time() + 3.0
            while not self.rows and self.proc.poll() is None and time.time() < deadline:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [v.strip() for v in line.split(",")]))

    def __exit__(self, *a):
        if self.proc:
            # one more sample after the timed region
            t_end, n0 = time.time(), len(self.rows)
            while (len(self.rows) == n0 and self.proc.poll() is None
                   and time.time() < t_end + 1.0):
                time.sleep(0.01)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t0=None, t1=None):
        rows = [r for ts, r in self.rows if (t0 is None or ts >= t0 - 0.05) and
                (t1 is None or ts <= t1 + 0.05)]
        inside = bool(rows)
        if not rows and self.rows:
            # a timed region shorter than the 50 ms sampling period: the
            # nearest sample on either side of it
            before = [r for ts, r in self.rows if t0 is not None and ts < t0]
            after = [r for ts, r in self.rows if t1 is not None and ts > t1]
            rows = before[-1:] + after[:1] or [r for _, r in self.rows]
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
                "samples": len(rows), "samples_inside_window": inside}


# ----------------------------------------------------------------- CPU side
def cpu_info():
    """CPU model, logical CPUs this process may use, physical cores."""
    model, cores = platform.processor() or "unknown", set()
    try:
        phys = core = None
        for line in open("/proc/cpuinfo"):
            k, _, v = line.partition(":")
            k, v = k.strip(), v.strip()
            if k == "model name":
                model = v
            elif k == "physical id":
                phys = v
            elif k == "core id":
                core = v
            elif not k and core is not None:
                cores.add((phys, core))
                phys = core = None
        if core is not None:
            cores.add((phys, core))
    except OSError:
        pass
    logical = len(os.sched_getaffinity(0))
    return {"model": model, "logical_cpus": logical, "physical_cores": len(cores) or logical}


def cpu_cycle(orc, w, n_cand, threads):
    """The reference CPU planner (oracle/_ref: the unmodified reference headers
    + the SPEC planner loop) on the first n_cand candidates of the workload.
    Returns (candidate-steps, seconds)."""
    from paper_2603_20525_b200 import planner as PL  # pure-Python struct marshalling
    ws = w.with_(n_samples=n_cand)
    p = ws.params()
    smp, _k = PL.make_sampling(ws.cfg, warm_seq=warm_seq_for(ws))
    sd = None if ws.sdist is None else PL.SignedDistanceMap(ws.grid, ws.sdist, True)
    terr, _t = PL.make_terrain(PL.Heightmap(ws.grid, ws.heights), sd)
    t0 = time.perf_counter()
    rc, res, *_ = orc.solve(p, smp, terr, ws.s0, threads=threads)
    return n_cand * p.n_steps, time.perf_counter() - t0


def reference_oracle():
    from oracle.oracle import Oracle
    kind = "reference" if Oracle.available("reference") else "port"
    return Oracle(kind), kind


def pick_pinning(orc, w, n_cand, threads):
    """Pinned (one thread per physical core, TMPC_REF_PIN) or scheduler-placed
    threads, whichever runs the reference faster on this host: the baseline
    is the reference at its best."""
    rates = {}
    for pin in ("1", "0"):
        os.environ["TMPC_REF_PIN"] = pin
        cs, dt = cpu_cycle(orc, w, min(n_cand, 2048), threads)
        rates[pin] = cs / dt
    best = max(rates, key=rates.get)
    os.environ["TMPC_REF_PIN"] = best
    return best == "1", rates


def cpu_baseline(w, name, min_seconds):
    """All physical cores on the first n_cand candidates (>= min_seconds of
    CPU work), plus a single-thread rate on a 1/16 sample."""
    info = cpu_info()
    threads = info["physical_cores"]
    orc, kind = reference_oracle()
    n_cand = min(w.cfg.n_samples, int(os.environ.get("TMPC_REF_SAMPLE", "16384")))
    pinned, rates = pick_pinning(orc, w, n_cand, threads)
    done, secs, reps = 0, 0.0, 0
    while secs < min_seconds or reps == 0:
        cs, dt = cpu_cycle(orc, w, n_cand, threads)
        done, secs, reps = done + cs, secs + dt, reps + 1
    n1 = max(1, n_cand // 16)
    cs1, dt1 = cpu_cycle(orc, w, n1, 1)
    return {"value": done / secs, "unit": "candidate-steps/s", "cores": threads, "kind": kind,
            "cpu_model": info["model"], "physical_cores": info["physical_cores"],
            "logical_cpus": info["logical_cpus"], "pinned": pinned,
            "pinning_probe": {"pinned": rates["1"], "unpinned": rates["0"]},
            "sample": f"{reps} x first {n_cand} of {w.cfg.n_samples} {name} candidates, full "
                      f"horizon, {secs:.1f} s of CPU work on {threads} threads "
                      f"({'pinned' if pinned else 'unpinned'}: the faster of the two)",
            "value_1_thread": cs1 / dt1,
            "sample_1_thread": f"first {n1} candidates, full horizon, {dt1:.1f} s on 1 thread",
            "cycle_ms_all_threads": w.cfg.n_samples * w.cfg.n_steps / (done / secs) * 1e3}


def run_reference(args):
    """The reference's own CPU planner on the box's host cores, on the same
    config, metric and unit as our arm at this N.  Its inputs come from
    oracle/libworkload.so (the same generator source), so this process never
    loads the product library."""
    topo = resolve_world(args, need_gpus=False)
    if topo["rank"] != 0:
        return  # rank 0 alone times the CPU reference
    from oracle.oracle import workload_lib
    name, w, scaling = make_workload(args, topo["n_gpus"], lib=workload_lib())
    info = cpu_info()
    threads = info["physical_cores"]
    orc, kind = reference_oracle()
    n_cand = min(w.cfg.n_samples, int(os.environ.get("TMPC_REF_SAMPLE", "16384")))
    pinned, _rates = pick_pinning(orc, w, n_cand, threads)
    for _ in range(args.warmup):
        cpu_cycle(orc, w, min(n_cand, 512), threads)
    rates, times = [], []
    for _ in range(args.steps):
        cs, dt = cpu_cycle(orc, w, n_cand, threads)
        rates.append(cs / dt)
        times.append(dt * w.cfg.n_samples / n_cand)  # full-cycle latency
    value = statistics.median(rates)
    line = {
        "metric": "candidate-steps/s", "value": value, "unit": "candidate-steps/s",
        "impl": "reference", "n_gpus": topo["n_gpus"], "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": statistics.median(times) * 1e3,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": w.label(), "planning_cycle_ms": statistics.median(times) * 1e3},
        "cpu_baseline": {"value": value, "unit": "candidate-steps/s", "cores": threads,
                         "kind": kind, "cpu_model": info["model"],
                         "physical_cores": info["physical_cores"], "pinned": pinned,
                         "sample": f"per step the first {n_cand} of {w.cfg.n_samples} "
                                   f"candidates, full horizon, {threads} threads "
                                   f"({'pinned' if pinned else 'unpinned'}: the faster)"},
        "e2e": {"value": value, "unit": "candidate-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "native_libs": native_libs(),
    }
    assert not any("libtmpc_b200" in s for s in line["native_libs"]), line["native_libs"]
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU side
class Timer:
    """Per-cycle device time on every GPU this process drives: CUDA events on
    each context stream around the cycle, the L2 of every GPU flushed (256 MB
    write) before the first event.  cycle time = max over the GPUs."""

    def __init__(self, pl):
        import torch
        self.torch = torch
        self.n = pl.n_devices
        self.streams, self.flush = [], []
        for i in range(self.n):
            dev = pl.device_ordinal(i)
            self.streams.append(torch.cuda.ExternalStream(pl.device_stream(i), device=dev))
            self.flush.append(torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32,
                                          device=f"cuda:{dev}"))

    def flush_l2(self):
        for s, f in zip(self.streams, self.flush):
            with self.torch.cuda.stream(s):
                f.zero_()

    def start(self):
        self.flush_l2()
        ev = []
        for s in self.streams:
            e0, e1 = (self.torch.cuda.Event(enable_timing=True),
                      self.torch.cuda.Event(enable_timing=True))
            e0.record(s)
            ev.append((e0, e1))
        return ev

    def stop(self, ev):
        for (e0, e1), s in zip(ev, self.streams):
            e1.record(s)

    @staticmethod
    def elapsed(ev):
        return max(e0.elapsed_time(e1) for e0, e1 in ev)

    def sync(self):
        for s in self.streams:
            s.synchronize()


def time_cycles(pl, w, smp, steps, warmup, dist=None, device=None):
    """Device-resident timing of `steps` cycles (inputs already in HBM):
    returns (per-cycle ms list, kernel ms list, substeps list, wall t0, t1)."""
    import torch
    from paper_2603_20525_b200 import _abi
    lib = pl.lib
    s0 = np.ascontiguousarray(w.s0)
    res = _abi.tmpc_result()
    tm = Timer(pl)

    def cycle():
        assert lib.tmpc_stage_cycle(pl.ctx, _abi.dptr(s0), C.byref(smp)) == 0, pl._err()
        assert lib.tmpc_launch_cycle(pl.ctx) == 0, pl._err()

    def finish():
        assert lib.tmpc_finish_cycle(pl.ctx, C.byref(res)) == 0, pl._err()

    def barrier():
        tm.sync()
        torch.cuda.synchronize(device)
        if dist:
            dist.barrier()
        tm.sync()

    for _ in range(warmup):
        cycle()
        finish()
    evs, kern, sub = [], [], []
    barrier()
    t0 = time.time()
    for _ in range(steps):
        ev = tm.start()
        cycle()
        tm.stop(ev)
        finish()
        evs.append(ev)
        kern.append(res.kernel_ms)
        sub.append(res.substeps_executed)
    barrier()
    t1 = time.time()
    cyc = [tm.elapsed(ev) for ev in evs]
    return cyc, kern, sub, t0, t1, tm


def time_e2e(pl, w, smp, steps, tm, dist=None):
    """The same cycle through the public API (tmpc_solve via Planner.solve_raw):
    host s0 in, result block + winner controls out, every step."""
    e2e = []
    s0 = np.ascontiguousarray(w.s0)
    for _ in range(steps):
        tm.flush_l2()
        tm.sync()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        r, ctrl = pl.solve_raw(s0, smp)
        e2e.append((time.perf_counter() - t0) * 1e3)
    return e2e


def roofline(name, kern_ms, substeps, n_parts, peak_tflops, ncu, ncu_key=None):
    """FP32-SIMT roofline of the rollout kernel: algorithmic flops per launch
    (ALGO_FLOPS_PER_SUBSTEP x substeps one launch executes) / its time."""
    kmean = statistics.mean(kern_ms)
    sub_launch = statistics.mean(substeps) / n_parts
    achieved = ALGO_FLOPS_PER_SUBSTEP.get(name, 600.0) * sub_launch / (kmean * 1e-3) / 1e12
    cfg = ncu.get(ncu_key or name, {})
    return {"bound": "fp32", "achieved": achieved, "peak": peak_tflops, "unit": "TFLOP/s",
            "frac": achieved / peak_tflops if peak_tflops else None,
            "traffic": cfg.get("dram_bytes_per_launch"),
            "peak_source": "FFMA probe on this GPU (tmpc_fp32_peak; MEASURED_PEAKS.json has "
                           "HBM and bf16 only)",
            "algo_flops_per_substep": ALGO_FLOPS_PER_SUBSTEP.get(name),
            "kernel_ms": kmean, "ncu_fma_pipe_pct": cfg.get("fma_pipe_pct"),
            "ncu_issue_active_pct": cfg.get("issue_active_pct"),
            "ncu_l1_sectors_per_request": cfg.get("l1_sectors_per_request"),
            "ncu_source": cfg.get("source")}


def exchange_mode():
    """Cross-rank exchange of the per-GPU records: the rollout kernel's own
    peer-memory stores (default) or NCCL (TMPC_EXCHANGE=nccl)."""
    from paper_2603_20525_b200 import _abi
    return (_abi.EXCHANGE_NCCL if os.environ.get("TMPC_EXCHANGE", "peer").lower() == "nccl"
            else _abi.EXCHANGE_PEER)


def nccl_unique_id(dist):
    """Rank 0's NCCL unique id, broadcast to every rank."""
    from paper_2603_20525_b200 import _abi
    buf = [None]
    if dist.get_rank() == 0:
        idb = C.create_string_buffer(128)
        assert _abi.load().tmpc_nccl_unique_id(idb) == 0
        buf[0] = idb.raw
    dist.broadcast_object_list(buf, src=0)
    return buf[0]


def open_planner(w, topo, prec, nccl_id=None, dist=None):
    from paper_2603_20525_b200 import _abi, planner as PL
    K_total, N = w.cfg.n_samples, w.cfg.n_steps
    if topo["mode"] == "ranks":
        import torch
        k0, kc = PL.shard_range(K_total, topo["rank"], topo["world"])
        xm = exchange_mode()
        pl = None
        if xm == _abi.EXCHANGE_PEER:
            # every rank's mailbox handle, rank order, over torch.distributed;
            # a box without GPU peer access falls back to NCCL on every rank
            ok, mine = 1, None
            try:
                pl = PL.Planner(device=topo["local"], rank=topo["rank"], world_size=topo["world"],
                                k_max=kc, n_steps_max=N, precision=prec, exchange=xm)
                mine = pl.peer_export()
            except RuntimeError as e:
                print(f"bench: peer exchange unavailable ({e})", file=sys.stderr)
                ok = 0
            handles = [mine]
            if dist is not None:
                handles = [None] * topo["world"]
                dist.all_gather_object(handles, mine)
            if ok and all(h is not None for h in handles):
                try:
                    pl.peer_connect(handles)
                except RuntimeError as e:
                    print(f"bench: peer_connect failed ({e})", file=sys.stderr)
                    ok = 0
            else:
                ok = 0
            if dist is not None:
                t = torch.tensor([ok], dtype=torch.int32, device=f"cuda:{topo['local']}")
                dist.all_reduce(t, op=dist.ReduceOp.MIN)
                ok = int(t.item())
            if not ok:
                print("bench: falling back to the NCCL exchange", file=sys.stderr)
                if pl is not None:
                    pl.close()
                pl, xm = None, _abi.EXCHANGE_NCCL
                if dist is not None and nccl_id is None:
                    nccl_id = nccl_unique_id(dist)
        if pl is None:
            pl = PL.Planner(device=topo["local"], rank=topo["rank"], world_size=topo["world"],
                            k_max=kc, n_steps_max=N, precision=prec, exchange=xm,
                            nccl_id=nccl_id)
        pl.exchange = xm
    else:
        k0, kc = 0, K_total
        pl = PL.Planner(devices=topo["devices"], k_max=kc, n_steps_max=N, precision=prec)
    pl.set_params(w.params())
    pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
    smp, keep = PL.make_sampling(w.cfg, k0, kc, warm_seq_for(w))
    return pl, smp, keep


def run_ours(args):
    import torch
    from paper_2603_20525_b200 import _abi
    topo = resolve_world(args)
    dist = None
    torch.cuda.set_device(topo["devices"][0])
    if topo["mode"] == "ranks":
        # the N ranks' NCCL init in the log -- on stderr, so stdout keeps the one JSON line
        # (forced: an inherited NCCL_DEBUG=VERSION would print its banner on stdout)
        os.environ["NCCL_DEBUG"] = "INFO"
        os.environ["NCCL_DEBUG_FILE"] = "/dev/stderr"
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", topo["local"]))
    name, w, scaling = make_workload(args, topo["n_gpus"])
    prec = _abi.PRECISION_FP64 if args.precision == "fp64" else _abi.PRECISION_FP32
    nccl_id = None
    if dist and exchange_mode() == _abi.EXCHANGE_NCCL:
        nccl_id = nccl_unique_id(dist)
    pl, smp, _keep = open_planner(w, topo, prec, nccl_id, dist)
    exch = getattr(pl, "exchange", None)
    K_total, N = w.cfg.n_samples, w.cfg.n_steps
    dev0 = topo["devices"][0]

    def max_over_ranks(v):
        if not dist:
            return v
        t = torch.tensor([v], device=f"cuda:{dev0}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    with ClockSampler(topo["devices"]) as clocks:
        cyc, kern, sub, t0, t1, tm = time_cycles(pl, w, smp, args.steps, args.warmup, dist, dev0)
        launches = int(pl.lib.tmpc_kernels_per_cycle(pl.ctx)) * args.steps
        ms_per_step = max_over_ranks(sum(cyc) / args.steps)
        value = K_total * N / (ms_per_step * 1e-3)
        e2e = time_e2e(pl, w, smp, args.steps, tm, dist)
        e2e_mean = max_over_ranks(statistics.mean(e2e))
    clk = dict(clocks.summary(t0, t1), window="timed region")
    e2e_value = K_total * N / (e2e_mean * 1e-3)
    peak = C.c_double(0.0)
    pl.lib.tmpc_fp32_peak(dev0, C.byref(peak))
    ncu = json.loads(NCU_SUMMARY.read_text()) if NCU_SUMMARY.exists() else {}
    n_parts = pl.n_devices if topo["mode"] != "ranks" else 1
    roof = roofline(name, kern, [s / (topo["world"]) for s in sub], n_parts, peak.value, ncu)
    launches = int(max_over_ranks(launches))
    if topo["rank"] != 0:
        pl.close()
        if dist:
            dist.destroy_process_group()
        return
    rows = {}
    if topo["n_gpus"] == 1 and not args.no_rows and not args.config:
        pl.close()
        pl = None
        for rname in ("c3", "c4"):
            rows[rname] = bench_row(rname, topo, prec, args, peak.value, ncu)
        # the per-GPU work of the 8-GPU c4 and c5 cycles (north-star scale)
        rows["c4_shard_of_8"] = shard_row("c4", 8, topo, prec, args, peak.value, ncu)
        rows["c5_shard_of_8"] = shard_row("c5", 8, topo, prec, args, peak.value, ncu)
        # BASELINE configs[4]: the receding-horizon loop, per-cycle shadow oracle
        rows["c5_closed_loop"] = closed_loop_row(topo, prec, args, cycles=200, warmup=3,
                                                 stride=max(args.shadow_stride, 256))
    cpu = None
    if not args.no_cpu_baseline and topo["n_gpus"] == 1:
        cpu = cpu_baseline(w, name, args.cpu_seconds)
    line = {
        "metric": "candidate-steps/s", "value": value, "unit": "candidate-steps/s",
        "n_gpus": topo["n_gpus"], "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
        "config": {"workload": w.label(),
                   "planning_cycle_ms": ms_per_step,
                   "planning_cycle_ms_p50": statistics.median(cyc),
                   "planning_cycle_ms_p99": float(np.percentile(cyc, 99)),
                   "parallelism": {"single": "one GPU",
                                   "devices": f"candidates sharded over {topo['n_gpus']} GPUs "
                                              "driven by one process (records folded on the host)",
                                   "ranks": f"candidates sharded over {topo['n_gpus']} ranks "
                                            "(one process per GPU; the per-GPU arg-min records "
                                            + ("exchanged by the rollout kernel over peer memory)"
                                               if exch == _abi.EXCHANGE_PEER
                                               else "all-gathered by NCCL)")}[topo["mode"]],
                   "l2": "flushed (256 MB write per GPU) between timed cycles",
                   "substeps_per_s": K_total * N * 10 / (ms_per_step * 1e-3),
                   # the paper's unit: 800-substep (4 s at 5 ms) rollouts per second
                   "paper_samples_per_s_800_substeps": K_total * N * 10 / (ms_per_step * 1e-3) / 800,
                   "executed_substep_fraction": statistics.mean(sub) / (K_total * N * 10),
                   "precision": args.precision, "rows": rows},
        "e2e": {"value": e2e_value, "unit": "candidate-steps/s", "h2d_bytes_per_step": 13 * 8,
                # per-GPU reduction records, 112 B each: written into mapped
                # host memory by the kernel's last block (one process), or
                # every rank's record copied home after the exchange
                "d2h_bytes_per_step": (112 * topo["world"] + 8 if topo["mode"] == "ranks"
                                       else 112 * topo["n_gpus"]),
                "cycle_ms": e2e_mean,
                "api": "tmpc_solve: host s0 (104 B) in, per-GPU records + result out, winner "
                       "controls regenerated on the host from (seed, index)"},
        "roofline": roof,
        "cpu_baseline": cpu,
        "clocks": clk,
        "gpu_launches": launches,
        "native_libs": native_libs(),
    }
    print(json.dumps(line), flush=True)
    if pl:
        pl.close()
    if dist:
        dist.destroy_process_group()


def bench_row(name, topo, prec, args, peak, ncu):
    """One more BASELINE config on the same GPU(s): device cycle time, the
    public-API cycle, roofline and clocks (config.rows of the N=1 line)."""
    from paper_2603_20525_b200 import workloads as W
    w = W.make_workload(name)
    pl, smp, keep = open_planner(w, topo, prec)
    with ClockSampler(topo["devices"]) as clocks:
        cyc, kern, sub, t0, t1, tm = time_cycles(pl, w, smp, args.row_steps, args.warmup)
        e2e = time_e2e(pl, w, smp, max(3, args.row_steps // 2), tm)
    K, N = w.cfg.n_samples, w.cfg.n_steps
    ms = sum(cyc) / len(cyc)
    row = {"workload": w.label(), "value": K * N / (ms * 1e-3), "unit": "candidate-steps/s",
           "ms_per_step": ms, "planning_cycle_ms_p50": statistics.median(cyc),
           "steps": args.row_steps,
           "e2e": {"value": K * N / (statistics.mean(e2e) * 1e-3),
                   "cycle_ms": statistics.mean(e2e)},
           "roofline": roofline(name, kern, sub, pl.n_devices, peak, ncu),
           "clocks": dict(clocks.summary(t0, t1), window="timed region"),
           "gpu_launches": int(pl.lib.tmpc_kernels_per_cycle(pl.ctx)) * args.row_steps}
    pl.close()
    return row


def shard_row(name, g, topo, prec, args, peak, ncu):
    """GPU 0's share of BASELINE config `name` sharded over g GPUs, timed on
    this GPU: the contiguous shard [0, K/g) with the whole problem's lane
    layout (k_total = K), i.e. the per-GPU work of the g-GPU cycle without the
    cross-GPU exchange (config.rows of the N=1 line)."""
    from paper_2603_20525_b200 import planner as PL, workloads as W
    w = W.make_workload(name)
    K, N = w.cfg.n_samples, w.cfg.n_steps
    k0, kc = PL.shard_range(K, 0, g)
    pl = PL.Planner(device=topo["devices"][0], k_max=kc, n_steps_max=N, precision=prec)
    pl.set_params(w.params())
    pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
    smp, keep = PL.make_sampling(w.cfg, k0, kc, warm_seq_for(w))
    with ClockSampler(topo["devices"]) as clocks:
        cyc, kern, sub, t0, t1, tm = time_cycles(pl, w, smp, args.row_steps, args.warmup)
    ms = sum(cyc) / len(cyc)
    row = {"workload": f"shard 0 of {g}: candidates [{k0}, {k0 + kc}) of {w.label()}",
           "value": kc * N / (ms * 1e-3), "unit": "candidate-steps/s", "ms_per_step": ms,
           "planning_cycle_ms_p50": statistics.median(cyc), "steps": args.row_steps,
           "roofline": roofline(name, kern, sub, 1, peak, ncu, ncu_key=f"{name}_shard_of_{g}"),
           "clocks": dict(clocks.summary(t0, t1), window="timed region"),
           "gpu_launches": int(pl.lib.tmpc_kernels_per_cycle(pl.ctx)) * args.row_steps}
    pl.close()
    return row


def closed_loop_row(topo, prec, args, cycles, warmup, stride):
    """BASELINE c5: `cycles` consecutive receding-horizon cycles (warm-started
    Gaussian candidates around the shifted previous winner, RK4 1 ms plant
    between cycles).  A step = one planning cycle through tmpc_solve (host
    state in, winner out) followed by the plant; p50/p99 cycle latency.  With
    stride > 0 the CPU oracle re-evaluates, every cycle and on the same plant
    state, every stride-th candidate plus the device's 64 best, and the
    north-star winner rule is applied per cycle (oracle/shadow.py: a checker
    outside the timed planning calls)."""
    from paper_2603_20525_b200 import closed_loop as CL, workloads as W
    w = W.make_workload("c5")
    loop = CL.ClosedLoop(w.heights, w.grid, w.sdist, w.goal, w.cfg)
    plan = loop.device_planner(devices=topo["devices"], precision=prec)
    loop.run(plan, w.s0, cycles=warmup)  # warm-up trial
    shadow = None
    if stride > 0:
        from oracle.shadow import ShadowCheck
        shadow = ShadowCheck(loop, reference_oracle()[0], stride=stride,
                             threads=cpu_info()["physical_cores"])
    with ClockSampler(topo["devices"]) as clocks:
        t0 = time.time()
        rec = loop.run(plan, w.s0, cycles=cycles, shadow=shadow)
        t1 = time.time()
    lat = rec.latencies()
    kern = np.array([c.kernel_ms for c in rec.cycles])
    K, N = w.cfg.n_samples, w.cfg.n_steps
    p50, p99 = rec.p50_p99()
    launches = int(plan.planner.lib.tmpc_kernels_per_cycle(plan.planner.ctx)) * len(rec.cycles)
    plan.planner.close()
    return {"workload": f"c5 closed loop: {w.label()}, warm-started Gaussian (sigma 10% range), "
                        "RK4 1 ms plant",
            "value": K * N / (kern.mean() * 1e-3), "unit": "candidate-steps/s",
            "ms_per_step": float(kern.mean()), "planning_cycle_ms_p50": p50,
            "planning_cycle_ms_p99": p99, "outcome": rec.outcome, "cycles": len(rec.cycles),
            "e2e": {"value": K * N / (lat.mean() * 1e-3), "unit": "candidate-steps/s",
                    "cycle_ms": float(lat.mean())},
            "shadow_oracle": shadow.summary() if shadow else None,
            "clocks": dict(clocks.summary(t0, t1), window="closed loop"),
            "gpu_launches": launches}


def run_closed_loop(args):
    """`bench.py --config c5`: the closed loop as its own line."""
    import torch
    from paper_2603_20525_b200 import _abi
    topo = resolve_world(args)
    torch.cuda.set_device(topo["devices"][0])
    prec = _abi.PRECISION_FP64 if args.precision == "fp64" else _abi.PRECISION_FP32
    row = closed_loop_row(topo, prec, args, cycles=args.steps, warmup=args.warmup,
                          stride=args.shadow_stride)
    line = {
        "metric": "candidate-steps/s", "value": row["value"], "unit": "candidate-steps/s",
        "n_gpus": topo["n_gpus"], "steps": row["cycles"], "warmup": args.warmup,
        "ms_per_step": row["ms_per_step"], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
        "config": {"workload": row["workload"],
                   "planning_cycle_ms_p50": row["planning_cycle_ms_p50"],
                   "planning_cycle_ms_p99": row["planning_cycle_ms_p99"],
                   "outcome": row["outcome"], "cycles": row["cycles"],
                   "shadow_oracle": row["shadow_oracle"]},
        "e2e": dict(row["e2e"], h2d_bytes_per_step=13 * 8 + 100 * 2 * 8, d2h_bytes_per_step=112),
        "clocks": row["clocks"],
        "gpu_launches": row["gpu_launches"],
        "native_libs": native_libs(),
    }
    print(json.dumps(line), flush=True)


def synthetic_outputs(k0, kc):
    """Deterministic stand-in per-candidate outputs of global candidates
    [k0, k0 + kc) (dry run): cost, flags, margin, substeps from a hash of k."""
    k = np.arange(k0, k0 + kc, dtype=np.uint64)
    h = (k * np.uint64(0x9E3779B97F4A7C15)) ^ (k >> np.uint64(7))
    cost = 50.0 + (h % np.uint64(1 << 20)).astype(np.float64) * 1e-3
    cost[(h % np.uint64(97)) == 0] = np.inf
    flags = np.where(np.isfinite(cost), ((h >> np.uint64(3)) % np.uint64(3) == 0).astype(np.uint8), 2)
    margin = ((h % np.uint64(1000)).astype(np.float32) - 500.0) * 1e-3
    sub = (h % np.uint64(1000)).astype(np.int64)
    return cost, flags.astype(np.uint8), margin, sub


def run_dry(args):
    """The N-rank code path without a GPU: torchrun env -> topology, the
    workload's contiguous shards, each rank's record (tmpc_make_record, the
    host mirror of the kernel's reduction), the records gathered in rank order
    (gloo all_gather in place of the library's ncclAllGather), the fold
    (tmpc_fold_records), max over ranks of the time."""
    import torch
    import torch.distributed as dist
    from paper_2603_20525_b200 import planner as PL
    topo = resolve_world(args, need_gpus=False)
    if topo["mode"] == "ranks":
        dist.init_process_group("gloo")
    else:
        dist = None
    name, w, scaling = make_workload(args, topo["n_gpus"])
    K = w.cfg.n_samples
    t0 = time.perf_counter()
    k0, kc = PL.shard_range(K, topo["rank"], topo["world"])
    rec = PL.make_record(*synthetic_outputs(k0, kc)[:3], k0, substeps=synthetic_outputs(k0, kc)[3])
    recs = [rec]
    if dist:
        got = [None] * topo["world"]
        dist.all_gather_object(got, PL.record_bytes(rec))
        recs = [PL.record_from_bytes(b) for b in got]
    res = PL.fold_records(recs)
    ms = (time.perf_counter() - t0) * 1e3
    if dist:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if topo["rank"] == 0:
        print(json.dumps({"dry_run": True, "n_gpus": topo["n_gpus"], "mode": topo["mode"],
                          "workload": w.label(), "scaling": scaling, "shard0": [k0, kc],
                          "best_index": int(res.best_index), "best_cost": res.best_cost,
                          "n_candidates": int(res.n_candidates),
                          "n_feasible": int(res.n_feasible), "mean_cost": res.mean_cost,
                          "result_hex": bytes(res).hex(), "ms": ms}), flush=True)
    if dist:
        dist.destroy_process_group()


def main(argv=None):
    args = parse(argv)
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    elif args.config == "c5":
        run_closed_loop(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
