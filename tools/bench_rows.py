"""Measurement of every SURVEY §8 row beside the reference CPU implementation
on the same box (dev tool; results -> profiles/r01_rows.json + DESIGN.md §7).

  python tools/bench_rows.py [--out gpurun_out/rows.json] [--quick]

Planning-cycle rows: device kernel time (CUDA events inside the ctx) and the
public-API cycle time of tmpc_solve, median of --cycles cycles after 3 warm-up
cycles, L2 flushed between cycles; the reference CPU planner (oracle/_ref, all
host threads) on a bounded prefix of the same candidates, rate scaled.
Terrain rows: device gaussian_smooth / build_sdist_map through the C ABI
(host arrays in and out) vs the reference functions (single-threaded, as the
reference is written)."""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle.oracle import Oracle  # noqa: E402  (checker / CPU baseline only)
from paper_2603_20525_b200 import _abi, planner as PL, terrain as TR, workloads as W  # noqa: E402


def flush_l2():
    import torch
    buf = getattr(flush_l2, "buf", None)
    if buf is None:
        buf = flush_l2.buf = torch.empty(64 << 20, dtype=torch.float32, device="cuda:0")
    buf.zero_()
    torch.cuda.synchronize()


def warm_for(w):
    """c5 samples around a warm-start sequence: a straight-ahead one here."""
    return np.zeros((w.cfg.n_steps, 2)) if w.cfg.sampler == PL.SAMPLE_WARM_GAUSS else None


def gpu_cycle(w, prec, model, scheme, cycles, lanes=0):
    p = w.params()
    p.model, p.scheme = model, scheme
    pl = PL.Planner(device=0, k_max=w.cfg.n_samples, n_steps_max=w.cfg.n_steps,
                    precision=prec, lanes=lanes)
    pl.set_params(p)
    pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
    smp, _keep = PL.make_sampling(w.cfg, warm_seq=warm_for(w))
    for _ in range(3):
        pl.solve_raw(w.s0, smp, want_controls=False)
    kern, wall, res = [], [], None
    for _ in range(cycles):
        flush_l2()
        t0 = time.perf_counter()
        res, _ = pl.solve_raw(w.s0, smp)
        wall.append((time.perf_counter() - t0) * 1e3)
        kern.append(res.kernel_ms)
    pl.close()
    return statistics.median(kern), statistics.median(wall), res


def cpu_cycle(w, model, scheme, n_cand, min_s):
    p = w.params()
    p.model, p.scheme = model, scheme
    ws = w.with_(n_samples=n_cand)
    smp, _k = PL.make_sampling(ws.cfg, warm_seq=warm_for(ws))
    sd = None if ws.sdist is None else PL.SignedDistanceMap(ws.grid, ws.sdist, True)
    terr, _t = PL.make_terrain(PL.Heightmap(ws.grid, ws.heights), sd)
    orc = Oracle("reference")
    threads = os.cpu_count() or 1
    secs, reps = 0.0, 0
    while secs < min_s or reps == 0:
        t0 = time.perf_counter()
        rc, res, *_ = orc.solve(p, smp, terr, ws.s0, threads=threads)
        secs += time.perf_counter() - t0
        reps += 1
    return n_cand * w.cfg.n_steps * reps / secs, threads, res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "rows.json"))
    ap.add_argument("--cycles", type=int, default=10)
    ap.add_argument("--cpu-seconds", type=float, default=3.0)
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    F32, F64 = _abi.PRECISION_FP32, _abi.PRECISION_FP64
    SRB, EST = _abi.MODEL_SRB, _abi.MODEL_EST
    EU, RK = _abi.SCHEME_EULER, _abi.SCHEME_RK4
    rows = [
        ("c1", F32, SRB, EU), ("c1", F64, SRB, EU),
        ("c2", F32, SRB, EU), ("c2", F64, SRB, EU),
        ("c3", F32, SRB, EU), ("c3", F64, SRB, EU),
        ("c4", F32, SRB, EU),
        ("c5", F32, SRB, EU),
        ("c2", F32, EST, EU), ("c2", F64, EST, EU), ("c3", F32, EST, EU), ("c4", F32, EST, EU),
        ("c2", F32, SRB, RK), ("c2", F64, SRB, RK), ("c2", F32, EST, RK),
    ]
    if a.quick:
        rows = rows[2:3]
    out = {"box": {"cpu_threads": os.cpu_count(), "gpu": "1x B200"}, "rows": []}
    wl = {}
    for name, prec, model, scheme in rows:
        if name not in wl:
            wl[name] = W.make_workload(name)
        w = wl[name]
        K, N = w.cfg.n_samples, w.cfg.n_steps
        kms, wms, res = gpu_cycle(w, prec, model, scheme, a.cycles)
        # CPU: bounded candidate prefix (~cpu_seconds of work), rate scaled
        n_cand = min(K, 1024 if scheme == RK else 4096)
        cpu_rate, thr, cres = cpu_cycle(w, model, scheme, n_cand, a.cpu_seconds)
        row = {
            "row": f"{name} {'fp32' if prec == F32 else 'fp64'} "
                   f"{'SRB' if model == SRB else 'EST'} {'Euler' if scheme == EU else 'RK4'}",
            "K": K, "N": N,
            "kernel_ms": kms, "api_cycle_ms": wms,
            "candidate_steps_per_s": K * N / (kms * 1e-3),
            "api_candidate_steps_per_s": K * N / (wms * 1e-3),
            "n_feasible": int(res.n_feasible), "n_diverged": int(res.n_diverged),
            "cpu_ref_candidate_steps_per_s": cpu_rate, "cpu_threads": thr,
            "cpu_ref_cycle_ms_scaled": K * N / cpu_rate * 1e3,
            "cpu_sample": f"first {n_cand} of {K} candidates",
            "speedup_api_vs_cpu": K * N / (wms * 1e-3) / cpu_rate,
        }
        print(json.dumps(row), flush=True)
        out["rows"].append(row)

    # ---- terrain preprocessing
    ref = Oracle("reference")
    w4 = wl.get("c4") or W.make_workload("c4")
    hm = PL.Heightmap(w4.grid, w4.heights)
    def med_ms(fn, n=5):
        fn()  # warm
        ts = []
        for _ in range(n):
            t0 = time.perf_counter()
            fn()
            ts.append((time.perf_counter() - t0) * 1e3)
        return statistics.median(ts)

    for sigma in (0.3, 1.5):
        g = med_ms(lambda: TR.gaussian_smooth(hm, sigma))
        t0 = time.perf_counter()
        ref.gaussian_smooth(w4.heights, w4.grid, sigma)
        c = (time.perf_counter() - t0) * 1e3
        row = {"row": f"gaussian_smooth sigma={sigma} m on c4 2048^2", "gpu_api_ms": g,
               "cpu_ref_ms": c, "cpu_threads": 1, "speedup": c / g}
        print(json.dumps(row), flush=True)
        out["rows"].append(row)
    for name in ("c2", "c4"):
        w = wl.get(name) or W.make_workload(name)
        off, verts = w.polys
        perims = [TR.Perimeter(vertices=verts[off[i]:off[i + 1]].copy()) for i in range(len(off) - 1)]
        g = med_ms(lambda: TR.build_sdist_map(w.grid, perims))
        row = {"row": f"build_sdist_map {name} {w.grid.nx}^2, {len(perims)} obstacles",
               "gpu_api_ms": g}
        if name == "c2":
            t0 = time.perf_counter()
            ref.build_sdist_map(w.grid, off, verts)
            c = (time.perf_counter() - t0) * 1e3
            row.update(cpu_ref_ms=c, cpu_threads=1, speedup=c / g)
        print(json.dumps(row), flush=True)
        out["rows"].append(row)
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    Path(a.out).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
