"""Host-side split of one public-API planning cycle (dev tool): stage, launch
(graph update + enqueue), finish (wait + fold), control regeneration, timed
from Python around each C call, median of 100 cycles.

  python tools/api_split_probe.py [c2|c5|...]"""
import ctypes as C
import statistics
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
from paper_2603_20525_b200 import _abi, planner as PL, workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = W.make_workload(name)
print(name, flush=True)
for graphs in (_abi.GRAPHS_AUTO, _abi.GRAPHS_OFF):
    pl = PL.Planner(device=0, k_max=w.cfg.n_samples, n_steps_max=w.cfg.n_steps, graphs=graphs)
    pl.set_params(w.params())
    pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
    warm = np.zeros((w.cfg.n_steps, 2)) if w.cfg.sampler == PL.SAMPLE_WARM_GAUSS else None
    smp, keep = PL.make_sampling(w.cfg, warm_seq=warm)
    lib = pl.lib
    s0 = np.ascontiguousarray(w.s0)
    s0p = _abi.dptr(s0)
    res = _abi.tmpc_result()
    ctrl = np.zeros((w.cfg.n_steps, 2))
    cp = _abi.dptr(ctrl)
    T = {k: [] for k in ("stage", "launch", "finish", "controls", "kernel", "solve_c")}
    for i in range(110):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lib.tmpc_stage_cycle(pl.ctx, s0p, C.byref(smp))
        t1 = time.perf_counter()
        lib.tmpc_launch_cycle(pl.ctx)
        t2 = time.perf_counter()
        lib.tmpc_finish_cycle(pl.ctx, C.byref(res))
        t3 = time.perf_counter()
        lib.tmpc_sample_controls(C.byref(pl._params), C.byref(smp), res.best_index, cp)
        t4 = time.perf_counter()
        if i >= 10:
            T["stage"].append((t1 - t0) * 1e6)
            T["launch"].append((t2 - t1) * 1e6)
            T["finish"].append((t3 - t2) * 1e6)
            T["controls"].append((t4 - t3) * 1e6)
            T["kernel"].append(res.kernel_ms * 1e3)
        r, _ = pl.solve_raw(w.s0, smp)
        if i >= 10:
            T["solve_c"].append(r.cycle_ms * 1e3)
    pl.close()
    print(f"graphs={'on' if graphs == _abi.GRAPHS_AUTO else 'off'}: " +
          ", ".join(f"{k} {statistics.median(v):.1f} us" for k, v in T.items()))
