import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
from dataclasses import replace
from paper_2603_20525_b200 import _abi, planner as PL, workloads as W, closed_loop as CL
w = W.make_workload("c5")
pl = PL.Planner(device=0, k_max=w.cfg.n_samples, n_steps_max=w.cfg.n_steps)
pl.set_params(w.params()); pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
warm = np.zeros((w.cfg.n_steps, 2))
for kind, ws in [("uniform", None), ("warm", warm)]:
    cfg = replace(w.cfg, sampler=PL.SAMPLE_UNIFORM) if ws is None else w.cfg
    smp, keep = PL.make_sampling(cfg, warm_seq=ws)
    for i in range(6):
        t0 = time.perf_counter(); res, ctrl = pl.solve_raw(w.s0, smp); t1 = time.perf_counter()
        print(kind, f"wall {1e3*(t1-t0):.3f} cycle {res.cycle_ms:.3f} kernel {res.kernel_ms:.3f}")
