"""Kernel time vs terrain size / features at small K (dev tool): separates the
L2-miss latency from the arithmetic critical path of one substep."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2603_20525_b200 import planner as PL, workloads as W

w0 = W.make_workload("c2")
def run(w, heights, sdist, grid, lanes, K):
    w = w.with_(n_samples=K)
    pl = PL.Planner(device=0, k_max=K, n_steps_max=w.cfg.n_steps, lanes=lanes)
    pl.set_params(w.params())
    pl.set_terrain_arrays(heights, sdist, grid)
    smp, _ = PL.make_sampling(w.cfg)
    ts = [pl.solve_raw(w.s0, smp, want_controls=False)[0].kernel_ms for _ in range(4)]
    pl.close()
    return min(ts[1:])

tiny = PL.GridSpec(0.0, 0.0, 8.0, 16, 16)
h_tiny = np.zeros((16, 16))
sd_tiny = np.full((16, 16), 50.0)
for K in (2048, 16384):
    for lanes in (1, 2, 4):
        a = run(w0, w0.heights, w0.sdist, w0.grid, lanes, K)
        b = run(w0, w0.heights, None, w0.grid, lanes, K)
        c = run(w0, h_tiny, sd_tiny, tiny, lanes, K)
        d = run(w0, h_tiny, None, tiny, lanes, K)
        print(f"K={K} L={lanes}: c2 {a:.3f}  c2-noSDF {b:.3f}  tiny {c:.3f}  tiny-noSDF {d:.3f} ms", flush=True)
