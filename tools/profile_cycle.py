"""One warm-up + `n` planning cycles of a workload (target for ncu)."""
import argparse, sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2603_20525_b200 import _abi, planner as PL, workloads as W

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--precision", type=int, default=0)
ap.add_argument("--cycles", type=int, default=2)
ap.add_argument("--K", type=int, default=0)
ap.add_argument("--lanes", type=int, default=0)
ap.add_argument("--ordering", type=int, default=0)
ap.add_argument("--model", type=int, default=0)
ap.add_argument("--scheme", type=int, default=0)
a = ap.parse_args()
w = W.make_workload(a.config)
if a.K:
    w = w.with_(n_samples=a.K)
pl = PL.Planner(device=0, k_max=w.cfg.n_samples, n_steps_max=w.cfg.n_steps, precision=a.precision,
                lanes=a.lanes, ordering=a.ordering)
p = w.params()
p.model, p.scheme = a.model, a.scheme
pl.set_params(p)
pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
smp, _ = PL.make_sampling(w.cfg)
for i in range(a.cycles):
    res, _ = pl.solve_raw(w.s0, smp)
    print(f"cycle {i}: kernel {res.kernel_ms:.3f} ms best {res.best_index} cost {res.best_cost:.4f}")
pl.close()
