"""Kernel time per lanes-per-candidate setting and batch size (dev tool)."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2603_20525_b200 import planner as PL, workloads as W

for name, Ks in [("c1", [1024]), ("c2", [1024, 2048, 4096, 8192, 12288, 16384, 32768]), ("c3", [8192, 65536])]:
    w0 = W.make_workload(name)
    for K in Ks:
        w = w0.with_(n_samples=K)
        row = []
        for lanes in (1, 2, 4, 0):
            pl = PL.Planner(device=0, k_max=K, n_steps_max=w.cfg.n_steps, lanes=lanes)
            pl.set_params(w.params())
            pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
            smp, _ = PL.make_sampling(w.cfg)
            ts = []
            for i in range(4):
                res, _ = pl.solve_raw(w.s0, smp, want_controls=False)
                ts.append(res.kernel_ms)
            c, f, m = pl.costs(K)
            pl.close()
            row.append((lanes, min(ts[1:]), res.best_index, float(np.nansum(np.where(np.isfinite(c), c, 0)))))
        print(name, K, " ".join(f"L{l}:{t:.3f}ms(best {b})" for l, t, b, cs in row), flush=True)
