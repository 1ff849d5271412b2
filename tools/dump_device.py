"""Dump device per-candidate outputs for offline parity analysis (dev tool)."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from paper_2603_20525_b200 import _abi, planner as PL
from parity_util import problem

out = {}
for name, K in [("c1", None), ("c2", 4096), ("c3", 4096)]:
    w, p, smp, terr, keep = problem(name, K)
    for prec in (0, 1):
        pl = PL.Planner(device=0, k_max=smp.k_count, n_steps_max=p.n_steps, precision=prec)
        pl.set_params(p)
        pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
        res, ctrl = pl.solve_raw(w.s0, smp)
        c, f, m = pl.costs(smp.k_count)
        out[f"{name}_{prec}_cost"], out[f"{name}_{prec}_flags"], out[f"{name}_{prec}_margin"] = c, f, m
        pl.close()
np.savez(ROOT / "gpurun_out" / "device_dump.npz", **out)
print("dumped", len(out))
