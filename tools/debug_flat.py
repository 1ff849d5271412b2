"""Flat-terrain sanity run of every kernel layout vs the oracle (debug tool)."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2603_20525_b200 import _abi, planner as PL
from oracle.oracle import Oracle

grid = PL.GridSpec(-20.0, -40.0, 0.2, 400, 400)
h = np.zeros((400, 400))
vp = PL.VehicleParams()
cfg = PL.PlannerConfig(n_samples=256, n_steps=20, dt_zoh=0.05, dt_int=0.005, seed=7)
p = PL.make_params(vp, PL.TireParams(), PL.ConstraintConfig(), PL.CostWeights(), PL.Goal(15.0, 0.0, 2.5), cfg)
smp, keep = PL.make_sampling(cfg)
s0 = np.zeros(13); s0[2] = vp.h + vp.R; s0[6] = 5.0
terr, tk = PL.make_terrain(PL.Heightmap(grid, h), None)
rc, ores, oc, of, om, osub, err = Oracle("port").solve(p, smp, terr, s0, threads=8)
print("oracle best", ores.best_index, ores.best_cost, "cost[:4]", oc[:4])
for prec in (0, 1):
    for lanes in ((1, 2, 4) if prec == 0 else (0,)):
        pl = PL.Planner(device=0, k_max=256, n_steps_max=20, precision=prec, lanes=lanes)
        pl.set_params(p)
        pl.set_terrain_arrays(h, None, grid)
        res, ctrl = pl.solve_raw(s0, smp)
        c, f, m = pl.costs(256)
        rel = np.abs(c - oc) / np.abs(oc)
        print(f"prec {prec} lanes {lanes}: best {res.best_index} {res.best_cost:.6f} max rel {rel.max():.3e} cost[:4] {c[:4]}")
        pl.close()
