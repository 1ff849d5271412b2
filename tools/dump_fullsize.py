"""Dump full-size device outputs (per candidate cost / flags / margin) of
c2, c3, c4 and the first warm-started c5 cycle for offline parity analysis
against oracle/_ref (dev tool; the parity tests themselves live in tests/).

  python tools/dump_fullsize.py [--precision fp32|fp64] [--out gpurun_out/full_fp32.npz]
"""
import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from paper_2603_20525_b200 import _abi, planner as PL  # noqa: E402
from parity_util import problem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--precision", default="fp32")
ap.add_argument("--configs", default="c2,c3,c4,c5")
ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "full_fp32.npz"))
a = ap.parse_args()
prec = _abi.PRECISION_FP64 if a.precision == "fp64" else _abi.PRECISION_FP32
out = {}
for name in a.configs.split(","):
    w, p, smp, terr, keep = problem(name)
    warm = np.zeros((w.cfg.n_steps, 2)) if w.cfg.sampler == PL.SAMPLE_WARM_GAUSS else None
    smp, k2 = PL.make_sampling(w.cfg, 0, w.cfg.n_samples, warm)
    pl = PL.Planner(device=0, k_max=smp.k_count, n_steps_max=p.n_steps, precision=prec)
    pl.set_params(p)
    pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
    res, ctrl = pl.solve_raw(w.s0, smp)
    c, f, m = pl.costs(smp.k_count)
    out[f"{name}_cost"], out[f"{name}_flags"], out[f"{name}_margin"] = c, f, m
    out[f"{name}_best"] = np.array([res.best_index])
    print(name, "best", res.best_index, res.best_cost, "feasible", res.n_feasible,
          "diverged", res.n_diverged, flush=True)
    pl.close()
np.savez(a.out, **out)
print("dumped", len(out))
