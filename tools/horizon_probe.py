"""Truncated-horizon probe of single candidates (dev tool): the device cost of
candidate k of a config for horizons N = 2, 4, ..., N_full (same goal, same
lane layout as the full cycle), so a device-vs-reference divergence can be
located in time by comparing with the reference on the CPU.

  python tools/horizon_probe.py c3 3331,19134 --out gpurun_out/hp.npz [--precision fp32]
      [--model 0|1 --scheme 0|1]
"""
import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2603_20525_b200 import _abi, planner as PL, workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("ks")
ap.add_argument("--out", required=True)
ap.add_argument("--precision", default="fp32")
ap.add_argument("--model", type=int, default=0)
ap.add_argument("--scheme", type=int, default=0)
a = ap.parse_args()
prec = _abi.PRECISION_FP64 if a.precision == "fp64" else _abi.PRECISION_FP32
w = W.make_workload(a.config)
ks = [int(x) for x in a.ks.split(",")]
Ns = list(range(2, w.cfg.n_steps + 1, 2))
pl = PL.Planner(device=0, k_max=1, n_steps_max=w.cfg.n_steps, precision=prec)
pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
out = {}
for N in Ns:
    p = w.params()
    p.n_steps = N
    p.model, p.scheme = a.model, a.scheme
    pl.set_params(p)
    for k in ks:
        smp, keep = PL.make_sampling(w.cfg, k, 1)
        smp.k_total = w.cfg.n_samples
        try:
            res, _ = pl.solve_raw(w.s0, smp, want_controls=False)
        except PL.NumericError:
            pass
        c, f, m = pl.costs(1)
        out.setdefault(f"k{k}_cost", []).append(c[0])
        out.setdefault(f"k{k}_flags", []).append(f[0])
np.savez(a.out, Ns=np.array(Ns), **{k: np.array(v) for k, v in out.items()})
print("done", len(Ns), "horizons x", len(ks), "candidates")
