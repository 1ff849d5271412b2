"""Open-loop model-error study: the
paper's Appendix-C analysis on the device.

Trajectories come from closed-loop c5 runs (BASELINE configs[4]: warm-started
planner on the GPU, RK4 1 ms plant): every plant state of a run that has 80
applied controls after it (4 s, the prediction horizon) starts one
trajectory, with those applied controls.  Each trajectory is re-simulated
open-loop by the plant (SRB RK4 1 ms, in-kernel) and by the two planner
models (SRB and EST, forward Euler 5 ms) from the same state
(Planner.open_loop_errors, fp64); per model the location and ESM errors are
the time averages of PAPER.md:1609-1612.  Reports medians, the SRB-vs-EST
relative improvement and a two-sided Mann-Whitney U test (scipy), and the
self-comparison (model = plant: SRB RK4 1 ms) that must give exactly 0.

  python tools/open_loop_study.py [--runs 4] [--out profiles/r02_open_loop.json]
"""
import argparse
import json
import sys
import time
from dataclasses import replace
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2603_20525_b200 import _abi, closed_loop as CL, planner as PL, terrain as TR  # noqa
from paper_2603_20525_b200 import workloads as W  # noqa

ap = argparse.ArgumentParser()
ap.add_argument("--runs", type=int, default=4)
ap.add_argument("--cycles", type=int, default=200)
ap.add_argument("--horizon-steps", type=int, default=80)  # 4 s at 0.05 s
ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "open_loop.json"))
a = ap.parse_args()

w = W.make_workload("c5")
H = a.horizon_steps
s0s, ctrls = [], []
t0 = time.time()
for run in range(a.runs):
    cfg = replace(w.cfg, seed=w.cfg.seed + 1000 * run)
    loop = CL.ClosedLoop(w.heights, w.grid, w.sdist, w.goal, cfg)
    plan = loop.device_planner()
    s_start = np.array(w.s0)
    s_start[1] += 0.5 * (run - (a.runs - 1) / 2) / max(1, a.runs - 1)  # +-0.25 m lateral
    rec = loop.run(plan, s_start, cycles=a.cycles)
    plan.planner.close()
    states = [c.state for c in rec.cycles] + [rec.final_state]
    u = np.array([c.control for c in rec.cycles])
    for i in range(len(rec.cycles) - H + 1):
        s0s.append(states[i])
        ctrls.append(u[i:i + H])
s0s, ctrls = np.array(s0s), np.array(ctrls)
t_loops = time.time() - t0

p = w.params()
p.n_steps = H
pl = PL.Planner(device=0, precision=_abi.PRECISION_FP64)
pl.set_params(p)
out = {}
t1 = time.time()
for name, model, sigma in (("srb", _abi.MODEL_SRB, 0.0), ("est", _abi.MODEL_EST, 0.0),
                           ("srb_lod", _abi.MODEL_SRB, 0.3), ("est_lod", _abi.MODEL_EST, 1.5)):
    # the paper's LODs: each model on its own smoothed
    # terrain (SRB sigma 0.3 m, EST 1.5 m), the plant on the unsmoothed one
    hm = PL.Heightmap(w.grid, w.heights)
    model_h = TR.gaussian_smooth(hm, sigma).heights if sigma > 0 else w.heights
    pl.set_terrain_arrays(model_h, None, w.grid)
    pl.set_plant_terrain(hm if sigma > 0 else None)
    loc, esm, fl = pl.open_loop_errors(model, s0s, ctrls, 0.001)
    ok = fl == 0
    out[name] = {"model_lod_sigma_m": sigma, "n": int(ok.sum()), "diverged": int((~ok).sum()),
                 "loc_median_m": float(np.median(loc[ok])), "loc_mean_m": float(loc[ok].mean()),
                 "loc_p90_m": float(np.percentile(loc[ok], 90)),
                 "esm_median_J": float(np.median(esm[ok])), "esm_mean_J": float(esm[ok].mean()),
                 "esm_p90_J": float(np.percentile(esm[ok], 90))}
    out[name + "_arrays"] = (loc, esm)
t_dev = time.time() - t1
# self-comparison: model = plant dynamics and LOD -> exactly 0
p_self = w.params()
p_self.n_steps, p_self.scheme, p_self.dt_int = H, _abi.SCHEME_RK4, 0.001
pl.set_params(p_self)
pl.set_terrain_arrays(w.heights, None, w.grid)
pl.set_plant_terrain(None)
loc_s, esm_s, fl_s = pl.open_loop_errors(_abi.MODEL_SRB, s0s[:16], ctrls[:16], 0.001)
pl.close()
res = {k: v for k, v in out.items() if not k.endswith("_arrays")}
for tag, (a_, b_) in (("same_lod", ("srb", "est")), ("paper_lods", ("srb_lod", "est_lod"))):
    ls, le = out[a_ + "_arrays"], out[b_ + "_arrays"]
    both = np.isfinite(ls[0]) & np.isfinite(le[0])
    entry = {"location": 1 - res[a_]["loc_median_m"] / res[b_]["loc_median_m"],
             "esm": 1 - res[a_]["esm_median_J"] / res[b_]["esm_median_J"]}
    try:
        from scipy.stats import mannwhitneyu
        entry["mann_whitney_p"] = {
            "location": float(mannwhitneyu(ls[0][both], le[0][both]).pvalue),
            "esm": float(mannwhitneyu(ls[1][both], le[1][both]).pvalue)}
    except Exception as e:  # scipy missing
        entry["mann_whitney_p"] = str(e)
    res["srb_vs_est_median_improvement_" + tag] = entry
res["self_comparison_max"] = {"loc": float(np.nanmax(loc_s)), "esm": float(np.nanmax(esm_s))}
res["setup"] = (f"{len(s0s)} trajectories from {a.runs} closed-loop c5 runs x {a.cycles} cycles "
                f"(K={w.cfg.n_samples}, GPU planner fp32), 4 s horizon ({H} ZOH steps of the "
                "applied controls); plant SRB RK4 1 ms in-kernel on the unsmoothed terrain, models "
                "SRB / EST forward Euler 5 ms, fp64; 'srb'/'est' on the plant's terrain, "
                "'srb_lod'/'est_lod' on the paper's model LODs (Gaussian sigma 0.3 / 1.5 m, "
                "PAPER.md:1184-1205)")
res["seconds"] = {"closed_loops": t_loops, "device_open_loop": t_dev}
Path(a.out).write_text(json.dumps(res, indent=1))
print(json.dumps(res, indent=1))
