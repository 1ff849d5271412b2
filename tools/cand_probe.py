"""Per-candidate cost of given indices under several kernel-variant libraries
(dev tool): full-size batch, so the lane layout is the production one.

  python tools/cand_probe.py c3 23102 --model 0 --scheme 1 --ref 452.27768746397066 variants/*/libtmpc_b200.so
"""
import argparse
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CHILD = r"""
import sys, json
sys.path.insert(0, %r)
from paper_2603_20525_b200 import planner as PL, workloads as W
name, ks, model, scheme = %r, %r, %d, %d
w = W.make_workload(name)
pl = PL.Planner(device=0, k_max=w.cfg.n_samples, n_steps_max=w.cfg.n_steps)
pp = w.params(); pp.model, pp.scheme = model, scheme
pl.set_params(pp); pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
smp, keep = PL.make_sampling(w.cfg)
pl.solve_raw(w.s0, smp, want_controls=False)
c, f, m = pl.costs(w.cfg.n_samples)
print("CP" + json.dumps([float(c[k]) for k in ks]))
"""
ap = argparse.ArgumentParser()
ap.add_argument("config"); ap.add_argument("ks"); ap.add_argument("libs", nargs="+")
ap.add_argument("--model", type=int, default=0); ap.add_argument("--scheme", type=int, default=0)
ap.add_argument("--ref", default="")
a = ap.parse_args()
ks = [int(x) for x in a.ks.split(",")]
ref = [float(x) for x in a.ref.split(",")] if a.ref else None
for lib in a.libs:
    env = dict(os.environ, TMPC_B200_LIB=str(Path(lib).resolve()))
    p = subprocess.run([sys.executable, "-c", CHILD % (str(ROOT), a.config, ks, a.model, a.scheme)],
                       env=env, capture_output=True, text=True, timeout=600)
    line = [ln for ln in p.stdout.splitlines() if ln.startswith("CP")]
    if not line:
        print(lib, "FAILED", p.stderr[-1500:]); continue
    c = json.loads(line[0][2:])
    rel = [abs(x - r) / abs(r) for x, r in zip(c, ref)] if ref else []
    print(f"{Path(lib).parent.name:12s} cost={c} rel={['%.3e' % r for r in rel]}", flush=True)
