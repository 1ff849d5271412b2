"""oracle/_ref costs + conditioning spread at full BASELINE sizes (dev tool,
pairs with tools/dump_fullsize.py for offline parity analysis).

  python tools/ref_fullsize.py --configs c2,c3 --out /tmp/ref_full.npz
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from paper_2603_20525_b200 import planner as PL  # noqa: E402
from parity_util import best_oracle, conditioning_spread, problem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c2,c3,c4,c5")
ap.add_argument("--threads", type=int, default=8)
ap.add_argument("--out", default="/tmp/ref_full.npz")
a = ap.parse_args()
orc = best_oracle()
out = {}
for name in a.configs.split(","):
    t0 = time.time()
    w, p, smp, terr, keep = problem(name)
    warm = np.zeros((w.cfg.n_steps, 2)) if w.cfg.sampler == PL.SAMPLE_WARM_GAUSS else None
    smp, k2 = PL.make_sampling(w.cfg, 0, w.cfg.n_samples, warm)
    rc, res, cost, flags, margin, sub, err = orc.solve(p, smp, terr, w.s0, threads=a.threads)
    spread = conditioning_spread(orc, p, smp, terr, w.s0, cost, threads=a.threads)
    out[f"{name}_cost"], out[f"{name}_flags"], out[f"{name}_margin"] = cost, flags, margin
    out[f"{name}_spread"] = spread
    out[f"{name}_best"] = np.array([res.best_index])
    print(name, "best", res.best_index, f"{time.time() - t0:.1f}s", flush=True)
np.savez(a.out, **out)
