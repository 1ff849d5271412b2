"""c2 with the footprint term on / off and the ESM on / off (dev probe): the
share of the substep chain the cost terms take (SRB, or EST with --est)."""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2603_20525_b200 import planner as PL, workloads as W  # noqa: E402

flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda:0")
args = sys.argv[1:] or ["c2"]
model = 1 if "--est" in args else 0
for name in [a for a in args if not a.startswith("--")]:
    w = W.make_workload(name)
    for dist, roll in ((1, 1), (0, 1), (1, 0), (0, 0)):
        pl = PL.Planner(device=0, k_max=w.cfg.n_samples, n_steps_max=w.cfg.n_steps)
        pp = w.params()
        pp.enable_dist, pp.enable_rollover = dist, roll
        pp.model = model
        pl.set_params(pp)
        pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
        smp, keep = PL.make_sampling(w.cfg)
        for _ in range(3):
            pl.solve_raw(w.s0, smp, want_controls=False)
        ts = []
        for _ in range(30):
            flush.zero_(); torch.cuda.synchronize()
            r, _ = pl.solve_raw(w.s0, smp, want_controls=False)
            ts.append(r.kernel_ms)
        print(f"{name} dist={dist} rollover={roll}: {statistics.median(ts):.4f} ms "
              f"(min {min(ts):.4f}) substeps={r.substeps_executed}", flush=True)
        pl.close()
