"""Kernel time of one warp alone on the GPU (K = 32 / L candidates) vs the full
c2 batch, per lanes-per-candidate layout (dev tool): how far a cycle is from
its single-warp dependency-chain bound."""
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
from paper_2603_20525_b200 import _abi, planner as PL, workloads as W  # noqa: E402

flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda:0")
for model in (_abi.MODEL_SRB, _abi.MODEL_EST):
    for lanes in ((1, 2, 4) if model == _abi.MODEL_SRB else (0,)):
        for K in (32 // max(lanes, 1), 16384):
            w = W.make_workload("c2").with_(n_samples=K)
            p = w.params()
            p.model = model
            pl = PL.Planner(device=0, k_max=K, n_steps_max=w.cfg.n_steps, lanes=lanes)
            pl.set_params(p)
            pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
            smp, _ = PL.make_sampling(w.cfg)
            for _ in range(3):
                pl.solve_raw(w.s0, smp, want_controls=False)
            ts, tw = [], []
            for _ in range(15):
                flush.zero_()
                torch.cuda.synchronize()
                r, _ = pl.solve_raw(w.s0, smp, want_controls=False)
                ts.append(r.kernel_ms)
                r, _ = pl.solve_raw(w.s0, smp, want_controls=False)  # L2 warm
                tw.append(r.kernel_ms)
            pl.close()
            print(f"{'SRB' if model == 0 else 'EST'} lanes {lanes} K {K:6d}: "
                  f"{statistics.median(ts):.4f} ms (L2 flushed)  {statistics.median(tw):.4f} ms "
                  f"(L2 warm)", flush=True)
