"""Where the public-API cycle time goes beyond the kernel (dev tool): python
wall of Planner.solve_raw vs the C-side cycle_ms vs the device kernel_ms, on
c2 and on a tiny K (fixed per-cycle overhead)."""
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
from paper_2603_20525_b200 import planner as PL, workloads as W  # noqa: E402

flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda:0")
from paper_2603_20525_b200 import _abi  # noqa: E402
for K, graphs in ((16384, _abi.GRAPHS_AUTO), (16384, _abi.GRAPHS_OFF), (32, _abi.GRAPHS_AUTO),
                  (32, _abi.GRAPHS_OFF)):
    w = W.make_workload("c2").with_(n_samples=K)
    pl = PL.Planner(device=0, k_max=K, n_steps_max=w.cfg.n_steps, graphs=graphs)
    pl.set_params(w.params())
    pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
    smp, _ = PL.make_sampling(w.cfg)
    for _ in range(5):
        pl.solve_raw(w.s0, smp)
    wall, cyc, kern, nocontrols = [], [], [], []
    for _ in range(50):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r, _ = pl.solve_raw(w.s0, smp)
        wall.append((time.perf_counter() - t0) * 1e3)
        cyc.append(r.cycle_ms)
        kern.append(r.kernel_ms)
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pl.solve_raw(w.s0, smp, want_controls=False)
        nocontrols.append((time.perf_counter() - t0) * 1e3)
    m = statistics.median
    print(f"K={K} graphs={'on' if graphs == _abi.GRAPHS_AUTO else 'off'}: python wall {m(wall):.4f} ms, C cycle {m(cyc):.4f} ms, kernel {m(kern):.4f} ms, "
          f"wall w/o controls {m(nocontrols):.4f} ms")
    pl.close()
