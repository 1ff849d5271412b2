"""EST footprint-skip statistics (dev probe): needs a library built with the
temporary ESTSTATS counters (gpurun_out/g59.log); runs one
EST cycle per config and lets the kernel print its counters."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2603_20525_b200 import _abi, planner as PL, workloads as W
for name in sys.argv[1:]:
    w = W.make_workload(name)
    pl = PL.Planner(device=0, k_max=w.cfg.n_samples, n_steps_max=w.cfg.n_steps, graphs=_abi.GRAPHS_OFF)
    p = w.params(); p.model = 1
    pl.set_params(p); pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
    smp, keep = PL.make_sampling(w.cfg)
    print(name, flush=True)
    pl.solve_raw(w.s0, smp, want_controls=False)
    pl.close()
