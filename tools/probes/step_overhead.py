"""Where the bench step's time outside the kernel goes (dev probe): for each
library (TMPC_B200_LIB per child process), the bench's device-timed c2 step
(torch events around stage + launch, L2 flushed before) against the ctx's own
kernel events, median of 100 cycles.  Libraries built with the
TMPC_PROBE_NO_* switches return garbage results; only timing is read."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
CHILD = r"""
import sys, json, statistics, ctypes as C
sys.path.insert(0, %r)
import numpy as np, torch
from paper_2603_20525_b200 import _abi, planner as PL, workloads as W
w = W.make_workload("c2")
pl = PL.Planner(device=0, k_max=w.cfg.n_samples, n_steps_max=w.cfg.n_steps)
pl.set_params(w.params()); pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
smp, keep = PL.make_sampling(w.cfg)
lib, s0, res = pl.lib, np.ascontiguousarray(w.s0), _abi.tmpc_result()
st = torch.cuda.ExternalStream(pl.device_stream(0), device=0)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda:0")
step, kern = [], []
for i in range(103):
    with torch.cuda.stream(st):
        flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    lib.tmpc_stage_cycle(pl.ctx, _abi.dptr(s0), C.byref(smp)); lib.tmpc_launch_cycle(pl.ctx)
    e1.record(st)
    lib.tmpc_finish_cycle(pl.ctx, C.byref(res))
    st.synchronize()
    if i >= 3:
        step.append(e0.elapsed_time(e1)); kern.append(res.kernel_ms)
print("SO" + json.dumps([statistics.median(step), statistics.median(kern)]))
"""
for lib in sys.argv[1:]:
    env = dict(os.environ, TMPC_B200_LIB=str(Path(lib).resolve()))
    p = subprocess.run([sys.executable, "-c", CHILD % str(ROOT)], env=env, capture_output=True,
                       text=True, timeout=600)
    line = [ln for ln in p.stdout.splitlines() if ln.startswith("SO")]
    if not line:
        print(lib, "FAILED", p.stderr[-800:]); continue
    a, b = json.loads(line[0][2:])
    print(f"{Path(lib).parent.name:10s} step {a * 1e3:8.1f} us  kernel events {b * 1e3:8.1f} us  "
          f"outside {1e3 * (a - b):6.1f} us", flush=True)
