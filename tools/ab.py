"""A/B timing of kernel variants (dev tool).

  python tools/variants.py build NAME "-DFLAG=1 ..."   # here: variants/NAME/libtmpc_b200.so
  python tools/ab.py [--configs c2,c3] [--cycles 30] variants/*/libtmpc_b200.so

Each library runs in its own process (TMPC_B200_LIB), median device kernel
time over --cycles cycles (L2 flushed between cycles), rounds interleaved
across variants so clock drift hits all of them alike."""
import argparse
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

CHILD = r"""
import sys, json, statistics
sys.path.insert(0, %r)
import torch
from paper_2603_20525_b200 import planner as PL, workloads as W
cfgs, cycles, K, lanes, ordering, model, scheme = %r, %d, %d, %d, %d, %d, %d
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda:0")
out = {}
for name in cfgs:
    w = W.make_workload(name)
    if K:
        w = w.with_(n_samples=K)
    pl = PL.Planner(device=0, k_max=w.cfg.n_samples, n_steps_max=w.cfg.n_steps, lanes=lanes, ordering=ordering)
    pp = w.params()
    pp.model, pp.scheme = model, scheme
    pl.set_params(pp)
    pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
    smp, keep = PL.make_sampling(w.cfg)
    for _ in range(3):
        pl.solve_raw(w.s0, smp, want_controls=False)
    ts = []
    for _ in range(cycles):
        flush.zero_(); torch.cuda.synchronize()
        r, _ = pl.solve_raw(w.s0, smp, want_controls=False)
        ts.append(r.kernel_ms)
    c, f, m = pl.costs(w.cfg.n_samples)
    out[name] = [statistics.median(ts), min(ts), int(r.best_index), float(r.best_cost)]
    pl.close()
print("AB" + json.dumps(out))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--configs", default="c2,c3")
    ap.add_argument("--cycles", type=int, default=30)
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--K", type=int, default=0)
    ap.add_argument("--lanes", type=int, default=0)
    ap.add_argument("--ordering", type=int, default=0, help="0 auto, 1 off, 2 on (_abi.ORDER_*)")
    ap.add_argument("--model", type=int, default=0, help="0 SRB, 1 EST")
    ap.add_argument("--scheme", type=int, default=0, help="0 Euler, 1 RK4")
    a = ap.parse_args()
    cfgs = a.configs.split(",")
    res = {lib: [] for lib in a.libs}
    for _ in range(a.rounds):
        for lib in a.libs:
            path, _, extra = lib.partition("@")  # "lib.so@NAME=VALUE" sets an env var
            env = dict(os.environ, TMPC_B200_LIB=str(Path(path).resolve()))
            if extra:
                k, _, v = extra.partition("=")
                env[k] = v
            p = subprocess.run([sys.executable, "-c", CHILD % (str(ROOT), cfgs, a.cycles, a.K, a.lanes, a.ordering, a.model, a.scheme)],
                               env=env, capture_output=True, text=True, timeout=600)
            line = [ln for ln in p.stdout.splitlines() if ln.startswith("AB")]
            if p.returncode or not line:
                print(lib, "FAILED", p.stderr[-2000:], flush=True)
                continue
            res[lib].append(json.loads(line[0][2:]))
    for lib, runs in res.items():
        cols = []
        for c in cfgs:
            vals = [r[c][0] for r in runs if c in r]
            best = runs[0][c][2:] if runs else None
            cols.append(f"{c}: {min(vals):.4f} ms (best {best})" if vals else f"{c}: -")
        tag = Path(lib.partition("@")[0]).parent.name + ("@" + lib.partition("@")[2] if "@" in lib else "")
        print(f"{tag:32s} " + "  ".join(cols), flush=True)


if __name__ == "__main__":
    main()
