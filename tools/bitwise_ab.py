"""Bit-for-bit comparison of two builds of the library (dev tool).

  python tools/bitwise_ab.py LIB_A LIB_B [--configs c1,c2,c3,c5] [--K 0] [--model 0 --scheme 0]

Each library solves the same workloads in its own process (TMPC_B200_LIB) and
dumps every candidate's cost, flags and margin; the parent compares the arrays
bitwise.  For layout / schedule changes that must not move a single bit."""
import argparse
import json
import os
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
CHILD = r"""
import sys
sys.path.insert(0, %r)
import numpy as np
from paper_2603_20525_b200 import planner as PL, workloads as W
cfgs, K, out, model, scheme, lanes = %r, %d, %r, %d, %d, %d
res = {}
for name in cfgs:
    w = W.make_workload(name)
    if K:
        w = w.with_(n_samples=min(K, w.cfg.n_samples))
    pl = PL.Planner(device=0, k_max=w.cfg.n_samples, n_steps_max=w.cfg.n_steps, lanes=lanes)
    p = w.params()
    p.model, p.scheme = model, scheme
    pl.set_params(p)
    pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
    smp, _ = PL.make_sampling(w.cfg)
    r, _ = pl.solve_raw(w.s0, smp, want_controls=False)
    c, f, m = pl.costs(w.cfg.n_samples)
    res[name + "_cost"], res[name + "_flags"], res[name + "_margin"] = c, f, m
    res[name + "_best"] = np.array([r.best_index, r.best_cost])
    pl.close()
np.savez(out, **res)
"""


def run(lib, cfgs, K, out, model, scheme, lanes):
    env = dict(os.environ, TMPC_B200_LIB=str(Path(lib).resolve()))
    subprocess.run([sys.executable, "-c", CHILD % (str(ROOT), cfgs, K, out, model, scheme, lanes)],
                   env=env, check=True)
    return np.load(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("a")
    ap.add_argument("b")
    ap.add_argument("--configs", default="c1,c2,c3,c5")
    ap.add_argument("--K", type=int, default=0)
    ap.add_argument("--model", type=int, default=0)
    ap.add_argument("--scheme", type=int, default=0)
    ap.add_argument("--lanes", type=int, default=0)
    a = ap.parse_args()
    cfgs = a.configs.split(",")
    with tempfile.TemporaryDirectory() as d:
        A = run(a.a, cfgs, a.K, f"{d}/a.npz", a.model, a.scheme, a.lanes)
        B = run(a.b, cfgs, a.K, f"{d}/b.npz", a.model, a.scheme, a.lanes)
        ok = True
        for tag, R in (("A", A), ("B", B)):
            for name in cfgs:
                bi, bc = R[name + "_best"]
                c = R[name + "_cost"]
                if c[int(bi)] != bc:
                    print(f"{tag} {name}: best_cost {bc!r} != cost[{int(bi)}] {c[int(bi)]!r}")
        for k in A.files:
            x, y = A[k], B[k]
            xb = x.view(np.uint8).reshape(x.shape[0], -1)
            yb = y.view(np.uint8).reshape(y.shape[0], -1)
            ndiff = int(np.sum(np.any(xb != yb, axis=1)))
            print(f"{k:16s} {'identical' if ndiff == 0 else 'DIFFER'} ({ndiff} of {len(x)} differ)")
            ok &= ndiff == 0
        tag = {"model": a.model, "scheme": a.scheme, "lanes": a.lanes}
        print("BITWISE", "OK" if ok else "MISMATCH", json.dumps(tag), flush=True)


if __name__ == "__main__":
    main()
