"""Generate the committed golden vectors from the REFERENCE itself.

Runs oracle/_ref/libtmpc_ref.so (the unmodified reference headers compiled
with the Eigen shim + the SPEC planner loop, oracle/ref_planner.cpp) on the
seeded BASELINE workloads and stores per-candidate cost / flags / margin,
the winner, sampled control sequences and the terrain digest.  Needs
/root/reference (this container); the fixtures travel with the repo.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle.oracle import Oracle  # noqa: E402
from paper_2603_20525_b200 import planner as PL  # noqa: E402
from parity_util import problem  # noqa: E402

OUT = Path(__file__).resolve().parent
CASES = {"c1": (None, None), "c2": (512, None), "c3": (512, None)}


def main():
    ref = Oracle("reference")
    meta = {}
    for name, (K, N) in CASES.items():
        w, p, smp, terr, keep = problem(name, K, N)
        rc, res, cost, flags, margin, sub, err = ref.solve(p, smp, terr, w.s0, threads=8)
        assert rc == 0, err
        ctrl = np.stack([ref.sample_controls(p, smp, k) for k in range(3)])
        np.savez_compressed(OUT / f"parity_{name}.npz", cost=cost, flags=flags, margin=margin,
                            substeps=sub, controls_k012=ctrl, s0=w.s0)
        meta[name] = {"K": int(smp.k_count), "N": int(p.n_steps), "seed": int(smp.seed),
                      "terrain_digest": w.terrain_digest(), "best_index": int(res.best_index),
                      "best_cost": float(res.best_cost), "n_feasible": int(res.n_feasible),
                      "n_diverged": int(res.n_diverged), "n_goal": int(res.n_goal)}
    (OUT / "parity_meta.json").write_text(json.dumps(meta, indent=1) + "\n")
    print(json.dumps(meta, indent=1))


if __name__ == "__main__":
    main()
