"""Shared helpers of the parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np

from oracle.oracle import Oracle
from paper_2603_20525_b200 import planner as PL
from paper_2603_20525_b200 import workloads as W

BETA = 1e-3        # feasibility-flag margin band
COST_RTOL = 1e-4   # north_star per-candidate cost tolerance
COND_SPREAD = 1e-5  # conditioning threshold of the reference's own cost


def best_oracle():
    return Oracle("reference") if Oracle.available("reference") else Oracle("port")


def problem(name, K=None, N=None):
    w = W.make_workload(name)
    kw = {}
    if K:
        kw["n_samples"] = K
    if N:
        kw["n_steps"] = N
    w = w.with_(**kw) if kw else w
    p = w.params()
    smp, keep = PL.make_sampling(w.cfg)
    sd = None if w.sdist is None else PL.SignedDistanceMap(w.grid, w.sdist, True)
    terr, tkeep = PL.make_terrain(PL.Heightmap(w.grid, w.heights), sd)
    return w, p, smp, terr, (keep, tkeep)


def rel_err(a, b):
    with np.errstate(invalid="ignore", divide="ignore"):
        both = np.isfinite(a) & np.isfinite(b)
        r = np.where(both, np.abs(a - b) / np.abs(b), np.where(np.isfinite(a) == np.isfinite(b), 0.0, np.inf))
    return r


def conditioning_spread(orc, p, smp, terr, s0, base_cost, threads=8):
    """Max relative change of the reference's own cost under +-1e-6 m (x, y)
    and +-1e-7 rad (psi) perturbations of s0 — the fp32 rounding scale of
    the state.  Candidates with spread < COND_SPREAD are 'well-conditioned'."""
    spread = np.zeros(len(base_cost))
    for idx, d in ((0, 1e-6), (1, 1e-6), (3, 1e-7)):
        for sg in (1.0, -1.0):
            s1 = np.array(s0, dtype=np.float64)
            s1[idx] += sg * d
            rc, _, c1, *_ = orc.solve(p, smp, terr, s1, threads=threads)
            spread = np.maximum(spread, rel_err(c1, base_cost))
    return spread


def runner_up_gap(cost, flags, feasible_first=True):
    """Relative gap between the best and second-best key of the oracle."""
    inf = (~(flags & 1).astype(bool)) if feasible_first else np.zeros(len(cost), bool)
    order = np.lexsort((np.arange(len(cost)), cost, inf))
    b, r = order[0], order[1]
    if inf[b] != inf[r]:
        return np.inf
    return (cost[r] - cost[b]) / abs(cost[b])


def oracle_plan(orc, loop, threads=8):
    """A ClosedLoop planner callable backed by the CPU oracle (shadow planner)."""
    import time
    from dataclasses import replace

    import numpy as np
    from paper_2603_20525_b200 import planner as PL
    sd = None if loop.sdist is None else PL.SignedDistanceMap(loop.grid, loop.sdist, True)
    terr, tkeep = PL.make_terrain(PL.Heightmap(loop.grid, loop.heights), sd)

    def plan(state, warm, cycle):
        smp, keep = PL.make_sampling(replace(loop.cfg, seed=loop.cfg.seed + cycle), warm_seq=warm)
        t0 = time.perf_counter()
        rc, res, cost, flags, margin, sub, err = orc.solve(loop.params, smp, terr, state,
                                                           threads=threads)
        if rc == 1:
            raise PL.NumericError(err)
        assert rc == 0, err
        ctrl = orc.sample_controls(loop.params, smp, res.best_index)
        return (ctrl, int(res.best_index), float(res.best_cost), bool(res.best_feasible),
                (time.perf_counter() - t0) * 1e3, 0.0)
    plan._keep = (terr, tkeep)
    return plan
