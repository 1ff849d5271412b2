"""Shared helpers of the parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np

from oracle.oracle import Oracle
from paper_2603_20525_b200 import planner as PL
from paper_2603_20525_b200 import workloads as W

BETA = 1e-3        # feasibility-flag margin band
COST_RTOL = 1e-4   # north_star per-candidate cost tolerance
# A candidate is excluded from the per-candidate comparison only when the
# reference's OWN cost moves by >= the tolerance under fp32-scale
# perturbations (extended_spread): the exclusion threshold is the tolerance.
COND_SPREAD = COST_RTOL


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


from oracle.conditioning import extended_spread, fp32_terrain, state_perturbations  # noqa: E402,F401


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


def check_parity(orc, w, p, smp, terr, s0, cost, flags, margin, best_index=None, threads=8,
                 label="", spread_all=True):
    """The north-star per-candidate parity rule (BASELINE north_star), every
    candidate of the batch against the reference CPU planner:

      * cost within COST_RTOL relative and identical divergence flags, unless
        the reference itself is ill-conditioned on that candidate
        (extended_spread >= COST_RTOL, computed for every candidate over the
        tolerance): every candidate over the tolerance must be in that set;
      * feasibility flags identical wherever |margin| > BETA (and not excluded);
      * the same winner whenever the reference's best-vs-runner-up gap exceeds
        COST_RTOL and neither of the two is ill-conditioned.

    Prints the counts (compared, over tolerance, excluded, the round-1 6-way
    spread's ill-conditioned count over all candidates) and returns them."""
    K = smp.k_count
    rc, ores, oc, of, om, osub, err = orc.solve(p, smp, terr, s0, threads=threads)
    assert rc in (0, 1), err
    rel = rel_err(cost, oc)
    divmis = (flags & 2) != (of & 2)
    over = (rel > COST_RTOL) | divmis
    idx_over = np.where(over)[0] + smp.k_begin
    sp_over = extended_spread(orc, w, p, smp, terr, s0, idx_over, threads)
    excluded = np.zeros(K, bool)
    excluded[idx_over - smp.k_begin] = sp_over >= COND_SPREAD
    missed = over & ~excluded
    n_ill6 = None
    if spread_all:
        n_ill6 = int((conditioning_spread(orc, p, smp, terr, s0, oc, threads) >= COND_SPREAD).sum())
    rest = ~excluded
    worst = float(rel[rest].max()) if rest.any() else 0.0
    band = (np.abs(om) > BETA) & rest
    feas_mis = int(((flags[band] & 1) != (of[band] & 1)).sum())
    stats = dict(label=label, K=K, over_tol=int(over.sum()), excluded=int(excluded.sum()),
                 missed=int(missed.sum()), max_rel_rest=worst, ill_6way_all=n_ill6,
                 feas_mismatch=feas_mis, div_mismatch_rest=int((divmis & rest).sum()))
    # winner identity
    if rc == 0 and best_index is not None:
        order = np.lexsort((np.arange(K), oc, (of & 1) == 0))
        b, r = order[0], order[1]
        gap = np.inf if (of[b] & 1) != (of[r] & 1) else (oc[r] - oc[b]) / abs(oc[b])
        ill_w = extended_spread(orc, w, p, smp, terr, s0,
                                [b + smp.k_begin, best_index], threads)
        stats.update(oracle_best=int(b + smp.k_begin), device_best=int(best_index),
                     gap=float(gap), winner_ill=bool((ill_w >= COND_SPREAD).any()))
        if gap > COST_RTOL and not stats["winner_ill"]:
            assert best_index == b + smp.k_begin, stats
    print(f"parity {label}: K={K} over_tol={stats['over_tol']} excluded={stats['excluded']} "
          f"missed={stats['missed']} max_rel_rest={worst:.2e} ill_6way_all={n_ill6} "
          f"feas_mismatch={feas_mis} winner dev/ref={stats.get('device_best')}/"
          f"{stats.get('oracle_best')} gap={stats.get('gap')}")
    bad = np.where(missed)[0][:10]
    assert not missed.any(), (stats, [(int(k + smp.k_begin), float(rel[k]), float(cost[k]),
                                       float(oc[k])) for k in bad])
    assert feas_mis == 0, stats
    return stats
