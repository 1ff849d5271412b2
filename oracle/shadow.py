"""Per-cycle shadow oracle of the c5 closed loop — TEST INFRASTRUCTURE ONLY.

After every device planning call of the closed loop (bench.py --config c5,
tests/test_gpu_api.py::test_closed_loop_fp32_shadow_oracle_every_cycle), the
reference CPU planner (oracle/_ref) is run
on the SAME plant state and the same sampler (seed + cycle, warm start) on

  * every `stride`-th candidate of the cycle (a deterministic strided sample),
  * the device's `top_m` best candidates by its own (infeasible, J, k) key,

and the north-star rules (BASELINE north_star) are
applied per cycle:

  * per candidate: cost within 1e-4 relative and identical divergence flags,
    except where the reference itself is ill-conditioned: its own cost moves
    by >= 1e-4 under fp32-scale perturbations of the plant state / terrain
    (oracle/conditioning.extended_spread, the rule of the parity tests),
    evaluated for every candidate over the tolerance and for both winners;
  * winner: the device's winner is the reference's arg-min over the evaluated
    set, or the reference's gap between the two is <= 1e-4, or one of the two
    is ill-conditioned.

The strided sample bounds the CPU work (K/stride + top_m candidates per
cycle, plus 27 perturbed runs of the few over the tolerance); the timed
planning calls never include it.
"""
from __future__ import annotations

import time

import numpy as np

from oracle.conditioning import extended_spread, rel_err

TOL = 1e-4


def key_order(cost, flags, idx):
    """(infeasible, J, k) order of the listed candidates."""
    return np.lexsort((idx, cost, (flags & 1) == 0))


class ShadowCheck:
    def __init__(self, loop, oracle, stride=64, top_m=64, threads=8):
        self.loop, self.orc, self.stride, self.top_m, self.threads = loop, oracle, stride, top_m, threads
        from paper_2603_20525_b200 import planner as PL
        sd = None if loop.sdist is None else PL.SignedDistanceMap(loop.grid, loop.sdist, True)
        self.terr, self._tkeep = PL.make_terrain(PL.Heightmap(loop.grid, loop.heights), sd)
        self.cycles = []
        self.seconds = 0.0

    def check(self, loop, cycle, state, warm, plan, rec):
        t0 = time.perf_counter()
        K = loop.cfg.n_samples
        pl = plan.planner
        dcost, dflags, _ = pl.costs(K)
        order = key_order(dcost, dflags, np.arange(K))
        idx = np.union1d(np.arange(0, K, self.stride), order[:self.top_m])
        idx = np.union1d(idx, [rec.best_index])
        smp, keep = loop.sampling(cycle, warm)
        rc, oc, of, om, err = self.orc.solve_indices(loop.params, smp, self.terr, state, idx,
                                                     threads=self.threads)
        assert rc == 0, err
        rel = rel_err(dcost[idx], oc)
        divmis = (dflags[idx] & 2) != (of & 2)
        over = (rel > TOL) | divmis
        o = key_order(oc, of, idx)[0]
        w = int(np.searchsorted(idx, rec.best_index))
        check = np.union1d(np.where(over)[0], [o, w])
        sp = extended_spread(self.orc, loop, loop.params, smp, self.terr, state, idx[check],
                             self.threads)
        ill = np.zeros(len(idx), bool)
        ill[check] = sp >= TOL
        divmis = divmis & ~ill
        # winner rule over the evaluated set
        if idx[o] == rec.best_index:
            verdict = "same"
        else:
            inf_w, inf_o = (of[w] & 1) == 0, (of[o] & 1) == 0
            gap = np.inf if inf_w != inf_o else (oc[w] - oc[o]) / abs(oc[o])
            if gap <= TOL:
                verdict = "within_tol"
            elif ill[w] or ill[o]:
                verdict = "ill_conditioned"
            else:
                verdict = "violation"
        self.cycles.append(dict(
            cycle=cycle, compared=int(len(idx)), ill=int(ill.sum()),
            max_rel_well=float(rel[~ill].max()) if (~ill).any() else 0.0,
            over_tol_well=int((over & ~ill).sum()), divflag_mismatch_well=int(divmis.sum()),
            winner=verdict, device_best=int(rec.best_index), oracle_best=int(idx[o])))
        self.seconds += time.perf_counter() - t0

    def summary(self):
        c = self.cycles
        if not c:
            return None
        verdicts = [x["winner"] for x in c]
        return {
            "cycles": len(c), "stride": self.stride, "top_m": self.top_m,
            "candidates_compared": int(sum(x["compared"] for x in c)),
            "over_tol_ill_conditioned": int(sum(x["ill"] for x in c)),
            "max_rel_err_well_conditioned": max(x["max_rel_well"] for x in c),
            "over_tol_well_conditioned": int(sum(x["over_tol_well"] for x in c)),
            "divflag_mismatch_well_conditioned": int(sum(x["divflag_mismatch_well"] for x in c)),
            "winner_same": verdicts.count("same"),
            "winner_within_tol": verdicts.count("within_tol"),
            "winner_ill_conditioned": verdicts.count("ill_conditioned"),
            "winner_violations": verdicts.count("violation"),
            "check_seconds": self.seconds,
            "rule": "per cycle, same plant state: candidates every `stride` + device top_m; "
                    "cost <= 1e-4 rel and equal divergence flags unless the reference's own "
                    "spread under fp32-scale perturbations of the 13 state components and the "
                    "terrain is >= 1e-4; winner equal, or reference gap <= 1e-4, or "
                    "ill-conditioned",
        }
