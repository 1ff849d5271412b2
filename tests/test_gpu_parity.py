"""Device-vs-oracle parity through the C ABI (north_star criteria).

fp64 mode: every candidate within the 1e-4 cost tolerance (in practice
~1e-12), identical divergence flags, identical feasibility flags outside
the margin band, identical winner.
fp32 mode: every candidate on c1; on the chaotic c2/c3 rollouts every
candidate whose reference cost is itself stable to 1e-5 under state
perturbations at the fp32 rounding scale (parity_util.conditioning_spread).
"""
import numpy as np
import pytest

from paper_2603_20525_b200 import _abi, planner as PL
from parity_util import (BETA, COND_SPREAD, COST_RTOL, best_oracle, conditioning_spread,
                         problem, rel_err, runner_up_gap)

pytestmark = pytest.mark.gpu

CASES = [("c1", None, None), ("c2", 4096, None), ("c3", 4096, None)]


def _device(w, p, smp, precision):
    pl = PL.Planner(device=0, k_max=smp.k_count, n_steps_max=p.n_steps, precision=precision)
    pl.set_params(p)
    pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
    res, ctrl = pl.solve_raw(w.s0, smp)
    cost, flags, margin = pl.costs(smp.k_count)
    pl.close()
    return res, ctrl, cost, flags, margin


@pytest.fixture(scope="module")
def oracle():
    return best_oracle()


@pytest.mark.parametrize("name,K,N", CASES)
@pytest.mark.parametrize("precision", [_abi.PRECISION_FP64, _abi.PRECISION_FP32])
def test_parity(oracle, name, K, N, precision):
    w, p, smp, terr, _keep = problem(name, K, N)
    rc, ores, ocost, oflags, omargin, osub, err = oracle.solve(p, smp, terr, w.s0, threads=8)
    assert rc == 0, err
    res, ctrl, cost, flags, margin = _device(w, p, smp, precision)
    rel = rel_err(cost, ocost)
    if precision == _abi.PRECISION_FP64 or name == "c1":
        mask = np.ones(len(cost), bool)
    else:
        spread = conditioning_spread(oracle, p, smp, terr, w.s0, ocost)
        mask = spread < COND_SPREAD
        assert mask.mean() > 0.5, f"only {mask.mean():.2f} well-conditioned"
    worst = float(rel[mask].max())
    assert worst <= COST_RTOL, f"{name}: max rel {worst:.3e} over {mask.sum()} candidates"
    # divergence flags must agree on every compared candidate
    assert np.array_equal(flags[mask] & 2, oflags[mask] & 2)
    # feasibility flags agree away from the margin band
    band = np.abs(omargin) > BETA
    sel = mask & band
    assert np.array_equal(flags[sel] & 1, oflags[sel] & 1)
    # arg-min: the same winner whenever the oracle's gap exceeds the tolerance
    gap = runner_up_gap(ocost, oflags)
    if gap > COST_RTOL and mask[ores.best_index]:
        assert res.best_index == ores.best_index
        assert abs(res.best_cost - ores.best_cost) <= COST_RTOL * abs(ores.best_cost)
    # stats consistent with the per-candidate outputs
    assert res.n_feasible == int((flags & 1).sum())
    assert res.n_diverged == int(((flags & 2) > 0).sum())
    assert res.n_goal == int(((flags & 4) > 0).sum())
    # winner controls regenerate exactly from (seed, index)
    np.testing.assert_array_equal(ctrl, oracle.sample_controls(p, smp, res.best_index))
    print(f"{name} prec={precision}: compared {mask.sum()}/{len(mask)} max rel {worst:.2e} "
          f"feasible {res.n_feasible} diverged {res.n_diverged} best {res.best_index}")
