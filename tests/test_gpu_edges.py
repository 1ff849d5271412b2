"""Edge cases of the planning cycle on the device: exact cost ties (arg-min
ties go to the lowest GLOBAL index), empty / oversize /
non-finite inputs rejected as ConfigError before any device work
(errors.hpp:9-18), and every (model, scheme, precision, lanes) kernel on a
ragged tiny batch."""
import dataclasses

import numpy as np
import pytest

from paper_2603_20525_b200 import _abi, planner as PL
from parity_util import best_oracle, problem, rel_err

pytestmark = pytest.mark.gpu


def _planner(w, p, K, **kw):
    pl = PL.Planner(device=0, k_max=K, n_steps_max=p.n_steps, **kw)
    pl.set_params(p)
    pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
    return pl


@pytest.mark.parametrize("precision", [_abi.PRECISION_FP32, _abi.PRECISION_FP64])
@pytest.mark.parametrize("k_begin", [0, 1000])
def test_start_inside_goal_ties_go_to_lowest_global_index(precision, k_begin):
    # starting inside the goal circle truncates every rollout at
    # t = 0, so J = Phi(s0) = 0 for every candidate -- an exact K-way tie
    w, p, smp, terr, keep = problem("c2", 256, 20)
    p.goal_x, p.goal_y = float(w.s0[0]), float(w.s0[1])
    smp, keep = PL.make_sampling(w.cfg, k_begin, 256)
    pl = _planner(w, p, 256, precision=precision)
    res, ctrl = pl.solve_raw(w.s0, smp)
    cost, flags, margin = pl.costs(256)
    pl.close()
    # every candidate is frozen at s0: bit-identical costs (Phi of the
    # position rebuilt from the cell anchor, ~1e-15 m from the goal centre)
    assert np.all(cost == cost[0]) and cost[0] < 1e-9 and np.all(flags & _abi.FLAG_GOAL)
    assert res.best_index == k_begin and res.best_cost == cost[0]
    assert res.n_goal == 256 and res.substeps_executed == 0


def test_equal_cost_candidates_resolve_to_lowest_index_across_warps():
    # the same rollout evaluated in two disjoint shards of one cycle is impossible
    # (controls come from the global index); instead force ties on the key:
    # with every constraint off and w_t = w_c = w_g = 0 all costs are exactly 0
    w, p, smp, terr, keep = problem("c1", 1000, 10)
    p.w_t = p.w_c = p.w_g = 0.0
    p.enable_dist = p.enable_rollover = 0
    for lanes in (1, 2, 4):
        pl = _planner(w, p, 1000, lanes=lanes)
        res, _ = pl.solve_raw(w.s0, smp)
        cost, flags, margin = pl.costs(1000)
        pl.close()
        assert np.all(cost == 0.0)
        assert res.best_index == 0


@pytest.mark.parametrize("bad", ["empty", "index_overflow", "nan_state", "inf_state"])
def test_bad_inputs_are_config_errors(bad):
    w, p, smp, terr, keep = problem("c1", 64, 5)
    pl = _planner(w, p, 64)
    s0 = w.s0.copy()
    if bad == "empty":
        smp.k_count = 0
    elif bad == "index_overflow":
        smp.k_begin = (1 << 31) - 10
    elif bad == "nan_state":
        s0[7] = np.nan
    else:
        s0[0] = np.inf
    with pytest.raises(PL.ConfigError):
        pl.solve_raw(s0, smp)
    # the context stays usable after a rejected cycle
    res, _ = pl.solve_raw(w.s0, PL.make_sampling(w.cfg)[0])
    assert res.n_candidates == 64
    pl.close()


@pytest.mark.parametrize("model,scheme", [(_abi.MODEL_SRB, _abi.SCHEME_EULER),
                                          (_abi.MODEL_SRB, _abi.SCHEME_RK4),
                                          (_abi.MODEL_EST, _abi.SCHEME_EULER),
                                          (_abi.MODEL_EST, _abi.SCHEME_RK4)])
def test_every_kernel_on_a_ragged_batch(model, scheme):
    # K = 37: one full warp + a 5-lane tail (and 37 x L lanes for L = 2, 4)
    w, p, smp, terr, keep = problem("c2", 37, 12)
    p.model, p.scheme = model, scheme
    orc = best_oracle()
    rc, ores, oc, of, om, osub, err = orc.solve(p, smp, terr, w.s0, threads=4)
    assert rc == 0, err
    lanes_set = (1, 2, 4) if model == _abi.MODEL_SRB else (0,)
    for precision in (_abi.PRECISION_FP32, _abi.PRECISION_FP64):
        for lanes in (lanes_set if precision == _abi.PRECISION_FP32 else (0,)):
            pl = _planner(w, p, 37, precision=precision, lanes=lanes)
            res, ctrl = pl.solve_raw(w.s0, smp)
            cost, flags, margin = pl.costs(37)
            pl.close()
            tol = 1e-9 if precision == _abi.PRECISION_FP64 else 1e-4
            assert rel_err(cost, oc).max() <= tol, (precision, lanes)
            np.testing.assert_array_equal(flags & 2, of & 2)
            assert res.n_candidates == 37


@pytest.mark.parametrize("dx,dy", [(-60.0, 0.0), (-60.0, -60.0), (0.0, 80.0)])
def test_off_map_starts_match_oracle(dx, dy):
    """Rollouts that start outside the heightmap (edge strip, corner, far
    side): the fp32 kernels clamp only the CoM and read the wheel points from
    the replicated pad (ctx.cu upload_terrain), which must equal the
    reference's clamped lookups (terrain.hpp:37-44, flat extension)."""
    w, p, smp, terr, keep = problem("c1", 256, 20)
    s0 = np.array(w.s0, dtype=np.float64)
    s0[0] += dx
    s0[1] += dy
    p.goal_x, p.goal_y = float(s0[0] + 10.0), float(s0[1])
    orc = best_oracle()
    rc, ores, oc, of, om, osub, err = orc.solve(p, smp, terr, s0, threads=8)
    assert rc == 0, err
    for precision, tol in ((_abi.PRECISION_FP32, 1e-4), (_abi.PRECISION_FP64, 1e-9)):
        pl = _planner(w, p, 256, precision=precision)
        res, ctrl = pl.solve_raw(s0, smp)
        cost, flags, margin = pl.costs(256)
        pl.close()
        assert rel_err(cost, oc).max() < tol
        np.testing.assert_array_equal(flags, of)
        assert res.best_index == ores.best_index


def test_terrain_pad_follows_params():
    """set_params after set_terrain with a vehicle reaching further than the
    terrain's replicated pad re-uploads it: the result equals a context that
    got the same params before the terrain, bit for bit."""
    w, p, smp, terr, keep = problem("c2", 512, 30)
    p2 = type(p).from_buffer_copy(p)
    p2.L_f, p2.L_r, p2.e = 2.5 * p.L_f, 2.5 * p.L_r, 2.0 * p.e
    a = _planner(w, p, 512)
    a.solve_raw(w.s0, smp)
    a.set_params(p2)  # wider pad -> re-upload from the context's host copy
    ra, _ = a.solve_raw(w.s0, smp)
    ca = a.costs(512)
    a.close()
    b = _planner(w, p2, 512)
    rb, _ = b.solve_raw(w.s0, smp)
    cb = b.costs(512)
    b.close()
    for x, y in zip(ca, cb):
        np.testing.assert_array_equal(x, y)
    assert ra.best_index == rb.best_index and ra.best_cost == rb.best_cost


def test_terrain_beyond_the_texture_limit_is_a_config_error():
    """The fp32 store is also read through 1-D linear textures whose width the
    device bounds (cudaDevAttrMaxTexture1DLinearWidth, 4 texels per padded
    cell): a heightmap past it is rejected as a ConfigError naming the limit
    (ADVICE round 1), while the fp64 context accepts it."""
    import torch
    n = 6200  # 6200^2 cells: > 2^27 / 4 padded cells
    g = PL.GridSpec(0.0, 0.0, 0.1, n, n)
    h = np.zeros((n, n))
    pl = PL.Planner(device=0)
    try:
        pl.set_terrain(PL.Heightmap(g, h))
        limited = False
    except PL.ConfigError as e:
        assert "texture limit" in str(e)
        limited = True
    pl.close()
    if not limited:
        pytest.skip("this device's 1-D texture limit is above 6200^2 padded cells")
    free, total = torch.cuda.mem_get_info()
    if free > 4 << 30:  # the fp64 store of 6200^2 is 1.5 GB
        p64 = PL.Planner(device=0, precision=_abi.PRECISION_FP64)
        p64.set_terrain(PL.Heightmap(g, h))
        p64.close()


@pytest.mark.parametrize("grow", [False, True])
def test_footprint_skip_on_an_arbitrary_sdf_map(grow):
    """The throughput-path launches (>= 131,072 candidates with the footprint
    term) let a warp skip the footprint term where the per-cell clearance
    proves it adds nothing (rollout_f32.cu, ctx.cu footprint_clearance); the
    bound is a min-filter of the map, so it must hold for ANY user SDF, not
    only a true distance field.  On a rough random map with pits (and, `grow`, a vehicle widened by set_params after the terrain: the
    re-uploaded clearance must cover it), the full launch equals the same
    candidates in two 65,536-candidate shards (latency path, no skip) bit for
    bit: cost, flags and margin."""
    K = 131072
    w, p, smp, terr, keep = problem("c2", K, 12)
    rng = np.random.default_rng(7)
    n = w.heights.shape[0]
    # not a distance field (node noise of +-0.2 m per 0.1 m cell), clear
    # (the warps skip) except 8 pits on the candidates' way (about half of
    # them hit one: the term decides feasibility)
    sd = 3.0 + rng.uniform(-0.2, 0.2, size=(n, n))
    for _ in range(8):
        i0, j0 = int(rng.uniform(8.0, 12.0) / 0.1), int(rng.uniform(22.0, 29.0) / 0.1)
        sd[j0 - 3:j0 + 4, i0 - 3:i0 + 4] = rng.uniform(-0.3, 0.1)
    w = dataclasses.replace(w, sdist=np.ascontiguousarray(sd, dtype=np.float64))
    p2 = type(p).from_buffer_copy(p)
    if grow:
        p2.L_f, p2.L_r, p2.e = 1.6 * p.L_f, 1.6 * p.L_r, 1.5 * p.e
    outs = []
    for shards in (1, 2):
        pl = PL.Planner(device=0, k_max=K, n_steps_max=p.n_steps, lanes=1)
        pl.set_params(p)
        pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
        pl.set_params(p2)
        cs = []
        for r in range(shards):
            k0, kc = PL.shard_range(K, r, shards)
            s, kk = PL.make_sampling(w.cfg, k0, kc)
            s.k_total = K
            pl.solve_raw(w.s0, s)
            cs.append(pl.costs(kc))
        pl.close()
        outs.append([np.concatenate([c[i] for c in cs]) for i in range(3)])
    for a, b in zip(*outs):
        np.testing.assert_array_equal(a, b)
    flags, margin = outs[0][1], outs[0][2]
    assert np.ptp(margin) > 0
    if not grow:
        assert 0 < int((flags & 1).sum()) < K  # the term decides feasibility somewhere


@pytest.mark.parametrize("devices", [[0], [0, 0]])
def test_cycle_after_all_diverged_equals_fresh_context(devices):
    """A one-process cycle is one kernel whose last block writes the host
    record and resets the reduction block for the next cycle (ctx.cu
    one_process).  A cycle whose every candidate diverges (100x suspension
    stiffness: forward Euler at 5 ms blows up; NumericError)
    and then normal cycles on the same context return exactly what a fresh
    context returns: nothing of the failed cycle leaks into the next."""
    w, p, smp, terr, keep = problem("c1", 1024, 50)
    stiff = type(p).from_buffer_copy(p)
    stiff.k_f, stiff.k_r = 100 * p.k_f, 100 * p.k_r
    pl = PL.Planner(devices=devices, k_max=1024, n_steps_max=50)
    pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
    pl.set_params(stiff)
    with pytest.raises(PL.NumericError):
        pl.solve_raw(w.s0, smp)
    pl.set_params(p)
    got = [pl.solve_raw(w.s0, smp)[0] for _ in range(2)]
    cost = pl.costs(1024)[0].copy()
    pl.close()
    fresh = _planner(w, p, 1024)
    ref, _ = fresh.solve_raw(w.s0, smp)
    ref_cost = fresh.costs(1024)[0].copy()
    fresh.close()
    np.testing.assert_array_equal(cost, ref_cost)
    for r in got:
        for f in ("best_index", "best_cost", "n_feasible", "n_diverged", "n_goal", "min_cost",
                  "mean_cost", "substeps_executed"):
            assert getattr(r, f) == getattr(ref, f), f
