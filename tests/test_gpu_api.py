"""Device path behaviour through the public APIs (C ABI via the Python host
mirror): golden vectors, sharding, lane layouts, samplers, selection order,
error codes and edge cases."""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle.oracle import Oracle
from paper_2603_20525_b200 import _abi
from paper_2603_20525_b200 import planner as PL
from paper_2603_20525_b200 import workloads as W
from parity_util import COST_RTOL, best_oracle, problem, rel_err

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"


def run(w, p, smp, precision=_abi.PRECISION_FP32, lanes=0, sd=True, ordering=_abi.ORDER_AUTO):
    pl = PL.Planner(device=0, k_max=smp.k_count, n_steps_max=p.n_steps, precision=precision,
                    lanes=lanes, ordering=ordering)
    pl.set_params(p)
    pl.set_terrain_arrays(w.heights, w.sdist if sd else None, w.grid)
    res, ctrl = pl.solve_raw(w.s0, smp)
    cost, flags, margin = pl.costs(smp.k_count)
    pl.close()
    return res, ctrl, cost, flags, margin


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_goldens_fp64(name):
    meta = json.loads((GOLDEN / "parity_meta.json").read_text())[name]
    gold = np.load(GOLDEN / f"parity_{name}.npz")
    w, p, smp, terr, keep = problem(name, meta["K"], meta["N"])
    assert w.terrain_digest() == meta["terrain_digest"]
    res, ctrl, cost, flags, margin = run(w, p, smp, _abi.PRECISION_FP64)
    assert rel_err(cost, gold["cost"]).max() < 1e-6
    np.testing.assert_array_equal(flags, gold["flags"])
    assert res.best_index == meta["best_index"]
    assert res.n_feasible == meta["n_feasible"] and res.n_diverged == meta["n_diverged"]


def test_goldens_fp32_c1():
    meta = json.loads((GOLDEN / "parity_meta.json").read_text())["c1"]
    gold = np.load(GOLDEN / "parity_c1.npz")
    w, p, smp, terr, keep = problem("c1")
    res, ctrl, cost, flags, margin = run(w, p, smp)
    assert rel_err(cost, gold["cost"]).max() < COST_RTOL
    np.testing.assert_array_equal(flags, gold["flags"])
    assert res.best_index == meta["best_index"]


@pytest.mark.parametrize("precision", [_abi.PRECISION_FP32, _abi.PRECISION_FP64])
def test_shards_reassemble_bitwise(precision):
    """Two shards (k_begin) give bit-identical per-candidate results to one
    solve: controls come from the global index (multi-GPU determinism)."""
    w, p, smp, terr, keep = problem("c2", 3000, 40)
    full = run(w, p, smp, precision)
    parts = []
    for k0, kc in (PL.shard_range(3000, 0, 2), PL.shard_range(3000, 1, 2)):
        s2, keep2 = PL.make_sampling(w.with_(n_samples=3000, n_steps=40).cfg, k0, kc)
        parts.append(run(w, p, s2, precision))
    np.testing.assert_array_equal(np.concatenate([parts[0][2], parts[1][2]]), full[2])
    np.testing.assert_array_equal(np.concatenate([parts[0][3], parts[1][3]]), full[3])
    lib = _abi.load()
    keys = [(lib.tmpc_key_hi(r[0].best_cost, r[0].best_feasible, p.selection), r[0].best_index)
            for r in parts]
    assert min(keys)[1] == full[0].best_index


def test_lane_layouts_agree():
    """1, 2 and 4 lanes per candidate evaluate the same algorithm (L = 1 with
    the axle-symmetric sums, L = 2 / 4 with per-wheel sums and shuffles):
    each layout meets the north-star parity rule against the reference on
    every candidate (parity_util.check_parity) and they pick the same winner."""
    from parity_util import check_parity
    w, p, smp, terr, keep = problem("c1", 2000, 50)
    orc = best_oracle()
    outs = {L: run(w, p, smp, lanes=L) for L in (1, 2, 4)}
    for L in (1, 2, 4):
        res, ctrl, cost, flags, margin = outs[L]
        check_parity(orc, w, p, smp, terr, w.s0, cost, flags, margin, res.best_index,
                     label=f"c1 lanes={L}", spread_all=False)
        assert outs[L][0].best_index == outs[1][0].best_index


def test_repeat_is_bitwise_deterministic():
    w, p, smp, terr, keep = problem("c3", 2048, 60)
    a = run(w, p, smp)
    b = run(w, p, smp)
    np.testing.assert_array_equal(a[2], b[2])
    assert a[0].best_index == b[0].best_index and a[0].best_cost == b[0].best_cost


@pytest.mark.parametrize("kind,vdot", [(PL.SAMPLE_UNIFORM, 1.0), (PL.SAMPLE_RANDOM_WALK, 0.0),
                                       (PL.SAMPLE_RANDOM_WALK, 1.0), (PL.SAMPLE_WARM_GAUSS, 0.0)])
def test_samplers_match_oracle(kind, vdot):
    w = W.make_workload("c1").with_(n_samples=512, n_steps=30, sampler=kind, vdot_max=vdot)
    p = w.params()
    warm = np.random.default_rng(2).uniform(-0.6, 0.6, (30, 2))
    warm[:, 1] = 0.0 if vdot == 0.0 else warm[:, 1]
    smp, keep = PL.make_sampling(w.cfg, warm_seq=warm if kind == PL.SAMPLE_WARM_GAUSS else None)
    t, tk = PL.make_terrain(PL.Heightmap(w.grid, w.heights), None)
    rc, ores, oc, of, om, osub, err = Oracle("port").solve(p, smp, t, w.s0, threads=8)
    assert rc == 0, err
    res, ctrl, cost, flags, margin = run(w, p, smp, _abi.PRECISION_FP64)
    assert rel_err(cost, oc).max() < 1e-9
    assert res.best_index == ores.best_index
    np.testing.assert_allclose(ctrl, Oracle("port").sample_controls(p, smp, res.best_index),
                               rtol=0, atol=1e-15)


def test_selection_orders():
    w, p, smp, terr, keep = problem("c3", 2048, 100)
    res_ff, _, cost, flags, _ = run(w, p, smp)
    feas = (flags & 1).astype(bool)
    assert res_ff.best_feasible == 1
    assert res_ff.best_index == np.flatnonzero(feas)[np.argmin(cost[feas])]
    p.selection = _abi.SELECT_PLAIN
    res_pl, _, cost2, _, _ = run(w, p, smp)
    assert res_pl.best_index == int(np.argmin(cost2))
    assert res_pl.best_cost <= res_ff.best_cost


def test_single_candidate_and_odd_sizes():
    # N = 1 returns that sample regardless of cost
    w, p, smp, terr, keep = problem("c2", 1, 100)
    res, ctrl, cost, flags, margin = run(w, p, smp)
    assert res.best_index == 0 and res.n_candidates == 1
    for K in (33, 1000, 4097):
        w, p, smp, terr, keep = problem("c1", K, 10)
        res, ctrl, cost, flags, margin = run(w, p, smp)
        assert res.n_candidates == K and np.isfinite(cost).all()


def test_all_diverged_is_numeric_error():
    # every rollout diverged -> solver error (NumericError)
    w, p, smp, terr, keep = problem("c1", 64, 5)
    s0 = w.s0.copy()
    s0[4] = np.pi / 2 - 1e-4  # past the gimbal guard at t = 0 (dynamics.hpp:311)
    for prec in (_abi.PRECISION_FP32, _abi.PRECISION_FP64):
        pl = PL.Planner(device=0, k_max=64, n_steps_max=5, precision=prec)
        pl.set_params(p)
        pl.set_terrain_arrays(w.heights, None, w.grid)
        with pytest.raises(PL.NumericError):
            pl.solve_raw(s0, smp)
        cost, flags, margin = pl.costs(64)
        assert np.isinf(cost).all() and (flags == _abi.FLAG_DIVERGED).all()
        pl.close()


def test_solve_ocp_and_plan_step_api():
    w = W.make_workload("c1")
    cfg = w.with_(n_samples=512, n_steps=20).cfg
    seq, rr, stats = PL.solve_ocp(PL.SrbState.from_array(w.s0), PL.Heightmap(w.grid, w.heights),
                                  None, w.goal, cfg)
    assert len(seq.entries) == 20 and seq.horizon() == pytest.approx(1.0)
    assert stats.n_samples == 512 and stats.min_cost == rr.cost
    pl = PL.Planner(device=0, k_max=512, n_steps_max=20)
    pl.set_terrain(PL.Heightmap(w.grid, w.heights))
    u = PL.plan_step(pl, PL.SrbState.from_array(w.s0), w.goal, cfg)
    assert u == seq.entries[0]
    pl.close()


def test_no_features_equals_far_features():
    """Without an SDF (has_features false) the distance term vanishes exactly
    (constraints.hpp:93); a map whose features are all >> eps_dist away gives
    the same costs."""
    w, p, smp, terr, keep = problem("c1", 256, 20)
    a = run(w, p, smp, _abi.PRECISION_FP64, sd=False)
    far = w.with_()
    far.sdist = np.full_like(w.heights, 1000.0)
    b = run(far, p, smp, _abi.PRECISION_FP64)
    np.testing.assert_array_equal(a[2], b[2])


def _c5_loop(K, N):
    from paper_2603_20525_b200 import closed_loop as CL
    w = W.make_workload("c5").with_(n_samples=K, n_steps=N)
    return w, CL.ClosedLoop(w.heights, w.grid, w.sdist, w.goal, w.cfg)


def test_closed_loop_fp64_matches_oracle_trajectory():
    """c5 closed loop (warm-started Gaussian candidates, RK4 plant): with the
    fp64 device planner every cycle picks the oracle's winner, so the plant
    trajectory is bit-identical to the all-CPU loop."""
    from parity_util import oracle_plan
    w, loop = _c5_loop(1024, 40)
    dev = loop.run(loop.device_planner(precision=_abi.PRECISION_FP64), w.s0, cycles=25)
    ref = loop.run(oracle_plan(best_oracle(), loop), w.s0, cycles=25)
    assert [c.best_index for c in dev.cycles] == [c.best_index for c in ref.cycles]
    np.testing.assert_array_equal(dev.final_state, ref.final_state)
    assert dev.outcome == ref.outcome


def test_closed_loop_fp32_shadow_oracle_every_cycle():
    """c5 closed loop with the fp32 planner: every cycle, on the same plant
    state, the reference re-evaluates a strided sample + the device's best 64
    (oracle/shadow.py); per cycle the per-candidate rule holds on every
    well-conditioned candidate and the winner is the reference's (or within
    the 1e-4 gap, or ill-conditioned)."""
    from oracle.shadow import ShadowCheck
    w, loop = _c5_loop(4096, 100)
    sh = ShadowCheck(loop, best_oracle(), stride=16, top_m=64, threads=16)
    rec = loop.run(loop.device_planner(), w.s0, cycles=25, shadow=sh)
    s = sh.summary()
    print("shadow", s)
    assert s["cycles"] == len(rec.cycles) >= 20
    assert s["over_tol_well_conditioned"] == 0 and s["divflag_mismatch_well_conditioned"] == 0
    assert s["winner_violations"] == 0


def test_nccl_path_single_rank():
    """The cross-GPU arg-min path (ncclAllGather of the per-GPU records, host
    fold in rank order) on a 1-rank communicator gives the plain result."""
    import ctypes as C
    w, p, smp, terr, keep = problem("c2", 2048, 40)
    plain = run(w, p, smp)
    idb = C.create_string_buffer(128)
    assert _abi.load().tmpc_nccl_unique_id(idb) == 0
    pl = PL.Planner(device=0, k_max=2048, n_steps_max=40, nccl_id=idb.raw)
    pl.set_params(p)
    pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
    res, ctrl = pl.solve_raw(w.s0, smp)
    assert pl.lib.tmpc_kernels_per_cycle(pl.ctx) == 2  # + NCCL's all-gather
    pl.close()
    r0 = plain[0]
    assert (res.best_index, res.best_cost, res.n_feasible, res.n_diverged, res.n_goal) == \
        (r0.best_index, r0.best_cost, r0.n_feasible, r0.n_diverged, r0.n_goal)
    assert res.min_cost == r0.min_cost and res.mean_cost == r0.mean_cost  # integer sums
    np.testing.assert_array_equal(ctrl, plain[1])


@pytest.mark.parametrize("name,K", [("c1", None), ("c2", None), ("c3", 8192)])
def test_est_model_parity(name, K):
    """EST formulation on the device vs the reference: fp64 mode to 1e-9 on
    every candidate; fp32 under the north-star rule on every candidate
    (parity_util.check_parity)."""
    from parity_util import check_parity
    w, p, smp, terr, keep = problem(name, K)
    p.model = _abi.MODEL_EST
    orc = best_oracle()
    rc, ores, oc, of, om, osub, err = orc.solve(p, smp, terr, w.s0, threads=16)
    assert rc == 0, err
    r64 = run(w, p, smp, _abi.PRECISION_FP64)
    assert rel_err(r64[2], oc).max() < 1e-9
    np.testing.assert_array_equal(r64[3], of)
    assert r64[0].best_index == ores.best_index
    r32 = run(w, p, smp)
    check_parity(orc, w, p, smp, terr, w.s0, r32[2], r32[3], r32[4], r32[0].best_index,
                 threads=16, label=f"EST {name} fp32", spread_all=False)


@pytest.mark.parametrize("model", [_abi.MODEL_SRB, _abi.MODEL_EST])
@pytest.mark.parametrize("name,K", [("c1", None), ("c2", 512), ("c3", 512)])
def test_rk4_scheme_parity(name, K, model):
    """In-kernel RK4 (Scheme::kRk4, dynamics.hpp:454-466) vs the fp64 oracle:
    fp64 mode on every candidate; fp32 under the north-star rule on every
    candidate (parity_util.check_parity)."""
    from parity_util import check_parity
    w, p, smp, terr, keep = problem(name, K)
    p.model = model
    p.scheme = _abi.SCHEME_RK4
    orc = best_oracle()
    rc, ores, oc, of, om, osub, err = orc.solve(p, smp, terr, w.s0, threads=8)
    assert rc == 0, err
    r64 = run(w, p, smp, _abi.PRECISION_FP64)
    rel64 = rel_err(r64[2], oc)
    # c3's rollover rollouts are chaotic: ~1e-16 differences in the device
    # trig grow to ~1e-7 on a few candidates over 4 stages x 800 substeps
    assert rel64.max() < COST_RTOL and np.quantile(rel64, 0.99) < 1e-9
    assert (r64[3] != of).mean() < 0.01
    assert r64[0].best_index == ores.best_index
    # the SRB fp32 RK4 kernel shares a candidate over 1, 2 or 4 lanes
    for lanes in ((1, 2, 4) if model == _abi.MODEL_SRB else (0,)):
        r32 = run(w, p, smp, lanes=lanes)
        check_parity(orc, w, p, smp, terr, w.s0, r32[2], r32[3], r32[4], r32[0].best_index,
                     threads=16, label=f"RK4 {name} model={model} lanes={lanes}",
                     spread_all=False)



@pytest.mark.parametrize("name,K,lanes", [("c2", 8192, 1), ("c3", 4096, 2), ("c1", None, 4)])
def test_path_ordering_leaves_outputs_unchanged(name, K, lanes):
    """The ordering pre-pass (order.cu) only permutes the candidate -> thread
    assignment: every per-candidate output and the winner are bit-identical."""
    w, p, smp, terr, keep = problem(name, K)
    a = run(w, p, smp, lanes=lanes, ordering=_abi.ORDER_OFF)
    b = run(w, p, smp, lanes=lanes, ordering=_abi.ORDER_ON)
    for x, y in zip(a[2:], b[2:]):
        np.testing.assert_array_equal(x, y)
    np.testing.assert_array_equal(a[1], b[1])
    assert a[0].best_index == b[0].best_index and a[0].best_cost == b[0].best_cost
    assert a[0].n_feasible == b[0].n_feasible and a[0].substeps_executed == b[0].substeps_executed


def test_solve_raw_returns_independent_controls():
    """solve_raw reuses its state / controls buffers across calls (prebuilt
    ctypes pointers): the returned controls are copies, and a state array
    the caller changes afterwards does not leak into the next solve."""
    w, p, smp, terr, keep = problem("c2", 256, 20)
    pl = PL.Planner(device=0, k_max=256, n_steps_max=p.n_steps)
    pl.set_params(p)
    pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
    s0 = np.array(w.s0, dtype=np.float64)
    r1, c1 = pl.solve_raw(s0, smp)
    keep_c1 = c1.copy()
    s1 = s0.copy()
    s1[0] += 3.0
    r2, c2 = pl.solve_raw(s1, smp)
    np.testing.assert_array_equal(c1, keep_c1)
    r3, c3 = pl.solve_raw(s0, smp)
    pl.close()
    assert r3.best_index == r1.best_index and r3.best_cost == r1.best_cost
    np.testing.assert_array_equal(c3, c1)
    assert c2 is not c1 and c3 is not c1


def test_shard_count_independent_lane_layout():
    """results do not depend on the GPU count.  K = 12000 runs one
    lane per candidate on one GPU; four shards of 3000 would pick four lanes
    from their own size, but the layout follows k_total (tmpc_sampling), so
    every shard reproduces the one-GPU solve bit for bit."""
    w, p, smp, terr, keep = problem("c2", 12000, 30)
    full = run(w, p, smp)
    parts = []
    for r in range(4):
        k0, kc = PL.shard_range(12000, r, 4)
        s_r, keep_r = PL.make_sampling(w.cfg, k0, kc)
        assert s_r.k_total == 12000
        res, ctrl, cost, flags, margin = run(w, p, s_r)
        parts.append((res, cost, flags, margin))
    np.testing.assert_array_equal(np.concatenate([q[1] for q in parts]), full[2])
    np.testing.assert_array_equal(np.concatenate([q[2] for q in parts]), full[3])
    np.testing.assert_array_equal(np.concatenate([q[3] for q in parts]), full[4])
    best = min(parts, key=lambda q: (not (q[0].best_feasible), q[0].best_cost, q[0].best_index))
    assert best[0].best_index == full[0].best_index and best[0].best_cost == full[0].best_cost


@pytest.mark.parametrize("scheme", [_abi.SCHEME_EULER, _abi.SCHEME_RK4])
def test_large_batch_variants_read_the_same_terrain(scheme):
    """A launch of >= 32768 candidates takes the throughput gather path (SRB:
    third contact-point quad via TEX, footprint SDF via LDG; EST: footprint
    SDF via TEX), a smaller one the latency path.  The gather path moves loads
    between the LSU and texture pipes, never the arithmetic: a 2048-candidate
    shard and the first 2048 candidates of a 32768-candidate launch of the
    same problem (k_total = 32768, so the packed-axle choice agrees) are bit
    for bit equal, in both models."""
    w, p, smp, terr, keep = problem("c2", 32768, 30)
    p.scheme = scheme
    shard = PL.make_sampling(w.cfg, 0, 2048)
    assert shard[0].k_total == 32768
    full = PL.make_sampling(w.cfg, 0, 32768)
    for model in (_abi.MODEL_EST, _abi.MODEL_SRB):
        p.model = model
        a = run(w, p, shard[0])
        b = run(w, p, full[0])
        np.testing.assert_array_equal(a[2], b[2][:2048])
        np.testing.assert_array_equal(a[3], b[3][:2048])
        np.testing.assert_array_equal(a[4], b[4][:2048])


@pytest.mark.parametrize("ndev", [2, 3])
def test_multi_device_context_equals_one_device(ndev):
    """One context driving several GPUs (here `ndev` shards on cuda:0, the
    single-process multi-GPU mode): identical
    per-candidate outputs and a bit-identical folded result (winner, counts,
    min / mean cost) to the one-GPU solve."""
    w, p, smp, terr, keep = problem("c2", 5000, 30)
    one = run(w, p, smp)
    pl = PL.Planner(devices=[0] * ndev, k_max=5000, n_steps_max=30)
    assert pl.n_devices == ndev
    pl.set_params(p)
    pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
    res, ctrl = pl.solve_raw(w.s0, smp)
    cost, flags, margin = pl.costs(5000)
    # first cycle: the reduction block reset + the rollout per GPU; from then
    # on one kernel per GPU (its last block writes the host record and resets
    # the block), with the same result
    assert pl.lib.tmpc_kernels_per_cycle(pl.ctx) == 2 * ndev
    res2, _ = pl.solve_raw(w.s0, smp)
    assert pl.lib.tmpc_kernels_per_cycle(pl.ctx) == ndev
    assert (res2.best_index, res2.best_cost, res2.mean_cost) == (res.best_index, res.best_cost,
                                                                 res.mean_cost)
    pl.close()
    np.testing.assert_array_equal(cost, one[2])
    np.testing.assert_array_equal(flags, one[3])
    r0 = one[0]
    for f in ("best_index", "best_cost", "n_feasible", "n_diverged", "n_goal", "n_candidates",
              "min_cost", "mean_cost", "substeps_executed"):
        assert getattr(res, f) == getattr(r0, f), f
    np.testing.assert_array_equal(ctrl, one[1])


def test_graph_replay_equals_direct_launches():
    """The cycle replayed as a CUDA graph with updated arguments (default)
    equals direct launches, across changing s0 / seed / shard."""
    w, p, smp, terr, keep = problem("c2", 3000, 30)
    outs = []
    for graphs in (_abi.GRAPHS_AUTO, _abi.GRAPHS_OFF):
        pl = PL.Planner(device=0, k_max=3000, n_steps_max=30, graphs=graphs)
        pl.set_params(p)
        pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
        got = []
        for i in range(4):
            s0 = np.array(w.s0)
            s0[1] += 0.1 * i
            smp2, k2 = PL.make_sampling(w.cfg.__class__(**{**w.cfg.__dict__, "seed": 5 + i}),
                                        100 * i, 3000 - 100 * i)
            res, ctrl = pl.solve_raw(s0, smp2)
            got.append((res.best_index, res.best_cost, pl.costs(3000 - 100 * i)[0].copy()))
        pl.close()
        outs.append(got)
    for a, b in zip(*outs):
        assert a[0] == b[0] and a[1] == b[1]
        np.testing.assert_array_equal(a[2], b[2])


def test_nccl_missing_peer_fails_instead_of_hanging():
    """A 2-rank communicator whose second rank never starts: the non-blocking
    NCCL init runs under the context's watchdog and ctx_create fails with a
    runtime error after timeout_ms instead of hanging.  Run in
    a subprocess so a regression cannot hang the test session."""
    import subprocess
    import sys
    code = r"""
import ctypes as C, sys, time
sys.path.insert(0, %r)
from paper_2603_20525_b200 import _abi, planner as PL
idb = C.create_string_buffer(128)
assert _abi.load().tmpc_nccl_unique_id(idb) == 0
t0 = time.time()
try:
    PL.Planner(device=0, rank=0, world_size=2, nccl_id=idb.raw, timeout_ms=3000)
    print("NO ERROR")
except RuntimeError as e:
    print("ERR", round(time.time() - t0, 1), e)
""" % str(Path(__file__).resolve().parents[1])
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "ERR" in r.stdout and "timed out" in r.stdout, r.stdout


def test_multi_device_context_with_idle_devices():
    """More GPUs than candidates: the idle GPUs contribute empty records."""
    w, p, smp, terr, keep = problem("c1", 3, 10)
    one = run(w, p, smp)
    pl = PL.Planner(devices=[0, 0, 0, 0, 0], k_max=3, n_steps_max=10)
    pl.set_params(p)
    pl.set_terrain_arrays(w.heights, w.sdist, w.grid)
    res, ctrl = pl.solve_raw(w.s0, smp)
    cost, flags, margin = pl.costs(3)
    pl.close()
    np.testing.assert_array_equal(cost, one[2])
    assert res.best_index == one[0].best_index and res.n_candidates == 3
    assert res.mean_cost == one[0].mean_cost
