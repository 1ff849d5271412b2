"""Closed-loop receding-horizon driver (c5) on CPU: the
plant is the reference RK4 model, the planner here the CPU oracle."""
import math

import numpy as np
import pytest

from oracle.oracle import Oracle
from paper_2603_20525_b200 import _abi
from paper_2603_20525_b200 import closed_loop as CL
from paper_2603_20525_b200 import planner as PL
from paper_2603_20525_b200 import workloads as W
from parity_util import oracle_plan


def test_shift_warm():
    seq = np.arange(10.0).reshape(5, 2)
    out = CL.shift_warm(seq)
    np.testing.assert_array_equal(out[:4], seq[1:])
    np.testing.assert_array_equal(out[4], seq[4])


@pytest.mark.parametrize("name", ["c1", "c3"])
def test_plant_is_reference_rk4(name):
    """tmpc_plant_step == reference integrate_step<SrbModel> kRk4 (bitwise)."""
    kind = "reference" if Oracle.available("reference") else "port"
    orc = Oracle(kind)
    w = W.make_workload(name)
    p = w.params()
    t, keep = PL.make_terrain(PL.Heightmap(w.grid, w.heights), None)
    lib = _abi.load()
    rng = np.random.default_rng(11)
    for _ in range(5):
        u = np.array([rng.uniform(-1, 1), 0.0])
        a = w.s0.copy()
        assert lib.tmpc_plant_step(p, t, _abi.dptr(u), 0.001, 50, _abi.dptr(a)) == 0
        b = w.s0.copy()
        for _ in range(50):
            rc, b = orc.integrate_step(p, t, b, u, 0.001, 1)
        if kind == "reference":
            np.testing.assert_array_equal(a, b)
        else:
            np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-12)


def test_plant_reports_divergence():
    w = W.make_workload("c1")
    p = w.params()
    t, keep = PL.make_terrain(PL.Heightmap(w.grid, w.heights), None)
    s = w.s0.copy()
    s[4] = math.pi / 2 - 1e-4  # gimbal guard
    u = np.zeros(2)
    assert _abi.load().tmpc_plant_step(p, t, _abi.dptr(u), 0.001, 5, _abi.dptr(s)) == 1


def test_flat_goal_reached_on_time():
    """SPEC.md:441-446 / AC11: flat terrain, goal 20 m ahead at 5 m/s ->
    success at t = 3.5 +- 0.3 s (goal radius reached after 17.5 m)."""
    n = 400
    grid = PL.GridSpec(-10.0, -20.0, 0.1, n, n)
    h = np.zeros((n, n))
    vp = PL.VehicleParams()
    s0 = np.zeros(13)
    s0[2], s0[6] = vp.h + vp.R, 5.0
    cfg = PL.PlannerConfig(n_samples=128, seed=3, n_steps=20, dt_zoh=0.05, dt_int=0.005,
                           sampler=PL.SAMPLE_WARM_GAUSS, warm_sigma_frac=0.1)
    loop = CL.ClosedLoop(h, grid, None, PL.Goal(20.0, 0.0, 2.5), cfg)
    rec = loop.run(oracle_plan(Oracle("port"), loop, threads=8), s0, cycles=120)
    assert rec.outcome == "success"
    t_goal = len(rec.cycles) * cfg.dt_zoh
    assert abs(t_goal - 3.5) <= 0.3, t_goal
