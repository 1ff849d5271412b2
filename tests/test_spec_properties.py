"""SPEC invariants and acceptance properties of the hot-path functions
(SPEC.md:40-62,101-107,166-176,215-240,377-383,559-562), checked on the
unmodified reference (oracle/_ref) and on the restatement (oracle port): the
pins SURVEY §4 lists beyond the single-value KATs of test_oracle.py."""
import math

import numpy as np
import pytest

from oracle.oracle import Oracle
from paper_2603_20525_b200 import _abi
from paper_2603_20525_b200 import planner as PL
from test_oracle import default_params, flat_terrain, needs_ref, rest_state, terr_struct

KINDS = ["port", pytest.param("reference", marks=needs_ref)]


def _q(orc, grid, hm, pts):
    t, keep = terr_struct(grid, hm)
    return orc.terrain_query(t, np.asarray(pts, dtype=np.float64))


# ---------------------------------------------------------------- terrain
@pytest.mark.parametrize("kind", KINDS)
def test_terrain_query_examples(kind):
    orc = Oracle(kind)
    grid, hm = flat_terrain(8, 1.0, h=2.0, origin=(0.0, 0.0))
    out = _q(orc, grid, hm, [(0.3, 4.7), (7.0, 7.0), (-3.0, 12.0)])
    assert np.all(out[:, 0] == 2.0) and np.all(out[:, 1:3] == 0.0)  # constant map
    # 2x2 map {0, 0, 1, 1} along y, mid-cell -> 0.5
    g2 = PL.GridSpec(0.0, 0.0, 1.0, 2, 2)
    h2 = np.array([[0.0, 0.0], [1.0, 1.0]])
    assert _q(orc, g2, h2, [(0.5, 0.5)])[0, 0] == pytest.approx(0.5, abs=1e-15)
    # exact at grid nodes
    rng = np.random.default_rng(1)
    hr = rng.uniform(-1, 1, (16, 16))
    g3 = PL.GridSpec(-2.0, 3.0, 0.25, 16, 16)
    nodes = [(-2.0 + 0.25 * i, 3.0 + 0.25 * j) for i, j in [(3, 4), (10, 2), (7, 13)]]
    out = _q(orc, g3, hr, nodes)
    assert np.allclose(out[:, 0], [hr[4, 3], hr[2, 10], hr[13, 7]], rtol=0, atol=1e-14)


@pytest.mark.parametrize("kind", KINDS)
def test_gradient_of_a_plane_is_exact_and_normal_is_unit(kind):
    orc = Oracle(kind)
    n, res = 32, 0.2
    x = np.arange(n) * res
    hm = np.tile(0.1 * x, (n, 1)) + 0.3 * np.arange(n)[:, None] * res  # z = 0.1 x + 0.3 y
    grid = PL.GridSpec(0.0, 0.0, res, n, n)
    rng = np.random.default_rng(2)
    pts = rng.uniform(1.0, (n - 1) * res - 1.0, (200, 2))
    out = _q(orc, grid, hm, pts)
    assert np.abs(out[:, 1] - 0.1).max() < 1e-9 and np.abs(out[:, 2] - 0.3).max() < 1e-9
    # normal_at = (-fx, -fy, 1) / |.| : unit length, positive z (terrain.hpp:97-100)
    nrm = np.stack([-out[:, 1], -out[:, 2], np.ones(len(out))], 1)
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    assert np.abs(np.linalg.norm(nrm, axis=1) - 1).max() < 1e-12 and np.all(nrm[:, 2] > 0)
    # continuity across a cell boundary
    b = 10 * res
    lo, hi = _q(orc, grid, hm, [(b - 1e-9, 1.3), (b + 1e-9, 1.3)])[:, 0]
    assert abs(lo - hi) < 1e-6 * res


# ---------------------------------------------------------------- tire
@needs_ref
def test_tire_is_odd_bounded_and_monotone():
    ref = Oracle("reference")
    p = PL.TireParams()
    alphas = np.linspace(-1.2, 1.2, 2001)
    fy = np.array([ref.lib.ref_tire_lateral_force(a, 1000.0, p.C, p.mu) for a in alphas])
    fyn = np.array([ref.lib.ref_tire_lateral_force(-a, 1000.0, p.C, p.mu) for a in alphas])
    assert np.array_equal(fy, -fyn)                   # odd in alpha
    assert np.all(np.abs(fy) < p.mu * 1000.0)         # |F_y| < mu F_z for finite alpha
    assert np.all(np.diff(fy) < 0)                    # monotone (sign: F_y opposes alpha)


# ---------------------------------------------------------------- SRB derivative
def _rand_states(rng, n, grid):
    vp = PL.VehicleParams()
    s = np.zeros((n, 13))
    ext = (grid.nx - 1) * grid.resolution
    s[:, 0:2] = rng.uniform(grid.origin_x + 3, grid.origin_x + ext - 3, (n, 2))
    s[:, 2] = vp.h + vp.R + rng.uniform(-0.15, 0.25, n)   # compressed .. near liftoff
    s[:, 3] = rng.uniform(-np.pi, np.pi, n)
    s[:, 4:6] = rng.uniform(-0.4, 0.4, (n, 2))
    s[:, 6] = rng.uniform(0.0, 15.0, n)
    s[:, 7:9] = rng.uniform(-2.0, 2.0, (n, 2))
    s[:, 9:12] = rng.uniform(-2.0, 2.0, (n, 3))
    s[:, 12] = rng.uniform(-0.6, 0.6, n)
    return s


def _rough(n=96, res=0.1, seed=5):
    rng = np.random.default_rng(seed)
    x = np.arange(n) * res
    hm = 0.2 * np.sin(x[None, :] * 1.3) * np.cos(x[:, None] * 0.9) + rng.uniform(-0.02, 0.02, (n, n))
    return PL.GridSpec(-4.8, -4.8, res, n, n), hm


@pytest.mark.parametrize("kind", KINDS)
def test_suspension_force_is_never_attractive(kind):
    # F_z,i >= 0 for random states (the damper is clamped at -F_k)
    orc = Oracle(kind)
    p = default_params()
    grid, hm = _rough()
    t, keep = terr_struct(grid, hm)
    rng = np.random.default_rng(3)
    n = 20000 if kind == "port" else 5000
    worst = np.inf
    for s in _rand_states(rng, n, grid):
        u = rng.uniform(-1, 1, 2)
        rc, d, diag = orc.srb_derivative(p, t, s, u)
        assert rc == 0
        worst = min(worst, diag[8:12].min())
    assert worst >= 0.0


@needs_ref
def test_airborne_wheels_carry_no_force():
    # chi large positive -> F_z,i = 0 and F_y,i = 0
    ref = Oracle("reference")
    p = default_params()
    grid, hm = flat_terrain()
    t, keep = terr_struct(grid, hm)
    s = rest_state(v=5.0)
    s[2] += 1.0  # one metre above the rest height: every wheel off the ground
    rc, d, diag = ref.srb_derivative(p, t, s, np.array([0.3, 0.0]))
    assert rc == 0 and np.all(diag[8:12] == 0.0) and np.all(diag[12:16] == 0.0)
    assert d[8] == pytest.approx(-p.g, rel=1e-12)  # free fall: v_bz' = g_bz


@pytest.mark.parametrize("kind", KINDS)
def test_left_right_mirror_symmetry(kind):
    # reflecting terrain and state across the x-z plane negates the
    # y / roll / yaw quantities of the derivative
    orc = Oracle(kind)
    p = default_params()
    n, res = 97, 0.1
    grid = PL.GridSpec(-4.8, -4.8, res, n, n)  # symmetric in y about 0
    rng = np.random.default_rng(4)
    hm = rng.uniform(-0.1, 0.1, (n, n))
    hmir = hm[::-1, :].copy()                   # H'(x, y) = H(x, -y)
    t1, k1 = terr_struct(grid, hm)
    t2, k2 = terr_struct(grid, hmir)
    flip_s = np.array([1, -1, 1, -1, 1, -1, 1, -1, 1, -1, 1, -1, -1], dtype=np.float64)
    for s in _rand_states(rng, 200, grid):
        s[0:2] = rng.uniform(-2.0, 2.0, 2)
        u = rng.uniform(-1, 1, 2)
        rc1, d1, _ = orc.srb_derivative(p, t1, s, u)
        rc2, d2, _ = orc.srb_derivative(p, t2, s * flip_s, u * np.array([-1.0, 1.0]))
        assert rc1 == 0 and rc2 == 0
        np.testing.assert_allclose(d2, d1 * flip_s, rtol=1e-9, atol=1e-9)


@needs_ref
def test_euler_rates_are_kinematically_consistent():
    # AC7: along an integrated SRB trajectory, the body rates
    # implied by the finite difference of rot_321 match omega within 10 dt
    ref = Oracle("reference")
    p = default_params()
    grid, hm = _rough(160, 0.1, 7)
    t, keep = terr_struct(grid, hm)
    s = rest_state(v=4.0)
    s[0], s[1] = -4.0, 0.0
    s[2] += float(np.interp(-4.0, np.arange(160) * 0.1 - 4.8, hm[48]))

    def rot321(psi, th, ph):
        cp, sp, ct, st, cf, sf = (math.cos(psi), math.sin(psi), math.cos(th), math.sin(th),
                                  math.cos(ph), math.sin(ph))
        return np.array([[cp * ct, cp * sf * st - cf * sp, sf * sp + cf * cp * st],
                         [ct * sp, cf * cp + sf * sp * st, cf * sp * st - cp * sf],
                         [-st, ct * sf, cf * ct]])

    dt = 0.005
    worst = 0.0
    for i in range(400):  # 2 s
        u = np.array([0.8 * math.sin(i * 0.02), 0.0])
        rc, s1 = ref.integrate_step(p, t, s, u, dt, _abi.SCHEME_EULER)
        assert rc == 0
        R0, R1 = rot321(*s[3:6]), rot321(*s1[3:6])
        W = (R0.T @ R1 - np.eye(3)) / dt
        w_fd = np.array([W[2, 1] - W[1, 2], W[0, 2] - W[2, 0], W[1, 0] - W[0, 1]]) / 2
        worst = max(worst, np.abs(w_fd - s[9:12]).max())
        s = s1
    assert worst < 10 * dt


def test_static_load_identity():
    # AC6: sum of the static loads 0.5 g K_zz,i over the wheels = M g
    rng = np.random.default_rng(6)
    for _ in range(100):
        vp = PL.VehicleParams(M=rng.uniform(100, 2000), L_f=rng.uniform(0.3, 2.0),
                              L_r=rng.uniform(0.3, 2.0), e=rng.uniform(0.5, 2.0))
        k = PL.load_transfer_coeffs(vp)
        total = 2 * (0.5 * vp.g * k[0]) + 2 * (0.5 * vp.g * k[1])
        assert total == pytest.approx(vp.M * vp.g, rel=1e-12)


# ---------------------------------------------------------------- sampler
def test_sampler_support_mean_and_determinism():
    import ctypes
    lib = _abi.load()
    p = default_params(n_steps=100)
    cfg = PL.PlannerConfig(n_samples=2000, n_steps=100, seed=99, sampler=PL.SAMPLE_UNIFORM)
    smp, keep = PL.make_sampling(cfg)
    draws = np.empty((2000, 100, 2))
    for k in range(2000):
        out = np.empty((100, 2))
        assert lib.tmpc_sample_controls(ctypes.byref(p), ctypes.byref(smp), k, _abi.dptr(out)) == 0
        draws[k] = out
    dr = draws[:, :, 0].ravel()
    assert np.all(np.abs(dr) <= 1.0) and np.all(draws[:, :, 1] == 0.0)  # support, v_bx_rate = 0
    sigma = 2.0 / math.sqrt(12.0)
    assert abs(dr.mean()) < 3 * sigma / math.sqrt(dr.size)           # mean -> 0
    again = np.empty((100, 2))
    lib.tmpc_sample_controls(ctypes.byref(p), ctypes.byref(smp), 17, _abi.dptr(again))
    assert np.array_equal(again, draws[17])                           # same seed, same sequence
