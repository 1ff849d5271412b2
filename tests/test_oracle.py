"""The CPU oracle, pinned: against the reference itself (oracle/_ref, the
unmodified reference headers), the SPEC known-answer tests and the committed
golden vectors.  No GPU needed."""
import json
import math
from pathlib import Path

import numpy as np
import pytest

from oracle.oracle import Oracle
from paper_2603_20525_b200 import planner as PL
from paper_2603_20525_b200 import workloads as W
from parity_util import problem, rel_err

GOLDEN = Path(__file__).resolve().parent / "golden"
HAVE_REF = Oracle.available("reference")
needs_ref = pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built (needs /root/reference)")


@pytest.fixture(scope="module")
def port():
    return Oracle("port")


@pytest.fixture(scope="module")
def ref():
    return Oracle("reference")


def default_params(**kw):
    cfg = PL.PlannerConfig(n_samples=1, n_steps=16, dt_zoh=0.25, dt_int=0.005)
    for k, v in kw.items():
        setattr(cfg, k, v)
    return PL.make_params(PL.VehicleParams(), PL.TireParams(), PL.ConstraintConfig(),
                          PL.CostWeights(), PL.Goal(1e3, 0.0, 2.5), cfg)


def flat_terrain(n=64, res=0.5, h=0.0, origin=(-16.0, -16.0)):
    hm = np.full((n, n), h, dtype=np.float64)
    grid = PL.GridSpec(origin[0], origin[1], res, n, n)
    return grid, hm


def terr_struct(grid, hm, sd=None):
    t, keep = PL.make_terrain(PL.Heightmap(grid, hm),
                              None if sd is None else PL.SignedDistanceMap(grid, sd, True))
    return t, keep


def rest_state(z=None, v=0.0):
    vp = PL.VehicleParams()
    s = np.zeros(13)
    s[2] = vp.h + vp.R if z is None else z
    s[6] = v
    return s


# ------------------------------------------------------------------ KATs
def test_tire_lateral_force_kat(ref):
    # C=6.1, mu=0.6, alpha=0.1, F_z=1000 -> ~ -427.7 N
    assert ref.lib.ref_tire_lateral_force(0.1, 1000.0, 6.1, 0.6) == pytest.approx(-427.7558, abs=1e-3)
    assert ref.lib.ref_tire_lateral_force(0.0, 1000.0, 6.1, 0.6) == 0.0


def test_load_transfer_kat():
    # K_zzf ~ 410.0 kg, K_zy ~ 507.9 kg, K_zzf + K_zzr = M
    kf, kr, kx, ky = PL.load_transfer_coeffs(PL.VehicleParams())
    assert kf == pytest.approx(410.0302, abs=1e-3)
    assert ky == pytest.approx(507.9680, abs=1e-3)
    assert kf + kr == pytest.approx(PL.VehicleParams().M, rel=1e-15)


def test_esm_kat(port, ref):
    p = default_params()
    vp = PL.VehicleParams()
    u_flat = port.lib.oracle_esm(p, 0.0, 0.0)
    assert u_flat == pytest.approx(2436.1326, abs=1e-3)  # SPEC.md:285 (~2.44e3 J)
    phi_bar = math.atan(2 * (vp.h + vp.R) / vp.e)
    mg_r = vp.M * vp.g * math.hypot(vp.h + vp.R, vp.e / 2)
    assert abs(port.lib.oracle_esm(p, math.pi / 2 - phi_bar, 0.0)) < 1e-9 * mg_r  # AC4
    assert port.lib.oracle_esm(p, math.pi / 2 - phi_bar + 0.1, 0.0) < 0.0
    if HAVE_REF:
        for phi, th in [(0.0, 0.0), (0.3, -0.2), (-1.2, 0.4), (2.0, 0.1)]:
            assert port.lib.oracle_esm(p, phi, th) == ref.lib.ref_esm(p, phi, th)
    assert PL.esm_normalization(vp) == pytest.approx(u_flat, rel=1e-15)


@needs_ref
def test_soft_cost_kat(ref):
    # pi=-eps -> 0, pi=0 -> sigma, pi=eps -> 4 sigma; dist 0.1 m inside band
    f = ref.lib.ref_soft_cost_rate
    assert f(-0.25, 0.25, 1e6) == 0.0
    assert f(0.0, 0.25, 1e6) == 1e6
    assert f(0.25, 0.25, 1e6) == 4e6
    assert f(-0.15, 0.25, 1e6) == pytest.approx(1.6e5, rel=1e-12)


@pytest.mark.parametrize("kind", ["port", "reference"])
def test_srb_static_equilibrium(kind):
    # SPEC.md:220 / AC5: at rest on flat ground with chi = 0, |sdot| < 1e-6
    if kind == "reference" and not HAVE_REF:
        pytest.skip("no _ref")
    orc = Oracle(kind)
    grid, hm = flat_terrain()
    t, keep = terr_struct(grid, hm)
    rc, d, diag = orc.srb_derivative(default_params(), t, rest_state(), [0.0, 0.0])
    assert rc == 0
    assert np.abs(np.delete(d, 0)).max() < 1e-6
    # static loads 0.5 g K_zz,i sum to M g (AC6)
    vp = PL.VehicleParams()
    assert diag[8:12].sum() == pytest.approx(vp.M * vp.g, rel=1e-12)


def test_srb_derivative_restatement_matches_reference(port):
    if not HAVE_REF:
        pytest.skip("no _ref")
    ref = Oracle("reference")
    w = W.make_workload("c3")
    t, keep = terr_struct(w.grid, w.heights)
    rng = np.random.default_rng(7)
    for _ in range(200):
        s = w.s0.copy()
        s[0] += rng.uniform(-3, 3)
        s[1] += rng.uniform(-3, 3)
        s[2] += rng.uniform(-0.2, 0.2)
        s[3:6] += rng.uniform(-0.5, 0.5, 3)
        s[6:9] += rng.uniform(-2, 2, 3)
        s[9:12] += rng.uniform(-1, 1, 3)
        s[12] = rng.uniform(-0.6, 0.6)
        u = [rng.uniform(-1, 1), 0.0]
        rc1, d1, g1 = port.srb_derivative(default_params(), t, s, u)
        rc2, d2, g2 = ref.srb_derivative(default_params(), t, s, u)
        assert rc1 == rc2 == 0
        np.testing.assert_allclose(d1, d2, rtol=1e-12, atol=1e-9)
        # F_z >= 0 always: the damper never makes the force attractive
        assert (g2[8:12] >= 0).all()


def test_gimbal_guard(port):
    grid, hm = flat_terrain()
    t, keep = terr_struct(grid, hm)
    s = rest_state()
    s[4] = math.pi / 2 - 1e-4
    assert port.srb_derivative(default_params(), t, s, [0, 0])[0] == 1
    if HAVE_REF:
        assert Oracle("reference").srb_derivative(default_params(), t, s, [0, 0])[0] == 1


def test_straight_line_and_euler_vs_rk4(port):
    # zero controls on flat terrain -> x = v t (Euler exact)
    grid, hm = flat_terrain(n=256, res=0.5, origin=(-10.0, -64.0))
    t, keep = terr_struct(grid, hm)
    p = default_params()
    s = rest_state(v=5.0)
    for _ in range(800):
        rc, s = port.integrate_step(p, t, s, [0.0, 0.0], 0.005, 0)
        assert rc == 0
    assert s[0] == pytest.approx(20.0, abs=1e-9)
    # Euler 5 ms vs RK4 1 ms on a sine ridge, 4 s -> within 0.2 m
    g2 = PL.GridSpec(-10.0, -32.0, 0.1, 700, 640)
    xs = g2.origin_x + 0.1 * np.arange(700)
    hm2 = np.tile(0.2 * np.sin(2 * np.pi * xs / 6.0), (640, 1))
    t2, keep2 = terr_struct(g2, hm2)
    s0 = rest_state(v=5.0)
    s0[2] += 0.2 * np.sin(0.0)
    se, sr = s0.copy(), s0.copy()
    for k in range(800):
        u = [0.5 if (k // 100) % 2 == 0 else -0.5, 0.0]
        rc, se = port.integrate_step(p, t2, se, u, 0.005, 0)
        assert rc == 0
        for _ in range(5):
            rc, sr = port.integrate_step(p, t2, sr, u, 0.001, 1)
            assert rc == 0
    assert math.hypot(se[0] - sr[0], se[1] - sr[1]) < 0.2


# ------------------------------------------------------------------ trajectory cost
def _single(port, p, grid, hm, s0, base_seq):
    smp = PL._abi.tmpc_sampling()
    smp.kind, smp.k_begin, smp.k_count, smp.warm_sigma_frac = PL.SAMPLE_WARM_GAUSS, 0, 1, 0.0
    seq = np.ascontiguousarray(base_seq, dtype=np.float64)
    smp.warm_seq = PL._abi.dptr(seq)
    t, keep = terr_struct(grid, hm)
    rc, res, cost, flags, margin, sub, err = port.solve(p, smp, t, s0)
    assert rc == 0, err
    return cost[0], flags[0]


def test_trajectory_cost_hand_values(port):
    # straight flat run, delta_rate = 0, no features, 4 s, ending
    # 10 m from the goal -> J = w_t * 4 + w_g * 10 (the SPEC prints "= 80";
    # with w_t = 5, w_g = 15 the closed form is 20 + 150 = 170).
    grid, hm = flat_terrain(n=512, res=0.25, origin=(-10.0, -64.0))
    p = default_params()
    p.goal_x, p.goal_y = 5.0 * 4.0 + 10.0, 0.0
    s0 = rest_state(v=5.0)
    J, fl = _single(port, p, grid, hm, s0, np.zeros((16, 2)))
    assert J == pytest.approx(5.0 * 4.0 + 15.0 * 10.0, rel=1e-9)
    assert fl & PL.FLAG_FEASIBLE
    # constant delta_rate 0.5 adds w_c * 0.25 * 4 = 8 (isolated
    # with w_t = w_g = 0)
    p.w_t, p.w_g = 0.0, 0.0
    seq = np.zeros((16, 2))
    seq[:, 0] = 0.5
    J, fl = _single(port, p, grid, hm, s0, seq)
    assert J == pytest.approx(8.0, rel=1e-9)


def test_start_inside_goal(port):
    # start inside the goal circle -> J = Phi only
    grid, hm = flat_terrain()
    p = default_params()
    p.goal_x, p.goal_y = 1.0, 0.0
    J, fl = _single(port, p, grid, hm, rest_state(v=5.0), np.zeros((16, 2)))
    assert J == pytest.approx(15.0 * 1.0, rel=1e-12)
    assert fl & PL.FLAG_GOAL


# ------------------------------------------------------------------ RNG / sampler
def test_random_access_rng_matches_stream(port):
    if not HAVE_REF:
        pytest.skip("no _ref")
    ref = Oracle("reference")
    rng = np.random.default_rng(1)
    for _ in range(50):
        seed = int(rng.integers(0, 2**63))
        k = int(rng.integers(0, 2**31))
        s = ref.lib.ref_substream(seed, k, 0, 0)
        assert port.lib.oracle_substream(seed, k, 0, 0) == s
        for j in (0, 1, 7, 199):
            assert port.lib.oracle_rng_draw(s, j) == ref.lib.ref_rng_draw(s, j)


@pytest.mark.parametrize("kind", [PL.SAMPLE_UNIFORM, PL.SAMPLE_RANDOM_WALK, PL.SAMPLE_WARM_GAUSS])
@pytest.mark.parametrize("vdot", [0.0, 1.5])
def test_sampler_bit_exact(port, kind, vdot):
    """oracle restatement == reference RngStream (sequential) == product host
    sampler (the device's random-access formula, tmpc_sample_controls)."""
    lib = PL._abi.load()
    cfg = PL.PlannerConfig(n_samples=64, seed=99, n_steps=40, dt_zoh=0.05, sampler=kind,
                           vdot_max=vdot, walk_step=0.3, warm_sigma_frac=0.1)
    p = PL.make_params(PL.VehicleParams(), PL.TireParams(), PL.ConstraintConfig(),
                       PL.CostWeights(), PL.Goal(10, 0, 2.5), cfg)
    warm = np.random.default_rng(3).uniform(-0.5, 0.5, (40, 2))
    smp, keep = PL.make_sampling(cfg, warm_seq=warm if kind == PL.SAMPLE_WARM_GAUSS else None)
    for k in (0, 1, 2, 63, 12345):
        a = port.sample_controls(p, smp, k)
        b = np.zeros((40, 2))
        assert lib.tmpc_sample_controls(p, smp, k, PL._abi.dptr(b)) == 0
        np.testing.assert_array_equal(a, b)
        if HAVE_REF:
            np.testing.assert_array_equal(a, Oracle("reference").sample_controls(p, smp, k))
        assert np.all(np.abs(a[:, 0]) <= 1.0)
        if vdot == 0.0:
            assert np.all(a[:, 1] == 0.0)
        else:
            assert np.all(np.abs(a[:, 1]) <= vdot)
    if kind == PL.SAMPLE_UNIFORM:  # mean -> 0 within 3 sigma / sqrt(n)
        draws = np.concatenate([port.sample_controls(p, smp, k)[:, 0] for k in range(2000)])
        assert abs(draws.mean()) < 3 * (1 / math.sqrt(3)) / math.sqrt(len(draws))


# ------------------------------------------------------------------ terrain
def test_padded_field_identity(port):
    """height_at / gradient_at / value_at == bilinear of the
    2-cell replicate-padded node fields with one clamp, everywhere (incl.
    outside the map), to fp32 storage precision."""
    w = W.make_workload("c2")
    t, keep = terr_struct(w.grid, w.heights, w.sdist)
    rng = np.random.default_rng(5)
    ext = w.grid.resolution * (w.grid.nx - 1)
    xy = np.concatenate([rng.uniform(-2.0, ext + 2.0, (20000, 2)),
                         np.stack(np.meshgrid(np.arange(0, 6) * 0.1, np.arange(0, 6) * 0.1), -1).reshape(-1, 2),
                         [[0.0, 0.0], [ext, ext], [-1.0, ext + 1.0], [ext + 5.0, -5.0]]])
    a = port.terrain_query(t, xy, variant=0)
    b = port.terrain_query(t, xy, variant=1)
    assert np.abs(a[:, 0] - b[:, 0]).max() < 1e-6
    assert np.abs(a[:, 1:3] - b[:, 1:3]).max() < 1e-5
    assert np.abs(a[:, 3] - b[:, 3]).max() < 1e-5
    if HAVE_REF:
        r = Oracle("reference").terrain_query(t, xy)
        np.testing.assert_array_equal(a, r)


def test_sdist_map_bit_exact_vs_reference():
    """Product build_sdist_map (culled, threaded) == reference build_sdist_map."""
    if not HAVE_REF:
        pytest.skip("no _ref")
    ts = W.TerrainSpec(160, 0.1, 77, n_obstacles=12)
    grid = PL.GridSpec(0.0, 0.0, 0.1, 160, 160)
    _, off, verts = W.synth_obstacles(ts, (1.0, 8.0), 2.0)
    kinds = np.zeros(len(off) - 1, np.int32)
    kinds[-1] = 1  # one path boundary exercises the unculled branch
    ours = W.build_sdist(grid, off, verts, kinds)
    theirs = Oracle("reference").build_sdist_map(grid, off, verts, kinds)
    np.testing.assert_array_equal(ours, theirs)
    restated = Oracle("port").build_sdist_map(grid, off, verts, kinds)
    np.testing.assert_array_equal(ours, restated)


# ------------------------------------------------------------------ planner
@pytest.mark.parametrize("name,K", [("c1", None), ("c2", 256), ("c3", 256)])
def test_restatement_matches_reference(port, name, K):
    if not HAVE_REF:
        pytest.skip("no _ref")
    w, p, smp, terr, keep = problem(name, K)
    rc1, r1, c1, f1, m1, s1, e1 = port.solve(p, smp, terr, w.s0, threads=8)
    rc2, r2, c2, f2, m2, s2, e2 = Oracle("reference").solve(p, smp, terr, w.s0, threads=8)
    assert rc1 == rc2 == 0
    assert rel_err(c1, c2).max() < 1e-9
    np.testing.assert_array_equal(f1, f2)
    assert r1.best_index == r2.best_index


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_goldens(port, name):
    """Committed reference outputs (tests/golden/make_golden.py) reproduce."""
    meta = json.loads((GOLDEN / "parity_meta.json").read_text())[name]
    gold = np.load(GOLDEN / f"parity_{name}.npz")
    w, p, smp, terr, keep = problem(name, meta["K"], meta["N"])
    assert w.terrain_digest() == meta["terrain_digest"]
    np.testing.assert_array_equal(w.s0, gold["s0"])
    rc, res, cost, flags, margin, sub, err = port.solve(p, smp, terr, w.s0, threads=8)
    assert rc == 0
    assert rel_err(cost, gold["cost"]).max() < 1e-9
    np.testing.assert_array_equal(flags, gold["flags"])
    assert res.best_index == meta["best_index"]
    for k in range(3):
        np.testing.assert_array_equal(port.sample_controls(p, smp, k), gold["controls_k012"][k])


def test_nested_prefix_monotone_and_deterministic(port):
    # SPEC.md:388-389,400 / AC10: best(N2) <= best(N1) for nested prefixes,
    # identical output for any worker count
    w, p, smp, terr, keep = problem("c1", 1024, 20)
    costs = {}
    for threads in (1, 4, 8):
        rc, res, c, f, m, s, e = port.solve(p, smp, terr, w.s0, threads=threads)
        costs[threads] = (res.best_index, c.copy())
    assert costs[1][0] == costs[4][0] == costs[8][0]
    np.testing.assert_array_equal(costs[1][1], costs[8][1])
    c = costs[1][1]
    best = [c[:n].min() for n in (64, 256, 1024)]
    assert best[0] >= best[1] >= best[2]


@pytest.mark.parametrize("name,K", [("c1", None), ("c2", 256), ("c3", 256)])
def test_est_restatement_matches_reference(port, name, K):
    """EST formulation: restated est_derivative + the
    lateral-acceleration constraint == the reference EstModel via oracle/_ref."""
    if not HAVE_REF:
        pytest.skip("no _ref")
    w, p, smp, terr, keep = problem(name, K)
    p.model = PL._abi.MODEL_EST
    rc1, r1, c1, f1, m1, s1, e1 = port.solve(p, smp, terr, w.s0, threads=8)
    rc2, r2, c2, f2, m2, s2, e2 = Oracle("reference").solve(p, smp, terr, w.s0, threads=8)
    assert rc1 == rc2 == 0
    assert rel_err(c1, c2).max() < 1e-12
    np.testing.assert_array_equal(f1, f2)
    assert r1.best_index == r2.best_index


def test_est_lateral_accel_constraint_semantics(port):
    """constraints.hpp:62-65: violation = |a_by - g_by| - a_by_bar; on flat
    ground driving straight at constant speed a_by = 0, so the EST rollout is
    feasible with margin 1 and the rollover soft cost is zero."""
    grid, hm = flat_terrain(n=512, res=0.25, origin=(-10.0, -64.0))
    p = default_params()
    p.model = PL._abi.MODEL_EST
    p.goal_x, p.goal_y = 30.0, 0.0
    J, fl = _single(port, p, grid, hm, rest_state(v=5.0), np.zeros((16, 2)))
    assert fl & PL.FLAG_FEASIBLE
    assert J == pytest.approx(5.0 * 4.0 + 15.0 * 10.0, rel=1e-9)


@pytest.mark.parametrize("model", ["srb", "est"])
@pytest.mark.parametrize("name,K", [("c1", None), ("c2", 128), ("c3", 128)])
def test_rk4_restatement_matches_reference(port, name, K, model):
    """RK4 scheme: the restated Scheme::kRk4 substep (four
    derivative stages, dynamics.hpp:454-466) == the reference
    integrate_step<Model>(..., Scheme::kRk4) via oracle/_ref."""
    if not HAVE_REF:
        pytest.skip("no _ref")
    w, p, smp, terr, keep = problem(name, K)
    p.scheme = PL._abi.SCHEME_RK4
    if model == "est":
        p.model = PL._abi.MODEL_EST
    rc1, r1, c1, f1, m1, s1, e1 = port.solve(p, smp, terr, w.s0, threads=8)
    rc2, r2, c2, f2, m2, s2, e2 = Oracle("reference").solve(p, smp, terr, w.s0, threads=8)
    assert rc1 == rc2 == 0
    assert rel_err(c1, c2).max() < 1e-9
    np.testing.assert_array_equal(f1, f2)
    np.testing.assert_array_equal(s1, s2)
    assert r1.best_index == r2.best_index
    # the scheme changes the rollout (not a silent Euler fallback)
    p.scheme = PL._abi.SCHEME_EULER
    rc3, r3, c3, *_ = port.solve(p, smp, terr, w.s0, threads=8)
    fin = np.isfinite(c1) & np.isfinite(c3)
    assert np.abs(c1[fin] - c3[fin]).max() > 1e-9
