"""Open-loop model-error analysis (
PAPER.md:1600-1621): the device batch (Planner.open_loop_errors) against
the reference restatement over the unmodified headers
(oracle/_ref ref_open_loop_errors), and the SPEC's own properties."""
import numpy as np
import pytest

from oracle.oracle import Oracle
from paper_2603_20525_b200 import _abi, planner as PL, workloads as W

needs_ref = pytest.mark.skipif(not Oracle.available("reference"), reason="oracle/_ref not built")


def _setup(name="c1", n=24, N=80, seed=0, flat=False):
    w = W.make_workload(name).with_(n_steps=N)
    heights = np.zeros_like(w.heights) if flat else w.heights
    p = w.params()
    rng = np.random.default_rng(seed)
    s0 = np.repeat(W.initial_state(heights, w.grid, w.s0[0], w.s0[1], w.v0)[None], n, 0)
    s0[:, 1] += rng.uniform(-0.5, 0.5, n)          # SPEC.md:475 lateral offset +-0.5 m
    s0[:, 3] += rng.uniform(-0.05, 0.05, n)        # heading +-0.05 rad
    u = np.zeros((n, N, 2))
    u[:, :, 0] = rng.uniform(-1.0, 1.0, (n, N)) * (0.0 if flat else 1.0)
    terr, keep = PL.make_terrain(PL.Heightmap(w.grid, heights), None)
    return w, p, heights, s0, u, terr, keep


@needs_ref
def test_reference_self_comparison_is_zero():
    """model = plant dynamics and LOD -> zero error."""
    w, p, h, s0, u, terr, keep = _setup(n=4, N=20)
    p.scheme = _abi.SCHEME_RK4
    p.dt_int = 0.001
    p.dt_zoh = 0.05
    rc, loc, esm, fl, err = Oracle("reference").open_loop_errors(p, terr, _abi.MODEL_SRB, s0, u,
                                                                 plant_dt=0.001, threads=4)
    assert rc == 0, err
    assert (fl == 0).all() and (loc == 0).all() and (esm == 0).all()


@needs_ref
@pytest.mark.parametrize("model", [_abi.MODEL_SRB, _abi.MODEL_EST])
def test_reference_straight_flat_run_small(model):
    """straight flat run, both models -> location error < 0.01 m."""
    w, p, h, s0, u, terr, keep = _setup(n=4, N=80, flat=True)
    s0[:, 3] = 0.0
    s0[:, 2] = p.h + p.R
    rc, loc, esm, fl, err = Oracle("reference").open_loop_errors(p, terr, model, s0, u,
                                                                 plant_dt=0.001, threads=4)
    assert rc == 0, err
    assert (fl == 0).all() and (loc < 0.01).all() and (esm >= 0).all()


def _device(p, heights, grid, model, s0, u, plant_heights=None):
    pl = PL.Planner(device=0, precision=_abi.PRECISION_FP64)
    pl.set_params(p)
    pl.set_terrain(PL.Heightmap(grid, heights))
    if plant_heights is not None:
        pl.set_plant_terrain(PL.Heightmap(grid, plant_heights))
    out = pl.open_loop_errors(model, s0, u, 0.001)
    pl.close()
    return out


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("name", ["c1", "c5"])
@pytest.mark.parametrize("model,scheme", [(_abi.MODEL_SRB, _abi.SCHEME_EULER),
                                          (_abi.MODEL_EST, _abi.SCHEME_EULER),
                                          (_abi.MODEL_SRB, _abi.SCHEME_RK4)])
def test_device_matches_reference(name, model, scheme):
    w, p, h, s0, u, terr, keep = _setup(name, n=48, N=80)
    p.scheme = scheme
    loc, esm, fl = _device(p, h, w.grid, model, s0, u)
    rc, rloc, resm, rfl, err = Oracle("reference").open_loop_errors(p, terr, model, s0, u,
                                                                    plant_dt=0.001, threads=16)
    assert rc == 0, err
    np.testing.assert_array_equal(fl, rfl)
    ok = fl == 0
    assert ok.mean() > 0.5
    np.testing.assert_allclose(loc[ok], rloc[ok], rtol=1e-7, atol=1e-10)
    np.testing.assert_allclose(esm[ok], resm[ok], rtol=1e-7, atol=1e-8)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("model", [_abi.MODEL_SRB, _abi.MODEL_EST])
def test_device_matches_reference_with_plant_lod(model):
    """The paper's setup: the model on a smoothed LOD of
    the terrain, the plant on the unsmoothed one (tmpc_set_plant_terrain)."""
    from paper_2603_20525_b200 import terrain as TR
    w, p, h, s0, u, terr, keep = _setup("c5", n=32, N=80)
    sigma = 0.3 if model == _abi.MODEL_SRB else 1.5
    lod = TR.gaussian_smooth(PL.Heightmap(w.grid, h), sigma).heights
    loc, esm, fl = _device(p, lod, w.grid, model, s0, u, plant_heights=h)
    t_lod, keep2 = PL.make_terrain(PL.Heightmap(w.grid, lod), None)
    rc, rloc, resm, rfl, err = Oracle("reference").open_loop_errors(
        p, t_lod, model, s0, u, plant_dt=0.001, threads=16, plant_terrain=terr)
    assert rc == 0, err
    np.testing.assert_array_equal(fl, rfl)
    ok = fl == 0
    np.testing.assert_allclose(loc[ok], rloc[ok], rtol=1e-7, atol=1e-10)
    np.testing.assert_allclose(esm[ok], resm[ok], rtol=1e-7, atol=1e-8)
    # the LOD gap makes the model differ from the plant
    assert np.median(loc[ok]) > 0


@pytest.mark.gpu
def test_device_self_comparison_is_zero():
    w, p, h, s0, u, terr, keep = _setup(n=8, N=20)
    p.scheme = _abi.SCHEME_RK4
    p.dt_int = 0.001
    loc, esm, fl = _device(p, h, w.grid, _abi.MODEL_SRB, s0, u)
    assert (fl == 0).all() and (loc == 0).all() and (esm == 0).all()


@pytest.mark.gpu
def test_device_needs_fp64_context():
    w = W.make_workload("c1").with_(n_steps=10)
    pl = PL.Planner(device=0)
    pl.set_params(w.params())
    pl.set_terrain(PL.Heightmap(w.grid, w.heights))
    with pytest.raises(PL.ConfigError):
        pl.open_loop_errors(_abi.MODEL_SRB, w.s0[None], np.zeros((1, 10, 2)))
    pl.close()
