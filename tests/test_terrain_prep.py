"""Terrain preprocessing and I/O: device gaussian_smooth /
build_sdist_map bit-identical to the reference (oracle/_ref), the heightmap
text format and the perimeter validation of terrain.hpp."""
import time

import numpy as np
import pytest

from oracle.oracle import Oracle
from paper_2603_20525_b200 import planner as PL
from paper_2603_20525_b200 import terrain as TR
from paper_2603_20525_b200 import workloads as W

HAVE_REF = Oracle.available("reference")
needs_ref = pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")


def _rough(n=96, res=0.1, seed=3, origin=(-4.8, -2.4)):
    rng = np.random.default_rng(seed)
    return PL.Heightmap(PL.GridSpec(origin[0], origin[1], res, n, n + 7),
                        rng.normal(0.0, 0.3, (n + 7, n)))


def _perimeters():
    ts = W.CONFIGS["c2"]["ts"]
    circles, off, verts = W.synth_obstacles(ts, (0.0, 0.0), 3.0)
    per = [TR.Perimeter(TR.PerimeterKind.OBSTACLE, verts[off[k]:off[k + 1]])
           for k in range(len(off) - 1)]
    # a corridor path boundary (violating outside) and a concave obstacle
    per.append(TR.Perimeter(TR.PerimeterKind.PATH_BOUNDARY,
                            np.array([[-24.0, -20.0], [24.0, -20.0], [24.0, 20.0], [-24.0, 20.0]])))
    per.append(TR.Perimeter(TR.PerimeterKind.OBSTACLE,
                            np.array([[5.0, 5.0], [9.0, 5.0], [9.0, 9.0], [7.0, 6.5], [5.0, 9.0]])))
    return per


# ------------------------------------------------------------------ host side
@needs_ref
@pytest.mark.parametrize("origin,res", [((-4.8, -2.4), 0.1), ((123.456789, -0.001), 0.25),
                                        ((0.0, 0.0), 1.0 / 3.0)])
def test_save_heightmap_matches_reference_text(tmp_path, origin, res):
    m = _rough(origin=origin, res=res)
    ours, theirs = tmp_path / "ours.txt", tmp_path / "ref.txt"
    TR.save_heightmap(m, ours)
    assert Oracle("reference").save_heightmap(m.heights, m.grid, theirs) == 0
    assert ours.read_text() == theirs.read_text()


@needs_ref
def test_load_heightmap_round_trip_and_reference(tmp_path):
    m = _rough()
    path = tmp_path / "t.txt"
    TR.save_heightmap(m, path)
    back = TR.load_heightmap(path)
    np.testing.assert_array_equal(back.heights, m.heights)  # %.17g round-trips exactly
    rc, err, hdr, h = Oracle("reference").load_heightmap(path)
    assert rc == 0
    np.testing.assert_array_equal(back.heights, h)
    assert (back.grid.origin_x, back.grid.origin_y, back.grid.resolution, back.grid.nx,
            back.grid.ny) == tuple(hdr[:3]) + (int(hdr[3]), int(hdr[4]))


BAD_FILES = {
    "header": "TERRAIN v2\n",
    "origin": "TERRAIN v1\norigin 1.0\n",
    "tag": "TERRAIN v1\norigen 1 2\n",
    "resolution": "TERRAIN v1\norigin 0 0\nresolution x\n",
    "size": "TERRAIN v1\norigin 0 0\nresolution 1\nsize 2\n",
    "small": "TERRAIN v1\norigin 0 0\nresolution 1\nsize 1 5\n",
    "short_row": "TERRAIN v1\norigin 0 0\nresolution 1\nsize 3 2\n1 2 3\n4 5\n",
    "eof": "TERRAIN v1\norigin 0 0\nresolution 1\nsize 2 3\n1 2\n3 4\n",
    "bad_res": "TERRAIN v1\norigin 0 0\nresolution -1\nsize 2 2\n1 2\n3 4\n",
}


@needs_ref
@pytest.mark.parametrize("case", sorted(BAD_FILES))
def test_load_heightmap_errors_match_reference(tmp_path, case):
    path = tmp_path / f"{case}.txt"
    path.write_text(BAD_FILES[case])
    with pytest.raises(PL.ConfigError) as ei:
        TR.load_heightmap(path)
    rc, err, _, _ = Oracle("reference").load_heightmap(path)
    assert rc == 2
    assert str(ei.value) == err


def test_perimeter_validation():
    TR.Perimeter(vertices=np.array([[0, 0], [1, 0], [0, 1.0]])).validate()
    for verts, msg in (([[0, 0], [1, 0]], "at least 3"),
                       ([[0, 0], [1, 0], [2, 0]], "zero area"),
                       ([[0, 0], [3, 3], [3, 0], [0, 1]], "self-intersecting")):
        with pytest.raises(PL.ConfigError, match=msg):
            TR.Perimeter(vertices=np.array(verts, dtype=float)).validate()


def test_device_preprocessing_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        TR.gaussian_smooth(_rough(), 0.3)
    with pytest.raises(RuntimeError):
        TR.build_sdist_map(PL.GridSpec(0, 0, 0.1, 16, 16), _perimeters()[:1])
    with pytest.raises(PL.ConfigError):  # validation precedes any device work
        TR.gaussian_smooth(_rough(), -1.0)


# ------------------------------------------------------------------ device
@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("sigma", [0.0, 0.05, 0.3, 1.5])
def test_gaussian_smooth_bit_identical(sigma):
    ref = Oracle("reference")
    for m in (_rough(), _rough(n=40, res=0.25, seed=9)):
        ours = TR.gaussian_smooth(m, sigma)
        rc, theirs = ref.gaussian_smooth(m.heights, m.grid, sigma)
        assert rc == 0
        np.testing.assert_array_equal(ours.heights, theirs)
    with pytest.raises(PL.ConfigError):
        TR.gaussian_smooth(_rough(), -0.1)


@pytest.mark.gpu
@needs_ref
def test_gaussian_smooth_lods_on_c2_terrain():
    w = W.make_workload("c2")
    ref = Oracle("reference")
    for sigma in (0.3, 1.5):  # the paper's planner LODs
        ours = TR.gaussian_smooth(PL.Heightmap(w.grid, w.heights), sigma)
        rc, theirs = ref.gaussian_smooth(w.heights, w.grid, sigma)
        np.testing.assert_array_equal(ours.heights, theirs)
        # smoothing keeps the mean and lowers the roughness
        assert abs(ours.heights.mean() - w.heights.mean()) < 1e-3
        assert np.abs(np.diff(ours.heights, axis=1)).mean() < np.abs(np.diff(w.heights, axis=1)).mean()


@pytest.mark.gpu
@needs_ref
def test_build_sdist_map_bit_identical():
    per = _perimeters()
    grid = PL.GridSpec(-25.6, -25.6, 0.1, 512, 512)
    ours = TR.build_sdist_map(grid, per)
    off, verts, kinds = TR.pack_perimeters(per)
    theirs = Oracle("reference").build_sdist_map(grid, off, verts, kinds)
    host = W.build_sdist(grid, off, verts, kinds)
    np.testing.assert_array_equal(ours.values, theirs)
    np.testing.assert_array_equal(ours.values, host)
    assert ours.has_features
    # inside the concave obstacle and outside the corridor are violating
    assert ours.values[int((7.0 + 25.6) / 0.1), int((8.5 + 25.6) / 0.1)] < 0
    assert (ours.values[:, 0] < 0).all()
    empty = TR.build_sdist_map(grid, [])
    assert not empty.has_features and np.isinf(empty.values).all()


@pytest.mark.gpu
def test_build_sdist_map_c4_scale_matches_host():
    """c4's map (2048^2 @ 0.1 m, 200 obstacles): device == exact host build."""
    ts = W.CONFIGS["c4"]["ts"]
    grid = PL.GridSpec(-102.4, -102.4, 0.1, 2048, 2048)
    circles, off, verts = W.synth_obstacles(ts, (0.0, 0.0), 3.0)
    per = [TR.Perimeter(TR.PerimeterKind.OBSTACLE, verts[off[k]:off[k + 1]])
           for k in range(len(off) - 1)]
    TR.build_sdist_map(PL.GridSpec(0, 0, 0.1, 8, 8), per)  # warm the context
    t0 = time.perf_counter()
    ours = TR.build_sdist_map(grid, per)
    t_dev = time.perf_counter() - t0
    t0 = time.perf_counter()
    host = W.build_sdist(grid, off, verts)
    t_host = time.perf_counter() - t0
    np.testing.assert_array_equal(ours.values, host)
    print(f"c4 sdist build: device {t_dev * 1e3:.1f} ms (incl. copies), host {t_host * 1e3:.1f} ms")
