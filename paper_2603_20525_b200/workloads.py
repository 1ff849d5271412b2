"""Seeded synthetic stand-ins for BASELINE.json configs c1-c5.

The reference publishes no dataset for this path; BASELINE.json describes
the workloads in words and SURVEY App. A (D3-D6, D11) lists what it leaves
open.  Every declared choice is here, in one place, shared by the device
path, the oracle parity tests and bench.py.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import math
from dataclasses import dataclass, field, replace
from typing import Optional

import numpy as np

from . import _abi
from .planner import (SAMPLE_RANDOM_WALK, SAMPLE_UNIFORM, SAMPLE_WARM_GAUSS, ConfigError,
                      ConstraintConfig, CostWeights, Goal, GridSpec, PlannerConfig, TireParams,
                      VehicleParams, make_params)

DT_ZOH = 0.05   # BASELINE dt = ZOH control period (D1)
DT_INT = 0.005  # forward-Euler substep, PAPER.md:1065 / SPEC.md:361


@dataclass
class TerrainSpec:
    n: int
    res: float
    seed: int
    sine_amp: float = 0.0
    sine_wavelength: float = 8.0
    noise_amp: float = 0.0
    fractal_octaves: int = 0
    fractal_persistence: float = 0.5
    fractal_lattice: float = 6.4
    fractal_pp: float = 0.0
    slope_deg: float = 0.0
    slope_period: float = 6.0
    slope_dir: float = math.pi / 4
    n_berms: int = 0
    berm_height: float = 0.4
    berm_length: float = 4.0
    berm_halfwidth: float = 0.5
    n_obstacles: int = 0
    obstacle_rmin: float = 0.5
    obstacle_rmax: float = 1.5
    obstacle_ngon: int = 32
    obstacle_stamp: float = 0.0  # height added inside obstacles (D5), 0 = SDF only


@dataclass
class Workload:
    name: str
    cfg: PlannerConfig
    goal: Goal
    grid: GridSpec
    heights: np.ndarray
    sdist: Optional[np.ndarray]
    s0: np.ndarray
    v0: float
    polys: Optional[tuple] = None  # (poly_off int32, verts float64)
    vp: VehicleParams = field(default_factory=VehicleParams)
    tp: TireParams = field(default_factory=TireParams)
    cc: ConstraintConfig = field(default_factory=ConstraintConfig)
    w: CostWeights = field(default_factory=CostWeights)

    def params(self) -> _abi.tmpc_params:
        return make_params(self.vp, self.tp, self.cc, self.w, self.goal, self.cfg)

    def terrain_digest(self) -> str:
        h = hashlib.sha256(np.ascontiguousarray(self.heights).tobytes())
        if self.sdist is not None:
            h.update(np.ascontiguousarray(self.sdist).tobytes())
        return h.hexdigest()[:16]

    def label(self) -> str:
        """The workload string both bench.py arms print (config.workload)."""
        n_obs = 0 if self.polys is None else len(self.polys[0]) - 1
        return (f"{self.name}: K={self.cfg.n_samples} N={self.cfg.n_steps} S=10 "
                f"grid={self.grid.nx}^2 obstacles={n_obs} v0={self.v0} m/s "
                f"terrain={self.terrain_digest()}")

    def with_(self, **kw) -> "Workload":
        """Copy with PlannerConfig fields replaced (n_samples, n_steps, ...)."""
        return replace(self, cfg=replace(self.cfg, **kw))


def synth_terrain(ts: TerrainSpec, lib=None):
    lib = lib or _abi.load()
    s = _abi.tmpc_synth_spec()
    s.nx = s.ny = ts.n
    s.origin_x = s.origin_y = 0.0
    s.resolution = ts.res
    s.seed = ts.seed
    for k in ("sine_amp", "sine_wavelength", "noise_amp", "fractal_octaves",
              "fractal_persistence", "fractal_lattice", "fractal_pp", "slope_deg",
              "slope_period", "slope_dir", "n_berms", "berm_height", "berm_length",
              "berm_halfwidth"):
        setattr(s, k, getattr(ts, k))
    h = np.zeros((ts.n, ts.n), dtype=np.float64)
    rc = lib.tmpc_synth_heightmap(C.byref(s), _abi.dptr(h))
    if rc:
        raise ConfigError("synth_heightmap: bad spec")
    return h


def synth_obstacles(ts: TerrainSpec, clear_xy, clear_r: float, lib=None):
    lib = lib or _abi.load()
    o = _abi.tmpc_obstacle_spec()
    o.seed, o.n, o.n_gon = ts.seed, ts.n_obstacles, ts.obstacle_ngon
    o.r_min, o.r_max = ts.obstacle_rmin, ts.obstacle_rmax
    ext = ts.res * (ts.n - 1)
    o.x_min, o.x_max, o.y_min, o.y_max = 1.0, ext - 1.0, 1.0, ext - 1.0
    o.clear_x, o.clear_y, o.clear_r = clear_xy[0], clear_xy[1], clear_r
    circles = np.zeros((ts.n_obstacles, 3))
    verts = np.zeros((ts.n_obstacles * ts.obstacle_ngon, 2))
    if lib.tmpc_synth_obstacles(C.byref(o), _abi.dptr(circles), _abi.dptr(verts)):
        raise ConfigError("synth_obstacles: bad spec")
    off = (np.arange(ts.n_obstacles + 1) * ts.obstacle_ngon).astype(np.int32)
    return circles, off, verts


def build_sdist(grid: GridSpec, off: np.ndarray, verts: np.ndarray, kinds=None, threads=0,
                lib=None):
    """build_sdist_map (terrain.hpp:241-260), exact, host."""
    lib = lib or _abi.load()
    n_poly = len(off) - 1
    if kinds is None:
        kinds = np.zeros(n_poly, dtype=np.int32)
    out = np.zeros((grid.ny, grid.nx))
    rc = lib.tmpc_build_sdist_map(grid.nx, grid.ny, grid.origin_x, grid.origin_y,
                                  grid.resolution, n_poly,
                                  off.ctypes.data_as(C.POINTER(C.c_int32)),
                                  _abi.dptr(np.ascontiguousarray(verts, dtype=np.float64)),
                                  np.ascontiguousarray(kinds, dtype=np.int32).ctypes.data_as(
                                      C.POINTER(C.c_int32)),
                                  _abi.dptr(out), threads)
    if rc:
        raise ConfigError("build_sdist_map failed")
    return out


def initial_state(heights, grid: GridSpec, x0: float, y0: float, v0: float, psi0=0.0,
                  vp: VehicleParams = VehicleParams()):
    """D11: z = h(x0, y0) + h + R, level attitude, body speed v0 along psi0."""
    gx = (x0 - grid.origin_x) / grid.resolution
    gy = (y0 - grid.origin_y) / grid.resolution
    i0, j0 = min(int(gx), grid.nx - 2), min(int(gy), grid.ny - 2)
    fx, fy = gx - i0, gy - j0
    a = heights[j0, i0] + fx * (heights[j0, i0 + 1] - heights[j0, i0])
    b = heights[j0 + 1, i0] + fx * (heights[j0 + 1, i0 + 1] - heights[j0 + 1, i0])
    hz = a + fy * (b - a)
    s0 = np.zeros(13)
    s0[0], s0[1], s0[2], s0[3], s0[6] = x0, y0, hz + vp.h + vp.R, psi0, v0
    return s0


# (terrain spec, K, N, v0, start (fraction of extent), sampler) per config.
CONFIGS = {
    # c1: 256^2 @ 0.2 m sinusoid (0.3 m, 8 m) + U(+-0.05); grid centre; 5 m/s; iid uniform
    "c1": dict(ts=TerrainSpec(256, 0.2, 1001, sine_amp=0.3, sine_wavelength=8.0, noise_amp=0.05),
               K=1024, N=50, v0=5.0, start=(0.5, 0.5), sampler=SAMPLE_UNIFORM),
    # c2: 512^2 @ 0.1 m value-noise fractal (4 oct, p 0.5, 1.0 m p-p) + 20 cylinders;
    #     10 m/s; random walk
    "c2": dict(ts=TerrainSpec(512, 0.1, 2002, fractal_octaves=4, fractal_pp=1.0,
                              n_obstacles=20),
               K=16384, N=100, v0=10.0, start=(0.1, 0.5), sampler=SAMPLE_RANDOM_WALK),
    # c3: 512^2 @ 0.1 m +-15 deg side slopes (sinusoid, 6 m period across the direction of
    #     travel) + 12 berms 0.4 m high / 3 m wide; 15 m/s; iid uniform.  Calibrated with
    #     the oracle: ~35% infeasible (BASELINE asks 30-60%), ~17% of those roll over.
    "c3": dict(ts=TerrainSpec(512, 0.1, 3003, slope_deg=15.0, slope_period=6.0,
                              slope_dir=math.pi / 2, n_berms=12, berm_height=0.4,
                              berm_halfwidth=1.5),
               K=65536, N=100, v0=15.0, start=(0.1, 0.5), sampler=SAMPLE_UNIFORM),
    # c4: 2048^2 @ 0.1 m fractal (2.0 m p-p) + 200 cylinders; 10 m/s; iid uniform.
    #     Obstacles keep 10 m clear of the start: with the default 4 m one cylinder
    #     sits 8.5 m dead ahead, inside the 0.85 s no candidate can steer around,
    #     and every candidate is infeasible (oracle, 512 candidates: 0 -> 45% feasible)
    "c4": dict(ts=TerrainSpec(2048, 0.1, 4004, fractal_octaves=4, fractal_pp=2.0,
                              fractal_lattice=12.8, n_obstacles=200),
               K=262144, N=100, v0=10.0, start=(0.1, 0.5), sampler=SAMPLE_UNIFORM,
               clear_r=10.0),
    # c5: 1024^2 @ 0.1 m fractal + side slopes; 8 m/s; warm-started Gaussian; the goal
    #     85 m ahead (200 cycles x 0.05 s x 8 m/s = 80 m of closed-loop driving)
    "c5": dict(ts=TerrainSpec(1024, 0.1, 5005, fractal_octaves=4, fractal_pp=1.0,
                              slope_deg=10.0, slope_period=8.0, slope_dir=math.pi / 2),
               K=131072, N=100, v0=8.0, start=(0.1, 0.5), sampler=SAMPLE_WARM_GAUSS,
               goal_dist=85.0),
}
GOAL_FRACTION = 1.0   # D3: goal v0 * horizon ahead along psi0
CLEAR_RADIUS = 4.0    # obstacle keep-out around the start (D5)
WALK_STEP = 0.25      # D6: random-walk increment bound, rad/s per step


def make_workload(name: str, seed: int = 12345, lib=None, **overrides) -> Workload:
    """The seeded inputs of BASELINE config `name`.  `lib`: the library whose
    generators (tmpc_synth_heightmap / _obstacles / tmpc_build_sdist_map, the
    same synth.cpp source) build them -- libtmpc_b200.so by default; the
    reference arm of bench.py passes oracle/libworkload.so so that it never
    loads the product."""
    spec = dict(CONFIGS[name])
    spec.update(overrides)
    ts: TerrainSpec = spec["ts"]
    grid = GridSpec(0.0, 0.0, ts.res, ts.n, ts.n)
    ext = ts.res * (ts.n - 1)
    x0, y0 = spec["start"][0] * ext, spec["start"][1] * ext
    heights = synth_terrain(ts, lib)
    sdist, polys = None, None
    if ts.n_obstacles:
        _, off, verts = synth_obstacles(ts, (x0, y0), spec.get("clear_r", CLEAR_RADIUS), lib)
        polys = (off, verts)
        if ts.obstacle_stamp:
            t = _abi.tmpc_terrain()
            t.nx, t.ny, t.resolution = ts.n, ts.n, ts.res
            (lib or _abi.load()).tmpc_stamp_obstacles(C.byref(t), _abi.dptr(heights), len(off) - 1,
                                             off.ctypes.data_as(C.POINTER(C.c_int32)),
                                             _abi.dptr(verts), ts.obstacle_stamp)
        sdist = build_sdist(grid, off, verts, lib=lib)
    v0 = spec["v0"]
    N = spec["N"]
    s0 = initial_state(heights, grid, x0, y0, v0)
    dist = spec.get("goal_dist", GOAL_FRACTION * v0 * N * DT_ZOH)
    goal = Goal(x0 + dist, y0, 2.5)
    cfg = PlannerConfig(n_samples=spec["K"], seed=seed, n_steps=N, dt_zoh=DT_ZOH, dt_int=DT_INT,
                        sampler=spec["sampler"], walk_step=WALK_STEP, warm_sigma_frac=0.10)
    return Workload(name, cfg, goal, grid, heights, sdist, s0, v0, polys)
