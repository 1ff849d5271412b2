"""Host-side mirror of the reference planner interface, over libtmpc_b200.so.

Reference types keep their names, fields and defaults:
  VehicleParams / TireParams        dynamics.hpp:20-58
  SrbState / Control / ControlSequence   dynamics.hpp:130-183
  GridSpec / Heightmap / SignedDistanceMap   terrain.hpp:20-75,230-239
  ConstraintConfig                  constraints.hpp:42-58
  ConfigError / NumericError        errors.hpp:8-18
SPEC-only planner types and entry points (absent from the reference code):
  CostWeights, Goal, PlannerConfig, RolloutResult, SolverStats
  solve_ocp(...)  SPEC.md:384-390     plan_step(...)

Everything from "parallel over candidates" to the arg-min runs in the CUDA
kernel behind the C ABI; this module only validates, marshals and unpacks.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _abi
from ._abi import (FLAG_DIVERGED, FLAG_FEASIBLE, FLAG_GOAL, SAMPLE_RANDOM_WALK,
                   SAMPLE_UNIFORM, SAMPLE_WARM_GAUSS, SELECT_FEASIBLE_FIRST, SELECT_PLAIN,
                   STATE_DIM, TMPC_ERR_CONFIG, TMPC_ERR_NUMERIC, TMPC_OK)

__all__ = [
    "ConfigError", "NumericError", "VehicleParams", "TireParams", "ConstraintConfig",
    "CostWeights", "Goal", "PlannerConfig", "SrbState", "Control", "ControlSequence", "GridSpec",
    "Heightmap", "SignedDistanceMap", "RolloutResult", "SolverStats", "Planner", "solve_ocp",
    "plan_step", "esm", "esm_normalization", "load_transfer_coeffs",
]


# --------------------------------------------------------------------- errors
class ConfigError(RuntimeError):
    """Invalid configuration (errors.hpp:9-12); CLI exit code 2."""


class NumericError(RuntimeError):
    """Numerical failure, e.g. every rollout diverged (errors.hpp:15-18); exit code 1."""


def _raise(rc: int, msg: str):
    if rc == TMPC_OK:
        return
    if rc == TMPC_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == TMPC_ERR_NUMERIC:
        raise NumericError(msg)
    raise RuntimeError(msg)


# --------------------------------------------------------------------- params
@dataclass
class VehicleParams:
    """dynamics.hpp:20-36 (Appendix-B full-scale test vehicle)."""
    M: float = 969.0
    J_xx: float = 280.9
    J_yy: float = 692.1
    J_zz: float = 810.7
    L_f: float = 1.565
    L_r: float = 1.148
    e: float = 1.280
    h: float = 0.380
    R: float = 0.291
    k_f: float = 4.2e4
    k_r: float = 5.8e4
    b_f: float = 3.1e3
    b_r: float = 4.3e3
    delta_max: float = 0.639
    delta_rate_max: float = 1.0
    g: float = 9.81


@dataclass
class TireParams:
    """dynamics.hpp:50-52."""
    C: float = 6.1
    mu: float = 0.6


@dataclass
class ConstraintConfig:
    """constraints.hpp:42-49.  esm_nominal=None => esm_normalization(vp)."""
    a_by_bar: float = 5.0
    esm_nominal: Optional[float] = None
    eps_dist: float = 0.25
    sigma: float = 1e6
    safety_factor: float = 0.10
    enable_dist: bool = True
    enable_rollover: bool = True


@dataclass
class CostWeights:
    """SPEC.md:349 / PAPER.md:880-883."""
    w_t: float = 5.0
    w_c: float = 8.0
    w_g: float = 15.0


@dataclass
class Goal:
    """SPEC.md:357 / PAPER.md:983-989."""
    x_g: float = 0.0
    y_g: float = 0.0
    r_g: float = 2.5


@dataclass
class PlannerConfig:
    """SPEC.md:360-363 plus the sampler/selection extensions of SURVEY App. A.

    n_steps ZOH segments of dt_zoh, each integrated with dt_zoh/dt_int forward
    Euler substeps (decision D1: BASELINE's dt=0.05 s is the ZOH period)."""
    n_samples: int = 1024
    seed: int = 0
    n_steps: int = 16
    dt_zoh: float = 0.25
    dt_int: float = 0.005
    sampler: int = SAMPLE_UNIFORM
    vdot_max: float = 0.0
    walk_step: float = 0.25
    warm_sigma_frac: float = 0.10
    selection: int = SELECT_FEASIBLE_FIRST
    model: int = _abi.MODEL_SRB
    scheme: int = _abi.SCHEME_EULER


@dataclass
class SrbState:
    """dynamics.hpp:167-183, 3-2-1 angles, body-frame velocities."""
    x: float = 0.0
    y: float = 0.0
    z: float = 0.0
    psi: float = 0.0
    theta: float = 0.0
    phi: float = 0.0
    v_bx: float = 0.0
    v_by: float = 0.0
    v_bz: float = 0.0
    omega_bx: float = 0.0
    omega_by: float = 0.0
    omega_bz: float = 0.0
    delta: float = 0.0

    def as_array(self) -> np.ndarray:
        return np.array([self.x, self.y, self.z, self.psi, self.theta, self.phi, self.v_bx,
                         self.v_by, self.v_bz, self.omega_bx, self.omega_by, self.omega_bz,
                         self.delta], dtype=np.float64)

    @staticmethod
    def from_array(a) -> "SrbState":
        return SrbState(*[float(v) for v in a])


@dataclass
class Control:
    """dynamics.hpp:130-133."""
    delta_rate: float = 0.0
    v_bx_rate: float = 0.0


@dataclass
class ControlSequence:
    """dynamics.hpp:135-145."""
    entries: list = field(default_factory=list)
    dt_zoh: float = 0.25

    def horizon(self) -> float:
        return self.dt_zoh * len(self.entries)

    def as_array(self) -> np.ndarray:
        return np.array([[c.delta_rate, c.v_bx_rate] for c in self.entries], dtype=np.float64)


@dataclass
class GridSpec:
    """terrain.hpp:20-29."""
    origin_x: float = 0.0
    origin_y: float = 0.0
    resolution: float = 1.0
    nx: int = 0
    ny: int = 0


@dataclass
class Heightmap:
    """terrain.hpp:56-75; heights[j, i] (row-major, j indexes y)."""
    grid: GridSpec
    heights: np.ndarray


@dataclass
class SignedDistanceMap:
    """terrain.hpp:230-239."""
    grid: GridSpec
    values: Optional[np.ndarray] = None
    has_features: bool = False


@dataclass
class RolloutResult:
    """SPEC.md:365-367 (the winner's total cost and flags)."""
    cost: float
    feasible: bool
    margin: float
    index: int


@dataclass
class SolverStats:
    """min/mean cost and rollout throughput (+ counts)."""
    best_cost: float
    min_cost: float
    mean_cost: float
    n_samples: int
    n_feasible: int
    n_diverged: int
    n_goal: int
    substeps_executed: int
    kernel_ms: float
    cycle_ms: float

    @property
    def rollouts_per_s(self) -> float:
        return self.n_samples / (self.cycle_ms * 1e-3) if self.cycle_ms > 0 else float("inf")


# --------------------------------------------------------------------- helpers
def load_transfer_coeffs(vp: VehicleParams):
    """dynamics.hpp:67-71 -> (K_zzf, K_zzr, K_zx, K_zy)."""
    L = vp.L_f + vp.L_r
    return (vp.M * vp.L_r / L, vp.M * vp.L_f / L, vp.M * (vp.h + vp.R) / L,
            vp.M * (vp.h + vp.R) / vp.e)


def esm(phi: float, theta: float, vp: VehicleParams) -> float:
    """constraints.hpp:16-23."""
    r_bar = math.hypot(vp.h + vp.R, vp.e / 2.0)
    phi_bar = math.atan(2.0 * (vp.h + vp.R) / vp.e)
    lever = abs(phi) + phi_bar
    dh = r_bar * (1.0 - math.sin(lever)) * math.cos(theta)
    return (1.0 if lever <= math.pi / 2.0 else -1.0) * vp.M * vp.g * dh


def esm_normalization(vp: VehicleParams) -> float:
    """constraints.hpp:26-28."""
    return esm(0.0, 0.0, vp)


def make_params(vp: VehicleParams, tp: TireParams, cc: ConstraintConfig, w: CostWeights,
                goal: Goal, cfg: PlannerConfig) -> _abi.tmpc_params:
    p = _abi.tmpc_params()
    for k in ("M", "J_xx", "J_yy", "J_zz", "L_f", "L_r", "e", "h", "R", "k_f", "k_r", "b_f",
              "b_r", "delta_max", "delta_rate_max", "g"):
        setattr(p, k, float(getattr(vp, k)))
    p.C, p.mu = float(tp.C), float(tp.mu)
    p.a_by_bar = cc.a_by_bar
    p.esm_nominal = esm_normalization(vp) if cc.esm_nominal is None else float(cc.esm_nominal)
    p.eps_dist, p.sigma, p.safety_factor = cc.eps_dist, cc.sigma, cc.safety_factor
    p.enable_dist, p.enable_rollover = int(cc.enable_dist), int(cc.enable_rollover)
    p.w_t, p.w_c, p.w_g = w.w_t, w.w_c, w.w_g
    p.goal_x, p.goal_y, p.goal_r = goal.x_g, goal.y_g, goal.r_g
    p.dt_zoh, p.dt_int = cfg.dt_zoh, cfg.dt_int
    p.n_steps, p.selection = int(cfg.n_steps), int(cfg.selection)
    p.model = int(cfg.model)
    p.scheme = int(cfg.scheme)
    return p


def make_sampling(cfg: PlannerConfig, k_begin: int = 0, k_count: Optional[int] = None,
                  warm_seq: Optional[np.ndarray] = None):
    s = _abi.tmpc_sampling()
    s.kind, s.seed = int(cfg.sampler), int(cfg.seed) & 0xFFFFFFFFFFFFFFFF
    s.vdot_max, s.walk_step, s.warm_sigma_frac = cfg.vdot_max, cfg.walk_step, cfg.warm_sigma_frac
    s.k_begin = int(k_begin)
    s.k_count = int(cfg.n_samples if k_count is None else k_count)
    # the whole problem's size picks the lane layout (bitwise G-independent)
    s.k_total = max(int(cfg.n_samples), int(s.k_begin + s.k_count))
    keep = None
    if warm_seq is not None:
        keep = np.ascontiguousarray(warm_seq, dtype=np.float64).reshape(-1)
        s.warm_seq = _abi.dptr(keep)
    return s, keep


def make_terrain(hm: Heightmap, sd: Optional[SignedDistanceMap]):
    h = np.ascontiguousarray(hm.heights, dtype=np.float64)
    t = _abi.tmpc_terrain()
    t.heights = _abi.dptr(h)
    sv = None
    if sd is not None and sd.has_features:
        if (sd.grid.nx, sd.grid.ny) != (hm.grid.nx, hm.grid.ny):
            raise ConfigError("sdist grid must match the heightmap grid")
        sv = np.ascontiguousarray(sd.values, dtype=np.float64)
        t.sdist = _abi.dptr(sv)
    t.nx, t.ny = int(hm.grid.nx), int(hm.grid.ny)
    t.origin_x, t.origin_y, t.resolution = hm.grid.origin_x, hm.grid.origin_y, hm.grid.resolution
    if h.shape != (t.ny, t.nx):
        raise ConfigError("heightmap: height count does not match grid size")
    return t, (h, sv)


def make_record(cost, flags, margin, k_begin: int, selection: int = SELECT_FEASIBLE_FIRST,
                substeps=None) -> _abi.tmpc_rank_record:
    """Host mirror of one GPU's reduction of its shard (tmpc_make_record)."""
    lib = _abi.load()
    cost = np.ascontiguousarray(cost, dtype=np.float64)
    flags = np.ascontiguousarray(flags, dtype=np.uint8)
    margin = np.ascontiguousarray(margin, dtype=np.float32)
    sub = None if substeps is None else np.ascontiguousarray(substeps, dtype=np.int64)
    r = _abi.tmpc_rank_record()
    rc = lib.tmpc_make_record(_abi.dptr(cost), flags.ctypes.data_as(C.POINTER(C.c_uint8)),
                              margin.ctypes.data_as(C.POINTER(C.c_float)),
                              None if sub is None else sub.ctypes.data_as(C.POINTER(C.c_int64)),
                              int(k_begin), len(cost), int(selection), C.byref(r))
    _raise(rc, lib.tmpc_last_error(None).decode())
    return r


def fold_records(records) -> _abi.tmpc_result:
    """Fold per-GPU / per-rank records in order (tmpc_fold_records): the
    cross-GPU arg-min and stats of one cycle.  Raises NumericError when every
    candidate diverged."""
    lib = _abi.load()
    arr = (_abi.tmpc_rank_record * len(records))(*records)
    out = _abi.tmpc_result()
    rc = lib.tmpc_fold_records(arr, len(records), C.byref(out))
    _raise(rc, lib.tmpc_last_error(None).decode())
    return out


def record_bytes(r: _abi.tmpc_rank_record) -> bytes:
    return bytes(r)


def record_from_bytes(b: bytes) -> _abi.tmpc_rank_record:
    return _abi.tmpc_rank_record.from_buffer_copy(b)


def shard_range(n: int, rank: int, world: int):
    """Contiguous global index range of `rank`."""
    base, rem = divmod(n, world)
    begin = rank * base + min(rank, rem)
    return begin, base + (1 if rank < rem else 0)


# --------------------------------------------------------------------- planner
class Planner:
    """One planning problem (a tmpc_ctx) on one GPU, or on several GPUs from
    this one process (`devices=[0, 1, ...]`: the library splits each cycle's
    candidates over them and folds the per-GPU arg-min records).

    Terrain and parameters are uploaded once and stay resident in HBM (one
    replica per GPU); each solve() is one planning cycle (solve_ocp,
    SPEC.md:384-390)."""

    def __init__(self, device: int = 0, rank: int = 0, world_size: int = 1, k_max: int = 0,
                 n_steps_max: int = 0, nccl_id: Optional[bytes] = None,
                 precision: int = _abi.PRECISION_FP32, lanes: int = 0,
                 ordering: int = _abi.ORDER_AUTO, devices=None, timeout_ms: int = 0,
                 graphs: int = _abi.GRAPHS_AUTO, exchange: int = _abi.EXCHANGE_NCCL):
        self.lib = _abi.load()
        o = _abi.tmpc_opts()
        o.device, o.rank, o.world_size, o.lanes = device, rank, world_size, lanes
        o.ordering = ordering
        o.k_max, o.n_steps_max, o.precision = k_max, n_steps_max, precision
        o.timeout_ms, o.graphs, o.exchange = int(timeout_ms), int(graphs), int(exchange)
        self._devs = None
        if devices is not None:
            self._devs = (C.c_int32 * len(devices))(*[int(d) for d in devices])
            o.n_devices = len(devices)
            o.devices = C.cast(self._devs, C.POINTER(C.c_int32))
        self._nid = None
        if nccl_id is not None:
            self._nid = C.create_string_buffer(bytes(nccl_id), 128)
            o.nccl_id = C.cast(self._nid, C.c_void_p)
        h = C.c_void_p()
        rc = self.lib.tmpc_ctx_create(C.byref(o), C.byref(h))
        _raise(rc, self.lib.tmpc_last_error(None).decode())
        self.ctx = h
        self.rank, self.world_size = rank, world_size
        self._params = None
        self._io = None  # (s0, its pointer, controls, their pointer) of solve_raw

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.tmpc_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _err(self) -> str:
        return self.lib.tmpc_last_error(self.ctx).decode()

    def peer_export(self) -> bytes:
        """This rank's mailbox as a 64-byte CUDA IPC handle (EXCHANGE_PEER)."""
        buf = C.create_string_buffer(64)
        _raise(self.lib.tmpc_peer_export(self.ctx, buf), self._err())
        return buf.raw

    def peer_connect(self, handles):
        """Every rank's handle, rank order (EXCHANGE_PEER): from now on the
        rollout kernel exchanges the per-GPU records over peer memory."""
        blob = b"".join(bytes(h) for h in handles)
        _raise(self.lib.tmpc_peer_connect(self.ctx, blob, len(handles)), self._err())

    def peer_inspect(self, src_rank: int, seq: int):
        """(record rank src_rank stored in this rank's mailbox for sequence
        number seq, the sequence number src_rank last published)."""
        rec = _abi.tmpc_rank_record()
        pub = C.c_uint64()
        _raise(self.lib.tmpc_peer_inspect(self.ctx, src_rank, seq, C.byref(rec), C.byref(pub)),
               self._err())
        return rec, int(pub.value)

    @property
    def n_devices(self) -> int:
        return int(self.lib.tmpc_num_devices(self.ctx))

    def device_stream(self, i: int = 0):
        """cudaStream_t of the context's i-th GPU (event timing)."""
        return self.lib.tmpc_get_device_stream(self.ctx, i)

    def device_ordinal(self, i: int = 0) -> int:
        return int(self.lib.tmpc_get_device_ordinal(self.ctx, i))

    def set_params(self, p: _abi.tmpc_params):
        _raise(self.lib.tmpc_set_params(self.ctx, C.byref(p)), self._err())
        self._params = p

    def set_terrain(self, hm: Heightmap, sd: Optional[SignedDistanceMap] = None):
        t, _keep = make_terrain(hm, sd)
        _raise(self.lib.tmpc_set_terrain(self.ctx, C.byref(t)), self._err())

    def set_terrain_arrays(self, heights, sdist, grid: GridSpec):
        self.set_terrain(Heightmap(grid, heights),
                         None if sdist is None else SignedDistanceMap(grid, sdist, True))

    def solve_raw(self, s0: np.ndarray, smp: _abi.tmpc_sampling, want_controls: bool = True):
        # the state and controls go through buffers owned by the planner whose
        # ctypes pointers are built once (numpy's data_as costs ~3 us a call,
        # a tenth of the per-cycle host overhead); the controls are returned
        # as a copy
        buf = self._io
        if buf is None or buf[2].shape[0] != self._params.n_steps:
            s0b, ctrl = np.zeros(STATE_DIM), np.zeros((self._params.n_steps, 2))
            buf = self._io = (s0b, _abi.dptr(s0b), ctrl, _abi.dptr(ctrl))
        s0b, s0p, ctrl, ctrlp = buf
        s0 = np.asarray(s0, dtype=np.float64)
        if s0.shape != (STATE_DIM,):
            raise ConfigError("state must have 13 entries")
        s0b[:] = s0
        res = _abi.tmpc_result()
        rc = self.lib.tmpc_solve(self.ctx, s0p, C.byref(smp), C.byref(res),
                                 ctrlp if want_controls else None)
        _raise(rc, self._err())
        return res, (ctrl.copy() if want_controls else None)

    def set_plant_terrain(self, hm: Optional[Heightmap]):
        """The plant LOD of open_loop_errors (same grid as the terrain); None =
        the planning terrain (tmpc_set_plant_terrain)."""
        if hm is None:
            _raise(self.lib.tmpc_set_plant_terrain(self.ctx, None), self._err())
            return
        t, keep = make_terrain(hm, None)
        _raise(self.lib.tmpc_set_plant_terrain(self.ctx, C.byref(t)), self._err())

    def open_loop_errors(self, model: int, s0, controls, plant_dt: float = 0.001):
        """open_loop_errors: for each trajectory (initial
        state s0[t], ZOH controls[t] of n_steps x 2) the time-averaged
        location error and |ESM error| of `model` (MODEL_SRB / MODEL_EST, the
        params' scheme at dt_int) against the SRB RK4 plant at plant_dt.
        Needs a PRECISION_FP64 planner.  Returns (loc, esm, flags); flags 1 =
        model diverged, 2 = plant diverged (errors NaN)."""
        s0 = np.ascontiguousarray(s0, dtype=np.float64).reshape(-1, STATE_DIM)
        n = len(s0)
        u = np.ascontiguousarray(controls, dtype=np.float64).reshape(n, -1, 2)
        if self._params is None or u.shape[1] != self._params.n_steps:
            raise ConfigError("open_loop_errors: controls must be n_traj x n_steps x 2")
        loc, esm_e, fl = np.empty(n), np.empty(n), np.empty(n, dtype=np.uint8)
        rc = self.lib.tmpc_open_loop_errors(self.ctx, int(model), _abi.dptr(s0), _abi.dptr(u), n,
                                            float(plant_dt), _abi.dptr(loc), _abi.dptr(esm_e),
                                            fl.ctypes.data_as(C.POINTER(C.c_uint8)))
        _raise(rc, self._err())
        return loc, esm_e, fl

    def costs(self, k_count: int):
        cost = np.empty(k_count, dtype=np.float64)
        flags = np.empty(k_count, dtype=np.uint8)
        margin = np.empty(k_count, dtype=np.float32)
        rc = self.lib.tmpc_get_costs(self.ctx, _abi.dptr(cost),
                                     flags.ctypes.data_as(C.POINTER(C.c_uint8)),
                                     margin.ctypes.data_as(C.POINTER(C.c_float)))
        _raise(rc, self._err())
        return cost, flags, margin

    def solve(self, state: SrbState, goal: Goal, cfg: PlannerConfig,
              weights: CostWeights = CostWeights(), cc: ConstraintConfig = ConstraintConfig(),
              vp: VehicleParams = VehicleParams(), tp: TireParams = TireParams(),
              warm_seq: Optional[np.ndarray] = None):
        """solve_ocp -> (ControlSequence, RolloutResult, SolverStats)."""
        self.set_params(make_params(vp, tp, cc, weights, goal, cfg))
        k0, kc = shard_range(cfg.n_samples, self.rank, self.world_size)
        smp, _keep = make_sampling(cfg, k0, kc, warm_seq)
        res, ctrl = self.solve_raw(state.as_array(), smp)
        seq = ControlSequence([Control(float(a), float(b)) for a, b in ctrl], cfg.dt_zoh)
        rr = RolloutResult(res.best_cost, bool(res.best_feasible), res.best_margin,
                           int(res.best_index))
        st = SolverStats(res.best_cost, res.min_cost, res.mean_cost, int(res.n_candidates),
                         int(res.n_feasible), int(res.n_diverged), int(res.n_goal),
                         int(res.substeps_executed), res.kernel_ms, res.cycle_ms)
        return seq, rr, st


def solve_ocp(state: SrbState, terrain: Heightmap, sdmap: Optional[SignedDistanceMap],
              goal: Goal, cfg: PlannerConfig, weights: CostWeights = CostWeights(),
              cc: ConstraintConfig = ConstraintConfig(), vp: VehicleParams = VehicleParams(),
              tp: TireParams = TireParams(), device: int = 0, warm_seq=None,
              precision: int = _abi.PRECISION_FP32):
    """One-shot solve_ocp.  For repeated cycles keep a Planner."""
    pl = Planner(device=device, k_max=cfg.n_samples, n_steps_max=cfg.n_steps,
                 precision=precision)
    try:
        pl.set_params(make_params(vp, tp, cc, weights, goal, cfg))
        pl.set_terrain(terrain, sdmap)
        return pl.solve(state, goal, cfg, weights, cc, vp, tp, warm_seq)
    finally:
        pl.close()


def plan_step(planner: Planner, state: SrbState, goal: Goal, cfg: PlannerConfig, **kw) -> Control:
    """plan_step: the first ZOH control of the best sequence."""
    seq, _, _ = planner.solve(state, goal, cfg, **kw)
    return seq.entries[0]
