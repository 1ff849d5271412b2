"""Closed-loop receding-horizon driver (BASELINE c5).

Every planning period the planner solves the OCP from the current plant
state (`plan_step`), the first ZOH control of the winner is
applied, and the plant — the reference SRB model integrated with RK4 at 1 ms
(`tmpc_plant_step`) — advances the state by one period.
Candidates of the next cycle are seeded around the previous winner, shifted
by one step (warm start; the reference planner has none,
SPEC.md:410).  The trial ends on goal acquisition, rollover
(|roll| or |pitch| > 72 deg) or plant divergence.
"""
from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field, replace
from typing import Callable, List, Optional

import numpy as np

from . import _abi
from .planner import (SAMPLE_WARM_GAUSS, ConstraintConfig, CostWeights, Goal, GridSpec,
                      NumericError, Planner, PlannerConfig, TireParams, VehicleParams,
                      make_params, make_terrain, Heightmap, SignedDistanceMap)

ROLLOVER_RAD = math.radians(72.0)


@dataclass
class CycleRecord:
    cycle: int
    state: np.ndarray          # plant state at planning time
    control: np.ndarray        # applied (delta_rate, v_bx_rate)
    best_index: int
    best_cost: float
    feasible: bool
    cycle_ms: float            # host wall time of the planning call
    kernel_ms: float           # device time of the rollout kernel


@dataclass
class TrialRecord:
    outcome: str = "running"   # success | rollover | diverged | timeout
    cycles: List[CycleRecord] = field(default_factory=list)
    final_state: Optional[np.ndarray] = None

    def latencies(self) -> np.ndarray:
        return np.array([c.cycle_ms for c in self.cycles])

    def p50_p99(self):
        lat = self.latencies()
        return float(np.percentile(lat, 50)), float(np.percentile(lat, 99))


def shift_warm(seq: np.ndarray) -> np.ndarray:
    """Previous winner shifted one ZOH step, last entry repeated (D7)."""
    out = np.empty_like(seq)
    out[:-1] = seq[1:]
    out[-1] = seq[-1]
    return out


class ClosedLoop:
    """Plan -> apply -> plant, `cycles` times.  `plan` is any callable
    (state, warm_seq, cycle) -> (controls n_steps x 2, index, cost, feasible,
    cycle_ms, kernel_ms); `device_planner` builds the one backed by the GPU."""

    def __init__(self, heights: np.ndarray, grid: GridSpec, sdist: Optional[np.ndarray],
                 goal: Goal, cfg: PlannerConfig, vp: VehicleParams = VehicleParams(),
                 tp: TireParams = TireParams(), cc: ConstraintConfig = ConstraintConfig(),
                 w: CostWeights = CostWeights(), plant_dt: float = 0.001):
        self.lib = _abi.load()
        self.goal, self.cfg = goal, cfg
        self.params = make_params(vp, tp, cc, w, goal, cfg)
        self.heights = np.ascontiguousarray(heights, dtype=np.float64)
        self.grid, self.sdist = grid, sdist
        self.terrain, self._keep = make_terrain(Heightmap(grid, self.heights), None)
        self.plant_dt = plant_dt
        self.plant_steps = int(round(cfg.dt_zoh / plant_dt))

    def sampling(self, cycle: int, warm, k0: int = 0, kc: Optional[int] = None):
        """The sampler of planning cycle `cycle` (seed + cycle, warm start)."""
        from .planner import make_sampling
        return make_sampling(replace(self.cfg, seed=self.cfg.seed + cycle), k0, kc, warm_seq=warm)

    def device_planner(self, device: int = 0, precision: int = _abi.PRECISION_FP32,
                       rank: int = 0, world_size: int = 1, nccl_id=None,
                       devices=None) -> Callable:
        """The GPU planner: one GPU, `devices` driven by this process, or one
        rank of a one-process-per-GPU job (rank / world_size / nccl_id)."""
        pl = Planner(device=device, rank=rank, world_size=world_size, k_max=self.cfg.n_samples,
                     n_steps_max=self.cfg.n_steps, nccl_id=nccl_id, precision=precision,
                     devices=devices)
        pl.set_params(self.params)
        pl.set_terrain_arrays(self.heights, self.sdist, self.grid)
        from .planner import shard_range
        k0, kc = shard_range(self.cfg.n_samples, rank, world_size)

        def plan(state, warm, cycle):
            smp, keep = self.sampling(cycle, warm, k0, kc)
            res, ctrl = pl.solve_raw(state, smp)
            return (ctrl, int(res.best_index), float(res.best_cost), bool(res.best_feasible),
                    float(res.cycle_ms), float(res.kernel_ms))
        plan.planner = pl
        return plan

    def plant(self, state: np.ndarray, control: np.ndarray) -> int:
        u = np.ascontiguousarray(control, dtype=np.float64)
        return self.lib.tmpc_plant_step(self.params, self.terrain, _abi.dptr(u), self.plant_dt,
                                        self.plant_steps, _abi.dptr(state))

    def run(self, plan: Callable, s0: np.ndarray, cycles: int,
            on_cycle: Optional[Callable[[CycleRecord], None]] = None,
            shadow=None) -> TrialRecord:
        """`shadow` (optional, a checker with .check(loop, cycle, state, warm,
        plan, record)) is called after every planning call, outside its timing."""
        rec = TrialRecord()
        state = np.array(s0, dtype=np.float64)
        warm = np.zeros((self.cfg.n_steps, 2))
        for c in range(cycles):
            dx, dy = state[0] - self.goal.x_g, state[1] - self.goal.y_g
            if dx * dx + dy * dy <= self.goal.r_g ** 2:
                rec.outcome = "success"
                break
            try:
                ctrl, idx, cost, feas, cyc_ms, k_ms = plan(state, warm, c)
            except NumericError:
                rec.outcome = "diverged"
                break
            cr = CycleRecord(c, state.copy(), ctrl[0].copy(), idx, cost, feas, cyc_ms, k_ms)
            rec.cycles.append(cr)
            if shadow is not None:
                shadow.check(self, c, state, warm, plan, cr)
            if on_cycle:
                on_cycle(cr)
            if self.plant(state, ctrl[0]) != _abi.TMPC_OK:
                rec.outcome = "diverged"
                break
            if abs(state[5]) > ROLLOVER_RAD or abs(state[4]) > ROLLOVER_RAD:
                rec.outcome = "rollover"
                break
            warm = shift_warm(ctrl)
        else:
            rec.outcome = "timeout"
        rec.final_state = state
        return rec
