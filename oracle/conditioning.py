"""Conditioning of the reference's own result -- TEST INFRASTRUCTURE ONLY.

The north-star parity rule (per-candidate cost within 1e-4, BASELINE
north_star) excludes exactly the candidates on which the REFERENCE itself is
ill-conditioned at the scale of the device's fp32 arithmetic: its own cost
moves by >= 1e-4 when its inputs are perturbed by fp32 rounding.  Used by
tests/parity_util.check_parity and by the c5 shadow check (oracle/shadow.py).
"""
from __future__ import annotations

import numpy as np

from paper_2603_20525_b200 import planner as PL


def rel_err(a, b):
    with np.errstate(invalid="ignore", divide="ignore"):
        both = np.isfinite(a) & np.isfinite(b)
        return np.where(both, np.abs(a - b) / np.abs(b),
                        np.where(np.isfinite(a) == np.isfinite(b), 0.0, np.inf))


# fp32 rounding scale of each SrbState component (as_array order,
# dynamics.hpp:175-178): absolute floors, or 2^-23 of the value when larger
STATE_EPS_FLOOR = np.array([1e-6, 1e-6, 1e-7, 1e-7, 1e-7, 1e-7, 1e-7, 1e-7, 1e-7, 1e-7, 1e-7,
                            1e-7, 1e-7])


def state_perturbations(s0):
    """+- the fp32 rounding scale of each of the 13 state components."""
    s0 = np.asarray(s0, dtype=np.float64)
    for i in range(13):
        d = max(STATE_EPS_FLOOR[i], abs(s0[i]) * 2.0 ** -23)
        for sg in (1.0, -1.0):
            s1 = s0.copy()
            s1[i] += sg * d
            yield s1


def fp32_terrain(w):
    """The workload's terrain with heights and SDF rounded to fp32 (the device
    store's rounding), as a tmpc_terrain (+ keep-alive)."""
    h32 = w.heights.astype(np.float32).astype(np.float64)
    sd = None
    if w.sdist is not None:
        sd = PL.SignedDistanceMap(w.grid, w.sdist.astype(np.float32).astype(np.float64), True)
    return PL.make_terrain(PL.Heightmap(w.grid, h32), sd)


def extended_spread(orc, w, p, smp, terr, s0, idx, threads=8):
    """Conditioning spread of the reference on the listed candidates over
    every fp32-scale perturbation the device's arithmetic applies: each of
    the 13 state components +- its rounding scale, and the terrain rounded to
    fp32.  For a candidate the reference diverges on, the continuous quantity
    is the running cost up to the divergence and its substep: a changed
    divergence substep or finiteness is an infinite spread."""
    idx = np.asarray(idx, dtype=np.int64)
    spread = np.zeros(len(idx))
    if len(idx) == 0:
        return spread
    rc, c0, f0, m0, sub0, j0, err = orc.solve_indices(p, smp, terr, s0, idx, threads, True)
    assert rc == 0, err
    t32, keep = fp32_terrain(w)
    runs = [(s1, terr) for s1 in state_perturbations(s0)] + [(np.asarray(s0), t32)]
    for s1, tt in runs:
        rc, c1, f1, m1, sub1, j1, err = orc.solve_indices(p, smp, tt, s1, idx, threads, True)
        assert rc == 0, err
        r = rel_err(c1, c0)
        both_div = ~np.isfinite(c1) & ~np.isfinite(c0)
        r = np.where(both_div, np.where(sub1 != sub0, np.inf, rel_err(j1, j0)), r)
        spread = np.maximum(spread, r)
    return spread


