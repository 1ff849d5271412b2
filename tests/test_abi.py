"""The C-ABI boundary (include/tmpc_b200.h) without a GPU: the library loads,
exports every declared symbol, validates like the reference validate()
methods, reports device absence as a runtime error, and its arg-min key
orders candidates like the reference's (infeasible, J, k)."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2603_20525_b200 import _abi
from paper_2603_20525_b200 import planner as PL

HEADER = Path(__file__).resolve().parents[1] / "include" / "tmpc_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:[\w\*\s]+?)\b(tmpc_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _abi.load()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) <= set(_abi.SIGNATURES), set(syms) - set(_abi.SIGNATURES)
    assert b"sm_100a" in lib.tmpc_build_info()


def good_params():
    cfg = PL.PlannerConfig(n_samples=16, n_steps=10, dt_zoh=0.05, dt_int=0.005)
    return PL.make_params(PL.VehicleParams(), PL.TireParams(), PL.ConstraintConfig(),
                          PL.CostWeights(), PL.Goal(10.0, 0.0, 2.5), cfg)


def validate(p):
    buf = C.create_string_buffer(256)
    return _abi.load().tmpc_validate_params(p, buf, 256), buf.value.decode()


def test_valid_params_pass():
    assert validate(good_params()) == (0, "")


@pytest.mark.parametrize("field,value,msg", [
    ("M", 0.0, "vehicle: M must be > 0"),           # dynamics.hpp:40-44
    ("k_r", -1.0, "vehicle: k_r must be > 0"),
    ("delta_max", 1.6, "vehicle: delta_max must be < pi/2"),  # dynamics.hpp:46
    ("C", 0.0, "tire: C must be > 0"),              # dynamics.hpp:55
    ("mu", 2.5, "tire: mu must be in (0, 2]"),      # dynamics.hpp:56
    ("eps_dist", 0.0, "constraints: eps_dist must be > 0"),  # constraints.hpp:53
    ("sigma", -1.0, "constraints: sigma must be > 0"),
    ("safety_factor", 0.0, "constraints: safety_factor must be > 0"),
    ("esm_nominal", 0.0, "esm_nominal must be > 0"),
    ("dt_int", 0.003, "dt_int must divide the ZOH period"),  # dynamics.hpp:477-481
    ("n_steps", 0, "n_steps must be >= 1"),
    ("goal_r", 0.0, "r_g must be > 0"),
    ("model", 5, "unknown vehicle model"),
    ("scheme", 7, "unknown integration scheme"),  # dynamics.hpp:419
])
def test_invalid_params_are_config_errors(field, value, msg):
    p = good_params()
    setattr(p, field, value)
    rc, text = validate(p)
    assert rc == _abi.TMPC_ERR_CONFIG
    assert msg in text


def test_terrain_validation():
    lib = _abi.load()
    buf = C.create_string_buffer(256)
    h = np.zeros((4, 4))
    t, keep = PL.make_terrain(PL.Heightmap(PL.GridSpec(0, 0, 0.1, 4, 4), h), None)
    assert lib.tmpc_validate_terrain(t, buf, 256) == 0
    h[1, 2] = np.nan  # terrain.hpp:72-73
    assert lib.tmpc_validate_terrain(t, buf, 256) == _abi.TMPC_ERR_CONFIG
    assert b"non-finite height" in buf.value
    t.nx = 1  # terrain.hpp:66-67
    assert lib.tmpc_validate_terrain(t, buf, 256) == _abi.TMPC_ERR_CONFIG


def test_ctx_create_config_errors_before_device():
    lib = _abi.load()
    o = _abi.tmpc_opts()
    o.world_size, o.rank = 2, 0  # world_size > 1 without an NCCL id
    h = C.c_void_p()
    assert lib.tmpc_ctx_create(o, C.byref(h)) == _abi.TMPC_ERR_CONFIG
    o.world_size, o.lanes = 1, 3
    assert lib.tmpc_ctx_create(o, C.byref(h)) == _abi.TMPC_ERR_CONFIG

    def bad(**kw):
        q = _abi.tmpc_opts()
        for k, v in kw.items():
            setattr(q, k, v)
        return lib.tmpc_ctx_create(q, C.byref(h))
    assert bad(graphs=7) == _abi.TMPC_ERR_CONFIG          # unknown graphs mode
    assert bad(exchange=5) == _abi.TMPC_ERR_CONFIG        # unknown exchange
    assert bad(timeout_ms=-1) == _abi.TMPC_ERR_CONFIG
    assert bad(n_devices=2) == _abi.TMPC_ERR_CONFIG       # no device list
    assert bad(exchange=_abi.EXCHANGE_PEER, world_size=65) == _abi.TMPC_ERR_CONFIG
    devs = (C.c_int32 * 2)(0, 0)
    # several devices and one process per GPU are exclusive
    assert bad(n_devices=2, devices=C.cast(devs, C.POINTER(C.c_int32)), world_size=2,
               exchange=_abi.EXCHANGE_PEER) == _abi.TMPC_ERR_CONFIG


@pytest.mark.skipif(PL._abi is None, reason="")
def test_no_device_is_a_runtime_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError, match="no CUDA device"):
        PL.Planner(device=0)


def test_python_errors_map_like_errors_hpp():
    with pytest.raises(PL.ConfigError):
        PL._raise(_abi.TMPC_ERR_CONFIG, "x")
    with pytest.raises(PL.NumericError):
        PL._raise(_abi.TMPC_ERR_NUMERIC, "x")
    with pytest.raises(RuntimeError):
        PL._raise(_abi.TMPC_ERR_RUNTIME, "x")


def test_key_order_is_feasible_first_then_cost_then_index():
    lib = _abi.load()

    def key(c, f, k, sel=_abi.SELECT_FEASIBLE_FIRST):
        return (lib.tmpc_key_hi(c, f, sel), k)
    assert key(100.0, 1, 5) < key(1.0, 0, 0)          # feasible beats cheaper infeasible
    assert key(1.0, 1, 9) < key(2.0, 1, 0)            # lower cost wins
    assert key(1.0, 1, 3) < key(1.0, 1, 4)            # ties -> lowest index
    assert key(float("inf"), 0, 0) > key(1e30, 0, 1)  # diverged last
    # the exact fp64 cost decides: costs one ulp apart are not tied (the f32
    # key of round 1 tied them and let the lower index win)
    c = 123.456
    assert key(np.nextafter(c, 0.0), 1, 9) < key(c, 1, 0)
    assert key(0.0, 1, 0) < key(5e-324, 1, 0)
    # plain (J, k) order ignores feasibility (the reference's argmin)
    assert key(1.0, 0, 0, _abi.SELECT_PLAIN) < key(100.0, 1, 5, _abi.SELECT_PLAIN)
    # the lexicographic MIN of (hi, index) is the oracle's arg-min order
    rng = np.random.default_rng(0)
    cost = rng.uniform(0, 100, 1000)
    cost[rng.integers(0, 1000, 50)] = float("inf")
    cost[7] = cost[3]  # an exact tie
    feas = rng.random(1000) < 0.3
    keys = [key(c, int(f), k) for k, (c, f) in enumerate(zip(cost, feas))]
    order = np.lexsort((np.arange(1000), cost, ~feas))
    assert min(keys)[1] == order[0]


def test_records_fold_like_one_shard():
    """tmpc_make_record / tmpc_fold_records (the per-GPU reduction and the
    cross-GPU fold): any split of the candidates into records folds to the
    same result, bit for bit (integer sums and MINs only), and equals the
    direct arg-min / counts / mean of the whole batch."""
    rng = np.random.default_rng(1)
    K = 5000
    cost = rng.uniform(0, 5e3, K)
    cost[rng.integers(0, K, 80)] = float("inf")
    flags = ((rng.random(K) < 0.4).astype(np.uint8) * _abi.FLAG_FEASIBLE)
    flags[~np.isfinite(cost)] = _abi.FLAG_DIVERGED
    flags[rng.integers(0, K, 100)] |= _abi.FLAG_GOAL
    margin = rng.uniform(-1, 1, K).astype(np.float32)
    sub = rng.integers(0, 1000, K)
    whole = PL.fold_records([PL.make_record(cost, flags, margin, 0, substeps=sub)])
    fin = np.isfinite(cost)
    order = np.lexsort((np.arange(K), cost, (flags & 1) == 0))
    assert whole.best_index == order[0] and whole.best_cost == cost[order[0]]
    assert whole.n_candidates == K and whole.substeps_executed == int(sub.sum())
    assert whole.n_feasible == int((flags & 1).sum())
    assert whole.n_diverged == int((~fin).sum()) and whole.n_goal == int(((flags & 4) > 0).sum())
    assert whole.min_cost == cost[fin].min()
    assert whole.mean_cost == pytest.approx(cost[fin].mean(), rel=1e-10)
    for G in (2, 3, 8):
        recs = []
        for r in range(G):
            k0, kc = PL.shard_range(K, r, G)
            recs.append(PL.make_record(cost[k0:k0 + kc], flags[k0:k0 + kc], margin[k0:k0 + kc], k0,
                                       substeps=sub[k0:k0 + kc]))
        for order_ in (recs, recs[::-1]):
            got = PL.fold_records(order_)
            assert bytes(got) == bytes(whole)
    # all diverged -> NumericError
    with pytest.raises(PL.NumericError):
        PL.fold_records([PL.make_record(np.full(4, np.inf), np.full(4, 2, np.uint8),
                                        np.zeros(4, np.float32), 0)])


def test_shard_ranges_partition():
    for n in (1, 7, 16384, 262144, 100003):
        for world in (1, 2, 3, 4, 8):
            spans = [PL.shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0
            for (a, c), (b, _) in zip(spans, spans[1:]):
                assert a + c == b
            assert spans[-1][0] + spans[-1][1] == n


def test_fold_skips_empty_records():
    """An idle GPU (fewer candidates than GPUs) contributes an empty record:
    it changes nothing in the fold."""
    cost = np.array([5.0, 3.0, 4.0])
    flags = np.array([1, 1, 0], dtype=np.uint8)
    margin = np.zeros(3, dtype=np.float32)
    empty = PL.make_record(np.zeros(0), np.zeros(0, np.uint8), np.zeros(0, np.float32), 3)
    assert empty.key_hi == _abi.KEY_NONE and empty.k_count == 0
    a = PL.fold_records([PL.make_record(cost, flags, margin, 0)])
    b = PL.fold_records([empty, PL.make_record(cost, flags, margin, 0), empty])
    assert bytes(a) == bytes(b) and a.best_index == 1
    with pytest.raises(PL.NumericError):
        PL.fold_records([empty])
