"""ctypes mirror of include/tmpc_b200.h and the loader of libtmpc_b200.so.

The shared library is the product: there is no Python or CPU fallback for the
hot path.  If the library is missing, importing the planner raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libtmpc_b200.so"

TMPC_OK, TMPC_ERR_NUMERIC, TMPC_ERR_CONFIG, TMPC_ERR_RUNTIME = 0, 1, 2, 3
FLAG_FEASIBLE, FLAG_DIVERGED, FLAG_GOAL = 1, 2, 4
SAMPLE_UNIFORM, SAMPLE_RANDOM_WALK, SAMPLE_WARM_GAUSS = 0, 1, 2
SELECT_FEASIBLE_FIRST, SELECT_PLAIN = 0, 1
PRECISION_FP32, PRECISION_FP64 = 0, 1
MODEL_SRB, MODEL_EST = 0, 1
SCHEME_EULER, SCHEME_RK4 = 0, 1
ORDER_AUTO, ORDER_OFF, ORDER_ON = 0, 1, 2
GRAPHS_AUTO, GRAPHS_OFF = 0, 1
EXCHANGE_NCCL, EXCHANGE_PEER = 0, 1
KEY_NONE = 0xFFFFFFFFFFFFFFFF
STATE_DIM = 13


class tmpc_params(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "M", "J_xx", "J_yy", "J_zz", "L_f", "L_r", "e", "h", "R", "k_f", "k_r", "b_f", "b_r",
        "delta_max", "delta_rate_max", "g", "C", "mu",
        "a_by_bar", "esm_nominal", "eps_dist", "sigma", "safety_factor")] + [
        ("enable_dist", C.c_int32), ("enable_rollover", C.c_int32)] + [
        (n, C.c_double) for n in ("w_t", "w_c", "w_g", "goal_x", "goal_y", "goal_r",
                                  "dt_zoh", "dt_int")] + [
        ("n_steps", C.c_int32), ("selection", C.c_int32), ("model", C.c_int32),
        ("scheme", C.c_int32)]


class tmpc_sampling(C.Structure):
    _fields_ = [("kind", C.c_int32), ("_pad0", C.c_int32), ("seed", C.c_uint64),
                ("vdot_max", C.c_double), ("walk_step", C.c_double),
                ("warm_sigma_frac", C.c_double), ("warm_seq", C.POINTER(C.c_double)),
                ("k_begin", C.c_int64), ("k_count", C.c_int64), ("k_total", C.c_int64)]


class tmpc_terrain(C.Structure):
    _fields_ = [("heights", C.POINTER(C.c_double)), ("sdist", C.POINTER(C.c_double)),
                ("nx", C.c_int32), ("ny", C.c_int32), ("origin_x", C.c_double),
                ("origin_y", C.c_double), ("resolution", C.c_double)]


class tmpc_result(C.Structure):
    _fields_ = [("best_index", C.c_int64), ("best_cost", C.c_double),
                ("best_feasible", C.c_int32), ("best_margin", C.c_float),
                ("n_candidates", C.c_int64), ("n_feasible", C.c_int64),
                ("n_diverged", C.c_int64), ("n_goal", C.c_int64),
                ("min_cost", C.c_double), ("mean_cost", C.c_double),
                ("substeps_executed", C.c_int64), ("kernel_ms", C.c_double),
                ("cycle_ms", C.c_double)]


class tmpc_opts(C.Structure):
    _fields_ = [("device", C.c_int32), ("rank", C.c_int32), ("world_size", C.c_int32),
                ("lanes", C.c_int32), ("k_max", C.c_int64), ("n_steps_max", C.c_int32),
                ("precision", C.c_int32), ("nccl_id", C.c_void_p), ("ordering", C.c_int32),
                ("n_devices", C.c_int32), ("devices", C.POINTER(C.c_int32)),
                ("timeout_ms", C.c_int32), ("graphs", C.c_int32), ("exchange", C.c_int32),
                ("_pad1", C.c_int32)]


class tmpc_rank_record(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "key_lo", "key_hi", "min_cost_bits", "done_blocks", "n_feasible", "n_diverged", "n_goal",
        "n_finite", "substeps")] + [
        ("cost_limb", C.c_uint64 * 3), ("best_cost", C.c_double), ("best_margin", C.c_float),
        ("best_flags", C.c_int32), ("k_begin", C.c_int64), ("k_count", C.c_int64)]


class tmpc_synth_spec(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("origin_x", C.c_double),
                ("origin_y", C.c_double), ("resolution", C.c_double), ("seed", C.c_uint64),
                ("sine_amp", C.c_double), ("sine_wavelength", C.c_double),
                ("noise_amp", C.c_double), ("fractal_octaves", C.c_int32),
                ("_pad0", C.c_int32), ("fractal_persistence", C.c_double),
                ("fractal_lattice", C.c_double), ("fractal_pp", C.c_double),
                ("slope_deg", C.c_double), ("slope_period", C.c_double),
                ("slope_dir", C.c_double), ("n_berms", C.c_int32), ("_pad1", C.c_int32),
                ("berm_height", C.c_double), ("berm_length", C.c_double),
                ("berm_halfwidth", C.c_double)]


class tmpc_obstacle_spec(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("n", C.c_int32), ("n_gon", C.c_int32),
                ("r_min", C.c_double), ("r_max", C.c_double), ("x_min", C.c_double),
                ("x_max", C.c_double), ("y_min", C.c_double), ("y_max", C.c_double),
                ("clear_x", C.c_double), ("clear_y", C.c_double), ("clear_r", C.c_double)]


_P = C.POINTER
_vp = C.c_void_p
# name -> (restype, argtypes); every symbol include/tmpc_b200.h declares.
SIGNATURES = {
    "tmpc_ctx_create": (C.c_int, [_P(tmpc_opts), _P(_vp)]),
    "tmpc_ctx_destroy": (None, [_vp]),
    "tmpc_last_error": (C.c_char_p, [_vp]),
    "tmpc_validate_params": (C.c_int, [_P(tmpc_params), C.c_char_p, C.c_size_t]),
    "tmpc_validate_terrain": (C.c_int, [_P(tmpc_terrain), C.c_char_p, C.c_size_t]),
    "tmpc_set_params": (C.c_int, [_vp, _P(tmpc_params)]),
    "tmpc_set_terrain": (C.c_int, [_vp, _P(tmpc_terrain)]),
    "tmpc_solve": (C.c_int, [_vp, _P(C.c_double), _P(tmpc_sampling), _P(tmpc_result),
                             _P(C.c_double)]),
    "tmpc_stage_cycle": (C.c_int, [_vp, _P(C.c_double), _P(tmpc_sampling)]),
    "tmpc_launch_cycle": (C.c_int, [_vp]),
    "tmpc_finish_cycle": (C.c_int, [_vp, _P(tmpc_result)]),
    "tmpc_get_costs": (C.c_int, [_vp, _P(C.c_double), _P(C.c_uint8), _P(C.c_float)]),
    "tmpc_get_stream": (C.c_void_p, [_vp]),
    "tmpc_kernels_per_cycle": (C.c_int, [_vp]),
    "tmpc_sample_controls": (C.c_int, [_P(tmpc_params), _P(tmpc_sampling), C.c_int64,
                                       _P(C.c_double)]),
    "tmpc_key_hi": (C.c_uint64, [C.c_double, C.c_int, C.c_int]),
    "tmpc_make_record": (C.c_int, [_P(C.c_double), _P(C.c_uint8), _P(C.c_float), _P(C.c_int64),
                                   C.c_int64, C.c_int64, C.c_int, _P(tmpc_rank_record)]),
    "tmpc_fold_records": (C.c_int, [_P(tmpc_rank_record), C.c_int32, _P(tmpc_result)]),
    "tmpc_num_devices": (C.c_int, [_vp]),
    "tmpc_get_device_stream": (C.c_void_p, [_vp, C.c_int32]),
    "tmpc_get_device_ordinal": (C.c_int, [_vp, C.c_int32]),
    "tmpc_nccl_unique_id": (C.c_int, [_vp]),
    "tmpc_peer_export": (C.c_int, [_vp, _vp]),
    "tmpc_peer_connect": (C.c_int, [_vp, _vp, C.c_int32]),
    "tmpc_peer_inspect": (C.c_int, [_vp, C.c_int32, C.c_uint64, C.POINTER(tmpc_rank_record),
                                    C.POINTER(C.c_uint64)]),
    "tmpc_synth_heightmap": (C.c_int, [_P(tmpc_synth_spec), _P(C.c_double)]),
    "tmpc_synth_obstacles": (C.c_int, [_P(tmpc_obstacle_spec), _P(C.c_double),
                                       _P(C.c_double)]),
    "tmpc_stamp_obstacles": (C.c_int, [_P(tmpc_terrain), _P(C.c_double), C.c_int32,
                                       _P(C.c_int32), _P(C.c_double), C.c_double]),
    "tmpc_build_sdist_map": (C.c_int, [C.c_int32, C.c_int32, C.c_double, C.c_double,
                                       C.c_double, C.c_int32, _P(C.c_int32), _P(C.c_double),
                                       _P(C.c_int32), _P(C.c_double), C.c_int32]),
    "tmpc_gaussian_smooth": (C.c_int, [C.c_int32, _P(C.c_double), C.c_int32, C.c_int32,
                                       C.c_double, C.c_double, _P(C.c_double)]),
    "tmpc_build_sdist_map_gpu": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_double,
                                           C.c_double, C.c_double, C.c_int32, _P(C.c_int32),
                                           _P(C.c_double), _P(C.c_int32), _P(C.c_double)]),
    "tmpc_plant_step": (C.c_int, [_P(tmpc_params), _P(tmpc_terrain), _P(C.c_double), C.c_double,
                                  C.c_int32, _P(C.c_double)]),
    "tmpc_open_loop_errors": (C.c_int, [_vp, C.c_int32, _P(C.c_double), _P(C.c_double), C.c_int64,
                                        C.c_double, _P(C.c_double), _P(C.c_double),
                                        _P(C.c_uint8)]),
    "tmpc_set_plant_terrain": (C.c_int, [_vp, _P(tmpc_terrain)]),
    "tmpc_fp32_peak": (C.c_int, [C.c_int32, _P(C.c_double)]),
    "tmpc_build_info": (C.c_char_p, []),
}

_lib = None


def load() -> C.CDLL:
    """Load libtmpc_b200.so (built in-tree by __graft_entry__.build()).

    Raises ImportError when it is missing: the planner has no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("TMPC_B200_LIB", LIB_PATH))
    if not path.exists():
        raise ImportError(f"libtmpc_b200.so not built at {path}; run __graft_entry__.build()")
    lib = C.CDLL(str(path))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def dptr(a):
    """numpy float64 array -> POINTER(c_double) (None passes NULL)."""
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(C.c_double))
