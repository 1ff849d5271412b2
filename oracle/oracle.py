"""ctypes loader for the CPU oracle libraries — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) import this module, and only as the checker / baseline.
  liboracle.so          restatement (oracle/tmpc_oracle.cpp), always built
  _ref/libtmpc_ref.so   SPEC planner over the unmodified reference headers
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from paper_2603_20525_b200 import _abi

HERE = Path(__file__).resolve().parent
P = C.POINTER

_SOLVE_ARGS = [P(_abi.tmpc_params), P(_abi.tmpc_sampling), P(_abi.tmpc_terrain), P(C.c_double),
               P(C.c_double), P(C.c_uint8), P(C.c_float), P(C.c_int64), C.c_int]


def _bind(lib, prefix):
    lib_solve = getattr(lib, prefix + "_solve")
    lib_solve.restype = C.c_int
    if prefix == "oracle":
        lib_solve.argtypes = _SOLVE_ARGS + [C.c_int, P(_abi.tmpc_result), C.c_char_p, C.c_size_t]
    else:
        lib_solve.argtypes = _SOLVE_ARGS + [P(_abi.tmpc_result), C.c_char_p, C.c_size_t]
    f = getattr(lib, prefix + "_sample_controls")
    f.restype, f.argtypes = C.c_int, [P(_abi.tmpc_params), P(_abi.tmpc_sampling), C.c_int64,
                                      P(C.c_double)]
    f = getattr(lib, prefix + "_srb_derivative")
    if prefix == "oracle":
        f.argtypes = [P(_abi.tmpc_params), P(_abi.tmpc_terrain), P(C.c_double), P(C.c_double),
                      C.c_int, P(C.c_double), P(C.c_double)]
    else:
        f.argtypes = [P(_abi.tmpc_params), P(_abi.tmpc_terrain), P(C.c_double), P(C.c_double),
                      P(C.c_double), P(C.c_double)]
    f.restype = C.c_int
    f = getattr(lib, prefix + "_integrate_step")
    f.restype = C.c_int
    f.argtypes = [P(_abi.tmpc_params), P(_abi.tmpc_terrain), P(C.c_double), P(C.c_double),
                  C.c_double, C.c_int, P(C.c_double)]
    f = getattr(lib, prefix + "_terrain_query")
    f.restype = C.c_int
    f.argtypes = ([P(_abi.tmpc_terrain), P(C.c_double), C.c_int64] +
                  ([C.c_int] if prefix == "oracle" else []) + [P(C.c_double)])
    f = getattr(lib, prefix + "_build_sdist_map")
    f.restype = C.c_int
    f.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_int, P(C.c_int),
                  P(C.c_double), P(C.c_int), P(C.c_double)]
    f = getattr(lib, prefix + "_esm")
    f.restype, f.argtypes = C.c_double, [P(_abi.tmpc_params), C.c_double, C.c_double]
    f = getattr(lib, prefix + "_substream")
    f.restype, f.argtypes = C.c_uint64, [C.c_uint64] * 4
    f = getattr(lib, prefix + "_rng_draw")
    f.restype, f.argtypes = C.c_uint64, [C.c_uint64, C.c_int64]
    return lib


_WL = None


def workload_lib():
    """oracle/libworkload.so: the workload generators (synth.cpp) for the
    reference arm of bench.py, which must not load the product library."""
    global _WL
    if _WL is None:
        path = HERE / "libworkload.so"
        if not path.exists():
            raise FileNotFoundError(f"{path} missing (run __graft_entry__.build())")
        lib = C.CDLL(str(path))
        for n in ("tmpc_synth_heightmap", "tmpc_synth_obstacles", "tmpc_stamp_obstacles",
                  "tmpc_build_sdist_map"):
            res, args = _abi.SIGNATURES[n]
            getattr(lib, n).restype, getattr(lib, n).argtypes = res, args
        _WL = lib
    return _WL


class Oracle:
    """Uniform Python face over liboracle.so (kind='port') or _ref (kind='reference')."""

    def __init__(self, kind: str = "port"):
        self.kind = kind
        if kind == "port":
            path, self.prefix = HERE / "liboracle.so", "oracle"
        elif kind == "reference":
            path, self.prefix = HERE / "_ref" / "libtmpc_ref.so", "ref"
        else:
            raise ValueError(kind)
        if not path.exists():
            raise FileNotFoundError(f"oracle library missing: {path} (run __graft_entry__.build())")
        self.lib = _bind(C.CDLL(str(path)), self.prefix)
        if kind == "reference":
            for n, res, args in (("ref_tire_lateral_force", C.c_double, [C.c_double] * 4),
                                 ("ref_soft_cost_rate", C.c_double, [C.c_double] * 3)):
                fn = getattr(self.lib, n)
                fn.restype, fn.argtypes = res, args
            self.lib.ref_gaussian_smooth.restype = C.c_int
            self.lib.ref_gaussian_smooth.argtypes = [P(_abi.tmpc_terrain), C.c_double, P(C.c_double)]

    def solve_indices(self, params, smp, terrain, s0, idx, threads=1, extended=False):
        """Candidates at arbitrary global indices (reference only).  With
        extended=True also (substeps, running cost when the rollout stopped)."""
        if self.prefix != "ref":
            raise NotImplementedError("solve_indices: oracle/_ref only")
        f = self.lib.ref_solve_indices
        f.restype = C.c_int
        f.argtypes = [P(_abi.tmpc_params), P(_abi.tmpc_sampling), P(_abi.tmpc_terrain),
                      P(C.c_double), P(C.c_int64), C.c_int64, P(C.c_double), P(C.c_uint8),
                      P(C.c_float), P(C.c_int64), P(C.c_double), C.c_int, C.c_char_p,
                      C.c_size_t]
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        n = len(idx)
        cost, flags = np.empty(n), np.empty(n, dtype=np.uint8)
        margin = np.empty(n, dtype=np.float32)
        sub, jrun = np.empty(n, dtype=np.int64), np.empty(n)
        err = C.create_string_buffer(256)
        s0 = np.ascontiguousarray(s0, dtype=np.float64)
        rc = f(C.byref(params), C.byref(smp), C.byref(terrain), _abi.dptr(s0),
               idx.ctypes.data_as(P(C.c_int64)), n, _abi.dptr(cost),
               flags.ctypes.data_as(P(C.c_uint8)), margin.ctypes.data_as(P(C.c_float)),
               sub.ctypes.data_as(P(C.c_int64)), _abi.dptr(jrun), threads, err, 256)
        if extended:
            return rc, cost, flags, margin, sub, jrun, err.value.decode()
        return rc, cost, flags, margin, err.value.decode()

    def open_loop_errors(self, params, terrain, model, s0, controls, plant_dt=0.001, threads=1,
                         plant_terrain=None):
        """ref_open_loop_errors (reference only): per trajectory the time-
        averaged location / ESM errors of `model` vs the RK4 plant."""
        if self.prefix != "ref":
            raise NotImplementedError("open_loop_errors: oracle/_ref only")
        f = self.lib.ref_open_loop_errors
        f.restype = C.c_int
        f.argtypes = [P(_abi.tmpc_params), P(_abi.tmpc_terrain), P(_abi.tmpc_terrain), C.c_int,
                      P(C.c_double),
                      P(C.c_double), C.c_int64, C.c_double, P(C.c_double), P(C.c_double),
                      P(C.c_uint8), C.c_int, C.c_char_p, C.c_size_t]
        s0 = np.ascontiguousarray(s0, dtype=np.float64).reshape(-1, 13)
        u = np.ascontiguousarray(controls, dtype=np.float64)
        n = len(s0)
        loc, esm, fl = np.empty(n), np.empty(n), np.empty(n, dtype=np.uint8)
        err = C.create_string_buffer(256)
        rc = f(C.byref(params), C.byref(terrain),
               None if plant_terrain is None else C.byref(plant_terrain), int(model),
               _abi.dptr(s0), _abi.dptr(u), n,
               plant_dt, _abi.dptr(loc), _abi.dptr(esm), fl.ctypes.data_as(P(C.c_uint8)), threads,
               err, 256)
        return rc, loc, esm, fl, err.value.decode()

    @staticmethod
    def available(kind: str) -> bool:
        return (HERE / ("liboracle.so" if kind == "port" else "_ref/libtmpc_ref.so")).exists()

    def solve(self, params, smp, terrain, s0, threads=1, variant=0):
        K = smp.k_count
        cost = np.empty(K)
        flags = np.empty(K, dtype=np.uint8)
        margin = np.empty(K, dtype=np.float32)
        sub = np.empty(K, dtype=np.int64)
        res = _abi.tmpc_result()
        err = C.create_string_buffer(256)
        s0 = np.ascontiguousarray(s0, dtype=np.float64)
        args = [C.byref(params), C.byref(smp), C.byref(terrain), _abi.dptr(s0), _abi.dptr(cost),
                flags.ctypes.data_as(P(C.c_uint8)), margin.ctypes.data_as(P(C.c_float)),
                sub.ctypes.data_as(P(C.c_int64)), threads]
        if self.prefix == "oracle":
            args.append(variant)
        rc = getattr(self.lib, self.prefix + "_solve")(*args, C.byref(res), err, 256)
        return rc, res, cost, flags, margin, sub, err.value.decode()

    def sample_controls(self, params, smp, k):
        out = np.zeros((params.n_steps, 2))
        getattr(self.lib, self.prefix + "_sample_controls")(C.byref(params), C.byref(smp), k,
                                                          _abi.dptr(out))
        return out

    def srb_derivative(self, params, terrain, s13, u2, variant=0):
        d = np.zeros(13)
        diag = np.zeros(23)
        s = np.ascontiguousarray(s13, dtype=np.float64)
        u = np.ascontiguousarray(u2, dtype=np.float64)
        f = getattr(self.lib, self.prefix + "_srb_derivative")
        if self.prefix == "oracle":
            rc = f(C.byref(params), C.byref(terrain), _abi.dptr(s), _abi.dptr(u), variant,
                   _abi.dptr(d), _abi.dptr(diag))
        else:
            rc = f(C.byref(params), C.byref(terrain), _abi.dptr(s), _abi.dptr(u), _abi.dptr(d),
                   _abi.dptr(diag))
        return rc, d, diag

    def integrate_step(self, params, terrain, s13, u2, dt, scheme):
        out = np.zeros(13)
        s = np.ascontiguousarray(s13, dtype=np.float64)
        u = np.ascontiguousarray(u2, dtype=np.float64)
        rc = getattr(self.lib, self.prefix + "_integrate_step")(
            C.byref(params), C.byref(terrain), _abi.dptr(s), _abi.dptr(u), dt, scheme,
            _abi.dptr(out))
        return rc, out

    def terrain_query(self, terrain, xy, variant=0):
        xy = np.ascontiguousarray(xy, dtype=np.float64)
        out = np.zeros((len(xy), 4))
        f = getattr(self.lib, self.prefix + "_terrain_query")
        if self.prefix == "oracle":
            f(C.byref(terrain), _abi.dptr(xy), len(xy), variant, _abi.dptr(out))
        else:
            f(C.byref(terrain), _abi.dptr(xy), len(xy), _abi.dptr(out))
        return out

    def build_sdist_map(self, grid, off, verts, kinds=None):
        n_poly = len(off) - 1
        kinds = np.zeros(n_poly, dtype=np.int32) if kinds is None else np.asarray(kinds, np.int32)
        out = np.zeros((grid.ny, grid.nx))
        off = np.ascontiguousarray(off, dtype=np.int32)
        verts = np.ascontiguousarray(verts, dtype=np.float64)
        getattr(self.lib, self.prefix + "_build_sdist_map")(
            grid.nx, grid.ny, grid.origin_x, grid.origin_y, grid.resolution, n_poly,
            off.ctypes.data_as(P(C.c_int)), _abi.dptr(verts), kinds.ctypes.data_as(P(C.c_int)),
            _abi.dptr(out))
        return out

    # ---- reference-only terrain hooks (terrain.hpp:102-138, 334-415)
    @staticmethod
    def _grid_terrain(heights, grid):
        h = np.ascontiguousarray(heights, dtype=np.float64)
        t = _abi.tmpc_terrain()
        t.heights = _abi.dptr(h)
        t.nx, t.ny = grid.nx, grid.ny
        t.origin_x, t.origin_y, t.resolution = grid.origin_x, grid.origin_y, grid.resolution
        return t, h

    def gaussian_smooth(self, heights, grid, sigma_m):
        t, keep = self._grid_terrain(heights, grid)
        out = np.zeros((grid.ny, grid.nx))
        rc = self.lib.ref_gaussian_smooth(C.byref(t), sigma_m, _abi.dptr(out))
        return rc, out

    @staticmethod
    def _io_tool():
        return str(HERE / "_ref" / "ref_terrain_io")

    def save_heightmap(self, heights, grid, path):
        """The reference save_heightmap (via the _ref/ref_terrain_io CLI)."""
        import subprocess
        import tempfile
        with tempfile.NamedTemporaryFile(suffix=".f64") as f:
            np.ascontiguousarray(heights, dtype=np.float64).tofile(f.name)
            r = subprocess.run([self._io_tool(), "save", f.name, str(grid.nx), str(grid.ny),
                                repr(grid.origin_x), repr(grid.origin_y), repr(grid.resolution),
                                str(path)], capture_output=True, text=True, timeout=120)
        return r.returncode

    def load_heightmap(self, path):
        """The reference load_heightmap: (rc, error text, header[5], heights)."""
        import subprocess
        import tempfile
        with tempfile.NamedTemporaryFile(suffix=".f64") as f:
            r = subprocess.run([self._io_tool(), "load", str(path), f.name], capture_output=True,
                               text=True, timeout=120)
            if r.returncode:
                return r.returncode, r.stdout, None, None
            a = np.fromfile(f.name, dtype=np.float64)
        nx, ny = int(a[3]), int(a[4])
        return 0, "", a[:5], a[5:5 + nx * ny].reshape(ny, nx)
