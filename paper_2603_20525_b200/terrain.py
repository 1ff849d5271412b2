"""Terrain preprocessing and I/O of the reference (terrain.hpp), B200 side.

  Perimeter / PerimeterKind / validate      terrain.hpp:142-181
  gaussian_smooth(m, sigma_m)               terrain.hpp:102-138   -> GPU (tmpc_gaussian_smooth)
  build_sdist_map(grid, perimeters)         terrain.hpp:241-260   -> GPU (tmpc_build_sdist_map_gpu)
  save_heightmap / load_heightmap           terrain.hpp:334-415   (host text format "TERRAIN v1")

The two grid transforms run as CUDA kernels behind the C ABI and are
bit-identical to the reference fp64 code (tests/test_terrain_prep.py checks
them against oracle/_ref).  There is no CPU fallback: without a GPU they
raise.  The planner LODs of the paper (sigma 0.3 / 1.5 m)
are gaussian_smooth(m, sigma) of the plant terrain.
"""
from __future__ import annotations

import ctypes as C
import enum
import io
import re
from dataclasses import dataclass, field
from pathlib import Path
from typing import List, Sequence, Union

import numpy as np

from . import _abi
from .planner import ConfigError, GridSpec, Heightmap, SignedDistanceMap

__all__ = ["PerimeterKind", "Perimeter", "gaussian_smooth", "build_sdist_map", "save_heightmap",
           "load_heightmap", "validate_heightmap"]


class PerimeterKind(enum.IntEnum):
    """terrain.hpp:140."""
    OBSTACLE = 0
    PATH_BOUNDARY = 1


def _segments_intersect(a, b, c, d) -> bool:
    def cross(u, v):
        return u[0] * v[1] - u[1] * v[0]
    d1 = cross((b[0] - a[0], b[1] - a[1]), (c[0] - a[0], c[1] - a[1]))
    d2 = cross((b[0] - a[0], b[1] - a[1]), (d[0] - a[0], d[1] - a[1]))
    d3 = cross((d[0] - c[0], d[1] - c[1]), (a[0] - c[0], a[1] - c[1]))
    d4 = cross((d[0] - c[0], d[1] - c[1]), (b[0] - c[0], b[1] - c[1]))
    return ((d1 > 0) != (d2 > 0)) and ((d3 > 0) != (d4 > 0))


@dataclass
class Perimeter:
    """Closed polygon marking an obstacle or a path boundary (terrain.hpp:142-181)."""
    kind: PerimeterKind = PerimeterKind.OBSTACLE
    vertices: np.ndarray = field(default_factory=lambda: np.zeros((0, 2)))

    def validate(self) -> None:
        v = np.asarray(self.vertices, dtype=np.float64)
        n = len(v)
        if n < 3:
            raise ConfigError("perimeter: needs at least 3 vertices")
        area2 = 0.0
        for i in range(n):
            a, b = v[i], v[(i + 1) % n]
            area2 += a[0] * b[1] - b[0] * a[1]
        if abs(area2) < 1e-12:
            raise ConfigError("perimeter: zero area")
        for i in range(n):
            for j in range(i + 1, n):
                if j == i or (j + 1) % n == i or (i + 1) % n == j:
                    continue
                if _segments_intersect(v[i], v[(i + 1) % n], v[j], v[(j + 1) % n]):
                    raise ConfigError("perimeter: self-intersecting polygon")


def validate_heightmap(m: Heightmap) -> None:
    """Heightmap::validate (terrain.hpp:63-72)."""
    g = m.grid
    if g.nx < 2 or g.ny < 2:
        raise ConfigError("heightmap: grid must be at least 2x2")
    if not g.resolution > 0.0:
        raise ConfigError("heightmap: resolution must be positive")
    h = np.asarray(m.heights)
    if h.size != g.nx * g.ny:
        raise ConfigError("heightmap: height count does not match grid size")
    if not np.isfinite(h).all():
        raise ConfigError("heightmap: non-finite height")


def _check(rc: int, what: str) -> None:
    if rc == _abi.TMPC_OK:
        return
    msg = (_abi.load().tmpc_last_error(None) or b"").decode() or what
    if rc == _abi.TMPC_ERR_CONFIG:
        raise ConfigError(msg)
    raise RuntimeError(msg)


def gaussian_smooth(m: Heightmap, sigma_m: float, device: int = 0) -> Heightmap:
    """gaussian_smooth (terrain.hpp:102-138) on GPU `device`; bit-identical."""
    lib = _abi.load()
    h = np.ascontiguousarray(m.heights, dtype=np.float64).reshape(m.grid.ny, m.grid.nx)
    out = np.empty_like(h)
    _check(lib.tmpc_gaussian_smooth(device, _abi.dptr(h), m.grid.nx, m.grid.ny, m.grid.resolution,
                                    float(sigma_m), _abi.dptr(out)), "gaussian_smooth failed")
    return Heightmap(GridSpec(**vars(m.grid)), out)


def pack_perimeters(perimeters: Sequence[Perimeter]):
    """(poly_off int32 [n+1], verts float64 [V, 2], kinds int32 [n]) of the C ABI."""
    off = np.zeros(len(perimeters) + 1, dtype=np.int32)
    for k, p in enumerate(perimeters):
        off[k + 1] = off[k] + len(p.vertices)
    verts = (np.concatenate([np.asarray(p.vertices, dtype=np.float64).reshape(-1, 2)
                             for p in perimeters]) if perimeters else np.zeros((0, 2)))
    kinds = np.array([int(p.kind) for p in perimeters], dtype=np.int32)
    return off, np.ascontiguousarray(verts), kinds


def build_sdist_map(grid: GridSpec, perimeters: Sequence[Perimeter],
                    device: int = 0) -> SignedDistanceMap:
    """build_sdist_map (terrain.hpp:249-260) on GPU `device`; bit-identical."""
    lib = _abi.load()
    off, verts, kinds = pack_perimeters(perimeters)
    out = np.empty((grid.ny, grid.nx))
    ip = C.POINTER(C.c_int32)
    _check(lib.tmpc_build_sdist_map_gpu(device, grid.nx, grid.ny, grid.origin_x, grid.origin_y,
                                        grid.resolution, len(perimeters), off.ctypes.data_as(ip),
                                        _abi.dptr(verts), kinds.ctypes.data_as(ip),
                                        _abi.dptr(out)), "build_sdist_map failed")
    return SignedDistanceMap(GridSpec(**vars(grid)), out, len(perimeters) > 0)


# ---------------------------------------------------------------- heightmap I/O
def save_heightmap(m: Heightmap, dest: Union[str, Path, io.TextIOBase]) -> None:
    """save_heightmap (terrain.hpp:334-353): header values at the stream's
    default precision (6 significant digits), heights at precision 17."""
    g = m.grid
    h = np.asarray(m.heights, dtype=np.float64).reshape(g.ny, g.nx)
    lines = ["TERRAIN v1", "origin %.6g %.6g" % (g.origin_x, g.origin_y),
             "resolution %.6g" % g.resolution, "size %d %d" % (g.nx, g.ny)]
    lines += [" ".join("%.17g" % v for v in row) for row in h]
    text = "\n".join(lines) + "\n"
    if isinstance(dest, (str, Path)):
        try:
            Path(dest).write_text(text)
        except OSError:
            raise ConfigError(f"cannot open for writing: {dest}") from None
    else:
        dest.write(text)


_FLOAT = re.compile(r"\s*([+-]?(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?)")
_INT = re.compile(r"\s*([+-]?\d+)")
_WORD = re.compile(r"\s*(\S+)")


class _LineScan:
    """Sequential extraction from one line like std::istringstream >>."""

    def __init__(self, line: str):
        self.s, self.pos = line, 0

    def _take(self, rx):
        m = rx.match(self.s, self.pos)
        if not m:
            raise ValueError
        self.pos = m.end()
        return m.group(1)

    def word(self):
        return self._take(_WORD)

    def real(self):
        return float(self._take(_FLOAT))

    def integer(self):
        return int(self._take(_INT))


def load_heightmap(src: Union[str, Path, io.TextIOBase], name: str = "<stream>") -> Heightmap:
    """load_heightmap (terrain.hpp:355-407), same messages ("name:line: why")."""
    if isinstance(src, (str, Path)):
        try:
            text = Path(src).read_text()
        except OSError:
            raise ConfigError(f"cannot open: {src}") from None
        name = str(src)
    else:
        text = src.read()
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()  # getline does not produce an empty final line
    lineno = 0

    def fail(ln, why):
        return ConfigError(f"{name}:{ln}: {why}")

    def next_line():
        nonlocal lineno
        if lineno >= len(lines):
            raise fail(lineno + 1, "unexpected end of file")
        lineno += 1
        return lines[lineno - 1]

    if next_line() != "TERRAIN v1":
        raise fail(lineno, "expected header 'TERRAIN v1'")
    g = GridSpec()
    sc = _LineScan(next_line())
    try:
        tag = sc.word()
        g.origin_x, g.origin_y = sc.real(), sc.real()
        if tag != "origin":
            raise ValueError
    except ValueError:
        raise fail(lineno, "expected 'origin <x> <y>'") from None
    sc = _LineScan(next_line())
    try:
        tag = sc.word()
        g.resolution = sc.real()
        if tag != "resolution":
            raise ValueError
    except ValueError:
        raise fail(lineno, "expected 'resolution <r>'") from None
    sc = _LineScan(next_line())
    try:
        tag = sc.word()
        g.nx, g.ny = sc.integer(), sc.integer()
        if tag != "size":
            raise ValueError
    except ValueError:
        raise fail(lineno, "expected 'size <nx> <ny>'") from None
    if g.nx < 2 or g.ny < 2:
        raise fail(lineno, "size must be at least 2x2")
    h = np.empty((g.ny, g.nx))
    for j in range(g.ny):
        sc = _LineScan(next_line())
        try:
            for i in range(g.nx):
                h[j, i] = sc.real()
        except ValueError:
            raise fail(lineno, f"expected {g.nx} heights") from None
    m = Heightmap(g, h)
    validate_heightmap(m)
    return m
