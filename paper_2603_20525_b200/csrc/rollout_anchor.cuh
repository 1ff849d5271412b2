// Cell-anchored planar position of the fp32 rollout kernels (SRB
// rollout_f32.cu, EST rollout_est_f32.cu): the position is kept in padded-grid
// cell units as an integer anchor + a compensated fp32 offset (DESIGN.md §4,
// SURVEY App. A D12), so a terrain lookup is a magic-number floor of a small
// fp32 sum and a row-pointer offset.
#pragma once
#include <cuda_runtime.h>

#include "fastmath.cuh"
#include "rollout.cuh"

namespace tmpcb {

// The planar anchor of a candidate: its integer cell (ax, ay) in the padded
// grid, row pointers of the two terrain fields at that cell, and the
// clamp window [lo, hi] = [1 - a, n + 2 - a] of a cell offset.  Changes only
// when the position is re-anchored (once per ZOH step).
struct Anchor {
  const float4* hq;
  const float4* sdq;
  float lox, hix, loy, hiy;
  int o;                          // record index of the anchor cell
  unsigned long long tex, hqtex;  // TerrainDev::sd_tex, hq_tex
};

__device__ __forceinline__ Anchor make_anchor(const KParams& P, const TerrainDev& td, int ax,
                                              int ay) {
  Anchor A;
  const long long o = static_cast<long long>(ay) * P.pitch + ax;
  A.hq = td.hq32 + 4 * o;
  A.sdq = td.sdq32 + o;
  A.o = static_cast<int>(o);
  A.tex = td.sd_tex;
  A.hqtex = td.hq_tex;
  A.lox = static_cast<float>(1 - ax);
  A.hix = static_cast<float>(P.nx + 2 - ax);
  A.loy = static_cast<float>(1 - ay);
  A.hiy = static_cast<float>(P.ny + 2 - ay);
  return A;
}

// Cell offset (from the anchor) + fraction of the offset coordinate t,
// clamped to the window: g' clamped to [1, n+2] exactly like axis_cell (out of
// range => the clamped integer cell, fraction 0).
__device__ __forceinline__ int cell(float t, float lo, float hi, float& f) {
  return fm::floor_frac(fminf(fmaxf(t, lo), hi), f);
}

// Both axes of one lookup at once: the cell offset t = (tx, ty) (anchor
// relative, clamped to the window per axis) -> row-major record offset
// iy * pitch + ix and the fractions (fx, fy).  The magic-number floor and the
// fraction run as FADD2 pairs (bit-identical to cell() per axis).
__device__ __forceinline__ int cell2(fm::f2 t, const Anchor& A, int pitch, float& fx, float& fy) {
  float tx, ty;
  fm::upk(t, tx, ty);
  const fm::f2 c = fm::pk(fminf(fmaxf(tx, A.lox), A.hix), fminf(fmaxf(ty, A.loy), A.hiy));
  const fm::f2 r = fm::fadd2_rd(c, fm::pk(fm::kMagic, fm::kMagic));  // exact floor + magic
  fm::upk(fm::fsub2(c, fm::fadd2(r, fm::pk(-fm::kMagic, -fm::kMagic))), fx, fy);
  float rx, ry;
  fm::upk(r, rx, ry);
  return (__float_as_int(ry) - 0x4B400000) * pitch + (__float_as_int(rx) - 0x4B400000);
}

}  // namespace tmpcb
