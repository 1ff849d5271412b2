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
// grid, row pointers of the two terrain fields at that cell, the clamp
// window [lo, hi] = [Q - 1 - a, n + Q - a] of a cell offset (the reference's
// clamp to [-1, n] of the gradient stencil) and the CoM window
// [clo, chi] = [lo - m, hi + m] (m = E0 + 1, KParams::cmargin) of the
// unclamped wheel lookups (prepare_frame).  Changes only when the position is
// re-anchored (once per ZOH step).
struct Anchor {
  const float4* hq;
  const float4* sdq;
  const float4* hq0;   // TerrainDev::hq32 (record 0)
  const float4* sdq0;  // TerrainDev::sdq32
  float lox, hix, loy, hiy;
  float clox, chix, cloy, chiy;
  unsigned bias;  // KParams::cell_bias + record index of the anchor cell (cell2u)
  int o;                          // record index of the anchor cell
  unsigned long long tex, hqtex;  // TerrainDev::sd_tex, hq_tex
};

__device__ __forceinline__ Anchor make_anchor(const KParams& P, const TerrainDev& td, int ax,
                                              int ay) {
  Anchor A;
  const long long o = static_cast<long long>(ay) * P.pitch + ax;
  A.hq = td.hq32 + 4 * o;
  A.sdq = td.sdq32 + o;
  A.hq0 = td.hq32;
  A.sdq0 = td.sdq32;
  A.o = static_cast<int>(o);
  A.tex = td.sd_tex;
  A.hqtex = td.hq_tex;
  A.lox = static_cast<float>(P.pad - 1 - ax);
  A.hix = static_cast<float>(P.nx + P.pad - ax);
  A.loy = static_cast<float>(P.pad - 1 - ay);
  A.hiy = static_cast<float>(P.ny + P.pad - ay);
  A.bias = P.cell_bias + static_cast<unsigned>(o);
  A.clox = static_cast<float>(P.pad - 1 - P.cmargin - ax);
  A.chix = static_cast<float>(P.nx + P.pad + P.cmargin - ax);
  A.cloy = static_cast<float>(P.pad - 1 - P.cmargin - ay);
  A.chiy = static_cast<float>(P.ny + P.pad + P.cmargin - ay);
  return A;
}

// Cell offset (from the anchor) + fraction of the offset coordinate t,
// clamped to the window: g' clamped to [Q-1, n+Q] exactly like axis_cell (out
// of range => the clamped integer cell, fraction 0).
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

// cell2 without the per-point clamp, for offsets from a CoM already clamped to
// [clo, chi]: t stays within E0 cells of it, inside the padded grid, and any
// point beyond [lo, hi] reads a record that is constant along that axis
// (ctx.cu upload_terrain), i.e. the clamped value.  Returns the absolute
// record index: the magic-number bias of both floors and the anchor's record
// index fold into one 32-bit constant, bits(ry) pitch + bits(rx) + A.bias ==
// o + iy pitch + ix (mod 2^32).  The one unsigned min against the last record
// only acts on a non-finite offset (the frozen state of a diverged candidate,
// whose result is discarded): it keeps that gather in bounds.
__device__ __forceinline__ unsigned cell2u(fm::f2 t, int pitch, unsigned bias, unsigned last,
                                           float& fx, float& fy) {
  const fm::f2 r = fm::fadd2_rd(t, fm::pk(fm::kMagic, fm::kMagic));  // exact floor + magic
  fm::upk(fm::fsub2(t, fm::fadd2(r, fm::pk(-fm::kMagic, -fm::kMagic))), fx, fy);
  float rx, ry;
  fm::upk(r, rx, ry);
  return min(static_cast<unsigned>(__float_as_int(ry)) * static_cast<unsigned>(pitch) +
                 static_cast<unsigned>(__float_as_int(rx)) + bias,
             last);
}

// Re-anchor the planar position at a ZOH boundary (exact: the integer part
// moves), branch-free so the boundary block stays one basic block.  A
// runaway offset (>= 2^21 cells, beyond the magic-number floor) stays
// un-anchored and the anchor stays within +-2^20 cells; the lookups clamp
// (cell / the CoM clamp of prepare_frame) so every gather stays in bounds.
__device__ __forceinline__ void reanchor(bool live, float& gxs, float& gys, int& ax, int& ay) {
  constexpr float kBig = 2097152.f;  // 2^21
  constexpr int kLim = 1 << 20;
  float fr;
  const int ix = fm::floor_frac(gxs, fr), iy = fm::floor_frac(gys, fr);
  const bool mvx = live && fabsf(gxs) < kBig && abs(ax + ix) < kLim;
  const bool mvy = live && fabsf(gys) < kBig && abs(ay + iy) < kLim;
  ax = mvx ? ax + ix : ax;
  gxs = mvx ? gxs - static_cast<float>(ix) : gxs;
  ay = mvy ? ay + iy : ay;
  gys = mvy ? gys - static_cast<float>(iy) : gys;
}

}  // namespace tmpcb
