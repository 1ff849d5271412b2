// SRB substep frame of the fp32 rollout kernels (Euler rollout_f32.cu, RK4
// rollout_rk4_f32.cu): the attitude trig split over the L lanes of a
// candidate, rot_321 (dynamics.hpp:96-105), this lane's contact-point and
// footprint cells and their terrain gathers.
#pragma once
#include <cuda_runtime.h>

#include "fastmath.cuh"
#include "rollout.cuh"
#include "rollout_anchor.cuh"
#include "rollout_dev.cuh"

// TEX-pipe gathers (A/B switches): the footprint SDF quads go through the
// texture path by default (c2 -4.8%, c4 -5.7%: the L1 LSU data pipe is the
// contended resource); TMPC_HQ_TEX=2 would move every contact-point record
// (measured +30% c2 / +33% c4: texture latency, 3 instead of 2 requests).
#ifndef TMPC_SD_TEX
#define TMPC_SD_TEX 1
#endif
#ifndef TMPC_HQ_TEX
#define TMPC_HQ_TEX 0
#endif

namespace tmpcb {

constexpr unsigned kFull = 0xffffffffu;

// Predicated select that ptxas keeps as FSEL (a runtime lane index in a
// ternary chain otherwise becomes a branch).
__device__ __forceinline__ float selp(bool p, float a, float b) {
  float r;
  asm("{\n .reg .pred q;\n setp.ne.b32 q, %3, 0;\n selp.f32 %0, %1, %2, q;\n}"
      : "=f"(r)
      : "f"(a), "f"(b), "r"(static_cast<int>(p)));
  return r;
}

// 32-byte read-only gather (LDG.E.256, sm_100): two consecutive float4.
__device__ __forceinline__ void ldg256(const float4* p, float4& a, float4& b) {
  asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
      : "l"(p));
}

template <int L>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
  for (int o = 1; o < L; o <<= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// Everything a substep needs that depends only on its (final) state: attitude
// trig, rotation, this lane's contact-point / footprint cells and the
// gathered terrain texels.
template <int W>
struct Frame {
  float sps, cps, sth, cth, sph, cph, cd;
  float r00, r01, r02, r10, r11, r12, r20, r21, r22;
  float rwz[W], hfx[W], hfy[W], sfx[W], sfy[W];
  float4 qh[W], qx[W], qy[W], sq[W];  // H / dH/dx / dH/dy / SDF corner quads
  float cl;    // SKIP: footprint clearance of the CoM cell (ctx.cu upload_terrain)
  bool sd_on;  // SKIP: the footprint cells / SDF quads were built (warp-uniform)
};


// Phase A + B of a substep: trig split over the group, rot_321
// (dynamics.hpp:96-105), contact points p_w = pos + R rho (335), planar
// footprints (wheel_footprint, constraints.hpp:104-113) and their gathers.
// (anchor + gxf, anchor + gyf) is the CoM in padded-grid cells.  SKIP (one
// lane per candidate): the footprint cells and SDF gathers only when the
// warp-uniform sd_fetch says so, plus the footprint clearance of the CoM cell
// for the caller's next skip test (rollout_f32.cu).
template <int L, int W, bool TRIG_SET = false, bool QT = false, bool SKIP = false>
__device__ __forceinline__ void prepare_frame(Frame<W>& F, const KParams& P, int s, int gbase,
                                              const Anchor& A, float gxf, float gyf, float psi,
                                              float th, float ph, float de, const float* rho_x,
                                              const float* rho_y, const float* rho_z,
                                              bool use_sd, bool sd_fetch = true) {
  static_assert(!SKIP || L == 1, "the footprint skip serves one-lane layouts");
  const KConsts<float>& K = P.cf;
  // one lane alone evaluates psi, theta, phi (cos delta by its short series)
  // (TRIG_SET, L = 1: the caller already holds sin / cos of psi, theta, phi in F)
  constexpr int NA = L == 1 ? (TRIG_SET ? 0 : 3) : W;
  float tsn[W], tcs[W];
#pragma unroll
  for (int m = 0; m < NA; ++m) {
    const int j = s + m * L;  // angle index: 0 psi, 1 theta, 2 phi, 3 delta
    const float a = selp(j & 2, selp(j & 1, de, ph), selp(j & 1, th, psi));
    fm::sincos(a, &tsn[m], &tcs[m]);
  }
  if constexpr (L == 1) {
    if constexpr (!TRIG_SET) {
      F.sps = tsn[0]; F.cps = tcs[0]; F.sth = tsn[1]; F.cth = tcs[1];
      F.sph = tsn[2]; F.cph = tcs[2];
    }
    F.cd = fm::cos_small(de);
  } else {
    F.sps = __shfl_sync(kFull, tsn[0 / L], gbase + 0 % L);
    F.cps = __shfl_sync(kFull, tcs[0 / L], gbase + 0 % L);
    F.sth = __shfl_sync(kFull, tsn[1 / L], gbase + 1 % L);
    F.cth = __shfl_sync(kFull, tcs[1 / L], gbase + 1 % L);
    F.sph = __shfl_sync(kFull, tsn[2 / L], gbase + 2 % L);
    F.cph = __shfl_sync(kFull, tcs[2 / L], gbase + 2 % L);
    F.cd = __shfl_sync(kFull, tcs[3 / L], gbase + 3 % L);
  }
  const float sps = F.sps, cps = F.cps, sth = F.sth, cth = F.cth, sph = F.sph, cph = F.cph;
  F.r00 = cps * cth; F.r01 = cps * sph * sth - cph * sps; F.r02 = sph * sps + cph * cps * sth;
  F.r10 = cth * sps; F.r11 = cph * cps + sph * sps * sth; F.r12 = cph * sps * sth - cps * sph;
  F.r20 = -sth;      F.r21 = cth * sph;                   F.r22 = cph * cth;
  const int pitch = P.pitch;
  const unsigned bias = A.bias, last = P.last_cell;
  unsigned hoff[W], soff[W];  // absolute record indices
  // the CoM clamped to [clo, chi] once; the wheel points are looked up
  // unclamped from it (cell2u, rollout_anchor.cuh)
  const fm::f2 g = fm::pk(fminf(fmaxf(gxf, A.clox), A.chix), fminf(fmaxf(gyf, A.cloy), A.chiy));
  const fm::f2 ir = fm::pk(K.inv_res, K.inv_res);
  if constexpr (L <= 2) {
    // wheel_offsets (dynamics.hpp:188-192) are axle-symmetric: rho = (x_a,
    // +-e/2, -(h+R)) with x_a = L_f (wheels 0, 1) or -L_r (2, 3) and the
    // left wheel first, so R rho = (R col0 x_a + R col2 rho_z) +- R col1 e/2.
    // This lane owns NAX = 2 / L axles (its wheels 2a, 2a + 1).
    constexpr int NAX = 2 / L;
    const float hw = rho_y[0], rz = rho_z[0];
    float ax[NAX], ay[NAX], az[NAX], oxa[NAX], oya[NAX];
#pragma unroll
    for (int a = 0; a < NAX; ++a) {
      const float xa = rho_x[2 * a];
      ax[a] = fmaf(F.r00, xa, F.r02 * rz);
      ay[a] = fmaf(F.r10, xa, F.r12 * rz);
      az[a] = fmaf(F.r20, xa, F.r22 * rz);
      oxa[a] = cps * xa;
      oya[a] = sps * xa;
    }
    const float bx = F.r01 * hw, by = F.r11 * hw, bz = F.r21 * hw;
    const float obx = sps * hw, oby = cps * hw;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const int a = w >> 1;
      const bool left = (w & 1) == 0;
      const float rwx = left ? ax[a] + bx : ax[a] - bx;
      const float rwy = left ? ay[a] + by : ay[a] - by;
      F.rwz[w] = left ? az[a] + bz : az[a] - bz;
      hoff[w] = cell2u(fm::ffma2(fm::pk(rwx, rwy), ir, g), pitch, bias, last, F.hfx[w], F.hfy[w]);
      // planar footprint (wheel_footprint, constraints.hpp:104-113)
      if constexpr (!SKIP) {
        const float ox = left ? oxa[a] - obx : oxa[a] + obx;
        const float oy = left ? oya[a] + oby : oya[a] - oby;
        soff[w] = cell2u(fm::ffma2(fm::pk(ox, oy), ir, g), pitch, bias, last, F.sfx[w], F.sfy[w]);
      }
    }
  } else {
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const float rx = rho_x[w], ry = rho_y[w], rz = rho_z[w];
      const float rwx = F.r00 * rx + F.r01 * ry + F.r02 * rz;
      const float rwy = F.r10 * rx + F.r11 * ry + F.r12 * rz;
      F.rwz[w] = F.r20 * rx + F.r21 * ry + F.r22 * rz;
      hoff[w] = cell2u(fm::ffma2(fm::pk(rwx, rwy), ir, g), pitch, bias, last, F.hfx[w], F.hfy[w]);
      const float ox = cps * rx - sps * ry;
      const float oy = sps * rx + cps * ry;
      soff[w] = cell2u(fm::ffma2(fm::pk(ox, oy), ir, g), pitch, bias, last, F.sfx[w], F.sfy[w]);
    }
  }
#pragma unroll
  for (int w = 0; w < W; ++w) {
    // one 256-bit + one 128-bit gather per contact point: each is one L1
    // wavefront per lane-line, so fewer, wider requests cut the L1 data-pipe
    // load (the binding resource once the gathers are batched)
#if TMPC_HQ_TEX == 2
    const int ti = 4 * hoff[w];
    F.qh[w] = tex1Dfetch<float4>(A.hqtex, ti);
    F.qx[w] = tex1Dfetch<float4>(A.hqtex, ti + 1);
    F.qy[w] = tex1Dfetch<float4>(A.hqtex, ti + 2);
#else
    const float4* r0 = A.hq0 + 4 * static_cast<size_t>(hoff[w]);
    ldg256(r0, F.qh[w], F.qx[w]);
    // QT: the third quad through the TEX pipe -- for throughput-bound launches
    // without the footprint term (c3 -11%); latency-bound ones lose (c2 +20%)
    if (QT || TMPC_HQ_TEX == 1)
      F.qy[w] = tex1Dfetch<float4>(A.hqtex, 4 * hoff[w] + 2);
    else
      F.qy[w] = __ldg(r0 + 2);
#endif
  }
  if constexpr (SKIP) {
    // the clearance sits in the spare texel of the CoM cell's record
    float fxc, fyc;
    const unsigned co = cell2u(g, pitch, bias, last, fxc, fyc);
    F.cl = __ldg(reinterpret_cast<const float*>(A.hq0 + 4 * static_cast<size_t>(co) + 3));
    F.sd_on = sd_fetch;
    if (use_sd && sd_fetch) {
      // the planar footprint as in the loop above (same operations, same
      // rounding), built only for a warp that needs it
      const float hw = rho_y[0];
      const float obx = sps * hw, oby = cps * hw;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const int a = w >> 1;
        const bool left = (w & 1) == 0;
        const float xa = rho_x[2 * a];
        const float oxa = cps * xa, oya = sps * xa;
        const float ox = left ? oxa - obx : oxa + obx;
        const float oy = left ? oya + oby : oya - oby;
        const unsigned so = cell2u(fm::ffma2(fm::pk(ox, oy), ir, g), pitch, bias, last, F.sfx[w],
                                   F.sfy[w]);
        F.sq[w] = __ldg(A.sdq0 + so);
      }
    }
  } else if (use_sd) {
#pragma unroll
    for (int w = 0; w < W; ++w) {
      // through the TEX pipe (c2 -7% vs LDG: the L1 LSU data pipe is the
      // contended resource), except in the QT launches, whose third
      // contact-point quad already loads the texture path (c4 -0.7% via LDG)
      if (TMPC_SD_TEX && !QT)
        F.sq[w] = tex1Dfetch<float4>(A.tex, soff[w]);
      else
        F.sq[w] = __ldg(A.sdq0 + soff[w]);
    }
  }
}

// Suspension + tire model (dynamics.hpp:333-371) of one axle's left / right
// wheels (frame slots wl, wl + 1) as fp32x2 pairs: the two wheels share the
// axle's spring / damper / static load and the point velocity's y component,
// so most of the per-wheel arithmetic runs as one FFMA2 / FADD2 / FMUL2 per
// operation; the clamps, selects, MUFU ops and the slip-angle interval
// selection stay per element.  Returns f_z and the lateral force (cos delta
// applied on the front axle) per wheel.
template <int W>
__device__ __forceinline__ void axle_pair_forces(const Frame<W>& F, int wl, const KConsts<float>& K,
                                                 float zs, float zc, float wx, float wy,
                                                 float vix_l, float vix_r, float viy, float viz_l,
                                                 float viz_r, float fs, float kk, float bb,
                                                 bool front, float de, float& fzl, float& fzr,
                                                 float& fyl, float& fyr) {
  using namespace fm;
  const int wr = wl + 1;
  const f2 H = pk(lerp_quad(F.qh[wl], F.hfx[wl], F.hfy[wl]), lerp_quad(F.qh[wr], F.hfx[wr], F.hfy[wr]));
  const f2 GX = pk(lerp_quad(F.qx[wl], F.hfx[wl], F.hfy[wl]), lerp_quad(F.qx[wr], F.hfx[wr], F.hfy[wr]));
  const f2 GY = pk(lerp_quad(F.qy[wl], F.hfx[wl], F.hfy[wl]), lerp_quad(F.qy[wr], F.hfx[wr], F.hfy[wr]));
  // tau_b = R^T (-fx, -fy, 1) (dynamics.hpp:339-341)
  const f2 TBX = ffma2(GY, pk(-F.r10, -F.r10), ffma2(GX, pk(-F.r00, -F.r00), pk(F.r20, F.r20)));
  const f2 TBY = ffma2(GY, pk(-F.r11, -F.r11), ffma2(GX, pk(-F.r01, -F.r01), pk(F.r21, F.r21)));
  const f2 TBZ = ffma2(GY, pk(-F.r12, -F.r12), ffma2(GX, pk(-F.r02, -F.r02), pk(F.r22, F.r22)));
  float tbz_l, tbz_r;
  upk(TBZ, tbz_l, tbz_r);
  const f2 INV = pk(rcp(fmaxf(tbz_l, K.tau_floor)), rcp(fmaxf(tbz_r, K.tau_floor)));
  // extension and rate (dynamics.hpp:343-346); z compensated (value zs - zc)
  const f2 CHI = fmul2(fsub2(fadd2(fsub2(pk(zs, zs), H), pk(F.rwz[wl], F.rwz[wr])), pk(zc, zc)), INV);
  const f2 A = ffma2(CHI, pk(-wy, -wy), pk(vix_l, vix_r));
  const f2 B = ffma2(CHI, pk(wx, wx), pk(viy, viy));
  const f2 CHD = fmul2(ffma2(TBZ, pk(viz_l, viz_r), ffma2(TBY, B, fmul2(TBX, A))), INV);
  // suspension (dynamics.hpp:348-351)
  float fk_l, fk_r, nb_l, nb_r;
  upk(ffma2(CHI, pk(-kk, -kk), pk(fs, fs)), fk_l, fk_r);
  upk(fmul2(CHD, pk(-bb, -bb)), nb_l, nb_r);
  fk_l = fmaxf(fk_l, 0.f);
  fk_r = fmaxf(fk_r, 0.f);
  const float fb_l = fk_l > 0.f ? fmaxf(nb_l, -fk_l) : 0.f;
  const float fb_r = fk_r > 0.f ? fmaxf(nb_r, -fk_r) : 0.f;
  const f2 FZ = fadd2(pk(fk_l, fk_r), pk(fb_l, fb_r));
  // slip and tire (dynamics.hpp:353-356, 74-77)
  f2 AL = atan_ratio2(viy, fmaxf(vix_l, K.vbx_floor), viy, fmaxf(vix_r, K.vbx_floor));
  if (front) AL = fsub2(AL, pk(de, de));
  const f2 CA = fmul2(AL, pk(K.C, K.C));
  float q_l, q_r;
  upk(ffma2(CA, CA, pk(K.mu2, K.mu2)), q_l, q_r);
  f2 FY = fmul2(fmul2(FZ, fmul2(CA, pk(-K.mu, -K.mu))), pk(rsqrt(q_l), rsqrt(q_r)));
  if (front) FY = fmul2(FY, pk(F.cd, F.cd));
  upk(FZ, fzl, fzr);
  upk(FY, fyl, fyr);
}

}  // namespace tmpcb
