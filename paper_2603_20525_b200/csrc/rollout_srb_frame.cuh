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
};


// Phase A + B of a substep: trig split over the group, rot_321
// (dynamics.hpp:96-105), contact points p_w = pos + R rho (335), planar
// footprints (wheel_footprint, constraints.hpp:104-113) and their gathers.
// (anchor + gxf, anchor + gyf) is the CoM in padded-grid cells.
template <int L, int W, bool TRIG_SET = false>
__device__ __forceinline__ void prepare_frame(Frame<W>& F, const KParams& P, int s, int gbase,
                                              const Anchor& A, float gxf, float gyf, float psi,
                                              float th, float ph, float de, const float* rho_x,
                                              const float* rho_y, const float* rho_z,
                                              bool use_sd) {
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
  int hoff[W], soff[W];
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
      const fm::f2 ir = fm::pk(K.inv_res, K.inv_res), g = fm::pk(gxf, gyf);
      hoff[w] = cell2(fm::ffma2(fm::pk(rwx, rwy), ir, g), A, pitch, F.hfx[w], F.hfy[w]);
      // planar footprint (wheel_footprint, constraints.hpp:104-113)
      const float ox = left ? oxa[a] - obx : oxa[a] + obx;
      const float oy = left ? oya[a] + oby : oya[a] - oby;
      soff[w] = cell2(fm::ffma2(fm::pk(ox, oy), ir, g), A, pitch, F.sfx[w], F.sfy[w]);
    }
  } else {
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const float rx = rho_x[w], ry = rho_y[w], rz = rho_z[w];
      const float rwx = F.r00 * rx + F.r01 * ry + F.r02 * rz;
      const float rwy = F.r10 * rx + F.r11 * ry + F.r12 * rz;
      F.rwz[w] = F.r20 * rx + F.r21 * ry + F.r22 * rz;
      hoff[w] = cell(fmaf(rwy, K.inv_res, gyf), A.loy, A.hiy, F.hfy[w]) * pitch +
                cell(fmaf(rwx, K.inv_res, gxf), A.lox, A.hix, F.hfx[w]);
      const float ox = cps * rx - sps * ry;
      const float oy = sps * rx + cps * ry;
      soff[w] = cell(fmaf(oy, K.inv_res, gyf), A.loy, A.hiy, F.sfy[w]) * pitch +
                cell(fmaf(ox, K.inv_res, gxf), A.lox, A.hix, F.sfx[w]);
    }
  }
#pragma unroll
  for (int w = 0; w < W; ++w) {
    // one 256-bit + one 128-bit gather per contact point: each is one L1
    // wavefront per lane-line, so fewer, wider requests cut the L1 data-pipe
    // load (the binding resource once the gathers are batched)
    const float4* r0 = A.hq + 4 * hoff[w];
    ldg256(r0, F.qh[w], F.qx[w]);
    F.qy[w] = __ldg(r0 + 2);
  }
  if (use_sd) {
#pragma unroll
    for (int w = 0; w < W; ++w) F.sq[w] = __ldg(A.sdq + soff[w]);
  }
}

}  // namespace tmpcb
