// fp32 fast path of the fused rollout + cost + feasibility + arg-min kernel
// (same per-candidate algorithm as rollout.cu).
//
// Written for the SASS it produces (ncu: the first version spent 50% of its
// warp samples on long-scoreboard waits, one gather round trip per terrain
// row, with one warp per scheduler):
//  * every terrain gather of a substep (4 SDF quad texels at the planar wheel
//    footprints, 16 {H, dH/dx, dH/dy} node texels at the 4 contact points)
//    is issued before any is consumed, so a substep costs one L1/L2 round
//    trip instead of twelve;
//  * branch-free math (fastmath.cuh): no FCHK/slow-path branches splitting
//    the substep, so ptxas can interleave the four wheel chains;
//  * double-float state accumulators instead of fp64 (no XU conversions), x
//    and y in fp64 for the absolute grid position, cell indices via the
//    magic-number floor (no F2I/FRND), the running cost of a ZOH step summed
//    in fp32 before one fp64 accumulate.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "fastmath.cuh"
#include "rollout.cuh"
#include "rollout_dev.cuh"
#include "tmpc_common.h"

namespace tmpcb {

namespace {

__device__ __forceinline__ void df_clamp(fm::DF& a, const fm::DF& lo, const fm::DF& hi) {
  if (a.hi > hi.hi || (a.hi == hi.hi && a.lo > hi.lo)) a = hi;
  if (a.hi < lo.hi || (a.hi == lo.hi && a.lo < lo.lo)) a = lo;
}

// Cell index + fraction of g' = gi + gf + off (off = a wheel offset in cells),
// clamped to [1, n+2] like axis_cell.
__device__ __forceinline__ int cell(int gi, float gf, float off, int n_hi, float& f) {
  int i = gi + fm::floor_frac(gf + off, f);
  if (i < 1) {
    i = 1;
    f = 0.f;
  } else if (i >= n_hi) {
    i = n_hi;
    f = 0.f;
  }
  return i;
}

}  // namespace

__global__ void __launch_bounds__(kBlock) rollout_kernel_f32(const KParams P, const TerrainDev td,
                                                             const double* __restrict__ warm,
                                                             double* __restrict__ out_cost,
                                                             uint8_t* __restrict__ out_flags,
                                                             float* __restrict__ out_margin,
                                                             DevStats* __restrict__ st) {
  const KConsts<float>& K = P.cf;
  const int64_t kl = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool active = kl < P.k_count;
  const int64_t kg = P.k_begin + kl;

  double J = 0.0;
  float margin = __int_as_float(0x7f800000);  // +inf
  bool feasible = true, diverged = false, goal = false;
  unsigned substeps = 0;

  // state: x, y in fp64 (absolute grid position), the rest double-float
  double x = P.s0[0], y = P.s0[1];
  fm::DF z = fm::df_make(P.s0[2]);
  fm::DF psi = fm::df_make(P.s0[3]), th = fm::df_make(P.s0[4]), ph = fm::df_make(P.s0[5]);
  fm::DF vx = fm::df_make(P.s0[6]), vy = fm::df_make(P.s0[7]), vz = fm::df_make(P.s0[8]);
  fm::DF wx = fm::df_make(P.s0[9]), wy = fm::df_make(P.s0[10]), wz = fm::df_make(P.s0[11]);
  fm::DF de = fm::df_make(P.s0[12]);
  const fm::DF de_max = fm::df_make(P.cd.delta_max), de_min = fm::df_make(-P.cd.delta_max);
  const float gim = __double2float_rd(P.gimbal_lim);  // <= the fp64 limit; refined below

  if (active) {
    const uint64_t base = mix64(substream(P.seed, static_cast<uint64_t>(kg)));
    double prev[2] = {0.0, 0.0};
    const int n_hi_x = P.nx + 2, n_hi_y = P.ny + 2;
    const int pitch = P.pitch;
    const bool use_sd = P.enable_dist && P.has_sdist;
    const float4* __restrict__ hg = td.hg32;
    const float4* __restrict__ sdq = td.sdq32;
    const float dt = K.dt;
    for (int t = 0; t < P.n_steps; ++t) {
      double u[2];
      sample_step(P.smp, base, kg == 0, t, warm, prev, u);
      const float u_dr = static_cast<float>(u[0]);
      const float u_vr = static_cast<float>(u[1]);
      const double L0 = P.w_t + P.w_c * u[0] * u[0];
      float rate_sum = 0.f;  // sum of L_soft over this ZOH step's substeps
      int nq = 0;
      for (int q = 0; q < P.S; ++q) {
        // goal truncation before accumulating
        const double gdx = x - P.goal_x, gdy = y - P.goal_y;
        if (gdx * gdx + gdy * gdy <= P.goal_r2) {
          goal = true;
          break;
        }
        if (fabsf(th.hi) >= gim && fabs(fm::df_value(th)) >= P.gimbal_lim) {
          diverged = true;  // srb_derivative gimbal guard, dynamics.hpp:311-312
          break;
        }
        // ---- phase A: attitude, rotation, gather addresses
        float sps, cps, sth, cth, sph, cph, sde, cd;
        fm::sincos(psi.hi, &sps, &cps);
        fm::sincos(th.hi, &sth, &cth);
        fm::sincos(ph.hi, &sph, &cph);
        fm::sincos(de.hi, &sde, &cd);
        // rot_321 (dynamics.hpp:96-105)
        const float r00 = cps * cth, r01 = cps * sph * sth - cph * sps, r02 = sph * sps + cph * cps * sth;
        const float r10 = cth * sps, r11 = cph * cps + sph * sps * sth, r12 = cph * sps * sth - cps * sph;
        const float r20 = -sth, r21 = cth * sph, r22 = cph * cth;
        float gxf, gyf;
        const int gxi = fm::floor_frac(x * P.gx_scale + P.gx_off, gxf);
        const int gyi = fm::floor_frac(y * P.gy_scale + P.gy_off, gyf);
        float rwz[4], hfx[4], hfy[4], sfx[4], sfy[4];
        int hoff[4], soff[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float rx = K.rho[i][0], ry = K.rho[i][1], rz = K.rho[i][2];
          // contact point p_w = pos + R rho (dynamics.hpp:335)
          const float rwx = r00 * rx + r01 * ry + r02 * rz;
          const float rwy = r10 * rx + r11 * ry + r12 * rz;
          rwz[i] = r20 * rx + r21 * ry + r22 * rz;
          const int i0 = cell(gxi, gxf, rwx * K.inv_res, n_hi_x, hfx[i]);
          const int j0 = cell(gyi, gyf, rwy * K.inv_res, n_hi_y, hfy[i]);
          hoff[i] = j0 * pitch + i0;
          // planar footprint (wheel_footprint, constraints.hpp:104-113)
          const float ox = cps * rx - sps * ry;
          const float oy = sps * rx + cps * ry;
          const int si = cell(gxi, gxf, ox * K.inv_res, n_hi_x, sfx[i]);
          const int sj = cell(gyi, gyf, oy * K.inv_res, n_hi_y, sfy[i]);
          soff[i] = sj * pitch + si;
        }
        // ---- phase B: issue every gather of the substep
        float4 ta[4], tb[4], tc[4], tdd[4], sq[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float4* r0 = hg + hoff[i];
          ta[i] = __ldg(r0);
          tb[i] = __ldg(r0 + 1);
          tc[i] = __ldg(r0 + pitch);
          tdd[i] = __ldg(r0 + pitch + 1);
        }
        if (use_sd) {
#pragma unroll
          for (int i = 0; i < 4; ++i) sq[i] = __ldg(sdq + soff[i]);
        }
        // ---- phase C: gather-independent terms
        float rate = 0.f;
        if (P.enable_rollover) {
          // esm (constraints.hpp:16-23); sin(|phi|+phi_bar) by the angle sum
          const float sin_abs = ph.hi < 0.f ? -sph : sph;
          const float sin_lever = sin_abs * K.esm_c_pb + cph * K.esm_s_pb;
          const float sgn = fabsf(ph.hi) <= K.esm_phi_lim ? 1.f : -1.f;
          const float U = sgn * K.esm_Mg * (K.esm_r_bar * (1.f - sin_lever) * cth);
          const float a = fmaxf(0.f, 1.f - U * K.inv_eps_esm);
          rate += K.sigma * a * a;
          feasible = feasible && (U > 0.f);
          margin = fminf(margin, U * K.inv_esm_nominal);
        }
        const float gbx = r20 * (-K.g), gby = r21 * (-K.g), gbz = r22 * (-K.g);
        const float f_x_rear = K.half_M * (u_vr - gbx + wy.hi * vz.hi - wz.hi * vy.hi);
        // euler_rates_321 (dynamics.hpp:109-118) and v_w = R v_b (374)
        const float inv_ct = fm::rcp(cth);
        const float tt = sth * inv_ct;
        const float d_psi = (sph * wy.hi + cph * wz.hi) * inv_ct;
        const float d_th = cph * wy.hi - sph * wz.hi;
        const float d_ph = wx.hi + sph * tt * wy.hi + cph * tt * wz.hi;
        const float dxw = r00 * vx.hi + r01 * vy.hi + r02 * vz.hi;
        const float dyw = r10 * vx.hi + r11 * vy.hi + r12 * vz.hi;
        const float dzw = r20 * vx.hi + r21 * vy.hi + r22 * vz.hi;
        // ---- phase D: consume the gathers
        if (use_sd) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float sd = lerp_quad(sq[i], sfx[i], sfy[i]);
            const float a = fmaxf(0.f, 1.f - sd * K.inv_eps_dist);  // soft_cost_rate(-sd)
            rate += K.sigma * a * a;
            feasible = feasible && (sd > 0.f);
            margin = fminf(margin, sd * K.inv_eps_dist);
          }
        }
        rate_sum += rate;
        ++nq;
        float fy_sum = 0.f, fz_sum = 0.f, mx = 0.f, my = 0.f, mz = 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const bool front = i < 2;
          const float rx = K.rho[i][0], ry = K.rho[i][1], rz = K.rho[i][2];
          // point velocity v_i = v + omega x rho (dynamics.hpp:336)
          const float vix = vx.hi + (wy.hi * rz - wz.hi * ry);
          const float viy = vy.hi + (wz.hi * rx - wx.hi * rz);
          const float viz = vz.hi + (wx.hi * ry - wy.hi * rx);
          float h, gsx, gsy;
          lerp_hg(ta[i], tb[i], tc[i], tdd[i], hfx[i], hfy[i], h, gsx, gsy);
          // tau_b = R^T (-fx, -fy, 1) (dynamics.hpp:339-341)
          const float tbx = r20 - r00 * gsx - r10 * gsy;
          const float tby = r21 - r01 * gsx - r11 * gsy;
          const float tbz = r22 - r02 * gsx - r12 * gsy;
          const float inv_tbz = fm::rcp(fmaxf(tbz, K.tau_floor));
          // extension and rate (dynamics.hpp:343-346), z in double-float
          const float chi = (((z.hi - h) + rwz[i]) + z.lo) * inv_tbz;
          const float chi_dot = (tbx * (vix - chi * wy.hi) + tby * (viy + chi * wx.hi) + tbz * viz) * inv_tbz;
          // suspension (dynamics.hpp:348-351)
          const float f_k = fmaxf(K.fs_i[i] - K.k_i[i] * chi, 0.f);
          const float f_b = f_k > 0.f ? fmaxf(-K.b_i[i] * chi_dot, -f_k) : 0.f;
          const float f_z = f_k + f_b;
          // slip and tire (dynamics.hpp:353-356, 74-77)
          const float alpha = fm::atan_ratio(viy, fmaxf(vix, K.vbx_floor)) - (front ? de.hi : 0.f);
          const float ca = K.C * alpha;
          const float f_y = f_z * (-ca * K.mu) * fm::rsqrt(K.mu2 + ca * ca);
          // sums and moment rho x F (dynamics.hpp:358-362)
          const float Fy = front ? f_y * cd : f_y;
          const float Fx = front ? 0.f : f_x_rear;
          fy_sum += Fy;
          fz_sum += f_z;
          mx += ry * f_z - rz * Fy;
          my += rz * Fx - rx * f_z;
          mz += rx * Fy - ry * Fx;
        }
        const float d_vy = fy_sum * K.inv_M + gby + wx.hi * vz.hi - wz.hi * vx.hi;
        const float d_vz = fz_sum * K.inv_M + gbz - wx.hi * vy.hi + wy.hi * vx.hi;
        const float d_wx = (mx + K.cJx * wy.hi * wz.hi) * K.inv_Jxx;
        const float d_wy = (my - K.cJy * wx.hi * wz.hi) * K.inv_Jyy;
        const float d_wz = (mz + K.cJz * wx.hi * wy.hi) * K.inv_Jzz;
        // ---- forward Euler + clamp_steering (dynamics.hpp:423-441,453,466)
        x += P.dt * static_cast<double>(dxw);
        y += P.dt * static_cast<double>(dyw);
        fm::df_add(z, dt * dzw);
        fm::df_add(psi, dt * d_psi);
        fm::df_add(th, dt * d_th);
        fm::df_add(ph, dt * d_ph);
        fm::df_add(vx, dt * u_vr);
        fm::df_add(vy, dt * d_vy);
        fm::df_add(vz, dt * d_vz);
        fm::df_add(wx, dt * d_wx);
        fm::df_add(wy, dt * d_wy);
        fm::df_add(wz, dt * d_wz);
        fm::df_add(de, dt * u_dr);
        df_clamp(de, de_min, de_max);
        ++substeps;
        const float fsum = z.hi + psi.hi + th.hi + ph.hi + vx.hi + vy.hi + vz.hi + wx.hi + wy.hi +
                           wz.hi + de.hi;
        if (!(isfinite(fsum) && isfinite(x + y))) {
          diverged = true;  // dynamics.hpp:491-492
          break;
        }
      }
      J += P.dt * (static_cast<double>(nq) * L0 + static_cast<double>(rate_sum));
      if (goal || diverged) break;
    }
  }

  if (active) {
    if (diverged) {
      J = __longlong_as_double(0x7ff0000000000000LL);
      feasible = false;
      margin = __int_as_float(0xff800000);
    } else {
      const double gdx = x - P.goal_x, gdy = y - P.goal_y;
      J += P.w_g * sqrt(gdx * gdx + gdy * gdy);
    }
  }
  reduce_and_finalize(P, active, kl, kg, J, feasible, diverged, goal, margin, substeps, out_cost,
                      out_flags, out_margin, st);
}

void launch_rollout_f32(unsigned blocks, const KParams& P, const TerrainDev& td,
                        const double* warm, double* cost, uint8_t* flags, float* margin,
                        DevStats* st, cudaStream_t stream) {
  rollout_kernel_f32<<<blocks, kBlock, 0, stream>>>(P, td, warm, cost, flags, margin, st);
}

}  // namespace tmpcb
