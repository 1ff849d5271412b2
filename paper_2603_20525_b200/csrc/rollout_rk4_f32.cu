// fp32 fast path of the SRB rollout with the reference's RK4 substep
// (Scheme::kRk4, dynamics.hpp:454-466).  Per candidate and
// substep, as oracle/tmpc_oracle.cpp rollout + rk4_update and oracle/_ref
// over integrate_step<SrbModel>(.., kRk4):
//   goal test; L_soft at the substep's start state (ESM + footprint SDF)
//   k1..k4 = srb_derivative at s, s + dt/2 k1, s + dt/2 k2, s + dt k3
//       (dynamics.hpp:308-398; the gimbal guard of any stage diverges the
//       candidate, as the reference's std::domain_error does)
//   s += dt/6 (k1 + 2 k2 + 2 k3 + k4); clamp_steering
// Same machinery as the Euler fast path (rollout_f32.cu): L lanes per
// candidate sharing the wheels (rollout_srb_frame.cuh), the planar position
// as a cell anchor + compensated offset, every state entry Kahan-compensated
// (the stage inputs s + f k fold the compensation in: fm::ks_stage), branch-free math and a
// warp-uniform `live` predicate.  The stage-1 frame of the next substep (trig,
// contact points, gathers incl. the footprint SDF quads) is built at the end
// of the iteration so its gathers cross the back-edge; stages 2-4 depend on
// the previous stage's rates and gather in line.
// The RK4 kernel refines its MUFU reciprocal / rsqrt with one Newton step
// (TMPC_ACC_MATH bits 1 | 2, fastmath.cuh): its four stages per substep feed
// more rounding into each candidate than the Euler kernel, and at c3's full
// size SRB candidate 23102 -- reference spread 9.80e-5 under the fp32-scale
// perturbations, just under the exclusion threshold -- sits at 1.006e-4 with
// the raw MUFU results and 9.85e-5 with the refined ones (c3 +2%, c2 +0.6%;
// full CUDA atanf / sincosf, bits 4 | 8, would cost +39%).
// Each .cu is its own device module (no -rdc): the other kernels keep the raw
// MUFU results.
#ifndef TMPC_ACC_MATH
#ifndef TMPC_RK4_ACC_MATH
#define TMPC_RK4_ACC_MATH 3
#endif
#define TMPC_ACC_MATH TMPC_RK4_ACC_MATH
#endif
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "fastmath.cuh"
#include "launch.cuh"
#include "rollout.cuh"
#include "rollout_anchor.cuh"
#include "rollout_dev.cuh"
#include "rollout_srb_frame.cuh"
#include "tmpc_common.h"

// TMPC_RK4_INCR_TRIG=1: stages 2-4 of a one-lane candidate rotate the
// substep's start trig by their angle offsets (3 x 9 instead of 3 x 22
// instructions) instead of exact sin / cos -- a few ulp more error, which the
// full-size parity rule does not absorb on chaotic c3 rollouts.
#ifndef TMPC_RK4_INCR_TRIG
#define TMPC_RK4_INCR_TRIG 0
#endif

namespace tmpcb {

namespace {

// srb_derivative rates of one stage (dynamics.hpp:308-398) in fp32.
struct Rates {
  float x, y, z, psi, th, ph, vy, vz, wx, wy, wz;  // x, y in m/s (world)
};

// The state a stage reads (plain fp32) + its frame F.
struct StageState {
  float z, zc, vx, vy, vz, wx, wy, wz, de;
};

template <int L, int W>
__device__ __forceinline__ Rates srb_rates(const Frame<W>& F, const KConsts<float>& K,
                                           const StageState& y, float u_vr, const float* rho_x,
                                           const float* rho_y, const float* rho_z,
                                           const float* k_w, const float* b_w,
                                           const float* fs_w, const bool* front) {
  const float gbx = F.r20 * (-K.g), gby = F.r21 * (-K.g), gbz = F.r22 * (-K.g);
  const float f_x_rear = K.half_M * (u_vr - gbx + y.wy * y.vz - y.wz * y.vy);
  float fy_sum = 0.f, fz_sum = 0.f, mx = 0.f, my = 0.f, mz = 0.f;
  // per-wheel suspension + tire model (dynamics.hpp:333-371)
  const auto wheel = [&](int w, float vix, float viy, float viz, bool is_front, float& f_z,
                         float& Fy) {
    const float h = lerp_quad(F.qh[w], F.hfx[w], F.hfy[w]);
    const float gsx = lerp_quad(F.qx[w], F.hfx[w], F.hfy[w]);
    const float gsy = lerp_quad(F.qy[w], F.hfx[w], F.hfy[w]);
    const float tbx = F.r20 - F.r00 * gsx - F.r10 * gsy;  // tau_b = R^T (-fx, -fy, 1)
    const float tby = F.r21 - F.r01 * gsx - F.r11 * gsy;
    const float tbz = F.r22 - F.r02 * gsx - F.r12 * gsy;
    const float inv_tbz = fm::rcp(fmaxf(tbz, K.tau_floor));
    const float chi = (((y.z - h) + F.rwz[w]) - y.zc) * inv_tbz;  // dynamics.hpp:343-346
    const float chi_dot =
        (tbx * (vix - chi * y.wy) + tby * (viy + chi * y.wx) + tbz * viz) * inv_tbz;
    const float f_k = fmaxf(fs_w[w] - k_w[w] * chi, 0.f);  // dynamics.hpp:348-351
    const float f_b = f_k > 0.f ? fmaxf(-b_w[w] * chi_dot, -f_k) : 0.f;
    f_z = f_k + f_b;
    const float alpha = fm::atan_ratio(viy, fmaxf(vix, K.vbx_floor)) - (is_front ? y.de : 0.f);
    const float ca = K.C * alpha;
    const float f_y = f_z * (-ca * K.mu) * fm::rsqrt(K.mu2 + ca * ca);
    Fy = is_front ? f_y * F.cd : f_y;
  };
  if constexpr (L <= 2) {
    // axle-symmetric offsets (rollout_srb_frame.cuh prepare_frame)
    constexpr int NAX = 2 / L;
    const float hw = rho_y[0], rz = rho_z[0];
    const float vxc = fmaf(y.wy, rz, y.vx), vxs = y.wz * hw;
    const float vyc = fmaf(-y.wx, rz, y.vy);
    const float vzs = y.wx * hw;
#pragma unroll
    for (int a = 0; a < NAX; ++a) {
      const float xa = rho_x[2 * a];
      const bool fr = front[2 * a];
      const float viy = fmaf(y.wz, xa, vyc), viz = fmaf(-y.wy, xa, y.vz);
      float fzl, fzr, fyl, fyr;
      axle_pair_forces<W>(F, 2 * a, K, y.z, y.zc, y.wx, y.wy, vxc - vxs, vxc + vxs, viy, viz + vzs,
                          viz - vzs, fs_w[2 * a], k_w[2 * a], b_w[2 * a], fr, y.de, fzl, fzr, fyl,
                          fyr);
      const float fya = fyl + fyr, fza = fzl + fzr;
      fy_sum += fya;
      fz_sum += fza;
      mx = fmaf(hw, fzl - fzr, fmaf(-rz, fya, mx));
      my = fmaf(-xa, fza, fr ? my : fmaf(rz, 2.f * f_x_rear, my));
      mz = fmaf(xa, fya, mz);
    }
  } else {
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const float rx = rho_x[w], ry = rho_y[w], rz = rho_z[w];
      const float vix = y.vx + (y.wy * rz - y.wz * ry);  // v + omega x rho (336)
      const float viy = y.vy + (y.wz * rx - y.wx * rz);
      const float viz = y.vz + (y.wx * ry - y.wy * rx);
      float f_z, Fy;
      wheel(w, vix, viy, viz, front[w], f_z, Fy);
      const float Fx = front[w] ? 0.f : f_x_rear;
      fy_sum += Fy;
      fz_sum += f_z;
      mx += ry * f_z - rz * Fy;
      my += rz * Fx - rx * f_z;
      mz += rx * Fy - ry * Fx;
    }
  }
  fy_sum = group_sum<L>(fy_sum);
  fz_sum = group_sum<L>(fz_sum);
  mx = group_sum<L>(mx);
  my = group_sum<L>(my);
  mz = group_sum<L>(mz);
  Rates d;
  // v_w = R v_b and euler_rates_321 (dynamics.hpp:109-118, 374-389)
  d.x = F.r00 * y.vx + F.r01 * y.vy + F.r02 * y.vz;
  d.y = F.r10 * y.vx + F.r11 * y.vy + F.r12 * y.vz;
  d.z = F.r20 * y.vx + F.r21 * y.vy + F.r22 * y.vz;
  const float inv_ct = fm::rcp(F.cth);
  const float tt = F.sth * inv_ct;
  d.psi = (F.sph * y.wy + F.cph * y.wz) * inv_ct;
  d.th = F.cph * y.wy - F.sph * y.wz;
  d.ph = y.wx + F.sph * tt * y.wy + F.cph * tt * y.wz;
  d.vy = fy_sum * K.inv_M + gby + y.wx * y.vz - y.wz * y.vx;
  d.vz = fz_sum * K.inv_M + gbz - y.wx * y.vy + y.wy * y.vx;
  d.wx = (mx + K.cJx * y.wy * y.wz) * K.inv_Jxx;
  d.wy = (my - K.cJy * y.wx * y.wz) * K.inv_Jyy;
  d.wz = (mz + K.cJz * y.wx * y.wy) * K.inv_Jzz;
  return d;
}

}  // namespace

template <int L, int SD>
__global__ void __launch_bounds__(kBlock, 1) rollout_kernel_rk4_f32(const KParams P,
                                                                   const TerrainDev td,
                                                                   const double* __restrict__ warm,
                                                                   double* __restrict__ out_cost,
                                                                   uint8_t* __restrict__ out_flags,
                                                                   float* __restrict__ out_margin,
                                                                   DevStats* __restrict__ st) {
  l2_prefetch_terrain(P, td);  // the reachable terrain into L2 (rollout_dev.cuh)
  constexpr int W = 4 / L;
  const KConsts<float>& K = P.cf;
  const int lane = threadIdx.x & 31;
  const int s = lane & (L - 1);
  const int gbase = lane & ~(L - 1);
  const int64_t slot = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / L;
  const bool active = slot < P.k_count;
  const int64_t kl = active && P.order ? static_cast<int64_t>(__ldg(P.order + slot)) : slot;
  const int64_t kg = P.k_begin + kl;

  double J = 0.0;
  float margin = __int_as_float(0x7f800000);
  bool feasible = true, diverged = false, goal = false;
  unsigned substeps = 0;

  int ax, ay;
  fm::KS gx, gy;
  {
    const double g0x = P.s0[0] * P.gx_scale + P.gx_off, g0y = P.s0[1] * P.gy_scale + P.gy_off;
    ax = static_cast<int>(floor(g0x));
    ay = static_cast<int>(floor(g0y));
    gx = fm::ks_make(g0x - ax);
    gy = fm::ks_make(g0y - ay);
  }
  const double ggx = P.goal_x * P.gx_scale + P.gx_off, ggy = P.goal_y * P.gy_scale + P.gy_off;
  const int gax = static_cast<int>(floor(ggx)), gay = static_cast<int>(floor(ggy));
  const float gfx = static_cast<float>(ggx - gax), gfy = static_cast<float>(ggy - gay);
  const float rg2 = static_cast<float>(P.goal_r2 * P.gx_scale * P.gy_scale);
  float bx = static_cast<float>(ax - gax) - gfx, by = static_cast<float>(ay - gay) - gfy;
  fm::KS z = fm::ks_make(P.s0[2]);
  fm::KS psi = fm::ks_make(P.s0[3]), th = fm::ks_make(P.s0[4]), ph = fm::ks_make(P.s0[5]);
  fm::KS vx = fm::ks_make(P.s0[6]), vy = fm::ks_make(P.s0[7]), vz = fm::ks_make(P.s0[8]);
  fm::KS wx = fm::ks_make(P.s0[9]), wy = fm::ks_make(P.s0[10]), wz = fm::ks_make(P.s0[11]);
  fm::KS de = fm::ks_make(P.s0[12]);
  const fm::KS de_max = fm::ks_make(P.cd.delta_max), de_min = fm::ks_make(-P.cd.delta_max);
  const float gim = __double2float_rd(P.gimbal_lim);

  float rho_x[W], rho_y[W], rho_z[W], k_w[W], b_w[W], fs_w[W];
  bool front[W];
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const int i = s * W + w;
    rho_x[w] = K.rho[i][0];
    rho_y[w] = K.rho[i][1];
    rho_z[w] = K.rho[i][2];
    k_w[w] = K.k_i[i];
    b_w[w] = K.b_i[i];
    fs_w[w] = K.fs_i[i];
    front[w] = i < 2;
  }

  const uint64_t base = mix64(substream(P.seed, static_cast<uint64_t>(kg)));
  double prev0 = 0.0, prev1 = 0.0;  // random-walk state per channel (sample_step)
  const bool use_sd = SD != 0 && P.enable_dist && P.has_sdist;  // SD = 0 compiles it out
  const bool use_rollover = P.enable_rollover && s == 0;
  const float dt = K.dt;
  const float dt_cells_x = static_cast<float>(P.dt * P.gx_scale);
  const float dt_cells_y = static_cast<float>(P.dt * P.gy_scale);
  const int S = P.S, total = P.n_steps * P.S;

  Frame<W> F;
  Anchor A = make_anchor(P, td, ax, ay);
  prepare_frame<L, W>(F, P, s, gbase, A, gx.s, gy.s, psi.s, th.s, ph.s, de.s, rho_x, rho_y, rho_z,
                      use_sd);
  bool live = active;
  float u_dr = 0.f, u_vr = 0.f;
  double L0 = 0.0;
  float rate_sum = 0.f;
  int nq = 0, q = 0;
  for (int it = 0; it < total; ++it) {
    if (q == 0) {  // ---- ZOH step boundary (warp-uniform), one basic block
      // (see rollout_f32.cu; at it == 0 only the first control is new)
      J += P.dt * ((s == 0 ? static_cast<double>(nq) : 0.0) * L0 + static_cast<double>(rate_sum));
      rate_sum = 0.f;
      nq = 0;
      const float fsum = ((gx.s + gy.s) + (z.s + psi.s)) + ((th.s + ph.s) + (vx.s + vy.s)) +
                         (((vz.s + wx.s) + (wy.s + wz.s)) + de.s);
      const bool bad = !isfinite(fsum);  // dynamics.hpp:491-492
      diverged = diverged || (live && bad);
      live = live && !bad;
      const bool stop = !__any_sync(kFull, live);
      reanchor(live, gx.s, gy.s, ax, ay);
      bx = static_cast<float>(ax - gax) - gfx;
      by = static_cast<float>(ay - gay) - gfy;
      A = make_anchor(P, td, ax, ay);
      double u0, u1;
      zoh_control(P, base, kg == 0, it / S, warm, prev0, prev1, u0, u1);
      u_dr = static_cast<float>(u0);
      u_vr = static_cast<float>(u1);
      L0 = P.w_t + P.w_c * u0 * u0;
      if (stop) break;
    }
    q = q + 1 == S ? 0 : q + 1;

    // ---- goal truncation and the stage-1 gimbal guard
    const float gdx = (bx + gx.s) - gx.c, gdy = (by + gy.s) - gy.c;
    const bool at_goal = live && gdx * gdx + gdy * gdy <= rg2;
    goal = goal || at_goal;
    live = live && !at_goal;
    bool gimbal = live && fabsf(th.s) >= gim && fabs(fm::ks_value(th)) >= P.gimbal_lim;

    // ---- L_soft at the start state (constraints.hpp:16-23, 87-113)
    float rate = 0.f;
    {
      const float sin_abs = ph.s < 0.f ? -F.sph : F.sph;
      const float sin_lever = sin_abs * K.esm_c_pb + F.cph * K.esm_s_pb;
      const float sgn = fabsf(ph.s) <= K.esm_phi_lim ? 1.f : -1.f;
      const float U = sgn * K.esm_Mg * (K.esm_r_bar * (1.f - sin_lever) * F.cth);
      const float a = fmaxf(0.f, 1.f - U * K.inv_eps_esm);
      const bool on = use_rollover && live && !gimbal;
      rate = on ? K.sigma * a * a : 0.f;
      feasible = feasible && (!on || U > 0.f);
      margin = on ? fminf(margin, U * K.inv_esm_nominal) : margin;
    }
    if (use_sd) {
      float srate = 0.f, sd_min = __int_as_float(0x7f800000);
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const float sd = lerp_quad(F.sq[w], F.sfx[w], F.sfy[w]);
        const float a = fmaxf(0.f, 1.f - sd * K.inv_eps_dist);
        srate = fmaf(K.sigma * a, a, srate);
        sd_min = fminf(sd_min, sd);
      }
      const bool on = live && !gimbal;
      rate = on ? rate + srate : rate;
      feasible = feasible && (!on || sd_min > 0.f);
      margin = on ? fminf(margin, sd_min * K.inv_eps_dist) : margin;
    }
    // the reference throws in srb_derivative before the cost of this substep
    // is added only when the guard trips; the cost of the state itself is
    // accumulated by the planner loop first (oracle rollout: cost, then step)
    rate_sum += (live && !gimbal) ? rate : 0.f;
    nq += live && !gimbal;

    // ---- Scheme::kRk4 (dynamics.hpp:454-465)
    StageState y{z.s, z.c, vx.s, vy.s, vz.s, wx.s, wy.s, wz.s, de.s};
    Rates k = srb_rates<L, W>(F, K, y, u_vr, rho_x, rho_y, rho_z, k_w, b_w, fs_w, front);
    Rates acc = k;
    // sin / cos of the substep's start attitude (stage 1); stages 2-4 rotate
    // them by their angle offsets f k (L = 1: 3 x 9 instead of 3 x 22)
    const float b_sps = F.sps, b_cps = F.cps, b_sth = F.sth, b_cth = F.cth, b_sph = F.sph,
                b_cph = F.cph;
    (void)b_sps; (void)b_cps; (void)b_sth; (void)b_cth; (void)b_sph; (void)b_cph;
#pragma unroll 1
    for (int stg = 1; stg < 4; ++stg) {
      const float fr = stg == 3 ? 1.f : 0.5f;
      const float f = fr * dt;
      const float th_y = fm::ks_stage(th, f, k.th);
      gimbal = gimbal || (live && fabsf(th_y) >= gim &&
                          fabs(fm::ks_value(th) + static_cast<double>(f) * k.th) >= P.gimbal_lim);
      const float de_y = fm::ks_stage(de, f, u_dr);
      if constexpr (L == 1 && TMPC_RK4_INCR_TRIG) {
        F.sps = b_sps; F.cps = b_cps; F.sth = b_sth; F.cth = b_cth; F.sph = b_sph; F.cph = b_cph;
        fm::rotate_sc(F.sps, F.cps, f * k.psi);
        fm::rotate_sc(F.sth, F.cth, f * k.th);
        fm::rotate_sc(F.sph, F.cph, f * k.ph);
        prepare_frame<L, W, true>(F, P, s, gbase, A, fm::ks_stage(gx, fr * dt_cells_x, k.x),
                                  fm::ks_stage(gy, fr * dt_cells_y, k.y), 0.f, 0.f, 0.f, de_y, rho_x,
                                  rho_y, rho_z, false);
      } else {
        prepare_frame<L, W>(F, P, s, gbase, A, fm::ks_stage(gx, fr * dt_cells_x, k.x),
                            fm::ks_stage(gy, fr * dt_cells_y, k.y), fm::ks_stage(psi, f, k.psi), th_y,
                            fm::ks_stage(ph, f, k.ph), de_y, rho_x, rho_y, rho_z, false);
      }
      y = StageState{fmaf(f, k.z, z.s), z.c, fm::ks_stage(vx, f, u_vr),
                     fm::ks_stage(vy, f, k.vy), fm::ks_stage(vz, f, k.vz),
                     fm::ks_stage(wx, f, k.wx), fm::ks_stage(wy, f, k.wy),
                     fm::ks_stage(wz, f, k.wz), de_y};
      k = srb_rates<L, W>(F, K, y, u_vr, rho_x, rho_y, rho_z, k_w, b_w, fs_w, front);
      const float wgt = stg == 3 ? 1.f : 2.f;
      acc.x = fmaf(wgt, k.x, acc.x); acc.y = fmaf(wgt, k.y, acc.y); acc.z = fmaf(wgt, k.z, acc.z);
      acc.psi = fmaf(wgt, k.psi, acc.psi); acc.th = fmaf(wgt, k.th, acc.th);
      acc.ph = fmaf(wgt, k.ph, acc.ph); acc.vy = fmaf(wgt, k.vy, acc.vy);
      acc.vz = fmaf(wgt, k.vz, acc.vz); acc.wx = fmaf(wgt, k.wx, acc.wx);
      acc.wy = fmaf(wgt, k.wy, acc.wy); acc.wz = fmaf(wgt, k.wz, acc.wz);
    }
    diverged = diverged || gimbal;
    live = live && !gimbal;
    // s += dt/6 (k1 + 2 k2 + 2 k3 + k4); d_vx = u_vr, d_delta = u_dr in every stage
    const float h6 = live ? dt * (1.f / 6.f) : 0.f;
    const float h = live ? dt : 0.f;
    fm::ks_axpy2(gx, gy, live ? dt_cells_x * (1.f / 6.f) : 0.f, live ? dt_cells_y * (1.f / 6.f) : 0.f,
                 acc.x, acc.y);
    fm::ks_axpy2(z, psi, h6, h6, acc.z, acc.psi);
    fm::ks_axpy2(th, ph, h6, h6, acc.th, acc.ph);
    fm::ks_axpy2(vx, vy, h, h6, u_vr, acc.vy);
    fm::ks_axpy2(vz, wx, h6, h6, acc.vz, acc.wx);
    fm::ks_axpy2(wy, wz, h6, h6, acc.wy, acc.wz);
    fm::ks_axpy(de, h, u_dr);
    fm::ks_clamp(de, de_min, de_max);
    substeps += live;
    // ---- stage-1 frame of the next substep: gathers cross the back-edge
    prepare_frame<L, W>(F, P, s, gbase, A, gx.s, gy.s, psi.s, th.s, ph.s, de.s, rho_x, rho_y,
                        rho_z, use_sd);
  }
  J += P.dt * ((s == 0 ? static_cast<double>(nq) : 0.0) * L0 + static_cast<double>(rate_sum));
  {
    const float fsum = gx.s + gy.s + z.s + psi.s + th.s + ph.s + vx.s + vy.s + vz.s + wx.s + wy.s +
                       wz.s + de.s;
    diverged = diverged || (live && !isfinite(fsum));
  }
  if constexpr (L > 1) {
#pragma unroll
    for (int o = 1; o < L; o <<= 1) {
      J += __shfl_xor_sync(kFull, J, o);
      margin = fminf(margin, __shfl_xor_sync(kFull, margin, o));
      feasible = __shfl_xor_sync(kFull, static_cast<int>(feasible), o) && feasible;
    }
  }
  const bool owner = active && s == 0;
  if (owner) {
    if (diverged) {
      J = __longlong_as_double(0x7ff0000000000000LL);
      feasible = false;
      margin = __int_as_float(0xff800000);
    } else {
      const double x = ((ax - P.gx_off) + (static_cast<double>(gx.s) - gx.c)) / P.gx_scale;
      const double yy = ((ay - P.gy_off) + (static_cast<double>(gy.s) - gy.c)) / P.gy_scale;
      const double gdx = x - P.goal_x, gdy = yy - P.goal_y;
      J += P.w_g * sqrt(gdx * gdx + gdy * gdy);
    }
  }
  reduce_and_finalize(P, owner, kl, kg, J, feasible, diverged, goal, margin,
                      owner ? substeps : 0u, out_cost, out_flags, out_margin, st);
}

void launch_rollout_rk4_f32(int lanes, const KParams& P, const TerrainDev& td, const double* warm,
                            double* cost, uint8_t* flags, float* margin, DevStats* st,
                            cudaStream_t stream) {
  const unsigned blocks = static_cast<unsigned>((P.k_count * lanes + kBlock - 1) / kBlock);
  const bool sd = P.enable_dist && P.has_sdist;
#define TMPC_LAUNCH(LN, SDV) \
  launch(rollout_kernel_rk4_f32<LN, SDV>, blocks, kBlock, stream, P, td, warm, cost, flags, margin, st)
  if (lanes == 4) {
    if (sd) TMPC_LAUNCH(4, 1); else TMPC_LAUNCH(4, 0);
  } else if (lanes == 2) {
    if (sd) TMPC_LAUNCH(2, 1); else TMPC_LAUNCH(2, 0);
  } else {
    if (sd) TMPC_LAUNCH(1, 1); else TMPC_LAUNCH(1, 0);
  }
#undef TMPC_LAUNCH
}

cudaError_t configure_rollout_rk4_f32() {
  cudaError_t e = cudaSuccess;
  const auto carve = [&](const void* f) {
    const cudaError_t r = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
    if (r != cudaSuccess) e = r;
  };
  carve(reinterpret_cast<const void*>(rollout_kernel_rk4_f32<1, 0>));
  carve(reinterpret_cast<const void*>(rollout_kernel_rk4_f32<2, 0>));
  carve(reinterpret_cast<const void*>(rollout_kernel_rk4_f32<4, 0>));
  carve(reinterpret_cast<const void*>(rollout_kernel_rk4_f32<1, 1>));
  carve(reinterpret_cast<const void*>(rollout_kernel_rk4_f32<2, 1>));
  carve(reinterpret_cast<const void*>(rollout_kernel_rk4_f32<4, 1>));
  return e;
}

}  // namespace tmpcb
