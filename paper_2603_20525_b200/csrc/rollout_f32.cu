// fp32 fast path of the fused rollout + cost + feasibility + arg-min kernel
// (same per-candidate algorithm as rollout.cu).
//
// Decomposition: L lanes (1, 2 or 4) of a warp share one candidate.  Lane s
// of the group owns wheels {s*W .. s*W+W-1} (W = 4/L): their contact-point
// terrain gathers, suspension / tire forces and planar-footprint SDF soft
// costs.  Body work is split where it is SIMT-parallel (lane s evaluates
// sin/cos of the attitude angles j = s mod L, shared by shuffles) and
// replicated otherwise; the per-wheel force / moment sums are combined with
// an xor-shuffle butterfly, which gives every lane bit-identical sums, so all
// lanes of a group integrate bit-identical states.  L = 4 exposes 4x the
// warps for the small per-GPU batches (K = 16-32 K on 148 SMs is < 1 warp per
// scheduler at one thread per candidate), L = 1 has the fewest instructions
// for large batches; the launcher picks L from K.
//
// Control flow is warp-uniform: every lane runs every substep of a ZOH step;
// goal truncation, the gimbal guard and divergence become a per-candidate
// `live` predicate that freezes the state (zero time step) and masks the cost
// accumulation, and the warp leaves the horizon loop once no lane is live.
//
// Software pipelining of the terrain gathers: a substep's contact points
// depend only on positions and attitude, and forward Euler advances those
// from the previous state alone, so the loop runs (1) the gather-independent
// head (goal / gimbal predicates, ESM, Euler rates, v_w), (2) the Euler step
// of the kinematic half of the state (x, y, z, psi, theta, phi, delta),
// (3) the wheel forces from the frame gathered one substep earlier, then
// (4) rebuilds that frame in place for substep n+1 (trig, rotation, cells,
// gathers) and (5) finishes with the velocity update.  The gathers are in
// flight during (5), across the back-edge (ptxas cannot sink them next to
// their use) and through the next head; the frame is never copied and holds
// the registers of one substep only.  (Measured, c2: issuing the gathers at
// the very end of the iteration left 30% of all stall samples on their first
// consumer; this order cut the cycle by 20%.)
//
// Arithmetic (all FFMA-pipe, no fp64 or XU conversion on the substep's
// critical path): branch-free math (fastmath.cuh); Kahan-compensated fp32
// state (fp64-grade over 1000 increments); the planar position kept in
// padded-grid cell units as an integer anchor + compensated fp32 offset,
// re-anchored every ZOH step (cell index and fraction of a wheel are then a
// magic-number floor of a small fp32 sum; world x, y are rebuilt in fp64 only
// for the terminal cost); the running cost of a ZOH step summed in fp32
// before one fp64 accumulate; sin / cos of the three attitude angles
// evaluated exactly every substep (TMPC_INCR_TRIG=0: carrying them by the
// angle-addition formulas between ZOH steps is 2.7% faster at c2 but
// accumulates ~2.5 ulp per substep, which the full-size parity rule does not
// allow).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "fastmath.cuh"
#include "rollout_anchor.cuh"
#include "rollout_srb_frame.cuh"
#include "launch.cuh"
#include "rollout.cuh"
#include "rollout_dev.cuh"
#include "tmpc_common.h"

// Build-time variant switch for A/B timing (tools/variants.py, tools/ab.py):
// TMPC_INCR_TRIG=0 evaluates sin/cos of psi, theta, phi every substep.
#ifndef TMPC_INCR_TRIG
#define TMPC_INCR_TRIG 0  // exact sin/cos per substep: parity, +2.5% c2
#endif
// TMPC_QT_SD=1 also routes the third contact-point quad through TEX in the
// large-batch launches with the footprint term (c4 -1%: the TEX pipe then
// carries 8 of the 12 gathers of a substep, the L1 LSU pipe 4).
#ifndef TMPC_QT_SD
#define TMPC_QT_SD 1
#endif
// TMPC_PACKED_AXLE=0 computes the two wheels of an axle with scalar code,
// 1 packed, 2 as the PK template flag says (packed for large problems).
#ifndef TMPC_PACKED_AXLE
#define TMPC_PACKED_AXLE 2  // c2 -0.75% scalar, c4 packed (A/B, v21)
#endif
// TMPC_SD_SKIP=1: in the throughput-path launches (QT), a warp whose
// candidates are all provably clear of the footprint obstacle term for the
// next substep skips the term's cells, gathers and soft cost (bit-identical:
// only where it adds exactly 0 and cannot lower the margin; see the loop).
// Latency-bound launches keep the straight-line body (c2 +4.5% with it).
#ifndef TMPC_SD_SKIP
#define TMPC_SD_SKIP 1
#endif

namespace tmpcb {


// SD = 0: no footprint obstacle term (ConstraintConfig::enable_dist off or a
// signed-distance map without features) -- compiled out, so the substep path
// is one basic block with ~35 fewer registers (c3 -5%, c5 -8%).
// QT: gather path of a throughput-bound batch (third contact-point quad via
// TEX, footprint SDF via LDG), from this launch's own K -- it moves loads,
// not arithmetic.  PK: axle wheels as fp32x2 pairs, from the whole problem's
// K -- it changes the rounding, so every shard of a G-GPU solve must agree.
template <int L, int SD, int QT, int PK>
__global__ void __launch_bounds__(4 * kBlock, 1) rollout_kernel_f32(const KParams P, const TerrainDev td,
                                                             const double* __restrict__ warm,
                                                             double* __restrict__ out_cost,
                                                             uint8_t* __restrict__ out_flags,
                                                             float* __restrict__ out_margin,
                                                             DevStats* __restrict__ st) {
  l2_prefetch_terrain(P, td);  // the reachable terrain into L2 (rollout_dev.cuh)
  constexpr int W = 4 / L;  // wheels per lane
  const KConsts<float>& K = P.cf;
  const int lane = threadIdx.x & 31;
  const int s = lane & (L - 1);       // index within the candidate group
  const int gbase = lane & ~(L - 1);  // first lane of the group
  const int64_t slot = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / L;
  const bool active = slot < P.k_count;
  // the candidate of this slot: path-ordered for terrain locality (order.cu)
  const int64_t kl = active && P.order ? static_cast<int64_t>(__ldg(P.order + slot)) : slot;
  const int64_t kg = P.k_begin + kl;

  double J = 0.0;
  float margin = __int_as_float(0x7f800000);  // +inf
  bool feasible = true, diverged = false, goal = false;
  unsigned substeps = 0;

  // planar position in padded-grid cells: anchor (int) + compensated offset
  int ax, ay;
  fm::KS gx, gy;
  {
    const double g0x = P.s0[0] * P.gx_scale + P.gx_off, g0y = P.s0[1] * P.gy_scale + P.gy_off;
    ax = static_cast<int>(floor(g0x));
    ay = static_cast<int>(floor(g0y));
    gx = fm::ks_make(g0x - ax);
    gy = fm::ks_make(g0y - ay);
  }
  // goal circle in cells: anchor + fraction, radius^2
  const double ggx = P.goal_x * P.gx_scale + P.gx_off, ggy = P.goal_y * P.gy_scale + P.gy_off;
  const int gax = static_cast<int>(floor(ggx)), gay = static_cast<int>(floor(ggy));
  const float gfx = static_cast<float>(ggx - gax), gfy = static_cast<float>(ggy - gay);
  const float rg2 = static_cast<float>(P.goal_r2 * P.gx_scale * P.gy_scale);
  float bx = static_cast<float>(ax - gax) - gfx, by = static_cast<float>(ay - gay) - gfy;
  // the rest of the state, compensated fp32 (SrbState order, dynamics.hpp:167-172)
  fm::KS z = fm::ks_make(P.s0[2]);
  fm::KS psi = fm::ks_make(P.s0[3]), th = fm::ks_make(P.s0[4]), ph = fm::ks_make(P.s0[5]);
  fm::KS vx = fm::ks_make(P.s0[6]), vy = fm::ks_make(P.s0[7]), vz = fm::ks_make(P.s0[8]);
  fm::KS wx = fm::ks_make(P.s0[9]), wy = fm::ks_make(P.s0[10]), wz = fm::ks_make(P.s0[11]);
  fm::KS de = fm::ks_make(P.s0[12]);
  const fm::KS de_max = fm::ks_make(P.cd.delta_max), de_min = fm::ks_make(-P.cd.delta_max);
  const float gim = __double2float_rd(P.gimbal_lim);  // <= the fp64 limit; refined below

  // this lane's wheel constants (dynamics.hpp:188-192,322-324,348)
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
  // launched with SD = 1 only when the term is on: a compile-time flag (v22:
  // c2 -0.8%, c4 -1.6% against the runtime test an older schedule preferred)
  constexpr bool use_sd = SD != 0;
  constexpr bool skip_sd = use_sd && L == 1 && (TMPC_SD_SKIP == 2 || (QT != 0 && TMPC_SD_SKIP));
  const bool use_rollover = P.enable_rollover && s == 0;  // the ESM term lives in lane 0
  const float dt = K.dt;
  const float dt_cells_x = static_cast<float>(P.dt * P.gx_scale);
  const float dt_cells_y = static_cast<float>(P.dt * P.gy_scale);
  const int S = P.S, total = P.n_steps * P.S;

  Frame<W> F;
  Anchor A = make_anchor(P, td, ax, ay);
  prepare_frame<L, W, false, QT != 0, skip_sd>(F, P, s, gbase, A, gx.s, gy.s, psi.s, th.s, ph.s,
                                               de.s, rho_x, rho_y, rho_z, use_sd);
  bool live = active;
  float u_dr = 0.f, u_vr = 0.f;
  double L0 = 0.0;
  float rate_sum = 0.f;  // this lane's share of sum L_soft over the ZOH step
  int nq = 0;
  int q = 0;
  for (int it = 0; it < total; ++it) {
    if (q == 0) {  // ---- ZOH step boundary (warp-uniform)
      // One basic block for the common samplers, so ptxas overlaps its
      // independent chains (cost accumulation, divergence test, re-anchor,
      // exact trig, the fp64 control draw): as separate blocks they ran back
      // to back, ~8% of c2's time.  At it == 0 the block is a no-op except for
      // the first control (the accumulators are zero, s0 is finite, gx, gy in
      // [0, 1) do not re-anchor).
      J += P.dt * ((s == 0 ? static_cast<double>(nq) : 0.0) * L0 + static_cast<double>(rate_sum));
      rate_sum = 0.f;
      nq = 0;
      // non-finite values persist in the accumulators, so one test per ZOH
      // step flags the same candidates as the per-substep test
      // (dynamics.hpp:491-492)
      const float fsum = ((gx.s + gy.s) + (z.s + psi.s)) + ((th.s + ph.s) + (vx.s + vy.s)) +
                         (((vz.s + wx.s) + (wy.s + wz.s)) + de.s);
      const bool bad = !isfinite(fsum);
      diverged = diverged || (live && bad);
      live = live && !bad;
      const bool stop = !__any_sync(kFull, live);  // warp-uniform exit, taken below
      reanchor(live, gx.s, gy.s, ax, ay);  // rollout_anchor.cuh
      bx = static_cast<float>(ax - gax) - gfx;
      by = static_cast<float>(ay - gay) - gfy;
      A = make_anchor(P, td, ax, ay);
#if TMPC_INCR_TRIG
      if constexpr (L == 1) {  // re-sync the rotated attitude trig once per ZOH step
        fm::sincos(psi.s, &F.sps, &F.cps);
        fm::sincos(th.s, &F.sth, &F.cth);
        fm::sincos(ph.s, &F.sph, &F.cph);
      }
#endif
      double u0, u1;
      zoh_control(P, base, kg == 0, it / S, warm, prev0, prev1, u0, u1);  // rollout_dev.cuh
      u_dr = static_cast<float>(u0);
      u_vr = static_cast<float>(u1);
      L0 = P.w_t + P.w_c * u0 * u0;
      if (stop) break;
    }
    q = q + 1 == S ? 0 : q + 1;

    // ---- goal truncation before accumulating and the
    // srb_derivative gimbal guard (dynamics.hpp:311-312) as predicates
    const float gdx = (bx + gx.s) - gx.c, gdy = (by + gy.s) - gy.c;
    const bool at_goal = live && gdx * gdx + gdy * gdy <= rg2;
    goal = goal || at_goal;
    live = live && !at_goal;
    const bool gimbal = live && fabsf(th.s) >= gim && fabs(fm::ks_value(th)) >= P.gimbal_lim;
    diverged = diverged || gimbal;
    live = live && !gimbal;

    // ---- phase C: gather-independent terms
    float rate = 0.f;
    {
      // esm (constraints.hpp:16-23); sin(|phi|+phi_bar) by the angle sum
      const float sin_abs = ph.s < 0.f ? -F.sph : F.sph;
      const float sin_lever = sin_abs * K.esm_c_pb + F.cph * K.esm_s_pb;
      const float sgn = fabsf(ph.s) <= K.esm_phi_lim ? 1.f : -1.f;
      const float U = sgn * K.esm_Mg * (K.esm_r_bar * (1.f - sin_lever) * F.cth);
      const float a = fmaxf(0.f, 1.f - U * K.inv_eps_esm);
      const bool on = use_rollover && live;
      rate = on ? K.sigma * a * a : 0.f;
      feasible = feasible && (!on || U > 0.f);
      margin = on ? fminf(margin, U * K.inv_esm_nominal) : margin;
    }
    const float gbx = F.r20 * (-K.g), gby = F.r21 * (-K.g), gbz = F.r22 * (-K.g);
    const float f_x_rear = K.half_M * (u_vr - gbx + wy.s * vz.s - wz.s * vy.s);
    // euler_rates_321 (dynamics.hpp:109-118) and v_w = R v_b (374)
    const float inv_ct = fm::rcp(F.cth);
    const float tt = F.sth * inv_ct;
    const float d_psi = (F.sph * wy.s + F.cph * wz.s) * inv_ct;
    const float d_th = F.cph * wy.s - F.sph * wz.s;
    const float d_ph = wx.s + F.sph * tt * wy.s + F.cph * tt * wz.s;
    const float dxw = F.r00 * vx.s + F.r01 * vy.s + F.r02 * vz.s;
    const float dyw = F.r10 * vx.s + F.r11 * vy.s + F.r12 * vz.s;
    const float dzw = F.r20 * vx.s + F.r21 * vy.s + F.r22 * vz.s;

    // ---- forward Euler of the kinematic half of the state (dynamics.hpp:
    // 423-441,453,466): positions, attitude and steering at n+1 depend only
    // on state n; a frozen (goal / diverged) candidate integrates with a
    // zero step
    const float h = live ? dt : 0.f;
    const float zs_n = z.s, zc_n = z.c, de_n = de.s;  // state-n values the forces read
    fm::ks_axpy2(gx, gy, live ? dt_cells_x : 0.f, live ? dt_cells_y : 0.f, dxw, dyw);
    fm::ks_axpy2(z, psi, h, h, dzw, d_psi);
    fm::ks_axpy2(th, ph, h, h, d_th, d_ph);
    fm::ks_axpy(de, h, u_dr);
    fm::ks_clamp(de, de_min, de_max);

    // ---- phase D: consume the gathers
    if (use_sd && (!skip_sd || F.sd_on)) {
      // soft_cost_rate(-sd) per footprint point; the minimum over the
      // lane's points decides feasibility (sd > 0) and the margin (sd / eps
      // is monotone in sd), so the live mask is applied once
      float srate = 0.f, sd_min = __int_as_float(0x7f800000);
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const float sd = lerp_quad(F.sq[w], F.sfx[w], F.sfy[w]);
        const float a = fmaxf(0.f, 1.f - sd * K.inv_eps_dist);
        srate = fmaf(K.sigma * a, a, srate);
        sd_min = fminf(sd_min, sd);
      }
      rate = live ? rate + srate : rate;
      feasible = feasible && (!live || sd_min > 0.f);
      margin = live ? fminf(margin, sd_min * K.inv_eps_dist) : margin;
    }
    rate_sum += rate;
    nq += live;
    float fy_sum = 0.f, fz_sum = 0.f, mx = 0.f, my = 0.f, mz = 0.f;
    // per-wheel suspension + tire model (dynamics.hpp:333-371) from the
    // point velocity, the terrain plane and the extension of one wheel
    const auto wheel = [&](int w, float vix, float viy, float viz, bool is_front, float& f_z,
                           float& Fy) {
      const float h = lerp_quad(F.qh[w], F.hfx[w], F.hfy[w]);
      const float gsx = lerp_quad(F.qx[w], F.hfx[w], F.hfy[w]);
      const float gsy = lerp_quad(F.qy[w], F.hfx[w], F.hfy[w]);
      // tau_b = R^T (-fx, -fy, 1) (dynamics.hpp:339-341)
      const float tbx = F.r20 - F.r00 * gsx - F.r10 * gsy;
      const float tby = F.r21 - F.r01 * gsx - F.r11 * gsy;
      const float tbz = F.r22 - F.r02 * gsx - F.r12 * gsy;
      const float inv_tbz = fm::rcp(fmaxf(tbz, K.tau_floor));
      // extension and rate (dynamics.hpp:343-346); z compensated (value zs - zc)
      const float chi = (((zs_n - h) + F.rwz[w]) - zc_n) * inv_tbz;
      const float chi_dot = (tbx * (vix - chi * wy.s) + tby * (viy + chi * wx.s) + tbz * viz) * inv_tbz;
      // suspension (dynamics.hpp:348-351)
      const float f_k = fmaxf(fs_w[w] - k_w[w] * chi, 0.f);
      const float f_b = f_k > 0.f ? fmaxf(-b_w[w] * chi_dot, -f_k) : 0.f;
      f_z = f_k + f_b;
      // slip and tire (dynamics.hpp:353-356, 74-77)
      const float alpha = fm::atan_ratio(viy, fmaxf(vix, K.vbx_floor)) - (is_front ? de_n : 0.f);
      const float ca = K.C * alpha;
      const float f_y = f_z * (-ca * K.mu) * fm::rsqrt(K.mu2 + ca * ca);
      Fy = is_front ? f_y * F.cd : f_y;
    };
    if constexpr (L <= 2) {
      // axle-symmetric offsets (see prepare_frame): v_i = v + omega x rho
      // (dynamics.hpp:336) shares its terms between wheels, and the moment
      // sum rho x F (358-362) collapses to per-axle / per-side force sums
      constexpr int NAX = 2 / L;
      const float hw = rho_y[0], rz = rho_z[0];
      const float vxc = fmaf(wy.s, rz, vx.s), vxs = wz.s * hw;  // vix = vxc -+ vxs
      const float vyc = fmaf(-wx.s, rz, vy.s);
      const float vzs = wx.s * hw;  // viz = viz_a +- vzs
#pragma unroll
      for (int a = 0; a < NAX; ++a) {
        const float xa = rho_x[2 * a];
        const bool fr = front[2 * a];
        const float viy = fmaf(wz.s, xa, vyc), viz = fmaf(-wy.s, xa, vz.s);
        float fzl, fzr, fyl, fyr;
        if (TMPC_PACKED_AXLE == 1 || (TMPC_PACKED_AXLE == 2 && PK != 0)) {
          axle_pair_forces<W>(F, 2 * a, K, zs_n, zc_n, wx.s, wy.s, vxc - vxs, vxc + vxs, viy,
                              viz + vzs, viz - vzs, fs_w[2 * a], k_w[2 * a], b_w[2 * a], fr, de_n,
                              fzl, fzr, fyl, fyr);
        } else {
          wheel(2 * a, vxc - vxs, viy, viz + vzs, fr, fzl, fyl);
          wheel(2 * a + 1, vxc + vxs, viy, viz - vzs, fr, fzr, fyr);
        }
        const float fya = fyl + fyr, fza = fzl + fzr;
        fy_sum += fya;
        fz_sum += fza;
        mx = fmaf(hw, fzl - fzr, fmaf(-rz, fya, mx));
        my = fmaf(-xa, fza, fr ? my : fmaf(rz, 2.f * f_x_rear, my));
        mz = fmaf(xa, fya, mz);  // the rear F_x pair cancels about z
      }
      fy_sum = group_sum<L>(fy_sum);
      fz_sum = group_sum<L>(fz_sum);
      mx = group_sum<L>(mx);
      my = group_sum<L>(my);
      mz = group_sum<L>(mz);
    } else {
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const float rx = rho_x[w], ry = rho_y[w], rz = rho_z[w];
        // point velocity v_i = v + omega x rho (dynamics.hpp:336)
        const float vix = vx.s + (wy.s * rz - wz.s * ry);
        const float viy = vy.s + (wz.s * rx - wx.s * rz);
        const float viz = vz.s + (wx.s * ry - wy.s * rx);
        float f_z, Fy;
        wheel(w, vix, viy, viz, front[w], f_z, Fy);
        // sums and moment rho x F (dynamics.hpp:358-362)
        const float Fx = front[w] ? 0.f : f_x_rear;
        fy_sum += Fy;
        fz_sum += f_z;
        mx += ry * f_z - rz * Fy;
        my += rz * Fx - rx * f_z;
        mz += rx * Fy - ry * Fx;
      }
      fy_sum = group_sum<L>(fy_sum);
      fz_sum = group_sum<L>(fz_sum);
      mx = group_sum<L>(mx);
      my = group_sum<L>(my);
      mz = group_sum<L>(mz);
    }
    // ---- phase A + B of substep n+1 (its kinematic state is final and the
    // frame of substep n is consumed, so it is rebuilt in place): the gathers
    // are in flight during the velocity update below and the next loop head
    bool sd_fetch = true;
    if constexpr (skip_sd) {
      // F.cl (gathered with frame n) bounds the SDF of every footprint point
      // of a CoM within kClearWindowMove cells of the CoM of substep n (the
      // store's clearance window, ctx.cu footprint_clearance); the CoM moves
      // by this substep's kinematic increment.  A lane is clear when its
      // bound gives a zero soft cost (sd / eps >= kClearCost) and cannot lower
      // the margin (fl(sd / eps) >= fl(bound / eps) >= margin: rounding is
      // monotone, and the margin only decreases): the term then leaves cost,
      // feasibility and margin exactly as they are.  NaN tests false.
      const float lb = F.cl * K.inv_eps_dist;
      const bool clear = lb >= fmaxf(kClearCost, margin) &&
                         fabsf(dxw) * dt_cells_x <= kClearMove &&
                         fabsf(dyw) * dt_cells_y <= kClearMove;
      sd_fetch = __any_sync(kFull, live && !clear);
    }
#if TMPC_INCR_TRIG
    if constexpr (L == 1) {
      // attitude trig of substep n+1: sin / cos of psi, theta, phi rotated by
      // this substep's angle increments (re-synced exactly at every ZOH
      // step, see the boundary block): 3 x 9 instead of 3 x 22 instructions
      fm::rotate_sc(F.sps, F.cps, h * d_psi);
      fm::rotate_sc(F.sth, F.cth, h * d_th);
      fm::rotate_sc(F.sph, F.cph, h * d_ph);
      prepare_frame<L, W, true, QT != 0, skip_sd>(F, P, s, gbase, A, gx.s, gy.s, psi.s, th.s, ph.s,
                                                  de.s, rho_x, rho_y, rho_z, use_sd, sd_fetch);
    } else
#endif
    prepare_frame<L, W, false, QT != 0, skip_sd>(F, P, s, gbase, A, gx.s, gy.s, psi.s, th.s, ph.s,
                                                 de.s, rho_x, rho_y, rho_z, use_sd, sd_fetch);
    const float d_vy = fy_sum * K.inv_M + gby + wx.s * vz.s - wz.s * vx.s;
    const float d_vz = fz_sum * K.inv_M + gbz - wx.s * vy.s + wy.s * vx.s;
    const float d_wx = (mx + K.cJx * wy.s * wz.s) * K.inv_Jxx;
    const float d_wy = (my - K.cJy * wx.s * wz.s) * K.inv_Jyy;
    const float d_wz = (mz + K.cJz * wx.s * wy.s) * K.inv_Jzz;
    // ---- forward Euler of the velocities (dynamics.hpp:446-453)
    fm::ks_axpy2(vx, vy, h, h, u_vr, d_vy);
    fm::ks_axpy2(vz, wx, h, h, d_vz, d_wx);
    fm::ks_axpy2(wy, wz, h, h, d_wy, d_wz);
    substeps += live;
  }
  J += P.dt * ((s == 0 ? static_cast<double>(nq) : 0.0) * L0 + static_cast<double>(rate_sum));
  {
    const float fsum = gx.s + gy.s + z.s + psi.s + th.s + ph.s + vx.s + vy.s + vz.s + wx.s + wy.s +
                       wz.s + de.s;
    diverged = diverged || (live && !isfinite(fsum));
  }

  // combine the group's partial cost / margin / feasibility into lane s == 0
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
      // world position from the cell representation (g' = (x - ox)/r + 2)
      const double x = ((ax - P.gx_off) + (static_cast<double>(gx.s) - gx.c)) / P.gx_scale;
      const double y = ((ay - P.gy_off) + (static_cast<double>(gy.s) - gy.c)) / P.gy_scale;
      const double gdx = x - P.goal_x, gdy = y - P.goal_y;
      J += P.w_g * sqrt(gdx * gdx + gdy * gdy);
    }
  }
  reduce_and_finalize(P, owner, kl, kg, J, feasible, diverged, goal, margin,
                      owner ? substeps : 0u, out_cost, out_flags, out_margin, st);
}

// Lanes per candidate for a shard of k candidates (measured on B200,
// tools/sweep_lanes.py): one lane per candidate once the batch gives ~0.55
// warps per scheduler (c2: K >= ~10 K), two down to ~0.3, four below, where
// the latency of one substep, not issue, bounds the cycle.
int pick_lanes(int64_t k, int sms) {
  const double warps_per_sched_l1 = static_cast<double>(k) / 32.0 / (4.0 * sms);
  if (warps_per_sched_l1 >= 0.55) return 1;
  if (warps_per_sched_l1 >= 0.3) return 2;
  return 4;
}

// The kernels use no shared memory: give the whole unified L1/shared array
// to L1 (terrain records of the resident candidates stay cached longer).
cudaError_t configure_rollout_f32() {
  cudaError_t e = cudaSuccess;
  const auto carve = [&](const void* f) {
    const cudaError_t r = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
    if (r != cudaSuccess) e = r;
  };
  carve(reinterpret_cast<const void*>(rollout_kernel_f32<1, 0, 0, 0>));
  carve(reinterpret_cast<const void*>(rollout_kernel_f32<1, 0, 0, 1>));
  carve(reinterpret_cast<const void*>(rollout_kernel_f32<1, 0, 1, 0>));
  carve(reinterpret_cast<const void*>(rollout_kernel_f32<1, 0, 1, 1>));
  carve(reinterpret_cast<const void*>(rollout_kernel_f32<1, 1, 0, 0>));
  carve(reinterpret_cast<const void*>(rollout_kernel_f32<1, 1, 0, 1>));
  carve(reinterpret_cast<const void*>(rollout_kernel_f32<1, 1, 1, 0>));
  carve(reinterpret_cast<const void*>(rollout_kernel_f32<1, 1, 1, 1>));
  carve(reinterpret_cast<const void*>(rollout_kernel_f32<2, 0, 0, 0>));
  carve(reinterpret_cast<const void*>(rollout_kernel_f32<2, 1, 0, 0>));
  carve(reinterpret_cast<const void*>(rollout_kernel_f32<4, 0, 0, 0>));
  carve(reinterpret_cast<const void*>(rollout_kernel_f32<4, 1, 0, 0>));
  return e;
}

// Launch configuration: lanes per candidate (pick_lanes, from the whole
// problem), the footprint term (SD), for one-lane launches with >= 2 warps per
// scheduler the throughput gather path (QT: at K = 65 K the L1 data pipe, not
// latency, limits; from this launch's K) and the packed axle wheels (PK: from
// the whole problem's K, so the rounding is the same on every shard).
void launch_rollout_f32(int lanes, const KParams& P, const TerrainDev& td, const double* warm,
                        double* cost, uint8_t* flags, float* margin, DevStats* st,
                        cudaStream_t stream) {
  const bool sd = P.enable_dist && P.has_sdist;
  // the throughput gather path from 32 K candidates per launch without the
  // footprint term (c3 / c5 shards of 32 K: -4% / -2% with it), from 128 K
  // with it: c4 shards of 32 K / 64 K (8 / 4 GPUs) run 16% / 9% faster on
  // the latency gather path (footprint SDF via TEX, contact quads via LDG;
  // 1.019 vs 1.212 ms, 2.243 vs 2.475 ms), 128 K is even
#ifndef TMPC_QT_MIN
#define TMPC_QT_MIN 32768
#endif
#ifndef TMPC_QT_MIN_SD
#define TMPC_QT_MIN_SD 131072
#endif
  const bool qt = P.k_count >= (sd ? TMPC_QT_MIN_SD : TMPC_QT_MIN) && (TMPC_QT_SD || !sd);
  const bool pk = P.k_layout >= 32768;
  // one-warp CTAs spread a latency-bound batch over every SM; four-warp CTAs
  // keep a throughput-bound one's warps evenly over the four schedulers of an
  // SM as CTAs retire and refill (c4 -1.4%, c2 +2.5% with them) -- from 64 K
  // candidates per launch: a 32 K shard (c4 on 8 GPUs) runs 5.6% faster with
  // one-warp CTAs (1.164 vs 1.233 ms; 64 K equal, 131 K 4.07 vs 3.58 ms)
#ifndef TMPC_QT_WARPS
#define TMPC_QT_WARPS 4
#endif
  const int bs = qt && P.k_count >= 65536 ? TMPC_QT_WARPS * kBlock : kBlock;
  const unsigned blocks = static_cast<unsigned>((P.k_count * lanes + bs - 1) / bs);
#define TMPC_LAUNCH(LN, SDV, QTV, PKV) \
  launch(rollout_kernel_f32<LN, SDV, QTV, PKV>, blocks, bs, stream, P, td, warm, cost, flags, margin, st)
#define TMPC_LAUNCH1(SDV)                         \
  do {                                            \
    if (qt && pk) TMPC_LAUNCH(1, SDV, 1, 1);      \
    else if (qt) TMPC_LAUNCH(1, SDV, 1, 0);       \
    else if (pk) TMPC_LAUNCH(1, SDV, 0, 1);       \
    else TMPC_LAUNCH(1, SDV, 0, 0);               \
  } while (0)
  if (lanes == 4) {
    if (sd) TMPC_LAUNCH(4, 1, 0, 0); else TMPC_LAUNCH(4, 0, 0, 0);
  } else if (lanes == 2) {
    if (sd) TMPC_LAUNCH(2, 1, 0, 0); else TMPC_LAUNCH(2, 0, 0, 0);
  } else if (sd) {
    TMPC_LAUNCH1(1);
  } else {
    TMPC_LAUNCH1(0);
  }
#undef TMPC_LAUNCH1
#undef TMPC_LAUNCH
}

}  // namespace tmpcb
