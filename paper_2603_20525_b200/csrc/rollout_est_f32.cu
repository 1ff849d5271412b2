// fp32 fast path of the EST formulation: the paper's
// baseline extended single-track model (dynamics.hpp:147-275) with the
// lateral-acceleration rollover constraint (constraints.hpp:62-65,78-80) and
// the footprint obstacle costs, forward Euler or RK4 (dynamics.hpp:446-468).
// The per-candidate algorithm is oracle/tmpc_oracle.cpp rollout_est; the fp64
// certification kernel is rollout_est.cu.
//
// One thread per candidate (an EST substep reads one terrain record at the
// CoM plus four footprint SDF quads).  Same machinery as the SRB fast path
// (rollout_f32.cu): the planar position as a cell anchor + compensated fp32
// offset (rollout_anchor.cuh), every other state entry Kahan-compensated,
// branch-free elementary functions, warp-uniform control flow (goal / divergence
// are a `live` predicate, the warp leaves once no lane is live).
//
// The critical path of a substep is the chain CoM gather -> plane attitude ->
// planar velocity -> next CoM cell, so the attitude avoids transcendental
// round trips: est_plane_attitude (dynamics.hpp:213-219) takes theta =
// asin(tau_x) and phi = asin(sphi) and rot_123 (84-93) then only needs their
// sines and cosines, which are sin(asin(a)) = a and cos(asin(a)) = sqrt(1-a^2)
// (theta, phi in [-pi/2, pi/2]): one rsqrt each instead of asin + sincos.
// The slip angles, tire saturation terms and cos(delta) depend on the state
// alone and sit off that chain; so do the footprint SDF gathers (x, y, psi).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "fastmath.cuh"
#include "launch.cuh"
#include "rollout.cuh"
#include "rollout_anchor.cuh"
#include "rollout_dev.cuh"
#include "tmpc_common.h"

// The footprint SDF quads through the TEX pipe in the large-batch launches
// (TEX template flag: c4 -5%; a latency-bound c2 batch +20%, so LDG there).
// Euler: sin / cos psi carried by angle addition between ZOH steps (c2 -0.9%,
// c3 -3.2%; RK4 +2.3%, so RK4 keeps the exact sincos)
#ifndef TMPC_EST_INCR_TRIG
#define TMPC_EST_INCR_TRIG 1
#endif
// Footprint-term skip (as the SRB kernel's, rollout_f32.cu): a warp whose
// live lanes are all provably clear of the obstacle term for the next substep
// skips its four SDF gathers and soft cost.  1: the TEX (throughput-path)
// Euler launches with the footprint term (c4 -3.4%; measured +6% in the
// latency-bound c2 launch, and the kernel without the term keeps its own
// instantiation: c3 +7.7% with the skip machinery compiled in), 0: off.
#ifndef TMPC_EST_SD_SKIP
#define TMPC_EST_SD_SKIP 1
#endif

namespace tmpcb {

namespace {

constexpr unsigned kFull = 0xffffffffu;

// Terrain of one derivative evaluation: the dH/dx, dH/dy coefficient quads of
// the CoM cell and the fractions of the CoM in it.
struct CoM {
  float4 qx, qy;
  float fx, fy;
  float cl;  // footprint clearance of the cell (spare texel; SKIP launches)
};

__device__ __forceinline__ void gather_com(CoM& c, const Anchor& A, int pitch, float gxf,
                                           float gyf) {
  const int o = cell(gyf, A.loy, A.hiy, c.fy) * pitch + cell(gxf, A.lox, A.hix, c.fx);
  const float4* r = A.hq + 4 * o;
  c.qx = __ldg(r + 1);
  c.qy = __ldg(r + 2);
}

// A CoM record gathered ahead of its substep: its address and this lane's
// shared-memory slots.  The prefetch is a cp.async (LDGSTS) group, not an
// LDG: ptxas puts every LDG of the loop on one scoreboard, so a consumer of a
// prefetched register would also wait for the footprint gathers issued just
// before it; cp.async.wait_group 1 waits for exactly the older group.
struct CoMBuf {
  float4* sx;
  float4* sy;
  float* sc;  // the record's spare texel's first word (footprint clearance), SKIP launches
  const float4* p;
};

__device__ __forceinline__ void cp_async16(float4* dst, const float4* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(float* dst, const float4* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}

template <bool CL = false>
__device__ __forceinline__ void issue_com(CoMBuf& b, const float4* r, bool cl_on = false) {
  b.p = r;
  cp_async16(b.sx, r + 1);
  cp_async16(b.sy, r + 2);
  if (CL && cl_on) cp_async4(b.sc, r + 3);
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// Misprediction fix-up (rare: ~0.5% of warp-substeps on c2): lanes whose
// extrapolated cell missed re-gather into their slots with cp.async and the
// warp drains every group.  A real call, so ptxas cannot if-convert the
// drain (a wait_group 0 on every substep would also wait for the next
// substep's prefetch) and no LDG shares the footprint gathers' scoreboard.
__device__ __noinline__ void regather_com(unsigned dx, unsigned dy, const float4* r, int miss) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.s32 p, %4, 0;\n"
      " @p cp.async.ca.shared.global [%0], [%2], 16;\n"
      " @p cp.async.ca.shared.global [%1], [%3], 16;\n"
      " cp.async.commit_group;\n"
      " cp.async.wait_group 0;\n}" ::"r"(dx), "r"(dy), "l"(r + 1), "l"(r + 2), "r"(miss)
      : "memory");
}
// the same with the clearance texel (SKIP launches)
__device__ __noinline__ void regather_com_cl(unsigned dx, unsigned dy, unsigned dc,
                                             const float4* r, int miss) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.s32 p, %6, 0;\n"
      " @p cp.async.ca.shared.global [%0], [%3], 16;\n"
      " @p cp.async.ca.shared.global [%1], [%4], 16;\n"
      " @p cp.async.ca.shared.global [%2], [%5], 4;\n"
      " cp.async.commit_group;\n"
      " cp.async.wait_group 0;\n}" ::"r"(dx), "r"(dy), "r"(dc), "l"(r + 1), "l"(r + 2),
      "l"(r + 3), "r"(miss)
      : "memory");
}

// The record of the current substep: the older prefetch group (+ fix-up).
template <bool CL = false>
__device__ __forceinline__ void take_com(CoM& c, const CoMBuf& b, const float4* r, bool miss,
                                         bool any_miss) {
  asm volatile("cp.async.wait_group 1;" ::: "memory");
  if (any_miss) {
    if constexpr (CL)
      regather_com_cl(static_cast<unsigned>(__cvta_generic_to_shared(b.sx)),
                      static_cast<unsigned>(__cvta_generic_to_shared(b.sy)),
                      static_cast<unsigned>(__cvta_generic_to_shared(b.sc)), r, miss);
    else
      regather_com(static_cast<unsigned>(__cvta_generic_to_shared(b.sx)),
                   static_cast<unsigned>(__cvta_generic_to_shared(b.sy)), r, miss);
  }
  c.qx = *b.sx;
  c.qy = *b.sy;
  if constexpr (CL) c.cl = *b.sc;
}

// est_plane_attitude + rot_123 + est_derivative (dynamics.hpp:213-275): the
// planar velocity (world), the two velocity rates, g_by and a_by.
struct EstRates {
  float dx, dy, dvby, dwz, g_by, a_by;
};

__device__ __forceinline__ EstRates est_rates(const KConsts<float>& K, const CoM& c, float sps,
                                              float cps, float vbx, float vby, float wz, float de,
                                              float cde, float u_vr) {
  // normal_at (terrain.hpp:97-100): tau = (-f_x, -f_y, 1) / n, n = |(f_x, f_y, 1)|;
  // theta = asin(tau_x), phi = asin(-tau_y / cos theta) (the clamps are
  // no-ops: |tau_x| < 1, and cos theta = sqrt(1 + f_y^2) / n >= 1 / n).  In
  // closed form, with m = 1 / sqrt(1 + f_y^2):
  //   sin theta = -f_x / n, cos theta = (1 + f_y^2) m / n, sin phi = f_y m,
  //   cos phi = m
  // -- two independent rsqrt instead of three rsqrt and a reciprocal in a
  // chain (the EST substep's critical path), no 1 - a^2 cancellation
  const float sx = lerp_quad(c.qx, c.fx, c.fy);
  const float sy = lerp_quad(c.qy, c.fx, c.fy);
  const float q = fmaf(sy, sy, 1.f);
  const float rn = fm::rsqrt(fmaf(sx, sx, q));
  const float m = fm::rsqrt(q);
  const float st = -sx * rn;
  const float ct = (q * m) * rn;
  const float sf = sy * m;
  const float cf = m;
  // rot_123(phi, theta, psi) rows used: r0 (planar x), r1 (planar y), r2 (g_b)
  const float r00 = ct * cps, r01 = -ct * sps;
  const float sfst = sf * st, cfst = cf * st;
  const float r10 = fmaf(cps, sfst, cf * sps), r11 = fmaf(-sfst, sps, cf * cps);
  const float r21 = fmaf(cfst, sps, cps * sf), r22 = cf * ct;
  EstRates o;
  o.dx = fmaf(r00, vbx, r01 * vby);
  o.dy = fmaf(r10, vbx, r11 * vby);
  o.g_by = -K.g * r21;
  const float g_bz = -K.g * r22;
  // virtual tires (dynamics.hpp:241-251, 74-77)
  // front / rear virtual tires as one fp32x2 pair (fastmath.cuh)
  using fm::f2;
  const float vxe = fmaxf(vbx, K.vbx_floor);
  const f2 AL = fm::fsub2(fm::atan_ratio2(fmaf(wz, K.L_f, vby), vxe, fmaf(-wz, K.L_r, vby), vxe),
                          fm::pk(de, 0.f));
  const f2 CA = fm::fmul2(AL, fm::pk(K.C, K.C));
  float q_f, q_r;
  fm::upk(fm::ffma2(CA, CA, fm::pk(K.mu2, K.mu2)), q_f, q_r);
  const f2 T = fm::fmul2(fm::fmul2(CA, fm::pk(-K.mu, -K.mu)), fm::pk(fm::rsqrt(q_f), fm::rsqrt(q_r)));
  const float a_bx = fmaf(-wz, vby, u_vr);
  const float f_zf = fmaxf(fmaf(-K.kzzf, g_bz, -K.kzx * a_bx), 0.f);
  const float f_zr = fmaxf(fmaf(-K.kzzr, g_bz, K.kzx * a_bx), 0.f);
  float f_yf, f_yr;
  fm::upk(fm::fmul2(fm::pk(f_zf, f_zr), T), f_yf, f_yr);
  o.a_by = (f_yf + f_yr) * K.inv_M + o.g_by;  // EstDiagnostics::a_by (265)
  o.dvby = fmaf(-wz, vbx, o.a_by);
  o.dwz = fmaf(f_yf * K.L_f, cde, -f_yr * K.L_r) * K.inv_Jzz;
  return o;
}

// Planar footprint SDF quads (wheel_footprint, constraints.hpp:104-113) at
// (x, y, psi): fractions in sfx / sfy, quads in sq.  The CoM is clamped once
// and the points looked up unclamped (cell2u, rollout_anchor.cuh).
template <bool TEX>
__device__ __forceinline__ void gather_sd(float4 sq[4], float sfx[4], float sfy[4],
                                          const KConsts<float>& K, const KParams& P,
                                          const Anchor& A, float gxf, float gyf, float sps,
                                          float cps) {
  const fm::f2 g = fm::pk(fminf(fmaxf(gxf, A.clox), A.chix), fminf(fmaxf(gyf, A.cloy), A.chiy));
  const fm::f2 ir = fm::pk(K.inv_res, K.inv_res);
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    const float ox = fmaf(cps, K.rho[w][0], -sps * K.rho[w][1]);
    const float oy = fmaf(sps, K.rho[w][0], cps * K.rho[w][1]);
    const unsigned o = cell2u(fm::ffma2(fm::pk(ox, oy), ir, g), P.pitch, A.bias, P.last_cell,
                              sfx[w], sfy[w]);
    if constexpr (TEX)
      sq[w] = tex1Dfetch<float4>(A.tex, o);
    else
      sq[w] = __ldg(A.sdq0 + o);
  }
}

}  // namespace

// TEX (throughput-path) launches: a residency target of 14 one-warp CTAs per
// SM (ptxas then allocates <= 128 registers, 16 warps per SM instead of 14 at
// 144): c3 -14%, c4 -1.8%, RK4 c3 -13%, bit-identical.  SKIP: the footprint-
// term skip (TEX Euler launches with the term).
template <bool RK4, bool TEX, bool SKIP>
__global__ void __launch_bounds__(kBlock, TEX ? 14 : 1) rollout_kernel_est_f32(const KParams P,
                                                                   const TerrainDev td,
                                                                   const double* __restrict__ warm,
                                                                   double* __restrict__ out_cost,
                                                                   uint8_t* __restrict__ out_flags,
                                                                   float* __restrict__ out_margin,
                                                                   DevStats* __restrict__ st) {
  l2_prefetch_terrain(P, td);  // the reachable terrain into L2 (rollout_dev.cuh)
  const KConsts<float>& K = P.cf;
  const int64_t slot = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool active = slot < P.k_count;
  const int64_t kl = active && P.order ? static_cast<int64_t>(__ldg(P.order + slot)) : slot;
  const int64_t kg = P.k_begin + kl;
  // the footprint-term skip: the clearance of the CoM cell comes with the
  // CoM record
  static_assert(!SKIP || (TEX && !RK4), "the skip serves the TEX Euler launches");

  double J = 0.0;
  float margin = __int_as_float(0x7f800000);  // +inf
  bool feasible = true, diverged = false, goal = false;
  unsigned substeps = 0;

  // planar position: cell anchor + compensated offset (rollout_anchor.cuh)
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
  // EstState (dynamics.hpp:148-155) from the SrbState slots of s0
  fm::KS psi = fm::ks_make(P.s0[3]), vby = fm::ks_make(P.s0[7]), wz = fm::ks_make(P.s0[11]);
  fm::KS de = fm::ks_make(P.s0[12]), vbx = fm::ks_make(P.s0[6]);
  const fm::KS de_max = fm::ks_make(P.cd.delta_max), de_min = fm::ks_make(-P.cd.delta_max);

  const uint64_t base = mix64(substream(P.seed, static_cast<uint64_t>(kg)));
  double prev[2] = {0.0, 0.0};
  const bool use_sd = P.enable_dist && P.has_sdist;
  const bool use_lat = P.enable_rollover;
  const float dt = K.dt;
  const float dtx = static_cast<float>(P.dt * P.gx_scale);  // m/s -> cells per substep
  const float dty = static_cast<float>(P.dt * P.gy_scale);
  const int S = P.S, total = P.n_steps * P.S;
  const int pitch = P.pitch;

  Anchor A = make_anchor(P, td, ax, ay);
  // Footprint SDF quads of the current substep (issued one substep ahead).
  float4 sq[4];
  float sfx[4], sfy[4];
  float sps, cps;
  fm::sincos(psi.s, &sps, &cps);
  if (use_sd) gather_sd<TEX>(sq, sfx, sfy, K, P, A, gx.s, gy.s, sps, cps);
  // CoM records, two substeps ahead: the record of substep n+2 is gathered
  // at the end of substep n at the position extrapolated from x(n+1) with
  // the velocity 2 v(n) - v(n-1) (error O(dt^3 jerk), far below a cell), so
  // the gather -> attitude -> position chain no longer waits on a gather; a
  // lane whose extrapolated cell misses re-gathers (warp-uniform test).
  // Substep parity selects the buffer, hence the 2x-unrolled loop below.
  __shared__ float4 s_com[2][2][kBlock];  // [buffer][qx, qy][lane]
  __shared__ float s_cl[2][SKIP ? kBlock : 1];  // [buffer][lane]: the clearance (SKIP)
  const int lane = threadIdx.x;
  CoMBuf b0{&s_com[0][0][lane], &s_com[0][1][lane], &s_cl[0][SKIP ? lane : 0], nullptr};
  CoMBuf b1{&s_com[1][0][lane], &s_com[1][1][lane], &s_cl[1][SKIP ? lane : 0], nullptr};
  bool sd_on = true;  // the footprint quads of the current substep were gathered (warp-uniform)
  float vxp, vyp;  // planar velocity (cells / substep) of the previous substep
  {
    const float vx0 = static_cast<float>(P.s0[6]), vy0 = static_cast<float>(P.s0[7]);
    vxp = fmaf(cps, vx0, -sps * vy0) * dtx;  // level-plane guess for substep 0
    vyp = fmaf(sps, vx0, cps * vy0) * dty;
    float f;
    issue_com<SKIP>(b0, A.hq + 4 * (cell(gy.s, A.loy, A.hiy, f) * pitch +
                                    cell(gx.s, A.lox, A.hix, f)), use_sd);
    const float px = gx.s + vxp, py = gy.s + vyp;
    issue_com<SKIP>(b1, A.hq + 4 * (cell(py, A.loy, A.hiy, f) * pitch + cell(px, A.lox, A.hix, f)),
                    use_sd);
  }

  bool live = active;
  float u_dr = 0.f, u_vr = 0.f;
  double L0 = 0.0;
  float rate_sum = 0.f;
  int nq = 0, q = 0, it = 0;
  const auto step = [&](CoMBuf& cur) -> bool {
    if (q == 0) {  // ---- ZOH step boundary (warp-uniform)
      if (it > 0) {
        J += P.dt * (static_cast<double>(nq) * L0 + static_cast<double>(rate_sum));
        rate_sum = 0.f;
        nq = 0;
        const float fsum = gx.s + gy.s + psi.s + vby.s + wz.s + de.s + vbx.s;
        const bool bad = !isfinite(fsum);  // dynamics.hpp:491-492
        diverged = diverged || (live && bad);
        live = live && !bad;
        if (!__any_sync(kFull, live)) return false;
      }
      float fr;
      const int ix = fm::floor_frac(gx.s, fr), iy = fm::floor_frac(gy.s, fr);
      if (live) {
        constexpr float kBig = 2097152.f;  // 2^21
        constexpr int kLim = 1 << 20;
        if (fabsf(gx.s) < kBig && abs(ax + ix) < kLim) {
          ax += ix;
          gx.s -= static_cast<float>(ix);
        }
        if (fabsf(gy.s) < kBig && abs(ay + iy) < kLim) {
          ay += iy;
          gy.s -= static_cast<float>(iy);
        }
        bx = static_cast<float>(ax - gax) - gfx;
        by = static_cast<float>(ay - gay) - gfy;
        A = make_anchor(P, td, ax, ay);
      }
      if (TMPC_EST_INCR_TRIG && !RK4) fm::sincos(psi.s, &sps, &cps);
      double u[2];
      sample_step(P.smp, base, kg == 0, it / S, warm, prev, u);
      u_dr = static_cast<float>(u[0]);
      u_vr = static_cast<float>(u[1]);
      L0 = P.w_t + P.w_c * u[0] * u[0];
    }
    q = q + 1 == S ? 0 : q + 1;
    ++it;

    // goal truncation before accumulating
    const float gdx = (bx + gx.s) - gx.c, gdy = (by + gy.s) - gy.c;
    const bool at_goal = live && gdx * gdx + gdy * gdy <= rg2;
    goal = goal || at_goal;
    live = live && !at_goal;

    // the CoM record of this substep: the extrapolated gather, or a re-gather
    CoM c;
    const float4* rec = A.hq + 4 * (cell(gy.s, A.loy, A.hiy, c.fy) * pitch +
                                    cell(gx.s, A.lox, A.hix, c.fx));
    const bool miss = rec != cur.p;
    take_com<SKIP>(c, cur, rec, miss, __any_sync(kFull, miss));
    // the CoM of this substep lies inside the reference's clamp window, so
    // its record's cell is also the footprint lookups' clamped CoM cell
    const bool in_window = gx.s >= A.lox && gx.s <= A.hix && gy.s >= A.loy && gy.s <= A.hiy;

    // derivative at the state (k1)
    const float cde = fm::cos_small(de.s);
    const EstRates k1 = est_rates(K, c, sps, cps, vbx.s, vby.s, wz.s, de.s, cde, u_vr);

    // increments over the substep (world velocities in cells)
    float ix_, iy_, ipsi, ivby, iwz;
    const float h = live ? dt : 0.f;
    if constexpr (!RK4) {
      ix_ = k1.dx;
      iy_ = k1.dy;
      ipsi = wz.s;
      ivby = k1.dvby;
      iwz = k1.dwz;
    } else {
      // Scheme::kRk4 (dynamics.hpp:454-465): stages at s + f k, f = dt/2,
      // dt/2, dt; each stage gathers the CoM record of its own position
      float sx, sy, spsi, svby, swz;  // sums k1 + 2 k2 + 2 k3 + k4
      float kx = k1.dx, ky = k1.dy, kpsi = wz.s, kvby = k1.dvby, kwz = k1.dwz;
      sx = kx; sy = ky; spsi = kpsi; svby = kvby; swz = kwz;
#pragma unroll
      for (int stg = 1; stg < 4; ++stg) {
        const float fr = stg == 3 ? 1.f : 0.5f;  // stage fraction of the substep
        const float f = fr * dt;
        const float wgt = stg == 3 ? 1.f : 2.f;
        const float px = fmaf(fr * dtx, kx, gx.s), py = fmaf(fr * dty, ky, gy.s);
        const float ppsi = fmaf(f, kpsi, psi.s);
        const float pvbx = fmaf(f, u_vr, vbx.s), pvby = fmaf(f, kvby, vby.s);
        const float pwz = fmaf(f, kwz, wz.s), pde = fmaf(f, u_dr, de.s);
        float s2, c2;
        fm::sincos(ppsi, &s2, &c2);
        CoM cs;
        gather_com(cs, A, pitch, px, py);
        const EstRates kr = est_rates(K, cs, s2, c2, pvbx, pvby, pwz, pde, fm::cos_small(pde), u_vr);
        kx = kr.dx; ky = kr.dy; kpsi = pwz; kvby = kr.dvby; kwz = kr.dwz;
        sx = fmaf(wgt, kx, sx); sy = fmaf(wgt, ky, sy); spsi = fmaf(wgt, kpsi, spsi);
        svby = fmaf(wgt, kvby, svby); swz = fmaf(wgt, kwz, swz);
      }
      constexpr float kSixth = 1.f / 6.f;
      ix_ = sx * kSixth; iy_ = sy * kSixth; ipsi = spsi * kSixth;
      ivby = svby * kSixth; iwz = swz * kSixth;
    }
    // forward Euler / RK4 update + clamp_steering (dynamics.hpp:423-441,453-466)
    const float hx = live ? dtx : 0.f, hy = live ? dty : 0.f;
    fm::ks_axpy(gx, hx, ix_);
    fm::ks_axpy(gy, hy, iy_);
    fm::ks_axpy(psi, h, ipsi);
    fm::ks_axpy(vby, h, ivby);
    fm::ks_axpy(wz, h, iwz);
    fm::ks_axpy(de, h, u_dr);
    fm::ks_axpy(vbx, h, u_vr);
    fm::ks_clamp(de, de_min, de_max);
    substeps += live;

    // the CoM record of substep n+2 (extrapolated; this buffer is free now)
    {
      const float vxn = hx * ix_, vyn = hy * iy_;
      const float px = gx.s + fmaf(2.f, vxn, -vxp), py = gy.s + fmaf(2.f, vyn, -vyp);
      vxp = vxn;
      vyp = vyn;
      float f;
      issue_com<SKIP>(cur, A.hq + 4 * (cell(py, A.loy, A.hiy, f) * pitch +
                                       cell(px, A.lox, A.hix, f)), use_sd);
    }

    // L_soft of this substep: footprint SDF (gathered one substep ago) +
    // lateral acceleration (constraints.hpp:62-65, 87-100)
    float rate = 0.f;
    if (use_sd && sd_on) {
      float srate = 0.f, sd_min = __int_as_float(0x7f800000);
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const float sd = lerp_quad(sq[w], sfx[w], sfy[w]);
        const float a = fmaxf(0.f, 1.f - sd * K.inv_eps_dist);
        srate = fmaf(K.sigma * a, a, srate);
        sd_min = fminf(sd_min, sd);
      }
      rate = h != 0.f ? srate : 0.f;
      feasible = feasible && (h == 0.f || sd_min > 0.f);
      margin = h != 0.f ? fminf(margin, sd_min * K.inv_eps_dist) : margin;
    }
    if (use_lat) {
      const float pi_aby = fabsf(k1.a_by - k1.g_by) - K.a_by_bar;
      const float a = fmaxf(0.f, fmaf(pi_aby, K.inv_eps_aby, 1.f));
      rate = h != 0.f ? fmaf(K.sigma * a, a, rate) : rate;
      feasible = feasible && (h == 0.f || pi_aby < 0.f);
      margin = h != 0.f ? fminf(margin, -pi_aby * K.inv_a_by_bar) : margin;
    }
    rate_sum += rate;
    nq += h != 0.f;

    // footprint of substep n+1: sin / cos psi rotated by this substep's
    // increment (re-synced exactly at every ZOH step, like the SRB kernel)
    if (TMPC_EST_INCR_TRIG && !RK4)
      fm::rotate_sc(sps, cps, h * ipsi);
    else
      fm::sincos(psi.s, &sps, &cps);
    if constexpr (SKIP) {
      // c.cl bounds the SDF of every footprint point of a CoM within
      // kClearWindowMove cells of this substep's CoM cell (ctx.cu
      // footprint_clearance); the next CoM is this one + the increment.  A
      // clear lane's term adds exactly 0 and cannot lower its margin (see
      // rollout_f32.cu); NaN tests false.
      const bool clear = c.cl * K.inv_eps_dist >= fmaxf(kClearCost, margin) && in_window &&
                         fabsf(hx * ix_) <= kClearMove && fabsf(hy * iy_) <= kClearMove;
      sd_on = __any_sync(kFull, live && !clear);
    }
    if (use_sd && sd_on) gather_sd<TEX>(sq, sfx, sfy, K, P, A, gx.s, gy.s, sps, cps);
    return true;
  };
  while (it < total) {
    if (!step(b0) || it >= total || !step(b1)) break;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  J += P.dt * (static_cast<double>(nq) * L0 + static_cast<double>(rate_sum));
  {
    const float fsum = gx.s + gy.s + psi.s + vby.s + wz.s + de.s + vbx.s;
    diverged = diverged || (live && !isfinite(fsum));
  }
  if (active) {
    if (diverged) {
      J = __longlong_as_double(0x7ff0000000000000LL);
      feasible = false;
      margin = __int_as_float(0xff800000);
    } else {
      const double x = ((ax - P.gx_off) + (static_cast<double>(gx.s) - gx.c)) / P.gx_scale;
      const double y = ((ay - P.gy_off) + (static_cast<double>(gy.s) - gy.c)) / P.gy_scale;
      const double gdx = x - P.goal_x, gdy = y - P.goal_y;
      J += P.w_g * sqrt(gdx * gdx + gdy * gdy);
    }
  }
  reduce_and_finalize(P, active, kl, kg, J, feasible, diverged, goal, margin,
                      active ? substeps : 0u, out_cost, out_flags, out_margin, st);
}

void launch_rollout_est_f32(const KParams& P, const TerrainDev& td, const double* warm,
                            double* cost, uint8_t* flags, float* margin, DevStats* st,
                            cudaStream_t stream) {
  const unsigned blocks = static_cast<unsigned>((P.k_count + kBlock - 1) / kBlock);
  const bool tex = P.k_count >= 32768;  // this launch's K: the gather path, not the arithmetic
  const bool skip = TMPC_EST_SD_SKIP && tex && P.enable_dist && P.has_sdist;
#define TMPC_LAUNCH(R, T, K) \
  launch(rollout_kernel_est_f32<R, T, K>, blocks, kBlock, stream, P, td, warm, cost, flags, margin, st)
  if (P.scheme == TMPC_SCHEME_RK4) {
    if (tex) TMPC_LAUNCH(true, true, false); else TMPC_LAUNCH(true, false, false);
  } else if (skip) {
    TMPC_LAUNCH(false, true, true);
  } else {
    if (tex) TMPC_LAUNCH(false, true, false); else TMPC_LAUNCH(false, false, false);
  }
#undef TMPC_LAUNCH
}

// Shared memory holds only the CoM prefetch slots, 2 KB per CTA (+256 B of
// clearance words in the skip launches): a 16% carveout (~36 KB) fits every
// CTA the registers allow on an SM (a 0%
// carveout would cap residency at 2-4 CTAs and split c2 into two waves);
// the rest stays L1.
cudaError_t configure_rollout_est_f32() {
  cudaError_t e = cudaSuccess;
  const auto carve = [&](const void* f, int pct) {  // 2 KB (+256 B) per CTA
    const cudaError_t r = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    if (r != cudaSuccess) e = r;
  };
  carve(reinterpret_cast<const void*>(rollout_kernel_est_f32<false, false, false>), 16);
  carve(reinterpret_cast<const void*>(rollout_kernel_est_f32<true, false, false>), 16);
  carve(reinterpret_cast<const void*>(rollout_kernel_est_f32<false, true, false>), 16);
  carve(reinterpret_cast<const void*>(rollout_kernel_est_f32<true, true, false>), 16);
  carve(reinterpret_cast<const void*>(rollout_kernel_est_f32<false, true, true>), 16);
  return e;
}

}  // namespace tmpcb
