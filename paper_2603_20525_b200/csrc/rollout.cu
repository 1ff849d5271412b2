// Fused rollout + cost + feasibility + arg-min kernel.
//
// One thread owns one candidate k for the whole horizon: the 13-entry SRB
// state lives in registers (stored in fp64 so 1000 Euler increments do not
// round away; the derivative is evaluated in the math type T), controls are
// drawn in-kernel from the counter RNG, and the terrain store is a padded
// {H, dH/dx, dH/dy} node field plus a signed-distance field read through the
// read-only path (L1/L2 resident).  Nothing per substep touches HBM; per
// candidate the kernel writes 13 bytes.
//
// Algorithm per candidate (identical to oracle/tmpc_oracle.cpp rollout and
// SURVEY §8a):
//   for t < N: u_t = sample(seed, k, t)
//     for q < S: if |p - p_g| <= r_g: stop (goal)
//                J += dt * (w_t + w_c u^2 + L_soft(s))   SPEC.md:372, constraints.hpp:87-100
//                feasibility / margin from s             DESIGN.md §3 (D9)
//                s = s + dt * srb_derivative(s, u)       dynamics.hpp:308-398,446-468
//                diverged if gimbal guard / non-finite   dynamics.hpp:311, 491
//   J += w_g |p - p_g|
// then a warp-shuffle / atomicMin arg-min over the packed key
// (infeasible, f32(J), k) and a last-block finalisation of the local winner.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "fastmath.cuh"
#include "rollout.cuh"
#include "tmpc_common.h"

namespace tmpcb {

namespace {

// ---- math dispatch -------------------------------------------------------
__device__ __forceinline__ void dsincos(float a, float* s, float* c) { sincosf(a, s, c); }
__device__ __forceinline__ void dsincos(double a, double* s, double* c) { sincos(a, s, c); }
__device__ __forceinline__ float datan(float a) { return atanf(a); }
__device__ __forceinline__ double datan(double a) { return atan(a); }
__device__ __forceinline__ float dcos(float a) { return cosf(a); }
__device__ __forceinline__ double dcos(double a) { return cos(a); }

// ---- terrain store access --------------------------------------------------
// Split a padded grid coordinate g' (fp64) into integer + fraction so
// per-wheel offsets (a few cells) are added in T without losing the absolute
// position.
template <typename T>
__device__ __forceinline__ void split_coord(double g, int& gi, T& gf) {
  const double fl = floor(g);
  gi = static_cast<int>(fl);
  gf = static_cast<T>(g - fl);
}

// Clamped cell index and fraction along one axis for g' = gi + gf + off,
// clamped to [1, n+2] (== the reference's clamp to [0, n-1] on the
// 2-cell replicate-padded grid, terrain.hpp:37-44).
template <typename T>
__device__ __forceinline__ void axis_cell(int gi, T gf, T off, int n_hi, int& i0, T& f) {
  const T t = gf + off;
  const T ft = floor(t);
  int i = gi + static_cast<int>(ft);
  T fr = t - ft;
  if (i < 1) {
    i = 1;
    fr = T(0);
  } else if (i >= n_hi) {
    i = n_hi;
    fr = T(0);
  }
  i0 = i;
  f = fr;
}

// detail::bilinear (terrain.hpp:45-49) on the padded node fields: one texel
// gather per corner gives height and both gradient components
// (gradient_at == bilinear of the node central differences).
__device__ __forceinline__ void lookup_hg(const TerrainDev& td, int pitch, int i0, int j0,
                                          float fx, float fy, float& h, float& gxs, float& gys) {
  const float4* r0 = td.hg32 + static_cast<size_t>(j0) * pitch + i0;
  const float4 a0 = __ldg(r0), a1 = __ldg(r0 + 1), b0 = __ldg(r0 + pitch), b1 = __ldg(r0 + pitch + 1);
  const float ha = a0.x + fx * (a1.x - a0.x), hb = b0.x + fx * (b1.x - b0.x);
  const float xa = a0.y + fx * (a1.y - a0.y), xb = b0.y + fx * (b1.y - b0.y);
  const float ya = a0.z + fx * (a1.z - a0.z), yb = b0.z + fx * (b1.z - b0.z);
  h = ha + fy * (hb - ha);
  gxs = xa + fy * (xb - xa);
  gys = ya + fy * (yb - ya);
}
__device__ __forceinline__ void lookup_hg(const TerrainDev& td, int pitch, int i0, int j0,
                                          double fx, double fy, double& h, double& gxs,
                                          double& gys) {
  const HG64* r0 = td.hg64 + static_cast<size_t>(j0) * pitch + i0;
  const double2 a0 = __ldg(&r0->a), a0b = __ldg(&r0->b);
  const double2 a1 = __ldg(&(r0 + 1)->a), a1b = __ldg(&(r0 + 1)->b);
  const double2 b0 = __ldg(&(r0 + pitch)->a), b0b = __ldg(&(r0 + pitch)->b);
  const double2 b1 = __ldg(&(r0 + pitch + 1)->a), b1b = __ldg(&(r0 + pitch + 1)->b);
  const double ha = a0.x + fx * (a1.x - a0.x), hb = b0.x + fx * (b1.x - b0.x);
  const double xa = a0.y + fx * (a1.y - a0.y), xb = b0.y + fx * (b1.y - b0.y);
  const double ya = a0b.x + fx * (a1b.x - a0b.x), yb = b0b.x + fx * (b1b.x - b0b.x);
  h = ha + fy * (hb - ha);
  gxs = xa + fy * (xb - xa);
  gys = ya + fy * (yb - ya);
}

template <typename T>
__device__ __forceinline__ T lookup_sd(const T* __restrict__ sd, int pitch, int i0, int j0, T fx,
                                       T fy) {
  const T* r0 = sd + static_cast<size_t>(j0) * pitch + i0;
  const T a0 = __ldg(r0), a1 = __ldg(r0 + 1), b0 = __ldg(r0 + pitch), b1 = __ldg(r0 + pitch + 1);
  const T a = a0 + fx * (a1 - a0), b = b0 + fx * (b1 - b0);
  return a + fy * (b - a);
}
__device__ __forceinline__ const float* sd_ptr(const TerrainDev& td, float) { return td.sd32; }
__device__ __forceinline__ const double* sd_ptr(const TerrainDev& td, double) { return td.sd64; }

template <typename V>
__device__ __forceinline__ V warp_min(V v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const V w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr int kBlock = 32;  // one warp per CTA: spreads small K over all 148 SMs

}  // namespace

template <typename T>
__global__ void __launch_bounds__(kBlock) rollout_kernel(const KParams P, const TerrainDev td,
                                                         const double* __restrict__ warm,
                                                         double* __restrict__ out_cost,
                                                         uint8_t* __restrict__ out_flags,
                                                         float* __restrict__ out_margin,
                                                         DevStats* __restrict__ st) {
  const KConsts<T>& K = consts<T>(P);
  const int64_t kl = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool active = kl < P.k_count;
  const int64_t kg = P.k_begin + kl;

  double J = 0.0;
  float margin = __int_as_float(0x7f800000);  // +inf
  bool feasible = true, diverged = false, goal = false;
  unsigned substeps = 0;

  // state (SrbState order, dynamics.hpp:167-172), fp64 storage
  double x = P.s0[0], y = P.s0[1], z = P.s0[2];
  double psi = P.s0[3], th = P.s0[4], ph = P.s0[5];
  double vx = P.s0[6], vy = P.s0[7], vz = P.s0[8];
  double wx = P.s0[9], wy = P.s0[10], wz = P.s0[11];
  double de = P.s0[12];

  if (active) {
    const uint64_t base = mix64(substream(P.seed, static_cast<uint64_t>(kg)));
    double prev[2] = {0.0, 0.0};
    const int n_hi_x = P.nx + 2, n_hi_y = P.ny + 2;
    const T* __restrict__ sdf = sd_ptr(td, T(0));
    for (int t = 0; t < P.n_steps; ++t) {
      double u[2];
      sample_step(P.smp, base, kg == 0, t, warm, prev, u);
      const T u_dr = static_cast<T>(u[0]);
      const T u_vr = static_cast<T>(u[1]);
      const double L0 = P.w_t + P.w_c * u[0] * u[0];
      for (int q = 0; q < P.S; ++q) {
        // goal truncation before accumulating
        const double gdx = x - P.goal_x, gdy = y - P.goal_y;
        if (gdx * gdx + gdy * gdy <= P.goal_r2) {
          goal = true;
          break;
        }
        // state in the math type
        const T tpsi = static_cast<T>(psi), tth = static_cast<T>(th), tph = static_cast<T>(ph);
        const T tvx = static_cast<T>(vx), tvy = static_cast<T>(vy), tvz = static_cast<T>(vz);
        const T twx = static_cast<T>(wx), twy = static_cast<T>(wy), twz = static_cast<T>(wz);
        const T tde = static_cast<T>(de);
        T sps, cps, sth, cth, sph, cph;
        dsincos(tpsi, &sps, &cps);
        dsincos(tth, &sth, &cth);
        dsincos(tph, &sph, &cph);

        // centre grid coordinates (fp64 -> int + fraction)
        int gxi, gyi;
        T gxf, gyf;
        split_coord(x * P.gx_scale + P.gx_off, gxi, gxf);
        split_coord(y * P.gy_scale + P.gy_off, gyi, gyf);

        // ---- L_soft(s): wheel SDF soft costs + ESM rollover (constraints.hpp:87-113)
        T rate = T(0);
        if (P.enable_dist && P.has_sdist) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            // wheel_footprint (constraints.hpp:104-113): planar, ignores roll/pitch
            const T ox = cps * K.rho[i][0] - sps * K.rho[i][1];
            const T oy = sps * K.rho[i][0] + cps * K.rho[i][1];
            int i0, j0;
            T fx, fy;
            axis_cell(gxi, gxf, ox * K.inv_res, n_hi_x, i0, fx);
            axis_cell(gyi, gyf, oy * K.inv_res, n_hi_y, j0, fy);
            const T sd = lookup_sd(sdf, P.pitch, i0, j0, fx, fy);
            const T a = fmax(T(0), T(1) - sd * K.inv_eps_dist);  // soft_cost_rate(-sd)
            rate += K.sigma * a * a;
            feasible = feasible && (sd > T(0));
            margin = fminf(margin, static_cast<float>(sd * K.inv_eps_dist));
          }
        }
        if (P.enable_rollover) {
          // esm (constraints.hpp:16-23): sin(|phi| + phi_bar) via the angle sum,
          // with sin|phi| = sign(phi) sin(phi) (exact for any phi, incl. |phi| > pi)
          const T sin_abs = tph < T(0) ? -sph : sph;
          const T sin_lever = sin_abs * K.esm_c_pb + cph * K.esm_s_pb;
          const T sgn = fabs(tph) <= K.esm_phi_lim ? T(1) : T(-1);
          const T U = sgn * K.esm_Mg * (K.esm_r_bar * (T(1) - sin_lever) * cth);
          const T a = fmax(T(0), T(1) - U * K.inv_eps_esm);
          rate += K.sigma * a * a;
          feasible = feasible && (U > T(0));
          margin = fminf(margin, static_cast<float>(U * K.inv_esm_nominal));
        }
        J += P.dt * (L0 + static_cast<double>(rate));

        // ---- srb_derivative (dynamics.hpp:308-398)
        if (fabs(th) >= P.gimbal_lim) {  // dynamics.hpp:311-312
          diverged = true;
          break;
        }
        // rot_321 (dynamics.hpp:96-105)
        const T r00 = cps * cth, r01 = cps * sph * sth - cph * sps, r02 = sph * sps + cph * cps * sth;
        const T r10 = cth * sps, r11 = cph * cps + sph * sps * sth, r12 = cph * sps * sth - cps * sph;
        const T r20 = -sth, r21 = cth * sph, r22 = cph * cth;
        const T gbx = r20 * (-K.g), gby = r21 * (-K.g), gbz = r22 * (-K.g);
        const T cd = dcos(tde);
        const T f_x_rear = K.half_M * (u_vr - gbx + twy * tvz - twz * tvy);
        T fy_sum = T(0), fz_sum = T(0), mx = T(0), my = T(0), mz = T(0);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const bool front = i < 2;
          const T rx = K.rho[i][0], ry = K.rho[i][1], rz = K.rho[i][2];
          const T rwx = r00 * rx + r01 * ry + r02 * rz;
          const T rwy = r10 * rx + r11 * ry + r12 * rz;
          const T rwz = r20 * rx + r21 * ry + r22 * rz;
          const T vix = tvx + (twy * rz - twz * ry);
          const T viy = tvy + (twz * rx - twx * rz);
          const T viz = tvz + (twx * ry - twy * rx);
          int i0, j0;
          T fx, fy;
          axis_cell(gxi, gxf, rwx * K.inv_res, n_hi_x, i0, fx);
          axis_cell(gyi, gyf, rwy * K.inv_res, n_hi_y, j0, fy);
          T h, sfx, sfy;
          lookup_hg(td, P.pitch, i0, j0, fx, fy, h, sfx, sfy);
          // tau_b = R^T (-fx, -fy, 1)
          const T tbx = r20 - r00 * sfx - r10 * sfy;
          const T tby = r21 - r01 * sfx - r11 * sfy;
          const T tbz = r22 - r02 * sfx - r12 * sfy;
          const T inv_tbz = T(1) / fmax(tbz, K.tau_floor);
          const T chi = static_cast<T>((z + static_cast<double>(rwz)) - static_cast<double>(h)) * inv_tbz;
          const T chi_dot = (tbx * (vix - chi * twy) + tby * (viy + chi * twx) + tbz * viz) * inv_tbz;
          const T f_k = fmax(K.fs_i[i] - K.k_i[i] * chi, T(0));
          const T f_b = f_k > T(0) ? fmax(-K.b_i[i] * chi_dot, -f_k) : T(0);
          const T f_z = f_k + f_b;
          const T alpha = datan(viy / fmax(vix, K.vbx_floor)) - (front ? tde : T(0));
          const T ca = K.C * alpha;
          const T f_y = f_z * (-ca * K.mu) / sqrt(K.mu2 + ca * ca);
          const T Fy = front ? f_y * cd : f_y;
          const T Fx = front ? T(0) : f_x_rear;
          fy_sum += Fy;
          fz_sum += f_z;
          mx += ry * f_z - rz * Fy;
          my += rz * Fx - rx * f_z;
          mz += rx * Fy - ry * Fx;
        }
        // euler_rates_321 (dynamics.hpp:109-118)
        const T inv_ct = T(1) / cth;
        const T tt = sth * inv_ct;
        const T d_psi = (sph * twy + cph * twz) * inv_ct;
        const T d_th = cph * twy - sph * twz;
        const T d_ph = twx + sph * tt * twy + cph * tt * twz;
        // v_w = R v_b and the 13-vector derivative (dynamics.hpp:374-389)
        const T dxw = r00 * tvx + r01 * tvy + r02 * tvz;
        const T dyw = r10 * tvx + r11 * tvy + r12 * tvz;
        const T dzw = r20 * tvx + r21 * tvy + r22 * tvz;
        const T d_vy = fy_sum * K.inv_M + gby + twx * tvz - twz * tvx;
        const T d_vz = fz_sum * K.inv_M + gbz - twx * tvy + twy * tvx;
        const T d_wx = (mx + K.cJx * twy * twz) * K.inv_Jxx;
        const T d_wy = (my - K.cJy * twx * twz) * K.inv_Jyy;
        const T d_wz = (mz + K.cJz * twx * twy) * K.inv_Jzz;
        // forward Euler + clamp_steering (dynamics.hpp:423-441,453,466), fp64 state
        x += P.dt * static_cast<double>(dxw);
        y += P.dt * static_cast<double>(dyw);
        z += P.dt * static_cast<double>(dzw);
        psi += P.dt * static_cast<double>(d_psi);
        th += P.dt * static_cast<double>(d_th);
        ph += P.dt * static_cast<double>(d_ph);
        vx += P.dt * static_cast<double>(u_vr);
        vy += P.dt * static_cast<double>(d_vy);
        vz += P.dt * static_cast<double>(d_vz);
        wx += P.dt * static_cast<double>(d_wx);
        wy += P.dt * static_cast<double>(d_wy);
        wz += P.dt * static_cast<double>(d_wz);
        de = fmin(fmax(de + P.dt * static_cast<double>(u_dr), -P.cd.delta_max), P.cd.delta_max);
        ++substeps;
        if (!isfinite(x + y + z + psi + th + ph + vx + vy + vz + wx + wy + wz + de)) {
          diverged = true;  // dynamics.hpp:491-492
          break;
        }
      }
      if (goal || diverged) break;
    }
  }

  // ---- terminal cost and per-candidate outputs
  float cost_f = 0.f;
  if (active) {
    if (diverged) {
      J = __longlong_as_double(0x7ff0000000000000LL);
      feasible = false;
      margin = __int_as_float(0xff800000);
    } else {
      const double gdx = x - P.goal_x, gdy = y - P.goal_y;
      J += P.w_g * sqrt(gdx * gdx + gdy * gdy);
    }
    out_cost[kl] = J;
    out_flags[kl] = static_cast<uint8_t>((feasible ? TMPC_FLAG_FEASIBLE : 0) |
                                         (diverged ? TMPC_FLAG_DIVERGED : 0) |
                                         (goal ? TMPC_FLAG_GOAL : 0));
    out_margin[kl] = margin;
    cost_f = static_cast<float>(J);
  }

  // ---- arg-min + stats: warp shuffle -> one atomic per warp
  const bool infeasible = P.selection == TMPC_SELECT_FEASIBLE_FIRST && !feasible;
  long long key = active ? pack_key(cost_f, infeasible, kg) : kKeyNone;
  key = warp_min(key);
  const bool fin = active && !diverged;
  const unsigned mfeas = __ballot_sync(0xffffffffu, active && feasible);
  const unsigned mdiv = __ballot_sync(0xffffffffu, active && diverged);
  const unsigned mgoal = __ballot_sync(0xffffffffu, active && goal);
  const unsigned mfin = __ballot_sync(0xffffffffu, fin);
  const double csum = warp_sum(fin ? J : 0.0);
  const long long cmin = warp_min(fin ? __double_as_longlong(J) : 0x7ff0000000000000LL);
  const unsigned ssum = __reduce_add_sync(0xffffffffu, substeps);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&st->key, key);
    atomicAdd(&st->n_feasible, static_cast<unsigned long long>(__popc(mfeas)));
    atomicAdd(&st->n_diverged, static_cast<unsigned long long>(__popc(mdiv)));
    atomicAdd(&st->n_goal, static_cast<unsigned long long>(__popc(mgoal)));
    atomicAdd(&st->n_finite, static_cast<unsigned long long>(__popc(mfin)));
    atomicAdd(&st->substeps, static_cast<unsigned long long>(ssum));
    if (mfin) {
      atomicAdd(&st->sum_cost, csum);
      atomicMin(&st->min_cost_bits, cmin);
    }
  }
  // ---- last block: gather the local winner's exact fp64 cost / flags / margin
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned long long ticket = atomicAdd(&st->done_blocks, 1ULL);
    if (ticket == gridDim.x - 1) {
      __threadfence();
      const long long kmin = *reinterpret_cast<volatile long long*>(&st->key);
      const int64_t w = key_index(kmin) - P.k_begin;
      if (kmin != kKeyNone && w >= 0 && w < P.k_count) {
        st->best_cost = *reinterpret_cast<volatile double*>(&out_cost[w]);
        st->best_flags = *reinterpret_cast<volatile uint8_t*>(&out_flags[w]);
        st->best_margin = *reinterpret_cast<volatile float*>(&out_margin[w]);
      }
    }
  }
}

// Warp-level arg-min + stats + last-block finalisation shared by the kernels.
__device__ __forceinline__ void reduce_and_finalize(const KParams& P, bool active, int64_t kl,
                                                    int64_t kg, double J, bool feasible,
                                                    bool diverged, bool goal, float margin,
                                                    unsigned substeps, double* out_cost,
                                                    uint8_t* out_flags, float* out_margin,
                                                    DevStats* st) {
  float cost_f = 0.f;
  if (active) {
    out_cost[kl] = J;
    out_flags[kl] = static_cast<uint8_t>((feasible ? TMPC_FLAG_FEASIBLE : 0) |
                                         (diverged ? TMPC_FLAG_DIVERGED : 0) |
                                         (goal ? TMPC_FLAG_GOAL : 0));
    out_margin[kl] = margin;
    cost_f = static_cast<float>(J);
  }
  const bool infeasible = P.selection == TMPC_SELECT_FEASIBLE_FIRST && !feasible;
  long long key = active ? pack_key(cost_f, infeasible, kg) : kKeyNone;
  key = warp_min(key);
  const bool fin = active && !diverged;
  const unsigned mfeas = __ballot_sync(0xffffffffu, active && feasible);
  const unsigned mdiv = __ballot_sync(0xffffffffu, active && diverged);
  const unsigned mgoal = __ballot_sync(0xffffffffu, active && goal);
  const unsigned mfin = __ballot_sync(0xffffffffu, fin);
  const double csum = warp_sum(fin ? J : 0.0);
  const long long cmin = warp_min(fin ? __double_as_longlong(J) : 0x7ff0000000000000LL);
  const unsigned ssum = __reduce_add_sync(0xffffffffu, substeps);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&st->key, key);
    atomicAdd(&st->n_feasible, static_cast<unsigned long long>(__popc(mfeas)));
    atomicAdd(&st->n_diverged, static_cast<unsigned long long>(__popc(mdiv)));
    atomicAdd(&st->n_goal, static_cast<unsigned long long>(__popc(mgoal)));
    atomicAdd(&st->n_finite, static_cast<unsigned long long>(__popc(mfin)));
    atomicAdd(&st->substeps, static_cast<unsigned long long>(ssum));
    if (mfin) {
      atomicAdd(&st->sum_cost, csum);
      atomicMin(&st->min_cost_bits, cmin);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned long long ticket = atomicAdd(&st->done_blocks, 1ULL);
    if (ticket == gridDim.x - 1) {
      __threadfence();
      const long long kmin = *reinterpret_cast<volatile long long*>(&st->key);
      const int64_t w = key_index(kmin) - P.k_begin;
      if (kmin != kKeyNone && w >= 0 && w < P.k_count) {
        st->best_cost = *reinterpret_cast<volatile double*>(&out_cost[w]);
        st->best_flags = *reinterpret_cast<volatile uint8_t*>(&out_flags[w]);
        st->best_margin = *reinterpret_cast<volatile float*>(&out_margin[w]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// fp32 fast path.  Same algorithm as rollout_kernel<float> but written for
// the SASS it produces: branch-free math (fastmath.cuh) so the four wheel
// blocks form one basic block ptxas can interleave, double-float state
// accumulators instead of fp64 (no XU conversions), terrain cell indices via
// the magic-number floor (no F2I/FRND), and the running cost of a ZOH step
// summed in fp32 before one fp64 accumulate.
__device__ __forceinline__ void df_clamp(fm::DF& a, const fm::DF& lo, const fm::DF& hi) {
  if (a.hi > hi.hi || (a.hi == hi.hi && a.lo > hi.lo)) a = hi;
  if (a.hi < lo.hi || (a.hi == lo.hi && a.lo < lo.lo)) a = lo;
}

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
    const float* __restrict__ sdf = td.sd32;
    const float4* __restrict__ hg = td.hg32;
    const float dt = K.dt;
    for (int t = 0; t < P.n_steps; ++t) {
      double u[2];
      sample_step(P.smp, base, kg == 0, t, warm, prev, u);
      const float u_dr = static_cast<float>(u[0]);
      const float u_vr = static_cast<float>(u[1]);
      const double L0 = P.w_t + P.w_c * u[0] * u[0];
      float rate_sum = 0.f;  // sum over this ZOH step's substeps of L_soft
      int nq = 0;
      for (int q = 0; q < P.S; ++q) {
        // goal truncation before accumulating
        const double gdx = x - P.goal_x, gdy = y - P.goal_y;
        if (gdx * gdx + gdy * gdy <= P.goal_r2) {
          goal = true;
          break;
        }
        float sps, cps, sth, cth, sph, cph;
        fm::sincos(psi.hi, &sps, &cps);
        fm::sincos(th.hi, &sth, &cth);
        fm::sincos(ph.hi, &sph, &cph);
        float gxf, gyf;
        const int gxi = fm::floor_frac(x * P.gx_scale + P.gx_off, gxf);
        const int gyi = fm::floor_frac(y * P.gy_scale + P.gy_off, gyf);

        // ---- L_soft(s) (constraints.hpp:87-113)
        float rate = 0.f;
        if (P.enable_dist && P.has_sdist) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float ox = cps * K.rho[i][0] - sps * K.rho[i][1];
            const float oy = sps * K.rho[i][0] + cps * K.rho[i][1];
            float fx, fy;
            int i0 = gxi + fm::floor_frac(fmaf(ox, K.inv_res, gxf), fx);
            int j0 = gyi + fm::floor_frac(fmaf(oy, K.inv_res, gyf), fy);
            if (i0 < 1) { i0 = 1; fx = 0.f; } else if (i0 >= n_hi_x) { i0 = n_hi_x; fx = 0.f; }
            if (j0 < 1) { j0 = 1; fy = 0.f; } else if (j0 >= n_hi_y) { j0 = n_hi_y; fy = 0.f; }
            const float sd = lookup_sd(sdf, P.pitch, i0, j0, fx, fy);
            const float a = fmaxf(0.f, 1.f - sd * K.inv_eps_dist);
            rate += K.sigma * a * a;
            feasible = feasible && (sd > 0.f);
            margin = fminf(margin, sd * K.inv_eps_dist);
          }
        }
        if (P.enable_rollover) {
          const float sin_abs = ph.hi < 0.f ? -sph : sph;
          const float sin_lever = sin_abs * K.esm_c_pb + cph * K.esm_s_pb;
          const float sgn = fabsf(ph.hi) <= K.esm_phi_lim ? 1.f : -1.f;
          const float U = sgn * K.esm_Mg * (K.esm_r_bar * (1.f - sin_lever) * cth);
          const float a = fmaxf(0.f, 1.f - U * K.inv_eps_esm);
          rate += K.sigma * a * a;
          feasible = feasible && (U > 0.f);
          margin = fminf(margin, U * K.inv_esm_nominal);
        }
        rate_sum += rate;
        ++nq;

        // ---- srb_derivative (dynamics.hpp:308-398)
        if (fabsf(th.hi) >= gim && fabs(fm::df_value(th)) >= P.gimbal_lim) {
          diverged = true;
          break;
        }
        const float r00 = cps * cth, r01 = cps * sph * sth - cph * sps, r02 = sph * sps + cph * cps * sth;
        const float r10 = cth * sps, r11 = cph * cps + sph * sps * sth, r12 = cph * sps * sth - cps * sph;
        const float r20 = -sth, r21 = cth * sph, r22 = cph * cth;
        const float gbx = r20 * (-K.g), gby = r21 * (-K.g), gbz = r22 * (-K.g);
        float sde, cd;
        fm::sincos(de.hi, &sde, &cd);
        const float f_x_rear = K.half_M * (u_vr - gbx + wy.hi * vz.hi - wz.hi * vy.hi);
        float fy_sum = 0.f, fz_sum = 0.f, mx = 0.f, my = 0.f, mz = 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const bool front = i < 2;
          const float rx = K.rho[i][0], ry = K.rho[i][1], rz = K.rho[i][2];
          const float rwx = r00 * rx + r01 * ry + r02 * rz;
          const float rwy = r10 * rx + r11 * ry + r12 * rz;
          const float rwz = r20 * rx + r21 * ry + r22 * rz;
          const float vix = vx.hi + (wy.hi * rz - wz.hi * ry);
          const float viy = vy.hi + (wz.hi * rx - wx.hi * rz);
          const float viz = vz.hi + (wx.hi * ry - wy.hi * rx);
          float fx, fy;
          int i0 = gxi + fm::floor_frac(fmaf(rwx, K.inv_res, gxf), fx);
          int j0 = gyi + fm::floor_frac(fmaf(rwy, K.inv_res, gyf), fy);
          if (i0 < 1) { i0 = 1; fx = 0.f; } else if (i0 >= n_hi_x) { i0 = n_hi_x; fx = 0.f; }
          if (j0 < 1) { j0 = 1; fy = 0.f; } else if (j0 >= n_hi_y) { j0 = n_hi_y; fy = 0.f; }
          float h, sfx, sfy;
          lookup_hg(td, P.pitch, i0, j0, fx, fy, h, sfx, sfy);
          const float tbx = r20 - r00 * sfx - r10 * sfy;
          const float tby = r21 - r01 * sfx - r11 * sfy;
          const float tbz = r22 - r02 * sfx - r12 * sfy;
          const float inv_tbz = fm::rcp(fmaxf(tbz, K.tau_floor));
          // chi: (z + rwz - h) with z double-float; z.hi - h is exact-ish
          const float chi = (((z.hi - h) + rwz) + z.lo) * inv_tbz;
          const float chi_dot = (tbx * (vix - chi * wy.hi) + tby * (viy + chi * wx.hi) + tbz * viz) * inv_tbz;
          const float f_k = fmaxf(K.fs_i[i] - K.k_i[i] * chi, 0.f);
          const float f_b = f_k > 0.f ? fmaxf(-K.b_i[i] * chi_dot, -f_k) : 0.f;
          const float f_z = f_k + f_b;
          const float alpha = fm::atan_ratio(viy, fmaxf(vix, K.vbx_floor)) - (front ? de.hi : 0.f);
          const float ca = K.C * alpha;
          const float f_y = f_z * (-ca * K.mu) * fm::rsqrt(K.mu2 + ca * ca);
          const float Fy = front ? f_y * cd : f_y;
          const float Fx = front ? 0.f : f_x_rear;
          fy_sum += Fy;
          fz_sum += f_z;
          mx += ry * f_z - rz * Fy;
          my += rz * Fx - rx * f_z;
          mz += rx * Fy - ry * Fx;
        }
        // euler_rates_321 (dynamics.hpp:109-118)
        const float inv_ct = fm::rcp(cth);
        const float tt = sth * inv_ct;
        const float d_psi = (sph * wy.hi + cph * wz.hi) * inv_ct;
        const float d_th = cph * wy.hi - sph * wz.hi;
        const float d_ph = wx.hi + sph * tt * wy.hi + cph * tt * wz.hi;
        const float dxw = r00 * vx.hi + r01 * vy.hi + r02 * vz.hi;
        const float dyw = r10 * vx.hi + r11 * vy.hi + r12 * vz.hi;
        const float dzw = r20 * vx.hi + r21 * vy.hi + r22 * vz.hi;
        const float d_vy = fy_sum * K.inv_M + gby + wx.hi * vz.hi - wz.hi * vx.hi;
        const float d_vz = fz_sum * K.inv_M + gbz - wx.hi * vy.hi + wy.hi * vx.hi;
        const float d_wx = (mx + K.cJx * wy.hi * wz.hi) * K.inv_Jxx;
        const float d_wy = (my - K.cJy * wx.hi * wz.hi) * K.inv_Jyy;
        const float d_wz = (mz + K.cJz * wx.hi * wy.hi) * K.inv_Jzz;
        // forward Euler + clamp_steering (dynamics.hpp:423-441,453,466)
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

// Zero the per-cycle reduction block.
__global__ void stats_reset_kernel(DevStats* st) {
  st->key = kKeyNone;
  st->done_blocks = 0;
  st->n_feasible = st->n_diverged = st->n_goal = st->n_finite = st->substeps = 0;
  st->sum_cost = 0.0;
  st->min_cost_bits = 0x7ff0000000000000LL;
  st->best_cost = __longlong_as_double(0x7ff0000000000000LL);
  st->best_margin = 0.f;
  st->best_flags = 0;
}

// Multi-GPU: after the NCCL MIN on the key, a rank keeps the winner fields
// only if it owns the global winner (others contribute zeros to the SUM).
__global__ void winner_mask_kernel(DevStats* st, const long long* global_key, int64_t k_begin,
                                   int64_t k_count) {
  const long long gk = *global_key;
  const int64_t w = key_index(gk) - k_begin;
  st->key = gk;
  if (!(gk != kKeyNone && w >= 0 && w < k_count)) {
    st->best_cost = 0.0;
    st->best_margin = 0.f;
    st->best_flags = 0;
  }
}

int rollout_block_size() { return kBlock; }

cudaError_t launch_cycle(const KParams& P, const TerrainDev& td, const double* warm, double* cost,
                         uint8_t* flags, float* margin, DevStats* st, cudaStream_t stream) {
  stats_reset_kernel<<<1, 1, 0, stream>>>(st);
  const unsigned blocks = static_cast<unsigned>((P.k_count + kBlock - 1) / kBlock);
  if (P.precision == kFp64)
    rollout_kernel<double><<<blocks, kBlock, 0, stream>>>(P, td, warm, cost, flags, margin, st);
  else
    rollout_kernel_f32<<<blocks, kBlock, 0, stream>>>(P, td, warm, cost, flags, margin, st);
  return cudaGetLastError();
}

cudaError_t launch_winner_mask(DevStats* st, const long long* gkey, int64_t k_begin,
                               int64_t k_count, cudaStream_t stream) {
  winner_mask_kernel<<<1, 1, 0, stream>>>(st, gkey, k_begin, k_count);
  return cudaGetLastError();
}

}  // namespace tmpcb
