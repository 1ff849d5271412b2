// fp64 certification kernel + per-cycle launch plumbing.
//
// rollout_kernel_f64 evaluates the same per-candidate algorithm as the fp32
// fast path (rollout_f32.cu) with fp64 math over fp64 terrain fields; it
// matches the fp64 reference planner to ~1e-12 relative even on the chaotic
// rollover rollouts of c3, and serves as the parity certification mode
// (TMPC_PRECISION_FP64).
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

#include "launch.cuh"
#include "rollout.cuh"
#include "rollout_dev.cuh"
#include "tmpc_common.h"

namespace tmpcb {

// MINB: resident CTAs per SM ptxas plans for -- 1 (up to 255 registers, no
// spills) for latency-bound batches (c2 -9%), 16 (128 registers) for
// throughput-bound ones (c3: the 1-CTA build is +42%); picked from this
// launch's K (register allocation does not change the arithmetic).
template <int MINB>
__global__ void __launch_bounds__(kBlock, MINB) rollout_kernel_f64(const KParams P, const TerrainDev td,
                                                             const double* __restrict__ warm,
                                                             double* __restrict__ out_cost,
                                                             uint8_t* __restrict__ out_flags,
                                                             float* __restrict__ out_margin,
                                                             DevStats* __restrict__ st) {
  l2_prefetch_terrain(P, td);  // the reachable terrain into L2 (rollout_dev.cuh)
  using T = double;
  const KConsts<T>& K = P.cd;
  const int64_t kl = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool active = kl < P.k_count;
  const int64_t kg = P.k_begin + kl;

  double J = 0.0;
  float margin = __int_as_float(0x7f800000);  // +inf
  bool feasible = true, diverged = false, goal = false;
  unsigned substeps = 0;

  // state (SrbState order, dynamics.hpp:167-172)
  double x = P.s0[0], y = P.s0[1], z = P.s0[2];
  double psi = P.s0[3], th = P.s0[4], ph = P.s0[5];
  double vx = P.s0[6], vy = P.s0[7], vz = P.s0[8];
  double wx = P.s0[9], wy = P.s0[10], wz = P.s0[11];
  double de = P.s0[12];

  if (active) {
    const uint64_t base = mix64(substream(P.seed, static_cast<uint64_t>(kg)));
    double prev[2] = {0.0, 0.0};
    const int n_lo = P.pad - 1, n_hi_x = P.nx + P.pad, n_hi_y = P.ny + P.pad;
    for (int t = 0; t < P.n_steps; ++t) {
      double u[2];
      sample_step(P.smp, base, kg == 0, t, warm, prev, u);
      const T u_dr = u[0], u_vr = u[1];
      const double L0 = P.w_t + P.w_c * u[0] * u[0];
      for (int q = 0; q < P.S; ++q) {
        // goal truncation before accumulating
        const double gdx = x - P.goal_x, gdy = y - P.goal_y;
        if (gdx * gdx + gdy * gdy <= P.goal_r2) {
          goal = true;
          break;
        }
        T sps, cps, sth, cth, sph, cph;
        dsincos(psi, &sps, &cps);
        dsincos(th, &sth, &cth);
        dsincos(ph, &sph, &cph);
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
            axis_cell(gxi, gxf, ox * K.inv_res, n_lo, n_hi_x, i0, fx);
            axis_cell(gyi, gyf, oy * K.inv_res, n_lo, n_hi_y, j0, fy);
            const T sd = lookup_sd(td.sd64, P.pitch, i0, j0, fx, fy);
            const T a = fmax(T(0), T(1) - sd * K.inv_eps_dist);  // soft_cost_rate(-sd)
            rate += K.sigma * a * a;
            feasible = feasible && (sd > T(0));
            margin = fminf(margin, static_cast<float>(sd * K.inv_eps_dist));
          }
        }
        if (P.enable_rollover) {
          // esm (constraints.hpp:16-23): sin(|phi| + phi_bar) via the angle sum,
          // with sin|phi| = sign(phi) sin(phi) (exact for any phi, incl. |phi| > pi)
          const T sin_abs = ph < T(0) ? -sph : sph;
          const T sin_lever = sin_abs * K.esm_c_pb + cph * K.esm_s_pb;
          const T sgn = fabs(ph) <= K.esm_phi_lim ? T(1) : T(-1);
          const T U = sgn * K.esm_Mg * (K.esm_r_bar * (T(1) - sin_lever) * cth);
          const T a = fmax(T(0), T(1) - U * K.inv_eps_esm);
          rate += K.sigma * a * a;
          feasible = feasible && (U > T(0));
          margin = fminf(margin, static_cast<float>(U * K.inv_esm_nominal));
        }
        J += P.dt * (L0 + rate);

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
        const T cd = dcos(de);
        const T f_x_rear = K.half_M * (u_vr - gbx + wy * vz - wz * vy);
        T fy_sum = T(0), fz_sum = T(0), mx = T(0), my = T(0), mz = T(0);
        // the four contact points' terrain first, so their gathers are in
        // flight together (ncu: 23% of the stall samples were gathers waited
        // for one wheel at a time)
        T hw[4], sxw[4], syw[4], rwzw[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const T rx = K.rho[i][0], ry = K.rho[i][1], rz = K.rho[i][2];
          const T rwx = r00 * rx + r01 * ry + r02 * rz;
          const T rwy = r10 * rx + r11 * ry + r12 * rz;
          rwzw[i] = r20 * rx + r21 * ry + r22 * rz;
          int i0, j0;
          T fx, fy;
          axis_cell(gxi, gxf, rwx * K.inv_res, n_lo, n_hi_x, i0, fx);
          axis_cell(gyi, gyf, rwy * K.inv_res, n_lo, n_hi_y, j0, fy);
          lookup_hg(td, P.pitch, i0, j0, fx, fy, hw[i], sxw[i], syw[i]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const bool front = i < 2;
          const T rx = K.rho[i][0], ry = K.rho[i][1], rz = K.rho[i][2];
          const T rwz = rwzw[i];
          const T vix = vx + (wy * rz - wz * ry);
          const T viy = vy + (wz * rx - wx * rz);
          const T viz = vz + (wx * ry - wy * rx);
          const T h = hw[i], sfx = sxw[i], sfy = syw[i];
          // tau_b = R^T (-fx, -fy, 1)
          const T tbx = r20 - r00 * sfx - r10 * sfy;
          const T tby = r21 - r01 * sfx - r11 * sfy;
          const T tbz = r22 - r02 * sfx - r12 * sfy;
          const T inv_tbz = T(1) / fmax(tbz, K.tau_floor);
          const T chi = ((z + rwz) - h) * inv_tbz;
          const T chi_dot = (tbx * (vix - chi * wy) + tby * (viy + chi * wx) + tbz * viz) * inv_tbz;
          const T f_k = fmax(K.fs_i[i] - K.k_i[i] * chi, T(0));
          const T f_b = f_k > T(0) ? fmax(-K.b_i[i] * chi_dot, -f_k) : T(0);
          const T f_z = f_k + f_b;
          const T alpha = datan(viy / fmax(vix, K.vbx_floor)) - (front ? de : T(0));
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
        const T d_psi = (sph * wy + cph * wz) * inv_ct;
        const T d_th = cph * wy - sph * wz;
        const T d_ph = wx + sph * tt * wy + cph * tt * wz;
        // v_w = R v_b and the 13-vector derivative (dynamics.hpp:374-389)
        const T dxw = r00 * vx + r01 * vy + r02 * vz;
        const T dyw = r10 * vx + r11 * vy + r12 * vz;
        const T dzw = r20 * vx + r21 * vy + r22 * vz;
        const T d_vy = fy_sum * K.inv_M + gby + wx * vz - wz * vx;
        const T d_vz = fz_sum * K.inv_M + gbz - wx * vy + wy * vx;
        const T d_wx = (mx + K.cJx * wy * wz) * K.inv_Jxx;
        const T d_wy = (my - K.cJy * wx * wz) * K.inv_Jyy;
        const T d_wz = (mz + K.cJz * wx * wy) * K.inv_Jzz;
        // forward Euler + clamp_steering (dynamics.hpp:423-441,453,466)
        x += P.dt * dxw;
        y += P.dt * dyw;
        z += P.dt * dzw;
        psi += P.dt * d_psi;
        th += P.dt * d_th;
        ph += P.dt * d_ph;
        vx += P.dt * u_vr;
        vy += P.dt * d_vy;
        vz += P.dt * d_vz;
        wx += P.dt * d_wx;
        wy += P.dt * d_wy;
        wz += P.dt * d_wz;
        de = fmin(fmax(de + P.dt * u_dr, -K.delta_max), K.delta_max);
        ++substeps;
        if (!isfinite(x + y + z + psi + th + ph + vx + vy + vz + wx + wy + wz + de)) {
          diverged = true;  // dynamics.hpp:491-492
          break;
        }
      }
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

void launch_rollout_f32(int lanes, const KParams& P, const TerrainDev& td, const double* warm,
                        double* cost, uint8_t* flags, float* margin, DevStats* st,
                        cudaStream_t stream);  // rollout_f32.cu
void launch_rollout_rk4_f32(int lanes, const KParams& P, const TerrainDev& td, const double* warm,
                            double* cost, uint8_t* flags, float* margin, DevStats* st,
                            cudaStream_t stream);  // rollout_rk4_f32.cu
void launch_rollout_est_f32(const KParams& P, const TerrainDev& td, const double* warm,
                            double* cost, uint8_t* flags, float* margin, DevStats* st,
                            cudaStream_t stream);
void launch_rollout_est(const KParams& P, const TerrainDev& td, const double* warm, double* cost,
                        uint8_t* flags, float* margin, DevStats* st,
                        cudaStream_t stream);  // rollout_est.cu
void launch_rollout_rk4(const KParams& P, const TerrainDev& td, const double* warm, double* cost,
                        uint8_t* flags, float* margin, DevStats* st,
                        cudaStream_t stream);  // rollout_rk4.cu

// Zero the per-cycle reduction block.
__global__ void stats_reset_kernel(DevStats* st) {
  st->key_lo = kKeyNone;
  st->key_hi = kKeyNone;
  st->done_blocks = 0;
  st->n_feasible = st->n_diverged = st->n_goal = st->n_finite = st->substeps = 0;
  st->cost_limb[0] = st->cost_limb[1] = st->cost_limb[2] = 0;
  st->min_cost_bits = 0x7ff0000000000000ULL;
  st->best_cost = __longlong_as_double(0x7ff0000000000000LL);
  st->best_margin = 0.f;
  st->best_flags = 0;
}

int rollout_block_size() { return kBlock; }

cudaError_t reset_stats(DevStats* st, cudaStream_t stream) {
  stats_reset_kernel<<<1, 1, 0, stream>>>(st);
  return cudaGetLastError();
}

cudaError_t launch_cycle(const KParams& P, const TerrainDev& td, const double* warm, double* cost,
                         uint8_t* flags, float* margin, DevStats* st, int lanes,
                         cudaStream_t stream) {
  // a one-process cycle (xn < 0) finds the block reset by the previous
  // cycle's last block (host_record) or by reset_stats (ctx.cu, when it may be dirty)
  if (P.xn >= 0) launch(stats_reset_kernel, 1, 1, stream, st);
  const unsigned blocks = static_cast<unsigned>((P.k_count + kBlock - 1) / kBlock);
  if (P.model == TMPC_MODEL_EST && P.precision != kFp64)
    launch_rollout_est_f32(P, td, warm, cost, flags, margin, st, stream);
  else if (P.model == TMPC_MODEL_EST)
    launch_rollout_est(P, td, warm, cost, flags, margin, st, stream);
  else if (P.scheme == TMPC_SCHEME_RK4 && P.precision != kFp64)
    launch_rollout_rk4_f32(lanes, P, td, warm, cost, flags, margin, st, stream);
  else if (P.scheme == TMPC_SCHEME_RK4)
    launch_rollout_rk4(P, td, warm, cost, flags, margin, st, stream);
  else if (P.precision == kFp64 && P.k_count < 32768)
    launch(rollout_kernel_f64<1>, blocks, kBlock, stream, P, td, warm, cost, flags, margin, st);
  else if (P.precision == kFp64)
    launch(rollout_kernel_f64<16>, blocks, kBlock, stream, P, td, warm, cost, flags, margin, st);
  else
    launch_rollout_f32(lanes, P, td, warm, cost, flags, margin, st, stream);
  return cudaGetLastError();
}

}  // namespace tmpcb
