// EST formulation of the rollout kernel: the paper's
// baseline extended single-track model as a second instantiation of K2.
//
// Per candidate and 5 ms substep (identical to oracle/tmpc_oracle.cpp
// rollout_est and oracle/_ref rollout_est):
//   goal test
//   est_plane_attitude: normal_at the CoM -> theta = asin(tau_x),
//       phi = asin(-tau_y / max(cos theta, 1e-9))          dynamics.hpp:213-219
//   est_derivative: rot_123(phi, theta, psi), g_b, virtual-tire slip angles,
//       normal loads (clamped at 0), sigmoid tire forces   dynamics.hpp:230-275
//   L_soft: wheel-footprint SDF costs + the lateral-acceleration constraint
//       |a_by - g_by| - a_by_bar, eps = safety_factor * a_by_bar
//                                                          constraints.hpp:62-65,78-80,87-113
//   forward Euler, or RK4 (P.scheme, three more derivative stages), then the
//       steering clamp                                     dynamics.hpp:446-468
// One gather of the {H, dH/dx, dH/dy} field per derivative (at the CoM)
// instead of the SRB's four, so one thread per candidate; the state is stored
// in fp64 (7 entries), the math runs in T (fp32 fast path / fp64
// certification).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "launch.cuh"
#include "rollout.cuh"
#include "rollout_dev.cuh"
#include "rollout_models.cuh"
#include "tmpc_common.h"

namespace tmpcb {

template <typename T>
__global__ void __launch_bounds__(kBlock) rollout_kernel_est(const KParams P, const TerrainDev td,
                                                             const double* __restrict__ warm,
                                                             double* __restrict__ out_cost,
                                                             uint8_t* __restrict__ out_flags,
                                                             float* __restrict__ out_margin,
                                                             DevStats* __restrict__ st) {
  l2_prefetch_terrain(P, td);  // the reachable terrain into L2 (rollout_dev.cuh)
  const KConsts<T>& K = consts<T>(P);
  const int64_t kl = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool active = kl < P.k_count;
  const int64_t kg = P.k_begin + kl;

  double J = 0.0;
  float margin = __int_as_float(0x7f800000);  // +inf
  bool feasible = true, diverged = false, goal = false;
  unsigned substeps = 0;
  // EstState (dynamics.hpp:148-155) from the SrbState slots of s0
  Est7 s{P.s0[0], P.s0[1], P.s0[3], P.s0[7], P.s0[11], P.s0[12], P.s0[6]};
  const bool rk4 = P.scheme == TMPC_SCHEME_RK4;

  if (active) {
    const uint64_t base = mix64(substream(P.seed, static_cast<uint64_t>(kg)));
    double prev[2] = {0.0, 0.0};
    const int n_lo = P.pad - 1, n_hi_x = P.nx + P.pad, n_hi_y = P.ny + P.pad;
    const bool use_sd = P.enable_dist && P.has_sdist;
    for (int t = 0; t < P.n_steps; ++t) {
      double u[2];
      sample_step(P.smp, base, kg == 0, t, warm, prev, u);
      const T u_dr = static_cast<T>(u[0]), u_vr = static_cast<T>(u[1]);
      const double L0 = P.w_t + P.w_c * u[0] * u[0];
      for (int q = 0; q < P.S; ++q) {
        const double gdx = s.x - P.goal_x, gdy = s.y - P.goal_y;
        if (gdx * gdx + gdy * gdy <= P.goal_r2) {
          goal = true;
          break;
        }
        T d_x, d_y, d_vby, d_wz, g_by, a_by, gxf, gyf, sp, cp;
        int gxi, gyi;
        est_deriv(P, K, td, s, u_dr, u_vr, d_x, d_y, d_vby, d_wz, g_by, a_by, gxi, gxf, gyi, gyf,
                  sp, cp);
        // ---- L_soft: footprint SDF + lateral-acceleration constraint
        T rate = T(0);
        if (use_sd) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const T ox = cp * K.rho[i][0] - sp * K.rho[i][1];
            const T oy = sp * K.rho[i][0] + cp * K.rho[i][1];
            int si, sj;
            T sfx, sfy;
            axis_cell(gxi, gxf, ox * K.inv_res, n_lo, n_hi_x, si, sfx);
            axis_cell(gyi, gyf, oy * K.inv_res, n_lo, n_hi_y, sj, sfy);
            const T sd = terrain_sd(td, P.pitch, si, sj, sfx, sfy);
            const T a = fmax(T(0), T(1) - sd * K.inv_eps_dist);
            rate += K.sigma * a * a;
            feasible = feasible && (sd > T(0));
            margin = fminf(margin, static_cast<float>(sd * K.inv_eps_dist));
          }
        }
        if (P.enable_rollover) {
          const T pi_aby = fabs(a_by - g_by) - K.a_by_bar;  // constraints.hpp:62-65
          const T a = fmax(T(0), T(1) + pi_aby * K.inv_eps_aby);
          rate += K.sigma * a * a;
          feasible = feasible && (pi_aby < T(0));
          margin = fminf(margin, static_cast<float>(-pi_aby * K.inv_a_by_bar));
        }
        J += P.dt * (L0 + static_cast<double>(rate));
        if (!rk4) {
          // forward Euler + clamp_steering (dynamics.hpp:423-441,453,466)
          s.x += P.dt * static_cast<double>(d_x);
          s.y += P.dt * static_cast<double>(d_y);
          s.psi += P.dt * static_cast<double>(static_cast<T>(s.wz));
          s.vby += P.dt * static_cast<double>(d_vby);
          s.wz += P.dt * static_cast<double>(d_wz);
          s.de = s.de + P.dt * u[0];
          s.vbx += P.dt * u[1];
        } else {
          // Scheme::kRk4 (dynamics.hpp:454-465): k1 is the derivative above
          double k1[7] = {static_cast<double>(d_x),   static_cast<double>(d_y),
                          static_cast<double>(static_cast<T>(s.wz)), static_cast<double>(d_vby),
                          static_cast<double>(d_wz),  static_cast<double>(u_dr),
                          static_cast<double>(u_vr)};
          double k2[7], k3[7], k4[7];
          est_rates(P, K, td, est_axpy(s, 0.5 * P.dt, k1), u_dr, u_vr, k2);
          est_rates(P, K, td, est_axpy(s, 0.5 * P.dt, k2), u_dr, u_vr, k3);
          est_rates(P, K, td, est_axpy(s, P.dt, k3), u_dr, u_vr, k4);
          const double h6 = P.dt / 6.0;
          double c[7];
#pragma unroll
          for (int i = 0; i < 7; ++i) c[i] = h6 * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
          s = Est7{s.x + c[0], s.y + c[1], s.psi + c[2], s.vby + c[3], s.wz + c[4], s.de + c[5],
                   s.vbx + c[6]};
        }
        s.de = fmin(fmax(s.de, -P.cd.delta_max), P.cd.delta_max);
        ++substeps;
        if (!isfinite(s.x + s.y + s.psi + s.vby + s.wz + s.de + s.vbx)) {
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
      const double gdx = s.x - P.goal_x, gdy = s.y - P.goal_y;
      J += P.w_g * sqrt(gdx * gdx + gdy * gdy);
    }
  }
  reduce_and_finalize(P, active, kl, kg, J, feasible, diverged, goal, margin, substeps, out_cost,
                      out_flags, out_margin, st);
}

void launch_rollout_est(const KParams& P, const TerrainDev& td, const double* warm, double* cost,
                        uint8_t* flags, float* margin, DevStats* st, cudaStream_t stream) {
  const unsigned blocks = static_cast<unsigned>((P.k_count + kBlock - 1) / kBlock);
  if (P.precision == kFp64)
    launch(rollout_kernel_est<double>, blocks, kBlock, stream, P, td, warm, cost, flags, margin, st);
  else
    launch(rollout_kernel_est<float>, blocks, kBlock, stream, P, td, warm, cost, flags, margin, st);
}

}  // namespace tmpcb
