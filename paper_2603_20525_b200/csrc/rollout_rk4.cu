// RK4 instantiation of the SRB rollout kernel: the
// reference's Scheme::kRk4 substep (dynamics.hpp:454-466) in-kernel.
//
// Per candidate and substep (identical to oracle/tmpc_oracle.cpp rollout +
// rk4_update and to oracle/_ref over integrate_step<SrbModel>(.., kRk4)):
//   goal test, L_soft at the substep's start state (SPEC.md:372,374,
//       constraints.hpp:16-23,87-113) — as in the Euler kernels
//   k1..k4 = srb_derivative at s, s + dt/2 k1, s + dt/2 k2, s + dt k3
//       (dynamics.hpp:308-398; the gimbal guard of ANY stage diverges the
//       candidate, as the reference's std::domain_error does)
//   s += dt/6 (k1 + 2 k2 + 2 k3 + k4); clamp_steering (dynamics.hpp:440,466)
// The 13-entry state, the stage states and the combination are fp64 in both
// precision modes; the derivative math runs in T over the fp32 (hq32) or fp64
// (hg64) terrain store.  One thread per candidate: RK4 quadruples the
// derivative work per substep, so even small K fill the machine with enough
// independent math per thread.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "launch.cuh"
#include "rollout.cuh"
#include "rollout_dev.cuh"
#include "rollout_models.cuh"
#include "tmpc_common.h"

namespace tmpcb {

template <typename T, int MINB>  // MINB as rollout_kernel_f64 (rollout.cu)
__global__ void __launch_bounds__(kBlock, MINB) rollout_kernel_rk4(const KParams P, const TerrainDev td,
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
  Srb13 s;
#pragma unroll
  for (int i = 0; i < 13; ++i) s.v[i] = P.s0[i];

  if (active) {
    const uint64_t base = mix64(substream(P.seed, static_cast<uint64_t>(kg)));
    double prev[2] = {0.0, 0.0};
    const int n_lo = P.pad - 1, n_hi_x = P.nx + P.pad, n_hi_y = P.ny + P.pad;
    for (int t = 0; t < P.n_steps; ++t) {
      double u[2];
      sample_step(P.smp, base, kg == 0, t, warm, prev, u);
      const T u_dr = static_cast<T>(u[0]), u_vr = static_cast<T>(u[1]);
      const double L0 = P.w_t + P.w_c * u[0] * u[0];
      for (int q = 0; q < P.S; ++q) {
        const double gdx = s.v[0] - P.goal_x, gdy = s.v[1] - P.goal_y;
        if (gdx * gdx + gdy * gdy <= P.goal_r2) {
          goal = true;
          break;
        }
        // ---- L_soft(s) at the start state (constraints.hpp:16-23,87-113)
        T rate = T(0);
        if (P.enable_dist && P.has_sdist) {
          T sps, cps;
          dsincos(static_cast<T>(s.v[3]), &sps, &cps);
          int gxi, gyi;
          T gxf, gyf;
          split_coord(s.v[0] * P.gx_scale + P.gx_off, gxi, gxf);
          split_coord(s.v[1] * P.gy_scale + P.gy_off, gyi, gyf);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const T ox = cps * K.rho[i][0] - sps * K.rho[i][1];
            const T oy = sps * K.rho[i][0] + cps * K.rho[i][1];
            int i0, j0;
            T fx, fy;
            axis_cell(gxi, gxf, ox * K.inv_res, n_lo, n_hi_x, i0, fx);
            axis_cell(gyi, gyf, oy * K.inv_res, n_lo, n_hi_y, j0, fy);
            const T sd = terrain_sd(td, P.pitch, i0, j0, fx, fy);
            const T a = fmax(T(0), T(1) - sd * K.inv_eps_dist);
            rate += K.sigma * a * a;
            feasible = feasible && (sd > T(0));
            margin = fminf(margin, static_cast<float>(sd * K.inv_eps_dist));
          }
        }
        if (P.enable_rollover) {
          T sth, cth, sph, cph;
          dsincos(static_cast<T>(s.v[4]), &sth, &cth);
          dsincos(static_cast<T>(s.v[5]), &sph, &cph);
          const T ph = static_cast<T>(s.v[5]);
          const T sin_abs = ph < T(0) ? -sph : sph;
          const T sin_lever = sin_abs * K.esm_c_pb + cph * K.esm_s_pb;
          const T sgn = fabs(ph) <= K.esm_phi_lim ? T(1) : T(-1);
          const T U = sgn * K.esm_Mg * (K.esm_r_bar * (T(1) - sin_lever) * cth);
          const T a = fmax(T(0), T(1) - U * K.inv_eps_esm);
          rate += K.sigma * a * a;
          feasible = feasible && (U > T(0));
          margin = fminf(margin, static_cast<float>(U * K.inv_esm_nominal));
        }
        J += P.dt * (L0 + static_cast<double>(rate));

        // ---- Scheme::kRk4 (dynamics.hpp:454-465)
        double k[13], acc[13];
        Srb13 y;
        bool ok = srb_rates(P, K, td, s, u_dr, u_vr, k);
#pragma unroll
        for (int i = 0; i < 13; ++i) {
          acc[i] = k[i];
          y.v[i] = s.v[i] + 0.5 * P.dt * k[i];
        }
        ok = ok && srb_rates(P, K, td, y, u_dr, u_vr, k);
#pragma unroll
        for (int i = 0; i < 13; ++i) {
          acc[i] += 2.0 * k[i];
          y.v[i] = s.v[i] + 0.5 * P.dt * k[i];
        }
        ok = ok && srb_rates(P, K, td, y, u_dr, u_vr, k);
#pragma unroll
        for (int i = 0; i < 13; ++i) {
          acc[i] += 2.0 * k[i];
          y.v[i] = s.v[i] + P.dt * k[i];
        }
        ok = ok && srb_rates(P, K, td, y, u_dr, u_vr, k);
        if (!ok) {
          diverged = true;  // gimbal guard in a stage (dynamics.hpp:311-312)
          break;
        }
        const double h6 = P.dt / 6.0;
        double fin = 0.0;
#pragma unroll
        for (int i = 0; i < 13; ++i) {
          s.v[i] += h6 * (acc[i] + k[i]);
          fin += s.v[i];
        }
        s.v[12] = fmin(fmax(s.v[12], -P.cd.delta_max), P.cd.delta_max);
        ++substeps;
        if (!isfinite(fin)) {
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
      const double gdx = s.v[0] - P.goal_x, gdy = s.v[1] - P.goal_y;
      J += P.w_g * sqrt(gdx * gdx + gdy * gdy);
    }
  }
  reduce_and_finalize(P, active, kl, kg, J, feasible, diverged, goal, margin, substeps, out_cost,
                      out_flags, out_margin, st);
}

void launch_rollout_rk4(const KParams& P, const TerrainDev& td, const double* warm, double* cost,
                        uint8_t* flags, float* margin, DevStats* st, cudaStream_t stream) {
  const unsigned blocks = static_cast<unsigned>((P.k_count + kBlock - 1) / kBlock);
  if (P.precision == kFp64)
    if (P.k_count < 32768)
      launch(rollout_kernel_rk4<double, 1>, blocks, kBlock, stream, P, td, warm, cost, flags, margin, st);
    else
      launch(rollout_kernel_rk4<double, 16>, blocks, kBlock, stream, P, td, warm, cost, flags, margin, st);
  else
    launch(rollout_kernel_rk4<float, 16>, blocks, kBlock, stream, P, td, warm, cost, flags, margin, st);
}

}  // namespace tmpcb
