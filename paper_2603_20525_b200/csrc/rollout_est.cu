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
//   forward Euler + steering clamp                         dynamics.hpp:446-468
// One gather of the {H, dH/dx, dH/dy} field per substep (at the CoM) instead
// of the SRB's four, so one thread per candidate; the state is stored in fp64
// (7 entries), the math runs in T (fp32 fast path / fp64 certification).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "rollout.cuh"
#include "rollout_dev.cuh"
#include "tmpc_common.h"

namespace tmpcb {

namespace {

__device__ __forceinline__ float dasin(float a) { return asinf(a); }
__device__ __forceinline__ double dasin(double a) { return asin(a); }
__device__ __forceinline__ float dsqrt(float a) { return sqrtf(a); }
__device__ __forceinline__ double dsqrt(double a) { return sqrt(a); }

// height + gradient (bilinear of the padded node fields)
__device__ __forceinline__ void terrain_hg(const TerrainDev& td, int pitch, int i0, int j0,
                                           float fx, float fy, float& h, float& gx, float& gy) {
  const float4* r = td.hq32 + 4 * (static_cast<size_t>(j0) * pitch + i0);
  h = lerp_quad(__ldg(r), fx, fy);
  gx = lerp_quad(__ldg(r + 1), fx, fy);
  gy = lerp_quad(__ldg(r + 2), fx, fy);
}
__device__ __forceinline__ void terrain_hg(const TerrainDev& td, int pitch, int i0, int j0,
                                           double fx, double fy, double& h, double& gx,
                                           double& gy) {
  lookup_hg(td, pitch, i0, j0, fx, fy, h, gx, gy);
}
__device__ __forceinline__ float terrain_sd(const TerrainDev& td, int pitch, int i0, int j0,
                                            float fx, float fy) {
  return lerp_quad(__ldg(td.sdq32 + static_cast<size_t>(j0) * pitch + i0), fx, fy);
}
__device__ __forceinline__ double terrain_sd(const TerrainDev& td, int pitch, int i0, int j0,
                                             double fx, double fy) {
  return lookup_sd(td.sd64, pitch, i0, j0, fx, fy);
}

}  // namespace

template <typename T>
__global__ void __launch_bounds__(kBlock) rollout_kernel_est(const KParams P, const TerrainDev td,
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
  // EstState (dynamics.hpp:148-155) from the SrbState slots of s0
  double x = P.s0[0], y = P.s0[1], psi = P.s0[3], vby = P.s0[7], wz = P.s0[11];
  double de = P.s0[12], vbx = P.s0[6];

  if (active) {
    const uint64_t base = mix64(substream(P.seed, static_cast<uint64_t>(kg)));
    double prev[2] = {0.0, 0.0};
    const int n_hi_x = P.nx + 2, n_hi_y = P.ny + 2;
    const bool use_sd = P.enable_dist && P.has_sdist;
    for (int t = 0; t < P.n_steps; ++t) {
      double u[2];
      sample_step(P.smp, base, kg == 0, t, warm, prev, u);
      const T u_dr = static_cast<T>(u[0]), u_vr = static_cast<T>(u[1]);
      const double L0 = P.w_t + P.w_c * u[0] * u[0];
      for (int q = 0; q < P.S; ++q) {
        const double gdx = x - P.goal_x, gdy = y - P.goal_y;
        if (gdx * gdx + gdy * gdy <= P.goal_r2) {
          goal = true;
          break;
        }
        int gxi, gyi;
        T gxf, gyf;
        split_coord(x * P.gx_scale + P.gx_off, gxi, gxf);
        split_coord(y * P.gy_scale + P.gy_off, gyi, gyf);
        // est_plane_attitude (dynamics.hpp:213-219) via normal_at (terrain.hpp:97-100)
        int i0, j0;
        T fx, fy;
        axis_cell(gxi, gxf, T(0), n_hi_x, i0, fx);
        axis_cell(gyi, gyf, T(0), n_hi_y, j0, fy);
        T h, sx, sy;
        terrain_hg(td, P.pitch, i0, j0, fx, fy, h, sx, sy);
        const T nrm = dsqrt(sx * sx + sy * sy + T(1));
        const T tx = -sx / nrm, ty = -sy / nrm;
        const T theta = dasin(fmin(fmax(tx, T(-1)), T(1)));
        T sth, cth;
        dsincos(theta, &sth, &cth);
        const T sphi = fmin(fmax(-ty / fmax(cth, T(1e-9)), T(-1)), T(1));
        const T phi = dasin(sphi);
        T sf, cf, sp, cp;
        dsincos(phi, &sf, &cf);
        dsincos(static_cast<T>(psi), &sp, &cp);
        // rot_123 (dynamics.hpp:84-93) and g_b = R^T (0, 0, -g)
        const T r00 = cth * cp, r01 = -cth * sp;
        const T r10 = cf * sp + cp * sf * sth, r11 = cf * cp - sf * sth * sp;
        const T r21 = cp * sf + cf * sth * sp, r22 = cf * cth;
        const T g_by = r21 * (-K.g), g_bz = r22 * (-K.g);
        // est_derivative (dynamics.hpp:237-258)
        const T tvbx = static_cast<T>(vbx), tvby = static_cast<T>(vby), twz = static_cast<T>(wz);
        const T tde = static_cast<T>(de);
        const T vbx_eff = fmax(tvbx, K.vbx_floor);
        const T alpha_f = datan((tvby + twz * K.L_f) / vbx_eff) - tde;
        const T alpha_r = datan((tvby - twz * K.L_r) / vbx_eff);
        const T a_bx = u_vr - twz * tvby;
        const T f_zf = fmax(-K.kzzf * g_bz - K.kzx * a_bx, T(0));
        const T f_zr = fmax(-K.kzzr * g_bz + K.kzx * a_bx, T(0));
        const T caf = K.C * alpha_f, car = K.C * alpha_r;
        const T f_yf = f_zf * (-caf * K.mu) / dsqrt(K.mu2 + caf * caf);
        const T f_yr = f_zr * (-car * K.mu) / dsqrt(K.mu2 + car * car);
        const T d_x = r00 * tvbx + r01 * tvby, d_y = r10 * tvbx + r11 * tvby;
        const T d_vby = (f_yf + f_yr) * K.inv_M + g_by - twz * tvbx;
        const T d_wz = (f_yf * K.L_f * dcos(tde) - f_yr * K.L_r) * K.inv_Jzz;
        const T a_by = d_vby + twz * tvbx;  // EstDiagnostics::a_by (dynamics.hpp:265)
        // ---- L_soft: footprint SDF + lateral-acceleration constraint
        T rate = T(0);
        if (use_sd) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const T ox = cp * K.rho[i][0] - sp * K.rho[i][1];
            const T oy = sp * K.rho[i][0] + cp * K.rho[i][1];
            int si, sj;
            T sfx, sfy;
            axis_cell(gxi, gxf, ox * K.inv_res, n_hi_x, si, sfx);
            axis_cell(gyi, gyf, oy * K.inv_res, n_hi_y, sj, sfy);
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
        // forward Euler + clamp_steering (dynamics.hpp:423-441,453,466)
        x += P.dt * static_cast<double>(d_x);
        y += P.dt * static_cast<double>(d_y);
        psi += P.dt * static_cast<double>(twz);
        vby += P.dt * static_cast<double>(d_vby);
        wz += P.dt * static_cast<double>(d_wz);
        de = fmin(fmax(de + P.dt * u[0], -P.cd.delta_max), P.cd.delta_max);
        vbx += P.dt * u[1];
        ++substeps;
        if (!isfinite(x + y + psi + vby + wz + de + vbx)) {
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

void launch_rollout_est(const KParams& P, const TerrainDev& td, const double* warm, double* cost,
                        uint8_t* flags, float* margin, DevStats* st, cudaStream_t stream) {
  const unsigned blocks = static_cast<unsigned>((P.k_count + kBlock - 1) / kBlock);
  if (P.precision == kFp64)
    rollout_kernel_est<double><<<blocks, kBlock, 0, stream>>>(P, td, warm, cost, flags, margin, st);
  else
    rollout_kernel_est<float><<<blocks, kBlock, 0, stream>>>(P, td, warm, cost, flags, margin, st);
}

}  // namespace tmpcb
