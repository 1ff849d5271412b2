// Open-loop model-error analysis (harness open_loop_errors
// SPEC.md:461-467): a batch of trajectories, each the
// plant -- the reference SRB model integrated with RK4 at plant_dt (the
// harness plant) -- and a planner model (SRB or EST, the
// context's scheme and dt_int) driven open-loop from the same initial state
// by the same ZOH controls.  One thread per trajectory, fp64 throughout over
// the fp64 terrain store; per trajectory the time averages over [0, T] of
//   location error |(x^, y^) - (x, y)|
//   ESM error      |U^_ESM - U_ESM|
// with the EST model's ESM from its local-plane roll / pitch
// (est_plane_attitude, dynamics.hpp:213-219; SPEC.md design decision), both
// sampled at the start of every model substep (left rectangle rule, as the
// planner's running cost).  The plant may run on its own terrain LOD (the
// paper's unsmoothed plant LOD vs the smoothed model LODs, PAPER.md:1184-1205:
// tmpc_set_plant_terrain), on the same grid.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "launch.cuh"
#include "rollout.cuh"
#include "rollout_dev.cuh"
#include "rollout_models.cuh"
#include "tmpc_common.h"

namespace tmpcb {

namespace {

// esm (constraints.hpp:16-23) in fp64 from the hoisted constants, every
// product rounded on its own (no contraction into the caller's difference:
// the self-comparison must give exactly 0, as the reference built with
// -ffp-contract=off does).
__device__ __forceinline__ double esm64(const KConsts<double>& K, double phi, double theta) {
  const double lever = __dadd_rn(fabs(phi), K.esm_phi_bar);
  const double dh = __dmul_rn(__dmul_rn(K.esm_r_bar, __dadd_rn(1.0, -sin(lever))), cos(theta));
  return __dmul_rn((lever <= 1.5707963267948966 ? 1.0 : -1.0) * K.esm_Mg, dh);
}

// est_plane_attitude (dynamics.hpp:213-219) at (x, y): normal_at of the
// padded node fields (terrain.hpp:97-100).
__device__ __forceinline__ void plane_attitude(const KParams& P, const TerrainDev& td, double x,
                                               double y, double& phi, double& theta) {
  const int n_lo = P.pad - 1, n_hi_x = P.nx + P.pad, n_hi_y = P.ny + P.pad;
  int gxi, gyi, i0, j0;
  double gxf, gyf, fx, fy, h, sx, sy;
  split_coord(x * P.gx_scale + P.gx_off, gxi, gxf);
  split_coord(y * P.gy_scale + P.gy_off, gyi, gyf);
  axis_cell(gxi, gxf, 0.0, n_lo, n_hi_x, i0, fx);
  axis_cell(gyi, gyf, 0.0, n_lo, n_hi_y, j0, fy);
  terrain_hg(td, P.pitch, i0, j0, fx, fy, h, sx, sy);
  const double nrm = sqrt(sx * sx + sy * sy + 1.0);
  const double tx = -sx / nrm, ty = -sy / nrm;
  theta = asin(fmin(fmax(tx, -1.0), 1.0));
  const double ct = cos(theta);
  phi = asin(fmin(fmax(-ty / fmax(ct, 1e-9), -1.0), 1.0));
}

// One RK4 step of the SRB model (dynamics.hpp:454-466) + clamp_steering;
// false on the gimbal guard or a non-finite state.
__device__ __forceinline__ bool srb_rk4(const KParams& P, const TerrainDev& td, Srb13& s,
                                        double u_dr, double u_vr, double dt) {
  const KConsts<double>& K = P.cd;
  double k[13], acc[13];
  Srb13 y;
  bool ok = srb_rates(P, K, td, s, u_dr, u_vr, k);
#pragma unroll
  for (int i = 0; i < 13; ++i) {
    acc[i] = k[i];
    y.v[i] = s.v[i] + 0.5 * dt * k[i];
  }
  ok = ok && srb_rates(P, K, td, y, u_dr, u_vr, k);
#pragma unroll
  for (int i = 0; i < 13; ++i) {
    acc[i] += 2.0 * k[i];
    y.v[i] = s.v[i] + 0.5 * dt * k[i];
  }
  ok = ok && srb_rates(P, K, td, y, u_dr, u_vr, k);
#pragma unroll
  for (int i = 0; i < 13; ++i) {
    acc[i] += 2.0 * k[i];
    y.v[i] = s.v[i] + dt * k[i];
  }
  ok = ok && srb_rates(P, K, td, y, u_dr, u_vr, k);
  if (!ok) return false;
  const double h6 = dt / 6.0;
  double fin = 0.0;
#pragma unroll
  for (int i = 0; i < 13; ++i) {
    s.v[i] += h6 * (acc[i] + k[i]);
    fin += s.v[i];
  }
  s.v[12] = fmin(fmax(s.v[12], -K.delta_max), K.delta_max);
  return isfinite(fin);
}

__device__ __forceinline__ bool srb_euler(const KParams& P, const TerrainDev& td, Srb13& s,
                                          double u_dr, double u_vr, double dt) {
  double k[13];
  if (!srb_rates(P, P.cd, td, s, u_dr, u_vr, k)) return false;
  double fin = 0.0;
#pragma unroll
  for (int i = 0; i < 13; ++i) {
    s.v[i] += dt * k[i];
    fin += s.v[i];
  }
  s.v[12] = fmin(fmax(s.v[12], -P.cd.delta_max), P.cd.delta_max);
  return isfinite(fin);
}

__device__ __forceinline__ bool est_step(const KParams& P, const TerrainDev& td, Est7& s,
                                         double u_dr, double u_vr, double dt, bool rk4) {
  const KConsts<double>& K = P.cd;
  double k[7];
  est_rates(P, K, td, s, u_dr, u_vr, k);
  if (rk4) {
    double acc[7];
    Est7 y = est_axpy(s, 0.5 * dt, k);
#pragma unroll
    for (int i = 0; i < 7; ++i) acc[i] = k[i];
    est_rates(P, K, td, y, u_dr, u_vr, k);
#pragma unroll
    for (int i = 0; i < 7; ++i) acc[i] += 2.0 * k[i];
    y = est_axpy(s, 0.5 * dt, k);
    est_rates(P, K, td, y, u_dr, u_vr, k);
#pragma unroll
    for (int i = 0; i < 7; ++i) acc[i] += 2.0 * k[i];
    y = est_axpy(s, dt, k);
    est_rates(P, K, td, y, u_dr, u_vr, k);
#pragma unroll
    for (int i = 0; i < 7; ++i) acc[i] += k[i];
    s = est_axpy(s, dt / 6.0, acc);  // s + dt/6 (k1 + 2 k2 + 2 k3 + k4), dynamics.hpp:463
  } else {
    s = est_axpy(s, dt, k);
  }
  s.de = fmin(fmax(s.de, -K.delta_max), K.delta_max);
  return isfinite(s.x + s.y + s.psi + s.vby + s.wz + s.de + s.vbx);
}

// One step of the SRB system `sys` (0 the model, 1 the plant) through ONE
// call site for both (the caller loops over the systems without unrolling):
// with equal scheme and dt the model and the plant then execute the same
// instructions, so the self-comparison is exactly zero.
__device__ __noinline__ bool srb_step(const KParams& P, const TerrainDev& td, Srb13& s,
                                      double u_dr, double u_vr, double dt, bool rk4) {
  return rk4 ? srb_rk4(P, td, s, u_dr, u_vr, dt) : srb_euler(P, td, s, u_dr, u_vr, dt);
}

template <int MODEL>
__global__ void __launch_bounds__(64) open_loop_kernel(const KParams P, const TerrainDev td,
                                                       const TerrainDev tdp,
                                                       const double* __restrict__ s0,
                                                       const double* __restrict__ ctrl,
                                                       int64_t n, double plant_dt, int plant_sub,
                                                       double* __restrict__ loc_err,
                                                       double* __restrict__ esm_err,
                                                       uint8_t* __restrict__ flags) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const KConsts<double>& K = P.cd;
  Srb13 sys[2];  // [0] the SRB model, [1] the plant
#pragma unroll
  for (int i = 0; i < 13; ++i) sys[1].v[i] = s0[13 * t + i];
  sys[0] = sys[1];
  Est7 es{sys[1].v[0], sys[1].v[1], sys[1].v[3], sys[1].v[7], sys[1].v[11], sys[1].v[12],
          sys[1].v[6]};
  const bool rk4 = P.scheme == TMPC_SCHEME_RK4;
  double L = 0.0, E = 0.0;
  uint8_t fl = 0;
  const double* u = ctrl + static_cast<int64_t>(2) * P.n_steps * t;
  for (int j = 0; j < P.n_steps && !fl; ++j) {
    const double u_dr = u[2 * j], u_vr = u[2 * j + 1];
    for (int q = 0; q < P.S; ++q) {
      double xy[2][2], att[2][2];  // (x, y), (phi, theta) of model / plant
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        xy[k][0] = sys[k].v[0];
        xy[k][1] = sys[k].v[1];
        att[k][0] = sys[k].v[5];
        att[k][1] = sys[k].v[4];
      }
      if (MODEL == TMPC_MODEL_EST) {
        xy[0][0] = es.x;
        xy[0][1] = es.y;
        plane_attitude(P, td, es.x, es.y, att[0][0], att[0][1]);
      }
      double U[2];
#pragma unroll 1
      for (int k = 0; k < 2; ++k) U[k] = esm64(K, att[k][0], att[k][1]);
      const double dx = xy[0][0] - xy[1][0], dy = xy[0][1] - xy[1][1];
      L += P.dt * sqrt(dx * dx + dy * dy);
      E += P.dt * fabs(U[0] - U[1]);
      if (MODEL == TMPC_MODEL_EST && !est_step(P, td, es, u_dr, u_vr, P.dt, rk4)) fl |= 1;
#pragma unroll 1
      for (int k = MODEL == TMPC_MODEL_EST ? 1 : 0; k < 2; ++k) {
        const bool plant = k == 1;
        const int reps = plant ? plant_sub : 1;
        for (int r = 0; r < reps; ++r)
          if (!srb_step(P, plant ? tdp : td, sys[k], u_dr, u_vr, plant ? plant_dt : P.dt,
                        plant || rk4)) {
            fl |= plant ? 2 : 1;
            break;
          }
      }
      if (fl) break;
    }
  }
  const double T = P.n_steps * P.S * P.dt;
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  loc_err[t] = fl ? nan : L / T;
  esm_err[t] = fl ? nan : E / T;
  flags[t] = fl;
}

}  // namespace

cudaError_t launch_open_loop(const KParams& P, const TerrainDev& td, const TerrainDev& tdp,
                             int model, const double* s0, const double* ctrl, int64_t n,
                             double plant_dt, int plant_sub, double* loc, double* esm,
                             uint8_t* flags, cudaStream_t stream) {
  const unsigned blocks = static_cast<unsigned>((n + 63) / 64);
  if (model == TMPC_MODEL_EST)
    return launch(open_loop_kernel<TMPC_MODEL_EST>, blocks, 64, stream, P, td, tdp, s0, ctrl, n,
                  plant_dt, plant_sub, loc, esm, flags);
  return launch(open_loop_kernel<TMPC_MODEL_SRB>, blocks, 64, stream, P, td, tdp, s0, ctrl, n,
                plant_dt, plant_sub, loc, esm, flags);
}

}  // namespace tmpcb
