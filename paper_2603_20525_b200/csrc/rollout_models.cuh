// Precision-generic model derivatives shared by the fp64 / generic rollout
// kernels (rollout_rk4.cu, rollout_est.cu) and the open-loop analysis kernel
// (open_loop.cu): srb_derivative (dynamics.hpp:308-398) and
// est_plane_attitude + est_derivative (dynamics.hpp:213-275) over the padded
// terrain store.  Internal linkage per translation unit, as when they lived
// in the kernels' own files.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "rollout.cuh"
#include "rollout_dev.cuh"

namespace tmpcb {
namespace {

struct Srb13 {
  double v[13];  // SrbState::as_array order (dynamics.hpp:167-172)
};

// srb_derivative (dynamics.hpp:308-398) of state s in math type T; false on
// the gimbal guard (dynamics.hpp:311-312).
template <typename T>
__device__ __forceinline__ bool srb_rates(const KParams& P, const KConsts<T>& K,
                                          const TerrainDev& td, const Srb13& s, T u_dr, T u_vr,
                                          double d[13]) {
  const double th = s.v[4];
  if (fabs(th) >= P.gimbal_lim) return false;
  const int n_lo = P.pad - 1, n_hi_x = P.nx + P.pad, n_hi_y = P.ny + P.pad;
  T sps, cps, sth, cth, sph, cph;
  dsincos(static_cast<T>(s.v[3]), &sps, &cps);
  dsincos(static_cast<T>(th), &sth, &cth);
  dsincos(static_cast<T>(s.v[5]), &sph, &cph);
  const T vx = static_cast<T>(s.v[6]), vy = static_cast<T>(s.v[7]), vz = static_cast<T>(s.v[8]);
  const T wx = static_cast<T>(s.v[9]), wy = static_cast<T>(s.v[10]), wz = static_cast<T>(s.v[11]);
  const T de = static_cast<T>(s.v[12]);
  int gxi, gyi;
  T gxf, gyf;
  split_coord(s.v[0] * P.gx_scale + P.gx_off, gxi, gxf);
  split_coord(s.v[1] * P.gy_scale + P.gy_off, gyi, gyf);
  // rot_321 (dynamics.hpp:96-105)
  const T r00 = cps * cth, r01 = cps * sph * sth - cph * sps, r02 = sph * sps + cph * cps * sth;
  const T r10 = cth * sps, r11 = cph * cps + sph * sps * sth, r12 = cph * sps * sth - cps * sph;
  const T r20 = -sth, r21 = cth * sph, r22 = cph * cth;
  const T gbx = r20 * (-K.g), gby = r21 * (-K.g), gbz = r22 * (-K.g);
  const T cd = dcos(de);
  const T f_x_rear = K.half_M * (u_vr - gbx + wy * vz - wz * vy);
  T fy_sum = T(0), fz_sum = T(0), mx = T(0), my = T(0), mz = T(0);
  // the four contact points' terrain first: their gathers in flight together
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
    terrain_hg(td, P.pitch, i0, j0, fx, fy, hw[i], sxw[i], syw[i]);
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
    // tau_b = R^T (-fx, -fy, 1) (dynamics.hpp:338-341)
    const T tbx = r20 - r00 * sfx - r10 * sfy;
    const T tby = r21 - r01 * sfx - r11 * sfy;
    const T tbz = r22 - r02 * sfx - r12 * sfy;
    const T inv_tbz = T(1) / fmax(tbz, K.tau_floor);
    // extension in fp64 position space (z + R rho_z - h), then T
    const T chi = static_cast<T>((s.v[2] + static_cast<double>(rwz)) - static_cast<double>(h)) *
                  inv_tbz;
    const T chi_dot = (tbx * (vix - chi * wy) + tby * (viy + chi * wx) + tbz * viz) * inv_tbz;
    const T f_k = fmax(K.fs_i[i] - K.k_i[i] * chi, T(0));
    const T f_b = f_k > T(0) ? fmax(-K.b_i[i] * chi_dot, -f_k) : T(0);
    const T f_z = f_k + f_b;
    const T alpha = datan(viy / fmax(vix, K.vbx_floor)) - (front ? de : T(0));
    const T ca = K.C * alpha;
    const T f_y = f_z * (-ca * K.mu) / dsqrt(K.mu2 + ca * ca);
    const T Fy = front ? f_y * cd : f_y;
    const T Fx = front ? T(0) : f_x_rear;
    fy_sum += Fy;
    fz_sum += f_z;
    mx += ry * f_z - rz * Fy;
    my += rz * Fx - rx * f_z;
    mz += rx * Fy - ry * Fx;
  }
  // euler_rates_321 (dynamics.hpp:109-118), v_w = R v_b (374-389)
  const T inv_ct = T(1) / cth;
  const T tt = sth * inv_ct;
  d[0] = static_cast<double>(r00 * vx + r01 * vy + r02 * vz);
  d[1] = static_cast<double>(r10 * vx + r11 * vy + r12 * vz);
  d[2] = static_cast<double>(r20 * vx + r21 * vy + r22 * vz);
  d[3] = static_cast<double>((sph * wy + cph * wz) * inv_ct);
  d[4] = static_cast<double>(cph * wy - sph * wz);
  d[5] = static_cast<double>(wx + sph * tt * wy + cph * tt * wz);
  d[6] = static_cast<double>(u_vr);
  d[7] = static_cast<double>(fy_sum * K.inv_M + gby + wx * vz - wz * vx);
  d[8] = static_cast<double>(fz_sum * K.inv_M + gbz - wx * vy + wy * vx);
  d[9] = static_cast<double>((mx + K.cJx * wy * wz) * K.inv_Jxx);
  d[10] = static_cast<double>((my - K.cJy * wx * wz) * K.inv_Jyy);
  d[11] = static_cast<double>((mz + K.cJz * wx * wy) * K.inv_Jzz);
  d[12] = static_cast<double>(u_dr);
  return true;
}

// EstState in fp64 (dynamics.hpp:148-155), SrbState slot order of s0 noted.
struct Est7 {
  double x, y, psi, vby, wz, de, vbx;  // s0[0], s0[1], s0[3], s0[7], s0[11], s0[12], s0[6]
};

// est_plane_attitude + est_derivative (dynamics.hpp:213-275) at state s.
// Writes the four non-trivial rates (d_psi = wz, d_delta = u_dr and
// d_vbx = u_vr are the inputs) and the diagnostics g_by / a_by; also hands
// back the CoM cell split and sin/cos psi for the footprint SDF lookups.
template <typename T>
__device__ __forceinline__ void est_deriv(const KParams& P, const KConsts<T>& K,
                                          const TerrainDev& td, const Est7& s, T u_dr, T u_vr,
                                          T& d_x, T& d_y, T& d_vby, T& d_wz, T& g_by, T& a_by,
                                          int& gxi, T& gxf, int& gyi, T& gyf, T& sp, T& cp) {
  (void)u_dr;
  const int n_lo = P.pad - 1, n_hi_x = P.nx + P.pad, n_hi_y = P.ny + P.pad;
  split_coord(s.x * P.gx_scale + P.gx_off, gxi, gxf);
  split_coord(s.y * P.gy_scale + P.gy_off, gyi, gyf);
  // est_plane_attitude (dynamics.hpp:213-219) via normal_at (terrain.hpp:97-100)
  int i0, j0;
  T fx, fy;
  axis_cell(gxi, gxf, T(0), n_lo, n_hi_x, i0, fx);
  axis_cell(gyi, gyf, T(0), n_lo, n_hi_y, j0, fy);
  T h, sx, sy;
  terrain_hg(td, P.pitch, i0, j0, fx, fy, h, sx, sy);
  const T nrm = dsqrt(sx * sx + sy * sy + T(1));
  const T tx = -sx / nrm, ty = -sy / nrm;
  const T theta = dasin(fmin(fmax(tx, T(-1)), T(1)));
  T sth, cth;
  dsincos(theta, &sth, &cth);
  const T sphi = fmin(fmax(-ty / fmax(cth, T(1e-9)), T(-1)), T(1));
  const T phi = dasin(sphi);
  T sf, cf;
  dsincos(phi, &sf, &cf);
  dsincos(static_cast<T>(s.psi), &sp, &cp);
  // rot_123 (dynamics.hpp:84-93) and g_b = R^T (0, 0, -g)
  const T r00 = cth * cp, r01 = -cth * sp;
  const T r10 = cf * sp + cp * sf * sth, r11 = cf * cp - sf * sth * sp;
  const T r21 = cp * sf + cf * sth * sp, r22 = cf * cth;
  g_by = r21 * (-K.g);
  const T g_bz = r22 * (-K.g);
  // est_derivative (dynamics.hpp:237-258)
  const T tvbx = static_cast<T>(s.vbx), tvby = static_cast<T>(s.vby), twz = static_cast<T>(s.wz);
  const T tde = static_cast<T>(s.de);
  const T vbx_eff = fmax(tvbx, K.vbx_floor);
  const T alpha_f = datan((tvby + twz * K.L_f) / vbx_eff) - tde;
  const T alpha_r = datan((tvby - twz * K.L_r) / vbx_eff);
  const T a_bx = u_vr - twz * tvby;
  const T f_zf = fmax(-K.kzzf * g_bz - K.kzx * a_bx, T(0));
  const T f_zr = fmax(-K.kzzr * g_bz + K.kzx * a_bx, T(0));
  const T caf = K.C * alpha_f, car = K.C * alpha_r;
  const T f_yf = f_zf * (-caf * K.mu) / dsqrt(K.mu2 + caf * caf);
  const T f_yr = f_zr * (-car * K.mu) / dsqrt(K.mu2 + car * car);
  d_x = r00 * tvbx + r01 * tvby;
  d_y = r10 * tvbx + r11 * tvby;
  d_vby = (f_yf + f_yr) * K.inv_M + g_by - twz * tvbx;
  d_wz = (f_yf * K.L_f * dcos(tde) - f_yr * K.L_r) * K.inv_Jzz;
  a_by = d_vby + twz * tvbx;  // EstDiagnostics::a_by (dynamics.hpp:265)
}

// The 7 rates of EstModel::derivative in fp64 (EstState order of Est7).
template <typename T>
__device__ __forceinline__ void est_rates(const KParams& P, const KConsts<T>& K,
                                          const TerrainDev& td, const Est7& s, T u_dr, T u_vr,
                                          double k[7]) {
  T d_x, d_y, d_vby, d_wz, g_by, a_by, gxf, gyf, sp, cp;
  int gxi, gyi;
  est_deriv(P, K, td, s, u_dr, u_vr, d_x, d_y, d_vby, d_wz, g_by, a_by, gxi, gxf, gyi, gyf, sp,
            cp);
  k[0] = static_cast<double>(d_x);
  k[1] = static_cast<double>(d_y);
  k[2] = static_cast<double>(static_cast<T>(s.wz));
  k[3] = static_cast<double>(d_vby);
  k[4] = static_cast<double>(d_wz);
  k[5] = static_cast<double>(u_dr);
  k[6] = static_cast<double>(u_vr);
}

__device__ __forceinline__ Est7 est_axpy(const Est7& s, double h, const double k[7]) {
  return Est7{s.x + h * k[0],   s.y + h * k[1],  s.psi + h * k[2], s.vby + h * k[3],
              s.wz + h * k[4],  s.de + h * k[5], s.vbx + h * k[6]};
}

}  // namespace
}  // namespace tmpcb
