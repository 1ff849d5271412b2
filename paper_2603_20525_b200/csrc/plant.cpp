// Host fp64 plant for the closed-loop receding-horizon driver (BASELINE c5,
// SURVEY §8f row 1, App. A D8): the reference SRB model integrated with RK4 at
// a fine step between planning cycles, like the SPEC harness plant_step
// ("SRB dynamics at RK4/1 ms substeps").
//
// Restates, in fp64 and in the reference's operation order, srb_derivative
// (dynamics.hpp:308-398) over height_at / gradient_at (terrain.hpp:35-50,
// 79-93) and integrate_step's RK4 branch + clamp_steering
// (dynamics.hpp:446-468).  Runs once per planning cycle on the CPU; the
// planning hot path never calls it.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>

#include "tmpc_b200.h"

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kVbxFloor = 0.1;       // dynamics.hpp:15
constexpr double kGimbalMargin = 1e-3;  // dynamics.hpp:16

struct Terr {
  const tmpc_terrain* t;
  // detail::bilinear (terrain.hpp:35-50)
  double bilinear(double x, double y) const {
    double gx = (x - t->origin_x) / t->resolution;
    double gy = (y - t->origin_y) / t->resolution;
    gx = std::clamp(gx, 0.0, static_cast<double>(t->nx - 1));
    gy = std::clamp(gy, 0.0, static_cast<double>(t->ny - 1));
    const int i0 = std::min(static_cast<int>(gx), t->nx - 2);
    const int j0 = std::min(static_cast<int>(gy), t->ny - 2);
    const double fx = gx - i0, fy = gy - j0;
    const double* r0 = t->heights + static_cast<size_t>(j0) * t->nx + i0;
    const double* r1 = r0 + t->nx;
    const double a = r0[0] + fx * (r0[1] - r0[0]);
    const double b = r1[0] + fx * (r1[1] - r1[0]);
    return a + fy * (b - a);
  }
};

// srb_derivative (dynamics.hpp:308-398); false on the gimbal guard.
bool srb_derivative(const tmpc_params& p, const Terr& T, const double* s, double u_dr,
                    double u_vr, double* d) {
  if (std::fabs(s[4]) >= kPi / 2 - kGimbalMargin) return false;
  const double psi = s[3], th = s[4], ph = s[5];
  const double cf = std::cos(ph), sf = std::sin(ph);
  const double ct = std::cos(th), st = std::sin(th);
  const double cp = std::cos(psi), sp = std::sin(psi);
  const double r[3][3] = {{cp * ct, cp * sf * st - cf * sp, sf * sp + cf * cp * st},
                          {ct * sp, cf * cp + sf * sp * st, cf * sp * st - cp * sf},
                          {-st, ct * sf, cf * ct}};
  const double g = p.g;
  const double gb[3] = {r[2][0] * (-g), r[2][1] * (-g), r[2][2] * (-g)};
  const double vb[3] = {s[6], s[7], s[8]}, w[3] = {s[9], s[10], s[11]};
  const double L = p.L_f + p.L_r;
  const double kzz[2] = {p.M * p.L_r / L, p.M * p.L_f / L};
  const double zo = -(p.h + p.R);
  const double rho[4][3] = {{p.L_f, p.e / 2, zo}, {p.L_f, -p.e / 2, zo},
                            {-p.L_r, p.e / 2, zo}, {-p.L_r, -p.e / 2, zo}};
  const double cd = std::cos(s[12]);
  double fy_sum = 0.0, fz_sum = 0.0, m[3] = {0.0, 0.0, 0.0};
  const double f_x_rear = 0.5 * p.M * (u_vr - gb[0] + w[1] * vb[2] - w[2] * vb[1]);
  const double res = T.t->resolution;
  for (int i = 0; i < 4; ++i) {
    const bool front = i < 2;
    const double* q = rho[i];
    const double pw[3] = {s[0] + (r[0][0] * q[0] + r[0][1] * q[1] + r[0][2] * q[2]),
                          s[1] + (r[1][0] * q[0] + r[1][1] * q[1] + r[1][2] * q[2]),
                          s[2] + (r[2][0] * q[0] + r[2][1] * q[1] + r[2][2] * q[2])};
    const double vi[3] = {vb[0] + (w[1] * q[2] - w[2] * q[1]), vb[1] + (w[2] * q[0] - w[0] * q[2]),
                          vb[2] + (w[0] * q[1] - w[1] * q[0])};
    // gradient_at: central differences of height_at (terrain.hpp:89-93)
    const double fx = (T.bilinear(pw[0] + res, pw[1]) - T.bilinear(pw[0] - res, pw[1])) / (2.0 * res);
    const double fyg = (T.bilinear(pw[0], pw[1] + res) - T.bilinear(pw[0], pw[1] - res)) / (2.0 * res);
    const double tw[3] = {-fx, -fyg, 1.0};
    const double tb[3] = {r[0][0] * tw[0] + r[1][0] * tw[1] + r[2][0] * tw[2],
                          r[0][1] * tw[0] + r[1][1] * tw[1] + r[2][1] * tw[2],
                          r[0][2] * tw[0] + r[1][2] * tw[1] + r[2][2] * tw[2]};
    const double tbz = std::max(tb[2], 1e-6);
    const double chi = (pw[2] - T.bilinear(pw[0], pw[1])) / tbz;
    const double a[3] = {vi[0] - chi * w[1], vi[1] - chi * (-w[0]), vi[2] - chi * 0.0};
    const double chi_dot = (tb[0] * a[0] + tb[1] * a[1] + tb[2] * a[2]) / tbz;
    const double f_s = 0.5 * g * kzz[front ? 0 : 1];
    const double k_i = front ? p.k_f : p.k_r, b_i = front ? p.b_f : p.b_r;
    const double f_k = std::max(f_s - k_i * chi, 0.0);
    const double f_b = f_k > 0.0 ? std::max(-b_i * chi_dot, -f_k) : 0.0;
    const double f_z = f_k + f_b;
    const double alpha = std::atan(vi[1] / std::max(vi[0], kVbxFloor)) - (front ? s[12] : 0.0);
    const double ca = p.C * alpha;
    const double f_y = f_z * (-ca * p.mu) / std::sqrt(p.mu * p.mu + ca * ca);
    const double cos_di = front ? cd : 1.0;
    fy_sum += f_y * cos_di;
    fz_sum += f_z;
    const double F[3] = {front ? 0.0 : f_x_rear, f_y * cos_di, f_z};
    m[0] += q[1] * F[2] - q[2] * F[1];
    m[1] += q[2] * F[0] - q[0] * F[2];
    m[2] += q[0] * F[1] - q[1] * F[0];
  }
  const double tt = std::tan(th);
  d[0] = r[0][0] * vb[0] + r[0][1] * vb[1] + r[0][2] * vb[2];
  d[1] = r[1][0] * vb[0] + r[1][1] * vb[1] + r[1][2] * vb[2];
  d[2] = r[2][0] * vb[0] + r[2][1] * vb[1] + r[2][2] * vb[2];
  d[3] = (sf * w[1] + cf * w[2]) / ct;
  d[4] = cf * w[1] - sf * w[2];
  d[5] = w[0] + sf * tt * w[1] + cf * tt * w[2];
  d[6] = u_vr;
  d[7] = fy_sum / p.M + gb[1] + w[0] * vb[2] - w[2] * vb[0];
  d[8] = fz_sum / p.M + gb[2] - w[0] * vb[1] + w[1] * vb[0];
  d[9] = (m[0] + (p.J_yy - p.J_zz) * w[1] * w[2]) / p.J_xx;
  d[10] = (m[1] - (p.J_xx - p.J_zz) * w[0] * w[2]) / p.J_yy;
  d[11] = (m[2] + (p.J_xx - p.J_yy) * w[0] * w[1]) / p.J_zz;
  d[12] = u_dr;
  return true;
}

}  // namespace

extern "C" int tmpc_plant_step(const tmpc_params* p, const tmpc_terrain* t, const double* control,
                               double dt, int32_t n_steps, double* state) {
  if (!p || !t || !control || !state || !(dt > 0.0) || n_steps < 0) return TMPC_ERR_CONFIG;
  char msg[8];
  if (tmpc_validate_terrain(t, msg, sizeof msg) != TMPC_OK) return TMPC_ERR_CONFIG;
  const Terr T{t};
  double s[13], k1[13], k2[13], k3[13], k4[13], tmp[13];
  std::memcpy(s, state, sizeof s);
  for (int n = 0; n < n_steps; ++n) {
    // integrate_step, Scheme::kRk4 (dynamics.hpp:454-465)
    if (!srb_derivative(*p, T, s, control[0], control[1], k1)) return TMPC_ERR_NUMERIC;
    for (int i = 0; i < 13; ++i) tmp[i] = s[i] + dt / 2 * k1[i];
    if (!srb_derivative(*p, T, tmp, control[0], control[1], k2)) return TMPC_ERR_NUMERIC;
    for (int i = 0; i < 13; ++i) tmp[i] = s[i] + dt / 2 * k2[i];
    if (!srb_derivative(*p, T, tmp, control[0], control[1], k3)) return TMPC_ERR_NUMERIC;
    for (int i = 0; i < 13; ++i) tmp[i] = s[i] + dt * k3[i];
    if (!srb_derivative(*p, T, tmp, control[0], control[1], k4)) return TMPC_ERR_NUMERIC;
    for (int i = 0; i < 13; ++i) s[i] += dt / 6.0 * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
    s[12] = std::clamp(s[12], -p->delta_max, p->delta_max);  // clamp_steering, 438-441
    for (double v : s)
      if (!std::isfinite(v)) return TMPC_ERR_NUMERIC;  // dynamics.hpp:491-492
  }
  std::memcpy(state, s, sizeof s);
  return TMPC_OK;
}
