// oracle/tmpc_oracle.cpp — CPU RESTATEMENT of the reference planning hot path.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load this library,
// and only as the checker — the product (paper_2603_20525_b200/) never links
// or calls it.
//
// Parity pinning: this restatement is checked (tests/test_oracle.py)
//   * against the reference itself, compiled from the unmodified headers in
//     oracle/_ref (ref_planner.cpp) — per-candidate cost to ~1e-12 relative;
//   * against the SPEC known-answer tests (SPEC.md:184-197,220-237,284-308,
//     374-376) and the committed golden vectors in tests/golden/.
//
// What it restates (all fp64 in variant 0, reference operation order):
//   RngStream / substream          rng.hpp:10-48
//   bilinear / height_at / gradient_at / SignedDistanceMap::value_at
//                                   terrain.hpp:35-50,79-93,235-238
//   load_transfer_coeffs            dynamics.hpp:67-71
//   tire_lateral_force              dynamics.hpp:74-77
//   rot_321 / euler_rates_321       dynamics.hpp:96-118
//   wheel_offsets                   dynamics.hpp:188-192
//   srb_derivative                  dynamics.hpp:308-398
//   integrate_step (Euler, RK4), clamp_steering   dynamics.hpp:423-468
//   esm / soft_cost_rate / constraint_set_cost / wheel_footprint
//                                   constraints.hpp:16-40,87-113
//   trajectory_cost / sample_controls / solve_ocp
//   signed_distance / build_sdist_map              terrain.hpp:186-260
//
// Variants (drift study):
//   0  fp64 everywhere, reference formulas (5 scalar bilinears per wheel)
//   1  DEVICE fp32 MODE emulation: fp32 math, fp64 storage of the whole state
//      and of the cost, padded fp32 {H,Dx,Dy} + SDF fields
//   2  fp32 math, fp32 angle/velocity state, fp64 x/y/z (rejected design)
//   3  fp32 math and fp32 state, fp64 cost only (rejected design)
//   4  op-counting run of variant 1 (ALGO_FLOPS_PER_SUBSTEP)
//   5  fp64 math and state over the fp32 fields (terrain-store error only)
//   6  DEVICE fp64 MODE emulation: fp64 math and state over fp64 padded fields
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <thread>
#include <type_traits>
#include <vector>

#include "tmpc_b200.h"

namespace orc {

constexpr double kVbxFloor = 0.1;       // dynamics.hpp:15
constexpr double kGimbalMargin = 1e-3;  // dynamics.hpp:16
constexpr double kPi = 3.14159265358979323846;

// ------------------------------------------------------------------ op counter
struct OpCount {
  uint64_t add = 0, mul = 0, div = 0, sqrt = 0, trig = 0, atan = 0, cmp = 0;
};
thread_local OpCount g_ops;

struct Cnt {  // float-valued scalar that counts arithmetic (variant 4)
  float v;
  Cnt() : v(0) {}
  Cnt(double x) : v(static_cast<float>(x)) {}
  explicit operator double() const { return v; }
};
inline Cnt operator+(Cnt a, Cnt b) { g_ops.add++; return Cnt(a.v + b.v); }
inline Cnt operator-(Cnt a, Cnt b) { g_ops.add++; return Cnt(a.v - b.v); }
inline Cnt operator-(Cnt a) { return Cnt(-a.v); }
inline Cnt operator*(Cnt a, Cnt b) { g_ops.mul++; return Cnt(a.v * b.v); }
inline Cnt operator/(Cnt a, Cnt b) { g_ops.div++; return Cnt(a.v / b.v); }
inline Cnt& operator+=(Cnt& a, Cnt b) { a = a + b; return a; }
inline bool operator<(Cnt a, Cnt b) { g_ops.cmp++; return a.v < b.v; }
inline bool operator>(Cnt a, Cnt b) { g_ops.cmp++; return a.v > b.v; }
inline bool operator<=(Cnt a, Cnt b) { g_ops.cmp++; return a.v <= b.v; }
inline bool operator>=(Cnt a, Cnt b) { g_ops.cmp++; return a.v >= b.v; }

// math dispatch
inline double m_sin(double x) { return std::sin(x); }
inline double m_cos(double x) { return std::cos(x); }
inline double m_tan(double x) { return std::tan(x); }
inline double m_atan(double x) { return std::atan(x); }
inline double m_sqrt(double x) { return std::sqrt(x); }
inline double m_abs(double x) { return std::fabs(x); }
inline double m_max(double a, double b) { return std::max(a, b); }
inline double m_min(double a, double b) { return std::min(a, b); }
inline float m_sin(float x) { return std::sin(x); }
inline float m_cos(float x) { return std::cos(x); }
inline float m_tan(float x) { return std::tan(x); }
inline float m_atan(float x) { return std::atan(x); }
inline float m_sqrt(float x) { return std::sqrt(x); }
inline float m_abs(float x) { return std::fabs(x); }
inline float m_max(float a, float b) { return std::max(a, b); }
inline float m_min(float a, float b) { return std::min(a, b); }
inline Cnt m_sin(Cnt x) { g_ops.trig++; return Cnt(std::sin(x.v)); }
inline Cnt m_cos(Cnt x) { g_ops.trig++; return Cnt(std::cos(x.v)); }
inline Cnt m_tan(Cnt x) { g_ops.trig++; return Cnt(std::tan(x.v)); }
inline Cnt m_atan(Cnt x) { g_ops.atan++; return Cnt(std::atan(x.v)); }
inline Cnt m_sqrt(Cnt x) { g_ops.sqrt++; return Cnt(std::sqrt(x.v)); }
inline Cnt m_abs(Cnt x) { return Cnt(std::fabs(x.v)); }
inline Cnt m_max(Cnt a, Cnt b) { g_ops.cmp++; return Cnt(std::max(a.v, b.v)); }
inline Cnt m_min(Cnt a, Cnt b) { g_ops.cmp++; return Cnt(std::min(a.v, b.v)); }
inline double m_asin(double x) { return std::asin(x); }
inline float m_asin(float x) { return std::asin(x); }
inline Cnt m_asin(Cnt x) { g_ops.trig++; return Cnt(std::asin(x.v)); }
inline bool m_finite(double x) { return std::isfinite(x); }
inline bool m_finite(float x) { return std::isfinite(x); }
inline bool m_finite(Cnt x) { return std::isfinite(x.v); }
template <class T> inline double dbl(T x) { return static_cast<double>(x); }

// ------------------------------------------------------------------ RNG
// RngStream::mix (rng.hpp:29-34) and substream (rng.hpp:41-48).
inline uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
inline uint64_t substream(uint64_t seed, uint64_t a, uint64_t b = 0, uint64_t c = 0) {
  uint64_t s = mix(seed);
  s = mix(s ^ (a + 0x9E3779B97F4A7C15ULL));
  s = mix(s ^ (b + 0xBF58476D1CE4E5B9ULL));
  s = mix(s ^ (c + 0x94D049BB133111EBULL));
  return s;
}
// Sequential stream (ctor rng.hpp:12, next_u64 14-17, next_double 20-22,
// uniform 25-27).
struct Stream {
  uint64_t state;
  explicit Stream(uint64_t seed) : state(mix(seed)) {}
  uint64_t next_u64() {
    state += 0x9E3779B97F4A7C15ULL;
    return mix(state);
  }
  double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * next_double(); }
};

// ------------------------------------------------------------------ params
struct Consts {
  tmpc_params p;
  double K_zzf, K_zzr, K_zx, K_zy;  // load_transfer_coeffs dynamics.hpp:67-71
  double rho[4][3];                 // wheel_offsets dynamics.hpp:188-192
  double k_i[4], b_i[4], kzz_i[4];  // dynamics.hpp:322-324
  double eps_esm;                   // esm_epsilon constraints.hpp:81-83
  int S;                            // substeps per ZOH segment
};

Consts make_consts(const tmpc_params& p) {
  Consts c;
  c.p = p;
  const double L = p.L_f + p.L_r;
  c.K_zzf = p.M * p.L_r / L;
  c.K_zzr = p.M * p.L_f / L;
  c.K_zx = p.M * (p.h + p.R) / L;
  c.K_zy = p.M * (p.h + p.R) / p.e;
  const double zo = -(p.h + p.R);
  const double rx[4] = {p.L_f, p.L_f, -p.L_r, -p.L_r};
  const double ry[4] = {p.e / 2, -p.e / 2, p.e / 2, -p.e / 2};
  for (int i = 0; i < 4; ++i) {
    c.rho[i][0] = rx[i];
    c.rho[i][1] = ry[i];
    c.rho[i][2] = zo;
    c.k_i[i] = i < 2 ? p.k_f : p.k_r;
    c.b_i[i] = i < 2 ? p.b_f : p.b_r;
    c.kzz_i[i] = i < 2 ? c.K_zzf : c.K_zzr;
  }
  c.eps_esm = p.safety_factor * p.esm_nominal;
  c.S = static_cast<int>(std::lround(p.dt_zoh / p.dt_int));
  return c;
}

// ------------------------------------------------------------------ terrain
// Reference terrain (terrain.hpp:35-50,79-93,235-238), fp64.
struct RefTerrain {
  const tmpc_terrain* t;
  double bilinear(const double* v, double x, double y) const {
    double gx = (x - t->origin_x) / t->resolution;
    double gy = (y - t->origin_y) / t->resolution;
    gx = std::clamp(gx, 0.0, static_cast<double>(t->nx - 1));
    gy = std::clamp(gy, 0.0, static_cast<double>(t->ny - 1));
    const int i0 = std::min(static_cast<int>(gx), t->nx - 2);
    const int j0 = std::min(static_cast<int>(gy), t->ny - 2);
    const double fx = gx - i0, fy = gy - j0;
    const double* r0 = v + static_cast<size_t>(j0) * t->nx + i0;
    const double* r1 = r0 + t->nx;
    const double a = r0[0] + fx * (r0[1] - r0[0]);
    const double b = r1[0] + fx * (r1[1] - r1[0]);
    return a + fy * (b - a);
  }
  template <class R>
  void height_grad(double x, double y, R& h, R& fx, R& fy) const {
    const double r = t->resolution;
    h = R(bilinear(t->heights, x, y));
    fx = R((bilinear(t->heights, x + r, y) - bilinear(t->heights, x - r, y)) / (2.0 * r));
    fy = R((bilinear(t->heights, x, y + r) - bilinear(t->heights, x, y - r)) / (2.0 * r));
  }
  template <class R>
  R sdist(double x, double y) const {
    if (!t->sdist) return R(std::numeric_limits<double>::infinity());
    return R(bilinear(t->sdist, x, y));
  }
  bool has_features() const { return t->sdist != nullptr; }
};

// Padded-field terrain (SURVEY §8a T2 identity), fields stored as float like
// the device terrain store: H' padded by 2 replicated cells per side, node
// central differences Dx=(H'[i+1]-H'[i-1])/2r, Dy likewise, SDF padded the
// same way; grid coordinates clamped to [-1, n] (== [1, n+2] padded).
template <class S>
struct FieldTerrainT {
  int nx, ny, px, py;  // original / padded sizes
  double ox, oy, res, inv_res;
  std::vector<S> H, Dx, Dy, SD;
  bool feat;
  explicit FieldTerrainT(const tmpc_terrain* t) {
    nx = t->nx;
    ny = t->ny;
    px = nx + 4;
    py = ny + 4;
    ox = t->origin_x;
    oy = t->origin_y;
    res = t->resolution;
    inv_res = 1.0 / res;
    feat = t->sdist != nullptr;
    std::vector<double> Hp(static_cast<size_t>(px) * py), Sp;
    if (feat) Sp.resize(Hp.size());
    for (int j = 0; j < py; ++j)
      for (int i = 0; i < px; ++i) {
        const int si = std::clamp(i - 2, 0, nx - 1), sj = std::clamp(j - 2, 0, ny - 1);
        Hp[static_cast<size_t>(j) * px + i] = t->heights[static_cast<size_t>(sj) * nx + si];
        if (feat) Sp[static_cast<size_t>(j) * px + i] = t->sdist[static_cast<size_t>(sj) * nx + si];
      }
    H.resize(Hp.size());
    Dx.assign(Hp.size(), S(0));
    Dy.assign(Hp.size(), S(0));
    if (feat) SD.resize(Hp.size());
    for (int j = 0; j < py; ++j)
      for (int i = 0; i < px; ++i) {
        const size_t o = static_cast<size_t>(j) * px + i;
        H[o] = static_cast<S>(Hp[o]);
        if (feat) SD[o] = static_cast<S>(Sp[o]);
        if (i >= 1 && i < px - 1) Dx[o] = static_cast<S>((Hp[o + 1] - Hp[o - 1]) / (2.0 * res));
        if (j >= 1 && j < py - 1) Dy[o] = static_cast<S>((Hp[o + px] - Hp[o - px]) / (2.0 * res));
      }
  }
  // grid coordinate in padded space, clamped to [1, n+2]; i0 <= n+2.
  template <class R>
  void coords(double x, double y, int& i0, int& j0, R& fx, R& fy) const {
    double gx = (x - ox) * inv_res + 2.0;
    double gy = (y - oy) * inv_res + 2.0;
    gx = std::clamp(gx, 1.0, static_cast<double>(nx + 2));
    gy = std::clamp(gy, 1.0, static_cast<double>(ny + 2));
    i0 = std::min(static_cast<int>(gx), nx + 2);
    j0 = std::min(static_cast<int>(gy), ny + 2);
    fx = R(gx - i0);
    fy = R(gy - j0);
  }
  template <class R>
  static R lerp2(const S* v, size_t o, int pitch, R fx, R fy) {
    const R a = R(v[o]) + fx * (R(v[o + 1]) - R(v[o]));
    const R b = R(v[o + pitch]) + fx * (R(v[o + pitch + 1]) - R(v[o + pitch]));
    return a + fy * (b - a);
  }
  template <class R>
  void height_grad(double x, double y, R& h, R& fx_, R& fy_) const {
    int i0, j0;
    R fx, fy;
    coords(x, y, i0, j0, fx, fy);
    const size_t o = static_cast<size_t>(j0) * px + i0;
    h = lerp2(H.data(), o, px, fx, fy);
    fx_ = lerp2(Dx.data(), o, px, fx, fy);
    fy_ = lerp2(Dy.data(), o, px, fx, fy);
  }
  template <class R>
  R sdist(double x, double y) const {
    if (!feat) return R(std::numeric_limits<double>::infinity());
    int i0, j0;
    R fx, fy;
    coords(x, y, i0, j0, fx, fy);
    return lerp2(SD.data(), static_cast<size_t>(j0) * px + i0, px, fx, fy);
  }
  bool has_features() const { return feat; }
};
using FieldTerrain = FieldTerrainT<float>;   // device fp32 terrain store
using FieldTerrain64 = FieldTerrainT<double>; // device fp64 terrain store

// ------------------------------------------------------------------ dynamics
// State: P for x, y, z; Q for the other 10 entries (storage types).
template <class P, class Q>
struct St {
  P x, y, z;
  Q psi, theta, phi, vbx, vby, vbz, wx, wy, wz, delta;
};
struct Deriv13 {
  double d[13];
};

// srb_derivative (dynamics.hpp:308-398) in math type R.  Returns false on the
// gimbal guard (dynamics.hpp:311-312).
template <class R, class P, class Q, class T>
bool srb_derivative(const St<P, Q>& s, R u_dr, R u_vr, const T& terr, const Consts& c,
                    R* d, double* diag = nullptr) {
  const tmpc_params& p = c.p;
  if (m_abs(dbl(s.theta)) >= kPi / 2 - kGimbalMargin) return false;
  const R psi = R(dbl(s.psi)), theta = R(dbl(s.theta)), phi = R(dbl(s.phi));
  // rot_321 (dynamics.hpp:96-105)
  const R cf = m_cos(phi), sf = m_sin(phi);
  const R ct = m_cos(theta), st = m_sin(theta);
  const R cp = m_cos(psi), sp = m_sin(psi);
  R r[3][3];
  r[0][0] = cp * ct; r[0][1] = cp * sf * st - cf * sp; r[0][2] = sf * sp + cf * cp * st;
  r[1][0] = ct * sp; r[1][1] = cf * cp + sf * sp * st; r[1][2] = cf * sp * st - cp * sf;
  r[2][0] = -st;     r[2][1] = ct * sf;                r[2][2] = cf * ct;
  // g_b = R^T (0,0,-g)  (dynamics.hpp:315)
  const R g = R(p.g);
  const R gbx = r[2][0] * (-g), gby = r[2][1] * (-g), gbz = r[2][2] * (-g);
  const R vbx = R(dbl(s.vbx)), vby = R(dbl(s.vby)), vbz = R(dbl(s.vbz));
  const R wx = R(dbl(s.wx)), wy = R(dbl(s.wy)), wz = R(dbl(s.wz));
  const R delta = R(dbl(s.delta));
  const R cd = m_cos(delta);
  R fy_sum = R(0.0), fz_sum = R(0.0);
  R mx = R(0.0), my = R(0.0), mz = R(0.0);
  // rear-axle constraining force (dynamics.hpp:330-331)
  const R f_x_rear = R(0.5) * R(p.M) * (u_vr - gbx + wy * vbz - wz * vby);
  for (int i = 0; i < 4; ++i) {
    const bool front = i < 2;
    const R rx = R(c.rho[i][0]), ry = R(c.rho[i][1]), rz = R(c.rho[i][2]);
    // p_w = pos + R rho (dynamics.hpp:335)
    const R rwx = r[0][0] * rx + r[0][1] * ry + r[0][2] * rz;
    const R rwy = r[1][0] * rx + r[1][1] * ry + r[1][2] * rz;
    const R rwz = r[2][0] * rx + r[2][1] * ry + r[2][2] * rz;
    const double pwx = dbl(s.x) + dbl(rwx), pwy = dbl(s.y) + dbl(rwy);
    const double pwz = dbl(s.z) + dbl(rwz);
    // v_i = v + omega x rho (dynamics.hpp:336)
    const R vix = vbx + (wy * rz - wz * ry);
    const R viy = vby + (wz * rx - wx * rz);
    const R viz = vbz + (wx * ry - wy * rx);
    // terrain plane (dynamics.hpp:338-341)
    R h, sfx, sfy;
    terr.height_grad(pwx, pwy, h, sfx, sfy);
    const R twx = -sfx, twy = -sfy, twz = R(1.0);
    const R tbx = r[0][0] * twx + r[1][0] * twy + r[2][0] * twz;
    const R tby = r[0][1] * twx + r[1][1] * twy + r[2][1] * twz;
    const R tbz_raw = r[0][2] * twx + r[1][2] * twy + r[2][2] * twz;
    const R tbz = m_max(tbz_raw, R(1e-6));
    // extension and rate (dynamics.hpp:343-346); omega x z = (wy, -wx, 0)
    const R chi = R(pwz - dbl(h)) / tbz;
    const R ax = vix - chi * wy, ay = viy - chi * (-wx), az = viz - chi * R(0.0);
    const R chi_dot = (tbx * ax + tby * ay + tbz_raw * az) / tbz;
    // suspension forces (dynamics.hpp:348-351)
    const R f_s = R(0.5) * g * R(c.kzz_i[i]);
    const R f_k = m_max(f_s - R(c.k_i[i]) * chi, R(0.0));
    const R f_b = f_k > R(0.0) ? m_max(-R(c.b_i[i]) * chi_dot, -f_k) : R(0.0);
    const R f_z = f_k + f_b;
    // slip and lateral force (dynamics.hpp:353-356, tire 74-77)
    const R delta_i = front ? delta : R(0.0);
    const R alpha = m_atan(viy / m_max(vix, R(kVbxFloor))) - delta_i;
    const R ca = R(p.C) * alpha;
    const R f_y = f_z * (-ca * R(p.mu)) / m_sqrt(R(p.mu) * R(p.mu) + ca * ca);
    // sums and moment rho x F (dynamics.hpp:358-362)
    const R cos_di = front ? cd : R(1.0);
    fy_sum += f_y * cos_di;
    fz_sum += f_z;
    const R Fx = front ? R(0.0) : f_x_rear, Fy = f_y * cos_di, Fz = f_z;
    mx += ry * Fz - rz * Fy;
    my += rz * Fx - rx * Fz;
    mz += rx * Fy - ry * Fx;
    if (diag) {
      diag[i] = dbl(chi);
      diag[4 + i] = dbl(chi_dot);
      diag[8 + i] = dbl(f_z);
      diag[12 + i] = dbl(f_y);
      diag[16 + i] = dbl(alpha);
    }
  }
  if (diag) {
    diag[20] = dbl(gbx);
    diag[21] = dbl(gby);
    diag[22] = dbl(gbz);
  }
  // euler_rates_321 (dynamics.hpp:109-118)
  const R tt = m_tan(theta);
  const R er_psi = (sf * wy + cf * wz) / ct;
  const R er_theta = cf * wy - sf * wz;
  const R er_phi = wx + sf * tt * wy + cf * tt * wz;
  // v_w = R v_b (dynamics.hpp:374)
  d[0] = r[0][0] * vbx + r[0][1] * vby + r[0][2] * vbz;
  d[1] = r[1][0] * vbx + r[1][1] * vby + r[1][2] * vbz;
  d[2] = r[2][0] * vbx + r[2][1] * vby + r[2][2] * vbz;
  d[3] = er_psi;
  d[4] = er_theta;
  d[5] = er_phi;
  d[6] = u_vr;
  const R M = R(p.M);
  d[7] = fy_sum / M + gby + wx * vbz - wz * vbx;
  d[8] = fz_sum / M + gbz - wx * vby + wy * vbx;
  d[9] = (mx + (R(p.J_yy) - R(p.J_zz)) * wy * wz) / R(p.J_xx);
  d[10] = (my - (R(p.J_xx) - R(p.J_zz)) * wx * wz) / R(p.J_yy);
  d[11] = (mz + (R(p.J_xx) - R(p.J_yy)) * wx * wy) / R(p.J_zz);
  d[12] = u_dr;
  return true;
}

// Euler step + clamp_steering (dynamics.hpp:423-441,446-453,466).
template <class R, class P, class Q>
void euler_update(St<P, Q>& s, const R* d, double dt, const Consts& c) {
  const R h = R(dt);
  auto upd_p = [&](P& v, R dv) { v = P(dbl(v) + dbl(h * dv)); };
  auto upd_q = [&](Q& v, R dv) {
    if constexpr (std::is_same_v<Q, double>) v = dbl(v) + dt * dbl(dv);
    else v = Q(dbl(R(dbl(v)) + h * dv));
  };
  if constexpr (std::is_same_v<P, double>) {
    s.x = s.x + dt * dbl(d[0]);
    s.y = s.y + dt * dbl(d[1]);
    s.z = s.z + dt * dbl(d[2]);
  } else {
    upd_p(s.x, d[0]);
    upd_p(s.y, d[1]);
    upd_p(s.z, d[2]);
  }
  upd_q(s.psi, d[3]);
  upd_q(s.theta, d[4]);
  upd_q(s.phi, d[5]);
  upd_q(s.vbx, d[6]);
  upd_q(s.vby, d[7]);
  upd_q(s.vbz, d[8]);
  upd_q(s.wx, d[9]);
  upd_q(s.wy, d[10]);
  upd_q(s.wz, d[11]);
  upd_q(s.delta, d[12]);
  const double dm = c.p.delta_max;
  s.delta = Q(std::clamp(dbl(s.delta), -dm, dm));
}

// integrate_step, Scheme::kRk4 (dynamics.hpp:454-466): four srb_derivative
// evaluations in R at stage states s + (dt/2) k1, s + (dt/2) k2, s + dt k3
// formed in fp64, combined as s + dt/6 (k1 + 2 k2 + 2 k3 + k4) in fp64, then
// clamp_steering.  The gimbal guard of any stage diverges the candidate
// (the reference's std::domain_error propagates out of integrate_step).
template <class P, class Q>
void st_to_arr(const St<P, Q>& s, double* a) {
  const double v[13] = {dbl(s.x),   dbl(s.y),   dbl(s.z),   dbl(s.psi), dbl(s.theta),
                        dbl(s.phi), dbl(s.vbx), dbl(s.vby), dbl(s.vbz), dbl(s.wx),
                        dbl(s.wy),  dbl(s.wz),  dbl(s.delta)};
  for (int i = 0; i < 13; ++i) a[i] = v[i];
}
template <class P, class Q>
St<P, Q> st_from_arr(const double* a) {
  St<P, Q> s;
  s.x = P(a[0]); s.y = P(a[1]); s.z = P(a[2]);
  s.psi = Q(a[3]); s.theta = Q(a[4]); s.phi = Q(a[5]);
  s.vbx = Q(a[6]); s.vby = Q(a[7]); s.vbz = Q(a[8]);
  s.wx = Q(a[9]); s.wy = Q(a[10]); s.wz = Q(a[11]); s.delta = Q(a[12]);
  return s;
}
template <class R, class P, class Q, class T>
bool rk4_update(St<P, Q>& s, R u_dr, R u_vr, const T& terr, const Consts& c, double dt) {
  double a[13], tmp[13], k[4][13];
  st_to_arr(s, a);
  const double frac[3] = {dt / 2, dt / 2, dt};
  for (int stage = 0; stage < 4; ++stage) {
    R d[13];
    const double* src = a;
    if (stage > 0) {
      for (int i = 0; i < 13; ++i) tmp[i] = a[i] + frac[stage - 1] * k[stage - 1][i];
      src = tmp;
    }
    if (!srb_derivative<R>(st_from_arr<P, Q>(src), u_dr, u_vr, terr, c, d)) return false;
    for (int i = 0; i < 13; ++i) k[stage][i] = dbl(d[i]);
  }
  for (int i = 0; i < 13; ++i)
    a[i] += dt / 6.0 * (k[0][i] + 2.0 * k[1][i] + 2.0 * k[2][i] + k[3][i]);
  a[12] = std::clamp(a[12], -c.p.delta_max, c.p.delta_max);
  s = st_from_arr<P, Q>(a);
  return true;
}

template <class P, class Q>
bool all_finite(const St<P, Q>& s) {
  return m_finite(s.x) && m_finite(s.y) && m_finite(s.z) && m_finite(s.psi) &&
         m_finite(s.theta) && m_finite(s.phi) && m_finite(s.vbx) && m_finite(s.vby) &&
         m_finite(s.vbz) && m_finite(s.wx) && m_finite(s.wy) && m_finite(s.wz) &&
         m_finite(s.delta);
}

// ------------------------------------------------------------------ constraints
// esm (constraints.hpp:16-23)
template <class R>
R esm(R phi, R theta, const tmpc_params& p) {
  const R r_bar = R(std::hypot(p.h + p.R, p.e / 2.0));
  const R phi_bar = R(std::atan(2.0 * (p.h + p.R) / p.e));
  const R lever = m_abs(phi) + phi_bar;
  const R dh = r_bar * (R(1.0) - m_sin(lever)) * m_cos(theta);
  const R sign = lever <= R(kPi / 2.0) ? R(1.0) : R(-1.0);
  return sign * R(p.M) * R(p.g) * dh;
}
// soft_cost_rate (constraints.hpp:37-40)
template <class R>
R soft_cost_rate(R pi, R eps, R sigma) {
  const R a = m_max(R(0.0), R(1.0) + pi / eps);
  return sigma * a * a;
}

// ------------------------------------------------------------------ sampler
// sample_controls with the BASELINE extensions; random
// access draw j of stream s_k = mix(mix(s_k) + (j+1) * golden) (rng.hpp:12-17).
void sample_controls(const tmpc_params& p, const tmpc_sampling& s, int64_t k, double* out) {
  const int nch = s.vdot_max > 0.0 ? 2 : 1;
  const double bound[2] = {p.delta_rate_max, s.vdot_max};
  Stream rng(substream(s.seed, static_cast<uint64_t>(k)));
  double prev[2] = {0.0, 0.0};
  for (int t = 0; t < p.n_steps; ++t) {
    double v[2] = {0.0, 0.0};
    for (int ch = 0; ch < nch; ++ch) {
      const double b = bound[ch];
      if (s.kind == TMPC_SAMPLE_UNIFORM) {
        v[ch] = rng.uniform(-b, b);
      } else if (s.kind == TMPC_SAMPLE_RANDOM_WALK) {
        const double a = ch == 0 ? s.walk_step : s.walk_step * s.vdot_max / p.delta_rate_max;
        v[ch] = std::clamp(prev[ch] + rng.uniform(-a, a), -b, b);
        prev[ch] = v[ch];
      } else {
        const double u1 = rng.next_double();
        const double u2 = rng.next_double();
        const double base = s.warm_seq ? s.warm_seq[2 * t + ch] : 0.0;
        const double z = std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(2.0 * kPi * u2);
        const double sigma = s.warm_sigma_frac * 2.0 * b;
        v[ch] = std::clamp(k == 0 ? base : base + sigma * z, -b, b);
      }
    }
    out[2 * t] = v[0];
    out[2 * t + 1] = v[1];
  }
}

// ------------------------------------------------------------------ rollout
struct CandOut {
  double cost;
  uint8_t flags;
  float margin;
  int64_t substeps;
};

// trajectory_cost for one candidate: goal test before
// accumulating, rectangle rule on the dt_int grid, soft
// constraints via constraint_set_cost (constraints.hpp:87-100), divergence ->
// +inf, terminal cost w_g |p - p_g|.
template <class R, class P, class Q, class T>
CandOut rollout(const Consts& c, const T& terr, const double* s0, const double* u) {
  const tmpc_params& p = c.p;
  St<P, Q> s;
  s.x = P(s0[0]); s.y = P(s0[1]); s.z = P(s0[2]);
  s.psi = Q(s0[3]); s.theta = Q(s0[4]); s.phi = Q(s0[5]);
  s.vbx = Q(s0[6]); s.vby = Q(s0[7]); s.vbz = Q(s0[8]);
  s.wx = Q(s0[9]); s.wy = Q(s0[10]); s.wz = Q(s0[11]); s.delta = Q(s0[12]);
  const double inf = std::numeric_limits<double>::infinity();
  double J = 0.0, margin = inf;
  bool feasible = true, diverged = false, goal = false;
  int64_t n = 0;
  const bool use_dist = p.enable_dist && terr.has_features();
  for (int t = 0; t < p.n_steps && !goal && !diverged; ++t) {
    const R u_dr = R(u[2 * t]), u_vr = R(u[2 * t + 1]);
    for (int q = 0; q < c.S; ++q) {
      const double dx = dbl(s.x) - p.goal_x, dy = dbl(s.y) - p.goal_y;
      if (dx * dx + dy * dy <= p.goal_r * p.goal_r) {
        goal = true;
        break;
      }
      // L_soft (constraints.hpp:87-100): wheel_footprint (104-113) + SDF
      R rate = R(0.0);
      const R psi = R(dbl(s.psi));
      const R cps = m_cos(psi), sps = m_sin(psi);
      if (use_dist) {
        for (int i = 0; i < 4; ++i) {
          const double wxp = dbl(s.x) + dbl(cps * R(c.rho[i][0]) - sps * R(c.rho[i][1]));
          const double wyp = dbl(s.y) + dbl(sps * R(c.rho[i][0]) + cps * R(c.rho[i][1]));
          const R sd = terr.template sdist<R>(wxp, wyp);
          if (!std::isinf(dbl(sd))) rate += soft_cost_rate(-sd, R(p.eps_dist), R(p.sigma));
          if (!(dbl(sd) > 0.0)) feasible = false;
          margin = std::min(margin, dbl(sd) / p.eps_dist);
        }
      }
      const R U = esm(R(dbl(s.phi)), R(dbl(s.theta)), p);
      if (p.enable_rollover) {
        if (m_finite(-U)) rate += soft_cost_rate(-U, R(c.eps_esm), R(p.sigma));
        if (!(dbl(U) > 0.0)) feasible = false;
        margin = std::min(margin, dbl(U) / p.esm_nominal);
      }
      const double L = p.w_t + p.w_c * u[2 * t] * u[2 * t] + dbl(rate);
      J += p.dt_int * L;
      if (p.scheme == TMPC_SCHEME_RK4) {
        if (!rk4_update<R>(s, u_dr, u_vr, terr, c, p.dt_int)) {
          diverged = true;
          break;
        }
      } else {
        R d[13];
        if (!srb_derivative<R>(s, u_dr, u_vr, terr, c, d)) {
          diverged = true;
          break;
        }
        euler_update<R>(s, d, p.dt_int, c);
      }
      ++n;
      if (!all_finite(s)) {
        diverged = true;
        break;
      }
    }
  }
  CandOut o;
  o.substeps = n;
  if (diverged) {
    o.cost = inf;
    o.flags = TMPC_FLAG_DIVERGED;
    o.margin = -std::numeric_limits<float>::infinity();
    return o;
  }
  const double dx = dbl(s.x) - p.goal_x, dy = dbl(s.y) - p.goal_y;
  o.cost = J + p.w_g * std::sqrt(dx * dx + dy * dy);
  o.flags = static_cast<uint8_t>((feasible ? TMPC_FLAG_FEASIBLE : 0) | (goal ? TMPC_FLAG_GOAL : 0));
  o.margin = static_cast<float>(margin);
  return o;
}

// ------------------------------------------------------------------ EST model
// est_plane_attitude (dynamics.hpp:213-219) + est_derivative (230-275) in the
// math type R; writes d[7] in EstState order and the diagnostics g_by, a_by.
template <class R, class T>
void est_derivative(const double* s7, R u_dr, R u_vr, const T& terr, const Consts& c, R* d,
                    R& g_by, R& a_by) {
  const tmpc_params& p = c.p;
  // normal_at (terrain.hpp:97-100): normalize(-fx, -fy, 1)
  R h, fx, fy;
  terr.height_grad(s7[0], s7[1], h, fx, fy);
  const R nrm = m_sqrt(fx * fx + fy * fy + R(1.0));
  const R tx = -fx / nrm, ty = -fy / nrm;
  const R theta = m_asin(m_min(m_max(tx, R(-1.0)), R(1.0)));
  const R ct0 = m_cos(theta);
  const R sphi = m_min(m_max(-ty / m_max(ct0, R(1e-9)), R(-1.0)), R(1.0));
  const R phi = m_asin(sphi);
  // rot_123 (dynamics.hpp:84-93)
  const R psi = R(s7[2]);
  const R cf = m_cos(phi), sf = m_sin(phi), ct = m_cos(theta), st = m_sin(theta);
  const R cp = m_cos(psi), sp = m_sin(psi);
  const R r00 = ct * cp, r01 = -ct * sp;
  const R r10 = cf * sp + cp * sf * st, r11 = cf * cp - sf * st * sp;
  const R r20 = sf * sp - cf * cp * st, r21 = cp * sf + cf * st * sp, r22 = cf * ct;
  const R g = R(p.g);
  const R gbx = r20 * (-g);
  g_by = r21 * (-g);
  const R gbz = r22 * (-g);
  (void)gbx;
  const R vbx = R(s7[6]), vby = R(s7[3]), wz = R(s7[4]), delta = R(s7[5]);
  const R vbx_eff = m_max(vbx, R(kVbxFloor));
  const R alpha_f = m_atan((vby + wz * R(p.L_f)) / vbx_eff) - delta;
  const R alpha_r = m_atan((vby - wz * R(p.L_r)) / vbx_eff);
  const R a_bx = u_vr - wz * vby;
  const R f_zf = m_max(-R(c.K_zzf) * gbz - R(c.K_zx) * a_bx, R(0.0));
  const R f_zr = m_max(-R(c.K_zzr) * gbz + R(c.K_zx) * a_bx, R(0.0));
  const R mu = R(p.mu);
  const R caf = R(p.C) * alpha_f, car = R(p.C) * alpha_r;
  const R f_yf = f_zf * (-caf * mu) / m_sqrt(mu * mu + caf * caf);
  const R f_yr = f_zr * (-car * mu) / m_sqrt(mu * mu + car * car);
  d[0] = r00 * vbx + r01 * vby;  // v_w = r (v_bx, v_by, 0)
  d[1] = r10 * vbx + r11 * vby;
  d[2] = wz;
  d[3] = (f_yf + f_yr) / R(p.M) + g_by - wz * vbx;
  d[4] = (f_yf * R(p.L_f) * m_cos(delta) - f_yr * R(p.L_r)) / R(p.J_zz);
  d[5] = u_dr;
  d[6] = u_vr;
  a_by = d[3] + wz * vbx;  // EstDiagnostics::a_by (dynamics.hpp:265)
}

// trajectory_cost for the EST formulation: the lateral-acceleration rollover
// constraint (constraints.hpp:62-65; eps = safety_factor * a_by_bar, 78-80)
// replaces the ESM; margin normalised by a_by_bar.  State in the SrbState
// slots (x, y, psi, v_by, omega_bz, delta, v_bx) of s0 (13 entries).
template <class R, class T>
CandOut rollout_est(const Consts& c, const T& terr, const double* s0, const double* u) {
  const tmpc_params& p = c.p;
  double s[7] = {s0[0], s0[1], s0[3], s0[7], s0[11], s0[12], s0[6]};
  const double inf = std::numeric_limits<double>::infinity();
  double J = 0.0, margin = inf;
  bool feasible = true, diverged = false, goal = false;
  int64_t n = 0;
  const bool use_dist = p.enable_dist && terr.has_features();
  const R eps_aby = R(p.safety_factor * p.a_by_bar);
  for (int t = 0; t < p.n_steps && !goal && !diverged; ++t) {
    const R u_dr = R(u[2 * t]), u_vr = R(u[2 * t + 1]);
    for (int q = 0; q < c.S; ++q) {
      const double dx = s[0] - p.goal_x, dy = s[1] - p.goal_y;
      if (dx * dx + dy * dy <= p.goal_r * p.goal_r) {
        goal = true;
        break;
      }
      R d[7], g_by, a_by;
      est_derivative<R>(s, u_dr, u_vr, terr, c, d, g_by, a_by);
      R rate = R(0.0);
      const R psi = R(s[2]);
      const R cps = m_cos(psi), sps = m_sin(psi);
      if (use_dist) {
        for (int i = 0; i < 4; ++i) {
          const double wxp = s[0] + dbl(cps * R(c.rho[i][0]) - sps * R(c.rho[i][1]));
          const double wyp = s[1] + dbl(sps * R(c.rho[i][0]) + cps * R(c.rho[i][1]));
          const R sd = terr.template sdist<R>(wxp, wyp);
          if (!std::isinf(dbl(sd))) rate += soft_cost_rate(-sd, R(p.eps_dist), R(p.sigma));
          if (!(dbl(sd) > 0.0)) feasible = false;
          margin = std::min(margin, dbl(sd) / p.eps_dist);
        }
      }
      const R pi_aby = m_abs(a_by - g_by) - R(p.a_by_bar);
      if (p.enable_rollover) {
        rate += soft_cost_rate(pi_aby, eps_aby, R(p.sigma));
        if (!(dbl(pi_aby) < 0.0)) feasible = false;
        margin = std::min(margin, -dbl(pi_aby) / p.a_by_bar);
      }
      J += p.dt_int * (p.w_t + p.w_c * u[2 * t] * u[2 * t] + dbl(rate));
      if (p.scheme == TMPC_SCHEME_RK4) {
        // integrate_step Scheme::kRk4 over EstModel (dynamics.hpp:454-466);
        // k1 is the derivative the cost diagnostics came from.
        double k[4][7], tmp[7];
        for (int i = 0; i < 7; ++i) k[0][i] = dbl(d[i]);
        const double frac[3] = {p.dt_int / 2, p.dt_int / 2, p.dt_int};
        for (int stage = 1; stage < 4; ++stage) {
          for (int i = 0; i < 7; ++i) tmp[i] = s[i] + frac[stage - 1] * k[stage - 1][i];
          R ds[7], gb, ab;
          est_derivative<R>(tmp, u_dr, u_vr, terr, c, ds, gb, ab);
          for (int i = 0; i < 7; ++i) k[stage][i] = dbl(ds[i]);
        }
        for (int i = 0; i < 7; ++i)
          s[i] += p.dt_int / 6.0 * (k[0][i] + 2.0 * k[1][i] + 2.0 * k[2][i] + k[3][i]);
      } else {
        for (int i = 0; i < 7; ++i) s[i] += p.dt_int * dbl(d[i]);
      }
      s[5] = std::clamp(s[5], -p.delta_max, p.delta_max);
      ++n;
      bool fin = true;
      for (double v : s) fin = fin && std::isfinite(v);
      if (!fin) {
        diverged = true;
        break;
      }
    }
  }
  CandOut o;
  o.substeps = n;
  if (diverged) {
    o.cost = inf;
    o.flags = TMPC_FLAG_DIVERGED;
    o.margin = -std::numeric_limits<float>::infinity();
    return o;
  }
  const double dx = s[0] - p.goal_x, dy = s[1] - p.goal_y;
  o.cost = J + p.w_g * std::sqrt(dx * dx + dy * dy);
  o.flags = static_cast<uint8_t>((feasible ? TMPC_FLAG_FEASIBLE : 0) | (goal ? TMPC_FLAG_GOAL : 0));
  o.margin = static_cast<float>(margin);
  return o;
}

// ------------------------------------------------------------------ geometry
// point_segment_distance / point_in_polygon / signed_distance
// (terrain.hpp:186-224).
double point_segment_distance(double px, double py, double ax, double ay, double bx, double by) {
  const double abx = bx - ax, aby = by - ay;
  const double len2 = abx * abx + aby * aby;
  if (len2 == 0.0) return std::sqrt((px - ax) * (px - ax) + (py - ay) * (py - ay));
  const double t = std::clamp(((px - ax) * abx + (py - ay) * aby) / len2, 0.0, 1.0);
  const double qx = px - (ax + t * abx), qy = py - (ay + t * aby);
  return std::sqrt(qx * qx + qy * qy);
}
double signed_distance(double px, double py, const double* v, int n, int kind) {
  double d = std::numeric_limits<double>::infinity();
  for (int i = 0; i < n; ++i) {
    const int j = (i + 1) % n;
    d = std::min(d, point_segment_distance(px, py, v[2 * i], v[2 * i + 1], v[2 * j], v[2 * j + 1]));
  }
  bool inside = false;
  for (int i = 0, j = n - 1; i < n; j = i++) {
    const double yi = v[2 * i + 1], yj = v[2 * j + 1], xi = v[2 * i], xj = v[2 * j];
    if ((yi > py) != (yj > py)) {
      const double x_at = xj + (py - yj) / (yi - yj) * (xi - xj);
      if (px < x_at) inside = !inside;
    }
  }
  const bool violating = kind == 0 ? inside : !inside;
  return violating ? -d : d;
}

}  // namespace orc

extern "C" {

using namespace orc;

int oracle_sample_controls(const tmpc_params* p, const tmpc_sampling* smp, int64_t k, double* out) {
  sample_controls(*p, *smp, k, out);
  return 0;
}

// solve_ocp: every candidate of the shard, then the arg-min
// (feasible-first or plain, lowest index on ties).
int oracle_solve(const tmpc_params* p, const tmpc_sampling* smp, const tmpc_terrain* t,
                 const double* s0, double* cost, uint8_t* flags, float* margin,
                 int64_t* substeps, int n_threads, int variant, tmpc_result* res, char* err,
                 size_t err_len) {
  const Consts c = make_consts(*p);
  if (c.S < 1 || std::fabs(c.S * p->dt_int - p->dt_zoh) > 1e-9) {
    std::snprintf(err, err_len, "integrate: dt_int must divide the ZOH period");
    return 2;
  }
  const RefTerrain rt{t};
  const FieldTerrain* ft = variant == 0 ? nullptr : new FieldTerrain(t);
  const FieldTerrain64* ft64 = variant == 6 ? new FieldTerrain64(t) : nullptr;
  const int64_t K = smp->k_count;
  std::atomic<int64_t> next{0};
  std::atomic<uint64_t> ops[7] = {};
  auto worker = [&]() {
    std::vector<double> u(2 * static_cast<size_t>(p->n_steps));
    g_ops = OpCount{};
    for (;;) {
      const int64_t i0 = next.fetch_add(8);
      if (i0 >= K) break;
      for (int64_t i = i0; i < std::min<int64_t>(K, i0 + 8); ++i) {
        sample_controls(*p, *smp, smp->k_begin + i, u.data());
        CandOut o;
        if (p->model == TMPC_MODEL_EST) {
          switch (variant) {
            case 0: o = rollout_est<double>(c, rt, s0, u.data()); break;
            case 6: o = rollout_est<double>(c, *ft64, s0, u.data()); break;
            case 4: o = rollout_est<Cnt>(c, *ft, s0, u.data()); break;
            default: o = rollout_est<float>(c, *ft, s0, u.data()); break;
          }
        } else switch (variant) {
          case 0: o = rollout<double, double, double>(c, rt, s0, u.data()); break;
          case 1: o = rollout<float, double, double>(c, *ft, s0, u.data()); break;
          case 2: o = rollout<float, double, float>(c, *ft, s0, u.data()); break;
          case 3: o = rollout<float, float, float>(c, *ft, s0, u.data()); break;
          case 5: o = rollout<double, double, double>(c, *ft, s0, u.data()); break;
          case 6: o = rollout<double, double, double>(c, *ft64, s0, u.data()); break;
          default: o = rollout<Cnt, double, double>(c, *ft, s0, u.data()); break;
        }
        if (cost) cost[i] = o.cost;
        if (flags) flags[i] = o.flags;
        if (margin) margin[i] = o.margin;
        if (substeps) substeps[i] = o.substeps;
      }
    }
    ops[0] += g_ops.add; ops[1] += g_ops.mul; ops[2] += g_ops.div; ops[3] += g_ops.sqrt;
    ops[4] += g_ops.trig; ops[5] += g_ops.atan; ops[6] += g_ops.cmp;
  };
  const int nt = std::max(1, n_threads);
  std::vector<std::thread> th;
  for (int i = 1; i < nt; ++i) th.emplace_back(worker);
  worker();
  for (auto& x : th) x.join();
  delete ft;
  delete ft64;
  if (variant == 4 && res) {  // op counts smuggled out through the result
    std::memset(res, 0, sizeof(*res));
    res->n_candidates = static_cast<int64_t>(ops[0]);  // adds
    res->n_feasible = static_cast<int64_t>(ops[1]);    // muls
    res->n_diverged = static_cast<int64_t>(ops[2]);    // divs
    res->n_goal = static_cast<int64_t>(ops[3]);        // sqrt
    res->best_index = static_cast<int64_t>(ops[4]);    // sin/cos/tan
    res->substeps_executed = static_cast<int64_t>(ops[5]);  // atan
    res->best_cost = static_cast<double>(ops[6]);      // compares/max/min
    return 0;
  }
  if (res && cost && flags) {
    std::memset(res, 0, sizeof(*res));
    const bool ff = p->selection == TMPC_SELECT_FEASIBLE_FIRST;
    int64_t best = 0;
    double sum = 0.0, mn = std::numeric_limits<double>::infinity();
    int64_t nfin = 0;
    for (int64_t i = 0; i < K; ++i) {
      if (flags[i] & TMPC_FLAG_FEASIBLE) res->n_feasible++;
      if (flags[i] & TMPC_FLAG_DIVERGED) res->n_diverged++;
      if (flags[i] & TMPC_FLAG_GOAL) res->n_goal++;
      if (std::isfinite(cost[i])) {
        sum += cost[i];
        ++nfin;
        mn = std::min(mn, cost[i]);
      }
      const bool inf_i = ff && !(flags[i] & TMPC_FLAG_FEASIBLE);
      const bool inf_b = ff && !(flags[best] & TMPC_FLAG_FEASIBLE);
      if (inf_i < inf_b || (inf_i == inf_b && cost[i] < cost[best])) best = i;
    }
    res->n_candidates = K;
    res->best_index = smp->k_begin + best;
    res->best_cost = cost[best];
    res->best_feasible = (flags[best] & TMPC_FLAG_FEASIBLE) ? 1 : 0;
    res->best_margin = margin ? margin[best] : 0.0f;
    res->min_cost = mn;
    res->mean_cost = nfin ? sum / nfin : std::numeric_limits<double>::infinity();
    if (substeps)
      for (int64_t i = 0; i < K; ++i) res->substeps_executed += substeps[i];
    if (res->n_diverged == K) {
      std::snprintf(err, err_len, "solve_ocp: all %lld rollouts diverged", (long long)K);
      return 1;
    }
  }
  return 0;
}

// srb_derivative restated (variant 0 = fp64 reference terrain, 1 = fp32 fields).
int oracle_srb_derivative(const tmpc_params* p, const tmpc_terrain* t, const double* s13,
                          const double* u2, int variant, double* d13, double* diag) {
  const Consts c = make_consts(*p);
  St<double, double> s{s13[0], s13[1], s13[2], s13[3], s13[4], s13[5], s13[6],
                       s13[7], s13[8], s13[9], s13[10], s13[11], s13[12]};
  if (variant == 0) {
    const RefTerrain rt{t};
    double d[13];
    if (!srb_derivative<double>(s, u2[0], u2[1], rt, c, d, diag)) return 1;
    for (int i = 0; i < 13; ++i) d13[i] = d[i];
  } else {
    const FieldTerrain ft(t);
    float d[13];
    if (!srb_derivative<float>(s, static_cast<float>(u2[0]), static_cast<float>(u2[1]), ft, c, d, diag))
      return 1;
    for (int i = 0; i < 13; ++i) d13[i] = d[i];
  }
  return 0;
}

// Restated RK4 / Euler step (dynamics.hpp:446-468), fp64 reference terrain.
int oracle_integrate_step(const tmpc_params* p, const tmpc_terrain* t, const double* s13,
                          const double* u2, double dt, int scheme, double* out13) {
  const Consts c = make_consts(*p);
  const RefTerrain rt{t};
  using S = St<double, double>;
  auto to = [](const double* a) { return S{a[0], a[1], a[2], a[3], a[4], a[5], a[6], a[7], a[8], a[9], a[10], a[11], a[12]}; };
  auto arr = [](const S& s, double* a) {
    const double v[13] = {s.x, s.y, s.z, s.psi, s.theta, s.phi, s.vbx, s.vby, s.vbz, s.wx, s.wy, s.wz, s.delta};
    for (int i = 0; i < 13; ++i) a[i] = v[i];
  };
  double a[13];
  for (int i = 0; i < 13; ++i) a[i] = s13[i];
  if (scheme == 0) {
    double d[13];
    if (!srb_derivative<double>(to(a), u2[0], u2[1], rt, c, d)) return 1;
    for (int i = 0; i < 13; ++i) a[i] += dt * d[i];
  } else {
    double k1[13], k2[13], k3[13], k4[13], tmp[13];
    if (!srb_derivative<double>(to(a), u2[0], u2[1], rt, c, k1)) return 1;
    for (int i = 0; i < 13; ++i) tmp[i] = a[i] + dt / 2 * k1[i];
    if (!srb_derivative<double>(to(tmp), u2[0], u2[1], rt, c, k2)) return 1;
    for (int i = 0; i < 13; ++i) tmp[i] = a[i] + dt / 2 * k2[i];
    if (!srb_derivative<double>(to(tmp), u2[0], u2[1], rt, c, k3)) return 1;
    for (int i = 0; i < 13; ++i) tmp[i] = a[i] + dt * k3[i];
    if (!srb_derivative<double>(to(tmp), u2[0], u2[1], rt, c, k4)) return 1;
    for (int i = 0; i < 13; ++i) a[i] += dt / 6.0 * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
  }
  a[12] = std::clamp(a[12], -p->delta_max, p->delta_max);
  (void)arr;
  for (int i = 0; i < 13; ++i) out13[i] = a[i];
  return 0;
}

// Terrain queries: variant 0 reference formulas (fp64), 1 padded float fields.
int oracle_terrain_query(const tmpc_terrain* t, const double* xy, int64_t n, int variant,
                         double* out) {
  const RefTerrain rt{t};
  const FieldTerrain* ft = variant ? new FieldTerrain(t) : nullptr;
  for (int64_t i = 0; i < n; ++i) {
    const double x = xy[2 * i], y = xy[2 * i + 1];
    if (variant) {
      float h, fx, fy;
      ft->height_grad(x, y, h, fx, fy);
      out[4 * i] = h; out[4 * i + 1] = fx; out[4 * i + 2] = fy;
      out[4 * i + 3] = ft->sdist<float>(x, y);
    } else {
      double h, fx, fy;
      rt.height_grad(x, y, h, fx, fy);
      out[4 * i] = h; out[4 * i + 1] = fx; out[4 * i + 2] = fy;
      out[4 * i + 3] = rt.sdist<double>(x, y);
    }
  }
  delete ft;
  return 0;
}

// build_sdist_map (terrain.hpp:241-260) restated, brute force.
int oracle_build_sdist_map(int nx, int ny, double ox, double oy, double res, int n_poly,
                           const int* poly_off, const double* verts, const int* kinds,
                           double* out) {
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const double x = ox + res * i, y = oy + res * j;
      double d = std::numeric_limits<double>::infinity();
      for (int k = 0; k < n_poly; ++k)
        d = std::min(d, signed_distance(x, y, verts + 2 * poly_off[k], poly_off[k + 1] - poly_off[k], kinds[k]));
      out[static_cast<size_t>(j) * nx + i] = d;
    }
  return 0;
}

double oracle_esm(const tmpc_params* p, double phi, double theta) { return esm<double>(phi, theta, *p); }
uint64_t oracle_substream(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) { return substream(seed, a, b, c); }
uint64_t oracle_rng_draw(uint64_t stream_seed, int64_t j) {
  // random-access form of draw j of RngStream(stream_seed)
  return mix(mix(stream_seed) + static_cast<uint64_t>(j + 1) * 0x9E3779B97F4A7C15ULL);
}

}  // extern "C"
