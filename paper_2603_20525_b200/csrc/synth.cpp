// Workload setup on the host: synthetic heightmaps, seeded cylinder
// obstacles and the signed-distance map (terrain preprocessing, once per
// terrain — SURVEY §3.3, App. A D4-D5).  Not on the per-cycle hot path.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <thread>
#include <vector>

#include "tmpc_b200.h"
#include "tmpc_common.h"

namespace {

using tmpcb::mix64;
using tmpcb::substream;

constexpr double kPi = 3.14159265358979323846;

// Sequential RngStream (rng.hpp:10-27).
struct Stream {
  uint64_t state;
  explicit Stream(uint64_t seed) : state(mix64(seed)) {}
  uint64_t next_u64() {
    state += tmpcb::kGolden;
    return mix64(state);
  }
  double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * next_double(); }
};

double smooth(double t) { return t * t * (3.0 - 2.0 * t); }

void parallel_rows(int ny, int n_threads, const auto& fn) {
  const int nt = std::max(1, std::min(n_threads, ny));
  std::vector<std::thread> th;
  for (int w = 0; w < nt; ++w)
    th.emplace_back([&, w]() {
      for (int j = w; j < ny; j += nt) fn(j);
    });
  for (auto& t : th) t.join();
}

int hw_threads() { return std::max(1u, std::thread::hardware_concurrency()); }

// point_segment_distance (terrain.hpp:186-194), same operation order as the
// reference compiled against the Eigen shim.
inline double seg_dist(double px, double py, double ax, double ay, double bx, double by) {
  const double abx = bx - ax, aby = by - ay;
  const double len2 = abx * abx + aby * aby;
  if (len2 == 0.0) {
    const double dx = px - ax, dy = py - ay;
    return std::sqrt(dx * dx + dy * dy);
  }
  const double t = std::clamp(((px - ax) * abx + (py - ay) * aby) / len2, 0.0, 1.0);
  const double qx = px - (ax + abx * t), qy = py - (ay + aby * t);
  return std::sqrt(qx * qx + qy * qy);
}

// point_in_polygon (terrain.hpp:196-209).
inline bool inside_poly(double px, double py, const double* v, int n) {
  bool inside = false;
  for (int i = 0, j = n - 1; i < n; j = i++) {
    const double yi = v[2 * i + 1], yj = v[2 * j + 1];
    if ((yi > py) != (yj > py)) {
      const double x_at = v[2 * j] + (py - yj) / (yi - yj) * (v[2 * i] - v[2 * j]);
      if (px < x_at) inside = !inside;
    }
  }
  return inside;
}

// signed_distance (terrain.hpp:215-224).
inline double signed_dist(double px, double py, const double* v, int n, int kind) {
  double d = std::numeric_limits<double>::infinity();
  for (int i = 0; i < n; ++i) {
    const int j = (i + 1) % n;
    d = std::min(d, seg_dist(px, py, v[2 * i], v[2 * i + 1], v[2 * j], v[2 * j + 1]));
  }
  const bool in = inside_poly(px, py, v, n);
  const bool violating = kind == 0 ? in : !in;
  return violating ? -d : d;
}

}  // namespace

extern "C" {

int tmpc_synth_heightmap(const tmpc_synth_spec* s, double* out) {
  if (!s || !out || s->nx < 2 || s->ny < 2 || !(s->resolution > 0.0)) return TMPC_ERR_CONFIG;
  const int nx = s->nx, ny = s->ny;
  const size_t n = static_cast<size_t>(nx) * ny;
  std::fill(out, out + n, 0.0);
  const double r = s->resolution;

  if (s->sine_amp != 0.0) {
    if (!(s->sine_wavelength > 0.0)) return TMPC_ERR_CONFIG;
    Stream rng(substream(s->seed, 0x51E));
    const double p1 = rng.uniform(0.0, 2.0 * kPi), p2 = rng.uniform(0.0, 2.0 * kPi);
    const double kk = 2.0 * kPi / s->sine_wavelength;
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i)
        out[static_cast<size_t>(j) * nx + i] +=
            s->sine_amp * std::sin(kk * (r * i) + p1) * std::sin(kk * (r * j) + p2);
  }
  if (s->noise_amp != 0.0) {
    Stream rng(substream(s->seed, 0x401));
    for (size_t c = 0; c < n; ++c) out[c] += rng.uniform(-s->noise_amp, s->noise_amp);
  }
  if (s->fractal_octaves > 0 && s->fractal_pp != 0.0) {
    if (!(s->fractal_lattice > 0.0)) return TMPC_ERR_CONFIG;
    std::vector<double> v(n, 0.0);
    const double ext_x = r * (nx - 1), ext_y = r * (ny - 1);
    double amp = 1.0;
    for (int o = 0; o < s->fractal_octaves; ++o) {
      const double L = s->fractal_lattice / std::ldexp(1.0, o);
      const int lx = static_cast<int>(std::ceil(ext_x / L)) + 2;
      const int ly = static_cast<int>(std::ceil(ext_y / L)) + 2;
      std::vector<double> lat(static_cast<size_t>(lx) * ly);
      for (int b = 0; b < ly; ++b)
        for (int a = 0; a < lx; ++a) {
          Stream rng(substream(s->seed, 0xF4AC + o, a, b));
          lat[static_cast<size_t>(b) * lx + a] = rng.uniform(-1.0, 1.0);
        }
      parallel_rows(ny, hw_threads(), [&](int j) {
        const double gy = r * j / L;
        const int b = static_cast<int>(gy);
        const double ty = smooth(gy - b);
        for (int i = 0; i < nx; ++i) {
          const double gx = r * i / L;
          const int a = static_cast<int>(gx);
          const double tx = smooth(gx - a);
          const double* l0 = lat.data() + static_cast<size_t>(b) * lx + a;
          const double* l1 = l0 + lx;
          const double top = l0[0] + tx * (l0[1] - l0[0]);
          const double bot = l1[0] + tx * (l1[1] - l1[0]);
          v[static_cast<size_t>(j) * nx + i] += amp * (top + ty * (bot - top));
        }
      });
      amp *= s->fractal_persistence;
    }
    const auto [mn, mx] = std::minmax_element(v.begin(), v.end());
    const double lo = *mn, hi = *mx;
    const double scale = hi > lo ? s->fractal_pp / (hi - lo) : 0.0;
    const double mid = 0.5 * (lo + hi);
    for (size_t c = 0; c < n; ++c) out[c] += (v[c] - mid) * scale;
  }
  if (s->slope_deg != 0.0) {
    if (!(s->slope_period > 0.0)) return TMPC_ERR_CONFIG;
    // smooth alternating side slopes: a sinusoid whose steepest slope is
    // +-tan(slope_deg), i.e. amplitude tan(slope_deg) * P / (2 pi)
    const double amp = std::tan(s->slope_deg * kPi / 180.0) * s->slope_period / (2.0 * kPi);
    const double cx = std::cos(s->slope_dir), cy = std::sin(s->slope_dir);
    const double kk = 2.0 * kPi / s->slope_period;
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i)
        out[static_cast<size_t>(j) * nx + i] += amp * std::sin(kk * (cx * (r * i) + cy * (r * j)));
  }
  if (s->n_berms > 0 && s->berm_height != 0.0) {
    if (!(s->berm_halfwidth > 0.0) || !(s->berm_length >= 0.0)) return TMPC_ERR_CONFIG;
    Stream rng(substream(s->seed, 0xBE4));
    struct Berm { double ax, ay, bx, by; };
    std::vector<Berm> berms(s->n_berms);
    const double ext_x = r * (nx - 1), ext_y = r * (ny - 1);
    for (auto& b : berms) {
      const double cx = rng.uniform(0.0, ext_x), cy = rng.uniform(0.0, ext_y);
      const double th = rng.uniform(0.0, kPi);
      const double hx = 0.5 * s->berm_length * std::cos(th), hy = 0.5 * s->berm_length * std::sin(th);
      b = {cx - hx, cy - hy, cx + hx, cy + hy};
    }
    const double w = s->berm_halfwidth;
    parallel_rows(ny, hw_threads(), [&](int j) {
      for (int i = 0; i < nx; ++i) {
        double add = 0.0;
        for (const auto& b : berms) {
          const double d = seg_dist(r * i, r * j, b.ax, b.ay, b.bx, b.by);
          if (d < w) add += s->berm_height * 0.5 * (1.0 + std::cos(kPi * d / w));
        }
        out[static_cast<size_t>(j) * nx + i] += add;
      }
    });
  }
  return TMPC_OK;
}

int tmpc_synth_obstacles(const tmpc_obstacle_spec* s, double* circles, double* verts) {
  if (!s || s->n < 0 || s->n_gon < 3 || !(s->r_min > 0.0) || s->r_max < s->r_min)
    return TMPC_ERR_CONFIG;
  Stream rng(substream(s->seed, 0x0B57));
  for (int k = 0; k < s->n; ++k) {
    double cx = 0, cy = 0, rad = 0;
    for (int tries = 0; tries < 100000; ++tries) {
      cx = rng.uniform(s->x_min, s->x_max);
      cy = rng.uniform(s->y_min, s->y_max);
      rad = rng.uniform(s->r_min, s->r_max);
      const double dx = cx - s->clear_x, dy = cy - s->clear_y;
      if (std::sqrt(dx * dx + dy * dy) > s->clear_r + rad) break;
    }
    circles[3 * k] = cx;
    circles[3 * k + 1] = cy;
    circles[3 * k + 2] = rad;
    for (int v = 0; v < s->n_gon; ++v) {
      const double a = 2.0 * kPi * v / s->n_gon;
      verts[2 * (k * s->n_gon + v)] = cx + rad * std::cos(a);
      verts[2 * (k * s->n_gon + v) + 1] = cy + rad * std::sin(a);
    }
  }
  return TMPC_OK;
}

int tmpc_stamp_obstacles(const tmpc_terrain* g, double* heights, int32_t n_poly,
                         const int32_t* poly_off, const double* verts, double height) {
  if (!g || !heights || n_poly < 0) return TMPC_ERR_CONFIG;
  for (int k = 0; k < n_poly; ++k) {
    const double* v = verts + 2 * poly_off[k];
    const int nv = poly_off[k + 1] - poly_off[k];
    double x0 = 1e300, x1 = -1e300, y0 = 1e300, y1 = -1e300;
    for (int q = 0; q < nv; ++q) {
      x0 = std::min(x0, v[2 * q]); x1 = std::max(x1, v[2 * q]);
      y0 = std::min(y0, v[2 * q + 1]); y1 = std::max(y1, v[2 * q + 1]);
    }
    const int i0 = std::max(0, static_cast<int>(std::floor((x0 - g->origin_x) / g->resolution)));
    const int i1 = std::min(g->nx - 1, static_cast<int>(std::ceil((x1 - g->origin_x) / g->resolution)));
    const int j0 = std::max(0, static_cast<int>(std::floor((y0 - g->origin_y) / g->resolution)));
    const int j1 = std::min(g->ny - 1, static_cast<int>(std::ceil((y1 - g->origin_y) / g->resolution)));
    for (int j = j0; j <= j1; ++j)
      for (int i = i0; i <= i1; ++i)
        if (inside_poly(g->origin_x + g->resolution * i, g->origin_y + g->resolution * j, v, nv))
          heights[static_cast<size_t>(j) * g->nx + i] += height;
  }
  return TMPC_OK;
}

int tmpc_build_sdist_map(int32_t nx, int32_t ny, double ox, double oy, double res,
                         int32_t n_poly, const int32_t* poly_off, const double* verts,
                         const int32_t* kinds, double* out, int32_t n_threads) {
  if (nx < 1 || ny < 1 || !(res > 0.0) || n_poly < 0 || !out) return TMPC_ERR_CONFIG;
  const double inf = std::numeric_limits<double>::infinity();
  const size_t n = static_cast<size_t>(nx) * ny;
  std::fill(out, out + n, inf);
  if (n_poly == 0) return TMPC_OK;
  // bounding circles (all polygon points lie within r of the vertex centroid)
  std::vector<double> ccx(n_poly), ccy(n_poly), crad(n_poly);
  std::vector<int> always;  // path boundaries: sign flips outside, no culling
  for (int k = 0; k < n_poly; ++k) {
    const double* v = verts + 2 * poly_off[k];
    const int nv = poly_off[k + 1] - poly_off[k];
    if (nv < 3) return TMPC_ERR_CONFIG;
    double sx = 0, sy = 0;
    for (int q = 0; q < nv; ++q) { sx += v[2 * q]; sy += v[2 * q + 1]; }
    ccx[k] = sx / nv;
    ccy[k] = sy / nv;
    double rr = 0;
    for (int q = 0; q < nv; ++q)
      rr = std::max(rr, std::hypot(v[2 * q] - ccx[k], v[2 * q + 1] - ccy[k]));
    crad[k] = rr * (1.0 + 1e-12) + 1e-12;
    if (kinds && kinds[k] != 0) always.push_back(k);
  }
  constexpr int T = 32;  // tiles of T x T cells share a sorted candidate list
  const int tx = (nx + T - 1) / T, ty = (ny + T - 1) / T;
  const int nt = n_threads > 0 ? n_threads : hw_threads();
  parallel_rows(ty, nt, [&](int tj) {
    std::vector<std::pair<double, int>> cand;
    cand.reserve(n_poly);
    for (int ti = 0; ti < tx; ++ti) {
      const int i0 = ti * T, i1 = std::min(nx, i0 + T), j0 = tj * T, j1 = std::min(ny, j0 + T);
      const double cx = ox + res * 0.5 * (i0 + i1 - 1), cy = oy + res * 0.5 * (j0 + j1 - 1);
      const double half = res * 0.5 * std::hypot(i1 - i0, j1 - j0);
      cand.clear();
      for (int k = 0; k < n_poly; ++k) {
        if (kinds && kinds[k] != 0) continue;
        cand.emplace_back(std::hypot(cx - ccx[k], cy - ccy[k]) - crad[k] - half, k);
      }
      std::sort(cand.begin(), cand.end());
      for (int j = j0; j < j1; ++j) {
        const double y = oy + res * j;
        for (int i = i0; i < i1; ++i) {
          const double x = ox + res * i;
          double d = inf;
          for (int k : always)
            d = std::min(d, signed_dist(x, y, verts + 2 * poly_off[k], poly_off[k + 1] - poly_off[k], 1));
          for (const auto& [lbt, k] : cand) {
            if (lbt - 1e-9 > d) break;  // every later polygon is farther
            const double lb = std::hypot(x - ccx[k], y - ccy[k]) - crad[k];
            if (lb - 1e-9 > d) continue;
            d = std::min(d, signed_dist(x, y, verts + 2 * poly_off[k], poly_off[k + 1] - poly_off[k], 0));
          }
          out[static_cast<size_t>(j) * nx + i] = d;
        }
      }
    }
  });
  return TMPC_OK;
}

}  // extern "C"
