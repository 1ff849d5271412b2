// Host/device helpers shared by the CUDA rollout kernel and the host side of
// libtmpc_b200: counter RNG, control sampler, arg-min key.
#pragma once
#include <stdint.h>

#include "tmpc_b200.h"

#ifdef __CUDACC__
#define TMPC_HD __host__ __device__ __forceinline__
#else
#include <algorithm>
#include <cmath>
#define TMPC_HD inline
#endif

namespace tmpcb {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

// SplitMix64 finaliser — RngStream::mix (rng.hpp:29-34).
TMPC_HD uint64_t mix64(uint64_t z) {
  z += kGolden;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// substream(seed, a, b, c) (rng.hpp:41-48).
TMPC_HD uint64_t substream(uint64_t seed, uint64_t a, uint64_t b = 0, uint64_t c = 0) {
  uint64_t s = mix64(seed);
  s = mix64(s ^ (a + kGolden));
  s = mix64(s ^ (b + 0xBF58476D1CE4E5B9ULL));
  s = mix64(s ^ (c + 0x94D049BB133111EBULL));
  return s;
}

// Random access into RngStream(stream_seed): the constructor stores
// mix(stream_seed) (rng.hpp:12) and draw j returns mix(state + (j+1)*golden)
// (rng.hpp:14-17).  `base` = mix(stream_seed).
TMPC_HD uint64_t draw_u64(uint64_t base, uint64_t j) { return mix64(base + (j + 1) * kGolden); }
// next_double (rng.hpp:20-22).
TMPC_HD double draw_unit(uint64_t base, uint64_t j) {
  return static_cast<double>(draw_u64(base, j) >> 11) * 0x1.0p-53;
}
TMPC_HD double clampd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }

// Correctly rounded fp64 multiply / add that the compiler may not contract
// into an FMA (nvcc contracts device code by default): the sampled controls
// must equal, bit for bit, the reference RngStream::uniform arithmetic
// (rng.hpp:25-27) evaluated in IEEE order.  Host objects are built with
// -ffp-contract=off for the same reason.
TMPC_HD double dmul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
TMPC_HD double dadd(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
// RngStream::uniform(lo, hi) = lo + (hi - lo) * u
TMPC_HD double uniform_lohi(double lo, double hi, double u) { return dadd(lo, dmul(dadd(hi, -lo), u)); }

// Sampler state of one candidate (SPEC.md:377-383 + BASELINE extensions).
struct Sampler {
  int kind;
  int nch;          // 1: delta_rate only (v_bx_rate = 0); 2: both
  double bound[2];  // delta_rate_max, vdot_max
  double step[2];   // random-walk increments
  double sigma[2];  // Gaussian sigmas (fraction * range)
};

TMPC_HD Sampler make_sampler(const tmpc_params& p, const tmpc_sampling& s) {
  Sampler z;
  z.kind = s.kind;
  z.nch = s.vdot_max > 0.0 ? 2 : 1;
  z.bound[0] = p.delta_rate_max;
  z.bound[1] = s.vdot_max;
  z.step[0] = s.walk_step;
  z.step[1] = s.walk_step * s.vdot_max / p.delta_rate_max;
  z.sigma[0] = s.warm_sigma_frac * 2.0 * p.delta_rate_max;
  z.sigma[1] = s.warm_sigma_frac * 2.0 * s.vdot_max;
  return z;
}

// Control of step t for the candidate whose stream base is `base`
// (= mix(substream(seed, k))).  `prev` carries the random-walk state and
// `warm` the base sequence (n_steps x 2) for TMPC_SAMPLE_WARM_GAUSS.
// Draw accounting matches sequential use of one RngStream: per step and
// channel one draw (uniform/walk) or two (Gaussian, Box-Muller).
TMPC_HD void sample_step(const Sampler& z, uint64_t base, bool is_k0, int t,
                         const double* warm, double prev[2], double out[2]) {
  out[0] = 0.0;
  out[1] = 0.0;
  for (int c = 0; c < z.nch; ++c) {
    const double b = z.bound[c];
    if (z.kind == TMPC_SAMPLE_UNIFORM) {
      const uint64_t j = static_cast<uint64_t>(t) * z.nch + c;
      out[c] = uniform_lohi(-b, b, draw_unit(base, j));  // uniform(lo, hi), rng.hpp:25-27
    } else if (z.kind == TMPC_SAMPLE_RANDOM_WALK) {
      const uint64_t j = static_cast<uint64_t>(t) * z.nch + c;
      const double a = z.step[c];
      out[c] = clampd(dadd(prev[c], uniform_lohi(-a, a, draw_unit(base, j))), -b, b);
      prev[c] = out[c];
    } else {
      const uint64_t j = 2 * (static_cast<uint64_t>(t) * z.nch + c);
      const double bs = warm ? warm[2 * t + c] : 0.0;
      if (is_k0) {
        out[c] = clampd(bs, -b, b);
      } else {
        const double u1 = draw_unit(base, j);
        const double u2 = draw_unit(base, j + 1);
#ifdef __CUDA_ARCH__
        const double zz = sqrt(-2.0 * log(1.0 - u1)) * cos(2.0 * 3.14159265358979323846 * u2);
#else
        const double zz = std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
#endif
        out[c] = clampd(dadd(bs, dmul(z.sigma[c], zz)), -b, b);
      }
    }
  }
}

// Arg-min key: the pair (hi, lo) in lexicographic order,
// hi = infeasible << 63 | IEEE bits of the fp64 cost, lo = global index.
// Costs are >= 0 or +inf (every term of J is non-negative),
// so their bit patterns order like their values and the pair's MIN is the
// (infeasible, J, k) arg-min with ties to the lowest index on
// the exact fp64 cost the reference compares (no rounding of J in the key).
TMPC_HD uint64_t dbits(double v) {
#ifdef __CUDA_ARCH__
  return static_cast<uint64_t>(__double_as_longlong(v));
#else
  uint64_t b;
  __builtin_memcpy(&b, &v, 8);
  return b;
#endif
}
TMPC_HD uint64_t key_hi(double cost, bool infeasible) {
  return (infeasible ? (1ULL << 63) : 0ULL) | (dbits(cost) & 0x7FFFFFFFFFFFFFFFULL);
}
TMPC_HD bool key_less(uint64_t ahi, uint64_t alo, uint64_t bhi, uint64_t blo) {
  return ahi < bhi || (ahi == bhi && alo < blo);
}
constexpr uint64_t kKeyNone = ~0ULL;  // (hi, lo) of "no candidate"

// Order-independent cost sum (the solver output, its mean cost
// included, must not depend on the worker count or scheduling): each finite
// cost is rounded once to the fixed-point grid 2^-24 and split into three
// 32-bit limbs; integer sums of the limbs are exact in any order, on any
// number of GPUs (each limb sum stays below 2^64 for < 2^32 candidates).
// Costs at or above 2^72 saturate (never reached: sigma * (1 + |pi|/eps)^2
// * horizon is ~1e10 for a vehicle lying on its roof for the whole horizon).
constexpr double kCostQuantum = 0x1.0p-24;
TMPC_HD void cost_limbs(double J, uint64_t limb[3]) {
  double q = J * 0x1.0p24;
  if (!(q < 0x1.0p96)) q = 0x1.fffffffffffffp95;
#ifdef __CUDA_ARCH__
  const double hi = floor(q * 0x1.0p-32);
  const double l2 = floor(hi * 0x1.0p-32);
  limb[0] = __double2ull_rn(q - hi * 0x1.0p32);
  limb[1] = __double2ull_rn(hi - l2 * 0x1.0p32);
  limb[2] = __double2ull_rn(l2);
#else
  const double hi = std::floor(q * 0x1.0p-32);
  const double l2 = std::floor(hi * 0x1.0p-32);
  limb[0] = static_cast<uint64_t>(std::nearbyint(q - hi * 0x1.0p32));
  limb[1] = static_cast<uint64_t>(hi - l2 * 0x1.0p32);
  limb[2] = static_cast<uint64_t>(l2);
#endif
}
// The sum of the limb sums as a double (exact integer arithmetic, one
// rounding; host only).
inline double limbs_value(const uint64_t s[3]) {
  const unsigned __int128 t = (static_cast<unsigned __int128>(s[2]) << 64) +
                              (static_cast<unsigned __int128>(s[1]) << 32) + s[0];
  return static_cast<double>(t) * kCostQuantum;
}

}  // namespace tmpcb
