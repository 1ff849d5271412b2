// Device helpers shared by the rollout kernels (terrain store access,
// warp reductions, per-cycle arg-min / stats finalisation).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fastmath.cuh"
#include "rollout.cuh"
#include "tmpc_common.h"

namespace tmpcb {

constexpr int kBlock = 32;  // one warp per CTA: spreads small K over all 148 SMs

// ---- math dispatch (fp64 certification kernel) ----------------------------
__device__ __forceinline__ void dsincos(float a, float* s, float* c) { sincosf(a, s, c); }
__device__ __forceinline__ void dsincos(double a, double* s, double* c) { sincos(a, s, c); }
__device__ __forceinline__ float datan(float a) { return atanf(a); }
__device__ __forceinline__ double datan(double a) { return atan(a); }
__device__ __forceinline__ float dcos(float a) { return cosf(a); }
__device__ __forceinline__ double dcos(double a) { return cos(a); }

// ---- terrain store access --------------------------------------------------
// Split a padded grid coordinate g' (fp64) into integer + fraction so
// per-wheel offsets (a few cells) are added in T without losing the absolute
// position.
template <typename T>
__device__ __forceinline__ void split_coord(double g, int& gi, T& gf) {
  const double fl = floor(g);
  gi = static_cast<int>(fl);
  gf = static_cast<T>(g - fl);
}

// Clamped cell index and fraction along one axis for g' = gi + gf + off,
// clamped to [n_lo, n_hi] = [Q-1, n+Q] (== the reference's clamp to [0, n-1]
// on the Q-cell replicate-padded grid, terrain.hpp:37-44).
template <typename T>
__device__ __forceinline__ void axis_cell(int gi, T gf, T off, int n_lo, int n_hi, int& i0, T& f) {
  const T t = gf + off;
  const T ft = floor(t);
  int i = gi + static_cast<int>(ft);
  T fr = t - ft;
  if (i < n_lo) {
    i = n_lo;
    fr = T(0);
  } else if (i >= n_hi) {
    i = n_hi;
    fr = T(0);
  }
  i0 = i;
  f = fr;
}

// detail::bilinear (terrain.hpp:45-49) on the padded node fields: one texel
// gather per corner gives height and both gradient components
// (gradient_at == bilinear of the node central differences).
__device__ __forceinline__ void lerp_hg(const float4& a0, const float4& a1, const float4& b0,
                                        const float4& b1, float fx, float fy, float& h, float& gxs,
                                        float& gys) {
  const float ha = a0.x + fx * (a1.x - a0.x), hb = b0.x + fx * (b1.x - b0.x);
  const float xa = a0.y + fx * (a1.y - a0.y), xb = b0.y + fx * (b1.y - b0.y);
  const float ya = a0.z + fx * (a1.z - a0.z), yb = b0.z + fx * (b1.z - b0.z);
  h = ha + fy * (hb - ha);
  gxs = xa + fy * (xb - xa);
  gys = ya + fy * (yb - ya);
}
__device__ __forceinline__ void lookup_hg(const TerrainDev& td, int pitch, int i0, int j0,
                                          double fx, double fy, double& h, double& gxs,
                                          double& gys) {
  const HG64* r0 = td.hg64 + static_cast<size_t>(j0) * pitch + i0;
  const double2 a0 = __ldg(&r0->a), a0b = __ldg(&r0->b);
  const double2 a1 = __ldg(&(r0 + 1)->a), a1b = __ldg(&(r0 + 1)->b);
  const double2 b0 = __ldg(&(r0 + pitch)->a), b0b = __ldg(&(r0 + pitch)->b);
  const double2 b1 = __ldg(&(r0 + pitch + 1)->a), b1b = __ldg(&(r0 + pitch + 1)->b);
  const double ha = a0.x + fx * (a1.x - a0.x), hb = b0.x + fx * (b1.x - b0.x);
  const double xa = a0.y + fx * (a1.y - a0.y), xb = b0.y + fx * (b1.y - b0.y);
  const double ya = a0b.x + fx * (a1b.x - a0b.x), yb = b0b.x + fx * (b1b.x - b0b.x);
  h = ha + fy * (hb - ha);
  gxs = xa + fy * (xb - xa);
  gys = ya + fy * (yb - ya);
}

// detail::bilinear (terrain.hpp:45-49) from a cell record in coefficient
// form {c0, c1, c2, c3} = {v00, v10 - v00, v01 - v00, v11 - v10 - v01 + v00}
// (built in fp64 on the host, rounded once): f = c0 + c1 fx + c2 fy +
// c3 fx fy as 3 dependent-pair FFMAs instead of 3 lerps (3 FADD + 3 FFMA).
// The two inner FMAs run as one FFMA2 on the record's natural register pairs
// (c0, c1) and (c2, c3), fy broadcast: 2 instructions instead of 3.
__device__ __forceinline__ float lerp_quad(const float4& q, float fx, float fy) {
  float a, b;  // a = c2 fy + c0, b = c3 fy + c1
  fm::upk(fm::ffma2(fm::pk(q.z, q.w), fm::pk(fy, fy), fm::pk(q.x, q.y)), a, b);
  return fmaf(b, fx, a);
}

__device__ __forceinline__ double lookup_sd(const double* __restrict__ sd, int pitch, int i0,
                                            int j0, double fx, double fy) {
  const double* r0 = sd + static_cast<size_t>(j0) * pitch + i0;
  const double a0 = __ldg(r0), a1 = __ldg(r0 + 1), b0 = __ldg(r0 + pitch), b1 = __ldg(r0 + pitch + 1);
  const double a = a0 + fx * (a1 - a0), b = b0 + fx * (b1 - b0);
  return a + fy * (b - a);
}

// ---- precision-generic terrain access (EST / RK4 kernels) -----------------
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


// Bulk L2 prefetch (TMA engine, cp.async.bulk.prefetch.L2) of the terrain
// rows the cycle can reach, spread over the launch's threads.  The planning
// cycle starts from a cold L2 (the bench flushes it; in a closed loop other
// work evicts it), and a latency-bound rollout would otherwise pay a DRAM
// round trip on the first touch of every terrain line along its path.
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, long long bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~static_cast<uintptr_t>(15);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~static_cast<uintptr_t>(15);
  for (uintptr_t c = a; c < e; c += 32768) {
    const unsigned n = static_cast<unsigned>(e - c < 32768 ? e - c : 32768);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(c), "r"(n) : "memory");
  }
}

__device__ __forceinline__ void l2_prefetch_terrain(const KParams& P, const TerrainDev& td) {
  const int rows = P.pf_j1 - P.pf_j0 + 1;
  if (rows <= 0) return;
  const long long cols = P.pf_i1 - P.pf_i0 + 1;
  const bool f64 = P.precision == kFp64;
  const int hq_b = f64 ? static_cast<int>(sizeof(HG64)) : 64, sd_b = f64 ? 8 : 16;
  const char* hq = f64 ? reinterpret_cast<const char*>(td.hg64) : reinterpret_cast<const char*>(td.hq32);
  const char* sd = f64 ? reinterpret_cast<const char*>(td.sd64) : reinterpret_cast<const char*>(td.sdq32);
  const int stride = gridDim.x * blockDim.x;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += stride) {
    const long long cell = static_cast<long long>(P.pf_j0 + r) * P.pitch + P.pf_i0;
    bulk_prefetch_l2(hq + cell * hq_b, cols * hq_b);
    if (P.has_sdist) bulk_prefetch_l2(sd + cell * sd_b, cols * sd_b);
  }
}

template <typename V>
__device__ __forceinline__ V warp_min(V v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const V w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  return v;
}
__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// 128-bit atomic MIN of the arg-min pair (hi, lo) at st->key_lo/key_hi: a CAS
// loop on atom.global.cas.b128 (sm_90+).  The first read may be torn; the CAS
// then fails and returns the true current pair.
__device__ __forceinline__ void atomic_min_key(DevStats* st, unsigned long long hi,
                                               unsigned long long lo) {
  unsigned long long* a = &st->key_lo;
  unsigned long long cur_lo = *reinterpret_cast<volatile unsigned long long*>(a);
  unsigned long long cur_hi = *reinterpret_cast<volatile unsigned long long*>(a + 1);
  while (key_less(hi, lo, cur_hi, cur_lo)) {
    unsigned long long o_lo, o_hi;
    asm volatile(
        "{\n\t.reg .b128 d, cmp, val;\n\t"
        "mov.b128 cmp, {%2, %3};\n\t"
        "mov.b128 val, {%4, %5};\n\t"
        "atom.global.cas.b128 d, [%6], cmp, val;\n\t"
        "mov.b128 {%0, %1}, d;\n\t}"
        : "=l"(o_lo), "=l"(o_hi)
        : "l"(cur_lo), "l"(cur_hi), "l"(lo), "l"(hi), "l"(a)
        : "memory");
    if (o_lo == cur_lo && o_hi == cur_hi) return;
    cur_lo = o_lo;
    cur_hi = o_hi;
  }
}

// The fused cross-GPU exchange of one cycle (KParams xpeers): this GPU's
// reduction record, final now that the last block holds it, is stored into
// slot xrank of every rank's mailbox over peer memory (NVLink), and its
// sequence number published with a system-scope release store; then
// the block waits (acquire loads, backing off) until every rank's record of
// this cycle sits in its own mailbox, or marks err after xtimeout_ns (a peer
// that never ran).  The host then copies the G records home and folds them
// in rank order (ctx.cu), as with the NCCL all-gather this replaces.
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
static __device__ __noinline__ void exchange_record(Mailbox* const* peers, int n, int rank,
                                                    unsigned long long seq,
                                                    unsigned long long timeout_ns, long long kb,
                                                    long long kc, const DevStats* st) {
  RankRecord r;
  {
    const volatile unsigned long long* a = reinterpret_cast<const volatile unsigned long long*>(st);
    unsigned long long* b = reinterpret_cast<unsigned long long*>(&r.s);
#pragma unroll 1
    for (int i = 0; i < static_cast<int>(sizeof(DevStats) / 8); ++i) b[i] = a[i];
  }
  r.k_begin = kb;
  r.k_count = kc;
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(&r);
#pragma unroll 1
  for (int g = 0; g < n; ++g) {
    volatile unsigned long long* dst =
        reinterpret_cast<volatile unsigned long long*>(&peers[g]->rec[seq & 1][rank]);
#pragma unroll 1
    for (int i = 0; i < static_cast<int>(sizeof(RankRecord) / 8); ++i) dst[i] = src[i];
  }
  // the release store at system scope orders this thread's record stores
  // before its sequence number for every observer (no separate fence)
#pragma unroll 1
  for (int g = 0; g < n; ++g) {
    unsigned long long* f = &peers[g]->seq[rank];
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(seq) : "memory");
  }
  Mailbox* me = peers[rank];
  const unsigned long long t0 = global_ns();
#pragma unroll 1
  for (int g = 0; g < n; ++g) {
    for (;;) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(&me->seq[g]) : "memory");
      if (v >= seq) break;
      if (global_ns() - t0 > timeout_ns) {
        // mark this rank's own slot of the cycle (only this kernel writes it,
        // and the host copies the records only: one D2H) and the mailbox
        me->rec[seq & 1][rank].k_begin = -1;
        me->err = 1;
        __threadfence_system();
        return;
      }
      __nanosleep(200);
    }
  }
}

// Per-candidate outputs, warp-level arg-min + stats (one atomic set per
// warp, all integer: order-independent), and the last-block finalisation
// that copies the local winner's exact fp64 cost / flags / margin into the
// stats block.
// The record of a one-process cycle (KParams::xn < 0), by the last block:
// the final reduction block and the shard into this GPU's host record
// (pinned, mapped; the kernel's completion -- the host's stream sync -- makes
// the stores visible, so no fence), then the reduction block reset for the
// next cycle (stats_reset_kernel's values; every other block has retired its
// atomics: this is the last ticket).
static __device__ __noinline__ void host_record(RankRecord* out, long long kb, long long kc,
                                                DevStats* st) {
  {
    const volatile unsigned long long* a = reinterpret_cast<const volatile unsigned long long*>(st);
    unsigned long long* b = reinterpret_cast<unsigned long long*>(&out->s);
#pragma unroll 1
    for (int i = 0; i < static_cast<int>(sizeof(DevStats) / 8); ++i) b[i] = a[i];
  }
  out->k_begin = kb;
  out->k_count = kc;
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

__device__ __forceinline__ void reduce_and_finalize(const KParams& P, bool active, int64_t kl,
                                                    int64_t kg, double J, bool feasible,
                                                    bool diverged, bool goal, float margin,
                                                    unsigned substeps, double* out_cost,
                                                    uint8_t* out_flags, float* out_margin,
                                                    DevStats* st) {
  if (active) {
    out_cost[kl] = J;
    out_flags[kl] = static_cast<uint8_t>((feasible ? TMPC_FLAG_FEASIBLE : 0) |
                                         (diverged ? TMPC_FLAG_DIVERGED : 0) |
                                         (goal ? TMPC_FLAG_GOAL : 0));
    out_margin[kl] = margin;
    // every writer fences its own outputs before the block's ticket: the
    // last block reads the winner's cost / flags / margin (written by any
    // lane of any block), and a fence by thread 0 alone orders only its own
    // stores
    __threadfence();
  }
  const bool infeasible = P.selection == TMPC_SELECT_FEASIBLE_FIRST && !feasible;
  unsigned long long khi = active ? key_hi(J, infeasible) : kKeyNone;
  unsigned long long klo = active ? static_cast<unsigned long long>(kg) : kKeyNone;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long h2 = __shfl_xor_sync(0xffffffffu, khi, o);
    const unsigned long long l2 = __shfl_xor_sync(0xffffffffu, klo, o);
    if (key_less(h2, l2, khi, klo)) {
      khi = h2;
      klo = l2;
    }
  }
  const bool fin = active && !diverged;
  const unsigned mfeas = __ballot_sync(0xffffffffu, active && feasible);
  const unsigned mdiv = __ballot_sync(0xffffffffu, active && diverged);
  const unsigned mgoal = __ballot_sync(0xffffffffu, active && goal);
  const unsigned mfin = __ballot_sync(0xffffffffu, fin);
  uint64_t limb[3] = {0, 0, 0};
  if (fin) cost_limbs(J, limb);
  limb[0] = warp_sum_u64(limb[0]);
  limb[1] = warp_sum_u64(limb[1]);
  limb[2] = warp_sum_u64(limb[2]);
  const long long cmin = warp_min(fin ? __double_as_longlong(J) : 0x7ff0000000000000LL);
  const unsigned ssum = __reduce_add_sync(0xffffffffu, substeps);
  if ((threadIdx.x & 31) == 0) {
    if (khi != kKeyNone) atomic_min_key(st, khi, klo);
    atomicAdd(&st->n_feasible, static_cast<unsigned long long>(__popc(mfeas)));
    atomicAdd(&st->n_diverged, static_cast<unsigned long long>(__popc(mdiv)));
    atomicAdd(&st->n_goal, static_cast<unsigned long long>(__popc(mgoal)));
    atomicAdd(&st->n_finite, static_cast<unsigned long long>(__popc(mfin)));
    atomicAdd(&st->substeps, static_cast<unsigned long long>(ssum));
    if (mfin) {
      atomicAdd(&st->cost_limb[0], limb[0]);
      atomicAdd(&st->cost_limb[1], limb[1]);
      atomicAdd(&st->cost_limb[2], limb[2]);
      atomicMin(&st->min_cost_bits, static_cast<unsigned long long>(cmin));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned long long ticket = atomicAdd(&st->done_blocks, 1ULL);
    if (ticket == gridDim.x - 1) {
      __threadfence();
      const unsigned long long kidx = *reinterpret_cast<volatile unsigned long long*>(&st->key_lo);
      const int64_t w = static_cast<int64_t>(kidx) - P.k_begin;
      if (kidx != kKeyNone && w >= 0 && w < P.k_count) {
        st->best_cost = *reinterpret_cast<volatile double*>(&out_cost[w]);
        st->best_flags = *reinterpret_cast<volatile uint8_t*>(&out_flags[w]);
        st->best_margin = *reinterpret_cast<volatile float*>(&out_margin[w]);
      }
      if (P.xn > 0)
        exchange_record(P.xpeers, P.xn, P.xrank, P.xseq, P.xtimeout_ns, P.k_begin, P.k_count, st);
      else if (P.xn < 0)
        host_record(P.xhost, P.k_begin, P.k_count, st);
    }
  }
}

// Control of ZOH step t (sample_step, tmpc_common.h; SPEC.md:377-383 + D6/D7)
// for the boundary block of the fp32 kernels: the uniform and random-walk
// draws of the steering channel inline and branch-free (bit-identical to
// sample_step), the Gaussian warm start and the throttle channel through the
// generic code.  prev0 / prev1: random-walk state per channel, in registers.
__device__ __forceinline__ void zoh_control(const KParams& P, uint64_t base, bool is_k0, int t,
                                            const double* warm, double& prev0, double& prev1,
                                            double& u0, double& u1) {
  const double prev0_in = prev0;
  const double ud = draw_unit(base, static_cast<uint64_t>(t));
  const double b = P.smp.bound[0], a = P.smp.step[0];
  const double uni = uniform_lohi(-b, b, ud);
  const double walk = clampd(dadd(prev0_in, uniform_lohi(-a, a, ud)), -b, b);
  const bool is_walk = P.smp.kind == TMPC_SAMPLE_RANDOM_WALK;
  u0 = is_walk ? walk : uni;
  u1 = 0.0;
  prev0 = is_walk ? walk : prev0_in;
  if (P.smp.nch != 1 || P.smp.kind == TMPC_SAMPLE_WARM_GAUSS) {
    double pv[2] = {prev0_in, prev1}, u[2];
    sample_step(P.smp, base, is_k0, t, warm, pv, u);
    prev0 = pv[0];
    prev1 = pv[1];
    u0 = u[0];
    u1 = u[1];
  }
}

}  // namespace tmpcb
