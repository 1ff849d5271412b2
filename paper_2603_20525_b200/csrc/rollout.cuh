// Device side of the planning hot path: per-candidate SRB rollout with fused
// constraint/cost evaluation and the per-GPU arg-min (SURVEY §8a rows
// R1-R10, T1-T3, C1-C3, P1-P3).  sm_100a, FP32 SIMT (+ fp64 accumulators),
// or all-fp64 in the certification mode.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "tmpc_common.h"

namespace tmpcb {

// Precision modes of the rollout kernel.
enum Precision : int {
  kFp32 = 0,  // fp32 math over fp32 terrain fields; fp64 state + cost storage
  kFp64 = 1,  // fp64 math over fp64 terrain fields (parity certification)
};

// Dynamics / constraint constants in the math type T (hoisted from
// dynamics.hpp:20-71,188-192,320-324 and constraints.hpp:16-58).
template <typename T>
struct KConsts {
  T g, half_M, inv_M;
  T cJx, cJy, cJz;  // (Jyy-Jzz), (Jxx-Jzz), (Jxx-Jyy)
  T inv_Jxx, inv_Jyy, inv_Jzz;
  T rho[4][3];                 // wheel_offsets
  T k_i[4], b_i[4], fs_i[4];   // spring, damper, static load 0.5 g K_zz,i
  T C, mu, mu2;
  T delta_max, vbx_floor, tau_floor;
  T esm_r_bar, esm_c_pb, esm_s_pb, esm_Mg, esm_phi_lim;  // R_bar, cos/sin phi_bar, M g, pi/2-phi_bar
  T inv_eps_esm, inv_esm_nominal;
  T sigma, inv_eps_dist;
  T dt;
  T inv_res;
  // EST formulation (dynamics.hpp:230-275, constraints.hpp:62-65,78-80)
  T kzzf, kzzr, kzx, L_f, L_r;
  T a_by_bar, inv_a_by_bar, inv_eps_aby;
  T esm_phi_bar;  // atan(2 (h + R) / e) (constraints.hpp:19)
};

struct Mailbox;     // the peer-memory record exchange (below)
struct RankRecord;  // one GPU's reduction record (below)

// Footprint clearance (fp32 store, spare texel of each cell record; built by
// ctx.cu footprint_clearance, read by the Euler kernel's skip test): a lower
// bound of the SDF over every footprint point of a CoM within
// kClearWindowMove cells of the cell, so one substep may move the CoM up to
// kClearMove cells; the soft cost is exactly 0 once sd / eps >= kClearCost.
constexpr int kClearWindowMove = 2;
constexpr float kClearMove = 1.9f;
constexpr float kClearCost = 1.0001f;

// Everything the kernel needs, passed by value (kernel parameter space), so
// several contexts on one device never share mutable constant memory.
struct KParams {
  KConsts<float> cf;
  KConsts<double> cd;
  int enable_dist, enable_rollover;
  // cost
  double w_t, w_c, w_g;
  double goal_x, goal_y, goal_r2;
  double dt;  // dt_int
  int n_steps, S;
  double gimbal_lim;  // pi/2 - kGimbalMargin (dynamics.hpp:16,311)
  // terrain store (padded by `pad` replicated cells per side: 2 in fp64 mode,
  // 2 E0 + 3 in fp32 mode, ctx.cu terrain_pad; grid coordinate g' = g + pad)
  double gx_scale, gx_off, gy_scale, gy_off;  // g' = x*scale + off
  int nx, ny, pitch;  // original sizes, padded row pitch (nx + 2 pad)
  int pad, cmargin;   // cmargin: CoM clamp margin E0 + 1 of the fp32 SRB kernels
  unsigned cell_bias;  // -0x4B400000 (pitch + 1) mod 2^32 (rollout_anchor.cuh cell2u)
  unsigned last_cell;  // index of the last record (pitch * rows - 1)
  int has_sdist;
  // sampler
  Sampler smp;
  uint64_t seed;
  int64_t k_begin, k_count;
  int64_t k_layout;  // the whole problem's K (tmpc_sampling.k_total): picks kernel variants
  int selection;
  int precision;
  int model;   // TMPC_MODEL_SRB / TMPC_MODEL_EST
  int scheme;  // TMPC_SCHEME_EULER / TMPC_SCHEME_RK4 (dynamics.hpp:419)
  // candidate of thread slot t is order[t] (order.cu); nullptr = identity
  const int32_t* order;
  // fused record exchange over peer memory (one process per GPU, IPC mode;
  // reduce_and_finalize): the last block writes this GPU's record into slot
  // xrank of every rank's mailbox (xpeers[g], NVLink stores), publishes
  // sequence number xseq, and waits until every rank's record of this cycle
  // has arrived in its own mailbox (xpeers[xrank]) or xtimeout_ns passes.
  // xn == 0: no exchange.  xn < 0 (one process, no collective): xhost is
  // this GPU's RankRecord in pinned mapped host memory; the last block writes
  // the record there and resets the reduction block for the next cycle
  // (reduce_and_finalize host_record): the cycle is one kernel, no D2H copy.
  union {
    Mailbox* const* xpeers;  // xn > 0
    RankRecord* xhost;       // xn < 0
  };
  int xn, xrank;
  unsigned long long xseq, xtimeout_ns;
  // terrain rows / columns (padded cells, inclusive) the cycle can reach,
  // prefetched into L2 at kernel start (rollout_dev.cuh l2_prefetch_terrain);
  // pf_j1 < pf_j0 disables
  int pf_i0, pf_i1, pf_j0, pf_j1;
  // initial state (SrbState::as_array order)
  double s0[13];
};

template <typename T>
__host__ __device__ inline const KConsts<T>& consts(const KParams& P);
template <>
__host__ __device__ inline const KConsts<float>& consts<float>(const KParams& P) { return P.cf; }
template <>
__host__ __device__ inline const KConsts<double>& consts<double>(const KParams& P) { return P.cd; }

// fp64 terrain texel of the certification mode ({H, dH/dx} and {dH/dy, 0}).
struct __align__(16) HG64 {
  double2 a, b;
};

// Per-cycle reduction block of one GPU (reset before each cycle).  Every
// field is reduced with integer atomics (or a 128-bit CAS-min), so the block
// is bit-identical for any launch order, block size or scheduling; across
// GPUs the blocks are gathered and folded in rank order (ctx.cu
// fold_records), so it is also independent of the GPU count.
struct __align__(16) DevStats {
  unsigned long long key_lo;  // arg-min (hi, lo) pair (tmpc_common.h key_hi),
  unsigned long long key_hi;  // 16-B aligned for atom.cas.b128; init kKeyNone
  unsigned long long min_cost_bits;  // bits of the least finite cost, init +inf
  unsigned long long done_blocks;
  unsigned long long n_feasible, n_diverged, n_goal, n_finite, substeps;
  unsigned long long cost_limb[3];  // fixed-point sum of finite costs (cost_limbs)
  // filled by the last block (this GPU's winner)
  double best_cost;
  float best_margin;
  int best_flags;
};

// One GPU's contribution to a multi-GPU cycle (ncclAllGather / host gather).
struct __align__(16) RankRecord {
  DevStats s;
  long long k_begin, k_count;
};

// A rank's mailbox in its own device memory, written by every rank's rollout
// kernel over peer memory: record slot g holds rank g's record of the cycle
// whose sequence number seq[g] carries; err: this rank's wait timed out.
constexpr int kMaxRanks = 64;
// Records are double-buffered by the cycle's parity: a rank can run at most
// one cycle ahead of another (its next wait needs the other's next record),
// so cycle n + 1 never overwrites the cycle-n records a slower rank is still
// copying home; sequence numbers only grow, so waits test seq >= this cycle.
struct __align__(16) Mailbox {
  RankRecord rec[2][kMaxRanks];
  unsigned long long seq[kMaxRanks];
  unsigned long long err;
};

// Terrain store on the device (padded by 2 replicated cells per side).
//  fp32: hq32 cell records of 4 float4 (64 B, one L1 half-line): the quads
//        {v(i,j), v(i+1,j), v(i,j+1), v(i+1,j+1)} of H, dH/dx, dH/dy and a pad,
//        so one contact-point lookup is 3 x 16-B loads from one line;
//        sdq32 SDF quad texels (one 16-B gather per lookup).
//  fp64: hg64 node texels; sd64 node SDF.
struct TerrainDev {
  const float4* hq32;
  const float4* sdq32;
  const HG64* hg64;
  const double* sd64;
  // the sdq32 / hq32 records as 1-D float4 textures (TEX-pipe gathers)
  unsigned long long sd_tex, hq_tex;
};

}  // namespace tmpcb
