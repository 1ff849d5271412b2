// Candidate ordering pre-pass of the fp32 rollout kernel (terrain locality).
//
// The rollout kernel's stalls at the headline batch (c2: < 1 warp per
// scheduler) are dominated by terrain gathers that miss L1: the 32 candidates
// of a warp follow 32 unrelated paths, so every lane's wheel records sit in
// different 128-B lines.  Before the rollout, this pass predicts each
// candidate's path with a kinematic single-track model (same sampled
// controls, ZOH steps, no terrain) and buckets the candidates by a Morton
// code of the predicted lateral offsets at half and full horizon (counting
// sort: histogram, one-CTA scan, scatter — three launches).  The rollout
// kernel then gives thread t the candidate order[t]: neighbours in a warp
// drive near-identical paths, gather the same lines, and L1 serves most of
// the warp's requests.  Only the assignment of candidates to threads
// changes: each candidate is still evaluated from its own global index, so
// every per-candidate output and the arg-min are unchanged (the order inside
// a bucket follows atomic arrival and does not matter).
#include <cub/block/block_scan.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include "launch.cuh"
#include "rollout.cuh"
#include "tmpc_common.h"

namespace tmpcb {

namespace {

__device__ __forceinline__ uint32_t spread16(uint32_t v) {
  v &= 0xffffu;
  v = (v | (v << 8)) & 0x00ff00ffu;
  v = (v | (v << 4)) & 0x0f0f0f0fu;
  v = (v | (v << 2)) & 0x33333333u;
  v = (v | (v << 1)) & 0x55555555u;
  return v;
}

__device__ __forceinline__ uint32_t quant16(float lat, float inv_range) {
  const float u = fminf(fmaxf(fmaf(lat, inv_range, 0.5f), 0.f), 0.99999f);
  return static_cast<uint32_t>(u * 65536.f);
}

constexpr int kOrderBits = 14;  // 7 bits per predicted lateral offset
constexpr int kBins = 1 << kOrderBits;
constexpr int kScanThreads = 1024;

__global__ void __launch_bounds__(128) order_key_kernel(const KParams P,
                                                        const double* __restrict__ warm,
                                                        uint16_t* __restrict__ bin,
                                                        unsigned* __restrict__ hist) {
  const int64_t kl = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (kl >= P.k_count) return;
  const int64_t kg = P.k_begin + kl;
  const uint64_t base = mix64(substream(P.seed, static_cast<uint64_t>(kg)));
  double prev[2] = {0.0, 0.0};
  const float dtz = static_cast<float>(P.dt * P.S);
  const float inv_wb = 1.f / (P.cf.L_f + P.cf.L_r);
  const float dmax = P.cf.delta_max;
  float v = static_cast<float>(P.s0[6]);
  float de = static_cast<float>(P.s0[12]);
  float psi = 0.f, y = 0.f;  // in the frame of the initial heading
  const int half = (P.n_steps + 1) / 2;
  float lat_half = 0.f;
  for (int t = 0; t < P.n_steps; ++t) {
    double u[2];
    sample_step(P.smp, base, kg == 0, t, warm, prev, u);
    de = fminf(fmaxf(de + static_cast<float>(u[0]) * dtz, -dmax), dmax);
    v += static_cast<float>(u[1]) * dtz;
    psi += v * __tanf(de) * inv_wb * dtz;
    y += v * __sinf(psi) * dtz;
    if (t + 1 == half) lat_half = y;
  }
  // lateral offsets relative to the reach of the horizon, 7 bits each
  const float reach = fabsf(static_cast<float>(P.s0[6])) * dtz * P.n_steps + 1.f;
  const uint32_t code = (spread16(quant16(lat_half, 1.f / reach) >> 9) << 1) |
                        spread16(quant16(y, 0.5f / reach) >> 9);
  bin[kl] = static_cast<uint16_t>(code);
  atomicAdd(&hist[code], 1u);
}

// Exclusive scan of the histogram into the scatter cursors; re-zeroes the
// histogram for the next cycle.
__global__ void __launch_bounds__(kScanThreads) order_scan_kernel(unsigned* __restrict__ hist,
                                                                  unsigned* __restrict__ cursor) {
  using Scan = cub::BlockScan<unsigned, kScanThreads>;
  __shared__ typename Scan::TempStorage tmp;
  constexpr int kPer = kBins / kScanThreads;
  unsigned v[kPer];
  unsigned sum = 0;
  const int b0 = threadIdx.x * kPer;
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    v[i] = hist[b0 + i];
    sum += v[i];
  }
  unsigned off;
  Scan(tmp).ExclusiveSum(sum, off);
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    cursor[b0 + i] = off;
    off += v[i];
    hist[b0 + i] = 0u;
  }
}

__global__ void __launch_bounds__(128) order_scatter_kernel(const KParams P,
                                                            const uint16_t* __restrict__ bin,
                                                            unsigned* __restrict__ cursor,
                                                            int32_t* __restrict__ order) {
  const int64_t kl = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (kl >= P.k_count) return;
  order[atomicAdd(&cursor[bin[kl]], 1u)] = static_cast<int32_t>(kl);
}

}  // namespace

// Device scratch of the ordering pass for n candidates (bytes): bins (u16),
// histogram + cursors (u32), order (i32).
size_t order_scratch_bytes(int64_t n) {
  return 2 * sizeof(unsigned) * kBins + static_cast<size_t>(n) * (sizeof(uint16_t) + sizeof(int32_t)) + 64;
}

// scratch: order_scratch_bytes(n) bytes whose histogram part is zero (the
// scan re-zeroes it every cycle).  Writes the candidate order for the rollout
// kernel to *order_out.  Three launches.
cudaError_t launch_order(const KParams& P, const double* warm, void* scratch,
                         const int32_t** order_out, cudaStream_t stream) {
  const int64_t n = P.k_count;
  unsigned* hist = static_cast<unsigned*>(scratch);
  unsigned* cursor = hist + kBins;
  int32_t* order = reinterpret_cast<int32_t*>(cursor + kBins);
  uint16_t* bin = reinterpret_cast<uint16_t*>(order + n);
  const unsigned blocks = static_cast<unsigned>((n + 127) / 128);
  launch(order_key_kernel, blocks, 128, stream, P, warm, bin, hist);
  launch(order_scan_kernel, 1, kScanThreads, stream, hist, cursor);
  launch(order_scatter_kernel, blocks, 128, stream, P, bin, cursor, order);
  *order_out = order;
  return cudaGetLastError();
}

// Histogram part of the scratch that must be zero before the first cycle.
size_t order_hist_bytes() { return sizeof(unsigned) * kBins; }

}  // namespace tmpcb
