// FP32 FFMA throughput probe: the roofline denominator of the rollout kernel
// (FP32 SIMT bound).  MEASURED_PEAKS.json carries only HBM and
// bf16 tensor peaks, so bench.py measures the FP32 pipe on the same box.
#include <cuda_runtime.h>

#include "tmpc_b200.h"

namespace {

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void __launch_bounds__(256) ffma_probe(float* out, float a, float b) {
  float v[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) v[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) v[c] = fmaf(v[c], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += v[c];
  if (s == 12345.678f) out[0] = s;  // keep the chains alive
}

}  // namespace

extern "C" int tmpc_fp32_peak(int device, double* tflops) {
  if (cudaSetDevice(device) != cudaSuccess) return TMPC_ERR_RUNTIME;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  float* d = nullptr;
  if (cudaMalloc(&d, sizeof(float)) != cudaSuccess) return TMPC_ERR_RUNTIME;
  const int blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  ffma_probe<<<blocks, threads>>>(d, 0.999999f, 1e-7f);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    ffma_probe<<<blocks, threads>>>(d, 0.999999f, 1e-7f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  const cudaError_t err = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  if (err != cudaSuccess) return TMPC_ERR_RUNTIME;
  const double flops = 2.0 * kChains * kIters * static_cast<double>(blocks) * threads;
  *tflops = flops / (best * 1e-3) / 1e12;
  return TMPC_OK;
}
