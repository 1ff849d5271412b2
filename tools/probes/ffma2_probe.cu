// FFMA2 (packed fp32x2) vs FFMA issue rate / latency on sm_100a (dev probe).
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
  u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r;
}
__device__ __forceinline__ float ffma1(float a, float b, float c) {
  float r; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r;
}
template <int MODE>  // 0 scalar indep, 1 packed indep, 2 scalar chain, 3 packed chain
__global__ void k(float* out, long long* cyc, int iters) {
  float s[16]; u64 p[8];
  for (int i = 0; i < 16; ++i) s[i] = threadIdx.x * 0.001f + i;
  for (int i = 0; i < 8; ++i) p[i] = (u64)__float_as_uint(s[2*i]) | ((u64)__float_as_uint(s[2*i+1]) << 32);
  const float a = 0.999f, b = 0.001f;
  const u64 a2 = (u64)__float_as_uint(a) | ((u64)__float_as_uint(a) << 32);
  const u64 b2 = (u64)__float_as_uint(b) | ((u64)__float_as_uint(b) << 32);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) s[i] = ffma1(s[i], a, b);
    } else if (MODE == 1) {
#pragma unroll
      for (int i = 0; i < 8; ++i) p[i] = ffma2(p[i], a2, b2);
    } else if (MODE == 2) {
#pragma unroll
      for (int i = 0; i < 16; ++i) s[0] = ffma1(s[0], a, b);
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) p[0] = ffma2(p[0], a2, b2);
    }
  }
  long long t1 = clock64();
  float acc = 0;
  for (int i = 0; i < 16; ++i) acc += s[i];
  for (int i = 0; i < 8; ++i) acc += __uint_as_float((unsigned)p[i]) + __uint_as_float((unsigned)(p[i] >> 32));
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int M> void run(const char* name, int blocks, int threads) {
  float* o; long long* c; cudaMalloc(&o, blocks * threads * 4); cudaMalloc(&c, blocks * 8);
  const int iters = 4096;
  k<M><<<blocks, threads>>>(o, c, iters); cudaDeviceSynchronize();
  k<M><<<blocks, threads>>>(o, c, iters); cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  const double per = (double)h / iters / 16.0;  // cycles per (16 FMAs-or-chain-links) / 16
  printf("%-28s blocks %4d threads %4d: %.3f cycles per instruction-slot-of-work\n", name, blocks, threads, per);
  cudaFree(o); cudaFree(c);
}
int main() {
  run<0>("scalar FFMA x16 indep", 1, 32);
  run<1>("packed FFMA2 x8 indep", 1, 32);
  run<2>("scalar FFMA chain", 1, 32);
  run<3>("packed FFMA2 chain", 1, 32);
  run<0>("scalar FFMA x16 indep", 148, 128);
  run<1>("packed FFMA2 x8 indep", 148, 128);
  run<0>("scalar FFMA x16 indep", 148, 512);
  run<1>("packed FFMA2 x8 indep", 148, 512);
  return 0;
}
