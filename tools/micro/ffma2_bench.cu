// Microbenchmark: throughput of FFMA vs FFMA2 (fma.rn.f32x2, sm_100a) per SM.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 f2(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
template <int ILP>
__global__ void k_ffma(float* out, int iters, float s) {
  float a[ILP];
  for (int i = 0; i < ILP; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = fmaf(a[i], s, 0.5f * s + i);
  float t = 0; for (int i = 0; i < ILP; ++i) t += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int ILP>
__global__ void k_ffma2(float* out, int iters, float s) {
  u64 a[ILP]; float2 ss = make_float2(s, s); float2 cc = make_float2(0.5f * s, 0.25f * s);
  u64 S = *(u64*)&ss, Cc = *(u64*)&cc;
  for (int i = 0; i < ILP; ++i) { float2 v = make_float2(threadIdx.x * 1e-3f + i, i); a[i] = *(u64*)&v; }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = f2(a[i], S, Cc);
  float t = 0; for (int i = 0; i < ILP; ++i) { float2 v = *(float2*)&a[i]; t += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 1024 * 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 4096; const int thr = 512, blocks = sms * 4;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(a); k_ffma<8><<<blocks, thr>>>(out, iters, 0.999f); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    double fmas = (double)blocks * thr * iters * 8;
    printf("FFMA : %.3f ms  %.1f TFMA/s  warp-instr/clk/SM(at 1.965GHz) %.2f\n", ms, fmas / ms / 1e9, fmas / 32 / (ms * 1e-3) / sms / 1.965e9);
    cudaEventRecord(a); k_ffma2<8><<<blocks, thr>>>(out, iters, 0.999f); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    fmas = (double)blocks * thr * iters * 8 * 2;
    printf("FFMA2: %.3f ms  %.1f TFMA/s  warp-instr/clk/SM(at 1.965GHz) %.2f\n", ms, fmas / ms / 1e9, fmas / 64 / (ms * 1e-3) / sms / 1.965e9);
  }
  return 0;
}
