// MUFU.EX2 / FMA throughput probe: ops per clock per SM (nvcc -arch=sm_100a -O3 mufu_rate.cu)
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, int iters) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = -0.001f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      else if (MODE == 1) a[i] = fmaf(a[i], 0.999f, 0.001f);
      else { asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(*(unsigned*)&a[i]) : "f"(a[i]), "f"(a[(i + 1) & 15])); }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 12345.f) out[0] = s;
}
int main() {
  float* d; cudaMalloc(&d, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096, threads = 1024, blocks = sms * 2;
  const char* names[3] = {"ex2.approx.f32", "ffma", "cvt.bf16x2"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<blocks, threads>>>(d, iters);
      else if (mode == 1) k<1><<<blocks, threads>>>(d, iters);
      else k<2><<<blocks, threads>>>(d, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)blocks * threads * iters * 16;
      double per_clk_sm = ops / (ms * 1e-3) / (clk * 1e3) / sms;
      if (rep) printf("%-16s %.2f ms  %.1f ops/clk/SM (at %d MHz nominal)\n", names[mode], ms, per_clk_sm, clk / 1000);
    }
  }
  return 0;
}
