// Deterministic substep (nsf_material.deterministic = 1): P2G reduced in 64-bit
// fixed point with integer atomics, so the grid, and hence the whole substep,
// is bitwise independent of the order in which particles are reduced (launch
// configuration, scheduling, binning).  Units: 2^-32 particle masses for the
// mass, 2^-32 particle-mass m/s for the momentum (each contribution is rounded
// once, then summed exactly; |values| < 2^31 units).  Same P2G arithmetic as
// k_p2g_direct (reading #1, Eq. (6)); grid update P:177.
#include <cuda_runtime.h>
#include <cstdint>
#include "kernels.h"
#include "pipeline.h"
#include "point_ops.cuh"

namespace nsf {

constexpr float kFx = 4294967296.0f;   // 2^32

__device__ __forceinline__ void det_touch(int* flags, int* list, int* list_count, int b) {
  if (flags[b] == 0 && atomicExch(&flags[b], 1) == 0) list[atomicAdd(list_count, 1)] = b;
}

__device__ __forceinline__ void fx_add(unsigned long long* a, float v) {
  atomicAdd(a, (unsigned long long)__float2ll_rn(v));   // two's complement: signed sums are exact
}

template <int FORCE>
__global__ void __launch_bounds__(128) k_p2g_fixed(int64_t n, const float* __restrict__ S,
                                                   const int64_t* __restrict__ scene_off, int n_scenes,
                                                   unsigned long long* __restrict__ fx, int* flags, int* list,
                                                   int* list_count, DevParams P) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int scene = scene_of(p, scene_off, n_scenes, n);
  float xp[3], vp[3], Cp[9], tp[6];
  nsf_load_point(S, p, xp, vp, Cp);
#pragma unroll
  for (int k = 0; k < 6; ++k) tp[k] = S[pbase(p) + (PT + k) * 32];
  Axis ax[3];
  int base[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    ax[a] = bspline_axis(xp[a], P.inv_dx);
    base[a] = ax[a].base = clamp_base(ax[a].base, P.N[a]);
  }
  const float m = P.mass;
  const float T[9] = {tp[0], tp[5], tp[4], tp[5], tp[1], tp[3], tp[4], tp[3], tp[2]};
  float Q[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) Q[k] = P.mC * Cp[k] - (FORCE == 0 ? P.mls_coef * T[k] : 0.0f);
  const float sm = kFx / m;   // momentum -> fixed point
  const int64_t so = (int64_t)scene * P.nodes_per_scene;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const float W = ax[0].w[a] * ax[1].w[b] * ax[2].w[c];
        const float d0 = ((float)a - ax[0].f) * P.dx, d1 = ((float)b - ax[1].f) * P.dx, d2 = ((float)c - ax[2].f) * P.dx;
        float mv0 = W * (m * vp[0] + Q[0] * d0 + Q[1] * d1 + Q[2] * d2);
        float mv1 = W * (m * vp[1] + Q[3] * d0 + Q[4] * d1 + Q[5] * d2);
        float mv2 = W * (m * vp[2] + Q[6] * d0 + Q[7] * d1 + Q[8] * d2);
        if (FORCE == 1) {
          const float g0 = ax[0].dw[a] * ax[1].w[b] * ax[2].w[c];
          const float g1 = ax[0].w[a] * ax[1].dw[b] * ax[2].w[c];
          const float g2 = ax[0].w[a] * ax[1].w[b] * ax[2].dw[c];
          mv0 -= P.gradw_coef * (T[0] * g0 + T[1] * g1 + T[2] * g2);
          mv1 -= P.gradw_coef * (T[3] * g0 + T[4] * g1 + T[5] * g2);
          mv2 -= P.gradw_coef * (T[6] * g0 + T[7] * g1 + T[8] * g2);
        }
        unsigned long long* nd = fx + 4 * (so + node_index(base[0] + a, base[1] + b, base[2] + c, P));
        fx_add(nd + 0, W * kFx);
        fx_add(nd + 1, mv0 * sm);
        fx_add(nd + 2, mv1 * sm);
        fx_add(nd + 3, mv2 * sm);
      }
  const int64_t sb = (int64_t)scene * P.blocks_per_scene;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int b0 = (base[0] + 2 * (k >> 2)) >> 2, b1 = (base[1] + 2 * ((k >> 1) & 1)) >> 2,
              b2 = (base[2] + 2 * (k & 1)) >> 2;
    det_touch(flags, list, list_count, (int)(sb + block_id(b0, b1, b2, P)));
  }
}

// Grid update of the touched blocks from the fixed-point accumulator (one warp
// per block); the accumulator, the flags and the list are reset.
__global__ void __launch_bounds__(128) k_grid_update_fixed(int* __restrict__ flags, const int* __restrict__ list,
                                                           int* __restrict__ list_count, int* __restrict__ done,
                                                           unsigned long long* __restrict__ fx,
                                                           float4* __restrict__ vel, DevParams P,
                                                           const int64_t* __restrict__ d_step) {
  const int nl = *(volatile int*)list_count;
  const int lane = threadIdx.x & 31;
  const int warp = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nwarps = (int)(((int64_t)gridDim.x * blockDim.x) >> 5);
  const float y_pl = plate_y(P, *d_step);
  const int bps = (int)P.blocks_per_scene;
  const float unit = P.mass / kFx;
  for (int e = warp; e < nl; e += nwarps) {
    const int key = list[e];
    const int scene = key / bps, local = key - scene * bps;
    const int plane = P.NB[1] * P.NB[2];
    const int b0 = local / plane, b1 = (local - b0 * plane) / P.NB[2], b2 = local - b0 * plane - b1 * P.NB[2];
    const int64_t gb = (int64_t)scene * P.nodes_per_scene + (int64_t)local * kBlockNodes;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int l = lane + 32 * h;
      unsigned long long* nd = fx + 4 * (gb + l);
      const float4 a = make_float4((float)(long long)nd[0] * unit, (float)(long long)nd[1] * unit,
                                   (float)(long long)nd[2] * unit, (float)(long long)nd[3] * unit);
      nd[0] = nd[1] = nd[2] = nd[3] = 0ull;
      const int i = 4 * b0 + (l >> 4), j = 4 * b1 + ((l >> 2) & 3), k = 4 * b2 + (l & 3);
      vel[gb + l] = grid_node_update(a, i, j, k, P, y_pl);
    }
    if (lane == 0) flags[key] = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(done, 1) == (int)gridDim.x - 1) {
      *list_count = 0;
      *done = 0;
    }
  }
}

void launch_p2g_fixed(cudaStream_t st, int64_t n, const float* S, const int64_t* scene_off, int n_scenes,
                      unsigned long long* fx, PipelineBuffers* pb, const DevParams& P) {
  if (n == 0) return;
  const unsigned g = (unsigned)((n + 127) / 128);
  int* list = pb->touched;
  int* count = pb->touched + pb->total_blocks;
  if (P.force_mode == 0) k_p2g_fixed<0><<<g, 128, 0, st>>>(n, S, scene_off, n_scenes, fx, pb->flags, list, count, P);
  else k_p2g_fixed<1><<<g, 128, 0, st>>>(n, S, scene_off, n_scenes, fx, pb->flags, list, count, P);
}

void launch_grid_update_fixed(cudaStream_t st, PipelineBuffers* pb, unsigned long long* fx, float4* vel,
                              const DevParams& P, const int64_t* d_step) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  k_grid_update_fixed<<<sms * 8, 128, 0, st>>>(pb->flags, pb->touched, pb->touched + pb->total_blocks,
                                               pb->touched + pb->total_blocks + 1, fx, vel, P, d_step);
}

}  // namespace nsf
