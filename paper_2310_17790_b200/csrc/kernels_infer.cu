// Network inference and the sample / integration particle sets of the reduced
// model (§5.1, §5.4); the MLP passes
// themselves run in kernels_nsf_tc.cu / kernels_nsf_simt.cu.
//
//   infer : x = g(X, z_n) and g(X, z_{n-1}) into the store's x / v planes, then
//           v = (x - v) / dt (k_backdiff); C = l(X, z_n) into the C planes
//   sets  : per scene, I = stencil nodes of the samples' g(X_S, z_n) as a bit
//           mask over the scene's grid (k_mark_stencils); N = reference points whose
//           stencil at g(X_p, z_n) hits I, minus S (k_member_flags), compacted in
//           index order (k_count_block, k_scene_scan, k_compact_block: the order
//           is deterministic, offsets carried on the device across scenes); the
//           new points are S then N \ S.
#include <cuda_runtime.h>
#include <cstdint>
#include "kernels.h"
#include "params.cuh"

namespace nsf {

__global__ void k_latent_at(int64_t m, const float* __restrict__ z, const float* __restrict__ dz, int64_t step,
                            float* __restrict__ out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < m) out[e] = z[e] + (float)step * (dz ? dz[e] : 0.0f);   // the MLP kernels' z(n)
}

void launch_latent_at(cudaStream_t st, int64_t m, const float* z, const float* dz, int64_t step, float* out) {
  if (m <= 0) return;
  k_latent_at<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(m, z, dz, step, out);
}

// v = (x - v) / dt on the store planes (v holds g(X, z_{n-1}) on entry)
__global__ void k_backdiff(int64_t n, float* __restrict__ S, float inv_dt) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  float* b = S + pbase(p);
#pragma unroll
  for (int a = 0; a < 3; ++a) b[(PV + a) * 32] = (b[(PX + a) * 32] - b[(PV + a) * 32]) * inv_dt;
}

void launch_backdiff(cudaStream_t st, int64_t n, float* S, float dt) {
  if (n <= 0) return;
  k_backdiff<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, S, 1.0f / dt);
}

__device__ __forceinline__ bool stencil_base(const float* x, const DevParams& P, int b[3]) {
  bool ok = true;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    b[a] = (int)floorf(x[a] * P.inv_dx - 0.5f);
    ok &= b[a] >= 0 && b[a] + 2 < P.N[a];
  }
  return ok;
}

__device__ __forceinline__ int64_t lin_node(int i, int j, int k, const DevParams& P) {
  return ((int64_t)i * P.N[1] + j) * P.N[2] + k;
}

// I: bit (i N1 + j) N2 + k of `mask` for every stencil node of the samples x[idx[q]]
// (x AoS m x 3); samples whose stencil leaves the grid flag ERR_OUT_OF_DOMAIN
__global__ void k_mark_stencils(int n_sample, const int32_t* __restrict__ idx, const float* __restrict__ x,
                                uint32_t* __restrict__ mask, DevParams P, DevErr* err) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n_sample) return;
  const float* xp = x + 3 * (int64_t)idx[q];
  int b[3];
  if (!stencil_base(xp, P, b)) {
    atomicOr(&err->bits, ERR_OUT_OF_DOMAIN);
    return;
  }
  for (int o = 0; o < 27; ++o) {
    const int64_t id = lin_node(b[0] + o / 9, b[1] + (o / 3) % 3, b[2] + o % 3, P);
    atomicOr(&mask[id >> 5], 1u << (id & 31));
  }
}

// flag[p] = 1 if point p's stencil at x[p] hits I and p is not a sample
__global__ void k_member_flags(int64_t n_ref, const float* __restrict__ x, const uint32_t* __restrict__ mask,
                               const uint8_t* __restrict__ is_sample, uint8_t* __restrict__ flag, DevParams P) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n_ref) return;
  int b[3];
  bool hit = false;
  if (stencil_base(x + 3 * p, P, b)) {
    for (int o = 0; o < 27 && !hit; ++o) {
      const int64_t id = lin_node(b[0] + o / 9, b[1] + (o / 3) % 3, b[2] + o % 3, P);
      hit = (mask[id >> 5] >> (id & 31)) & 1u;
    }
  }
  flag[p] = (hit && !is_sample[p]) ? 1 : 0;
}

__global__ void k_set_samples(int n_sample, const int32_t* __restrict__ idx, uint8_t* __restrict__ is_sample,
                              uint8_t v) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n_sample) is_sample[idx[q]] = v;
}

constexpr int kCompactBlock = 1024;

// per 1024-point block: number of flagged points
__global__ void __launch_bounds__(kCompactBlock) k_count_block(int64_t n, const uint8_t* __restrict__ flag,
                                                               int32_t* __restrict__ cnt) {
  const int64_t p = blockIdx.x * (int64_t)kCompactBlock + threadIdx.x;
  const int f = p < n ? flag[p] : 0;
  const int c = __syncthreads_count(f);
  if (threadIdx.x == 0) cnt[blockIdx.x] = c;
}

// out[base[block] + rank] = p for flagged p, in index order (block-local ranks by
// warp ballots, then the warps' prefix)
__global__ void __launch_bounds__(kCompactBlock) k_compact_block(int64_t n, const uint8_t* __restrict__ flag,
                                                                 const int32_t* __restrict__ base,
                                                                 int32_t* __restrict__ out) {
  __shared__ int wsum[kCompactBlock / 32];
  const int64_t p = blockIdx.x * (int64_t)kCompactBlock + threadIdx.x;
  const bool f = p < n && flag[p];
  const unsigned bal = __ballot_sync(0xffffffffu, f);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) wsum[warp] = __popc(bal);
  __syncthreads();
  int off = 0;
  for (int w = 0; w < warp; ++w) off += wsum[w];
  if (f) out[base[blockIdx.x] + off + __popc(bal & ((1u << lane) - 1))] = (int32_t)p;
}

// per scene, on the device (no host round trip): the scene's points start at *cursor
// (samples first), the flagged points of block k at base[k]; *cursor advances by
// the scene's count, which is also written to scene_count[scene]
__global__ void __launch_bounds__(kCompactBlock) k_scene_scan(int64_t nblk, const int32_t* __restrict__ cnt,
                                                              int n_sample, int64_t* __restrict__ cursor,
                                                              int32_t* __restrict__ base,
                                                              int64_t* __restrict__ scene_count, int scene,
                                                              int64_t* __restrict__ sample_base) {
  __shared__ int64_t carry;
  __shared__ int64_t wsum[kCompactBlock / 32];
  const int64_t c0 = *cursor;
  if (threadIdx.x == 0) carry = c0 + n_sample;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t k0 = 0; k0 < nblk; k0 += kCompactBlock) {
    const int64_t k = k0 + threadIdx.x;
    const int64_t c = k < nblk ? cnt[k] : 0;
    int64_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int64_t woff = 0;
    for (int w = 0; w < warp; ++w) woff += wsum[w];
    if (k < nblk) base[k] = (int32_t)(carry + woff + incl - c);
    __syncthreads();
    if (threadIdx.x == kCompactBlock - 1) carry += woff + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    scene_count[scene] = carry - c0;
    *sample_base = c0;
    *cursor = carry;
  }
}

// list[*sample_base + q] = sample_idx[q]
__global__ void k_put_samples(int n_sample, const int32_t* __restrict__ idx, const int64_t* __restrict__ sample_base,
                              int32_t* __restrict__ list) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n_sample) list[*sample_base + q] = idx[q];
}

void launch_scene_scan(cudaStream_t st, int64_t nblk, const int32_t* cnt, int n_sample, int64_t* cursor,
                       int32_t* base, int64_t* scene_count, int scene, int64_t* sample_base) {
  k_scene_scan<<<1, kCompactBlock, 0, st>>>(nblk, cnt, n_sample, cursor, base, scene_count, scene, sample_base);
}

void launch_put_samples(cudaStream_t st, int n_sample, const int32_t* idx, const int64_t* sample_base,
                        int32_t* list) {
  if (n_sample <= 0) return;
  k_put_samples<<<(n_sample + 127) / 128, 128, 0, st>>>(n_sample, idx, sample_base, list);
}

// X_new[j] = X_all[list[j]] (AoS 3)
__global__ void k_gather_rows3(int64_t m, const int32_t* __restrict__ list, const float* __restrict__ X_all,
                               float* __restrict__ X_new) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= m) return;
  const int64_t p = list[j];
#pragma unroll
  for (int a = 0; a < 3; ++a) X_new[3 * j + a] = X_all[3 * p + a];
}

void launch_mark_stencils(cudaStream_t st, int n_sample, const int32_t* idx, const float* x, uint32_t* mask,
                          const DevParams& P, DevErr* err) {
  if (n_sample <= 0) return;
  k_mark_stencils<<<(n_sample + 127) / 128, 128, 0, st>>>(n_sample, idx, x, mask, P, err);
}

void launch_member_flags(cudaStream_t st, int64_t n_ref, const float* x, const uint32_t* mask,
                         const uint8_t* is_sample, uint8_t* flag, const DevParams& P) {
  if (n_ref <= 0) return;
  k_member_flags<<<(unsigned)((n_ref + 255) / 256), 256, 0, st>>>(n_ref, x, mask, is_sample, flag, P);
}

void launch_set_samples(cudaStream_t st, int n_sample, const int32_t* idx, uint8_t* is_sample, uint8_t v) {
  if (n_sample <= 0) return;
  k_set_samples<<<(n_sample + 127) / 128, 128, 0, st>>>(n_sample, idx, is_sample, v);
}

int64_t compact_blocks(int64_t n) { return (n + kCompactBlock - 1) / kCompactBlock; }

void launch_count_blocks(cudaStream_t st, int64_t n, const uint8_t* flag, int32_t* cnt) {
  if (n <= 0) return;
  k_count_block<<<(unsigned)compact_blocks(n), kCompactBlock, 0, st>>>(n, flag, cnt);
}

void launch_compact(cudaStream_t st, int64_t n, const uint8_t* flag, const int32_t* base, int32_t* out) {
  if (n <= 0) return;
  k_compact_block<<<(unsigned)compact_blocks(n), kCompactBlock, 0, st>>>(n, flag, base, out);
}

void launch_gather_rows3(cudaStream_t st, int64_t m, const int32_t* list, const float* X_all, float* X_new) {
  if (m <= 0) return;
  k_gather_rows3<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(m, list, X_all, X_new);
}

}  // namespace nsf
