// Neural stress field h(X, z) (architecture P:498-500) on
// CUDA cores: the reference-layout kernel used for eval_stress_field and for
// widths the tensor-core kernel (kernels_nsf_tc.cu) does not cover.
// Numerics (reading #20): layer-1 input fp32; W bf16; activations rounded to
// bf16 (RNE) before layers 2..L+1; fp32 accumulate; bias + ELU in fp32.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include "kernels.h"
#include "point_ops.cuh"

namespace nsf {

constexpr int kTile = 128;        // points per CTA tile (one per thread)
constexpr int kMaxWidth = 128;
constexpr int kMaxOut = 16;       // output width (stress 6, deformation 3, affine velocity 9)

__device__ __forceinline__ float bf16_bits_to_f32(uint16_t b) { return __uint_as_float(((uint32_t)b) << 16); }

__device__ __forceinline__ float elu(float a) { return a > 0.0f ? a : expm1f(a); }

// dynamic smem: weights transposed [in][out] as bf16 for every layer, then two
// activation buffers [width][kTile] bf16
__global__ void __launch_bounds__(kTile) k_nsf_mlp_simt(int64_t n, const float* __restrict__ X, int64_t xpitch,
                                                        const int64_t* __restrict__ scene_off, int n_scenes,
                                                        const float* __restrict__ z, const float* __restrict__ dz,
                                                        int r, const int64_t* __restrict__ d_step, MlpDev mlp,
                                                        float stress_scale, float* __restrict__ tau_out,
                                                        int64_t tau_pitch, int aos_out, NsfP2G q) {
  extern __shared__ __align__(16) uint16_t sm[];
  const int L = mlp.n_hidden + 1;   // number of linear layers
  const int width = mlp.width;
  // stage transposed weights
  int64_t total_w = mlp.w_off[L];
  for (int64_t e = threadIdx.x; e < total_w; e += blockDim.x) {
    int layer = 0;
    while (e >= mlp.w_off[layer + 1]) ++layer;
    int in = layer == 0 ? mlp.in_dim : width;
    int out = layer == L - 1 ? mlp.out_dim : width;
    int64_t loc = e - mlp.w_off[layer];
    int o = (int)(loc / in), i = (int)(loc % in);
    sm[mlp.w_off[layer] + (int64_t)i * out + o] = mlp.W[e];
  }
  uint16_t* hA = sm + ((total_w + 7) & ~7ll);
  uint16_t* hB = hA + kMaxWidth * kTile;
  __syncthreads();
  const int64_t step = d_step ? *d_step : 0;
  const int t = threadIdx.x;
  for (int64_t tile0 = (int64_t)blockIdx.x * kTile; tile0 < n; tile0 += (int64_t)gridDim.x * kTile) {
    int64_t p = tile0 + t;
    bool live = p < n;
    float u[16];
    const int scene = live ? scene_of(p, scene_off, n_scenes, n) : 0;
#pragma unroll
    for (int a = 0; a < 16; ++a) u[a] = 0.0f;
    if (live) {
      if (xpitch >= 0) {
        u[0] = X[0 * xpitch + p];
        u[1] = X[1 * xpitch + p];
        u[2] = X[2 * xpitch + p];
      } else {   // AoSoA planes of the particle store
        u[0] = X[pbase(p) + 0 * 32];
        u[1] = X[pbase(p) + 1 * 32];
        u[2] = X[pbase(p) + 2 * 32];
      }
      for (int k = 0; k < r; ++k)
        u[3 + k] = z[scene * r + k] + (float)step * (dz ? dz[scene * r + k] : 0.0f);
    }
    // layer 1 (fp32 inputs)
    {
      const uint16_t* Wt = sm + mlp.w_off[0];
      const float* b = mlp.b + mlp.b_off[0];
      for (int j = 0; j < width; ++j) {
        float a = b[j];
        for (int i = 0; i < mlp.in_dim; ++i) a = fmaf(bf16_bits_to_f32(Wt[i * width + j]), u[i], a);
        a = elu(a);
        __nv_bfloat16 hb = __float2bfloat16_rn(a);
        hA[j * kTile + t] = *reinterpret_cast<uint16_t*>(&hb);
      }
    }
    __syncthreads();
    // hidden layers 2..n_hidden
    for (int layer = 1; layer < L - 1; ++layer) {
      const uint16_t* Wt = sm + mlp.w_off[layer];
      const float* b = mlp.b + mlp.b_off[layer];
      float acc[kMaxWidth];
#pragma unroll
      for (int j = 0; j < kMaxWidth; ++j) acc[j] = (j < width) ? b[j] : 0.0f;
      for (int k = 0; k < width; ++k) {
        float hk = bf16_bits_to_f32(hA[k * kTile + t]);
        const uint4* wrow = reinterpret_cast<const uint4*>(Wt + k * width);
#pragma unroll
        for (int j8 = 0; j8 < kMaxWidth / 8; ++j8) {
          if (j8 * 8 < width) {
            uint4 wv = wrow[j8];
            uint32_t wa[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              acc[j8 * 8 + 2 * q] = fmaf(__uint_as_float(wa[q] << 16), hk, acc[j8 * 8 + 2 * q]);
              acc[j8 * 8 + 2 * q + 1] = fmaf(__uint_as_float(wa[q] & 0xffff0000u), hk, acc[j8 * 8 + 2 * q + 1]);
            }
          }
        }
      }
#pragma unroll
      for (int j = 0; j < kMaxWidth; ++j) {
        if (j < width) {
          __nv_bfloat16 hb = __float2bfloat16_rn(elu(acc[j]));
          hB[j * kTile + t] = *reinterpret_cast<uint16_t*>(&hb);
        }
      }
      __syncthreads();
      uint16_t* tmp = hA; hA = hB; hB = tmp;
    }
    // output layer
    {
      const uint16_t* Wt = sm + mlp.w_off[L - 1];
      const float* b = mlp.b + mlp.b_off[L - 1];
      float y[kMaxOut];
#pragma unroll
      for (int o = 0; o < kMaxOut; ++o) y[o] = (o < mlp.out_dim) ? b[o] : 0.0f;
      for (int k = 0; k < width; ++k) {
        float hk = bf16_bits_to_f32(hA[k * kTile + t]);
#pragma unroll
        for (int o = 0; o < kMaxOut; ++o)
          if (o < mlp.out_dim) y[o] = fmaf(bf16_bits_to_f32(Wt[k * mlp.out_dim + o]), hk, y[o]);
      }
      if (live) {
        float tau[kMaxOut];
#pragma unroll
        for (int o = 0; o < kMaxOut; ++o) tau[o] = stress_scale * y[o];
        for (int o = 0; o < mlp.out_dim; ++o) {
          if (aos_out) tau_out[p * mlp.out_dim + o] = tau[o];
          else tau_out[pbase(p) + o * 32] = tau[o];   // AoSoA particle store
        }
        if (q.enabled) {   // reduced P2G
          float xp[3], vp[3], Cp[9];
          nsf_load_point(q.S, p, xp, vp, Cp);
          nsf_p2g_point(q, scene, xp, vp, Cp, tau, step);
        }
      }
    }
    __syncthreads();
  }
}

void launch_nsf_mlp(cudaStream_t st, int64_t n, const float* X, int64_t xpitch, const int64_t* scene_off,
                    int n_scenes, const float* z, const float* dz, int r, const int64_t* d_step,
                    const MlpDev& mlp, float stress_scale, float* tau_out, int64_t tau_pitch, int aos_out,
                    const NsfP2G* qp) {
  if (n == 0) return;
  NsfP2G q{};
  if (qp) q = *qp;
  static int force_simt = -1;
  if (force_simt < 0) {
    const char* e = getenv("NSF_MLP_SIMT");
    force_simt = (e && atoi(e) != 0) ? 1 : 0;
  }
  if (!force_simt && nsf_mlp_tc_supported(mlp)) {
    launch_nsf_mlp_tc(st, n, X, xpitch, scene_off, n_scenes, z, dz, r, d_step, mlp, stress_scale, tau_out, aos_out,
                      qp);
    return;
  }
  int L = mlp.n_hidden + 1;
  size_t wbytes = (size_t)((mlp.w_off[L] + 7) & ~7ll) * 2;
  size_t smem = wbytes + 2 * (size_t)kMaxWidth * kTile * 2;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_nsf_mlp_simt, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr_set = true;
  }
  int64_t tiles = (n + kTile - 1) / kTile;
  int grid = (int)(tiles < 148 ? tiles : 148);
  k_nsf_mlp_simt<<<grid, kTile, smem, st>>>(n, X, xpitch, scene_off, n_scenes, z, dz, r, d_step, mlp,
                                            stress_scale, tau_out, tau_pitch, aos_out, q);
}

}  // namespace nsf
