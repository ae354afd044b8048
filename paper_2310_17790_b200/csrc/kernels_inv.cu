// Network inversion (§5.3, Eq. (10)): per scene,
//   z <- argmin_z sum_{p in S} || g(X_p, z) - x_p ||^2
// by Gauss-Newton from the current latent.  g is the neural deformation field
// (lines 204-209, architecture lines 498-500) with the stress field's numerics
// (reading #20: bf16 weights, layer-1 input fp32, activations rounded to bf16
// before each later layer, fp32 accumulation, bias and ELU).
//
// Jacobian dg/dz by forward mode, evaluated as extra rows of the same MLP pass:
// a tile holds 128 rows = (128 / rp) points x rp rows, rp = next power of two
// >= 1 + r; row 0 of a point is the primal (input (X, z)), row 1 + k the tangent
// of z_k (input e_{3+k}, no bias); rows beyond r are padding.  After each hidden
// layer the primal row publishes ELU'(a) (fp32) and the tangent rows multiply by
// it; tangents are rounded to bf16 at the same points as activations.
// Per point, J^T J and J^T (g - x) are reduced in fp64 into per-scene
// accumulators; one thread per scene then solves the r x r normal equations
// (Cholesky, fp64) and updates z.  Sample set S of a scene: its first n_sample
// points in load order (found through ids, since the store is reordered).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include "kernels.h"
#include "params.cuh"

namespace nsf {

namespace inv {
constexpr int kRows = 128;        // rows per tile (threads per CTA)
constexpr int kMaxWidth = 128;

__device__ __forceinline__ float bf(uint16_t b) { return __uint_as_float(((uint32_t)b) << 16); }
__device__ __forceinline__ uint16_t to_bf(float x) {
  __nv_bfloat16 h = __float2bfloat16_rn(x);
  return *reinterpret_cast<uint16_t*>(&h);
}
}  // namespace inv

// sample slot of (scene s, load-order index i < n_sample), -1 if the scene is smaller
__global__ void k_gn_samples(int64_t n, const int32_t* __restrict__ ids, const int64_t* __restrict__ scene_off,
                             int n_scenes, int n_sample, int32_t* __restrict__ slots) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int id = ids[j];
  int lo = 0, hi = n_scenes;   // scene of load index id (scenes are contiguous in both orders)
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (scene_off[mid] <= id) lo = mid; else hi = mid;
  }
  const int64_t i = id - scene_off[lo];
  if (i < n_sample) slots[(int64_t)lo * n_sample + i] = (int32_t)j;
}

// z_work = z + step dz (the latent the reduced substep of this step used)
__global__ void k_gn_zcur(int nz, const float* __restrict__ z, const float* __restrict__ dz,
                          const int64_t* __restrict__ d_step, float* __restrict__ zw) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nz) zw[i] = z[i] + (float)(*d_step) * (dz ? dz[i] : 0.0f);
}

__global__ void __launch_bounds__(inv::kRows) k_gn_accumulate(int n_scenes, int n_sample, int r, int rp,
                                                              const int32_t* __restrict__ slots,
                                                              const float* __restrict__ S,
                                                              const float* __restrict__ zw, MlpDev g,
                                                              double* __restrict__ accum) {
  using namespace inv;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int L = g.n_hidden + 1;
  const int width = g.width;
  const int64_t total_w = g.w_off[L];
  uint16_t* Wt = reinterpret_cast<uint16_t*>(smraw);                       // [layer][in][out] bf16
  uint16_t* hA = Wt + ((total_w + 7) & ~7ll);                              // [width][kRows]
  uint16_t* hB = hA + kMaxWidth * kRows;
  float* dbuf = reinterpret_cast<float*>(hB + kMaxWidth * kRows);          // [points][width]
  float* outb = dbuf + (kRows / 2) * kMaxWidth;                            // [kRows][4]
  const int t = threadIdx.x;
  for (int64_t e = t; e < total_w; e += kRows) {
    int layer = 0;
    while (e >= g.w_off[layer + 1]) ++layer;
    const int in = layer == 0 ? g.in_dim : width;
    const int out = layer == L - 1 ? g.out_dim : width;
    const int64_t loc = e - g.w_off[layer];
    const int o = (int)(loc / in), i = (int)(loc % in);
    Wt[g.w_off[layer] + (int64_t)i * out + o] = g.W[e];
  }
  __syncthreads();
  const int ppt = kRows / rp;                    // points per tile
  const int point = t / rp, k = t % rp;          // k = 0 primal, 1..r tangent of z_{k-1}
  const bool primal = k == 0, tangent = k >= 1 && k <= r;
  const int64_t n_pts = (int64_t)n_scenes * n_sample;
  const int nterm = r * (r + 1) / 2 + r;
  for (int64_t t0 = (int64_t)blockIdx.x * ppt; t0 < n_pts; t0 += (int64_t)gridDim.x * ppt) {
    const int64_t e = t0 + point;
    const int scene = e < n_pts ? (int)(e / n_sample) : 0;
    const int slot = e < n_pts ? slots[e] : -1;
    const bool live = slot >= 0;
    float xt[3] = {0.f, 0.f, 0.f};
    float u[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) u[i] = 0.0f;
    if (live) {
      if (primal) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          u[a] = S[pbase(slot) + (PXR + a) * 32];
          xt[a] = S[pbase(slot) + (PX + a) * 32];
        }
        for (int q = 0; q < r && q < 13; ++q) u[3 + q] = zw[scene * r + q];
      } else if (tangent) {
        u[3 + (k - 1)] = 1.0f;
      }
    }
    const float bsc = primal ? 1.0f : 0.0f;      // tangents carry no bias
    uint16_t* hin = hA;
    uint16_t* hout = hB;
    // ---- layers 1 .. L-1 (ELU) ----
    for (int layer = 0; layer < L - 1; ++layer) {
      const uint16_t* W = Wt + g.w_off[layer];
      const float* b = g.b + g.b_off[layer];
      float acc[kMaxWidth];
#pragma unroll
      for (int j = 0; j < kMaxWidth; ++j) acc[j] = (j < width) ? bsc * b[j] : 0.0f;
      if (layer == 0) {
        for (int i = 0; i < g.in_dim; ++i) {
          const float ui = u[i];
          if (ui == 0.0f) continue;
#pragma unroll
          for (int j = 0; j < kMaxWidth; ++j)
            if (j < width) acc[j] = fmaf(bf(W[i * width + j]), ui, acc[j]);
        }
      } else {
        for (int q = 0; q < width; ++q) {
          const float hk = bf(hin[q * kRows + t]);
          const uint4* wrow = reinterpret_cast<const uint4*>(W + q * width);   // 8 bf16 per load (broadcast)
#pragma unroll
          for (int j8 = 0; j8 < kMaxWidth / 8; ++j8) {
            if (j8 * 8 < width) {
              const uint4 wv = wrow[j8];
              const uint32_t wa[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                acc[j8 * 8 + 2 * c] = fmaf(__uint_as_float(wa[c] << 16), hk, acc[j8 * 8 + 2 * c]);
                acc[j8 * 8 + 2 * c + 1] = fmaf(__uint_as_float(wa[c] & 0xffff0000u), hk, acc[j8 * 8 + 2 * c + 1]);
              }
            }
          }
        }
      }
      // primal: ELU and ELU'(a) for the point's tangent rows
      if (primal) {
#pragma unroll
        for (int j = 0; j < kMaxWidth; ++j) {
          if (j < width) {
            const float a = acc[j];
            hout[j * kRows + t] = to_bf(a > 0.0f ? a : expm1f(a));
            dbuf[point * kMaxWidth + j] = a > 0.0f ? 1.0f : expf(a);
          }
        }
      }
      __syncthreads();
      if (!primal) {
#pragma unroll
        for (int j = 0; j < kMaxWidth; ++j)
          if (j < width) hout[j * kRows + t] = to_bf(tangent ? dbuf[point * kMaxWidth + j] * acc[j] : 0.0f);
      }
      __syncthreads();
      uint16_t* tmp = hin;
      hin = hout;
      hout = tmp;
    }
    // ---- output layer (linear, out_dim = 3) ----
    {
      const uint16_t* W = Wt + g.w_off[L - 1];
      const float* b = g.b + g.b_off[L - 1];
      float y[3] = {bsc * b[0], bsc * b[1], bsc * b[2]};
      for (int q = 0; q < width; ++q) {
        const float hk = bf(hin[q * kRows + t]);
#pragma unroll
        for (int o = 0; o < 3; ++o) y[o] = fmaf(bf(W[q * 3 + o]), hk, y[o]);
      }
#pragma unroll
      for (int o = 0; o < 3; ++o) outb[t * 4 + o] = y[o];
    }
    __syncthreads();
    // ---- per point: J^T J and J^T (g - x) into the scene's fp64 accumulators ----
    if (primal && live) {
      double res[3], J[3][13];
#pragma unroll
      for (int o = 0; o < 3; ++o) res[o] = (double)outb[t * 4 + o] - (double)xt[o];
      for (int q = 0; q < r; ++q)
#pragma unroll
        for (int o = 0; o < 3; ++o) J[o][q] = (double)outb[(t + 1 + q) * 4 + o];
      double* A = accum + (int64_t)scene * nterm;
      int idx = 0;
      for (int a = 0; a < r; ++a)
        for (int c = a; c < r; ++c, ++idx)
          atomicAdd(A + idx, J[0][a] * J[0][c] + J[1][a] * J[1][c] + J[2][a] * J[2][c]);
      for (int a = 0; a < r; ++a) atomicAdd(A + idx + a, J[0][a] * res[0] + J[1][a] * res[1] + J[2][a] * res[2]);
    }
    __syncthreads();
  }
}

// one thread per scene: solve (J^T J) dz = J^T res (Cholesky, fp64), z <- z - dz;
// the accumulators are cleared for the next iteration
__global__ void k_gn_solve(int n_scenes, int r, double* __restrict__ accum, float* __restrict__ zw) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_scenes) return;
  const int nterm = r * (r + 1) / 2 + r;
  double* A = accum + (int64_t)s * nterm;
  double H[13][13], gv[13], Lm[13][13];
  int idx = 0;
  for (int a = 0; a < r; ++a)
    for (int c = a; c < r; ++c, ++idx) H[a][c] = H[c][a] = A[idx];
  for (int a = 0; a < r; ++a) gv[a] = A[idx + a];
  bool ok = true;
  for (int i = 0; i < r && ok; ++i) {
    for (int j = 0; j <= i; ++j) {
      double sum = H[i][j];
      for (int q = 0; q < j; ++q) sum -= Lm[i][q] * Lm[j][q];
      if (i == j) {
        if (!(sum > 0.0)) { ok = false; break; }
        Lm[i][i] = sqrt(sum);
      } else {
        Lm[i][j] = sum / Lm[j][j];
      }
    }
  }
  if (ok) {
    double y[13], dzv[13];
    for (int i = 0; i < r; ++i) {
      double sum = gv[i];
      for (int q = 0; q < i; ++q) sum -= Lm[i][q] * y[q];
      y[i] = sum / Lm[i][i];
    }
    for (int i = r - 1; i >= 0; --i) {
      double sum = y[i];
      for (int q = i + 1; q < r; ++q) sum -= Lm[q][i] * dzv[q];
      dzv[i] = sum / Lm[i][i];
    }
    for (int i = 0; i < r; ++i) zw[s * r + i] = (float)((double)zw[s * r + i] - dzv[i]);
  }
  for (int i = 0; i < nterm; ++i) A[i] = 0.0;
}

size_t gn_smem_bytes(const MlpDev& g) {
  const int L = g.n_hidden + 1;
  return (size_t)((g.w_off[L] + 7) & ~7ll) * 2 + 2 * (size_t)inv::kMaxWidth * inv::kRows * 2 +
         (size_t)(inv::kRows / 2) * inv::kMaxWidth * 4 + (size_t)inv::kRows * 4 * 4;
}

void launch_gn_invert(cudaStream_t st, int64_t n, const int32_t* ids, const int64_t* scene_off, int n_scenes,
                      int n_sample, int r, const float* S, const float* z, const float* dz, const int64_t* d_step,
                      const MlpDev& g, int n_iters, int32_t* slots, float* zw, double* accum) {
  const int nz = n_scenes * r;
  cudaMemsetAsync(slots, 0xff, sizeof(int32_t) * (size_t)n_scenes * n_sample, st);
  cudaMemsetAsync(accum, 0, sizeof(double) * (size_t)n_scenes * (r * (r + 1) / 2 + r), st);
  if (n > 0) k_gn_samples<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, ids, scene_off, n_scenes, n_sample, slots);
  k_gn_zcur<<<(nz + 127) / 128, 128, 0, st>>>(nz, z, dz, d_step, zw);
  int rp = 1;
  while (rp < 1 + r) rp <<= 1;
  const size_t smem = gn_smem_bytes(g);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_gn_accumulate, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = ((int64_t)n_scenes * n_sample + (inv::kRows / rp) - 1) / (inv::kRows / rp);
  const int grid = (int)(tiles < sms ? tiles : sms);
  const char* e = getenv("NSF_GN_SIMT");   // read per call (tests run both passes)
  const int force_simt = (e && e[0] != '0') ? 1 : 0;
  const bool tc = !force_simt && gn_tc_supported(g, r);
  for (int it = 0; it < n_iters; ++it) {
    if (tc) launch_gn_tc(st, n_scenes, n_sample, r, slots, S, zw, g, accum);
    else k_gn_accumulate<<<grid > 0 ? grid : 1, inv::kRows, smem, st>>>(n_scenes, n_sample, r, rp, slots, S, zw, g, accum);
    k_gn_solve<<<(n_scenes + 127) / 128, 128, 0, st>>>(n_scenes, r, accum, zw);
  }
}

}  // namespace nsf
