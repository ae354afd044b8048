// Neural stress field MLP on the 5th-generation tensor cores (tcgen05 + TMEM).
//
//   tau = sigma_tau * h(X, z),  h = W_out r(ELU(W_L r(... ELU(W_1 u + b_1) ...)) + b_L) + b_out
//   (Eq. (9); architecture P:498-500; numerics reading #20:
//    layer-1 input fp32, activations rounded to bf16 before every later layer,
//    fp32 accumulation, bias and ELU in fp32)
//
// One persistent CTA per SM, 384 threads = three independent "streams" of 128
// points (one warpgroup each), so that the streams' CUDA-core epilogues (bias,
// ELU, bf16 rounding) overlap each other's MMAs.  Per stream and tile:
//   layer 1 (K = in_dim <= 16): tcgen05.mma kind::tf32 with the fp32 input split
//     as hi + lo (hi = tf32(u), lo = tf32(u - hi)) against W_1 stacked twice
//     (bf16 weights are exact in tf32), K = 32: the sum is u W_1 to fp32 accuracy,
//     as reading #20 requires; then bias + ELU, rounded to bf16 into the stream's
//     A tile (128 x 128, K-major, 128B-swizzled, the canonical UMMA layout);
//   hidden layers 2..L: tcgen05.mma.cta_group::1.kind::f16, M = N = 128,
//     K = 8 x 16, A = activations (smem), B = W_l (smem, resident for the whole
//     kernel), D = fp32 in TMEM (128 lanes x 128 columns); the epilogue reads D
//     with tcgen05.ld (thread = TMEM lane = point) and rewrites the A tile;
//   output layer: the same MMA with N = 16 (W_out zero-padded to 16 rows).
// TMEM: stream s uses columns [160 s, 160 s + 144).  Completion of each MMA
// group is signalled by tcgen05.commit to a per-stream mbarrier.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include "kernels.h"
#include "params.cuh"
#include "point_ops.cuh"

namespace nsf {

namespace tc {

constexpr int kStreams = 3;         // independent 128-point tile streams per CTA
constexpr int kThreads = 128 * kStreams;
constexpr int kTmemStride = 160;    // TMEM columns per stream (128 hidden + 16 output, 32-aligned)
constexpr int kM = 128;             // points per tile (MMA M)
constexpr int kW = 128;             // layer width (MMA N and K)
constexpr int kMaxHiddenMMA = 3;    // hidden layers on tensor cores (n_hidden <= 4)
constexpr int kOutN = 16;           // padded output width
constexpr int kTileBytes = kM * kW * 2;        // 32 KB bf16, two 64-wide K atoms of 16 KB
constexpr int kOutBBytes = kOutN * kW * 2;     // 4 KB

struct __align__(1024) Smem {
  uint8_t wB[kMaxHiddenMMA][kTileBytes];   // W_2..W_L as B operands (N x K, K-major, SW128)
  uint8_t wOut[kOutBBytes];                 // W_out padded to 16 rows
  uint8_t a[kStreams][kTileBytes];          // per-stream activation tile (layer 1: tf32 [hi | lo] inputs)
  uint8_t w1t[kW * 128];                     // layer-1 B operand: 128 rows x [W_1 | W_1] tf32, SW128
  float bias[kMaxHiddenMMA + 1][kW];        // b_1 .. b_L
  float bout[kOutN];
  unsigned long long bar[kStreams];          // per-stream MMA-completion mbarriers
  unsigned int tk[kStreams];                 // per-stream next tile (dynamic tickets)
  uint32_t tmem_base;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// byte offset of element (row, k) in a K-major, 128B-swizzled tile of `rows` rows
// (Swizzle<3,4,3>: the 16-byte chunk index within a 128-byte row is XORed with row % 8)
__device__ __forceinline__ uint32_t sw128_offset(int row, int k, int rows) {
  const int atom = k >> 6, kk = k & 63;
  return (uint32_t)(atom * rows * 128 + row * 128 + ((((kk >> 3) ^ (row & 7))) << 4) + ((kk & 7) << 1));
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, SBO = 1024 B, LBO = 16 B, version 1
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);          // start address
  d |= (uint64_t)1 << 16;                          // leading byte offset (16 B units)
  d |= (uint64_t)(1024 >> 4) << 32;                // stride byte offset: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                          // descriptor version (Blackwell)
  d |= (uint64_t)2 << 61;                          // layout: SWIZZLE_128B
  return d;
}

// instruction descriptor: D f32, A/B bf16 (fmt 1) or tf32 (fmt 2), both K-major, M x N
__host__ __device__ constexpr uint32_t make_idesc(int M, int N, uint32_t fmt = 1u) {
  return (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(unsigned long long* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void stream_barrier(int s) {
  asm volatile("bar.sync %0, 128;" ::"r"(1 + s) : "memory");
}

// 32 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// the same without the wait (the caller issues tmem_wait() before using r)
__device__ __forceinline__ void tmem_ld32_nw(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// ELU(a) = a (a > 0), e^a - 1 (a <= 0), fp32 with ex2.approx (MUFU)
__device__ __forceinline__ float elu(float a) {
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(a * 1.4426950408889634f));
  return a > 0.0f ? a : e - 1.0f;
}

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(src_bytes) : "memory");
}

__device__ __forceinline__ float4 lds_f4(uint32_t saddr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(saddr));
  return v;
}
__device__ __forceinline__ void sts_u4(uint32_t saddr, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(saddr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);   // RNE
  return *reinterpret_cast<uint32_t*>(&h);
}

// write 32 activations (columns c0..c0+31, c0 % 32 == 0) of row `row` into the swizzled A tile at shared
// address `tile`: 16-byte chunk (c0 % 64) / 8 + q of the row's 128-byte line, XORed with row % 8
__device__ __forceinline__ void store_act32(uint32_t tile, int row, int c0, const float* h) {
  const uint32_t rbase = tile + (uint32_t)((c0 >> 6) * (kM * 128) + row * 128);
  const uint32_t sw = (uint32_t)(row & 7), cb = (uint32_t)((c0 & 63) >> 3);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 u;
    u.x = pack_bf16(h[8 * q + 0], h[8 * q + 1]);
    u.y = pack_bf16(h[8 * q + 2], h[8 * q + 3]);
    u.z = pack_bf16(h[8 * q + 4], h[8 * q + 5]);
    u.w = pack_bf16(h[8 * q + 6], h[8 * q + 7]);
    sts_u4(rbase + (((cb + (uint32_t)q) ^ sw) << 4), u);
  }
}

}  // namespace tc

using namespace tc;

template <bool WIDE>   // WIDE: out_dim in (8, 16] (the affine-velocity field), a second TMEM load
__global__ void __launch_bounds__(kThreads, 1)
k_nsf_mlp_tc(int64_t n, const float* __restrict__ X, int64_t xpitch, const int64_t* __restrict__ scene_off,
             int n_scenes, const float* __restrict__ z, const float* __restrict__ dz, int r,
             const int64_t* __restrict__ d_step, MlpDev mlp, float stress_scale, float* __restrict__ tau_out,
             int aos_out, NsfP2G q) {
  extern __shared__ uint8_t smem_raw[];
  // align to 1024 B (SWIZZLE_128B atoms)
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x;
  const int s = tid >> 7;          // stream
  const int t = tid & 127;         // point within the tile == TMEM lane
  const int warp = tid >> 5;
  const int L = mlp.n_hidden + 1;  // linear layers
  const int n_mma_hidden = mlp.n_hidden - 1;
  const int in_dim = mlp.in_dim;

  // ---- one-time setup: weights into smem (swizzled B operands), biases, TMEM, barriers
  // (16-byte cp.async chunks, all in flight at once; the weights are L2-resident after the first CTA)
  for (int l = 0; l < n_mma_hidden; ++l) {
    const uint16_t* W = mlp.W + mlp.w_off[l + 1];   // [128 out][128 in]
    for (int c = tid; c < kW * (kW / 8); c += kThreads) {
      const int nrow = c >> 4, kc = c & 15;
      cp_async16(smem_u32(sm.wB[l] + sw128_offset(nrow, kc * 8, kW)), W + nrow * kW + kc * 8, 16);
    }
  }
  {
    const uint16_t* W = mlp.W + mlp.w_off[L - 1];   // [out_dim][128], rows >= out_dim zero-filled
    for (int c = tid; c < kOutN * (kW / 8); c += kThreads) {
      const int nrow = c >> 4, kc = c & 15;
      const bool in = nrow < mlp.out_dim;
      cp_async16(smem_u32(sm.wOut + sw128_offset(nrow, kc * 8, kOutN)), in ? W + nrow * kW + kc * 8 : W, in ? 16 : 0);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  // layer-1 B: row j = [W_1[j][0..in) b_hi b_lo 0.. | the same] (the inputs carry 1, 1 at columns in_dim,
  // in_dim + 1, so the MMA adds the fp32 bias b_1 = b_hi + b_lo, split in two tf32 parts); 16-byte chunk c of
  // row j at j*128 + ((c ^ (j & 7)) << 4)
  for (int e = tid; e < kW * 32; e += kThreads) {
    const int j = e >> 5, k = e & 31, i = k & 15;
    const float bj = mlp.b[mlp.b_off[0] + j];
    const float b_hi = __uint_as_float(to_tf32(bj));
    float w = 0.0f;
    if (i < in_dim) w = __uint_as_float(((uint32_t)mlp.W[mlp.w_off[0] + j * in_dim + i]) << 16);
    else if (i == in_dim) w = b_hi;
    else if (i == in_dim + 1) w = __uint_as_float(to_tf32(bj - b_hi));
    *reinterpret_cast<float*>(sm.w1t + j * 128 + ((((k >> 2) ^ (j & 7))) << 4) + (k & 3) * 4) = w;
  }
  for (int e = tid; e < (kMaxHiddenMMA + 1) * kW; e += kThreads) {
    const int l = e / kW, j = e % kW;
    sm.bias[l][j] = l < mlp.n_hidden ? mlp.b[mlp.b_off[l] + j] : 0.0f;
  }
  if (tid < kOutN) sm.bout[tid] = tid < mlp.out_dim ? mlp.b[mlp.b_off[L - 1] + tid] : 0.0f;
  if (tid == 0) {
    for (int k = 0; k < kStreams; ++k) mbar_init(&sm.bar[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&sm.tmem_base))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  fence_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = sm.tmem_base;
  const uint32_t d_col = tmem + (uint32_t)(kTmemStride * s);          // hidden-layer accumulator (128 cols)
  const uint32_t o_col = tmem + (uint32_t)(kTmemStride * s) + 128u;   // output accumulator (16 cols)
  const uint32_t lane_sel = ((uint32_t)(32 * (warp & 3))) << 16;
  const int64_t step = d_step ? *d_step : 0;
  const uint32_t a_saddr = smem_u32(sm.a[s]);
  const uint32_t w1_saddr = smem_u32(sm.w1t);
  const uint32_t bias_saddr = smem_u32(&sm.bias[0][0]);
  constexpr uint32_t kIdesc1 = make_idesc(kM, kW, 2u);
  constexpr uint32_t kIdescH = make_idesc(kM, kW);
  constexpr uint32_t kIdescO = make_idesc(kM, kOutN);
  uint32_t phase = 0;

  const int64_t n_tiles = (n + kM - 1) / kM;
  const int64_t tile_stride = (int64_t)gridDim.x * kStreams;
  // layer-1 inputs u = (X, z(n)) of point `tile * 128 + t`, fp32 (reading #20); loaded one tile ahead
  // (X and the scene are fetched a whole tile ahead, z(n) when the row is built)
  auto fetch_x = [&](int64_t tile_, float* x_, int& scene_) {
    const int64_t p_ = tile_ * kM + t;
    scene_ = -1;
    x_[0] = x_[1] = x_[2] = 0.0f;
    if (tile_ >= n_tiles || p_ >= n) return;
    scene_ = scene_of(p_, scene_off, n_scenes, n);
    if (xpitch >= 0) {
      x_[0] = X[0 * xpitch + p_];
      x_[1] = X[1 * xpitch + p_];
      x_[2] = X[2 * xpitch + p_];
    } else {   // AoSoA planes of the particle store
      x_[0] = X[pbase(p_) + 0 * 32];
      x_[1] = X[pbase(p_) + 1 * 32];
      x_[2] = X[pbase(p_) + 2 * 32];
    }
  };
  auto build_inputs = [&](const float* x_, int scene_, float* u_) {
#pragma unroll
    for (int i = 0; i < 16; ++i) u_[i] = 0.0f;
    if (scene_ < 0) return;
    u_[0] = x_[0];
    u_[1] = x_[1];
    u_[2] = x_[2];
    for (int k = 0; k < r && k < 13; ++k)
      u_[3 + k] = z[scene_ * r + k] + (float)step * (dz ? dz[scene_ * r + k] : 0.0f);
    u_[in_dim] = 1.0f;       // bias columns of the layer-1 B operand
    u_[in_dim + 1] = 1.0f;
  };
  // tiles: dynamic tickets (each stream claims its next tile while working on
  // the current one) or, without a counter, round robin
  int64_t tile = (int64_t)blockIdx.x * kStreams + s;
  if (mlp.ctr) {
    if (t == 0) sm.tk[s] = atomicAdd(mlp.ctr, 1u);
    stream_barrier(s);
    tile = sm.tk[s];
  }
  float xf[3];
  int scene_f;
  fetch_x(tile, xf, scene_f);
  while (tile < n_tiles) {
    const int64_t p = tile * kM + t;
    const bool live = p < n;
    const int scene = scene_f < 0 ? 0 : scene_f;
    float u[16];
    build_inputs(xf, scene_f, u);
    // A row t = [hi(u) | lo(u)], 32 tf32 = one 128-byte swizzled line
    {
      const uint32_t row = a_saddr + (uint32_t)t * 128u;
      const uint32_t sw = (uint32_t)(t & 7);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint4 hi, lo;
        uint32_t* ph = &hi.x;
        uint32_t* pl = &lo.x;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float x = u[4 * c + e];
          const uint32_t xh = to_tf32(x);
          ph[e] = xh;
          pl[e] = to_tf32(x - __uint_as_float(xh));
        }
        sts_u4(row + (((uint32_t)c ^ sw) << 4), hi);
        sts_u4(row + (((uint32_t)(c + 4) ^ sw) << 4), lo);
      }
    }
    if (mlp.ctr && t == 0) sm.tk[s] = atomicAdd(mlp.ctr, 1u);   // read after the tile's last barrier
    fence_async_smem();
    stream_barrier(s);
    if (t == 0) {
      fence_after();
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)   // K = 32 in steps of 8 (32 bytes)
        mma_tf32(d_col, make_desc(a_saddr + kk * 32), make_desc(w1_saddr + kk * 32), kIdesc1, kk > 0 ? 1u : 0u);
      mma_commit(&sm.bar[s]);
    }
    mbar_wait(&sm.bar[s], phase);
    phase ^= 1;
    fence_after();
#pragma unroll 1
    for (int c0 = 0; c0 < kW; c0 += 64) {   // 64 columns per TMEM round trip
      uint32_t r2[64];
      tmem_ld32_nw(d_col + lane_sel + c0, r2);   // bias already added by the MMA
      tmem_ld32_nw(d_col + lane_sel + c0 + 32, r2 + 32);
      tmem_wait();
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        float h[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) h[q] = elu(__uint_as_float(r2[32 * hh + q]));
        store_act32(a_saddr, t, c0 + 32 * hh, h);
      }
    }
    fence_before();
    fence_async_smem();
    stream_barrier(s);
    // the next tile (its ticket was claimed before the layer-1 barrier): X now,
    // so that the loads are in flight across the hidden layers
    const int64_t next = mlp.ctr ? (int64_t)sm.tk[s] : tile + tile_stride;
    fetch_x(next, xf, scene_f);
    // ---- hidden layers on tensor cores ----
    for (int l = 0; l < n_mma_hidden; ++l) {
      if (t == 0) {
        fence_after();
        const uint32_t b_saddr = smem_u32(sm.wB[l]);
#pragma unroll
        for (int kk = 0; kk < kW / 16; ++kk) {
          const uint32_t koff = (uint32_t)((kk >> 2) * (kM * 128) + (kk & 3) * 32);
          const uint32_t kofb = (uint32_t)((kk >> 2) * (kW * 128) + (kk & 3) * 32);
          mma_bf16(d_col, make_desc(a_saddr + koff), make_desc(b_saddr + kofb), kIdescH, kk > 0 ? 1u : 0u);
        }
        mma_commit(&sm.bar[s]);
      }
      mbar_wait(&sm.bar[s], phase);
      phase ^= 1;
      fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < kW; c0 += 64) {   // 64 columns per TMEM round trip
        uint32_t r2[64];
        tmem_ld32_nw(d_col + lane_sel + c0, r2);
        tmem_ld32_nw(d_col + lane_sel + c0 + 32, r2 + 32);
        tmem_wait();
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          float h[32];
          const int cc = c0 + 32 * hh;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 b = lds_f4(bias_saddr + (uint32_t)((l + 1) * kW + cc + 4 * q) * 4u);
            h[4 * q] = elu(__uint_as_float(r2[32 * hh + 4 * q]) + b.x);
            h[4 * q + 1] = elu(__uint_as_float(r2[32 * hh + 4 * q + 1]) + b.y);
            h[4 * q + 2] = elu(__uint_as_float(r2[32 * hh + 4 * q + 2]) + b.z);
            h[4 * q + 3] = elu(__uint_as_float(r2[32 * hh + 4 * q + 3]) + b.w);
          }
          store_act32(a_saddr, t, cc, h);
        }
      }
      fence_before();
      fence_async_smem();
      stream_barrier(s);
    }
    // ---- output layer (N = 16, zero-padded) ----
    if (t == 0) {
      fence_after();
      const uint32_t b_saddr = smem_u32(sm.wOut);
#pragma unroll
      for (int kk = 0; kk < kW / 16; ++kk) {
        const uint32_t koff = (uint32_t)((kk >> 2) * (kM * 128) + (kk & 3) * 32);
        const uint32_t kofb = (uint32_t)((kk >> 2) * (kOutN * 128) + (kk & 3) * 32);
        mma_bf16(o_col, make_desc(a_saddr + koff), make_desc(b_saddr + kofb), kIdescO, kk > 0 ? 1u : 0u);
      }
      mma_commit(&sm.bar[s]);
    }
    // the point's P2G inputs load while the output MMA runs
    float xp[3], vp[3], Cp[9];
    if (q.enabled && live) nsf_load_point(q.S, p, xp, vp, Cp);
    mbar_wait(&sm.bar[s], phase);
    phase ^= 1;
    fence_after();
    float y[8];
    tmem_ld8(o_col + lane_sel, y);
    if (live) {
      float tau[8];
#pragma unroll
      for (int o = 0; o < 8; ++o) tau[o] = stress_scale * (y[o] + sm.bout[o]);
      for (int o = 0; o < mlp.out_dim && o < 8; ++o) {
        if (aos_out) tau_out[p * mlp.out_dim + o] = tau[o];
        else tau_out[pbase(p) + o * 32] = tau[o];   // AoSoA particle store (tau fields)
      }
      if (q.enabled) nsf_p2g_point(q, scene, xp, vp, Cp, tau, step);   // reduced P2G, tau from registers
    }
    if (WIDE) {   // outputs 8..15 (the affine-velocity field l has 9; tcgen05.ld is warp-collective)
      float y2[8];
      tmem_ld8(o_col + lane_sel + 8, y2);
      if (live)
        for (int o = 8; o < mlp.out_dim; ++o) {
          const float val = stress_scale * (y2[o - 8] + sm.bout[o]);
          if (aos_out) tau_out[p * mlp.out_dim + o] = val;
          else tau_out[pbase(p) + o * 32] = val;
        }
    }
    fence_before();
    stream_barrier(s);   // the A tile and accumulators are free for the next tile
    tile = next;
  }
  __syncthreads();
  if (warp == 0) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
  if (mlp.ctr && tid == 0) {   // the last CTA resets the counters for the next launch
    __threadfence();
    if (atomicAdd(mlp.ctr + 1, 1u) == gridDim.x - 1) {
      mlp.ctr[0] = 0u;
      mlp.ctr[1] = 0u;
    }
  }
}

// ---------------------------------------------------------------------------
// Network inversion pass on the tensor cores (kernels_inv.cu has the CUDA-core
// version and the Gauss-Newton solve): per tile of 128 rows = 16 points x 8
// rows (primal, r <= 7 tangents of z, padding), the deformation field g and its
// forward-mode tangents go through the same MMAs as the stress field: layer 1
// tf32 on [hi | lo] inputs (primal: (X, z, 1, 1) -> bias by the MMA; tangent k:
// e_{3+k}, no bias), hidden layers bf16, output N = 16 (3 used).  Hidden
// epilogues in two phases: primal rows apply bias + ELU and publish ELU'(a)
// (fp32, shared memory); after a stream barrier the tangent rows scale their
// pre-activations by it (no bias).  Tangents are rounded to bf16 like
// activations.  Per point, J^T J and J^T (g - x) go into fp64 per-scene sums.
namespace gn {
constexpr int kS = 2;              // streams (128 rows each)
constexpr int kRP = 8;             // rows per point
constexpr int kPts = kM / kRP;     // 16 points per tile
struct __align__(1024) GnSmem {
  uint8_t wB[kMaxHiddenMMA][kTileBytes];
  uint8_t wOut[kOutBBytes];
  uint8_t a[kS][kTileBytes];
  uint8_t w1t[kW * 128];
  float bias[kMaxHiddenMMA + 1][kW];
  float bout[kOutN];
  float dbuf[kS][kPts][kW];        // ELU'(a) of each point's primal row
  float outb[kS][kM][4];
  unsigned long long bar[kS];
  uint32_t tmem_base;
};
}  // namespace gn

__global__ void __launch_bounds__(gn::kS * 128, 1)
k_gn_tc(int n_scenes, int n_sample, int r, const int32_t* __restrict__ slots, const float* __restrict__ S,
        const float* __restrict__ zw, MlpDev g, double* __restrict__ accum) {
  using namespace gn;
  extern __shared__ uint8_t smem_raw[];
  GnSmem& sm = *reinterpret_cast<GnSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x;
  const int s = tid >> 7;
  const int t = tid & 127;
  const int warp = tid >> 5;
  const int L = g.n_hidden + 1;
  const int n_mma_hidden = g.n_hidden - 1;
  const int in_dim = g.in_dim;
  // ---- weights (same layout as the stress-field kernel) ----
  for (int l = 0; l < n_mma_hidden; ++l) {
    const uint16_t* W = g.W + g.w_off[l + 1];
    for (int c = tid; c < kW * (kW / 8); c += kS * 128) {
      const int nrow = c >> 4, kc = c & 15;
      cp_async16(smem_u32(sm.wB[l] + sw128_offset(nrow, kc * 8, kW)), W + nrow * kW + kc * 8, 16);
    }
  }
  {
    const uint16_t* W = g.W + g.w_off[L - 1];
    for (int c = tid; c < kOutN * (kW / 8); c += kS * 128) {
      const int nrow = c >> 4, kc = c & 15;
      const bool in = nrow < g.out_dim;
      cp_async16(smem_u32(sm.wOut + sw128_offset(nrow, kc * 8, kOutN)), in ? W + nrow * kW + kc * 8 : W, in ? 16 : 0);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  for (int e = tid; e < kW * 32; e += kS * 128) {
    const int j = e >> 5, k = e & 31, i = k & 15;
    const float bj = g.b[g.b_off[0] + j];
    const float b_hi = __uint_as_float(to_tf32(bj));
    float w = 0.0f;
    if (i < in_dim) w = __uint_as_float(((uint32_t)g.W[g.w_off[0] + j * in_dim + i]) << 16);
    else if (i == in_dim) w = b_hi;
    else if (i == in_dim + 1) w = __uint_as_float(to_tf32(bj - b_hi));
    *reinterpret_cast<float*>(sm.w1t + j * 128 + ((((k >> 2) ^ (j & 7))) << 4) + (k & 3) * 4) = w;
  }
  for (int e = tid; e < (kMaxHiddenMMA + 1) * kW; e += kS * 128) {
    const int l = e / kW, j = e % kW;
    sm.bias[l][j] = l < g.n_hidden ? g.b[g.b_off[l] + j] : 0.0f;
  }
  if (tid < kOutN) sm.bout[tid] = tid < g.out_dim ? g.b[g.b_off[L - 1] + tid] : 0.0f;
  if (tid == 0) {
    for (int k = 0; k < kS; ++k) mbar_init(&sm.bar[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&sm.tmem_base))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  fence_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = sm.tmem_base;
  const uint32_t d_col = tmem + (uint32_t)(kTmemStride * s);
  const uint32_t o_col = d_col + 128u;
  const uint32_t lane_sel = ((uint32_t)(32 * (warp & 3))) << 16;
  const uint32_t a_saddr = smem_u32(sm.a[s]);
  const uint32_t w1_saddr = smem_u32(sm.w1t);
  const uint32_t bias_saddr = smem_u32(&sm.bias[0][0]);
  constexpr uint32_t kIdesc1 = make_idesc(kM, kW, 2u);
  constexpr uint32_t kIdescH = make_idesc(kM, kW);
  constexpr uint32_t kIdescO = make_idesc(kM, kOutN);
  uint32_t phase = 0;
  const int point = t / kRP, kk = t % kRP;
  const bool primal = kk == 0, tangent = kk >= 1 && kk <= r;
  const int64_t n_pts = (int64_t)n_scenes * n_sample;
  const int64_t n_tiles = (n_pts + kPts - 1) / kPts;
  const int nterm = r * (r + 1) / 2 + r;
  for (int64_t tile = (int64_t)blockIdx.x * kS + s; tile < n_tiles; tile += (int64_t)gridDim.x * kS) {
    const int64_t e = tile * kPts + point;
    const int scene = e < n_pts ? (int)(e / n_sample) : 0;
    const int slot = e < n_pts ? slots[e] : -1;
    const bool live = slot >= 0;
    // ---- layer-1 A row: [hi(u) | lo(u)] ----
    float u[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) u[i] = 0.0f;
    float xt[3] = {0.f, 0.f, 0.f};
    if (live && primal) {
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        u[a] = S[pbase(slot) + (PXR + a) * 32];
        xt[a] = S[pbase(slot) + (PX + a) * 32];
      }
      for (int q = 0; q < r; ++q) u[3 + q] = zw[scene * r + q];
      u[in_dim] = 1.0f;        // bias columns of the layer-1 B operand
      u[in_dim + 1] = 1.0f;
    } else if (live && tangent) {
      u[3 + (kk - 1)] = 1.0f;
    }
    {
      const uint32_t row = a_saddr + (uint32_t)t * 128u;
      const uint32_t sw = (uint32_t)(t & 7);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint4 hi, lo;
        uint32_t* ph = &hi.x;
        uint32_t* pl = &lo.x;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float x = u[4 * c + q];
          const uint32_t xh = to_tf32(x);
          ph[q] = xh;
          pl[q] = to_tf32(x - __uint_as_float(xh));
        }
        sts_u4(row + (((uint32_t)c ^ sw) << 4), hi);
        sts_u4(row + (((uint32_t)(c + 4) ^ sw) << 4), lo);
      }
    }
    fence_async_smem();
    stream_barrier(s);
    for (int layer = 0; layer <= n_mma_hidden; ++layer) {   // layer 0: tf32 layer 1; then the hidden MMAs
      if (t == 0) {
        fence_after();
        if (layer == 0) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            mma_tf32(d_col, make_desc(a_saddr + q * 32), make_desc(w1_saddr + q * 32), kIdesc1, q > 0 ? 1u : 0u);
        } else {
          const uint32_t b_saddr = smem_u32(sm.wB[layer - 1]);
#pragma unroll
          for (int q = 0; q < kW / 16; ++q) {
            const uint32_t koff = (uint32_t)((q >> 2) * (kM * 128) + (q & 3) * 32);
            const uint32_t kofb = (uint32_t)((q >> 2) * (kW * 128) + (q & 3) * 32);
            mma_bf16(d_col, make_desc(a_saddr + koff), make_desc(b_saddr + kofb), kIdescH, q > 0 ? 1u : 0u);
          }
        }
        mma_commit(&sm.bar[s]);
      }
      mbar_wait(&sm.bar[s], phase);
      phase ^= 1;
      fence_after();
      // per 32-column chunk (tcgen05.ld is warp-collective: every row loads its
      // chunk): primal rows add the bias (layers >= 2; layer 1's came from the
      // MMA), publish ELU'(a) and store ELU(a); then tangent rows store
      // ELU'(a) * (W t_prev); padding rows store zeros
#pragma unroll 1
      for (int c0 = 0; c0 < kW; c0 += 32) {
        float h[32];
        tmem_ld32(d_col + lane_sel + c0, h);
        if (primal) {
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            const float a = h[q] + (layer > 0 ? sm.bias[layer][c0 + q] : 0.0f);
            sm.dbuf[s][point][c0 + q] = a > 0.0f ? 1.0f : __expf(a);
            h[q] = elu(a);
          }
          store_act32(a_saddr, t, c0, h);
        }
        stream_barrier(s);
        if (!primal) {
#pragma unroll
          for (int q = 0; q < 32; ++q) h[q] = tangent ? sm.dbuf[s][point][c0 + q] * h[q] : 0.0f;
          store_act32(a_saddr, t, c0, h);
        }
      }
      fence_before();
      fence_async_smem();
      stream_barrier(s);
    }
    // ---- output layer (N = 16, 3 used): primal -> g, tangent k -> dg/dz_k ----
    if (t == 0) {
      fence_after();
      const uint32_t b_saddr = smem_u32(sm.wOut);
#pragma unroll
      for (int q = 0; q < kW / 16; ++q) {
        const uint32_t koff = (uint32_t)((q >> 2) * (kM * 128) + (q & 3) * 32);
        const uint32_t kofb = (uint32_t)((q >> 2) * (kOutN * 128) + (q & 3) * 32);
        mma_bf16(o_col, make_desc(a_saddr + koff), make_desc(b_saddr + kofb), kIdescO, q > 0 ? 1u : 0u);
      }
      mma_commit(&sm.bar[s]);
    }
    mbar_wait(&sm.bar[s], phase);
    phase ^= 1;
    fence_after();
    {
      float y[8];
      tmem_ld8(o_col + lane_sel, y);
#pragma unroll
      for (int o = 0; o < 3; ++o) sm.outb[s][t][o] = y[o] + (primal ? sm.bout[o] : 0.0f);
    }
    fence_before();
    stream_barrier(s);
    if (primal && live) {
      double res[3], J[3][8];
#pragma unroll
      for (int o = 0; o < 3; ++o) res[o] = (double)sm.outb[s][t][o] - (double)xt[o];
      for (int q = 0; q < r; ++q)
#pragma unroll
        for (int o = 0; o < 3; ++o) J[o][q] = (double)sm.outb[s][t + 1 + q][o];
      double* A = accum + (int64_t)scene * nterm;
      int idx = 0;
      for (int a = 0; a < r; ++a)
        for (int c = a; c < r; ++c, ++idx)
          atomicAdd(A + idx, J[0][a] * J[0][c] + J[1][a] * J[1][c] + J[2][a] * J[2][c]);
      for (int a = 0; a < r; ++a) atomicAdd(A + idx + a, J[0][a] * res[0] + J[1][a] * res[1] + J[2][a] * res[2]);
    }
    stream_barrier(s);   // outb, the A tile and the accumulators are free for the next tile
  }
  __syncthreads();
  if (warp == 0) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

bool gn_tc_supported(const MlpDev& g, int r) {
  return g.width == kW && g.n_hidden >= 2 && g.n_hidden - 1 <= kMaxHiddenMMA && g.in_dim <= 14 && g.out_dim == 3 &&
         r >= 1 && r + 1 <= gn::kRP;
}

void launch_gn_tc(cudaStream_t st, int n_scenes, int n_sample, int r, const int32_t* slots, const float* S,
                  const float* zw, const MlpDev& g, double* accum) {
  static int n_sms = 0;
  static bool attr = false;
  const size_t smem = sizeof(gn::GnSmem) + 1024;
  if (!attr) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_gn_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int64_t tiles = ((int64_t)n_scenes * n_sample + gn::kPts - 1) / gn::kPts;
  int64_t grid = (tiles + gn::kS - 1) / gn::kS;
  if (grid > n_sms) grid = n_sms;
  if (grid < 1) grid = 1;
  k_gn_tc<<<(unsigned)grid, gn::kS * 128, smem, st>>>(n_scenes, n_sample, r, slots, S, zw, g, accum);
}

bool nsf_mlp_tc_supported(const MlpDev& mlp) {
  return mlp.width == kW && mlp.n_hidden >= 2 && mlp.n_hidden - 1 <= kMaxHiddenMMA && mlp.in_dim <= 14 &&
         mlp.out_dim <= kOutN;
}

void launch_nsf_mlp_tc(cudaStream_t st, int64_t n, const float* X, int64_t xpitch, const int64_t* scene_off,
                       int n_scenes, const float* z, const float* dz, int r, const int64_t* d_step,
                       const MlpDev& mlp, float stress_scale, float* tau_out, int aos_out, const NsfP2G* qp) {
  if (n == 0) return;
  NsfP2G q{};
  if (qp) q = *qp;
  static int n_sms = 0;
  static bool attr = false;
  const size_t smem = sizeof(Smem) + 1024;
  if (!attr) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_nsf_mlp_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_nsf_mlp_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int64_t tiles = (n + kM - 1) / kM;
  int64_t grid = (tiles + kStreams - 1) / kStreams;
  if (grid > n_sms) grid = n_sms;
  if (mlp.out_dim > 8)
    k_nsf_mlp_tc<true><<<(unsigned)grid, kThreads, smem, st>>>(n, X, xpitch, scene_off, n_scenes, z, dz, r, d_step,
                                                               mlp, stress_scale, tau_out, aos_out, q);
  else
    k_nsf_mlp_tc<false><<<(unsigned)grid, kThreads, smem, st>>>(n, X, xpitch, scene_off, n_scenes, z, dz, r, d_step,
                                                                mlp, stress_scale, tau_out, aos_out, q);
}

}  // namespace nsf
