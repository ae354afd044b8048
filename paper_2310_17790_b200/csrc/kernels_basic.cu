// Particle-parallel kernels: load/unpack, read-back/pack, direct-atomic P2G,
// dense grid update, per-particle G2P.  These are the first correct path and
// remain the sparse path (reduced variant, one point per ~8 cells) of the
// library; the dense path is in kernels_tiled.cu.
#include <cuda_runtime.h>
#include <cstdint>
#include "kernels.h"
#include "mpm_math.cuh"
#include "point_ops.cuh"

namespace nsf {

// ---------------------------------------------------------------------------
// unpack AoS caller arrays into SoA planes; ids = load order; tau^0 = tau(F^0)
__global__ void k_unpack(int64_t n, const float* __restrict__ x, const float* __restrict__ v,
                         const float* __restrict__ C, const float* __restrict__ F, float* S,
                         int64_t pitch, int32_t* ids, DevParams P, DevErr* err, int with_F) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  float xp[3], Fp[9];
  bool finite = true;   // every input value and tau^0 (else NSF_ERR_NONFINITE at load)
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    xp[a] = x[p * 3 + a];
    const float vp = v[p * 3 + a];
    S[pbase(p) + (PX + a) * 32] = xp[a];
    S[pbase(p) + (PV + a) * 32] = vp;
    finite &= isfinite(xp[a]) && isfinite(vp);
  }
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const float c = C ? C[p * 9 + k] : 0.0f;
    S[pbase(p) + (PC + k) * 32] = c;
    Fp[k] = F ? F[p * 9 + k] : ((k % 4 == 0) ? 1.0f : 0.0f);
    if (with_F) S[pbase(p) + (PF + k) * 32] = Fp[k];
    finite &= isfinite(c) && isfinite(Fp[k]);
  }
  ids[p] = (int32_t)p;
  bool ok = true;
#pragma unroll
  for (int a = 0; a < 3; ++a) ok &= in_safe_region(xp[a] * P.inv_dx, P.N[a]);
  if (!ok && finite) flag_error(err, ERR_OUT_OF_DOMAIN, (int)p);
  if (with_F) {
    float tau[6];
    elastic_tau(Fp, P.model, P.mu, P.lam, tau, P.kappa);
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      S[pbase(p) + (PT + k) * 32] = tau[k];
      finite &= isfinite(tau[k]);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 6; ++k) S[pbase(p) + (PT + k) * 32] = 0.0f;
  }
  S[pbase(p) + PTY * 32] = P.tau_Y;   // per-particle yield stress starts at the material's
  if (!finite) flag_error(err, ERR_NONFINITE, (int)p);
}

void launch_unpack(cudaStream_t st, int64_t n, const float* x, const float* v, const float* C,
                   const float* F, float* S, int64_t pitch, int32_t* ids, const DevParams& P,
                   DevErr* err, int with_F) {
  if (n == 0) return;
  int bs = 128;
  k_unpack<<<(unsigned)((n + bs - 1) / bs), bs, 0, st>>>(n, x, v, C, F, S, pitch, ids, P, err, with_F);
}

// scatter SoA planes back to caller order (dst row-major AoS, particle id order)
__global__ void k_pack(int64_t n, const float* __restrict__ S, int64_t pitch,
                       const int32_t* __restrict__ ids, int plane0, int ncomp, float* out) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  int64_t id = ids[j];
  for (int k = 0; k < ncomp; ++k) out[id * ncomp + k] = S[pbase(j) + (plane0 + k) * 32];
}

void launch_pack(cudaStream_t st, int64_t n, const float* S, int64_t pitch, const int32_t* ids,
                 int plane0, int ncomp, float* out) {
  if (n == 0) return;
  int bs = 256;
  k_pack<<<(unsigned)((n + bs - 1) / bs), bs, 0, st>>>(n, S, pitch, ids, plane0, ncomp, out);
}

// ---------------------------------------------------------------------------
// P2G, one thread per particle, 27 x red.global.add.v4.f32 (m, m v) per particle.
// scene_of(p) from offsets (NSF batches); node = scene * nodes_per_scene + local.
template <int FORCE>
__global__ void __launch_bounds__(128) k_p2g_direct(int64_t n, const float* __restrict__ S, int64_t pitch,
                                                    const int64_t* __restrict__ scene_off, int n_scenes,
                                                    float4* acc, DevParams P) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  int scene = 0;
  if (n_scenes > 1) {
    int lo = 0, hi = n_scenes;   // find s with off[s] <= p < off[s+1]
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (scene_off[mid] <= p) lo = mid; else hi = mid;
    }
    scene = lo;
  }
  float xp[3], vp[3], Cp[9], tp[6];
#pragma unroll
  for (int a = 0; a < 3; ++a) { xp[a] = S[pbase(p) + (PX + a) * 32]; vp[a] = S[pbase(p) + (PV + a) * 32]; }
#pragma unroll
  for (int k = 0; k < 9; ++k) Cp[k] = S[pbase(p) + (PC + k) * 32];
#pragma unroll
  for (int k = 0; k < 6; ++k) tp[k] = S[pbase(p) + (PT + k) * 32];
  Axis ax[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    ax[a] = bspline_axis(xp[a], P.inv_dx);
    ax[a].base = clamp_base(ax[a].base, P.N[a]);
  }
  const float m = P.mass;
  // tau as a full symmetric matrix
  float T[9] = {tp[0], tp[5], tp[4], tp[5], tp[1], tp[3], tp[4], tp[3], tp[2]};
  // Q = m C - (MLS) dt V0 4/dx^2 tau
  float Q[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) Q[k] = P.mC * Cp[k] - (FORCE == 0 ? P.mls_coef * T[k] : 0.0f);
  float4* base_ptr = acc + (int64_t)scene * P.nodes_per_scene;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        float W = ax[0].w[a] * ax[1].w[b] * ax[2].w[c];
        float d0 = ((float)a - ax[0].f) * P.dx;
        float d1 = ((float)b - ax[1].f) * P.dx;
        float d2 = ((float)c - ax[2].f) * P.dx;
        float mv0 = m * vp[0] + Q[0] * d0 + Q[1] * d1 + Q[2] * d2;
        float mv1 = m * vp[1] + Q[3] * d0 + Q[4] * d1 + Q[5] * d2;
        float mv2 = m * vp[2] + Q[6] * d0 + Q[7] * d1 + Q[8] * d2;
        mv0 *= W; mv1 *= W; mv2 *= W;
        if (FORCE == 1) {
          float g0 = ax[0].dw[a] * ax[1].w[b] * ax[2].w[c];
          float g1 = ax[0].w[a] * ax[1].dw[b] * ax[2].w[c];
          float g2 = ax[0].w[a] * ax[1].w[b] * ax[2].dw[c];
          mv0 -= P.gradw_coef * (T[0] * g0 + T[1] * g1 + T[2] * g2);
          mv1 -= P.gradw_coef * (T[3] * g0 + T[4] * g1 + T[5] * g2);
          mv2 -= P.gradw_coef * (T[6] * g0 + T[7] * g1 + T[8] * g2);
        }
        int64_t ni = node_index(ax[0].base + a, ax[1].base + b, ax[2].base + c, P);
        red_add_v4(base_ptr + ni, W * m, mv0, mv1, mv2);
      }
}

void launch_p2g_direct(cudaStream_t st, int64_t n, const float* S, int64_t pitch,
                       const int64_t* scene_off, int n_scenes, float4* acc, const DevParams& P) {
  if (n == 0) return;
  int bs = 128;
  unsigned g = (unsigned)((n + bs - 1) / bs);
  if (P.force_mode == 0) k_p2g_direct<0><<<g, bs, 0, st>>>(n, S, pitch, scene_off, n_scenes, acc, P);
  else k_p2g_direct<1><<<g, bs, 0, st>>>(n, S, pitch, scene_off, n_scenes, acc, P);
}


// ---------------------------------------------------------------------------
// G2P + constitutive, one thread per particle, in place (reads and writes index p).
// WITH_F = 0 is the reduced (NSF) variant: no F, no SVD, tau untouched.
template <int FORCE, int WITH_F>
__global__ void __launch_bounds__(128) k_g2p_direct(int64_t n, float* S, int64_t pitch,
                                                    const int64_t* __restrict__ scene_off, int n_scenes,
                                                    const float4* __restrict__ vel, DevParams P,
                                                    DevErr* err, int64_t* d_step, const int32_t* __restrict__ ids) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p == 0 && d_step) atomicAdd((unsigned long long*)d_step, 1ull);
  if (p >= n) return;
  int scene = 0;
  if (n_scenes > 1) {
    int lo = 0, hi = n_scenes;
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (scene_off[mid] <= p) lo = mid; else hi = mid;
    }
    scene = lo;
  }
  float xp[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) xp[a] = S[pbase(p) + (PX + a) * 32];
  Axis ax[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    ax[a] = bspline_axis(xp[a], P.inv_dx);
    ax[a].base = clamp_base(ax[a].base, P.N[a]);
  }
  const float4* vb = vel + (int64_t)scene * P.nodes_per_scene;
  float v[3] = {0.f, 0.f, 0.f};
  float Bm[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  float G[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        float W = ax[0].w[a] * ax[1].w[b] * ax[2].w[c];
        float4 vi = __ldg(vb + node_index(ax[0].base + a, ax[1].base + b, ax[2].base + c, P));
        float wv0 = W * vi.x, wv1 = W * vi.y, wv2 = W * vi.z;
        v[0] += wv0; v[1] += wv1; v[2] += wv2;
        float d0 = ((float)a - ax[0].f) * P.dx;
        float d1 = ((float)b - ax[1].f) * P.dx;
        float d2 = ((float)c - ax[2].f) * P.dx;
        Bm[0] += wv0 * d0; Bm[1] += wv0 * d1; Bm[2] += wv0 * d2;
        Bm[3] += wv1 * d0; Bm[4] += wv1 * d1; Bm[5] += wv1 * d2;
        Bm[6] += wv2 * d0; Bm[7] += wv2 * d1; Bm[8] += wv2 * d2;
        if (FORCE == 1 && WITH_F) {
          float g0 = ax[0].dw[a] * ax[1].w[b] * ax[2].w[c];
          float g1 = ax[0].w[a] * ax[1].dw[b] * ax[2].w[c];
          float g2 = ax[0].w[a] * ax[1].w[b] * ax[2].dw[c];
          G[0] += vi.x * g0; G[1] += vi.x * g1; G[2] += vi.x * g2;
          G[3] += vi.y * g0; G[4] += vi.y * g1; G[5] += vi.y * g2;
          G[6] += vi.z * g0; G[7] += vi.z * g1; G[8] += vi.z * g2;
        }
      }
  const float cC = 4.0f * P.inv_dx * P.inv_dx;   // 12/(dx^2 (b+1)), b = 2
  float Cn[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) Cn[k] = cC * Bm[k];
  if (FORCE == 0) {   // MLS: the F update's gradient is the full C
#pragma unroll
    for (int k = 0; k < 9; ++k) G[k] = Cn[k];
  }
  if (P.rpic) skew_part(Cn);   // RPIC (#38): the stored / transferred C_p
  float xn[3];
  bool ok = true;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    xn[a] = xp[a] + P.dt * v[a];
    ok &= in_safe_region(xn[a] * P.inv_dx, P.N[a]);
  }
  bool finite = true;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    S[pbase(p) + (PX + a) * 32] = xn[a];
    S[pbase(p) + (PV + a) * 32] = v[a];
    finite &= isfinite(xn[a]) && isfinite(v[a]);
  }
#pragma unroll
  for (int k = 0; k < 9; ++k) S[pbase(p) + (PC + k) * 32] = Cn[k];
  if (WITH_F) {
    float Fp[9], Ft[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) Fp[k] = S[pbase(p) + (PF + k) * 32];
    // F_trial = (I + dt G) F
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        Ft[i * 3 + j] = Fp[i * 3 + j] + P.dt * (G[i * 3 + 0] * Fp[0 * 3 + j] + G[i * 3 + 1] * Fp[1 * 3 + j] +
                                                G[i * 3 + 2] * Fp[2 * 3 + j]);
    float FE[9], tau[6];
    float J;
    if (P.vm_hs) {   // per-particle yield stress
      float tY = S[pbase(p) + PTY * 32];
      J = vm_hs_update(Ft, P.mu, P.lam, P.vm_hard_k, P.vm_soft, tY, FE, tau);
      S[pbase(p) + PTY * 32] = tY;
    } else {
      J = P.model == 5 ? hb_update(Ft, P.mu, P.kappa, P.hb_yield, P.hb_relax, FE, tau)
                       : elastoplastic(Ft, P.model, P.mu, P.lam, P.alpha, P.tau_Y, FE, tau);
    }
    if (!(J > 0.0f)) atomicAdd(&err->inverted, 1ull);
#pragma unroll
    for (int k = 0; k < 9; ++k) { S[pbase(p) + (PF + k) * 32] = FE[k]; finite &= isfinite(FE[k]); }
#pragma unroll
    for (int k = 0; k < 6; ++k) { S[pbase(p) + (PT + k) * 32] = tau[k]; finite &= isfinite(tau[k]); }
  }
  if (!ok) flag_error(err, ERR_OUT_OF_DOMAIN, ids[p]);
  if (!finite) flag_error(err, ERR_NONFINITE, ids[p]);
}

void launch_g2p_direct(cudaStream_t st, int64_t n, float* S, int64_t pitch, const int64_t* scene_off,
                       int n_scenes, const float4* vel, const DevParams& P, DevErr* err, int64_t* d_step,
                       int with_F, const int32_t* ids) {
  int bs = 128;
  unsigned g = (unsigned)((n + bs - 1) / bs);
  if (g == 0) g = 1;   // still bump the step counter
  if (with_F) {
    if (P.force_mode == 0) k_g2p_direct<0, 1><<<g, bs, 0, st>>>(n, S, pitch, scene_off, n_scenes, vel, P, err, d_step, ids);
    else k_g2p_direct<1, 1><<<g, bs, 0, st>>>(n, S, pitch, scene_off, n_scenes, vel, P, err, d_step, ids);
  } else {
    k_g2p_direct<0, 0><<<g, bs, 0, st>>>(n, S, pitch, scene_off, n_scenes, vel, P, err, d_step, ids);
  }
}

// ---------------------------------------------------------------------------
// Reduced (NSF) G2P (see point_ops.cuh): reads acc[step & 1], applies
// the grid update to each of the 27 stencil nodes, updates x, v, C in place,
// clears the point's previous stencil in acc[(step + 1) & 1] and records the
// current base.  The last CTA advances the step counter (every thread reads it
// first).
// 256-bit global accesses (sm_100): a node pair at an even node index is 32-byte
// aligned.  These accesses go to the two grid arrays h->acc / h->vel, allocated
// in nsf_mpm_create through dalloc (runtime.cu), which rejects any pointer that is
// not 256-byte aligned; scenes start at multiples of 64 nodes.
__device__ __forceinline__ void ld_nc8(const float4* p, float4& a, float4& b) {
  asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
      : "l"(p));
}
__device__ __forceinline__ void st_zero8(float4* p) {
  asm volatile("st.global.v8.f32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "f"(0.0f) : "memory");
}

#ifndef NSF_G2P_NSF_MINB
#define NSF_G2P_NSF_MINB 6   // 80 registers: 24 warps per SM for the gather latency (C5 -2.4%)
#endif
__global__ void __launch_bounds__(128, NSF_G2P_NSF_MINB) k_g2p_nsf(int64_t n, float* S, const int64_t* __restrict__ scene_off,
                                                 int n_scenes, float4* acc0, float4* acc1, DevParams P, DevErr* err,
                                                 int64_t* d_step, int* done, const int32_t* __restrict__ ids) {
  const int64_t step = *(volatile const int64_t*)d_step;
  // reverse sweep: the MLP/P2G kernel just reduced into the accumulator in
  // forward point order, so its most recent (L2-resident) lines come first
  const int64_t p = n - 1 - (blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
  if (p >= 0) {
    const int scene = scene_of(p, scene_off, n_scenes, n);
    const float y_pl = plate_y(P, step);
    const int64_t so = (int64_t)scene * P.nodes_per_scene;
    float xp[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) xp[a] = S[pbase(p) + (PX + a) * 32];
    const int packed = __float_as_int(S[pbase(p) + PF * 32]);
    Axis ax[3];
    int base[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      ax[a] = bspline_axis(xp[a], P.inv_dx);
      base[a] = ax[a].base = clamp_base(ax[a].base, P.N[a]);
    }
    S[pbase(p) + PF * 32] = __int_as_float(pack_base(base[0], base[1], base[2]));
    int X[3], Y[3], Z[3];
    if (packed != kNoBase) {   // previous stencil, in the accumulator P2G(step + 1) will use
      const int pb_[3] = {packed >> 20, (packed >> 10) & 1023, packed & 1023};
      stencil_offsets(pb_, P, X, Y, Z);
      NSF_CHECK(X[0] + Y[0] + Z[0] >= 0 && X[2] + Y[2] + Z[2] < P.nodes_per_scene && pb_[0] + 2 < P.N[0] &&
                pb_[1] + 2 < P.N[1] && pb_[2] + 2 < P.N[2]);
      float4* clr = ((step & 1) ? acc0 : acc1) + so;
      // each z-run of 3 nodes as a 32-byte pair at an even node index plus one node
      const int zp = pb_[2] & 1;
      const int zpair = zp ? Z[1] : Z[0], zone = zp ? Z[0] : Z[2];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          float4* r = clr + (X[a] + Y[b]);
          st_zero8(r + zpair);
          r[zone] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
    stencil_offsets(base, P, X, Y, Z);
    NSF_CHECK(X[0] + Y[0] + Z[0] >= 0 && X[2] + Y[2] + Z[2] < P.nodes_per_scene);
    const float4* ab = ((step & 1) ? acc1 : acc0) + so;
    // interior stencil (no wall band, no plate): the node update is v = mv/m + dt g
    bool simple = !(P.plate_enabled && (float)(base[1] + 2) * P.dx >= y_pl);
#pragma unroll
    for (int face = 0; face < 6; ++face) {
      const int axis = face >> 1;
      const bool hit = (face & 1) ? (base[axis] + 2 >= P.N[axis] - P.bc_width) : (base[axis] < P.bc_width);
      simple &= !(P.bc[face] != 0 && hit);
    }
    float v[3] = {0.f, 0.f, 0.f};
    float Bm[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    auto accumulate_w = [&](float W, float d0, float d1, float d2, float4 vi) {
      const float wv0 = W * vi.x, wv1 = W * vi.y, wv2 = W * vi.z;
      v[0] += wv0; v[1] += wv1; v[2] += wv2;
      Bm[0] += wv0 * d0; Bm[1] += wv0 * d1; Bm[2] += wv0 * d2;
      Bm[3] += wv1 * d0; Bm[4] += wv1 * d1; Bm[5] += wv1 * d2;
      Bm[6] += wv2 * d0; Bm[7] += wv2 * d1; Bm[8] += wv2 * d2;
    };
    auto accumulate = [&](int a, int b, int c, float4 vi) {
      accumulate_w(ax[0].w[a] * ax[1].w[b] * ax[2].w[c], ((float)a - ax[0].f) * P.dx, ((float)b - ax[1].f) * P.dx,
                   ((float)c - ax[2].f) * P.dx, vi);
    };
    if (simple) {
      const float gx = P.dt * P.g[0], gy = P.dt * P.g[1], gz = P.dt * P.g[2];
      // z-runs as a 32-byte pair at an even node index (c = zp, zp + 1) plus one
      // node (c = zp ? 0 : 2): 6 loads per x-plane; the z weights and offsets
      // follow that order (slot s holds c = zc[s])
      const int zp = base[2] & 1;
      const int zpair = zp ? Z[1] : Z[0], zone = zp ? Z[0] : Z[2];
      const float zc[3] = {(float)zp, (float)(zp + 1), zp ? 0.0f : 2.0f};
      const float wz[3] = {zp ? ax[2].w[1] : ax[2].w[0], zp ? ax[2].w[2] : ax[2].w[1], zp ? ax[2].w[0] : ax[2].w[2]};
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        float4 an[9];
#pragma unroll
        for (int b = 0; b < 3; ++b) {   // 9 nodes in flight
          const float4* r = ab + (X[a] + Y[b]);
          ld_nc8(r + zpair, an[3 * b], an[3 * b + 1]);
          an[3 * b + 2] = __ldg(r + zone);
        }
#pragma unroll
        for (int q = 0; q < 9; ++q) {
          const float rm = an[q].x > 0.0f ? __frcp_rn(an[q].x) : 0.0f;
          const float4 vi = an[q].x > 0.0f ? make_float4(fmaf(an[q].y, rm, gx), fmaf(an[q].z, rm, gy),
                                                         fmaf(an[q].w, rm, gz), an[q].x)
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
          const int b = q / 3, sl = q % 3;
          const float W = ax[0].w[a] * ax[1].w[b] * wz[sl];
          const float d0 = ((float)a - ax[0].f) * P.dx, d1 = ((float)b - ax[1].f) * P.dx, d2 = (zc[sl] - ax[2].f) * P.dx;
          accumulate_w(W, d0, d1, d2, vi);
        }
      }
    } else {
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
          for (int c = 0; c < 3; ++c)
            accumulate(a, b, c, grid_node_update(__ldg(ab + (X[a] + Y[b] + Z[c])), base[0] + a, base[1] + b,
                                                 base[2] + c, P, y_pl));
    }
    const float cC = 4.0f * P.inv_dx * P.inv_dx;   // C = 4/dx^2 B (b = 2)
    bool ok = true, finite = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float xn = xp[a] + P.dt * v[a];
      ok &= in_safe_region(xn * P.inv_dx, P.N[a]);
      finite &= isfinite(xn) && isfinite(v[a]);
      S[pbase(p) + (PX + a) * 32] = xn;
      S[pbase(p) + (PV + a) * 32] = v[a];
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) Bm[k] *= cC;
    if (P.rpic) skew_part(Bm);   // RPIC (#38)
#pragma unroll
    for (int k = 0; k < 9; ++k) S[pbase(p) + (PC + k) * 32] = Bm[k];
    if (!ok) flag_error(err, ERR_OUT_OF_DOMAIN, ids[p]);
    if (!finite) flag_error(err, ERR_NONFINITE, ids[p]);
  }
  __syncthreads();
  if (threadIdx.x == 0) {   // every CTA read d_step at its start (no fence needed)
    if (atomicAdd(done, 1) == (int)gridDim.x - 1) {
      *d_step = step + 1;
      *done = 0;
    }
  }
}

void launch_g2p_nsf(cudaStream_t st, int64_t n, float* S, const int64_t* scene_off, int n_scenes,
                    float4* acc0, float4* acc1, const DevParams& P, DevErr* err, int64_t* d_step, int* done,
                    const int32_t* ids) {
  const int bs = 128;
  unsigned g = (unsigned)((n + bs - 1) / bs);
  if (g == 0) g = 1;   // still advances the step counter
  k_g2p_nsf<<<g, bs, 0, st>>>(n, S, scene_off, n_scenes, acc0, acc1, P, err, d_step, done, ids);
}

// Marks every point's previous stencil as absent (after a load).
__global__ void k_nsf_reset_base(int64_t n, float* S) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p < n) S[pbase(p) + PF * 32] = __int_as_float(kNoBase);
}

void launch_nsf_reset_base(cudaStream_t st, int64_t n, float* S) {
  if (n > 0) k_nsf_reset_base<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, S);
}

// ---------------------------------------------------------------------------
// debug: copy the blocked grid into natural order (scene, i, j, k, 4)
__global__ void k_grid_to_dense(int64_t total_nodes, const float4* __restrict__ g, float* out, DevParams P) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= total_nodes) return;
  int64_t scene = q / P.nodes_per_scene;
  int64_t r = q % P.nodes_per_scene;
  int k = (int)(r % P.N[2]);
  int j = (int)((r / P.N[2]) % P.N[1]);
  int i = (int)(r / ((int64_t)P.N[2] * P.N[1]));
  float4 a = g[scene * P.nodes_per_scene + node_index(i, j, k, P)];
  out[q * 4 + 0] = a.x; out[q * 4 + 1] = a.y; out[q * 4 + 2] = a.z; out[q * 4 + 3] = a.w;
}

// debug: grid update that keeps the accumulator (stage-1 dump), natural order out
__global__ void k_grid_update_debug(int64_t total_nodes, const float4* __restrict__ acc, float4* vel,
                                    DevParams P, const int64_t* d_step) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= total_nodes) return;
  int64_t local = g % P.nodes_per_scene;
  int64_t blk = local >> 6;
  int l = (int)(local & 63);
  int b2 = (int)(blk % P.NB[2]);
  int b1 = (int)((blk / P.NB[2]) % P.NB[1]);
  int b0 = (int)(blk / ((int64_t)P.NB[2] * P.NB[1]));
  int i = b0 * 4 + (l >> 4), j = b1 * 4 + ((l >> 2) & 3), k = b2 * 4 + (l & 3);
  vel[g] = grid_node_update(acc[g], i, j, k, P, plate_y(P, *d_step));
}

void launch_grid_debug(cudaStream_t st, int stage, int64_t total_nodes, const float4* acc, float4* vel,
                       float* out, const DevParams& P, const int64_t* d_step) {
  int bs = 256;
  unsigned g = (unsigned)((total_nodes + bs - 1) / bs);
  if (stage == 1) {
    k_grid_update_debug<<<g, bs, 0, st>>>(total_nodes, acc, vel, P, d_step);
    k_grid_to_dense<<<g, bs, 0, st>>>(total_nodes, vel, out, P);
  } else {
    k_grid_to_dense<<<g, bs, 0, st>>>(total_nodes, acc, out, P);
  }
}

}  // namespace nsf
