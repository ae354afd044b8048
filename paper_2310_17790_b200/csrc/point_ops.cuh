// Per-point device helpers shared by the particle-parallel kernels
// (kernels_basic.cu) and the reduced-variant MLP kernels (P2G epilogue).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include "mpm_math.cuh"
#include "params.cuh"

namespace nsf {

// ---------------------------------------------------------------------------
__device__ __forceinline__ void red_add_v4(float4* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b),
               "f"(c), "f"(d)
               : "memory");
}

__device__ __forceinline__ void flag_error(DevErr* err, uint32_t bit, int idx) {
  atomicOr(&err->bits, bit);
  atomicMin(&err->first_index, idx);
}

// (a NaN coordinate counts as in the region: it is reported as non-finite)
__device__ __forceinline__ bool in_safe_region(float t, int N) {
  return !(t < 0.5f || t >= (float)N - 1.5f);
}

// clamp a base index so that base..base+2 stays inside [0, N)
__device__ __forceinline__ int clamp_base(int b, int N) { return min(max(b, 0), N - 3); }

// ---------------------------------------------------------------------------
// Grid update for one node: v = mv/m + dt g, walls, plate.  Returns (v, m).
__device__ __forceinline__ float4 grid_node_update(float4 a, int i, int j, int k, const DevParams& P,
                                                   float y_plate) {
  float m = a.x;
  if (!(m > 0.0f)) return make_float4(0.f, 0.f, 0.f, 0.f);
  const float rm = __frcp_rn(m);   // v = (m v) (1/m) + dt g: the form every reduced-path gather uses
  float v[3] = {fmaf(a.y, rm, P.dt * P.g[0]), fmaf(a.z, rm, P.dt * P.g[1]), fmaf(a.w, rm, P.dt * P.g[2])};
  int idx[3] = {i, j, k};
#pragma unroll
  for (int face = 0; face < 6; ++face) {
    int kind = P.bc[face];
    if (kind == 0) continue;
    int axis = face >> 1;
    bool high = face & 1;
    bool in = high ? (idx[axis] >= P.N[axis] - P.bc_width) : (idx[axis] < P.bc_width);
    if (!in) continue;
    if (kind == 1) { v[0] = v[1] = v[2] = 0.0f; }
    else v[axis] = high ? fminf(v[axis], 0.0f) : fmaxf(v[axis], 0.0f);
  }
  if (P.plate_enabled && (float)j * P.dx >= y_plate) {
    v[0] = P.plate_v[0]; v[1] = P.plate_v[1]; v[2] = P.plate_v[2];
  }
  return make_float4(v[0], v[1], v[2], m);
}

__device__ __forceinline__ float plate_y(const DevParams& P, int64_t step) {
  // y_p(t_n) = y0 + v_y * n dt (reading #12); computed in double to keep t exact
  return (float)((double)P.plate_y0 + (double)P.plate_v[1] * ((double)step * (double)P.dt));
}

// Blocked-layout offsets of the 3 stencil nodes per axis (node_index split per
// axis, 32-bit: one scene's grid has < 2^31 nodes)
__device__ __forceinline__ void stencil_offsets(const int base[3], const DevParams& P, int X[3], int Y[3], int Z[3]) {
  const int plane = P.NB[1] * P.NB[2] * kBlockNodes;
#pragma unroll
  for (int o = 0; o < 3; ++o) {
    const int i = base[0] + o, j = base[1] + o, k = base[2] + o;
    X[o] = (i >> 2) * plane + ((i & 3) << 4);
    Y[o] = (j >> 2) * (P.NB[2] * kBlockNodes) + ((j & 3) << 2);
    Z[o] = (k >> 2) * kBlockNodes + (k & 3);
  }
}

// scene of point p among n: first the guess of equal-size scenes (two
// independent loads), else a binary search over the scene offsets
__device__ __forceinline__ int scene_of(int64_t p, const int64_t* scene_off, int n_scenes, int64_t n) {
  int lo = 0;
  if (n_scenes > 1 && scene_off) {
    const int g = (int)min((int64_t)n_scenes - 1, p * n_scenes / (n > 0 ? n : 1));
    if (__ldg(scene_off + g) <= p && p < __ldg(scene_off + g + 1)) return g;
    int hi = n_scenes;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (scene_off[mid] <= p) lo = mid; else hi = mid;
    }
  }
  return lo;
}

// ---------------------------------------------------------------------------
// Reduced (NSF) substep: points carry x, v, C; tau comes from
// the MLP.  Two accumulators alternate by step parity: P2G(n) reduces into
// acc[n & 1]; G2P(n) reads acc[n & 1] and applies the grid update node by
// node, and clears in acc[(n+1) & 1] (read by G2P(n-1), next written by P2G(n+1))
// the 27 nodes of each point's stencil at x_{n-1}: the base G2P(n-1) packed into
// the otherwise unused F plane.
struct NsfP2G {
  float* S;            // particle store (AoSoA)
  float4* acc0;
  float4* acc1;
  DevParams P;
  int enabled;         // 0: MLP only (tau to the store / AoS output)
};

constexpr int kNoBase = -1;

__device__ __forceinline__ int pack_base(int b0, int b1, int b2) { return (b0 << 20) | (b1 << 10) | b2; }

// P2G of one point (state x, v, C, Kirchhoff stress tau in Voigt order) of
// `scene`, MLS force (reading #1): 27 vector reductions into acc[step & 1].
__device__ __forceinline__ void nsf_p2g_point(const NsfP2G& q, int scene, const float xp[3], const float vp[3],
                                              const float Cp[9], const float tp[6], int64_t step) {
  const DevParams& P = q.P;
  float4* out = ((step & 1) ? q.acc1 : q.acc0) + (int64_t)scene * P.nodes_per_scene;
  Axis ax[3];
  int base[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    ax[a] = bspline_axis(xp[a], P.inv_dx);
    base[a] = ax[a].base = clamp_base(ax[a].base, P.N[a]);
  }
  int X[3], Y[3], Z[3];
  stencil_offsets(base, P, X, Y, Z);
  const float m = P.mass;
  const float T[9] = {tp[0], tp[5], tp[4], tp[5], tp[1], tp[3], tp[4], tp[3], tp[2]};
  float Q[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) Q[k] = P.mC * Cp[k] - P.mls_coef * T[k];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const float W = ax[0].w[a] * ax[1].w[b] * ax[2].w[c];
        const float d0 = ((float)a - ax[0].f) * P.dx, d1 = ((float)b - ax[1].f) * P.dx, d2 = ((float)c - ax[2].f) * P.dx;
        const float mv0 = W * (m * vp[0] + Q[0] * d0 + Q[1] * d1 + Q[2] * d2);
        const float mv1 = W * (m * vp[1] + Q[3] * d0 + Q[4] * d1 + Q[5] * d2);
        const float mv2 = W * (m * vp[2] + Q[6] * d0 + Q[7] * d1 + Q[8] * d2);
        NSF_CHECK(X[a] + Y[b] + Z[c] >= 0 && X[a] + Y[b] + Z[c] < P.nodes_per_scene);
        red_add_v4(out + (X[a] + Y[b] + Z[c]), W * m, mv0, mv1, mv2);
      }
}

// the point's x, v, C from the particle store
__device__ __forceinline__ void nsf_load_point(const float* S, int64_t p, float xp[3], float vp[3], float Cp[9]) {
#pragma unroll
  for (int a = 0; a < 3; ++a) { xp[a] = S[pbase(p) + (PX + a) * 32]; vp[a] = S[pbase(p) + (PV + a) * 32]; }
#pragma unroll
  for (int k = 0; k < 9; ++k) Cp[k] = S[pbase(p) + (PC + k) * 32];
}

}  // namespace nsf
