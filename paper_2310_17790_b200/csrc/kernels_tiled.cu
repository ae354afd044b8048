// Dense-path kernels: one CTA per non-empty 4x4x4-cell block (persistent over
// the compacted block list produced by the binning scan).
//
//  p2g_tiled: particles of the block are
//              staged in shared memory, counting-sorted by cell into a padded
//              [row][cell] layout (conflict-free reads); thread (cell, ox)
//              accumulates the 9 nodes of its stencil plane in registers over
//              the cell's particles; per-cell partials are reduced node by node
//              over the 6x6x6 tile and flushed with one red.global.add.v4.f32
//              per touched node.  No shared-memory float atomics (they are CAS
//              loops on sm_100a).
//  grid_update_blocks (a4): each node of every block touched by P2G is
//              updated exactly once (ownership rule below) and its accumulator
//              cleared for the next substep.
//  g2p         (a5 + a6): one thread per block-sorted slot gathers
//              its 27 grid velocities (through L1: neighbouring lanes share
//              stencils), updates x, v, C, F, runs the constitutive update and
//              writes the particle to the other buffer at its sorted slot
//              (sort-on-write), with its next block key and the histogram for
//              the next binning.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include "mpm_math.cuh"
#include "pipeline.h"

namespace nsf {

#if NSF_STATS
__device__ unsigned long long g_nsf_stats[kStCount];
__device__ unsigned long long g_tail_sum = 0, g_tail_start = ~0ull;
__device__ unsigned int g_tail_done = 0;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// per-launch tail statistics: called by thread 0 of every CTA at its start / exit
__device__ __forceinline__ void tail_stat_begin() { atomicMin(&g_tail_start, gtimer()); }
__device__ __forceinline__ void tail_stat_end() {
  const unsigned long long t = gtimer();
  atomicAdd(&g_tail_sum, t);
  __threadfence();
  if (atomicAdd(&g_tail_done, 1u) == gridDim.x - 1) {
    __threadfence();
    const unsigned long long s = atomicAdd(&g_tail_sum, 0ull), t0 = atomicAdd(&g_tail_start, 0ull);
    NSF_STAT_ADD(kStTailNs, (unsigned long long)gridDim.x * t - s);
    NSF_STAT_ADD(kStKernNs, t - t0);
    NSF_STAT_ADD(kStCtas, gridDim.x);
    g_tail_sum = 0;
    g_tail_start = ~0ull;
    g_tail_done = 0;
  }
}
#endif

__device__ __forceinline__ void red_add_v4_t(float4* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

struct BlockCoord {
  int scene;
  int b[3];
};

__device__ __forceinline__ BlockCoord decode_block(int key, const DevParams& P) {
  BlockCoord bc;
  if (P.n_scenes == 1 && P.nb_shift[1] >= 0 && P.nb_shift[2] >= 0) {   // power-of-two grids: shifts
    bc.scene = 0;
    bc.b[0] = key >> (P.nb_shift[1] + P.nb_shift[2]);
    bc.b[1] = (key >> P.nb_shift[2]) & (P.NB[1] - 1);
    bc.b[2] = key & (P.NB[2] - 1);
    return bc;
  }
  const int bps = (int)P.blocks_per_scene;
  bc.scene = key / bps;
  const int local = key - bc.scene * bps;
  const int plane = P.NB[1] * P.NB[2];
  bc.b[0] = local / plane;
  const int rem = local - bc.b[0] * plane;
  bc.b[1] = rem / P.NB[2];
  bc.b[2] = rem - bc.b[1] * P.NB[2];
  return bc;
}

// ---------------------------------------------------------------------------
// P2G (MLS force form)
constexpr int kP2GThreads = 192;   // 64 cells x 3 stencil planes (ox)
#ifndef NSF_P2G_ROWS
#define NSF_P2G_ROWS 12
#endif
#ifndef NSF_FUSED_MIN_BLOCKS
#define NSF_FUSED_MIN_BLOCKS 3
#endif
constexpr int kRows = NSF_P2G_ROWS;   // particles per cell per round
constexpr int kSlotFields = 21;    // w(9), u0(3), q0(3), q1(3), q2(3)
constexpr int kSlotStride = kRows * 64;   // floats per field
constexpr int kSegment = 1024;     // particles of one block handled per segment (smem: 3 CTAs/SM)

struct __align__(16) P2GSmem {
  union {
    float slot[kSlotFields * kSlotStride];   // [field][row][cell]
    float part[27 * 4 * 64];                 // [(node*4 + comp)][cell]
  } u;
  uint32_t cr[kSegment];   // (cell << 16) | rank within the cell, per particle of the segment
  int pop[64];             // cell populations of the segment
  int max_pop;
  int next;                // dynamically fetched block index
  uint16_t tbl[1728];      // tile-node reduction pairs (stencil node k << 6 | cell), grouped by tile node
  uint16_t tbl_off[218];   // pair range of tile node t: [tbl_off[t], tbl_off[t+1])
};

// (cell, stencil-offset) pairs feeding each of the 216 tile nodes, built once
__device__ __align__(16) uint16_t g_p2g_tbl[1728];
__device__ __align__(16) uint16_t g_p2g_tbl_off[224];   // 217 used; padded to 16-byte chunks

__global__ void k_p2g_tables() {
  const int t = threadIdx.x;   // tile node 0..215
  if (t >= 216) return;
  auto cnt1 = [](int n) { return min(3, n) - max(0, n - 2) + 1; };
  int off = 0;
  for (int u = 0; u < t; ++u) off += cnt1(u / 36) * cnt1((u / 6) % 6) * cnt1(u % 6);
  g_p2g_tbl_off[t] = (uint16_t)off;
  if (t == 215) g_p2g_tbl_off[216] = (uint16_t)(off + 1);
  const int nx = t / 36, ny = (t / 6) % 6, nz = t % 6;
  for (int cx = max(0, nx - 2); cx <= min(3, nx); ++cx)
    for (int cy = max(0, ny - 2); cy <= min(3, ny); ++cy)
      for (int cz = max(0, nz - 2); cz <= min(3, nz); ++cz) {
        const int k = ((nx - cx) * 3 + (ny - cy)) * 3 + (nz - cz);
        g_p2g_tbl[off++] = (uint16_t)((k << 6) | (cx << 4) | (cy << 2) | cz);
      }
}

void p2g_tables_init(cudaStream_t st) { k_p2g_tables<<<1, 256, 0, st>>>(); }

// one particle -> 21 floats of slot data at s = row*64 + cell
__device__ __forceinline__ void p2g_stage_particle(const float* __restrict__ S, int64_t pitch, int p, int s,
                                                   float* sl, const DevParams& P) {
  const float m = P.mass;
  const Axis a0 = bspline_axis(S[pbase(p) + (PX + 0) * 32], P.inv_dx);
  const Axis a1 = bspline_axis(S[pbase(p) + (PX + 1) * 32], P.inv_dx);
  const Axis a2 = bspline_axis(S[pbase(p) + (PX + 2) * 32], P.inv_dx);
  const float v0 = S[pbase(p) + (PV + 0) * 32], v1 = S[pbase(p) + (PV + 1) * 32], v2 = S[pbase(p) + (PV + 2) * 32];
  float Cm[9], T[6];
#pragma unroll
  for (int k = 0; k < 9; ++k) Cm[k] = S[pbase(p) + (PC + k) * 32];
#pragma unroll
  for (int k = 0; k < 6; ++k) T[k] = S[pbase(p) + (PT + k) * 32];
  const float Tm[9] = {T[0], T[5], T[4], T[5], T[1], T[3], T[4], T[3], T[2]};
  float Q[9];   // Q = m C - dt V0 (4/dx^2) tau  (MLS, reading #1)
#pragma unroll
  for (int k = 0; k < 9; ++k) Q[k] = P.mC * Cm[k] - P.mls_coef * Tm[k];
  // contribution to node base + o:  W_o [ m ; m v + Q (o - f) dx ] = W_o [ m ; u0 + dx Q o ]
  const float f0 = a0.f, f1 = a1.f, f2 = a2.f;
  const float u0x = m * v0 - P.dx * (Q[0] * f0 + Q[1] * f1 + Q[2] * f2);
  const float u0y = m * v1 - P.dx * (Q[3] * f0 + Q[4] * f1 + Q[5] * f2);
  const float u0z = m * v2 - P.dx * (Q[6] * f0 + Q[7] * f1 + Q[8] * f2);
  const float vals[kSlotFields] = {a0.w[0], a0.w[1], a0.w[2], a1.w[0], a1.w[1], a1.w[2], a2.w[0], a2.w[1], a2.w[2],
                                   u0x, u0y, u0z,
                                   P.dx * Q[0], P.dx * Q[3], P.dx * Q[6],
                                   P.dx * Q[1], P.dx * Q[4], P.dx * Q[7],
                                   P.dx * Q[2], P.dx * Q[5], P.dx * Q[8]};
#pragma unroll
  for (int k = 0; k < kSlotFields; ++k) sl[k * kSlotStride + s] = vals[k];
}

// one particle's slot data from its state values (same arithmetic as above)
__device__ __forceinline__ void p2g_stage_values(const float x[3], const float v[3], const float Cm[9], const float T[6],
                                                 int s, float* sl, const DevParams& P) {
  const float m = P.mass;
  const Axis a0 = bspline_axis(x[0], P.inv_dx), a1 = bspline_axis(x[1], P.inv_dx), a2 = bspline_axis(x[2], P.inv_dx);
  const float Tm[9] = {T[0], T[5], T[4], T[5], T[1], T[3], T[4], T[3], T[2]};
  float Q[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) Q[k] = P.mC * Cm[k] - P.mls_coef * Tm[k];
  const float f0 = a0.f, f1 = a1.f, f2 = a2.f;
  const float u0x = m * v[0] - P.dx * (Q[0] * f0 + Q[1] * f1 + Q[2] * f2);
  const float u0y = m * v[1] - P.dx * (Q[3] * f0 + Q[4] * f1 + Q[5] * f2);
  const float u0z = m * v[2] - P.dx * (Q[6] * f0 + Q[7] * f1 + Q[8] * f2);
  const float vals[kSlotFields] = {a0.w[0], a0.w[1], a0.w[2], a1.w[0], a1.w[1], a1.w[2], a2.w[0], a2.w[1], a2.w[2],
                                   u0x, u0y, u0z,
                                   P.dx * Q[0], P.dx * Q[3], P.dx * Q[6],
                                   P.dx * Q[1], P.dx * Q[4], P.dx * Q[7],
                                   P.dx * Q[2], P.dx * Q[5], P.dx * Q[8]};
#pragma unroll
  for (int k = 0; k < kSlotFields; ++k) sl[k * kSlotStride + s] = vals[k];
}

// MLS P2G of one particle straight to the global accumulator (27 x red.v4), marking
// every touched grid block in `flags` (used for particles outside their segment's
// block, and for cells with more than kRows particles)
// mark grid block `b` as touched; the first marker appends it to the work list of
// the next grid update
__device__ __forceinline__ void touch_block(int* flags, int* list, int* list_count, int b, const DevParams& P) {
  NSF_CHECK(b >= 0 && b < P.blocks_per_scene * P.n_scenes);
  if (flags[b] == 0 && atomicExch(&flags[b], 1) == 0) {
    const int e = atomicAdd(list_count, 1);
    NSF_CHECK(e < P.blocks_per_scene * P.n_scenes);
    list[e] = b;
  }
}

// Where a scattered particle's grid blocks are marked for the grid update.  With
// the halo list (HALO, separate grid-update pass): every block in the 27-block
// neighbourhood of a non-empty segment is updated anyway (k_halo, at each
// re-binning), so only a block outside it -- reached by a particle that drifted
// more than 4 cells from its segment -- goes through the flags and the touched list.
struct TouchCtx {
  int* flags;
  int* list;
  int* list_count;
  const int* hmark;   // HALO: per block, the epoch tag of the last halo list that held it
  const unsigned long long* scan_ticket;   // HALO: the current tag = scan ticket / scan tiles
  int64_t scan_tiles;
  int seg[3];         // HALO: the segment's block
  int64_t scene_block0;
};

template <bool HALO>
__device__ __forceinline__ void touch(const TouchCtx& t, int b0, int b1, int b2, const DevParams& P) {
  if (HALO) {
    if (abs(b0 - t.seg[0]) <= 1 && abs(b1 - t.seg[1]) <= 1 && abs(b2 - t.seg[2]) <= 1) return;
    const int B = (int)(t.scene_block0 + block_id(b0, b1, b2, P));
    if (t.hmark[B] == (int)(*(volatile const unsigned long long*)t.scan_ticket / (unsigned long long)t.scan_tiles))
      return;   // in the current halo (an older tag: a block that left it)
    touch_block(t.flags, t.list, t.list_count, B, P);
    return;
  }
  touch_block(t.flags, t.list, t.list_count, (int)(t.scene_block0 + block_id(b0, b1, b2, P)), P);
}

template <bool HALO>
__device__ __forceinline__ void p2g_scatter_direct(const float x[3], const float v[3], const float Cm[9],
                                                   const float T[6], float4* gbase, const TouchCtx& tc,
                                                   const DevParams& P) {
  const float m = P.mass;
  Axis ax[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    ax[a] = bspline_axis(x[a], P.inv_dx);
    ax[a].base = min(max(ax[a].base, 0), P.N[a] - 3);
  }
  const float Tm[9] = {T[0], T[5], T[4], T[5], T[1], T[3], T[4], T[3], T[2]};
  float Q[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) Q[k] = P.mC * Cm[k] - P.mls_coef * Tm[k];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const float W = ax[0].w[a] * ax[1].w[b] * ax[2].w[c];
        const float d0 = ((float)a - ax[0].f) * P.dx, d1 = ((float)b - ax[1].f) * P.dx, d2 = ((float)c - ax[2].f) * P.dx;
        const float mv0 = W * (m * v[0] + Q[0] * d0 + Q[1] * d1 + Q[2] * d2);
        const float mv1 = W * (m * v[1] + Q[3] * d0 + Q[4] * d1 + Q[5] * d2);
        const float mv2 = W * (m * v[2] + Q[6] * d0 + Q[7] * d1 + Q[8] * d2);
        NSF_CHECK(node_index(ax[0].base + a, ax[1].base + b, ax[2].base + c, P) < P.nodes_per_scene);
        red_add_v4_t(gbase + node_index(ax[0].base + a, ax[1].base + b, ax[2].base + c, P), W * m, mv0, mv1, mv2);
      }
  // touched blocks: per axis the blocks of base and base+2
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int b0 = (ax[0].base + 2 * a) >> 2, b1 = (ax[1].base + 2 * b) >> 2, b2 = (ax[2].base + 2 * c) >> 2;
        touch<HALO>(tc, b0, b1, b2, P);
      }
}

// Warp-cooperative form of p2g_scatter_direct: the lanes with `direct` set are
// taken one at a time, their particle broadcast by shuffles, and the active
// lanes of the warp each scatter some of its 27 nodes (and touch its 8 corner
// blocks).  A few direct particles per warp then cost ~21 shuffles + one node
// each instead of serialising 27 reductions while the other lanes idle.
template <bool HALO>
__device__ __forceinline__ void p2g_scatter_warp(bool direct, const float x[3], const float v[3], const float Cm[9],
                                                 const float T[6], float4* gbase, const TouchCtx& tc,
                                                 const DevParams& P) {
  const unsigned act = __activemask();
  unsigned pend = __ballot_sync(act, direct);
  if (!pend) return;
  const int lane = threadIdx.x & 31;
  const int r = __popc(act & ((1u << lane) - 1u));
  const int nact = __popc(act);
  const float m = P.mass;
  while (pend) {
    const int src = __ffs(pend) - 1;
    pend &= pend - 1;
    float px[3], pv[3], pC[9], pT[6];
#pragma unroll
    for (int a = 0; a < 3; ++a) { px[a] = __shfl_sync(act, x[a], src); pv[a] = __shfl_sync(act, v[a], src); }
#pragma unroll
    for (int k = 0; k < 9; ++k) pC[k] = __shfl_sync(act, Cm[k], src);
#pragma unroll
    for (int k = 0; k < 6; ++k) pT[k] = __shfl_sync(act, T[k], src);
    Axis ax[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      ax[a] = bspline_axis(px[a], P.inv_dx);
      ax[a].base = min(max(ax[a].base, 0), P.N[a] - 3);
    }
    const float Tm[9] = {pT[0], pT[5], pT[4], pT[5], pT[1], pT[3], pT[4], pT[3], pT[2]};
    float Q[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) Q[k] = P.mC * pC[k] - P.mls_coef * Tm[k];
    for (int node = r; node < 27; node += nact) {
      const int a = node / 9, b = (node / 3) % 3, c = node % 3;
      const float wa = a == 0 ? ax[0].w[0] : (a == 1 ? ax[0].w[1] : ax[0].w[2]);
      const float wb = b == 0 ? ax[1].w[0] : (b == 1 ? ax[1].w[1] : ax[1].w[2]);
      const float wc = c == 0 ? ax[2].w[0] : (c == 1 ? ax[2].w[1] : ax[2].w[2]);
      const float W = wa * wb * wc;
      const float d0 = ((float)a - ax[0].f) * P.dx, d1 = ((float)b - ax[1].f) * P.dx, d2 = ((float)c - ax[2].f) * P.dx;
      const float mv0 = W * (m * pv[0] + Q[0] * d0 + Q[1] * d1 + Q[2] * d2);
      const float mv1 = W * (m * pv[1] + Q[3] * d0 + Q[4] * d1 + Q[5] * d2);
      const float mv2 = W * (m * pv[2] + Q[6] * d0 + Q[7] * d1 + Q[8] * d2);
      NSF_CHECK(node_index(ax[0].base + a, ax[1].base + b, ax[2].base + c, P) < P.nodes_per_scene);
      red_add_v4_t(gbase + node_index(ax[0].base + a, ax[1].base + b, ax[2].base + c, P), W * m, mv0, mv1, mv2);
    }
    // touched blocks: per axis the blocks of base and base+2
    for (int k = r; k < 8; k += nact) {
      const int b0 = (ax[0].base + 2 * (k >> 2)) >> 2, b1 = (ax[1].base + 2 * ((k >> 1) & 1)) >> 2,
                b2 = (ax[2].base + 2 * (k & 1)) >> 2;
      touch<HALO>(tc, b0, b1, b2, P);
    }
  }
}

// thread (my_cell, ox) accumulates its cell's staged rows for stencil plane ox
__device__ __forceinline__ void p2g_accumulate(const float* sl, int my_cell, int ox, int rows, float accm[9],
                                               float accp[9][3]) {
  const float fox = (float)ox;
  for (int r = 0; r < rows; ++r) {
    const int s = r * 64 + my_cell;
    const float wx = sl[ox * kSlotStride + s];
    const float wyv[3] = {sl[3 * kSlotStride + s], sl[4 * kSlotStride + s], sl[5 * kSlotStride + s]};
    const float wzv[3] = {sl[6 * kSlotStride + s], sl[7 * kSlotStride + s], sl[8 * kSlotStride + s]};
    const float ux = fmaf(fox, sl[12 * kSlotStride + s], sl[9 * kSlotStride + s]);
    const float uy = fmaf(fox, sl[13 * kSlotStride + s], sl[10 * kSlotStride + s]);
    const float uz = fmaf(fox, sl[14 * kSlotStride + s], sl[11 * kSlotStride + s]);
    const float q1x = sl[15 * kSlotStride + s], q1y = sl[16 * kSlotStride + s], q1z = sl[17 * kSlotStride + s];
    const float q2x = sl[18 * kSlotStride + s], q2y = sl[19 * kSlotStride + s], q2z = sl[20 * kSlotStride + s];
#pragma unroll
    for (int oy = 0; oy < 3; ++oy) {
      const float wxy = wx * wyv[oy];
      const float uyx = oy ? fmaf((float)oy, q1x, ux) : ux, uyy = oy ? fmaf((float)oy, q1y, uy) : uy,
                  uyz = oy ? fmaf((float)oy, q1z, uz) : uz;   // fmaf(0, q, u) is not folded
#pragma unroll
      for (int oz = 0; oz < 3; ++oz) {
        const float W = wxy * wzv[oz];
        const int k = oy * 3 + oz;
        accm[k] += W;
        accp[k][0] = fmaf(W, oz ? fmaf((float)oz, q2x, uyx) : uyx, accp[k][0]);
        accp[k][1] = fmaf(W, oz ? fmaf((float)oz, q2y, uyy) : uyy, accp[k][1]);
        accp[k][2] = fmaf(W, oz ? fmaf((float)oz, q2z, uyz) : uyz, accp[k][2]);
      }
    }
  }
}

__device__ __forceinline__ int cell_in_block(const float* __restrict__ S, int64_t pitch, int p, const BlockCoord& bc,
                                             const DevParams& P) {
  int c[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float t = S[pbase(p) + (PX + a) * 32] * P.inv_dx;
    int base = (int)floorf(t - 0.5f);
    base = min(max(base, 0), P.N[a] - 3);
    c[a] = base - 4 * bc.b[a];
  }
  return (c[0] << 4) | (c[1] << 2) | c[2];
}

__global__ void __launch_bounds__(kP2GThreads, 3)
k_p2g_tiled(const float* __restrict__ S, int64_t pitch, const int32_t* __restrict__ perm,
            const int32_t* __restrict__ block_start, const int32_t* __restrict__ nonempty,
            int32_t* __restrict__ counters, float4* acc, DevParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  P2GSmem& sm = *reinterpret_cast<P2GSmem*>(smem_raw);
  const int tid = threadIdx.x;
  const int my_cell = tid & 63;
  const int ox = tid >> 6;
  const float fox = (float)ox;
  const int nblk = *(volatile int32_t*)&counters[0];
  for (int q = tid; q < 1728; q += kP2GThreads) sm.tbl[q] = g_p2g_tbl[q];
  for (int q = tid; q < 217; q += kP2GThreads) sm.tbl_off[q] = g_p2g_tbl_off[q];
  while (true) {
    if (tid == 0) sm.next = atomicAdd(&counters[3], 1);
    __syncthreads();
    const int bi = sm.next;
    if (bi >= nblk) break;
    const int key = nonempty[bi];
    const BlockCoord bc = decode_block(key, P);
    const int start = block_start[key], end = block_start[key + 1];
    float accm[9], accp[9][3];
#pragma unroll
    for (int k = 0; k < 9; ++k) { accm[k] = 0.f; accp[k][0] = accp[k][1] = accp[k][2] = 0.f; }
    for (int seg = start; seg < end; seg += kSegment) {
      const int cnt = min(kSegment, end - seg);
      __syncthreads();   // previous users of pop / part are done
      if (tid < 64) sm.pop[tid] = 0;
      if (tid == 0) sm.max_pop = 0;
      __syncthreads();
      // pass A: cell and rank of every particle of the segment; rows of round 0
      // are staged right away (the particle's x is already in registers)
      for (int i = tid; i < cnt; i += kP2GThreads) {
        const int p = perm[seg + i];
        const int cell = cell_in_block(S, pitch, p, bc, P);
        const int rank = atomicAdd(&sm.pop[cell], 1);
        sm.cr[i] = ((uint32_t)cell << 16) | (uint32_t)rank;
        if (rank < kRows) p2g_stage_particle(S, pitch, p, rank * 64 + cell, sm.u.slot, P);
      }
      __syncthreads();
      if (tid < 64) atomicMax(&sm.max_pop, sm.pop[tid]);
      __syncthreads();
      const int rounds = (sm.max_pop + kRows - 1) / kRows;
      const int my_pop = sm.pop[my_cell];
      for (int round = 0; round < rounds; ++round) {
        if (round > 0) {
          // pass B (rare: cells with more than kRows particles): stage this round's rows
          for (int i = tid; i < cnt; i += kP2GThreads) {
            const uint32_t cr = sm.cr[i];
            const int r = (int)(cr & 0xffffu) - round * kRows;
            if (r < 0 || r >= kRows) continue;
            p2g_stage_particle(S, pitch, perm[seg + i], r * 64 + (int)(cr >> 16), sm.u.slot, P);
          }
          __syncthreads();
        }
        // accumulate: thread (my_cell, ox) over its cell's rows in this round
        int rows = my_pop - round * kRows;
        rows = rows < 0 ? 0 : (rows > kRows ? kRows : rows);
        const float* sl = sm.u.slot;
        for (int r = 0; r < rows; ++r) {
          const int s = r * 64 + my_cell;
          const float wx = sl[ox * kSlotStride + s];
          const float wyv[3] = {sl[3 * kSlotStride + s], sl[4 * kSlotStride + s], sl[5 * kSlotStride + s]};
          const float wzv[3] = {sl[6 * kSlotStride + s], sl[7 * kSlotStride + s], sl[8 * kSlotStride + s]};
          const float ux = fmaf(fox, sl[12 * kSlotStride + s], sl[9 * kSlotStride + s]);
          const float uy = fmaf(fox, sl[13 * kSlotStride + s], sl[10 * kSlotStride + s]);
          const float uz = fmaf(fox, sl[14 * kSlotStride + s], sl[11 * kSlotStride + s]);
          const float q1x = sl[15 * kSlotStride + s], q1y = sl[16 * kSlotStride + s], q1z = sl[17 * kSlotStride + s];
          const float q2x = sl[18 * kSlotStride + s], q2y = sl[19 * kSlotStride + s], q2z = sl[20 * kSlotStride + s];
#pragma unroll
          for (int oy = 0; oy < 3; ++oy) {
            const float wxy = wx * wyv[oy];
            const float uyx = oy ? fmaf((float)oy, q1x, ux) : ux, uyy = oy ? fmaf((float)oy, q1y, uy) : uy,
                  uyz = oy ? fmaf((float)oy, q1z, uz) : uz;   // fmaf(0, q, u) is not folded
#pragma unroll
            for (int oz = 0; oz < 3; ++oz) {
              const float W = wxy * wzv[oz];
              const int k = oy * 3 + oz;
              accm[k] += W;
              accp[k][0] = fmaf(W, oz ? fmaf((float)oz, q2x, uyx) : uyx, accp[k][0]);
              accp[k][1] = fmaf(W, oz ? fmaf((float)oz, q2y, uyy) : uyy, accp[k][1]);
              accp[k][2] = fmaf(W, oz ? fmaf((float)oz, q2z, uyz) : uyz, accp[k][2]);
            }
          }
        }
        __syncthreads();   // slot buffer reused by the next round
      }
    }
    // partials -> shared memory [(node*4 + comp)][cell]   (aliases the slot buffer)
    float* part = sm.u.part;
    const float m = P.mass;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const int node = ox * 9 + k;
      part[(node * 4 + 0) * 64 + my_cell] = accm[k] * m;
      part[(node * 4 + 1) * 64 + my_cell] = accp[k][0];
      part[(node * 4 + 2) * 64 + my_cell] = accp[k][1];
      part[(node * 4 + 3) * 64 + my_cell] = accp[k][2];
    }
    __syncthreads();
    // reduce each node of the 6x6x6 tile over the cells whose stencil covers it
    float4* gbase = acc + (int64_t)bc.scene * P.nodes_per_scene;
    for (int t = tid; t < 216; t += kP2GThreads) {
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
      const int q1 = sm.tbl_off[t + 1];
      for (int q = sm.tbl_off[t]; q < q1; ++q) {
        const int pr = sm.tbl[q];
        const float* pp = part + (pr >> 6) * 256 + (pr & 63);   // [(k*4 + comp)*64 + cell]
        s0 += pp[0];
        s1 += pp[64];
        s2 += pp[128];
        s3 += pp[192];
      }
      if (s0 > 0.0f) {
        const int nx = t / 36, ny = (t / 6) % 6, nz = t % 6;
        const int gi = 4 * bc.b[0] + nx, gj = 4 * bc.b[1] + ny, gk = 4 * bc.b[2] + nz;
        if (gi < P.N[0] && gj < P.N[1] && gk < P.N[2])
          red_add_v4_t(gbase + node_index(gi, gj, gk, P), s0, s1, s2, s3);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// grid update over the blocks touched by P2G.  Target block t = b + d,
// d in {0,1}^3, is owned by the first non-empty block t - d' in the fixed order
// d' = (0,0,0), (0,0,1), ..., (1,1,1); the owner updates its 64 nodes.

__device__ __forceinline__ int count_of(const int32_t* bs, int scene, int b0, int b1, int b2, const DevParams& P) {
  if (b0 < 0 || b1 < 0 || b2 < 0) return 0;
  int64_t k = (int64_t)scene * P.blocks_per_scene + block_id(b0, b1, b2, P);
  return bs[k + 1] - bs[k];
}

__device__ __forceinline__ float4 grid_node_update_t(float4 a, int i, int j, int k, const DevParams& P, float y_plate) {
  float m = a.x;
  if (!(m > 0.0f)) return make_float4(0.f, 0.f, 0.f, 0.f);
  float v[3] = {a.y / m + P.dt * P.g[0], a.z / m + P.dt * P.g[1], a.w / m + P.dt * P.g[2]};
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
  if (P.plate_enabled && (float)j * P.dx >= y_plate) { v[0] = P.plate_v[0]; v[1] = P.plate_v[1]; v[2] = P.plate_v[2]; }
  return make_float4(v[0], v[1], v[2], m);
}

// The same update (readings #11-#14) for nodes updated inside the fused
// kernel: one correctly rounded reciprocal of m_i and three products instead of
// three IEEE divisions (<= 1.5 ulp apart); `in_walls` is false when the caller
// knows the node lies outside every wall region (then only the plate applies).
__device__ __forceinline__ float4 grid_node_update_rcp(float4 a, int i, int j, int k, const DevParams& P, float y_plate,
                                                       bool in_walls = true) {
  const float m = a.x;
  if (!(m > 0.0f)) return make_float4(0.f, 0.f, 0.f, 0.f);
  const float r = __frcp_rn(m);
  float v[3] = {fmaf(a.y, r, P.dt * P.g[0]) , fmaf(a.z, r, P.dt * P.g[1]), fmaf(a.w, r, P.dt * P.g[2])};
  if (in_walls) {
    const int idx[3] = {i, j, k};
#pragma unroll
    for (int face = 0; face < 6; ++face) {
      const int kind = P.bc[face];
      if (kind == 0) continue;
      const int axis = face >> 1;
      const bool high = face & 1;
      const bool in = high ? (idx[axis] >= P.N[axis] - P.bc_width) : (idx[axis] < P.bc_width);
      if (!in) continue;
      if (kind == 1) { v[0] = v[1] = v[2] = 0.0f; }
      else v[axis] = high ? fminf(v[axis], 0.0f) : fmaxf(v[axis], 0.0f);
    }
  }
  if (P.plate_enabled && (float)j * P.dx >= y_plate) { v[0] = P.plate_v[0]; v[1] = P.plate_v[1]; v[2] = P.plate_v[2]; }
  return make_float4(v[0], v[1], v[2], m);
}

__device__ __forceinline__ float plate_y_at(const DevParams& P, int64_t step) {
  return (float)((double)P.plate_y0 + (double)P.plate_v[1] * ((double)step * (double)P.dt));
}

__global__ void __launch_bounds__(128)
k_grid_update_blocks(const int32_t* __restrict__ block_start, const int32_t* __restrict__ nonempty,
                     int32_t* __restrict__ n_nonempty, float4* acc, float4* vel,
                     DevParams P, const int64_t* __restrict__ d_step) {
  // one warp per non-empty source block b; it owns target t = b + d (d in {0,1}^3)
  // when no source t - e with e < d (in the enumeration order) is non-empty.
  const int nblk = *n_nonempty;
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const float y_plate = (float)((double)P.plate_y0 + (double)P.plate_v[1] * ((double)(*d_step) * (double)P.dt));
  for (int bi = warp; bi < nblk; bi += nwarps) {
    const int key = nonempty[bi];
    const BlockCoord bc = decode_block(key, P);
    // bit s of `nb`: source b + (s0-1, s1-1, s2-1) is non-empty, s = s0*9 + s1*3 + s2
    bool has = false;
    if (lane < 27) {
      const int n0 = bc.b[0] + lane / 9 - 1, n1 = bc.b[1] + (lane / 3) % 3 - 1, n2 = bc.b[2] + lane % 3 - 1;
      has = n0 >= 0 && n1 >= 0 && n2 >= 0 && n0 < P.NB[0] && n1 < P.NB[1] && n2 < P.NB[2] &&
            count_of(block_start, bc.scene, n0, n1, n2, P) > 0;
    }
    const unsigned nb = __ballot_sync(0xffffffffu, has);
    float4 a[8][2];
    int64_t g[8];
    unsigned own = 0;
#pragma unroll
    for (int d = 0; d < 8; ++d) {
      const int d0 = (d >> 2) & 1, d1 = (d >> 1) & 1, d2 = d & 1;
      const int t0 = bc.b[0] + d0, t1 = bc.b[1] + d1, t2 = bc.b[2] + d2;
      bool owner = t0 < P.NB[0] && t1 < P.NB[1] && t2 < P.NB[2];
#pragma unroll
      for (int e = 0; e < d; ++e) {
        const int e0 = (e >> 2) & 1, e1 = (e >> 1) & 1, e2 = e & 1;
        if (nb & (1u << (((d0 - e0 + 1) * 3 + (d1 - e1 + 1)) * 3 + (d2 - e2 + 1)))) owner = false;
      }
      g[d] = (int64_t)bc.scene * P.nodes_per_scene + block_id(t0, t1, t2, P) * kBlockNodes;
      if (owner) {
        own |= 1u << d;
        a[d][0] = acc[g[d] + lane];
        a[d][1] = acc[g[d] + lane + 32];
      }
    }
#pragma unroll
    for (int d = 0; d < 8; ++d) {
      if (!(own & (1u << d))) continue;
      const int t0 = bc.b[0] + ((d >> 2) & 1), t1 = bc.b[1] + ((d >> 1) & 1), t2 = bc.b[2] + (d & 1);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int l = lane + 32 * h;
        const int i = t0 * 4 + (l >> 4), j = t1 * 4 + ((l >> 2) & 3), k = t2 * 4 + (l & 3);
        vel[g[d] + l] = grid_node_update_t(a[d][h], i, j, k, P, y_plate);
        acc[g[d] + l] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// G2P + constitutive (a5 + a6), sort-on-write.
struct PState {
  float x[3];
  float F[9];
  int id;
};

__device__ __forceinline__ void load_pstate(PState& s, const float* __restrict__ S, int p,
                                            const int32_t* __restrict__ ids) {
  const float* base = S + pbase(p);
#pragma unroll
  for (int a = 0; a < 3; ++a) s.x[a] = __ldg(base + (PX + a) * 32);
#pragma unroll
  for (int k = 0; k < 9; ++k) s.F[k] = __ldg(base + (PF + k) * 32);
  s.id = __ldg(ids + p);
}

// G2P gather: v_p = sum w v_i, C_p = 4/dx^2 sum w v_i (x_i - x_p)^T and the
// velocity gradient G for the F update (= C_p in MLS form, sum v_i grad(w)^T in GRADW
// form), from the blocked grid velocities vb (read through L1).  Separable sums:
// per stencil plane a, T = sum w_y w_z v, Ty = sum o_y w_y w_z v, Tz = sum o_z w_y w_z v;
// then v = sum w_x T and B = dx (M - v f^T) with M_ij = sum W v_i o_j.
template <int FORCE, bool RAW = false>
__device__ __forceinline__ void g2p_gather(const float x[3], const float4* __restrict__ vb, const DevParams& P,
                                           float v[3], float Cn[9], float G[9], float y_plate = 0.0f) {
#pragma unroll
  for (int k = 0; k < 3; ++k) v[k] = 0.f;
#pragma unroll
  for (int k = 0; k < 9; ++k) G[k] = 0.f;
  const float cC = 4.0f * P.inv_dx;   // C = (4/dx) (M - v f^T) = 4/dx^2 B (b = 2)
  Axis ax[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    ax[a] = bspline_axis(x[a], P.inv_dx);
    ax[a].base = min(max(ax[a].base, 0), P.N[a] - 3);
  }
  int X[3], Y[3], Z[3];
  {
    const int plane = P.NB[1] * P.NB[2] * kBlockNodes;
#pragma unroll
    for (int o = 0; o < 3; ++o) {
      const int i = ax[0].base + o, jj = ax[1].base + o, k = ax[2].base + o;
      X[o] = (i >> 2) * plane + ((i & 3) << 4);
      Y[o] = (jj >> 2) * (P.NB[2] * kBlockNodes) + ((jj & 3) << 2);
      Z[o] = (k >> 2) * kBlockNodes + (k & 3);
    }
  }
  float wyz[9];
#pragma unroll
  for (int b = 0; b < 3; ++b)
#pragma unroll
    for (int c = 0; c < 3; ++c) wyz[b * 3 + c] = ax[1].w[b] * ax[2].w[c];
  float M[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    float Tt[3] = {0.f, 0.f, 0.f}, Ty[3] = {0.f, 0.f, 0.f}, Tz[3] = {0.f, 0.f, 0.f};
    float Dy[3] = {0.f, 0.f, 0.f}, Dz[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        // RAW: vb holds the P2G sums (m, m v); the node is updated here
        const float4 vi = RAW ? grid_node_update_rcp(__ldcg(vb + (X[a] + Y[b] + Z[c])), ax[0].base + a,
                                                     ax[1].base + b, ax[2].base + c, P, y_plate)
                              : __ldg(vb + (X[a] + Y[b] + Z[c]));
        const float wgt = wyz[b * 3 + c];
        Tt[0] = fmaf(wgt, vi.x, Tt[0]); Tt[1] = fmaf(wgt, vi.y, Tt[1]); Tt[2] = fmaf(wgt, vi.z, Tt[2]);
        if (b) {
          const float wb = (float)b * wgt;
          Ty[0] = fmaf(wb, vi.x, Ty[0]); Ty[1] = fmaf(wb, vi.y, Ty[1]); Ty[2] = fmaf(wb, vi.z, Ty[2]);
        }
        if (c) {
          const float wc = (float)c * wgt;
          Tz[0] = fmaf(wc, vi.x, Tz[0]); Tz[1] = fmaf(wc, vi.y, Tz[1]); Tz[2] = fmaf(wc, vi.z, Tz[2]);
        }
        if (FORCE == 1) {
          const float gy = ax[1].dw[b] * ax[2].w[c], gz = ax[1].w[b] * ax[2].dw[c];
          Dy[0] = fmaf(gy, vi.x, Dy[0]); Dy[1] = fmaf(gy, vi.y, Dy[1]); Dy[2] = fmaf(gy, vi.z, Dy[2]);
          Dz[0] = fmaf(gz, vi.x, Dz[0]); Dz[1] = fmaf(gz, vi.y, Dz[1]); Dz[2] = fmaf(gz, vi.z, Dz[2]);
        }
      }
    const float wx = ax[0].w[a];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      v[i] = fmaf(wx, Tt[i], v[i]);
      if (a) M[i * 3 + 0] = fmaf((float)a * wx, Tt[i], M[i * 3 + 0]);
      M[i * 3 + 1] = fmaf(wx, Ty[i], M[i * 3 + 1]);
      M[i * 3 + 2] = fmaf(wx, Tz[i], M[i * 3 + 2]);
      if (FORCE == 1) {
        G[i * 3 + 0] = fmaf(ax[0].dw[a], Tt[i], G[i * 3 + 0]);
        G[i * 3 + 1] = fmaf(wx, Dy[i], G[i * 3 + 1]);
        G[i * 3 + 2] = fmaf(wx, Dz[i], G[i * 3 + 2]);
      }
    }
  }
  const float f[3] = {ax[0].f, ax[1].f, ax[2].f};
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int jj = 0; jj < 3; ++jj) Cn[i * 3 + jj] = cC * fmaf(-v[i], f[jj], M[i * 3 + jj]);
  if (FORCE == 0) {
#pragma unroll
    for (int k = 0; k < 9; ++k) G[k] = Cn[k];
  }
  if (P.rpic) skew_part(Cn);   // RPIC: the transfer's C_p; G keeps the full gradient
}

#ifndef NSF_G2P_FLAT_MIN_BLOCKS
#define NSF_G2P_FLAT_MIN_BLOCKS 7
#endif
template <int FORCE>
__global__ void __launch_bounds__(128, NSF_G2P_FLAT_MIN_BLOCKS)
k_g2p_flat(const float* __restrict__ Sin, float* __restrict__ Sout, int64_t n,
           const int32_t* __restrict__ ids_in, int32_t* __restrict__ ids_out,
           const int32_t* __restrict__ perm, const float4* __restrict__ vel, const int64_t* __restrict__ scene_off,
           int n_scenes, int32_t* __restrict__ keys, int32_t* __restrict__ counts, DevParams P, DevErr* err,
           int64_t* d_step) {
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd((unsigned long long*)d_step, 1ull);
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const unsigned active = __ballot_sync(0xffffffffu, j < n);
  if (j >= n) return;
  const int lane = threadIdx.x & 31;
  const int p = perm[j];
  PState st;
  load_pstate(st, Sin, p, ids_in);
  // scenes stay contiguous and in order in the sorted slot order
  const int bps = (int)P.blocks_per_scene;
  int scene = 0;
  if (n_scenes > 1) {
    int lo = 0, hi = n_scenes;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (scene_off[mid] <= j) lo = mid; else hi = mid;
    }
    scene = lo;
  }
  const float4* vb = vel + (int64_t)scene * P.nodes_per_scene;
  float v[3], Cn[9], G[9];
  g2p_gather<FORCE>(st.x, vb, P, v, Cn, G);
  float xn[3];
  bool ok = true;
  float* ob = Sout + pbase(j);
  float chk = 0.0f;   // any NaN/Inf makes the sum non-finite
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    xn[a] = st.x[a] + P.dt * v[a];
    const float tt = xn[a] * P.inv_dx;
    ok &= !(tt < 0.5f || tt >= (float)P.N[a] - 1.5f);   // NaN: non-finite, not out of domain
    ob[(PX + a) * 32] = xn[a];
    ob[(PV + a) * 32] = v[a];
    chk += xn[a] + v[a];
  }
#pragma unroll
  for (int k = 0; k < 9; ++k) ob[(PC + k) * 32] = Cn[k];
  ids_out[j] = st.id;
  // next block key + histogram (needs only x^{n+1})
  {
    int nb[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      int base = (int)floorf(xn[a] * P.inv_dx - 0.5f);
      base = min(max(base, 0), P.N[a] - 3);
      nb[a] = base >> 2;
    }
    const int nkey = scene * bps + (int)block_id(nb[0], nb[1], nb[2], P);
    keys[j] = nkey;
    const unsigned peers = __match_any_sync(active, nkey);
    if (lane == __ffs(peers) - 1) atomicAdd(&counts[nkey], __popc(peers));
  }
  float Ft[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int jj = 0; jj < 3; ++jj)
      Ft[i * 3 + jj] = st.F[i * 3 + jj] + P.dt * (G[i * 3 + 0] * st.F[0 * 3 + jj] + G[i * 3 + 1] * st.F[1 * 3 + jj] +
                                                  G[i * 3 + 2] * st.F[2 * 3 + jj]);
  float FE[9], tau[6];
  float J;
  float tY = Sin[pbase(p) + PTY * 32];
  if (P.vm_hs) {   // per-particle yield stress
    J = vm_hs_update(Ft, P.mu, P.lam, P.vm_hard_k, P.vm_soft, tY, FE, tau);
  } else {
    J = P.model == 5 ? hb_update(Ft, P.mu, P.kappa, P.hb_yield, P.hb_relax, FE, tau)
                     : elastoplastic_fast(Ft, P.model, P.mu, P.lam, P.alpha, P.tau_Y, FE, tau);
  }
  ob[PTY * 32] = tY;
#pragma unroll
  for (int k = 0; k < 9; ++k) { ob[(PF + k) * 32] = FE[k]; chk += FE[k]; }
#pragma unroll
  for (int k = 0; k < 6; ++k) { ob[(PT + k) * 32] = tau[k]; chk += tau[k]; }
  if (!(J > 0.0f)) atomicAdd(&err->inverted, 1ull);
  if (!ok) { atomicOr(&err->bits, ERR_OUT_OF_DOMAIN); atomicMin(&err->first_index, st.id); }
  if (!isfinite(chk)) { atomicOr(&err->bits, ERR_NONFINITE); atomicMin(&err->first_index, st.id); }
}

// ---------------------------------------------------------------------------
static int g_num_sms = 0;
int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return g_num_sms;
}

void launch_p2g_tiled(cudaStream_t st, const float* S, int64_t pitch, const int32_t* perm, const PipelineBuffers* pb,
                      float4* acc, const DevParams& P) {
  static bool attr = false;
  const size_t smem = sizeof(P2GSmem);
  if (!attr) {
    cudaFuncSetAttribute(k_p2g_tiled, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  int grid = num_sms() * 3;
  k_p2g_tiled<<<grid, kP2GThreads, smem, st>>>(S, pitch, perm, pb->block_start, pb->nonempty, pb->n_nonempty, acc, P);
  (void)0;
}

void launch_grid_update_blocks(cudaStream_t st, const PipelineBuffers* pb, float4* acc, float4* vel,
                               const DevParams& P, const int64_t* d_step) {
  // about one touched-source block per CTA: latency of the ownership lookups is
  // hidden by many resident CTAs rather than by a persistent loop
  int grid = num_sms() * 8;   // 4 warps per CTA, one source block per warp iteration
  k_grid_update_blocks<<<grid, 128, 0, st>>>(pb->block_start, pb->nonempty, pb->n_nonempty, acc, vel, P, d_step);
}

__global__ void k_bump_step(int64_t* d_step) { atomicAdd((unsigned long long*)d_step, 1ull); }

void launch_g2p_tiled(cudaStream_t st, const float* Sin, float* Sout, int64_t n, const int32_t* ids_in,
                      int32_t* ids_out, const PipelineBuffers* pb, const float4* vel, const int64_t* scene_off,
                      int n_scenes, const DevParams& P, DevErr* err, int64_t* d_step) {
  if (n == 0) {
    k_bump_step<<<1, 1, 0, st>>>(d_step);
    return;
  }
  const unsigned g = (unsigned)((n + 127) / 128);
  if (P.force_mode == 0)
    k_g2p_flat<0><<<g, 128, 0, st>>>(Sin, Sout, n, ids_in, ids_out, pb->perm, vel, scene_off, n_scenes, pb->keys,
                                     pb->counts, P, err, d_step);
  else
    k_g2p_flat<1><<<g, 128, 0, st>>>(Sin, Sout, n, ids_in, ids_out, pb->perm, vel, scene_off, n_scenes, pb->keys,
                                     pb->counts, P, err, d_step);
}

}  // namespace nsf

namespace nsf {
static_assert(sizeof(P2GSmem) + 1024 <= 228 * 1024 / NSF_FUSED_MIN_BLOCKS, "shared memory must allow the CTAs per SM");
// ===========================================================================
// Fused pipeline (MLS, full-order models): G2P of substep n and P2G of substep
// n+1 in one kernel, over storage segments.
//
// Storage is sorted by 4x4x4-cell block at the last re-binning (every
// kRebinEvery substeps, or at load); segment k = the particles that were in
// block k then.  For each segment one CTA
//   1. runs G2P(n) + the constitutive update for its particles (grid velocities
//      gathered through L1) and writes the new state in place;
//   2. stages the new state's P2G data by cell for the particles still inside
//      block k (register accumulation per (cell, stencil plane), then one
//      red.global.add.v4 per node of the thread's 3x3 plane: the L2 sums the
//      up to 27 cell partials of a node), and scatters particles that left the
//      block (or overflow a cell) directly with 27 red.global.add.v4;
//   3. marks every grid block it touched in `flags`.
// The grid update then visits exactly the flagged blocks.  Re-binning only
// restores locality; correctness does not depend on it.
#ifndef NSF_FUSED_VTILE
#define NSF_FUSED_VTILE 1                      // G2P reads a shared-memory velocity tile (else global gathers)
#endif
#ifndef NSF_DENSE_THREADS
#define NSF_DENSE_THREADS 256                  // dense variant: threads per CTA (>= 192): a full 512-particle
#endif                                         // block is exactly two phase-1 passes
#ifndef NSF_DENSE_MIN_BLOCKS
#define NSF_DENSE_MIN_BLOCKS NSF_FUSED_MIN_BLOCKS   // dense variant: CTAs per SM
#endif
#ifndef NSF_DENSE_ROWS
#define NSF_DENSE_ROWS 10
#endif
constexpr int kRowsF = NSF_DENSE_ROWS;         // dense variant: staged rows per cell
#ifndef NSF_SPARSE_ROWS
#define NSF_SPARSE_ROWS 6                      // sparse variant (few particles per block)
#endif
#ifndef NSF_SPARSE_MIN_BLOCKS
#define NSF_SPARSE_MIN_BLOCKS 4
#endif
#ifndef NSF_WARP_SCATTER
#define NSF_WARP_SCATTER 1                     // direct scatters are done warp-cooperatively
#endif   // staged rows per cell in the fused kernel

// Particles whose new cell lies outside the segment's block (or beyond the
// staged rows of their cell) are listed in shared memory during phase 1 and
// scattered node-parallel in phase 2, by the warps that do not accumulate (NT >
// 192) or by all threads before accumulating; only list overflow is scattered
// inline (warp-cooperatively), which stalls its warp on the block-flag loads.
#ifndef NSF_PF_NEXT
#define NSF_PF_NEXT 1                          // phase 1 loads the next particle's x, F a pass ahead
#endif
#ifndef NSF_SCATTER_CAP
#define NSF_SCATTER_CAP 40
#endif
constexpr int kScatterCap = NSF_SCATTER_CAP;

constexpr int kVT = 8;                         // velocity tile edge: nodes [4b-1, 4b+7)
// padded strides of the tile (in float4): a warp's lanes differ mostly within one
// 4-cell block, so with 8-float4 rows the 16-byte bank group (index mod 8) would
// take only 4 values; strides 9 (y) and 74 (x) spread (x, y, z) over all 8
// (simulated: 13.2 -> 9.5 shared wavefronts per warp-wide LDS.128)
constexpr int kVTy = 9, kVTx = 74;
constexpr int kVTSize = (kVT - 1) * (kVTx + kVTy + 1) + 1;   // 589

// Staged P2G row of one particle (24 floats = 6 float4): w_x(3) w_y(3) w_z(3),
// u = m v - dx Q f (3), dx Q e_x (3), dx Q e_y (3), dx Q e_z (3), packed stencil
// base (scatter list only), 2 pad.  Slots are [cell][row] with an odd cell
// stride in float4, so a warp of 32 cells reading the same row is conflict-free.
constexpr int kRowF4 = 6;
template <int ROWS>
struct FusedSlots {
  static constexpr int kCellStride4 = ROWS * kRowF4 + 1;
};

template <int ROWS>
struct __align__(16) FusedSmemT {
  float4 vt[NSF_FUSED_VTILE ? kVTSize : 1];   // G2P velocity tile (9.4 KB, padded strides)
  float4 slot[64 * FusedSlots<ROWS>::kCellStride4];
  float4 sc[kScatterCap * kRowF4];             // out-of-block particles: staged rows (+ packed base)
  int pop[64];
  int next;                                    // the next segment: ticket, block key and storage range
  int nkey, ns0, ns1;                          //   (fetched by thread NT - 1 during phase 1)
  int nsc;                                     // entries of sc this segment
  unsigned long long tbar;                     // mbarrier of the velocity tile's bulk copies (NSF_TILE_TMA)
};
static_assert(sizeof(FusedSmemT<kRowsF>) + 1024 <= 228 * 1024 / NSF_DENSE_MIN_BLOCKS, "fused kernel: CTAs per SM");
static_assert(sizeof(FusedSmemT<NSF_SPARSE_ROWS>) + 1024 <= 228 * 1024 / NSF_SPARSE_MIN_BLOCKS,
              "fused kernel (sparse): CTAs per SM");

__device__ __forceinline__ void cp_async16_f(void* smem, const void* gmem, int src_bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(src_bytes) : "memory");
}

// Velocity tile by TMA bulk copies (cp.async.bulk, SASS UBLKCP; north star: "TMA-staged
// grid tiles").  The grid is stored in 4x4x4-node blocks, so a tile row (fixed x, y; 8
// nodes in z from 4 b_z - 1) is three contiguous runs: 1 node of block b_z - 1 (16 B),
// 4 of block b_z (64 B), 3 of block b_z + 1 (48 B); 64 rows x 3 runs = 192 copies, one
// per thread, straight into the padded tile layout, all completing on one mbarrier
// (every thread arrives, the copying ones with their byte count).  Runs outside the
// grid are zero-filled by their thread.
// Measured (same-box A/B, -DNSF_TILE_TMA=1, parity-green): C3 103.0 vs 88.2 us per substep,
// C2 37.9 vs 35.2, C4 1363 vs 1174 -- 192 requests of 16-64 bytes per tile cost the TMA
// unit more than the 512 16-byte LDGSTS they replace (and the 96-register instantiation
// spills 128 bytes with them), so the default stays cp.async; kept as an A/B option.
#ifndef NSF_TILE_TMA
#define NSF_TILE_TMA 0
#endif
__device__ __forceinline__ unsigned smem_addr_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void tile_bar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// (the arrival's state token names the phase to wait for: no loop-carried parity register)
__device__ __forceinline__ unsigned long long tile_bar_arrive(unsigned long long* bar, int tx_bytes) {
  unsigned long long tok;
  if (tx_bytes)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 %0, [%1], %2;"
                 : "=l"(tok) : "r"(smem_addr_u32(bar)), "r"(tx_bytes) : "memory");
  else
    asm volatile("mbarrier.arrive.shared::cta.b64 %0, [%1];" : "=l"(tok) : "r"(smem_addr_u32(bar)) : "memory");
  return tok;
}
__device__ __forceinline__ void tile_bar_wait(unsigned long long* bar, unsigned long long tok) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "TILE_WAIT_%=:\n\t"
      "mbarrier.try_wait.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TILE_WAIT_%=;\n\t}" ::"r"(smem_addr_u32(bar)), "l"(tok)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, int bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr_u32(smem)),
               "l"(gmem), "r"(bytes), "r"(smem_addr_u32(bar))
               : "memory");
}

#ifndef NSF_P2G_ROW_UNROLL
#define NSF_P2G_ROW_UNROLL 1   // 2: phase-2 row loop unrolled by two
#endif
#ifndef NSF_F2_G2P
#define NSF_F2_G2P 1   // G2P gather on paired fp32 FMA (FFMA2, sm_100)
#endif
#ifndef NSF_F2_P2G
#define NSF_F2_P2G 1   // P2G accumulation on paired fp32 FMA / MUL / ADD (sm_100)
#endif

// G2P gather (MLS) from the shared 8^3 velocity tile whose node (0,0,0) is grid
// node o[]; the 27 reads are one shared base address plus immediate offsets.
// NSF_F2_G2P: the x, y components of every sum run as one paired FMA (the weight is a
// broadcast scalar operand, the pair is the node's (v_x, v_y) straight from its
// 16-byte shared load); the same operations per component as the scalar form.
__device__ __forceinline__ void g2p_gather_tile(const float x[3], const float4* vt, const int o[3], const DevParams& P,
                                                float v[3], float Cn[9]) {
  Axis ax[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) ax[a] = bspline_axis(x[a], P.inv_dx);
  NSF_CHECK(ax[0].base - o[0] >= 0 && ax[0].base - o[0] <= kVT - 3 && ax[1].base - o[1] >= 0 &&
            ax[1].base - o[1] <= kVT - 3 && ax[2].base - o[2] >= 0 && ax[2].base - o[2] <= kVT - 3);
  const float4* tp = vt + (ax[0].base - o[0]) * kVTx + (ax[1].base - o[1]) * kVTy + (ax[2].base - o[2]);
  float wyz[9];
#pragma unroll
  for (int b = 0; b < 3; ++b)
#pragma unroll
    for (int c = 0; c < 3; ++c) wyz[b * 3 + c] = ax[1].w[b] * ax[2].w[c];
#if NSF_F2_G2P
  // M[i][j] = sum W v_i o_j as pairs over i = (x, y) plus the z scalar
  float2 v01 = make_float2(0.f, 0.f), M01[3] = {v01, v01, v01};
  float v2 = 0.f, M2[3] = {0.f, 0.f, 0.f};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    float2 T01 = make_float2(0.f, 0.f), Ty01 = T01, Tz01 = T01;
    float T2 = 0.f, Ty2 = 0.f, Tz2 = 0.f;
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const float4 vi = tp[a * kVTx + b * kVTy + c];
        const float2 vxy = make_float2(vi.x, vi.y);
        const float wgt = wyz[b * 3 + c];
        T01 = __ffma2_rn(make_float2(wgt, wgt), vxy, T01);
        T2 = fmaf(wgt, vi.z, T2);
        if (b) {
          const float wb = (float)b * wgt;
          Ty01 = __ffma2_rn(make_float2(wb, wb), vxy, Ty01);
          Ty2 = fmaf(wb, vi.z, Ty2);
        }
        if (c) {
          const float wc = (float)c * wgt;
          Tz01 = __ffma2_rn(make_float2(wc, wc), vxy, Tz01);
          Tz2 = fmaf(wc, vi.z, Tz2);
        }
      }
    const float wx = ax[0].w[a];
    v01 = __ffma2_rn(make_float2(wx, wx), T01, v01);
    v2 = fmaf(wx, T2, v2);
    if (a) {
      const float awx = (float)a * wx;
      M01[0] = __ffma2_rn(make_float2(awx, awx), T01, M01[0]);
      M2[0] = fmaf(awx, T2, M2[0]);
    }
    M01[1] = __ffma2_rn(make_float2(wx, wx), Ty01, M01[1]);
    M2[1] = fmaf(wx, Ty2, M2[1]);
    M01[2] = __ffma2_rn(make_float2(wx, wx), Tz01, M01[2]);
    M2[2] = fmaf(wx, Tz2, M2[2]);
  }
  v[0] = v01.x; v[1] = v01.y; v[2] = v2;
  float M[9];
#pragma unroll
  for (int j = 0; j < 3; ++j) { M[0 * 3 + j] = M01[j].x; M[1 * 3 + j] = M01[j].y; M[2 * 3 + j] = M2[j]; }
#else
  float M[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  v[0] = v[1] = v[2] = 0.f;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    float Tt[3] = {0.f, 0.f, 0.f}, Ty[3] = {0.f, 0.f, 0.f}, Tz[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const float4 vi = tp[a * kVTx + b * kVTy + c];
        const float wgt = wyz[b * 3 + c];
        Tt[0] = fmaf(wgt, vi.x, Tt[0]); Tt[1] = fmaf(wgt, vi.y, Tt[1]); Tt[2] = fmaf(wgt, vi.z, Tt[2]);
        if (b) {
          const float wb = (float)b * wgt;
          Ty[0] = fmaf(wb, vi.x, Ty[0]); Ty[1] = fmaf(wb, vi.y, Ty[1]); Ty[2] = fmaf(wb, vi.z, Ty[2]);
        }
        if (c) {
          const float wc = (float)c * wgt;
          Tz[0] = fmaf(wc, vi.x, Tz[0]); Tz[1] = fmaf(wc, vi.y, Tz[1]); Tz[2] = fmaf(wc, vi.z, Tz[2]);
        }
      }
    const float wx = ax[0].w[a];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      v[i] = fmaf(wx, Tt[i], v[i]);
      if (a) M[i * 3 + 0] = fmaf((float)a * wx, Tt[i], M[i * 3 + 0]);
      M[i * 3 + 1] = fmaf(wx, Ty[i], M[i * 3 + 1]);
      M[i * 3 + 2] = fmaf(wx, Tz[i], M[i * 3 + 2]);
    }
  }
#endif
  const float cC = 4.0f * P.inv_dx;
  const float f[3] = {ax[0].f, ax[1].f, ax[2].f};
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int jj = 0; jj < 3; ++jj) Cn[i * 3 + jj] = cC * fmaf(-v[i], f[jj], M[i * 3 + jj]);
}

// Staged P2G row of one particle (6 float4), laid out so that every pair the
// paired-FMA accumulation needs sits 8-byte aligned:
//   [0] w_x0 w_x1 w_x2 w_y0   [1] u_x u_y u_z w_y1   [2] q0_x q0_y q0_z w_y2
//   [3] q1_x q1_y q1_z w_z2   [4] q2_x q2_y w_z0 w_z1   [5] 0 q2_z base 0
// u = m v - dx Q f, q_a = dx Q e_a (Q = m C - dt V0 4/dx^2 tau, MLS), base = the
// packed stencil base (scatter list only).
enum RowIdx : int { kRwWx = 0, kRwWy0 = 3, kRwU = 4, kRwWy1 = 7, kRwQ0 = 8, kRwWy2 = 11, kRwQ1 = 12, kRwWz2 = 15,
                    kRwQ2 = 16, kRwWz0 = 18, kRwWz1 = 19, kRwQ2z = 21, kRwBase = 22 };

__device__ __forceinline__ void p2g_stage_row(const float x[3], const float v[3], const float Cm[9], const float T[6],
                                              float4* row, const DevParams& P, float packed_base = 0.0f) {
  const float m = P.mass;
  const Axis a0 = bspline_axis(x[0], P.inv_dx), a1 = bspline_axis(x[1], P.inv_dx), a2 = bspline_axis(x[2], P.inv_dx);
  const float Tm[9] = {T[0], T[5], T[4], T[5], T[1], T[3], T[4], T[3], T[2]};
  float Q[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) Q[k] = P.mC * Cm[k] - P.mls_coef * Tm[k];
  const float f0 = a0.f, f1 = a1.f, f2 = a2.f;
  row[0] = make_float4(a0.w[0], a0.w[1], a0.w[2], a1.w[0]);
  row[1] = make_float4(m * v[0] - P.dx * (Q[0] * f0 + Q[1] * f1 + Q[2] * f2),
                       m * v[1] - P.dx * (Q[3] * f0 + Q[4] * f1 + Q[5] * f2),
                       m * v[2] - P.dx * (Q[6] * f0 + Q[7] * f1 + Q[8] * f2), a1.w[1]);
  row[2] = make_float4(P.dx * Q[0], P.dx * Q[3], P.dx * Q[6], a1.w[2]);
  row[3] = make_float4(P.dx * Q[1], P.dx * Q[4], P.dx * Q[7], a2.w[2]);
  row[4] = make_float4(P.dx * Q[2], P.dx * Q[5], a2.w[0], a2.w[1]);
  row[5] = make_float4(0.0f, P.dx * Q[8], packed_base, 0.0f);
}

// Thread (cell, ox): sums, over the cell's staged rows, the P2G contributions to
// its 9 nodes (ox, oy, oz) -- mass weight and affine momentum W (u + ox q0 + oy q1 + oz q2).
// NSF_F2_P2G: (p_x, p_y) of each node is one paired FMA with the node weight as a
// broadcast operand; the z momenta and the masses of nodes oz = 0, 1 of a row pair
// up across the two nodes (weights (W_0, W_1) from one paired multiply); every
// lane performs the scalar form's operation, so the sums are the same.
template <int ROWS>
__device__ __forceinline__ void p2g_accumulate_rows(const float4* slot, int my_cell, int ox, int rows, float accm[9],
                                                    float accp[9][3]) {
  const float fox = (float)ox;
  const float4* rp = slot + my_cell * FusedSlots<ROWS>::kCellStride4;
#if NSF_F2_P2G
  float2 pxy[9], pz01[3], m01[3];
  float pz2[3], m2[3];
#pragma unroll
  for (int k = 0; k < 9; ++k) pxy[k] = make_float2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < 3; ++k) { pz01[k] = m01[k] = make_float2(0.f, 0.f); pz2[k] = m2[k] = 0.f; }
#if NSF_P2G_ROW_UNROLL == 2
#pragma unroll 2
#endif
  for (int r = 0; r < rows; ++r, rp += kRowF4) {
    const float4 A = rp[0], U = rp[1], Q0 = rp[2], Q1 = rp[3], Q2 = rp[4], Z = rp[5];
    const float wx = ox == 0 ? A.x : (ox == 1 ? A.y : A.z);
    const float wyv[3] = {A.w, U.w, Q0.w};
    const float2 wz01 = make_float2(Q2.z, Q2.w);
    const float wz2 = Q1.w;
    const float2 q1 = make_float2(Q1.x, Q1.y), q2 = make_float2(Q2.x, Q2.y), zq2 = make_float2(Z.x, Z.y);
    const float2 uxy = __ffma2_rn(make_float2(fox, fox), make_float2(Q0.x, Q0.y), make_float2(U.x, U.y));
    const float uz = fmaf(fox, Q0.z, U.z);
#pragma unroll
    for (int oy = 0; oy < 3; ++oy) {
      const float wxy = wx * wyv[oy];
      const float2 uy = oy ? __ffma2_rn(make_float2((float)oy, (float)oy), q1, uxy) : uxy;
      const float uyz = oy ? fmaf((float)oy, Q1.z, uz) : uz;
      const float2 W01 = __fmul2_rn(make_float2(wxy, wxy), wz01);   // (W_oz0, W_oz1)
      const float W2 = wxy * wz2;
      const int k = oy * 3;
      pxy[k] = __ffma2_rn(make_float2(W01.x, W01.x), uy, pxy[k]);
      pxy[k + 1] = __ffma2_rn(make_float2(W01.y, W01.y), __fadd2_rn(q2, uy), pxy[k + 1]);
      pxy[k + 2] = __ffma2_rn(make_float2(W2, W2), __ffma2_rn(make_float2(2.f, 2.f), q2, uy), pxy[k + 2]);
      const float2 uz01 = __fadd2_rn(make_float2(uyz, uyz), zq2);   // (u_z + 0, u_z + q2_z)
      pz01[oy] = __ffma2_rn(W01, uz01, pz01[oy]);
      pz2[oy] = fmaf(W2, fmaf(2.0f, Z.y, uyz), pz2[oy]);
      m01[oy] = __fadd2_rn(W01, m01[oy]);
      m2[oy] += W2;
    }
  }
#pragma unroll
  for (int oy = 0; oy < 3; ++oy) {
    const int k = oy * 3;
#pragma unroll
    for (int oz = 0; oz < 3; ++oz) {
      accp[k + oz][0] += pxy[k + oz].x;
      accp[k + oz][1] += pxy[k + oz].y;
    }
    accp[k][2] += pz01[oy].x; accp[k + 1][2] += pz01[oy].y; accp[k + 2][2] += pz2[oy];
    accm[k] += m01[oy].x; accm[k + 1] += m01[oy].y; accm[k + 2] += m2[oy];
  }
#else
  for (int r = 0; r < rows; ++r, rp += kRowF4) {
    const float4 A = rp[0], U = rp[1], Q0 = rp[2], Q1 = rp[3], Q2 = rp[4], Z = rp[5];
    const float wx = ox == 0 ? A.x : (ox == 1 ? A.y : A.z);
    const float wyv[3] = {A.w, U.w, Q0.w};
    const float wzv[3] = {Q2.z, Q2.w, Q1.w};
    const float ux = fmaf(fox, Q0.x, U.x), uy = fmaf(fox, Q0.y, U.y), uz = fmaf(fox, Q0.z, U.z);
    const float q1x = Q1.x, q1y = Q1.y, q1z = Q1.z;
    const float q2x = Q2.x, q2y = Q2.y, q2z = Z.y;
#pragma unroll
    for (int oy = 0; oy < 3; ++oy) {
      const float wxy = wx * wyv[oy];
      const float uyx = oy ? fmaf((float)oy, q1x, ux) : ux, uyy = oy ? fmaf((float)oy, q1y, uy) : uy,
                  uyz = oy ? fmaf((float)oy, q1z, uz) : uz;   // fmaf(0, q, u) is not folded
#pragma unroll
      for (int oz = 0; oz < 3; ++oz) {
        const float W = wxy * wzv[oz];
        const int k = oy * 3 + oz;
        accm[k] += W;
        accp[k][0] = fmaf(W, oz ? fmaf((float)oz, q2x, uyx) : uyx, accp[k][0]);
        accp[k][1] = fmaf(W, oz ? fmaf((float)oz, q2y, uyy) : uyy, accp[k][1]);
        accp[k][2] = fmaf(W, oz ? fmaf((float)oz, q2z, uyz) : uyz, accp[k][2]);
      }
    }
  }
#endif
}

// Phase 1 of the fused kernels for storage slot j: G2P from the
// segment's velocity tile (global gather if the stencil left it), x/v/C/F/tau
// updated in place, and the new state returned for the next substep's P2G.
// P2G-only launches (DO_G2P = false) just read the state.
#ifndef NSF_STREAM_HINTS
#define NSF_STREAM_HINTS 0   // particle state read / written with evict-first cache hints (.cs)
#endif
__device__ __forceinline__ float ld_state(const float* p) {
#if NSF_STREAM_HINTS
  return __ldcs(p);
#else
  return *p;
#endif
}
__device__ __forceinline__ void st_state(float* p, float v) {
#if NSF_STREAM_HINTS
  __stcs(p, v);
#else
  *p = v;
#endif
}
// v, C, tau: written for the caller, never read back by the substep loop, so their
// lines are stored evict-first and leave the L2 to x, F and the grid (same-box A/B on C3:
// flushed 87.9 -> 87.4 us, single-substep calls back to back 84.3 -> 81.8; st.global.wt
// and evict-first on every state access: no gain)
#ifndef NSF_OUT_HINT
#define NSF_OUT_HINT 1   // 0: default policy, 1: st.global.cs (evict first), 2: st.global.wt
#endif
__device__ __forceinline__ void st_out(float* p, float v) {
#if NSF_OUT_HINT == 1
  __stcs(p, v);
#elif NSF_OUT_HINT == 2
  __stwt(p, v);
#else
  st_state(p, v);
#endif
}
__device__ __forceinline__ void load_xF(const float* __restrict__ S, int j, float x[3], float F[9]) {
  const float* base = S + pbase(j);
#pragma unroll
  for (int a = 0; a < 3; ++a) x[a] = ld_state(base + (PX + a) * 32);
#pragma unroll
  for (int k = 0; k < 9; ++k) F[k] = ld_state(base + (PF + k) * 32);
}

// The substep after a periodic re-binning reorders the store on the way (no copy
// pass): storage slot j of the new order is particle map[j] of the previous buffer
// S, whose x, F (and tau_Y, id) are gathered from there; the substep writes its new
// state to the new buffer in order.  S == nullptr: in place.
template <bool GATH>
__device__ __forceinline__ void load_xF_g(const float* __restrict__ S, const GatherIn& gi, int j, float x[3],
                                          float F[9]) {
  if (GATH) load_xF(gi.S, gi.map[j], x, F);
  else load_xF(S, j, x, F);
}

template <bool DO_G2P, bool HS, bool ROT, bool GATH, bool WR>
__device__ __forceinline__ void fused_g2p_particle(float* __restrict__ S, int j, const float xin[3], const float Fin[9],
                                                   const int o[3], const float4* vt, const float4* __restrict__ gvel,
                                                   const DevParams& P, DevErr* err, float xn[3], float vn[3],
                                                   float Cn[9], float tau[6], float y_plate,
                                                   const int32_t* __restrict__ ids, const GatherIn& gi) {
  float* base = S + pbase(j);
      if (DO_G2P) {
    float x[3], F[9], G[9];
#pragma unroll
    for (int a = 0; a < 3; ++a) x[a] = xin[a];
#pragma unroll
    for (int k = 0; k < 9; ++k) F[k] = Fin[k];
    // stencil inside the tile (drift <= 1 cell since the last re-binning)?
    bool in_tile = NSF_FUSED_VTILE;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int bb = (int)floorf(x[a] * P.inv_dx - 0.5f);
      in_tile &= (bb >= o[a]) && (bb + 2 < o[a] + kVT);
    }
    if (in_tile) {
      g2p_gather_tile(x, vt, o, P, vn, Cn);
#pragma unroll
      for (int k = 0; k < 9; ++k) G[k] = Cn[k];
      if (P.rpic) skew_part(Cn);   // RPIC: the transfer's C_p; G keeps the full gradient
    } else {
      NSF_STAT_ADD(kStOutOfTile, 1);
      g2p_gather<0, ROT>(x, gvel, P, vn, Cn, G, y_plate);   // ROT: gvel holds raw P2G sums
    }
    bool ok = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      xn[a] = x[a] + P.dt * vn[a];
      const float tt = xn[a] * P.inv_dx;
      ok &= !(tt < 0.5f || tt >= (float)P.N[a] - 1.5f);   // NaN: non-finite, not out of domain
      st_state(base + (PX + a) * 32, xn[a]);
      // v, C (and tau below) only feed the P2G of this kernel: they are stored when the
      // caller can read them, i.e. by the last substep of a nsf_mpm_substep(n) call (WR)
      if (WR) st_out(base + (PV + a) * 32, vn[a]);
    }
#pragma unroll
    for (int k = 0; k < 9; ++k)
      if (WR) st_out(base + (PC + k) * 32, Cn[k]);
    float Ft[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int jj = 0; jj < 3; ++jj)
        Ft[i * 3 + jj] = F[i * 3 + jj] + P.dt * (G[i * 3 + 0] * F[0 * 3 + jj] + G[i * 3 + 1] * F[1 * 3 + jj] +
                                                 G[i * 3 + 2] * F[2 * 3 + jj]);
    float FE[9];
    float J;
    if (HS) {   // per-particle yield stress (#30-#32)
      float tY = GATH ? gi.S[pbase(gi.map[j]) + PTY * 32] : base[PTY * 32];
      J = vm_hs_update(Ft, P.mu, P.lam, P.vm_hard_k, P.vm_soft, tY, FE, tau);
      base[PTY * 32] = tY;
    } else {
      J = P.model == 5 ? hb_update(Ft, P.mu, P.kappa, P.hb_yield, P.hb_relax, FE, tau)
                       : elastoplastic_fast(Ft, P.model, P.mu, P.lam, P.alpha, P.tau_Y, FE, tau);
    }
    float chk = xn[0] + xn[1] + xn[2] + vn[0] + vn[1] + vn[2];
#pragma unroll
    for (int k = 0; k < 9; ++k) { st_state(base + (PF + k) * 32, FE[k]); chk += FE[k]; }
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      if (WR) st_out(base + (PT + k) * 32, tau[k]);
      chk += tau[k];
    }
    if (!(J > 0.0f)) atomicAdd(&err->inverted, 1ull);
    if (!ok || !isfinite(chk)) {
      atomicOr(&err->bits, (ok ? 0u : (uint32_t)ERR_OUT_OF_DOMAIN) | (isfinite(chk) ? 0u : (uint32_t)ERR_NONFINITE));
      atomicMin(&err->first_index, GATH ? gi.ids[gi.map[j]] : ids[j]);
    }
  } else {
#pragma unroll
    for (int a = 0; a < 3; ++a) { xn[a] = base[(PX + a) * 32]; vn[a] = base[(PV + a) * 32]; }
#pragma unroll
    for (int k = 0; k < 9; ++k) Cn[k] = base[(PC + k) * 32];
#pragma unroll
    for (int k = 0; k < 6; ++k) tau[k] = base[(PT + k) * 32];
  }
}

// Phase-2 scatter of the listed particles: work item i = (entry i / 35; its
// stencil node i % 35 < 27, else one of its 8 corner blocks to mark touched).
// Node (a, b, c) gets m W, W (u0 + a q0 + b q1 + c q2) as in p2g_accumulate_rows.
template <bool HALO>
__device__ __forceinline__ void scatter_listed(const float4* sc, int nsc, int i0, int stride, float4* gacc,
                                               const TouchCtx& tc, const DevParams& P) {
  for (int i = i0; i < nsc * 35; i += stride) {
    const int e = i / 35, q = i - 35 * e;
    const float* s = reinterpret_cast<const float*>(sc + e * kRowF4);
    const int pb = __float_as_int(s[kRwBase]);
    const int bx = pb >> 20, by = (pb >> 10) & 1023, bz = pb & 1023;
    if (q < 27) {
      const int a = q / 9, b = (q / 3) % 3, c = q % 3;
      const float wy = b == 0 ? s[kRwWy0] : (b == 1 ? s[kRwWy1] : s[kRwWy2]);
      const float wz = c == 0 ? s[kRwWz0] : (c == 1 ? s[kRwWz1] : s[kRwWz2]);
      const float W = s[kRwWx + a] * wy * wz;
      const float fa = (float)a, fb = (float)b, fc = (float)c;
      const float ux = fmaf(fc, s[kRwQ2], fmaf(fb, s[kRwQ1], fmaf(fa, s[kRwQ0], s[kRwU])));
      const float uy = fmaf(fc, s[kRwQ2 + 1], fmaf(fb, s[kRwQ1 + 1], fmaf(fa, s[kRwQ0 + 1], s[kRwU + 1])));
      const float uz = fmaf(fc, s[kRwQ2z], fmaf(fb, s[kRwQ1 + 2], fmaf(fa, s[kRwQ0 + 2], s[kRwU + 2])));
      NSF_CHECK(node_index(bx + a, by + b, bz + c, P) < P.nodes_per_scene);
      red_add_v4_t(gacc + node_index(bx + a, by + b, bz + c, P), W * P.mass, W * ux, W * uy, W * uz);
    } else {
      const int k = q - 27;
      const int b0 = (bx + 2 * (k >> 2)) >> 2, b1 = (by + 2 * ((k >> 1) & 1)) >> 2, b2 = (bz + 2 * (k & 1)) >> 2;
      touch<HALO>(tc, b0, b1, b2, P);
    }
  }
}

// The fused kernel's next segment: its ticket, and (if any) its block key and
// storage range, into shared memory.  Called by one thread: at the kernel start,
// then during phase 1 by the last thread, which usually idles in the last pass, so
// the three dependent global round trips stay off the segment's critical path.
template <class SM>
__device__ __forceinline__ void claim_segment(SM& sm, int32_t* counters, const int32_t* __restrict__ nonempty,
                                              const int32_t* __restrict__ block_start, int nblk) {
  const int t = atomicAdd(&counters[3], 1);
  sm.next = t;
  if (t < nblk) {
    const int key = nonempty[t];
    sm.nkey = key;
    sm.ns0 = block_start[key];
    sm.ns1 = block_start[key + 1];
  }
}

// ROT: the grid update runs inside this kernel (RotGrid, pipeline.h): `vel`,
// `acc`, `flags`, `list` and `list_count` are ignored and taken from the
// rotation instead; the segment's velocity tile is staged from the raw P2G sums
// with every node updated on the way, the blocks of the cleared buffer
// are zeroed, and the last CTA to finish advances the step counter.
// GUM: where the grid update of the P2G reduced here runs:
//   0  in k_grid_update_list before the next substep;
//   1  (ROT) in the next k_g2p2g as it stages its velocity tiles (three rotating grids);
//   2  (GUB) at the end of this kernel, after a grid-wide barrier (every CTA of the
//      persistent grid is resident): all CTAs update the touched blocks, so a substep
//      is one launch and the next G2P reads `vel` directly.
// WR: v, C, tau are stored (false: a substep that is not the last of its call).
template <bool DO_G2P, int ROWS, int MINB, int NT, bool HS = false, int GUM = 0, bool GATH = false, bool WR = true>
__global__ void __launch_bounds__(NT, MINB)
k_g2p2g(float* __restrict__ S, const int32_t* __restrict__ ids, const float4* __restrict__ vel, float4* __restrict__ acc, int* __restrict__ flags,
        int* __restrict__ list, int* __restrict__ list_count, const int32_t* __restrict__ block_start,
        const int32_t* __restrict__ nonempty, int32_t* __restrict__ counters, DevParams P, DevErr* err,
        int64_t* d_step, RotGrid rg, const int* __restrict__ hmark, GatherIn gi,
        const unsigned long long* __restrict__ scan_ticket, int64_t scan_tiles) {
  constexpr bool ROT = GUM == 1, GUB = GUM == 2;
  constexpr bool HALO = GUM == 0;   // the grid-update pass visits the halo list (k_halo) + far-touched blocks
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FusedSmemT<ROWS>& sm = *reinterpret_cast<FusedSmemT<ROWS>*>(smem_raw);
  const int tid = threadIdx.x;
  const int my_cell = tid & 63;
  const int ox = tid >> 6;
  pdl_wait();   // the grid update (or the re-binning) before it
  const int nblk = *(volatile int32_t*)&counters[0];
#if NSF_STATS
  if (tid == 0) tail_stat_begin();
#endif
  int64_t kstep = 0;
  float y_plate = 0.0f;
  int* const cnt2 = list_count;   // GUB: the two count slots (+ [2] sel, [3] barrier generation)
  if (GUB) {
    // every CTA reads the step counter before anyone advances it (at the end);
    // the P2G written here is that of state kw + 1 and appends to slot kw & 1
    kstep = *(volatile const int64_t*)d_step;
    const int64_t kw = DO_G2P ? kstep : kstep - 1;
    list_count = cnt2 + (int)(kw & 1);
  } else if (ROT) {
    // kernel index kw: the P2G written here is that of state kw + 1 (kw = -1 for
    // the P2G of the loaded state); it reads buffer kw % 3, writes (kw + 1) % 3,
    // clears (kw + 2) % 3
    kstep = *(volatile const int64_t*)d_step;
    const int64_t kw = DO_G2P ? kstep : kstep - 1;
    const int rb = (int)(((kw % 3) + 3) % 3), wb = (rb + 1) % 3, zb = (rb + 2) % 3;
    const int64_t TB = rg.total_blocks;
    vel = rg.buf[rb];
    acc = rg.buf[wb];
    flags = rg.flags + wb * TB;
    list = rg.list + wb * TB;
    list_count = rg.cnt + (int)(kw & 3);
    y_plate = plate_y_at(P, kstep);
    if (DO_G2P) {
      // clear the blocks of buffer zb (the P2G of kernel kw - 2) and their flags;
      // CTA c takes list entries c, c + grid, ...
      const int nz = *(volatile const int*)&rg.cnt[(int)((kw + 2) & 3)];
      const int* zl = rg.list + zb * TB;
      int* zf = rg.flags + zb * TB;
      float4* zbuf = rg.buf[zb];
      for (int i = tid;; i += NT) {
        const int e = (int)blockIdx.x + (i >> 6) * (int)gridDim.x;
        if (e >= nz) break;
        const int key = zl[e];
        NSF_CHECK(nz <= TB && key >= 0 && key < TB);
        zbuf[(int64_t)key * kBlockNodes + (i & 63)] = make_float4(0.f, 0.f, 0.f, 0.f);
        if ((i & 63) == 0) zf[key] = 0;
      }
    }
  } else {
    // list count slot published by the grid update (or 0 after a load)
    list_count += *(volatile const int*)(list_count + 2);
    if (DO_G2P && blockIdx.x == 0 && tid == 0) atomicAdd((unsigned long long*)d_step, 1ull);
  }
  (void)cnt2;
  // segment tickets: the first here, each next one claimed (with its key and
  // range) during phase 1 of the current segment
  if (tid == 0) claim_segment(sm, counters, nonempty, block_start, nblk);
  if (DO_G2P && NSF_FUSED_VTILE && NSF_TILE_TMA && !ROT && tid == 0) tile_bar_init(&sm.tbar, NT);   // (barrier at the loop top)
#if NSF_STATS
  long long t_mark = clock64();
#endif
  while (true) {
    __syncthreads();   // also: previous segment's readers of slot are done
#if NSF_STATS
    if (tid == 0) { const long long t = clock64(); NSF_STAT_ADD(kStCycPhase2, t - t_mark); t_mark = t; }
#endif
    const int bi = sm.next;
    if (bi >= nblk) break;
    const int key = sm.nkey;
    const BlockCoord bc = decode_block(key, P);
    const int s0 = sm.ns0, s1 = sm.ns1;
    if (tid == 0) {
      NSF_STAT_ADD(kStSegments, 1);
      NSF_STAT_ADD(kStParticles, s1 - s0);
      NSF_STAT_ADD(kStPasses, (s1 - s0 + NT - 1) / NT);
    }
    const int64_t scene_block0 = (int64_t)bc.scene * P.blocks_per_scene;
    TouchCtx tc;
    tc.flags = flags;
    tc.list = list;
    tc.list_count = list_count;
    tc.hmark = hmark;
    tc.scan_ticket = scan_ticket;
    tc.scan_tiles = scan_tiles;
    tc.seg[0] = bc.b[0];
    tc.seg[1] = bc.b[1];
    tc.seg[2] = bc.b[2];
    tc.scene_block0 = scene_block0;
    float4* gacc = acc + (int64_t)bc.scene * P.nodes_per_scene;
    const float4* gvel = vel + (int64_t)bc.scene * P.nodes_per_scene;
    if (tid < 64) sm.pop[tid] = 0;
    if (tid == 0) sm.nsc = 0;
    const int o[3] = {4 * bc.b[0] - 1, 4 * bc.b[1] - 1, 4 * bc.b[2] - 1};   // tile origin (grid node)

    float x0[3], F0[9];   // the first particle's x, F: loaded under the tile copy
    unsigned long long ttok = 0;
    if (DO_G2P && NSF_FUSED_VTILE && ROT) {
      // raw P2G sums of the tile's nodes (L2-resident: reduced by the previous
      // kernel) copied asynchronously; after the wait each thread updates the
      // nodes it copied in place, so the first particle's loads overlap
      // the copy and the update, and no extra barrier is needed
      constexpr int kPer = (kVT * kVT * kVT + NT - 1) / NT;
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int e = tid + q * NT;
        if (e < kVT * kVT * kVT) {
          const int i = o[0] + (e >> 6), jn = o[1] + ((e >> 3) & 7), k = o[2] + (e & 7);
          const bool in = i >= 0 && jn >= 0 && k >= 0 && i < P.N[0] && jn < P.N[1] && k < P.N[2];
          cp_async16_f(&sm.vt[(e >> 6) * kVTx + ((e >> 3) & 7) * kVTy + (e & 7)],
                       in ? gvel + node_index(i, jn, k, P) : gvel, in ? 16 : 0);
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      if (s0 + tid < s1) load_xF_g<GATH>(S, gi, s0 + tid, x0, F0);
      // walls: skip the per-face tests when the tile lies inside [w, N - w) on every axis
      bool walls = false;
#pragma unroll
      for (int ax_ = 0; ax_ < 3; ++ax_)
        walls |= (o[ax_] < P.bc_width) || (o[ax_] + kVT > P.N[ax_] - P.bc_width);
      asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int e = tid + q * NT;
        if (e < kVT * kVT * kVT) {
          const int i = o[0] + (e >> 6), jn = o[1] + ((e >> 3) & 7), k = o[2] + (e & 7);
          float4* t = &sm.vt[(e >> 6) * kVTx + ((e >> 3) & 7) * kVTy + (e & 7)];
          *t = grid_node_update_rcp(*t, i, jn, k, P, y_plate, walls);
        }
      }
    } else if (DO_G2P && NSF_FUSED_VTILE && NSF_TILE_TMA) {
      int tx = 0;
      if (tid < 192) {
        const int r = tid / 3, pc = tid - 3 * r;            // tile row (x, y), run in z
        const int ti = r >> 3, tj = r & 7;
        const int k0 = pc == 0 ? 0 : (pc == 1 ? 1 : 5), nk = pc == 0 ? 1 : (pc == 1 ? 4 : 3);
        const int i = o[0] + ti, jn = o[1] + tj, k = o[2] + k0;
        float4* dst = &sm.vt[ti * kVTx + tj * kVTy + k0];
        if (i >= 0 && jn >= 0 && k >= 0 && i < P.N[0] && jn < P.N[1] && k < P.N[2]) {
          tx = 16 * nk;
          // (the tile's readers of the previous segment passed two barriers; order them,
          // and any zero fill, before the async-proxy writes)
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          ttok = tile_bar_arrive(&sm.tbar, tx);
          bulk_g2s(dst, gvel + node_index(i, jn, k, P), tx, &sm.tbar);
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (q < nk) dst[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      if (tx == 0) ttok = tile_bar_arrive(&sm.tbar, 0);
    } else if (DO_G2P && NSF_FUSED_VTILE) {
      for (int e = tid; e < kVT * kVT * kVT; e += NT) {
        const int i = o[0] + (e >> 6), jn = o[1] + ((e >> 3) & 7), k = o[2] + (e & 7);
        const bool in = i >= 0 && jn >= 0 && k >= 0 && i < P.N[0] && jn < P.N[1] && k < P.N[2];
        cp_async16_f(&sm.vt[(e >> 6) * kVTx + ((e >> 3) & 7) * kVTy + (e & 7)], in ? gvel + node_index(i, jn, k, P) : gvel,
                     in ? 16 : 0);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    if (DO_G2P && !ROT && s0 + tid < s1) load_xF_g<GATH>(S, gi, s0 + tid, x0, F0);
    if (DO_G2P && NSF_FUSED_VTILE && NSF_TILE_TMA && !ROT) {
      // every thread arrived after its stores above (pop, nsc, zero fill): the phase
      // completes when all have and the copies' bytes landed -- also the CTA barrier
      tile_bar_wait(&sm.tbar, ttok);
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncthreads();
    }
#if NSF_STATS
    if (tid == 0) { const long long t = clock64(); NSF_STAT_ADD(kStCycTile, t - t_mark); t_mark = t; }
#endif
    // ---- phase 1: per particle ----
    for (int j = s0 + tid; j < s1; j += NT) {
      float xn[3], vn[3], Cn[9], tau[6];
#if NSF_PF_NEXT
      // the next particle's x, F load under this one's G2P (needs the registers of
      // 2 CTAs per SM)
      float x1[3], F1[9];
      if (DO_G2P && j + NT < s1) load_xF_g<GATH>(S, gi, j + NT, x1, F1);
#else
      if (DO_G2P && j != s0 + tid) load_xF_g<GATH>(S, gi, j, x0, F0);
#endif
      fused_g2p_particle<DO_G2P, HS, ROT, GATH, WR>(S, j, x0, F0, o, sm.vt, gvel, P, err, xn, vn, Cn, tau, y_plate,
                                                    ids, gi);
      if (GATH) {   // the rest of the gathered particle: id, and tau_Y unless the update above wrote it
        const int g = gi.map[j];
        gi.ids_out[j] = gi.ids[g];
        if (!HS) S[pbase(j) + PTY * 32] = gi.S[pbase(g) + PTY * 32];
      }
#if NSF_PF_NEXT
      if (DO_G2P && j + NT < s1) {
#pragma unroll
        for (int a = 0; a < 3; ++a) x0[a] = x1[a];
#pragma unroll
        for (int k = 0; k < 9; ++k) F0[k] = F1[k];
      }
#endif
      // ---- P2G of the new state: by cell if still inside this block, else direct ----
      int c[3];
      bool core = true;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        int b = (int)floorf(xn[a] * P.inv_dx - 0.5f);
        b = min(max(b, 0), P.N[a] - 3);
        c[a] = b - 4 * bc.b[a];
        core &= (c[a] >= 0) && (c[a] < 4);
      }
      int rank = ROWS;
      int cell = 0;
      if (core) {
        cell = (c[0] << 4) | (c[1] << 2) | c[2];
        rank = atomicAdd(&sm.pop[cell], 1);
      } else {
        NSF_STAT_ADD(kStOutOfBlock, 1);
      }
      bool inline_scatter = false;
      if (rank < ROWS) {
        NSF_STAT_ADD(kStStaged, 1);
        NSF_CHECK(cell >= 0 && cell < 64 && (cell + 1) * FusedSlots<ROWS>::kCellStride4 > rank * kRowF4 + 5);
        p2g_stage_row(xn, vn, Cn, tau, sm.slot + cell * FusedSlots<ROWS>::kCellStride4 + rank * kRowF4, P);
      } else {
        const int e = atomicAdd(&sm.nsc, 1);
        if (e < kScatterCap) {
          NSF_STAT_ADD(kStListed, 1);
          int pb = 0;
#pragma unroll
          for (int a = 0; a < 3; ++a)
            pb = (pb << 10) | min(max((int)floorf(xn[a] * P.inv_dx - 0.5f), 0), P.N[a] - 3);
          p2g_stage_row(xn, vn, Cn, tau, sm.sc + e * kRowF4, P, __int_as_float(pb));
        } else {
          inline_scatter = true;
          NSF_STAT_ADD(kStInline, 1);
        }
      }
#if NSF_WARP_SCATTER
      p2g_scatter_warp<HALO>(inline_scatter, xn, vn, Cn, tau, gacc, tc, P);
#else
      if (inline_scatter) p2g_scatter_direct<HALO>(xn, vn, Cn, tau, gacc, tc, P);
#endif
    }
    // (every thread read the current segment's slots at the loop top, before the tile
    // barrier).  192 threads: the last one idles in the last phase-1 pass; more: it
    // is a phase-2 helper, and claims after the barrier
    if (NT <= 192 && tid == NT - 1) claim_segment(sm, counters, nonempty, block_start, nblk);
    __syncthreads();
    if (NT > 192 && tid == NT - 1) claim_segment(sm, counters, nonempty, block_start, nblk);
#if NSF_STATS
    if (tid == 0) { const long long t = clock64(); NSF_STAT_ADD(kStCycPhase1, t - t_mark); t_mark = t; }
#endif
#if NSF_STATS
    long long t_p2 = clock64();
#endif
    // ---- phase 2: per (cell, stencil plane) register accumulation ----
    float accm[9], accp[9][3];
#pragma unroll
    for (int k = 0; k < 9; ++k) { accm[k] = 0.f; accp[k][0] = accp[k][1] = accp[k][2] = 0.f; }
    // the grid blocks the segment's cell sums reduce into (its block and the +1
    // neighbours) are flagged by the last 8 helper threads, whose flag round trips
    // then overlap the accumulation instead of trailing it
    if (!HALO && NT > 192 && tid >= NT - 8) {
      const int t8 = tid - (NT - 8);
      const int b0 = bc.b[0] + (t8 >> 2), b1 = bc.b[1] + ((t8 >> 1) & 1), b2 = bc.b[2] + (t8 & 1);
      if (b0 < P.NB[0] && b1 < P.NB[1] && b2 < P.NB[2])
        touch_block(flags, list, list_count, (int)(scene_block0 + block_id(b0, b1, b2, P)), P);
    }
    {
      const int nsc = min(sm.nsc, kScatterCap);
      if (NT > 192) {
        if (ox >= 3) scatter_listed<HALO>(sm.sc, nsc, tid - 192, NT - 192, gacc, tc, P);
        else p2g_accumulate_rows<ROWS>(sm.slot, my_cell, ox, min(sm.pop[my_cell], ROWS), accm, accp);
      } else {
        scatter_listed<HALO>(sm.sc, nsc, tid, NT, gacc, tc, P);
        p2g_accumulate_rows<ROWS>(sm.slot, my_cell, ox, min(sm.pop[my_cell], ROWS), accm, accp);
      }
    }
    // each (cell, plane) thread reduces its 9 node sums straight into the grid
    // accumulator (one red.global.add.v4 per node); the segment's tile blocks
    // (4x4x4 nodes at 4b and the +1 neighbours its stencils reach) are flagged
    if (ox < 3 && sm.pop[my_cell] > 0) {
      const float m = P.mass;
      const int gi = 4 * bc.b[0] + (my_cell >> 4) + ox;
      const int cy = 4 * bc.b[1] + ((my_cell >> 2) & 3), cz = 4 * bc.b[2] + (my_cell & 3);
      const int x_part = (gi >> 2) * (P.NB[1] * P.NB[2] * kBlockNodes) + ((gi & 3) << 4);
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        const int gj = cy + k / 3, gk = cz + k % 3;
        const int off = x_part + ((gj >> 2) * P.NB[2] + (gk >> 2)) * kBlockNodes + ((gj & 3) << 2) + (gk & 3);
        NSF_CHECK(off >= 0 && off < P.nodes_per_scene);
        red_add_v4_t(gacc + off, accm[k] * m, accp[k][0], accp[k][1], accp[k][2]);
      }
    }
#if NSF_STATS
    if (tid == 0) NSF_STAT_ADD(kStCycP2Acc, clock64() - t_p2);
    if (tid == NT - 1) NSF_STAT_ADD(kStCycP2Help, clock64() - t_p2);
#endif
    if (!HALO && NT <= 192 && tid < 8) {   // (no helper threads)
      const int b0 = bc.b[0] + (tid >> 2), b1 = bc.b[1] + ((tid >> 1) & 1), b2 = bc.b[2] + (tid & 1);
      if (b0 < P.NB[0] && b1 < P.NB[1] && b2 < P.NB[2])
        touch_block(flags, list, list_count, (int)(scene_block0 + block_id(b0, b1, b2, P)), P);
    }
  }
  if (GUB) {
    // grid-wide barrier (generation counter; all CTAs are resident: the grid is one
    // wave of the persistent kernel): every CTA's reductions are complete and visible
    __syncthreads();
    if (tid == 0) {
      volatile int* genp = cnt2 + 3;
      const int g0 = *genp;
      __threadfence();
      if (atomicAdd(&counters[2], 1) == (int)gridDim.x - 1) {
        counters[2] = 0;
        __threadfence();
        atomicAdd(cnt2 + 3, 1);
      } else {
        while (*genp == g0) __nanosleep(20);
      }
      __threadfence();
    }
    __syncthreads();
    // grid update of the touched blocks, warp per block, for the next G2P
    const int64_t kw = DO_G2P ? kstep : kstep - 1;
    const int nl = *(volatile const int*)list_count;
    const float y_next = plate_y_at(P, kw + 1);
    const int lane = tid & 31;
    const int gw = (int)((blockIdx.x * NT + tid) >> 5), nw = (int)((gridDim.x * NT) >> 5);
    const int bps = (int)P.blocks_per_scene;
    float4* velw = const_cast<float4*>(vel);
    NSF_CHECK(nl >= 0 && nl <= P.blocks_per_scene * P.n_scenes);
    for (int e = gw; e < nl; e += nw) {
      const int key = *(volatile const int*)(list + e);
      NSF_CHECK(key >= 0 && key < P.blocks_per_scene * P.n_scenes);
      const int scene = key / bps;
      const BlockCoord bc = decode_block(key, P);
      const int64_t gb = (int64_t)scene * P.nodes_per_scene + (int64_t)(key - scene * bps) * kBlockNodes;
      float4 a[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) a[h] = __ldcg(acc + gb + lane + 32 * h);
      bool walls = false;
#pragma unroll
      for (int ax_ = 0; ax_ < 3; ++ax_)
        walls |= (4 * bc.b[ax_] < P.bc_width) || (4 * bc.b[ax_] + 4 > P.N[ax_] - P.bc_width);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int l = lane + 32 * h;
        const int i = bc.b[0] * 4 + (l >> 4), j = bc.b[1] * 4 + ((l >> 2) & 3), k = bc.b[2] * 4 + (l & 3);
        velw[gb + l] = grid_node_update_rcp(a[h], i, j, k, P, y_next, walls);
        acc[gb + l] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if (lane == 0) flags[key] = 0;
    }
    if (blockIdx.x == 0 && tid == 0) {
      counters[3] = 0;                     // segment ticket of the next kernel
      cnt2[(int)((kw + 1) & 1)] = 0;       // the list the next kernel appends to
      if (DO_G2P) *d_step = kstep + 1;
    }
  }
#if NSF_STATS
  if (tid == 0) tail_stat_end();
#endif
  if (ROT && tid == 0) {
    // every CTA has read the step counter and claimed its last ticket: the last
    // one to finish resets the ticket and the completion counter, and (G2P)
    // advances the step and empties the count slot the next kernel appends to
    if (atomicAdd(&rg.cnt[4], 1) == (int)gridDim.x - 1) {
      rg.cnt[4] = 0;
      counters[3] = 0;
      if (DO_G2P) {
        *d_step = kstep + 1;
        rg.cnt[(int)((kstep + 1) & 3)] = 0;
      }
    }
  }
}

// Grid update over the touched blocks: v = mv/m + dt g, walls, plate; the
// accumulator and the block's flag are cleared.  One warp per listed block.  The
// list count alternates between two slots by step parity: this kernel reads slot
// n & 1, empties slot (n + 1) & 1 and publishes it (sel) for the next G2P2G to
// append to -- no completion counter or fence is needed.
//
// The blocks visited are the halo list (`halo`, `nhalo` entries: every block in
// the 27-block neighbourhood of a non-empty segment, k_halo) followed by the
// touched list (blocks outside the halo, flagged by far particles).  Halo blocks
// nothing reached hold m = 0 and get v = 0 (never gathered).
__global__ void __launch_bounds__(128)
k_grid_update_list(int* __restrict__ flags, const int* __restrict__ list, int* __restrict__ cnt2,
                   const int* __restrict__ halo, const int* __restrict__ nhalo, const int* __restrict__ hmark,
                   const unsigned long long* __restrict__ scan_ticket, int64_t scan_tiles,
                   float4* __restrict__ acc, float4* __restrict__ vel, DevParams P,
                   const int64_t* __restrict__ d_step, int32_t* __restrict__ counters) {
  // the step, both count slots and this warp's first halo entry are loaded
  // together (the entry speculatively: the halo list has room for every block)
  const int lane = threadIdx.x & 31;
  const int warp = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nwarps = (int)(((int64_t)gridDim.x * blockDim.x) >> 5);
  pdl_launch_dependents();   // the fused kernel's CTAs may be scheduled now (they wait for this grid)
  pdl_wait();                // the previous substep's kernels
  const int64_t n = *d_step;
  const int c0 = cnt2[0], c1 = cnt2[1];
  const int nh = *nhalo;
  int key_next = warp < P.blocks_per_scene * P.n_scenes ? halo[warp] : 0;
  const int s = (int)(n & 1);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    counters[3] = 0;    // segment ticket of the next k_g2p2g
    cnt2[s ^ 1] = 0;    // the list the next k_g2p2g appends to
    cnt2[2] = s ^ 1;
  }
  const int nl = nh + (s ? c1 : c0);
  const float y_plate = plate_y_at(P, n);
  const int bps = (int)P.blocks_per_scene;
  NSF_CHECK(nl >= 0 && nl <= 2 * P.blocks_per_scene * P.n_scenes);
  if (warp >= nh && warp < nl) key_next = list[warp - nh];
  for (int e = warp; e < nl; e += nwarps) {
    const int key = key_next;
    NSF_CHECK(key >= 0 && key < P.blocks_per_scene * P.n_scenes);
    const int en = e + nwarps;
    if (en < nl) key_next = en < nh ? halo[en] : list[en - nh];
    // a far-touched block listed before a re-binning may be in the new halo: updated
    // there once (a second update would read the cleared sums)
    if (e >= nh && hmark[key] == (int)(*scan_ticket / (unsigned long long)scan_tiles)) {
      if (lane == 0) flags[key] = 0;
      continue;
    }
    const int scene = key / bps;
    const BlockCoord bc = decode_block(key, P);
    const int64_t gb = (int64_t)scene * P.nodes_per_scene + (int64_t)(key - scene * bps) * kBlockNodes;
    float4 a[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) a[h] = acc[gb + lane + 32 * h];
    // the per-face wall tests only for blocks that reach a wall band (uniform per warp)
    bool walls = false;
#pragma unroll
    for (int ax_ = 0; ax_ < 3; ++ax_)
      walls |= (4 * bc.b[ax_] < P.bc_width) || (4 * bc.b[ax_] + 4 > P.N[ax_] - P.bc_width);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int l = lane + 32 * h;
      const int i = bc.b[0] * 4 + (l >> 4), j = bc.b[1] * 4 + ((l >> 2) & 3), k = bc.b[2] * 4 + (l & 3);
      vel[gb + l] = grid_node_update_rcp(a[h], i, j, k, P, y_plate, walls);
      acc[gb + l] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (lane == 0 && e >= nh) flags[key] = 0;
  }
}

// Halo of the segments (GUM 0), at every re-binning: block B is in it when a
// non-empty block lies in its 27-neighbourhood (the blocks a segment's P2G can
// reach while its particles drift <= 4 cells).  Thread per (segment, neighbour):
// the first to mark B (hmark zeroed before) lists it for the grid update.
__global__ void __launch_bounds__(512)
k_halo(const int32_t* __restrict__ nonempty, const int32_t* __restrict__ n_nonempty, int* __restrict__ hmark,
       int* __restrict__ halo, int* __restrict__ nhalo, const unsigned long long* __restrict__ scan_ticket,
       int64_t scan_tiles, DevParams P) {
  // one wave of CTAs, each over a contiguous range of (segment, neighbour) items in
  // rounds of blockDim; a round's new members are counted in shared memory and
  // appended with one global atomic (a per-thread append serialised ~3,400 atomics
  // on one counter, and a thread per item launched 27 x 262,144 threads: 27 us)
  __shared__ int cnt, base;
  pdl_launch_dependents();
  pdl_wait();
  // marks carry the re-binning's scan epoch (>= 1), so hmark needs no clearing
  const int tag = (int)(*scan_ticket / (unsigned long long)scan_tiles);
  const int64_t items = 27 * (int64_t)(*n_nonempty);
  const int64_t per = (items + gridDim.x - 1) / gridDim.x;
  const int64_t c0 = blockIdx.x * per, c1 = min(items, c0 + per);
  for (int64_t r0 = c0; r0 < c1; r0 += blockDim.x) {
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    const int64_t t = r0 + threadIdx.x;
    int B = -1, slot = -1;
    if (t < c1) {
      const int e = (int)(t / 27), d = (int)(t % 27);
      const BlockCoord bc = decode_block(nonempty[e], P);
      const int n0 = bc.b[0] + d / 9 - 1, n1 = bc.b[1] + (d / 3) % 3 - 1, n2 = bc.b[2] + d % 3 - 1;
      if (n0 >= 0 && n1 >= 0 && n2 >= 0 && n0 < P.NB[0] && n1 < P.NB[1] && n2 < P.NB[2]) {
        B = (int)((int64_t)bc.scene * P.blocks_per_scene + block_id(n0, n1, n2, P));
        if (atomicExch(hmark + B, tag) != tag) slot = atomicAdd(&cnt, 1);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) base = cnt ? atomicAdd(nhalo, cnt) : 0;
    __syncthreads();
    if (slot >= 0) halo[base + slot] = B;
  }
}

// (nhalo is reset by the scan of the same re-binning)
void launch_halo(cudaStream_t st, PipelineBuffers* pb, const DevParams& P) {
  launch_pdl(k_halo, dim3(num_sms()), dim3(512), 0, st, (const int32_t*)pb->nonempty, (const int32_t*)pb->n_nonempty,
             pb->hmark, pb->halo, pb->nhalo, (const unsigned long long*)pb->scan_ticket, pb->scan_tiles, P);
}

// physical reorder into binned order: out[j] = in[perm[j]] (all 30 fields + id)
__global__ void k_reorder(const float* __restrict__ Sin, float* __restrict__ Sout, int64_t n,
                          const int32_t* __restrict__ ids_in, int32_t* __restrict__ ids_out,
                          const int32_t* __restrict__ perm) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int p = perm[j];
  const float* src = Sin + pbase(p);
  float* dst = Sout + pbase(j);
#pragma unroll
  for (int k = 0; k < kPlanes; ++k) dst[k * 32] = __ldg(src + k * 32);
  ids_out[j] = __ldg(ids_in + p);
}

// Physical reorder of the re-binning with each block's particles sorted by cell
// (counting sort over the block's 64 cells): consecutive particles of a segment
// then share a stencil, so the fused kernel's velocity-tile reads are mostly
// broadcasts.  Persistent CTAs claim blocks by ticket (counters[1], reset by the
// scan).  The order within a cell is not specified.
__global__ void __launch_bounds__(256) k_reorder_cells(const float* __restrict__ Sin, float* __restrict__ Sout,
                                                      const int32_t* __restrict__ ids_in, int32_t* __restrict__ ids_out,
                                                      const int32_t* __restrict__ perm,
                                                      const int32_t* __restrict__ block_start,
                                                      const int32_t* __restrict__ nonempty, int32_t* counters,
                                                      DevParams P) {
  __shared__ int cnt[64];
  __shared__ int next;
  const int tid = threadIdx.x;
  const int nblk = *(volatile int32_t*)&counters[0];
  auto cell_of = [&](int src, const BlockCoord& bc) {
    int c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      int b = (int)floorf(__ldg(Sin + pbase(src) + (PX + a) * 32) * P.inv_dx - 0.5f);
      b = min(max(b, 0), P.N[a] - 3);
      c[a] = min(max(b - 4 * bc.b[a], 0), 3);
    }
    return (c[0] << 4) | (c[1] << 2) | c[2];
  };
  while (true) {
    if (tid == 0) next = atomicAdd(&counters[1], 1);
    if (tid < 64) cnt[tid] = 0;
    __syncthreads();
    const int bi = next;
    if (bi >= nblk) break;
    const int key = nonempty[bi];
    const BlockCoord bc = decode_block(key, P);
    const int s0 = block_start[key], s1 = block_start[key + 1];
    for (int j = s0 + tid; j < s1; j += 256) atomicAdd(&cnt[cell_of(perm[j], bc)], 1);
    __syncthreads();
    if (tid < 32) {   // exclusive scan of the 64 counts, two per lane
      const int v0 = cnt[2 * tid], v1 = cnt[2 * tid + 1];
      int incl = v0 + v1;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, d);
        if (tid >= d) incl += t;
      }
      const int excl = incl - v0 - v1;
      cnt[2 * tid] = excl;
      cnt[2 * tid + 1] = excl + v0;
    }
    __syncthreads();
    for (int j = s0 + tid; j < s1; j += 256) {
      const int src = perm[j];
      const int dst = s0 + atomicAdd(&cnt[cell_of(src, bc)], 1);
      const float* sp = Sin + pbase(src);
      float* dp = Sout + pbase(dst);
#pragma unroll
      for (int k = 0; k < kPlanes; ++k) dp[k * 32] = __ldg(sp + k * 32);
      ids_out[dst] = __ldg(ids_in + src);
    }
    __syncthreads();
  }
}

void launch_reorder_cells(cudaStream_t st, const float* Sin, float* Sout, int64_t n, const int32_t* ids_in,
                          int32_t* ids_out, const PipelineBuffers* pb, const DevParams& P) {
  if (n == 0) return;
  k_reorder_cells<<<num_sms() * 6, 256, 0, st>>>(Sin, Sout, ids_in, ids_out, pb->perm, pb->block_start, pb->nonempty,
                                                 pb->n_nonempty, P);
}

// NSF_PDL=0 launches without programmatic dependent launch (A/B)
static bool pdl_enabled() {
  static int f = -1;
  if (f < 0) {
    const char* e = getenv("NSF_PDL");
    f = (e && e[0] == '0') ? 0 : 1;
  }
  return f == 1;
}

template <bool DO_G2P, int ROWS, int MINB, int NT, bool HS, int ROT, bool GATH, bool WR>
static void launch_g2p2g_tg(cudaStream_t st, float* S, const int32_t* ids, const float4* vel, float4* acc, PipelineBuffers* pb,
                           const DevParams& P, DevErr* err, int64_t* d_step) {
  static bool attr = false;
  const size_t smem = sizeof(FusedSmemT<ROWS>);
  if (!attr) {
    cudaFuncSetAttribute(k_g2p2g<DO_G2P, ROWS, MINB, NT, HS, ROT, GATH, WR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    // the persistent grid is one wave of MINB CTAs per SM (the barrier mode relies on it).
    // (Measured: a register cap above 96 for 3 x 192 threads -- __maxnreg__(104 / 112) --
    // leaves 2 CTAs per SM: C3 102.7 / 104.6 vs 88.5 us.)
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_g2p2g<DO_G2P, ROWS, MINB, NT, HS, ROT, GATH, WR>, NT, smem);
    if (nb < MINB) fprintf(stderr, "nsf_mpm: k_g2p2g<%d x %d> fits %d CTAs per SM, %d wanted\n", NT, MINB, nb, MINB);
    attr = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(num_sms() * MINB);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = la;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_g2p2g<DO_G2P, ROWS, MINB, NT, HS, ROT, GATH, WR>, S, ids, vel, acc, pb->flags, pb->touched,
                     pb->touched + pb->total_blocks, pb->block_start, pb->nonempty, pb->n_nonempty, P, err, d_step,
                     pb->rg, pb->hmark, pb->gather, (const unsigned long long*)pb->scan_ticket, pb->scan_tiles);
}

template <bool DO_G2P, int ROWS, int MINB, int NT, bool HS = false, int ROT = 0>
static void launch_g2p2g_t(cudaStream_t st, float* S, const int32_t* ids, const float4* vel, float4* acc, PipelineBuffers* pb,
                           const DevParams& P, DevErr* err, int64_t* d_step) {
  // the substep after a deferred re-binning gathers (its own instantiation: the
  // gather's registers must not reach the regular one)
  // (and one that keeps v, C, tau in registers: pb->skip_vct)
  if (DO_G2P && pb->gather.S) {
    if (pb->skip_vct) launch_g2p2g_tg<DO_G2P, ROWS, MINB, NT, HS, ROT, true, false>(st, S, ids, vel, acc, pb, P, err, d_step);
    else launch_g2p2g_tg<DO_G2P, ROWS, MINB, NT, HS, ROT, true, true>(st, S, ids, vel, acc, pb, P, err, d_step);
  } else if (DO_G2P && pb->skip_vct) {
    launch_g2p2g_tg<DO_G2P, ROWS, MINB, NT, HS, ROT, false, false>(st, S, ids, vel, acc, pb, P, err, d_step);
  } else {
    launch_g2p2g_tg<DO_G2P, ROWS, MINB, NT, HS, ROT, false, true>(st, S, ids, vel, acc, pb, P, err, d_step);
  }
}

template <int ROT>
static void launch_g2p2g_r(cudaStream_t st, bool do_g2p, float* S, const int32_t* ids, const float4* vel, float4* acc,
                           PipelineBuffers* pb, const DevParams& P, DevErr* err, int64_t* d_step) {
  if (do_g2p && P.vm_hs) {   // von Mises with a per-particle yield stress
    if (pb->sparse)
      launch_g2p2g_t<true, NSF_SPARSE_ROWS, NSF_SPARSE_MIN_BLOCKS, 192, true, ROT>(st, S, ids, vel, acc, pb, P, err, d_step);
    else
      launch_g2p2g_t<true, kRowsF, NSF_DENSE_MIN_BLOCKS, NSF_DENSE_THREADS, true, ROT>(st, S, ids, vel, acc, pb, P, err,
                                                                                      d_step);
    return;
  }
  if (do_g2p && pb->dense3s) {   // dense, 3 CTAs per SM of 192 threads (A/B)
    launch_g2p2g_t<true, kRowsF, 3, 192, false, ROT>(st, S, ids, vel, acc, pb, P, err, d_step);
    return;
  }
  if (do_g2p && pb->dense2) {   // dense, 2 CTAs per SM
    launch_g2p2g_t<true, kRowsF, 2, NSF_DENSE_THREADS, false, ROT>(st, S, ids, vel, acc, pb, P, err, d_step);
    return;
  }
  if (pb->sparse) {
    if (do_g2p)
      launch_g2p2g_t<true, NSF_SPARSE_ROWS, NSF_SPARSE_MIN_BLOCKS, 192, false, ROT>(st, S, ids, vel, acc, pb, P, err, d_step);
    else
      launch_g2p2g_t<false, NSF_SPARSE_ROWS, NSF_SPARSE_MIN_BLOCKS, 192, false, ROT>(st, S, ids, vel, acc, pb, P, err,
                                                                                    d_step);
  } else {
    if (do_g2p)
      launch_g2p2g_t<true, kRowsF, NSF_DENSE_MIN_BLOCKS, NSF_DENSE_THREADS, false, ROT>(st, S, ids, vel, acc, pb, P, err,
                                                                                       d_step);
    else
      launch_g2p2g_t<false, kRowsF, NSF_DENSE_MIN_BLOCKS, NSF_DENSE_THREADS, false, ROT>(st, S, ids, vel, acc, pb, P, err,
                                                                                        d_step);
  }
}

void launch_g2p2g(cudaStream_t st, bool do_g2p, float* S, const int32_t* ids, const float4* vel, float4* acc,
                  PipelineBuffers* pb,
                  const DevParams& P, DevErr* err, int64_t* d_step) {
  if (pb->gub) launch_g2p2g_r<2>(st, do_g2p, S, ids, vel, acc, pb, P, err, d_step);
  else if (pb->rot) launch_g2p2g_r<1>(st, do_g2p, S, ids, vel, acc, pb, P, err, d_step);
  else launch_g2p2g_r<0>(st, do_g2p, S, ids, vel, acc, pb, P, err, d_step);
}

#ifndef NSF_GU_CTAS_PER_SM
#define NSF_GU_CTAS_PER_SM 8
#endif
void launch_grid_update_flags(cudaStream_t st, PipelineBuffers* pb, float4* acc, float4* vel, const DevParams& P,
                              const int64_t* d_step) {
  const int grid = num_sms() * NSF_GU_CTAS_PER_SM;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_grid_update_list, pb->flags, (const int*)pb->touched, pb->touched + pb->total_blocks,
                     (const int*)pb->halo, (const int*)pb->nhalo, (const int*)pb->hmark,
                     (const unsigned long long*)pb->scan_ticket, pb->scan_tiles, acc, vel, P, d_step,
                     pb->n_nonempty);
}

void launch_reorder(cudaStream_t st, const float* Sin, float* Sout, int64_t n, const int32_t* ids_in, int32_t* ids_out,
                    const int32_t* perm) {
  if (n == 0) return;
  k_reorder<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(Sin, Sout, n, ids_in, ids_out, perm);
}

}  // namespace nsf

namespace nsf {
// statistics build: copy out and clear the counters (nsf_mpm_debug_stats)
int stats_read(cudaStream_t st, int64_t* out, int n) {
#if NSF_STATS
  unsigned long long h[kStCount];
  if (cudaStreamSynchronize(st) != cudaSuccess) return -1;
  if (cudaMemcpyFromSymbol(h, g_nsf_stats, sizeof(h)) != cudaSuccess) return -1;
  for (int i = 0; i < n && i < kStCount; ++i) out[i] = (int64_t)h[i];
  const unsigned long long z[kStCount] = {};
  if (cudaMemcpyToSymbol(g_nsf_stats, z, sizeof(z)) != cudaSuccess) return -1;
  return kStCount;
#else
  (void)st; (void)out; (void)n;
  return 0;
#endif
}
}  // namespace nsf
