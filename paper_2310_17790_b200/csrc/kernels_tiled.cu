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
//  g2p_tiled   (a5 + a6): the block's 6x6x6 velocity tile is staged
//              in shared memory, then one thread per particle gathers 27 nodes,
//              updates x, v, C, F, runs the SVD + return map, and writes the
//              particle to the other buffer at its sorted slot (sort-on-write),
//              with its next block key and the histogram for the next binning.
#include <cuda_runtime.h>
#include <cstdint>
#include "mpm_math.cuh"
#include "pipeline.h"

namespace nsf {

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
  bc.scene = (int)(key / P.blocks_per_scene);
  int local = (int)(key % P.blocks_per_scene);
  bc.b[2] = local % P.NB[2];
  bc.b[1] = (local / P.NB[2]) % P.NB[1];
  bc.b[0] = local / (P.NB[2] * P.NB[1]);
  return bc;
}

// ---------------------------------------------------------------------------
// P2G (MLS force form)
constexpr int kP2GThreads = 192;   // 64 cells x 3 stencil planes (ox)
constexpr int kRows = 12;          // particles per cell per round
constexpr int kSlotFields = 21;    // w(9), u0(3), q0(3), q1(3), q2(3)
constexpr int kSlotStride = kRows * 64;   // floats per field
constexpr int kSegment = 2048;     // particles of one block handled per segment

struct __align__(16) P2GSmem {
  union {
    float slot[kSlotFields * kSlotStride];   // [field][row][cell]
    float part[27 * 4 * 64];                 // [(node*4 + comp)][cell]
  } u;
  uint32_t cr[kSegment];   // (cell << 16) | rank within the cell, per particle of the segment
  int pop[64];             // cell populations of the segment
  int max_pop;
};

// one particle -> 21 floats of slot data at s = row*64 + cell
__device__ __forceinline__ void p2g_stage_particle(const float* __restrict__ S, int64_t pitch, int p, int s,
                                                   float* sl, const DevParams& P) {
  const float m = P.mass;
  const Axis a0 = bspline_axis(S[(PX + 0) * pitch + p], P.inv_dx);
  const Axis a1 = bspline_axis(S[(PX + 1) * pitch + p], P.inv_dx);
  const Axis a2 = bspline_axis(S[(PX + 2) * pitch + p], P.inv_dx);
  const float v0 = S[(PV + 0) * pitch + p], v1 = S[(PV + 1) * pitch + p], v2 = S[(PV + 2) * pitch + p];
  float Cm[9], T[6];
#pragma unroll
  for (int k = 0; k < 9; ++k) Cm[k] = S[(PC + k) * pitch + p];
#pragma unroll
  for (int k = 0; k < 6; ++k) T[k] = S[(PT + k) * pitch + p];
  const float Tm[9] = {T[0], T[5], T[4], T[5], T[1], T[3], T[4], T[3], T[2]};
  float Q[9];   // Q = m C - dt V0 (4/dx^2) tau  (MLS, reading #1)
#pragma unroll
  for (int k = 0; k < 9; ++k) Q[k] = m * Cm[k] - P.mls_coef * Tm[k];
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

__device__ __forceinline__ int cell_in_block(const float* __restrict__ S, int64_t pitch, int p, const BlockCoord& bc,
                                             const DevParams& P) {
  int c[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float t = S[(PX + a) * pitch + p] * P.inv_dx;
    int base = (int)floorf(t - 0.5f);
    base = min(max(base, 0), P.N[a] - 3);
    c[a] = base - 4 * bc.b[a];
  }
  return (c[0] << 4) | (c[1] << 2) | c[2];
}

__global__ void __launch_bounds__(kP2GThreads, 3)
k_p2g_tiled(const float* __restrict__ S, int64_t pitch, const int32_t* __restrict__ perm,
            const int32_t* __restrict__ block_start, const int32_t* __restrict__ nonempty,
            const int32_t* __restrict__ n_nonempty, float4* acc, DevParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  P2GSmem& sm = *reinterpret_cast<P2GSmem*>(smem_raw);
  const int tid = threadIdx.x;
  const int my_cell = tid & 63;
  const int ox = tid >> 6;
  const float fox = (float)ox;
  const int nblk = *n_nonempty;
  for (int bi = blockIdx.x; bi < nblk; bi += gridDim.x) {
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
      // pass A: cell and rank of every particle of the segment
      for (int i = tid; i < cnt; i += kP2GThreads) {
        const int cell = cell_in_block(S, pitch, perm[seg + i], bc, P);
        const int rank = atomicAdd(&sm.pop[cell], 1);
        sm.cr[i] = ((uint32_t)cell << 16) | (uint32_t)rank;
      }
      __syncthreads();
      if (tid < 64) atomicMax(&sm.max_pop, sm.pop[tid]);
      __syncthreads();
      const int rounds = (sm.max_pop + kRows - 1) / kRows;
      const int my_pop = sm.pop[my_cell];
      for (int round = 0; round < rounds; ++round) {
        // pass B: stage the particles whose rank falls in this round
        for (int i = tid; i < cnt; i += kP2GThreads) {
          const uint32_t cr = sm.cr[i];
          const int r = (int)(cr & 0xffffu) - round * kRows;
          if (r < 0 || r >= kRows) continue;
          p2g_stage_particle(S, pitch, perm[seg + i], r * 64 + (int)(cr >> 16), sm.u.slot, P);
        }
        __syncthreads();
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
            const float uyx = fmaf((float)oy, q1x, ux), uyy = fmaf((float)oy, q1y, uy), uyz = fmaf((float)oy, q1z, uz);
#pragma unroll
            for (int oz = 0; oz < 3; ++oz) {
              const float W = wxy * wzv[oz];
              const int k = oy * 3 + oz;
              accm[k] += W;
              accp[k][0] = fmaf(W, fmaf((float)oz, q2x, uyx), accp[k][0]);
              accp[k][1] = fmaf(W, fmaf((float)oz, q2y, uyy), accp[k][1]);
              accp[k][2] = fmaf(W, fmaf((float)oz, q2z, uyz), accp[k][2]);
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
      const int nx = t / 36, ny = (t / 6) % 6, nz = t % 6;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
      for (int cx = max(0, nx - 2); cx <= min(3, nx); ++cx)
        for (int cy = max(0, ny - 2); cy <= min(3, ny); ++cy)
          for (int cz = max(0, nz - 2); cz <= min(3, nz); ++cz) {
            const int node = ((nx - cx) * 3 + (ny - cy)) * 3 + (nz - cz);
            const int c = (cx << 4) | (cy << 2) | cz;
            s0 += part[(node * 4 + 0) * 64 + c];
            s1 += part[(node * 4 + 1) * 64 + c];
            s2 += part[(node * 4 + 2) * 64 + c];
            s3 += part[(node * 4 + 3) * 64 + c];
          }
      if (s0 > 0.0f) {
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
constexpr int kGridThreads = 512;   // 8 targets x 64 nodes

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

__global__ void __launch_bounds__(kGridThreads)
k_grid_update_blocks(const int32_t* __restrict__ block_start, const int32_t* __restrict__ nonempty,
                     const int32_t* __restrict__ n_nonempty, float4* acc, float4* vel, DevParams P,
                     const int64_t* __restrict__ d_step) {
  const int nblk = *n_nonempty;
  const int d = threadIdx.x >> 6;        // target offset index 0..7
  const int l = threadIdx.x & 63;        // node within the target block
  const int d0 = (d >> 2) & 1, d1 = (d >> 1) & 1, d2 = d & 1;
  const float y_plate = (float)((double)P.plate_y0 + (double)P.plate_v[1] * ((double)(*d_step) * (double)P.dt));
  for (int bi = blockIdx.x; bi < nblk; bi += gridDim.x) {
    const int key = nonempty[bi];
    const BlockCoord bc = decode_block(key, P);
    const int t0 = bc.b[0] + d0, t1 = bc.b[1] + d1, t2 = bc.b[2] + d2;
    if (t0 >= P.NB[0] || t1 >= P.NB[1] || t2 >= P.NB[2]) continue;
    // ownership: no earlier offset d' < d (same enumeration) has a non-empty source
    bool owner = true;
    for (int e = 0; e < d && owner; ++e) {
      const int e0 = (e >> 2) & 1, e1 = (e >> 1) & 1, e2 = e & 1;
      if (count_of(block_start, bc.scene, t0 - e0, t1 - e1, t2 - e2, P) > 0) owner = false;
    }
    if (!owner) continue;
    const int64_t g = (int64_t)bc.scene * P.nodes_per_scene + block_id(t0, t1, t2, P) * kBlockNodes + l;
    const float4 a = acc[g];
    const int i = t0 * 4 + (l >> 4), j = t1 * 4 + ((l >> 2) & 3), k = t2 * 4 + (l & 3);
    vel[g] = grid_node_update_t(a, i, j, k, P, y_plate);
    acc[g] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// ---------------------------------------------------------------------------
// G2P + constitutive, sort-on-write
constexpr int kG2PThreads = 256;

template <int FORCE>
__global__ void __launch_bounds__(kG2PThreads, 2)
k_g2p_tiled(const float* __restrict__ Sin, float* __restrict__ Sout, int64_t pitch,
            const int32_t* __restrict__ ids_in, int32_t* __restrict__ ids_out,
            const int32_t* __restrict__ perm, const int32_t* __restrict__ block_start,
            const int32_t* __restrict__ nonempty, const int32_t* __restrict__ n_nonempty,
            const float4* __restrict__ vel, int32_t* __restrict__ keys, int32_t* __restrict__ counts,
            DevParams P, DevErr* err, int64_t* d_step) {
  __shared__ float4 tile[8 * 64];   // the 2x2x2 blocks b + d, each 64 nodes
  const int nblk = *n_nonempty;
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd((unsigned long long*)d_step, 1ull);
  const float cC = 4.0f * P.inv_dx * P.inv_dx;
  for (int bi = blockIdx.x; bi < nblk; bi += gridDim.x) {
    const int key = nonempty[bi];
    const BlockCoord bc = decode_block(key, P);
    const float4* vb = vel + (int64_t)bc.scene * P.nodes_per_scene;
    __syncthreads();   // previous block's readers are done with the tile
    for (int e = threadIdx.x; e < 8 * 64; e += kG2PThreads) {
      const int d = e >> 6, l = e & 63;
      const int t0 = bc.b[0] + ((d >> 2) & 1), t1 = bc.b[1] + ((d >> 1) & 1), t2 = bc.b[2] + (d & 1);
      float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
      if (t0 < P.NB[0] && t1 < P.NB[1] && t2 < P.NB[2]) val = vb[block_id(t0, t1, t2, P) * kBlockNodes + l];
      tile[e] = val;
    }
    __syncthreads();
    const int start = block_start[key], end = block_start[key + 1];
    for (int j = start + threadIdx.x; j < end; j += kG2PThreads) {
      const unsigned active = __activemask();
      const int p = perm[j];
      float xp[3] = {Sin[(PX + 0) * pitch + p], Sin[(PX + 1) * pitch + p], Sin[(PX + 2) * pitch + p]};
      Axis ax[3];
      int lo[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        ax[a] = bspline_axis(xp[a], P.inv_dx);
        ax[a].base = min(max(ax[a].base, 0), P.N[a] - 3);
        lo[a] = ax[a].base - 4 * bc.b[a];   // 0..3
      }
      float v[3] = {0.f, 0.f, 0.f};
      float Bm[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      float G[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const int la = lo[0] + a;
        const int sa = la >> 2, wa = la & 3;
        const float da = ((float)a - ax[0].f) * P.dx;
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          const int lb = lo[1] + b;
          const int sb = lb >> 2, wb = lb & 3;
          const float db = ((float)b - ax[1].f) * P.dx;
          const float wab = ax[0].w[a] * ax[1].w[b];
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const int lc = lo[2] + c;
            const int sc = lc >> 2, wc = lc & 3;
            const float dc = ((float)c - ax[2].f) * P.dx;
            const float W = wab * ax[2].w[c];
            const float4 vi = tile[(((sa << 2) | (sb << 1) | sc) << 6) | (wa << 4) | (wb << 2) | wc];
            const float wv0 = W * vi.x, wv1 = W * vi.y, wv2 = W * vi.z;
            v[0] += wv0; v[1] += wv1; v[2] += wv2;
            Bm[0] = fmaf(wv0, da, Bm[0]); Bm[1] = fmaf(wv0, db, Bm[1]); Bm[2] = fmaf(wv0, dc, Bm[2]);
            Bm[3] = fmaf(wv1, da, Bm[3]); Bm[4] = fmaf(wv1, db, Bm[4]); Bm[5] = fmaf(wv1, dc, Bm[5]);
            Bm[6] = fmaf(wv2, da, Bm[6]); Bm[7] = fmaf(wv2, db, Bm[7]); Bm[8] = fmaf(wv2, dc, Bm[8]);
            if (FORCE == 1) {
              const float g0 = ax[0].dw[a] * ax[1].w[b] * ax[2].w[c];
              const float g1 = ax[0].w[a] * ax[1].dw[b] * ax[2].w[c];
              const float g2 = ax[0].w[a] * ax[1].w[b] * ax[2].dw[c];
              G[0] += vi.x * g0; G[1] += vi.x * g1; G[2] += vi.x * g2;
              G[3] += vi.y * g0; G[4] += vi.y * g1; G[5] += vi.y * g2;
              G[6] += vi.z * g0; G[7] += vi.z * g1; G[8] += vi.z * g2;
            }
          }
        }
      }
      float Cn[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) Cn[k] = cC * Bm[k];
      if (FORCE == 0) {
#pragma unroll
        for (int k = 0; k < 9; ++k) G[k] = Cn[k];
      }
      float xn[3];
      bool ok = true, finite = true;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        xn[a] = xp[a] + P.dt * v[a];
        const float t = xn[a] * P.inv_dx;
        ok &= (t >= 0.5f) && (t < (float)P.N[a] - 1.5f);
        finite &= isfinite(xn[a]) && isfinite(v[a]);
      }
      float Fp[9], Ft[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) Fp[k] = Sin[(PF + k) * pitch + p];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int jj = 0; jj < 3; ++jj)
          Ft[i * 3 + jj] = Fp[i * 3 + jj] + P.dt * (G[i * 3 + 0] * Fp[0 * 3 + jj] + G[i * 3 + 1] * Fp[1 * 3 + jj] +
                                                    G[i * 3 + 2] * Fp[2 * 3 + jj]);
      float FE[9], tau[6];
      const float J = elastoplastic(Ft, P.model, P.mu, P.lam, P.alpha, P.tau_Y, FE, tau);
      // sorted write (coalesced over j)
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        Sout[(PX + a) * pitch + j] = xn[a];
        Sout[(PV + a) * pitch + j] = v[a];
      }
#pragma unroll
      for (int k = 0; k < 9; ++k) Sout[(PC + k) * pitch + j] = Cn[k];
#pragma unroll
      for (int k = 0; k < 9; ++k) { Sout[(PF + k) * pitch + j] = FE[k]; finite &= isfinite(FE[k]); }
#pragma unroll
      for (int k = 0; k < 6; ++k) { Sout[(PT + k) * pitch + j] = tau[k]; finite &= isfinite(tau[k]); }
      const int id = ids_in[p];
      ids_out[j] = id;
      if (!(J > 0.0f)) atomicAdd(&err->inverted, 1ull);
      if (!ok) { atomicOr(&err->bits, ERR_OUT_OF_DOMAIN); atomicMin(&err->first_index, id); }
      if (!finite) { atomicOr(&err->bits, ERR_NONFINITE); atomicMin(&err->first_index, id); }
      // next block key + histogram (warp-aggregated)
      int nb[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        int base = (int)floorf(xn[a] * P.inv_dx - 0.5f);
        base = min(max(base, 0), P.N[a] - 3);
        nb[a] = base >> 2;
      }
      const int nkey = (int)(bc.scene * P.blocks_per_scene + block_id(nb[0], nb[1], nb[2], P));
      keys[j] = nkey;
      const unsigned peers = __match_any_sync(active, nkey);
      const int lane = threadIdx.x & 31;
      const int leader = __ffs(peers) - 1;
      if (lane == leader) atomicAdd(&counts[nkey], __popc(peers));
    }
  }
}

// ---------------------------------------------------------------------------
static int g_num_sms = 0;
static int num_sms() {
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
}

void launch_grid_update_blocks(cudaStream_t st, const PipelineBuffers* pb, float4* acc, float4* vel,
                               const DevParams& P, const int64_t* d_step) {
  int grid = num_sms() * 4;
  k_grid_update_blocks<<<grid, kGridThreads, 0, st>>>(pb->block_start, pb->nonempty, pb->n_nonempty, acc, vel, P,
                                                      d_step);
}

void launch_g2p_tiled(cudaStream_t st, const float* Sin, float* Sout, int64_t pitch, const int32_t* ids_in,
                      int32_t* ids_out, const PipelineBuffers* pb, const float4* vel, const DevParams& P, DevErr* err,
                      int64_t* d_step) {
  int grid = num_sms() * 2;
  if (P.force_mode == 0)
    k_g2p_tiled<0><<<grid, kG2PThreads, 0, st>>>(Sin, Sout, pitch, ids_in, ids_out, pb->perm, pb->block_start,
                                                 pb->nonempty, pb->n_nonempty, vel, pb->keys, pb->counts, P, err,
                                                 d_step);
  else
    k_g2p_tiled<1><<<grid, kG2PThreads, 0, st>>>(Sin, Sout, pitch, ids_in, ids_out, pb->perm, pb->block_start,
                                                 pb->nonempty, pb->n_nonempty, vel, pb->keys, pb->counts, P, err,
                                                 d_step);
}

}  // namespace nsf
