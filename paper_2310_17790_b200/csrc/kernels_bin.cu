// Binning: counting sort of particle slots by the
// 4x4x4-cell block containing base_p = floor(x_p/dx - 1/2), so that the P2G and
// G2P CTAs own grid tiles.  Keys are integers computed from exact fp32 products
// (reading #10), so counts and block_start are bit-exact against the oracle's
// block_keys; the order inside a block is not unique.
//
//   keys_hist : key[j], counts[key]++            (warp-aggregated atomics)
//   scan      : single-pass decoupled look-back exclusive scan of counts ->
//               block_start, scatter cursors, compacted non-empty block list;
//               zeroes counts for the next substep
//   scatter   : perm[cursor[key]++] = j          (warp-aggregated atomics)
#include <cuda_runtime.h>
#include <cstdint>
#include "pipeline.h"

namespace nsf {

__device__ __forceinline__ int block_key_of(float x0, float x1, float x2, int scene, const DevParams& P) {
  int b[3];
  float xs[3] = {x0, x1, x2};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    float t = xs[a] * P.inv_dx;
    int base = (int)floorf(t - 0.5f);
    base = min(max(base, 0), P.N[a] - 3);
    b[a] = base >> 2;
  }
  return (int)(scene * P.blocks_per_scene + block_id(b[0], b[1], b[2], P));
}

// warp-aggregated atomicAdd(&arr[key], 1): returns this lane's slot
__device__ __forceinline__ int aggregated_increment(int* arr, int key, unsigned active) {
  unsigned peers = __match_any_sync(active, key);
  int lane = threadIdx.x & 31;
  int leader = __ffs(peers) - 1;
  int rank = __popc(peers & ((1u << lane) - 1));
  int base = 0;
  if (lane == leader) base = atomicAdd(&arr[key], __popc(peers));
  base = __shfl_sync(peers, base, leader);
  return base + rank;
}

__global__ void k_keys_hist(int64_t n, const float* __restrict__ S, int64_t pitch,
                            const int64_t* __restrict__ scene_off, int n_scenes, int32_t* keys,
                            int32_t* counts, DevParams P) {
  pdl_launch_dependents();
  pdl_wait();
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  unsigned active = __ballot_sync(0xffffffffu, j < n);
  if (j >= n) return;
  int scene = 0;
  if (n_scenes > 1) {
    int lo = 0, hi = n_scenes;
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (scene_off[mid] <= j) lo = mid; else hi = mid;
    }
    scene = lo;
  }
  int key = block_key_of(S[pbase(j) + (PX + 0) * 32], S[pbase(j) + (PX + 1) * 32], S[pbase(j) + (PX + 2) * 32], scene, P);
  keys[j] = key;
  aggregated_increment(counts, key, active);
}

void launch_keys_hist(cudaStream_t st, int64_t n, const float* S, int64_t pitch, const int64_t* scene_off,
                      int n_scenes, int32_t* keys, int32_t* counts, const DevParams& P) {
  if (n == 0) return;
  int bs = 256;
  launch_pdl(k_keys_hist, dim3((unsigned)((n + bs - 1) / bs)), dim3(bs), 0, st, n, S, pitch, scene_off, n_scenes, keys,
             counts, P);
}

// ---------------------------------------------------------------------------
// Decoupled look-back scan (single pass).  Packed 64-bit running value: particle
// count in bits 0..31, non-empty-block count in bits 32..57.  Status word of a
// tile: value | epoch (bits 58..61) | flag (bits 62..63).  Tiles take tickets
// from a monotone counter: tile = ticket % n_tiles, epoch = ticket / n_tiles, so
// a status written by an earlier launch never matches and no reset is needed
// (the kernel is one graph node, no memsets).  Items are read and written
// warp-striped (coalesced); each warp scans its 16 x 32 items group by group.
constexpr int kScanThreads = 256;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;
constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagInc = 2ull << 62;
constexpr unsigned long long kFlagMask = 3ull << 62;
constexpr unsigned long long kEpochMask = 15ull << 58;
constexpr unsigned long long kValMask = (1ull << 58) - 1;

__device__ __forceinline__ unsigned long long packed(int c) {
  return (unsigned long long)c + ((c > 0 ? 1ull : 0ull) << 32);
}

__global__ void __launch_bounds__(kScanThreads) k_scan(int64_t total, int32_t* counts, int32_t* block_start,
                                                       int32_t* cursor, int32_t* nonempty, int32_t* n_nonempty,
                                                       unsigned long long* status, unsigned long long* ticket,
                                                       int64_t n_tiles, int32_t* ne_of, int4* cellcnt) {
  pdl_launch_dependents();
  pdl_wait();
  __shared__ unsigned long long warp_sums[kScanThreads / 32];
  __shared__ unsigned long long s_prefix;
  __shared__ unsigned long long s_ticket;
  if (threadIdx.x == 0) s_ticket = atomicAdd(ticket, 1ull);
  __syncthreads();
  const int64_t tile = (int64_t)(s_ticket % (unsigned long long)n_tiles);
  const unsigned long long ep = ((s_ticket / (unsigned long long)n_tiles) & 15ull) << 58;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t wbase = tile * kScanTile + (int64_t)warp * (kScanItems * 32);
  int c[kScanItems];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = wbase + k * 32 + lane;
    c[k] = i < total ? counts[i] : 0;
  }
  // per group k: inclusive warp scan of packed values; keep exclusive offsets
  unsigned long long excl[kScanItems];
  unsigned long long run = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    unsigned long long x = packed(c[k]);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    excl[k] = run + x - packed(c[k]);
    run += __shfl_sync(0xffffffffu, x, 31);
  }
  if (lane == 0) warp_sums[warp] = run;
  __syncthreads();
  unsigned long long warp_off = 0, agg = 0;
#pragma unroll
  for (int w = 0; w < kScanThreads / 32; ++w) {
    if (w < warp) warp_off += warp_sums[w];
    agg += warp_sums[w];
  }
  if (warp == 0) {
    unsigned long long prefix = 0;
    if (tile == 0) {
      if (lane == 0) atomicExch(&status[0], kFlagInc | ep | agg);
      // work counters of the kernels that follow (grid update, P2G, G2P)
      // ([4]: the halo list's length, built after this scan)
      if (lane >= 1 && lane <= 4) n_nonempty[lane] = 0;
    } else {
      if (lane == 0) atomicExch(&status[tile], kFlagAgg | ep | agg);
      int64_t base_t = tile - 1;
      while (true) {
        const int64_t t = base_t - lane;
        unsigned long long s = kFlagInc | ep;   // t < 0 behaves as an inclusive zero
        if (t >= 0) {
          do {
            s = *(volatile unsigned long long*)&status[t];
          } while ((s & kFlagMask) == 0 || (s & kEpochMask) != ep);
        }
        const unsigned inc_mask = __ballot_sync(0xffffffffu, (s & kFlagMask) == kFlagInc);
        unsigned long long val = s & kValMask;
        const bool done = inc_mask != 0;
        if (done && lane > __ffs(inc_mask) - 1) val = 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
        prefix += val;
        if (done) break;
        base_t -= 32;
      }
      if (lane == 0) atomicExch(&status[tile], kFlagInc | ep | (prefix + agg));
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  const unsigned long long off = s_prefix + warp_off;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = wbase + k * 32 + lane;
    if (i < total) {
      const unsigned long long r = off + excl[k];
      const int start = (int)(r & 0xffffffffull);
      block_start[i] = start;
      cursor[i] = start;
      if (c[k] > 0) {
        const int e = (int)((r >> 32) & 0x3ffffffull);
        nonempty[e] = (int)i;
        if (cellcnt) {   // cell-ordered re-binning: block -> list index, zeroed cell counters
          ne_of[i] = e;
#pragma unroll
          for (int q = 0; q < 16; ++q) cellcnt[16 * (int64_t)e + q] = make_int4(0, 0, 0, 0);
        }
      }
      counts[i] = 0;
    }
  }
  if (tile == n_tiles - 1 && threadIdx.x == 0) {
    const unsigned long long r = s_prefix + agg;
    block_start[total] = (int)(r & 0xffffffffull);
    *n_nonempty = (int)((r >> 32) & 0x3ffffffull);
  }
}

void launch_scan(cudaStream_t st, PipelineBuffers* pb) {
  launch_pdl(k_scan, dim3((unsigned)pb->scan_tiles), dim3(kScanThreads), 0, st, pb->total_blocks, pb->counts, pb->block_start,
                                                             pb->cursor, pb->nonempty, pb->n_nonempty,
                                                             pb->scan_status, pb->scan_ticket, pb->scan_tiles,
                                                             pb->ne_of, reinterpret_cast<int4*>(pb->cellcnt));
}

int64_t scan_tiles_for(int64_t total_blocks) { return (total_blocks + kScanTile - 1) / kScanTile; }

// ---------------------------------------------------------------------------
__global__ void k_scatter(int64_t n, const int32_t* __restrict__ keys, int32_t* cursor, int32_t* perm) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  unsigned active = __ballot_sync(0xffffffffu, j < n);
  if (j >= n) return;
  int slot = aggregated_increment(cursor, keys[j], active);
  perm[slot] = (int32_t)j;
}

void launch_scatter(cudaStream_t st, int64_t n, const int32_t* keys, int32_t* cursor, int32_t* perm) {
  if (n == 0) return;
  int bs = 256;
  k_scatter<<<(unsigned)((n + bs - 1) / bs), bs, 0, st>>>(n, keys, cursor, perm);
}

__global__ void k_gather_ids(int64_t n, const int32_t* __restrict__ perm, const int32_t* __restrict__ ids,
                             int32_t* out) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < n) out[k] = ids[perm[k]];
}

void launch_gather_ids(cudaStream_t st, int64_t n, const int32_t* perm, const int32_t* ids, int32_t* out) {
  if (n == 0) return;
  k_gather_ids<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, perm, ids, out);
}

// X reference planes (load order, pitch) -> the AoSoA X planes of the store, slot j
// holding particle ids[j]
__global__ void k_gather_xref(int64_t n, const float* __restrict__ X, int64_t pitch, const int32_t* __restrict__ ids,
                              float* S) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int32_t id = ids[j];
#pragma unroll
  for (int a = 0; a < 3; ++a) S[pbase(j) + (PXR + a) * 32] = X[a * pitch + id];
}

void launch_gather_xref(cudaStream_t st, int64_t n, const float* X, int64_t pitch, const int32_t* ids, float* S) {
  if (n > 0) k_gather_xref<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, X, pitch, ids, S);
}

__global__ void k_aos_to_planes(int64_t n, const float* __restrict__ aos, int ncomp, float* planes, int64_t pitch) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int k = 0; k < ncomp; ++k) planes[k * pitch + i] = aos[i * ncomp + k];
}

void launch_aos_to_planes(cudaStream_t st, int64_t n, const float* aos, int ncomp, float* planes, int64_t pitch) {
  if (n == 0) return;
  k_aos_to_planes<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, aos, ncomp, planes, pitch);
}

// ---------------------------------------------------------------------------
// Cell-ordered re-binning (storage sorted by block, and by cell inside each
// block), as three flat passes over the particles in their current order:
//   k_cell_rank : rank[j] = arrival rank of j among its cell's particles
//                 (counters cellcnt[64 e + cell], e = the block's list index)
//   k_cell_scan : one warp per non-empty block: counts -> absolute cell starts
//   k_copy_cells: out[cellcnt[64 e + cell] + rank[j]] = in[j]  (30 planes + id)
// Reads are sequential; the writes of a warp land in runs (one per cell).  The
// order inside a cell is not specified.
__device__ __forceinline__ int cell_of_x(float x0, float x1, float x2, const DevParams& P) {
  const float xs[3] = {x0, x1, x2};
  int c = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    int base = (int)floorf(xs[a] * P.inv_dx - 0.5f);   // as block_key_of
    base = min(max(base, 0), P.N[a] - 3);
    c = (c << 2) | (base & 3);
  }
  return c;
}

__global__ void k_cell_rank(int64_t n, const float* __restrict__ S, const int32_t* __restrict__ keys,
                            const int32_t* __restrict__ ne_of, int32_t* cellcnt, int32_t* __restrict__ rank,
                            DevParams P) {
  pdl_launch_dependents();
  pdl_wait();
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const unsigned active = __ballot_sync(0xffffffffu, j < n);
  if (j >= n) return;
  const float* b = S + pbase(j);
  const int cell = cell_of_x(b[(PX + 0) * 32], b[(PX + 1) * 32], b[(PX + 2) * 32], P);
  const int slot = 64 * ne_of[keys[j]] + cell;
  rank[j] = aggregated_increment(cellcnt, slot, active);
}

__global__ void k_cell_scan(int32_t* cellcnt, const int32_t* __restrict__ nonempty,
                            const int32_t* __restrict__ n_nonempty, const int32_t* __restrict__ block_start) {
  pdl_launch_dependents();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int nblk = *n_nonempty;
  for (int e = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); e < nblk;
       e += (int)((gridDim.x * (int64_t)blockDim.x) >> 5)) {
    int2* c2 = reinterpret_cast<int2*>(cellcnt + 64 * (int64_t)e);
    const int2 v = c2[lane];
    int incl = v.x + v.y;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += y;
    }
    const int s = block_start[nonempty[e]] + incl - v.x - v.y;
    c2[lane] = make_int2(s, s + v.x);
  }
}

__global__ void __launch_bounds__(128) k_copy_cells(int64_t n, const float* __restrict__ Sin, float* __restrict__ Sout,
                                                    const int32_t* __restrict__ ids_in, int32_t* __restrict__ ids_out,
                                                    const int32_t* __restrict__ keys, const int32_t* __restrict__ ne_of,
                                                    const int32_t* __restrict__ cellcnt,
                                                    const int32_t* __restrict__ rank, DevParams P) {
  pdl_launch_dependents();
  pdl_wait();
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const float* sp = Sin + pbase(j);
  float v[kPlanes];
#pragma unroll
  for (int k = 0; k < kPlanes; ++k) v[k] = __ldcs(sp + k * 32);   // read once: streaming
  const int id = __ldcs(ids_in + j);
  const int cell = cell_of_x(v[PX + 0], v[PX + 1], v[PX + 2], P);
  const int64_t dst = cellcnt[64 * ne_of[keys[j]] + cell] + rank[j];
  NSF_CHECK(dst >= 0 && dst < n);
  float* dp = Sout + pbase(dst);
#pragma unroll
  for (int k = 0; k < kPlanes; ++k) dp[k * 32] = v[k];
  ids_out[dst] = id;
}

// deferred reorder: only the map of the new order, gmap[dst(j)] = j
__global__ void __launch_bounds__(256) k_cell_map(int64_t n, const float* __restrict__ S,
                                                  const int32_t* __restrict__ keys, const int32_t* __restrict__ ne_of,
                                                  const int32_t* __restrict__ cellcnt, const int32_t* __restrict__ rank,
                                                  int32_t* __restrict__ gmap, DevParams P) {
  pdl_launch_dependents();
  pdl_wait();
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const float* b = S + pbase(j);
  const int cell = cell_of_x(b[(PX + 0) * 32], b[(PX + 1) * 32], b[(PX + 2) * 32], P);
  const int64_t dst = cellcnt[64 * ne_of[keys[j]] + cell] + rank[j];
  NSF_CHECK(dst >= 0 && dst < n);
  gmap[dst] = (int32_t)j;
}

void launch_reorder_map(cudaStream_t st, const float* S, int64_t n, PipelineBuffers* pb, const DevParams& P) {
  if (n == 0) return;
  const unsigned g = (unsigned)((n + 255) / 256);
  launch_pdl(k_cell_rank, dim3(g), dim3(256), 0, st, n, S, (const int32_t*)pb->keys, (const int32_t*)pb->ne_of,
             pb->cellcnt, pb->perm, P);
  launch_pdl(k_cell_scan, dim3(num_sms() * 4), dim3(256), 0, st, pb->cellcnt, (const int32_t*)pb->nonempty,
             (const int32_t*)pb->n_nonempty, (const int32_t*)pb->block_start);
  launch_pdl(k_cell_map, dim3(g), dim3(256), 0, st, n, S, (const int32_t*)pb->keys, (const int32_t*)pb->ne_of,
             (const int32_t*)pb->cellcnt, (const int32_t*)pb->perm, pb->gmap, P);
}

void launch_reorder_cells_flat(cudaStream_t st, const float* Sin, float* Sout, int64_t n, const int32_t* ids_in,
                               int32_t* ids_out, PipelineBuffers* pb, const DevParams& P) {
  if (n == 0) return;
  const unsigned g = (unsigned)((n + 255) / 256);
  launch_pdl(k_cell_rank, dim3(g), dim3(256), 0, st, n, Sin, (const int32_t*)pb->keys, (const int32_t*)pb->ne_of,
             pb->cellcnt, pb->perm, P);
  launch_pdl(k_cell_scan, dim3(num_sms() * 4), dim3(256), 0, st, pb->cellcnt, (const int32_t*)pb->nonempty,
             (const int32_t*)pb->n_nonempty, (const int32_t*)pb->block_start);
  launch_pdl(k_copy_cells, dim3((unsigned)((n + 127) / 128)), dim3(128), 0, st, n, Sin, Sout, ids_in, ids_out,
             (const int32_t*)pb->keys, (const int32_t*)pb->ne_of, (const int32_t*)pb->cellcnt,
             (const int32_t*)pb->perm, P);
}

// Processing order of the fused kernel's segments (longest first): the
// persistent CTAs claim segments by ticket in list order, so with the largest
// segments first the last claims are the small (surface) blocks and the CTAs
// finish closer together (LPT scheduling).  One CTA: counting sort of the
// non-empty list by descending particle count (buckets of 4).  The storage
// order and ne_of are not affected (ne_of is only used inside the re-binning).
__global__ void __launch_bounds__(1024) k_lpt_order(int32_t* __restrict__ nonempty,
                                                    const int32_t* __restrict__ n_nonempty,
                                                    const int32_t* __restrict__ block_start, int32_t* __restrict__ tmp) {
  pdl_launch_dependents();
  pdl_wait();
  __shared__ int hist[256];
  const int tid = threadIdx.x;
  const int nblk = *n_nonempty;
  auto bucket = [&](int key) { return 255 - min((block_start[key + 1] - block_start[key]) >> 2, 255); };
  for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  for (int e = tid; e < nblk; e += blockDim.x) {
    const int key = nonempty[e];
    tmp[e] = key;
    atomicAdd(&hist[bucket(key)], 1);
  }
  __syncthreads();
  if (tid < 32) {   // exclusive scan of the 256 buckets, 8 per lane
    int v[8], sum = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) { v[k] = hist[8 * tid + k]; sum += v[k]; }
    int incl = sum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, d);
      if (tid >= d) incl += y;
    }
    int run = incl - sum;
#pragma unroll
    for (int k = 0; k < 8; ++k) { hist[8 * tid + k] = run; run += v[k]; }
  }
  __syncthreads();
  for (int e = tid; e < nblk; e += blockDim.x) {
    const int key = tmp[e];
    nonempty[atomicAdd(&hist[bucket(key)], 1)] = key;
  }
}

void launch_lpt_order(cudaStream_t st, PipelineBuffers* pb) {
  launch_pdl(k_lpt_order, dim3(1), dim3(1024), 0, st, pb->nonempty, (const int32_t*)pb->n_nonempty,
             (const int32_t*)pb->block_start, pb->ne_tmp);
}

}  // namespace nsf
