// Substep pipeline: the order of kernels for one MLS-MPM substep (PAPER.md
// §3.3) and for the reduced variant.
#include <cuda_runtime.h>
#include <cstdlib>
#include <cstring>
#include "pipeline.h"
#include "point_ops.cuh"

namespace nsf {

int64_t scan_tiles_for(int64_t total_blocks);

#define PLAUNCH(h, name, ...)           \
  do {                                  \
    cudaEvent_t _ev = nullptr;          \
    prof_begin(h, name, &_ev);          \
    __VA_ARGS__;                        \
    prof_end(h, name, _ev);             \
  } while (0)

// particles of a block stored in cell order.  NSF_REORDER_CELLS=0: block order
// only; =block: one CTA per block (counting sort in shared memory); default:
// flat passes (kernels_bin.cu)
static int reorder_mode() {
  static int f = -1;
  if (f < 0) {
    const char* e = getenv("NSF_REORDER_CELLS");
    f = (e && e[0] == '0') ? 0 : (e && strcmp(e, "block") == 0) ? 2 : 1;
  }
  return f;
}

int pipeline_create(nsf_mpm* h, PipelineBuffers* pb, const DevParams& P, int64_t total_blocks) {
  pb->total_blocks = total_blocks;
  pb->scan_tiles = scan_tiles_for(total_blocks);
  pb->counts = (int32_t*)pipeline_alloc(h, sizeof(int32_t) * total_blocks);
  pb->block_start = (int32_t*)pipeline_alloc(h, sizeof(int32_t) * (total_blocks + 1));
  pb->cursor = (int32_t*)pipeline_alloc(h, sizeof(int32_t) * total_blocks);
  pb->nonempty = (int32_t*)pipeline_alloc(h, sizeof(int32_t) * total_blocks);
  pb->ne_tmp = (int32_t*)pipeline_alloc(h, sizeof(int32_t) * total_blocks);
  if (reorder_mode() == 1) {
    pb->ne_of = (int32_t*)pipeline_alloc(h, sizeof(int32_t) * total_blocks);
    if (!pb->ne_of) return -1;
  }
  pb->n_nonempty = (int32_t*)pipeline_alloc(h, sizeof(int32_t) * 8);
  pb->scan_status = (unsigned long long*)pipeline_alloc(h, sizeof(unsigned long long) * pb->scan_tiles);
  pb->scan_ticket = (unsigned long long*)pipeline_alloc(h, sizeof(unsigned long long) * 4);
  if (!pb->counts || !pb->block_start || !pb->cursor || !pb->nonempty || !pb->ne_tmp || !pb->n_nonempty || !pb->scan_status ||
      !pb->scan_ticket)
    return -1;
  HandleView v = view(h);
  if (cudaMemsetAsync(pb->counts, 0, sizeof(int32_t) * total_blocks, v.stream) != cudaSuccess) return -1;
  // scan status words carry an epoch; start from a clean slate once
  if (cudaMemsetAsync(pb->scan_status, 0, sizeof(unsigned long long) * pb->scan_tiles, v.stream) != cudaSuccess)
    return -1;
  if (cudaMemsetAsync(pb->scan_ticket, 0, sizeof(unsigned long long) * 4, v.stream) != cudaSuccess) return -1;
  if (cudaMemsetAsync(pb->n_nonempty, 0, sizeof(int32_t) * 8, v.stream) != cudaSuccess) return -1;
  pb->flags = (int*)pipeline_alloc(h, sizeof(int) * total_blocks);
  pb->touched = (int*)pipeline_alloc(h, sizeof(int) * (total_blocks + 4));
  pb->hmark = (int*)pipeline_alloc(h, sizeof(int) * total_blocks);
  pb->halo = (int*)pipeline_alloc(h, sizeof(int) * total_blocks);
  pb->nhalo = pb->n_nonempty ? pb->n_nonempty + 4 : nullptr;   // reset by every scan
  if (!pb->flags || !pb->touched || !pb->hmark || !pb->halo || !pb->nhalo) return -1;
  if (cudaMemsetAsync(pb->hmark, 0, sizeof(int) * total_blocks, v.stream) != cudaSuccess) return -1;
  if (cudaMemsetAsync(pb->flags, 0, sizeof(int) * total_blocks, v.stream) != cudaSuccess) return -1;
  if (cudaMemsetAsync(pb->touched, 0, sizeof(int) * (total_blocks + 4), v.stream) != cudaSuccess) return -1;
  p2g_tables_init(v.stream);
  if (cudaGetLastError() != cudaSuccess) return -1;
  pb->tiled = false;
  (void)P;
  return 0;
}

nsf_status pipeline_particles(nsf_mpm* h, PipelineBuffers* pb, int64_t pitch) {
  if (pb->keys) pipeline_free(h, pb->keys);
  if (pb->perm) pipeline_free(h, pb->perm);
  if (pb->gmap) pipeline_free(h, pb->gmap);
  if (pb->cellcnt) pipeline_free(h, pb->cellcnt);
  pb->cellcnt = nullptr;

  pb->keys = (int32_t*)pipeline_alloc(h, sizeof(int32_t) * pitch);
  pb->perm = (int32_t*)pipeline_alloc(h, sizeof(int32_t) * pitch);
  pb->gmap = (int32_t*)pipeline_alloc(h, sizeof(int32_t) * pitch);
  pb->pitch = pitch;
  pb->gather_pending = false;
  if (!pb->keys || !pb->perm || !pb->gmap) return NSF_ERR_OUT_OF_MEMORY;
  if (reorder_mode() == 1) {   // a non-empty block holds >= 1 particle
    const int64_t max_nonempty = pitch < pb->total_blocks ? pitch : pb->total_blocks;
    pb->cellcnt = (int32_t*)pipeline_alloc(h, sizeof(int32_t) * 64 * (max_nonempty > 0 ? max_nonempty : 1));
    if (!pb->cellcnt) return NSF_ERR_OUT_OF_MEMORY;
  }
  return NSF_OK;
}

// Re-binning with a physical reorder of buffer `cur` into 1 - cur (fused pipeline):
// keys + histogram, scan (block_start, non-empty list), scatter (perm), reorder.
static bool lpt_enabled() {
  static int f = -1;
  if (f < 0) {
    const char* e = getenv("NSF_LPT");
    f = (e && e[0] == '0') ? 0 : 1;
  }
  return f == 1;
}

static int enqueue_rebin_body(nsf_mpm* h, PipelineBuffers* pb, const HandleView& v, int cur, bool deferred);

// periodic re-binnings of the fused pipeline leave the reorder to the next substep
// (GatherIn); NSF_DEFERRED_REORDER=0 copies the store as the re-binning's last pass
static bool deferred_reorder() {
  static int f = -1;
  if (f < 0) {
    const char* e = getenv("NSF_DEFERRED_REORDER");
    f = (e && e[0] == '0') ? 0 : 1;
  }
  return f == 1 && reorder_mode() == 1;
}

// longest-first only for dense scenes: in sparse ones (C4: 1237 vs 1296 us) the
// spatial order of the non-empty list keeps neighbouring segments' grid lines in L2
static bool lpt_active(const PipelineBuffers* pb) {
  return pb->fused && pb->mode_ready && !pb->sparse && lpt_enabled();
}
// the halo list only serves the separate grid-update pass
static bool halo_active(const PipelineBuffers* pb) { return pb->fused && pb->mode_ready && !pb->rot && !pb->gub; }

// kernels one re-binning launches: keys + histogram, scan, reorder (flat: rank,
// cell scan, copy; else scatter + copy), and the longest-first order (fused)
static int rebin_launches(const PipelineBuffers* pb, int64_t n) {
  if (n == 0) return 1 + (halo_active(pb) ? 1 : 0);
  return 2 + (reorder_mode() == 1 ? 3 : 2) + (lpt_active(pb) ? 1 : 0) + (halo_active(pb) ? 1 : 0);
}

// the fused kernel then processes its segments longest first (k_lpt_order)
static int enqueue_rebin(nsf_mpm* h, PipelineBuffers* pb, const HandleView& v, int cur, bool deferred = false) {
  const int nxt = enqueue_rebin_body(h, pb, v, cur, deferred);
  if (lpt_active(pb) && v.n > 0) PLAUNCH(h, "bin_lpt", launch_lpt_order(v.stream, pb));
  if (halo_active(pb)) PLAUNCH(h, "bin_halo", launch_halo(v.stream, pb, *v.P));
  return nxt;
}

static int enqueue_rebin_body(nsf_mpm* h, PipelineBuffers* pb, const HandleView& v, int cur, bool deferred) {
  const int nxt = 1 - cur;
  PLAUNCH(h, "bin_keys_hist",
          launch_keys_hist(v.stream, v.n, v.S[cur], v.pitch, v.scene_off, v.n_scenes, pb->keys, pb->counts, *v.P));
  PLAUNCH(h, "bin_scan", launch_scan(v.stream, pb));
  if (deferred) {   // the map only; the store stays in buffer cur until the next substep
    PLAUNCH(h, "reorder_map", launch_reorder_map(v.stream, v.S[cur], v.n, pb, *v.P));
    return cur;
  }
  if (reorder_mode() == 1) {
    PLAUNCH(h, "reorder",
            launch_reorder_cells_flat(v.stream, v.S[cur], v.S[nxt], v.n, v.ids[cur], v.ids[nxt], pb, *v.P));
    return nxt;
  }
  PLAUNCH(h, "bin_scatter", launch_scatter(v.stream, v.n, pb->keys, pb->cursor, pb->perm));
  if (reorder_mode() == 2)
    PLAUNCH(h, "reorder",
            launch_reorder_cells(v.stream, v.S[cur], v.S[nxt], v.n, v.ids[cur], v.ids[nxt], pb, *v.P));
  else
    PLAUNCH(h, "reorder", launch_reorder(v.stream, v.S[cur], v.S[nxt], v.n, v.ids[cur], v.ids[nxt], pb->perm));
  return nxt;
}

static bool nsf_sort_enabled() {
  static int f = -1;
  if (f < 0) {
    const char* e = getenv("NSF_REDUCED_SORT");
    f = (e && strcmp(e, "0") == 0) ? 0 : 1;
  }
  return f == 1;
}

// grid update inside the fused kernel (three rotating accumulators, RotGrid) or
// the separate k_grid_update_list pass: NSF_FUSED_GU=rot|kernel forces one
// (read at every load, so a test can run both in one process)
static int rot_mode() {
  const char* e = getenv("NSF_FUSED_GU");
  return (e && strcmp(e, "kernel") == 0) ? 0 : (e && strcmp(e, "rot") == 0) ? 1
         : (e && strcmp(e, "barrier") == 0) ? 2 : -1;
}

static nsf_status rot_setup(nsf_mpm* h, PipelineBuffers* pb, const HandleView& v) {
  RotGrid& rg = pb->rg;
  const int64_t TB = pb->total_blocks;
  if (!pb->grid3) {
    pb->grid3 = (float4*)pipeline_alloc(h, sizeof(float4) * v.total_nodes);
    if (!pb->grid3) return NSF_ERR_OUT_OF_MEMORY;
  }
  if (!rg.flags) {
    rg.flags = (int*)pipeline_alloc(h, sizeof(int) * 3 * TB);
    rg.list = (int*)pipeline_alloc(h, sizeof(int) * 3 * TB);
    rg.cnt = (int*)pipeline_alloc(h, sizeof(int) * 8);
    if (!rg.flags || !rg.list || !rg.cnt) return NSF_ERR_OUT_OF_MEMORY;
  }
  rg.buf[0] = v.acc;
  rg.buf[1] = v.vel;
  rg.buf[2] = pb->grid3;
  rg.total_blocks = TB;
  if (cudaMemsetAsync(v.vel, 0, sizeof(float4) * v.total_nodes, v.stream) != cudaSuccess ||
      cudaMemsetAsync(pb->grid3, 0, sizeof(float4) * v.total_nodes, v.stream) != cudaSuccess ||
      cudaMemsetAsync(rg.flags, 0, sizeof(int) * 3 * TB, v.stream) != cudaSuccess ||
      cudaMemsetAsync(rg.cnt, 0, sizeof(int) * 8, v.stream) != cudaSuccess)
    return NSF_ERR_CUDA;
  return NSF_OK;
}

static bool fused_enabled() {
  static int f = -1;
  if (f < 0) {
    const char* e = getenv("NSF_PIPELINE");
    f = (e && strcmp(e, "split") == 0) ? 0 : 1;
  }
  return f == 1;
}

// Invariants between substeps.
//  split path : keys[] and counts[] describe the particles of the current buffer
//               (written by the last G2P, or here after a load).
//  fused path : storage is sorted by block at the last re-binning (segments =
//               block_start / non-empty list); the accumulator holds P2G of the
//               current state and `flags` marks its touched blocks; counts = 0.
nsf_status pipeline_on_load(nsf_mpm* h, PipelineBuffers* pb) {
  HandleView v = view(h);
  const bool det = v.P->deterministic != 0;
  pb->tiled = v.model != NSF_NEURAL_STRESS && !det;
  // (the fused kernel packs a stencil base into 3 x 10 bits: N <= 1024 per axis)
  pb->fused = pb->tiled && v.P->force_mode == NSF_FORCE_MLS && fused_enabled() && v.P->N[0] <= 1024 &&
              v.P->N[1] <= 1024 && v.P->N[2] <= 1024;
  pb->since_rebin = 0;
  pb->launch_total = 0;
  // re-binning every 32 substeps (measured over whole 500-substep runs: 64 and 128
  // are slower on C3, as the order inside segments decays, and no faster on C2)
  pb->rebin_every = 32;
  if (const char* e = getenv("NSF_REBIN_EVERY")) pb->rebin_every = atoi(e) > 0 ? atoi(e) : 32;
  pb->nsf_sorted = false;
  if (cudaMemsetAsync(pb->counts, 0, sizeof(int32_t) * pb->total_blocks, v.stream) != cudaSuccess)
    return NSF_ERR_CUDA;
  if (cudaMemsetAsync(v.acc, 0, sizeof(float4) * v.total_nodes, v.stream) != cudaSuccess) return NSF_ERR_CUDA;
  if (cudaMemsetAsync(pb->flags, 0, sizeof(int) * pb->total_blocks, v.stream) != cudaSuccess) return NSF_ERR_CUDA;
  if (cudaMemsetAsync(pb->touched + pb->total_blocks, 0, sizeof(int) * 4, v.stream) != cudaSuccess)
    return NSF_ERR_CUDA;
  if (det) {
    // fixed-point accumulator (deterministic P2G); nothing is sorted
    if (!pb->fx) {
      pb->fx = (unsigned long long*)pipeline_alloc(h, sizeof(unsigned long long) * 4 * v.total_nodes);
      if (!pb->fx) return NSF_ERR_OUT_OF_MEMORY;
    }
    if (cudaMemsetAsync(pb->fx, 0, sizeof(unsigned long long) * 4 * v.total_nodes, v.stream) != cudaSuccess)
      return NSF_ERR_CUDA;
    if (v.model == NSF_NEURAL_STRESS && v.X)
      launch_gather_xref(v.stream, v.n, v.X, v.pitch, v.ids[0], v.S[0]);
  } else if (pb->fused) {
    pb->mode_ready = false;   // (the variant is chosen below; the segment order and halo follow)
    pb->gather_pending = false;
    const int cur = enqueue_rebin(h, pb, v, 0);
    set_cur(h, cur);
    v = view(h);
    if (cudaMemsetAsync(pb->n_nonempty + 3, 0, sizeof(int32_t), v.stream) != cudaSuccess) return NSF_ERR_CUDA;
    // kernel variant by density: fewer staged rows and more CTAs per SM when the
    // non-empty blocks hold few particles; among dense scenes, 2 CTAs per SM (more
    // registers per thread) when there are fewer than 2 segments per CTA of the
    // 3-per-SM variant (NSF_FUSED_VARIANT=dense|dense2|sparse overrides)
    int32_t nblk = 0;
    if (cudaMemcpyAsync(&nblk, pb->n_nonempty, sizeof(int32_t), cudaMemcpyDeviceToHost, v.stream) != cudaSuccess ||
        cudaStreamSynchronize(v.stream) != cudaSuccess)
      return NSF_ERR_CUDA;
    const char* fv = getenv("NSF_FUSED_VARIANT");
    if (fv && strncmp(fv, "dense", 5) == 0) pb->sparse = false;
    else if (fv && strcmp(fv, "sparse") == 0) pb->sparse = true;
    else pb->sparse = nblk > 0 && v.n < (int64_t)kSparseParticlesPerBlock * nblk;
    // dense scenes: 3 CTAs/SM of 192 threads (96 registers, no spill with the
    // paired-FMA loops; a 512-particle segment is three passes either way) when
    // there are at least 2 segments per CTA of that grid (C3: 95.9 -> 92.3 us),
    // else 2 CTAs/SM of 256 threads (128 registers; C2: 36.6 vs 40.8 us)
    const bool many = nblk >= 2 * 3 * num_sms();
    pb->dense3s = fv ? strcmp(fv, "dense3s") == 0 : (!pb->sparse && many);
    if (fv && strcmp(fv, "dense2") == 0) pb->dense2 = true;
    else if (fv) pb->dense2 = false;
    else pb->dense2 = !pb->sparse && !many;
    // where the grid update runs (NSF_FUSED_GU=kernel|rot|barrier forces one): at the
    // end of k_g2p2g after a grid-wide barrier for dense scenes with few segments per
    // CTA (C2: 36.5 us with the separate pass or the rotating grids -> 35.5); else
    // its own pass (C3: 92.5 us vs 97.0 barrier / 109 rotation; C4 1308 vs 1315; C1
    // 43.8 vs 46.5)
    const int gm = rot_mode();
    pb->rot = gm == 1;
    pb->gub = gm == 2 || (gm < 0 && !pb->sparse && nblk < 2 * 3 * num_sms());
    if (cudaMemsetAsync(pb->n_nonempty + 2, 0, sizeof(int32_t), v.stream) != cudaSuccess) return NSF_ERR_CUDA;
    pb->mode_ready = true;
    if (lpt_active(pb) && v.n > 0) launch_lpt_order(v.stream, pb);
    if (halo_active(pb)) launch_halo(v.stream, pb, *v.P);
    if (pb->rot) {
      const nsf_status rs = rot_setup(h, pb, v);
      if (rs != NSF_OK) return rs;
    }
    launch_g2p2g(v.stream, false, v.S[cur], v.ids[cur], v.vel, v.acc, pb, *v.P, v.err, v.d_step);   // P2G of state 0
  } else if (pb->tiled) {
    launch_keys_hist(v.stream, v.n, v.S[0], v.pitch, v.scene_off, v.n_scenes, pb->keys, pb->counts, *v.P);
  } else {
    // reduced path: acc and vel are the two P2G accumulators (point_ops.cuh)
    if (!pb->nsf_done) {
      pb->nsf_done = (int*)pipeline_alloc(h, sizeof(int) * 4);
      if (!pb->nsf_done) return NSF_ERR_OUT_OF_MEMORY;
    }
    if (cudaMemsetAsync(pb->nsf_done, 0, sizeof(int) * 4, v.stream) != cudaSuccess ||
        cudaMemsetAsync(v.vel, 0, sizeof(float4) * v.total_nodes, v.stream) != cudaSuccess)
      return NSF_ERR_CUDA;
    launch_nsf_reset_base(v.stream, v.n, v.S[0]);
    // keep the points in block order (periodic re-binning, as the fused path):
    // neighbouring threads then share stencil nodes in the P2G reductions and
    // the G2P gathers.  X moves with them (planes PXR..).
    if (v.X) launch_gather_xref(v.stream, v.n, v.X, v.pitch, v.ids[0], v.S[0]);
    pb->nsf_sorted = nsf_sort_enabled();
    pb->since_rebin = 0;
    if (pb->nsf_sorted && v.n > 0) {
      const int cur = enqueue_rebin(h, pb, v, 0);
      set_cur(h, cur);
    }
  }
  if (cudaGetLastError() != cudaSuccess) return NSF_ERR_CUDA;
  return NSF_OK;
}

void pipeline_on_mlp(nsf_mpm* h, PipelineBuffers* pb) {
  (void)pb;
  HandleView v = view(h);
  if (v.model == NSF_NEURAL_STRESS && v.X && v.n > 0)   // X planes of the store follow the points
    launch_gather_xref(v.stream, v.n, v.X, v.pitch, v.ids[v.cur], v.S[v.cur]);
}

bool pipeline_graphable(nsf_mpm* h, PipelineBuffers* pb) {
  (void)h;
  (void)pb;
  return true;
}

// build the binning of buffer `cur` (keys + counts -> block_start, perm, non-empty list)
static void enqueue_binning(nsf_mpm* h, PipelineBuffers* pb, const HandleView& v, int cur) {
  PLAUNCH(h, "bin_keys_hist",
          launch_keys_hist(v.stream, v.n, v.S[cur], v.pitch, v.scene_off, v.n_scenes, pb->keys, pb->counts, *v.P));
  PLAUNCH(h, "bin_scan", launch_scan(v.stream, pb));
  PLAUNCH(h, "bin_scatter", launch_scatter(v.stream, v.n, pb->keys, pb->cursor, pb->perm));
}

// bit 0: the substep ends with a re-binning; bit 1: it gathers through the
// deferred reorder map of the previous one (its kernel's buffers differ); bit 2
// (added by the caller, runtime.cu enqueue_substeps): not the last substep of its
// call, so the fused kernel keeps v, C, tau in registers only
int pipeline_variant(nsf_mpm* h, PipelineBuffers* pb) {
  (void)h;
  const int rebin = ((pb->fused || pb->nsf_sorted) && pb->since_rebin + 1 >= pb->rebin_every) ? 1 : 0;
  return rebin | ((pb->fused && pb->gather_pending) ? 2 : 0);
}

void pipeline_advance(nsf_mpm* h, PipelineBuffers* pb, int variant, int launches) {
  (void)h;
  pb->since_rebin = (variant & 1) ? 0 : pb->since_rebin + 1;
  pb->gather_pending = pb->fused && (variant & 1) && deferred_reorder();
  pb->launch_total += launches;
}

// One substep.
//  fused (full-order, MLS): grid update of the flagged blocks -> G2P(n) + P2G(n+1)
//    in place over storage segments -> (every rebin_every substeps) re-binning
//    with a physical reorder.
//  split (GRADW): scan -> scatter -> P2G (direct) -> grid update -> G2P
//    (sort-on-write into the other buffer, next keys + histogram).
//  reduced (NSF): keys + hist -> scan -> MLP -> direct P2G -> grid update -> direct G2P
//    (points are ~0.1 per cell: tiles do not pay).
int pipeline_substep(nsf_mpm* h, PipelineBuffers* pb, int cur, int variant) {
  HandleView v = view(h);
  const bool nsf_model = v.model == NSF_NEURAL_STRESS;
  int launches = 0;
  if (v.P->deterministic) {
    // deterministic: [MLP ->] fixed-point P2G -> grid update of the touched blocks -> G2P (in place)
    if (nsf_model) {
      PLAUNCH(h, "nsf_mlp",
              launch_nsf_mlp(v.stream, v.n, v.S[cur] + PXR * kTileP, -1, v.scene_off, v.n_scenes, v.z, v.dz, v.r,
                             v.d_step, *v.mlp, v.P->stress_scale, v.S[cur] + PT * kTileP, v.pitch, 0));
      launches += (v.n > 0);
    }
    PLAUNCH(h, "p2g_fixed", launch_p2g_fixed(v.stream, v.n, v.S[cur], v.scene_off, v.n_scenes, pb->fx, pb, *v.P));
    PLAUNCH(h, "grid_update", launch_grid_update_fixed(v.stream, pb, pb->fx, v.vel, *v.P, v.d_step));
    PLAUNCH(h, "g2p_direct", launch_g2p_direct(v.stream, v.n, v.S[cur], v.pitch, v.scene_off, v.n_scenes, v.vel, *v.P,
                                               v.err, v.d_step, nsf_model ? 0 : 1, v.ids[cur]));
    launches += (v.n > 0) + 2;
    pb->launches = launches;
    return cur;
  }
  if (pb->fused) {
    if (!pb->rot && !pb->gub)
      PLAUNCH(h, "grid_update", launch_grid_update_flags(v.stream, pb, v.acc, v.vel, *v.P, v.d_step));
    int next = cur;
    if (variant & 2) {   // reorder on the way: gather from buffer cur, write buffer 1 - cur in order
      next = 1 - cur;
      pb->gather.S = v.S[cur];
      pb->gather.map = pb->gmap;
      pb->gather.ids = v.ids[cur];
      pb->gather.ids_out = v.ids[next];
    }
    pb->skip_vct = (variant & 4) != 0;
    PLAUNCH(h, "g2p2g", launch_g2p2g(v.stream, true, v.S[next], v.ids[next], v.vel, v.acc, pb, *v.P, v.err, v.d_step));
    pb->skip_vct = false;
    pb->gather = GatherIn{};
    launches = (pb->rot || pb->gub) ? 1 : 2;
    if (variant & 1) {
      next = enqueue_rebin(h, pb, v, next, deferred_reorder());
      launches += rebin_launches(pb, v.n);
    }
    pb->launches = launches;
    return next;
  }
  if (!nsf_model) {
    const int nxt = 1 - cur;
    PLAUNCH(h, "bin_scan", launch_scan(v.stream, pb));
    PLAUNCH(h, "bin_scatter", launch_scatter(v.stream, v.n, pb->keys, pb->cursor, pb->perm));
    launches += 1 + (v.n > 0);
    if (v.P->force_mode == NSF_FORCE_MLS) {
      PLAUNCH(h, "p2g_tiled", launch_p2g_tiled(v.stream, v.S[cur], v.pitch, pb->perm, pb, v.acc, *v.P));
      ++launches;
    } else {
      PLAUNCH(h, "p2g_direct",
              launch_p2g_direct(v.stream, v.n, v.S[cur], v.pitch, v.scene_off, v.n_scenes, v.acc, *v.P));
      launches += (v.n > 0);
    }
    PLAUNCH(h, "grid_update", launch_grid_update_blocks(v.stream, pb, v.acc, v.vel, *v.P, v.d_step));
    PLAUNCH(h, "g2p",
            launch_g2p_tiled(v.stream, v.S[cur], v.S[nxt], v.n, v.ids[cur], v.ids[nxt], pb, v.vel, v.scene_off,
                             v.n_scenes, *v.P, v.err, v.d_step));
    launches += 2;
    pb->launches = launches;
    return nxt;
  }
  // reduced: MLP with the P2G of each point in its epilogue ->
  // G2P with the grid update applied per gathered node
  NsfP2G q;
  q.S = v.S[cur];
  q.acc0 = v.acc;
  q.acc1 = v.vel;
  q.P = *v.P;
  q.enabled = 1;
  // MLP input X from the store's X planes (xpitch < 0: AoSoA addressing)
  PLAUNCH(h, "nsf_mlp",
          launch_nsf_mlp(v.stream, v.n, v.S[cur] + PXR * kTileP, -1, v.scene_off, v.n_scenes, v.z, v.dz, v.r,
                         v.d_step, *v.mlp, v.P->stress_scale, v.S[cur] + PT * kTileP, v.pitch, 0, &q));
  PLAUNCH(h, "g2p_nsf", launch_g2p_nsf(v.stream, v.n, v.S[cur], v.scene_off, v.n_scenes, v.acc, v.vel, *v.P, v.err,
                                       v.d_step, pb->nsf_done, v.ids[cur]));
  launches += (v.n > 0 ? 2 : 1);
  if (variant && v.n > 0) {
    pb->launches = launches + rebin_launches(pb, v.n);
    return enqueue_rebin(h, pb, v, cur);
  }
  pb->launches = launches;
  return cur;
}

void pipeline_aos_to_planes(cudaStream_t st, int64_t n, const float* aos, int ncomp, float* planes, int64_t pitch) {
  launch_aos_to_planes(st, n, aos, ncomp, planes, pitch);
}

void pipeline_eval_mlp(nsf_mpm* h, PipelineBuffers* pb, int64_t m, const float* planes, int64_t pitch,
                       const float* z, int r, float* tau_aos) {
  (void)pb;
  HandleView v = view(h);
  PLAUNCH(h, "nsf_mlp_eval",
          launch_nsf_mlp(v.stream, m, planes, pitch, nullptr, 1, z, nullptr, r, nullptr, *v.mlp, v.P->stress_scale,
                         tau_aos, 0, 1));
}

int pipeline_debug_bins(nsf_mpm* h, PipelineBuffers* pb, int cur, int32_t* counts, int32_t* perm, int on_device) {
  HandleView v = view(h);
  // counts: histogram only (then clear), perm: full binning mapped to load order;
  // finally restore the between-substep invariant (keys/counts of buffer cur)
  if (cudaMemsetAsync(pb->counts, 0, sizeof(int32_t) * pb->total_blocks, v.stream) != cudaSuccess) return -1;
  if (counts) {
    launch_keys_hist(v.stream, v.n, v.S[cur], v.pitch, v.scene_off, v.n_scenes, pb->keys, pb->counts, *v.P);
    if (cudaMemcpyAsync(counts, pb->counts, sizeof(int32_t) * pb->total_blocks,
                        on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, v.stream) != cudaSuccess)
      return -1;
    if (cudaMemsetAsync(pb->counts, 0, sizeof(int32_t) * pb->total_blocks, v.stream) != cudaSuccess) return -1;
  }
  if (perm) {
    enqueue_binning(h, pb, v, cur);
    int32_t* tmp = (int32_t*)pipeline_alloc(h, sizeof(int32_t) * (v.n + 1));
    if (!tmp) return -1;
    launch_gather_ids(v.stream, v.n, pb->perm, v.ids[cur], tmp);
    cudaError_t e = cudaMemcpyAsync(perm, tmp, sizeof(int32_t) * v.n,
                                    on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, v.stream);
    cudaStreamSynchronize(v.stream);
    pipeline_free(h, tmp);
    if (e != cudaSuccess) return -1;
  }
  if (cudaMemsetAsync(pb->counts, 0, sizeof(int32_t) * pb->total_blocks, v.stream) != cudaSuccess) return -1;
  if (pb->fused) {
    // segments must describe the storage order again: re-bin and reorder (the
    // accumulator only depends on the state, which is unchanged)
    set_cur(h, enqueue_rebin(h, pb, v, cur));
    pb->since_rebin = 0;
    pb->gather_pending = false;
  } else if (pb->tiled) {
    launch_keys_hist(v.stream, v.n, v.S[cur], v.pitch, v.scene_off, v.n_scenes, pb->keys, pb->counts, *v.P);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int pipeline_debug_grid(nsf_mpm* h, PipelineBuffers* pb, int cur, int stage, float* out) {
  HandleView v = view(h);
  if (pb->fused && pb->gub) {
    // the kernel already updated and cleared its accumulator: P2G of the current
    // state again, into scratch grids (MLS form, as the fused kernel)
    if (!pb->dbg_acc) {
      pb->dbg_acc = (float4*)pipeline_alloc(h, sizeof(float4) * v.total_nodes);
      pb->dbg_vel = (float4*)pipeline_alloc(h, sizeof(float4) * v.total_nodes);
      if (!pb->dbg_acc || !pb->dbg_vel) return -1;
    }
    if (cudaMemsetAsync(pb->dbg_acc, 0, sizeof(float4) * v.total_nodes, v.stream) != cudaSuccess) return -1;
    launch_p2g_direct(v.stream, v.n, v.S[cur], v.pitch, v.scene_off, v.n_scenes, pb->dbg_acc, *v.P);
    launch_grid_debug(v.stream, stage, v.total_nodes, pb->dbg_acc, pb->dbg_vel, out, *v.P, v.d_step);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
  }
  if (pb->fused) {
    // the accumulator already holds P2G of the current state; keep it (rotation:
    // buffer step % 3, updated into a scratch grid: the other two are in use)
    if (pb->rot) {
      if (!pb->dbg_vel) {
        pb->dbg_vel = (float4*)pipeline_alloc(h, sizeof(float4) * v.total_nodes);
        if (!pb->dbg_vel) return -1;
      }
      launch_grid_debug(v.stream, stage, v.total_nodes, pb->rg.buf[v.host_step % 3], pb->dbg_vel, out, *v.P,
                        v.d_step);
    } else {
      launch_grid_debug(v.stream, stage, v.total_nodes, v.acc, v.vel, out, *v.P, v.d_step);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
  }
  float4* acc = v.acc;
  float4* vel = v.vel;
  if (v.model == NSF_NEURAL_STRESS) {
    // acc / vel hold the reduced path's accumulators: use scratch grids
    if (!pb->dbg_acc) {
      pb->dbg_acc = (float4*)pipeline_alloc(h, sizeof(float4) * v.total_nodes);
      pb->dbg_vel = (float4*)pipeline_alloc(h, sizeof(float4) * v.total_nodes);
      if (!pb->dbg_acc || !pb->dbg_vel) return -1;
    }
    acc = pb->dbg_acc;
    vel = pb->dbg_vel;
    if (cudaMemsetAsync(acc, 0, sizeof(float4) * v.total_nodes, v.stream) != cudaSuccess) return -1;
    launch_nsf_mlp(v.stream, v.n, v.S[cur] + PXR * kTileP, -1, v.scene_off, v.n_scenes, v.z, v.dz, v.r, v.d_step,
                   *v.mlp, v.P->stress_scale, v.S[cur] + PT * kTileP, v.pitch, 0);
  }
  launch_p2g_direct(v.stream, v.n, v.S[cur], v.pitch, v.scene_off, v.n_scenes, acc, *v.P);
  launch_grid_debug(v.stream, stage, v.total_nodes, acc, vel, out, *v.P, v.d_step);
  if (cudaMemsetAsync(acc, 0, sizeof(float4) * v.total_nodes, v.stream) != cudaSuccess) return -1;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int pipeline_launches_per_substep(nsf_mpm* h, PipelineBuffers* pb) {
  (void)h;
  return pb->launches;
}

int64_t pipeline_launch_total(nsf_mpm* h, PipelineBuffers* pb) {
  (void)h;
  return pb->launch_total;
}

void pipeline_destroy(nsf_mpm* h, PipelineBuffers* pb) {
  (void)h;
  (void)pb;   // buffers are tracked and freed by the handle's allocation list
}

}  // namespace nsf
