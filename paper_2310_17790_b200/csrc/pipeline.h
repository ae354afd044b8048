// Substep pipeline (internal): which kernels run, in which order, on which
// buffers.  runtime.cu owns the handle; this layer only sees a HandleView.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include "../../include/nsf_mpm.h"
#include "kernels.h"
#include "params.cuh"

namespace nsf {

// fused kernel variant threshold: mean particles per non-empty 4^3-cell block
constexpr int kSparseParticlesPerBlock = 256;

// Fused full-order pipeline with the grid update inside the G2P2G kernel: three
// grid accumulators used in rotation.  Kernel k (k = substeps done) reads the
// raw P2G sums of buffer k % 3 (updating each node as it stages its velocity
// tile), reduces the next P2G into buffer (k + 1) % 3 and clears the
// blocks of buffer (k + 2) % 3 (written two kernels ago, read by kernel k - 1;
// nobody touches it during kernel k).  Each buffer has its own touched-block
// flags and list; the list of the P2G written by kernel k counts in cnt[k & 3]
// (kernel k resets cnt[(k + 1) & 3], which kernel k - 1 read last).  cnt[4]
// counts finished CTAs: the last one advances the step counter.
struct RotGrid {
  float4* buf[3] = {nullptr, nullptr, nullptr};
  int* flags = nullptr;             // [3][total_blocks]
  int* list = nullptr;              // [3][total_blocks]
  int* cnt = nullptr;               // [8]
  int64_t total_blocks = 0;
};

// Deferred reorder (fused pipeline): a periodic re-binning computes only the map of
// the new storage order (map[j] = the particle of the previous buffer that goes to
// slot j); the next substep's k_g2p2g gathers x, F (tau_Y, id) through it and
// writes its new state into the other buffer in order, so the store is reordered
// without a copy pass.  S == nullptr: in place.
struct GatherIn {
  const float* S = nullptr;
  const int32_t* map = nullptr;
  const int32_t* ids = nullptr;
  int32_t* ids_out = nullptr;
};

struct PipelineBuffers {
  // binning: block key per particle slot, per-block counts,
  // start offsets (exclusive scan), scatter cursors, permutation, active list
  int32_t* keys = nullptr;          // [pitch]
  int32_t* counts = nullptr;        // [total_blocks]      (zero between substeps)
  int32_t* block_start = nullptr;   // [total_blocks + 1]
  int32_t* cursor = nullptr;        // [total_blocks]
  int32_t* perm = nullptr;          // [pitch]  sorted slot -> storage slot
  int32_t* nonempty = nullptr;      // [total_blocks] list of non-empty block ids
  int32_t* ne_of = nullptr;         // [total_blocks] list index of a non-empty block (cell-ordered re-binning)
  int32_t* ne_tmp = nullptr;        // [total_blocks] scratch of the longest-first segment order (fused)
  int32_t* cellcnt = nullptr;       // [64 * min(total_blocks, pitch)] per-cell counts, then starts (idem)
  int32_t* n_nonempty = nullptr;    // [8]: n_nonempty, (unused), barrier count, segment ticket, halo length
                                    //      (1-4 reset by the scan)
  unsigned long long* scan_status = nullptr;  // [scan tiles]
  unsigned long long* scan_ticket = nullptr;  // [1] monotone ticket counter
  int64_t scan_tiles = 0;
  int64_t total_blocks = 0;
  int64_t pitch = 0;
  bool tiled = false;               // dense tiled path (full-order models)
  bool fused = false;               // fused G2P2G pipeline (full-order, MLS)
  bool sparse = false;
  bool dense2 = false;      // dense variant at 2 CTAs per SM (128 registers)
  bool dense3s = false;     // dense variant at 3 CTAs per SM of 192 threads (96 registers): many segments
  bool mode_ready = false;  // fused: variant and grid-update mode chosen (pipeline_on_load)
  bool nsf_sorted = false;          // reduced path: points kept in block order (periodic re-binning)              // fused kernel variant for few particles per block (chosen at load)
  int* flags = nullptr;             // [total_blocks] grid blocks touched by P2G (fused pipeline)
  int* touched = nullptr;           // [total_blocks] list of touched blocks, then [count], [done]
  int* hmark = nullptr;             // [total_blocks] halo membership (fused, separate grid update; k_halo)
  int* halo = nullptr;              // [total_blocks] halo list
  int* nhalo = nullptr;             // its length (= n_nonempty + 4)
  int* nsf_done = nullptr;          // reduced path: CTA completion counter of the G2P kernel
  bool rot = false;                 // fused pipeline with the in-kernel grid update (RotGrid)
  bool gub = false;                 // fused pipeline with the grid update at the end of k_g2p2g (barrier)
  float4* grid3 = nullptr;          // its third grid accumulator
  RotGrid rg;
  float4* dbg_acc = nullptr;        // reduced path: scratch grids for debug_grid
  unsigned long long* fx = nullptr; // deterministic mode: fixed-point P2G accumulator [total_nodes][4]
  float4* dbg_vel = nullptr;
  int32_t* gmap = nullptr;          // [pitch] deferred reorder map (fused)
  bool gather_pending = false;      // the next fused substep gathers through gmap
  bool skip_vct = false;            // set around a k_g2p2g launch: v, C, tau are not written back (a substep
                                    // that is not the last of its nsf_mpm_substep(n) call: nothing can read them)
  GatherIn gather;                  // the gather of the k_g2p2g being enqueued
  int rebin_every = 32;             // fused pipeline: substeps between re-binnings
  int since_rebin = 0;              // host counter
  int64_t launch_total = 0;         // kernel launches enqueued since load
  int launches = 0;                 // kernels per substep (last enqueued)
};

struct HandleView {
  const DevParams* P;
  cudaStream_t stream;
  int64_t n, pitch;
  float* S[2];
  int32_t* ids[2];
  const int64_t* scene_off;
  const int64_t* scene_off_host;
  int n_scenes;
  float4* acc;
  float4* vel;
  int64_t total_nodes, total_blocks;
  DevErr* err;
  int64_t* d_step;
  int cur;                          // current particle buffer
  int64_t host_step;                // substeps enqueued since load
  const MlpDev* mlp;
  const float* X;
  const float* z;
  const float* dz;
  int r;
  int model;
};

// provided by runtime.cu
HandleView view(nsf_mpm* h);
void set_cur(nsf_mpm* h, int cur);
void* pipeline_alloc(nsf_mpm* h, size_t bytes);
void pipeline_free(nsf_mpm* h, void* p);
void prof_begin(nsf_mpm* h, const char* name, cudaEvent_t* a);
void prof_end(nsf_mpm* h, const char* name, cudaEvent_t a);

// provided by pipeline.cu
int pipeline_create(nsf_mpm* h, PipelineBuffers* pb, const DevParams& P, int64_t total_blocks);
nsf_status pipeline_particles(nsf_mpm* h, PipelineBuffers* pb, int64_t pitch);
nsf_status pipeline_on_load(nsf_mpm* h, PipelineBuffers* pb);
void pipeline_on_mlp(nsf_mpm* h, PipelineBuffers* pb);
bool pipeline_graphable(nsf_mpm* h, PipelineBuffers* pb);
inline bool pipeline_fused(const PipelineBuffers* pb) { return pb->fused; }   // k_g2p2g path (full-order, MLS)
int pipeline_variant(nsf_mpm* h, PipelineBuffers* pb);             // graph variant of the next substep
int pipeline_substep(nsf_mpm* h, PipelineBuffers* pb, int cur, int variant);   // returns next buffer or -1
void pipeline_advance(nsf_mpm* h, PipelineBuffers* pb, int variant, int launches);          // host bookkeeping after one substep
void pipeline_aos_to_planes(cudaStream_t st, int64_t n, const float* aos, int ncomp, float* planes,
                            int64_t pitch);
void pipeline_eval_mlp(nsf_mpm* h, PipelineBuffers* pb, int64_t m, const float* planes, int64_t pitch,
                       const float* z, int r, float* tau_aos);
int pipeline_debug_bins(nsf_mpm* h, PipelineBuffers* pb, int cur, int32_t* counts, int32_t* perm,
                        int on_device);
int pipeline_debug_grid(nsf_mpm* h, PipelineBuffers* pb, int cur, int stage, float* out);
int pipeline_launches_per_substep(nsf_mpm* h, PipelineBuffers* pb);
int64_t pipeline_launch_total(nsf_mpm* h, PipelineBuffers* pb);
void pipeline_destroy(nsf_mpm* h, PipelineBuffers* pb);

// kernels_bin.cu
void launch_keys_hist(cudaStream_t st, int64_t n, const float* S, int64_t pitch, const int64_t* scene_off,
                      int n_scenes, int32_t* keys, int32_t* counts, const DevParams& P);
void launch_scan(cudaStream_t st, PipelineBuffers* pb);
void launch_scatter(cudaStream_t st, int64_t n, const int32_t* keys, int32_t* cursor, int32_t* perm);
void launch_lpt_order(cudaStream_t st, PipelineBuffers* pb);
void launch_halo(cudaStream_t st, PipelineBuffers* pb, const DevParams& P);
void launch_gather_ids(cudaStream_t st, int64_t n, const int32_t* perm, const int32_t* ids, int32_t* out);
void launch_gather_xref(cudaStream_t st, int64_t n, const float* X, int64_t pitch, const int32_t* ids, float* S);
void launch_aos_to_planes(cudaStream_t st, int64_t n, const float* aos, int ncomp, float* planes, int64_t pitch);

// kernels_tiled.cu
void launch_p2g_tiled(cudaStream_t st, const float* S, int64_t pitch, const int32_t* perm, const PipelineBuffers* pb,
                      float4* acc, const DevParams& P);
void launch_grid_update_blocks(cudaStream_t st, const PipelineBuffers* pb, float4* acc, float4* vel,
                               const DevParams& P, const int64_t* d_step);
void p2g_tables_init(cudaStream_t st);
void launch_g2p2g(cudaStream_t st, bool do_g2p, float* S, const int32_t* ids, const float4* vel, float4* acc,
                  PipelineBuffers* pb,
                  const DevParams& P, DevErr* err, int64_t* d_step);
void launch_grid_update_flags(cudaStream_t st, PipelineBuffers* pb, float4* acc, float4* vel, const DevParams& P,
                              const int64_t* d_step);
void launch_reorder(cudaStream_t st, const float* Sin, float* Sout, int64_t n, const int32_t* ids_in, int32_t* ids_out,
                    const int32_t* perm);
// kernels_det.cu (deterministic mode)
void launch_p2g_fixed(cudaStream_t st, int64_t n, const float* S, const int64_t* scene_off, int n_scenes,
                      unsigned long long* fx, PipelineBuffers* pb, const DevParams& P);
void launch_grid_update_fixed(cudaStream_t st, PipelineBuffers* pb, unsigned long long* fx, float4* vel,
                              const DevParams& P, const int64_t* d_step);
void launch_reorder_cells(cudaStream_t st, const float* Sin, float* Sout, int64_t n, const int32_t* ids_in,
                          int32_t* ids_out, const PipelineBuffers* pb, const DevParams& P);
void launch_reorder_cells_flat(cudaStream_t st, const float* Sin, float* Sout, int64_t n, const int32_t* ids_in,
                               int32_t* ids_out, PipelineBuffers* pb, const DevParams& P);
void launch_reorder_map(cudaStream_t st, const float* S, int64_t n, PipelineBuffers* pb, const DevParams& P);
int num_sms();
int stats_read(cudaStream_t st, int64_t* out, int n);   // statistics build only (else 0)
void launch_g2p_tiled(cudaStream_t st, const float* Sin, float* Sout, int64_t n, const int32_t* ids_in,
                      int32_t* ids_out, const PipelineBuffers* pb, const float4* vel, const int64_t* scene_off,
                      int n_scenes, const DevParams& P, DevErr* err, int64_t* d_step);

}  // namespace nsf
