// Host runtime behind the C ABI (include/nsf_mpm.h): handle, device memory,
// stream, CUDA graph of the substep, deferred device errors, per-kernel
// event timing.  Every entry point validates its arguments, then enqueues
// kernels from kernels_*.cu; no arithmetic of the method runs on the host
// except the material constants (Lame parameters P:504-512, DP alpha P:536).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/nsf_mpm.h"
#include "kernels.h"
#include "pipeline.h"
#include "params.cuh"

using namespace nsf;

struct nsf_mpm {
  int32_t grid_res[3] = {0, 0, 0};
  double dx = 0, dt = 0;
  nsf_material mat{};
  DevParams P{};
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;   // default: a non-blocking stream owned by the handle
  void* (*ualloc)(size_t, void*, void*) = nullptr;
  void (*ufree)(void*, void*, void*) = nullptr;
  void* uctx = nullptr;
  struct Alloc {                                // a live device allocation and how to release it
    void* p;
    void (*release)(void*, void*, void*);       // NULL: cudaFree; else the hook that was current at allocation
    void* ctx;
  };
  std::vector<Alloc> allocs;

  // particles
  int64_t n = 0, pitch = 0;
  bool loaded = false;
  float* S[2] = {nullptr, nullptr};
  int32_t* ids[2] = {nullptr, nullptr};
  int cur = 0;
  int64_t* scene_off = nullptr;    // device, n_scenes + 1
  std::vector<int64_t> scene_off_host;
  // grid
  int64_t total_nodes = 0, total_blocks = 0;
  float4* acc = nullptr;
  float4* vel = nullptr;
  // pipeline scratch (binning etc.)
  PipelineBuffers pb{};
  // errors / counters
  DevErr* err = nullptr;        // device
  DevErr* err_host = nullptr;   // pinned
  int64_t* d_step = nullptr;    // device step counter
  int64_t host_step = 0;
  // NSF
  uint16_t* W = nullptr;
  float* b = nullptr;
  unsigned int* mlp_ctr = nullptr;   // MLP tile ticket + completion counter (kernels_nsf_tc.cu)
  MlpDev gdef{};                      // deformation field g (network inversion, inference)
  MlpDev ldef{};                      // affine-velocity field l (inference)
  uint16_t* lW = nullptr;
  float* lb = nullptr;
  bool ldef_loaded = false;
  float* zprev = nullptr;             // z_{n-1} of inference (n_scenes x r)
  float* zrom = nullptr;              // rom_step: the latent the last step started from (its z_{n-1})
  bool zrom_valid = false;
  uint16_t* gW = nullptr;
  float* gb = nullptr;
  bool gdef_loaded = false;
  int32_t* inv_slots = nullptr;       // inversion scratch: sample slots, working latents, fp64 sums
  float* inv_z = nullptr;
  double* inv_acc = nullptr;
  size_t inv_cap[3] = {0, 0, 0};      // their capacities (bytes); grown, never shrunk
  MlpDev mlp{};
  bool mlp_loaded = false;
  float* X = nullptr;            // 3 planes, pitch
  float* z = nullptr;
  float* dz = nullptr;
  int r = 0;
  bool latents_loaded = false;
  // staging
  void* staging = nullptr;
  size_t staging_bytes = 0;
  // graphs: one captured substep per source buffer (the pipeline may ping-pong
  // particle buffers, so the substep starting from buffer k is graph[k])
  // [source buffer][variant]; variant = pipeline_variant: bit 0 re-binning at the end,
  // bit 1 the gather of a deferred reorder, bit 2 v, C, tau not stored (not the last substep of a call)
  static constexpr int kVariants = 8;
  cudaGraphExec_t graph[2][kVariants] = {};
  int graph_next[2][kVariants] = {{0, 0, 0, 0, 0, 0, 0, 0}, {1, 1, 1, 1, 1, 1, 1, 1}};
  int graph_launches[2][kVariants] = {};   // kernels in each captured graph
  // profiling
  bool profiling = false;
  struct Pending { std::string name; cudaEvent_t a, b; };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> free_events;
  std::map<std::string, std::pair<double, int64_t>> ktimes;
  std::vector<std::string> knames_storage;
  // status
  std::string last_error;
  bool poisoned = false;
};

// ---------------------------------------------------------------------------
namespace {

nsf_status fail(nsf_mpm* h, nsf_status s, const char* fmt, ...) {
  if (h) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    h->last_error = buf;
  }
  return s;
}

nsf_status cuda_fail(nsf_mpm* h, cudaError_t e, const char* where) {
  h->poisoned = true;
  return fail(h, NSF_ERR_CUDA, "CUDA error in %s: %s", where, cudaGetErrorString(e));
}

#define CK(expr)                                                   \
  do {                                                             \
    cudaError_t _e = (expr);                                       \
    if (_e != cudaSuccess) return cuda_fail(h, _e, #expr);         \
  } while (0)

// Every device allocation goes through here.  Kernels use 256-bit accesses
// (grid node pairs) and 128-byte particle tiles, so a pointer from an allocator
// hook that is not 256-byte aligned is released again and the allocation fails.
void* dalloc(nsf_mpm* h, size_t bytes, bool* misaligned = nullptr) {
  if (misaligned) *misaligned = false;
  if (bytes == 0) bytes = 256;
  bytes = (bytes + 255) & ~size_t(255);
  void* p = nullptr;
  if (h->ualloc) {
    p = h->ualloc(bytes, (void*)h->stream, h->uctx);
    if (p && ((uintptr_t)p & 255u) != 0) {
      h->ufree(p, (void*)h->stream, h->uctx);
      if (misaligned) *misaligned = true;
      return nullptr;
    }
    if (p) h->allocs.push_back({p, h->ufree, h->uctx});
  } else {
    if (cudaMalloc(&p, bytes) != cudaSuccess) p = nullptr;
    if (p) h->allocs.push_back({p, nullptr, nullptr});
  }
  return p;
}

// releases through the function recorded with the allocation (the hook may have
// been changed or removed since)
void dfree(nsf_mpm* h, void* p) {
  if (!p) return;
  for (size_t i = 0; i < h->allocs.size(); ++i) {
    if (h->allocs[i].p == p) {
      const nsf_mpm::Alloc a = h->allocs[i];
      h->allocs.erase(h->allocs.begin() + i);
      if (a.release) a.release(p, (void*)h->stream, a.ctx);
      else cudaFree(p);
      return;
    }
  }
}

// (re)allocates *dst; on any failure *dst is NULL (the old buffer is released first)
template <class T>
nsf_status alloc_into(nsf_mpm* h, T** dst, size_t bytes) {
  if (*dst) dfree(h, *dst);
  *dst = nullptr;
  bool misaligned = false;
  T* p = (T*)dalloc(h, bytes, &misaligned);
  if (misaligned)
    return fail(h, NSF_ERR_INVALID_ARGUMENT, "device allocator returned a pointer that is not 256-byte aligned");
  if (!p) return fail(h, NSF_ERR_OUT_OF_MEMORY, "device allocation of %zu bytes failed", bytes);
  *dst = p;
  return NSF_OK;
}

nsf_status ensure_staging(nsf_mpm* h, size_t bytes) {
  if (h->staging_bytes >= bytes) return NSF_OK;
  h->staging_bytes = 0;
  nsf_status s = alloc_into(h, (char**)&h->staging, bytes);
  if (s == NSF_OK) h->staging_bytes = bytes;
  return s;
}

// copy caller data (host or device) into device memory; returns device pointer
nsf_status to_device(nsf_mpm* h, const void* src, size_t bytes, int on_device, void* dst) {
  if (bytes == 0) return NSF_OK;
  CK(cudaMemcpyAsync(dst, src, bytes, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                     h->stream));
  return NSF_OK;
}

void invalidate_graph(nsf_mpm* h) {
  for (int k = 0; k < 2; ++k)
    for (int v = 0; v < nsf_mpm::kVariants; ++v) {
      if (h->graph[k][v]) cudaGraphExecDestroy(h->graph[k][v]);
      h->graph[k][v] = nullptr;
    }
}

nsf_status check_device_errors(nsf_mpm* h) {
  CK(cudaMemcpyAsync(h->err_host, h->err, sizeof(DevErr), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  const DevErr& e = *h->err_host;
  if (e.bits & ERR_OUT_OF_DOMAIN)
    return fail(h, NSF_ERR_OUT_OF_DOMAIN, "particle %d (load order) left the safe region x/dx in [0.5, N-1.5) "
                "by substep %lld", e.first_index, (long long)h->host_step);
  if (e.bits & ERR_NONFINITE)
    return fail(h, NSF_ERR_NONFINITE, "non-finite state at particle %d (load order) by substep %lld",
                e.first_index, (long long)h->host_step);
  return NSF_OK;
}

nsf_status reset_errors(nsf_mpm* h) {
  DevErr z{};
  z.first_index = 0x7fffffff;
  *h->err_host = z;
  CK(cudaMemcpyAsync(h->err, h->err_host, sizeof(DevErr), cudaMemcpyHostToDevice, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return NSF_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// Kernel launch bracketing for nsf_mpm_set_profiling.
namespace nsf {
void prof_begin(nsf_mpm* h, const char* name, cudaEvent_t* a) {
  if (!h->profiling) return;
  cudaEvent_t e;
  if (!h->free_events.empty()) { e = h->free_events.back(); h->free_events.pop_back(); }
  else cudaEventCreate(&e);
  cudaEventRecord(e, h->stream);
  *a = e;
  (void)name;
}
void prof_end(nsf_mpm* h, const char* name, cudaEvent_t a) {
  if (!h->profiling) return;
  cudaEvent_t e;
  if (!h->free_events.empty()) { e = h->free_events.back(); h->free_events.pop_back(); }
  else cudaEventCreate(&e);
  cudaEventRecord(e, h->stream);
  h->pending.push_back({name, a, e});
}
}  // namespace nsf

static void resolve_profiling(nsf_mpm* h) {
  if (h->pending.empty()) return;
  cudaStreamSynchronize(h->stream);
  for (auto& p : h->pending) {
    float ms = 0;
    cudaEventElapsedTime(&ms, p.a, p.b);
    auto& t = h->ktimes[p.name];
    t.first += ms;
    t.second += 1;
    h->free_events.push_back(p.a);
    h->free_events.push_back(p.b);
  }
  h->pending.clear();
}

// ---------------------------------------------------------------------------
extern "C" {

int32_t nsf_mpm_abi_version(void) { return NSF_MPM_ABI_VERSION; }

nsf_status nsf_mpm_create(const int32_t grid_res[3], double dx, double dt, const nsf_material* m,
                          nsf_mpm** out) {
  if (!out) return NSF_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  if (!grid_res || !m) return NSF_ERR_INVALID_ARGUMENT;
  if (!(dx > 0) || !(dt > 0) || !std::isfinite(dx) || !std::isfinite(dt)) return NSF_ERR_INVALID_ARGUMENT;
  if (!(m->E > 0) || !(m->nu >= 0 && m->nu < 0.5) || !(m->rho > 0)) return NSF_ERR_INVALID_ARGUMENT;
  if (m->model < 0 || m->model > 5) return NSF_ERR_INVALID_ARGUMENT;
  if (m->model == NSF_HERSCHEL_BULKLEY && !(m->viscosity >= 0 && std::isfinite(m->viscosity)))
    return NSF_ERR_INVALID_ARGUMENT;
  if (m->transfer != NSF_TRANSFER_APIC && m->transfer != NSF_TRANSFER_PIC && m->transfer != NSF_TRANSFER_RPIC)
    return NSF_ERR_INVALID_ARGUMENT;
  if (m->model == NSF_DRUCKER_PRAGER && !(m->friction_angle_deg > 0 && m->friction_angle_deg < 90))
    return NSF_ERR_INVALID_ARGUMENT;
  if (!(m->yield_stress >= 0)) return NSF_ERR_INVALID_ARGUMENT;
  if (!(m->hardening >= 0 && std::isfinite(m->hardening)) || !(m->softening >= 0 && std::isfinite(m->softening)))
    return NSF_ERR_INVALID_ARGUMENT;
  if (m->bc_width < 0) return NSF_ERR_INVALID_ARGUMENT;
  for (int f = 0; f < 6; ++f)
    if (m->bc[f] < 0 || m->bc[f] > 2) return NSF_ERR_INVALID_ARGUMENT;
  for (int a = 0; a < 3; ++a)
    if (grid_res[a] < 4 || grid_res[a] % 4 != 0 || grid_res[a] < 2 * m->bc_width + 3)
      return NSF_ERR_INVALID_ARGUMENT;
  if (m->force_mode < 0 || m->force_mode > 1) return NSF_ERR_INVALID_ARGUMENT;
  if (m->deterministic != 0 && m->deterministic != 1) return NSF_ERR_INVALID_ARGUMENT;
  if (m->n_scenes < 1) return NSF_ERR_INVALID_ARGUMENT;
  if (m->model == NSF_NEURAL_STRESS && !std::isfinite(m->stress_scale)) return NSF_ERR_INVALID_ARGUMENT;
  // the reduced G2P packs the previous stencil base in 10 bits per axis and uses
  // 32-bit node offsets within a scene (kernels_basic.cu k_g2p_nsf)
  if (m->model == NSF_NEURAL_STRESS &&
      (grid_res[0] > 1024 || grid_res[1] > 1024 || grid_res[2] > 1024 ||
       (int64_t)grid_res[0] * grid_res[1] * grid_res[2] >= (int64_t(1) << 31)))
    return NSF_ERR_INVALID_ARGUMENT;
  int device = 0;
  if (cudaGetDevice(&device) != cudaSuccess) return NSF_ERR_CUDA;

  nsf_mpm* h = new nsf_mpm();
  if (cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete h;
    return NSF_ERR_CUDA;
  }
  h->stream = h->own_stream;
  for (int a = 0; a < 3; ++a) h->grid_res[a] = grid_res[a];
  h->dx = dx;
  h->dt = dt;
  h->mat = *m;
  // material constants
  double mu = m->E / (2.0 * (1.0 + m->nu));
  double lam = m->E * m->nu / ((1.0 + m->nu) * (1.0 - 2.0 * m->nu));
  double s = std::sin(m->friction_angle_deg * M_PI / 180.0);
  double alpha = std::sqrt(2.0 / 3.0) * 2.0 * s / (3.0 - s);
  double V0 = m->particle_volume > 0 ? m->particle_volume : dx * dx * dx / 8.0;
  DevParams& P = h->P;
  for (int a = 0; a < 3; ++a) { P.N[a] = grid_res[a]; P.NB[a] = grid_res[a] / 4; }
  P.n_scenes = m->n_scenes;
  P.nodes_per_scene = (long long)grid_res[0] * grid_res[1] * grid_res[2];
  P.blocks_per_scene = (long long)P.NB[0] * P.NB[1] * P.NB[2];
  for (int a = 0; a < 3; ++a) {
    P.nb_shift[a] = -1;
    for (int k = 0; k < 31; ++k)
      if ((1 << k) == P.NB[a]) P.nb_shift[a] = k;
  }
  P.dx = (float)dx;
  P.inv_dx = (float)(1.0 / dx);
  P.dt = (float)dt;
  P.V0 = (float)V0;
  P.mass = (float)(m->rho * V0);
  P.mu = (float)mu;
  P.lam = (float)lam;
  P.alpha = (float)alpha;
  P.tau_Y = (float)m->yield_stress;
  for (int a = 0; a < 3; ++a) { P.g[a] = (float)m->gravity[a]; P.plate_v[a] = (float)m->plate_velocity[a]; }
  for (int f = 0; f < 6; ++f) P.bc[f] = m->bc[f];
  P.bc_width = m->bc_width;
  P.plate_enabled = m->plate_enabled;
  P.plate_y0 = (float)m->plate_y0;
  P.model = m->model;
  if (m->model == NSF_HENCKY) {   // Hencky without a return map = the von Mises code path that never yields
    P.model = NSF_VON_MISES;
    P.tau_Y = INFINITY;
  }
  P.mC = m->transfer == NSF_TRANSFER_PIC ? 0.0f : P.mass;
  P.rpic = m->transfer == NSF_TRANSFER_RPIC ? 1 : 0;
  P.kappa = (float)(m->E / (3.0 * (1.0 - 2.0 * m->nu)));
  P.hb_yield = (float)(std::sqrt(2.0 / 3.0) * m->yield_stress);
  P.hb_relax = (float)(1.0 / (1.0 + m->viscosity / (2.0 * mu * dt)));
  P.vm_hs = m->model == NSF_VON_MISES && (m->hardening > 0 || m->softening > 0);
  P.vm_hard_k = (float)(2.0 * mu * m->hardening);
  P.vm_soft = (float)m->softening;
  P.force_mode = m->force_mode;
  P.mls_coef = (float)(dt * V0 * 4.0 / (dx * dx));
  P.gradw_coef = (float)(dt * V0);
  P.stress_scale = (float)m->stress_scale;
  P.deterministic = m->deterministic;
  h->total_nodes = P.nodes_per_scene * m->n_scenes;
  h->total_blocks = P.blocks_per_scene * m->n_scenes;

  nsf_status st;
  if ((st = alloc_into(h, &h->err, sizeof(DevErr))) != NSF_OK ||
      (st = alloc_into(h, &h->d_step, sizeof(int64_t))) != NSF_OK ||
      (st = alloc_into(h, &h->acc, sizeof(float4) * h->total_nodes)) != NSF_OK ||
      (st = alloc_into(h, &h->vel, sizeof(float4) * h->total_nodes)) != NSF_OK) {
    nsf_mpm_destroy(h);
    return st;
  }
  if (cudaMallocHost(&h->err_host, sizeof(DevErr)) != cudaSuccess) { nsf_mpm_destroy(h); return NSF_ERR_CUDA; }
  if (cudaMemsetAsync(h->acc, 0, sizeof(float4) * h->total_nodes, h->stream) != cudaSuccess ||
      cudaMemsetAsync(h->vel, 0, sizeof(float4) * h->total_nodes, h->stream) != cudaSuccess ||
      cudaMemsetAsync(h->d_step, 0, sizeof(int64_t), h->stream) != cudaSuccess) {
    nsf_mpm_destroy(h);
    return NSF_ERR_CUDA;
  }
  if (pipeline_create(h, &h->pb, P, h->total_blocks) != 0) { nsf_mpm_destroy(h); return NSF_ERR_OUT_OF_MEMORY; }
  if (reset_errors(h) != NSF_OK) { nsf_mpm_destroy(h); return NSF_ERR_CUDA; }
  *out = h;
  return NSF_OK;
}

nsf_status nsf_mpm_set_stream(nsf_mpm* h, void* s) {
  if (!h) return NSF_ERR_INVALID_ARGUMENT;
  if (h->poisoned) return NSF_ERR_CUDA;
  cudaStream_t ns = s ? (cudaStream_t)s : h->own_stream;   // NULL -> the handle's own stream
  if (h->stream != ns) {
    cudaStreamSynchronize(h->stream);
    h->stream = ns;
    invalidate_graph(h);
  }
  return NSF_OK;
}

nsf_status nsf_mpm_set_allocator(nsf_mpm* h, void* (*alloc)(size_t, void*, void*),
                                 void (*release)(void*, void*, void*), void* ctx) {
  if (!h) return NSF_ERR_INVALID_ARGUMENT;
  if ((alloc == nullptr) != (release == nullptr)) return fail(h, NSF_ERR_INVALID_ARGUMENT, "alloc/release pair");
  h->ualloc = alloc;
  h->ufree = release;
  h->uctx = ctx;
  return NSF_OK;
}

nsf_status nsf_mpm_load_particles(nsf_mpm* h, int64_t n, const float* x, const float* v, const float* C,
                                  const float* F, const int64_t* scene_offsets, int32_t on_device) {
  if (!h) return NSF_ERR_INVALID_ARGUMENT;
  if (h->poisoned) return fail(h, NSF_ERR_CUDA, "handle poisoned by an earlier CUDA error");
  if (n < 0 || n >= (int64_t(1) << 31)) return fail(h, NSF_ERR_INVALID_ARGUMENT, "n out of range");
  if (n > 0 && (!x || !v)) return fail(h, NSF_ERR_INVALID_ARGUMENT, "x and v are required");
  int ns = h->mat.n_scenes;
  std::vector<int64_t> off(ns + 1);
  if (scene_offsets) {
    if (on_device) {
      CK(cudaMemcpyAsync(off.data(), scene_offsets, sizeof(int64_t) * (ns + 1), cudaMemcpyDeviceToHost, h->stream));
      CK(cudaStreamSynchronize(h->stream));
    } else {
      memcpy(off.data(), scene_offsets, sizeof(int64_t) * (ns + 1));
    }
    if (off[0] != 0 || off[ns] != n) return fail(h, NSF_ERR_INVALID_ARGUMENT, "scene_offsets must span [0, n]");
    for (int s = 0; s < ns; ++s)
      if (off[s + 1] < off[s]) return fail(h, NSF_ERR_INVALID_ARGUMENT, "scene_offsets not monotone");
  } else {
    if (ns != 1) return fail(h, NSF_ERR_INVALID_ARGUMENT, "scene_offsets required for n_scenes > 1");
    off[0] = 0;
    off[1] = n;
  }
  CK(cudaStreamSynchronize(h->stream));
  invalidate_graph(h);
  h->loaded = false;   // until every buffer below is in place: a failed load leaves no usable state
  bool with_F = h->mat.model != NSF_NEURAL_STRESS;
  int64_t pitch = ((n + 127) / 128) * 128;
  if (pitch == 0) pitch = 128;
  if (pitch != h->pitch || !h->S[0] || !h->S[1] || !h->ids[0] || !h->ids[1]) {
    nsf_status s;
    h->pitch = 0;
    for (int k = 0; k < 2; ++k) {
      if ((s = alloc_into(h, &h->S[k], sizeof(float) * kPlanes * pitch)) != NSF_OK) return s;
      if ((s = alloc_into(h, &h->ids[k], sizeof(int32_t) * pitch)) != NSF_OK) return s;
    }
    if ((s = pipeline_particles(h, &h->pb, pitch)) != NSF_OK) return s;
    h->pitch = pitch;
    if (h->X) { dfree(h, h->X); h->X = nullptr; }
  }
  nsf_status s;
  if ((s = alloc_into(h, &h->scene_off, sizeof(int64_t) * (ns + 1))) != NSF_OK) return s;
  CK(cudaMemcpyAsync(h->scene_off, off.data(), sizeof(int64_t) * (ns + 1), cudaMemcpyHostToDevice, h->stream));
  h->scene_off_host = off;
  h->n = n;
  h->cur = 0;
  // stage caller arrays (AoS) on the device
  size_t bx = sizeof(float) * 3 * n, bC = sizeof(float) * 9 * n;
  const float *dx_ = x, *dv_ = v, *dC_ = C, *dF_ = F;
  if (!on_device && n > 0) {
    if ((s = ensure_staging(h, 2 * bx + 2 * bC)) != NSF_OK) return s;
    char* st = (char*)h->staging;
    if ((s = to_device(h, x, bx, 0, st)) != NSF_OK) return s;
    if ((s = to_device(h, v, bx, 0, st + bx)) != NSF_OK) return s;
    dx_ = (const float*)st;
    dv_ = (const float*)(st + bx);
    if (C) { if ((s = to_device(h, C, bC, 0, st + 2 * bx)) != NSF_OK) return s; dC_ = (const float*)(st + 2 * bx); }
    if (F) { if ((s = to_device(h, F, bC, 0, st + 2 * bx + bC)) != NSF_OK) return s; dF_ = (const float*)(st + 2 * bx + bC); }
  }
  if ((s = reset_errors(h)) != NSF_OK) return s;
  launch_unpack(h->stream, n, dx_, dv_, dC_, dF_, h->S[0], pitch, h->ids[0], h->P, h->err, with_F ? 1 : 0);
  CK(cudaGetLastError());
  CK(cudaMemsetAsync(h->d_step, 0, sizeof(int64_t), h->stream));
  h->host_step = 0;
  CK(cudaMemcpyAsync(h->err_host, h->err, sizeof(DevErr), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  if (h->err_host->bits & (ERR_OUT_OF_DOMAIN | ERR_NONFINITE)) {
    const int idx = h->err_host->first_index;
    const bool nonfinite = h->err_host->bits & ERR_NONFINITE;
    reset_errors(h);
    h->loaded = false;
    if (nonfinite)
      return fail(h, NSF_ERR_NONFINITE, "particle %d (load order): non-finite x, v, C, F or tau(F)", idx);
    return fail(h, NSF_ERR_OUT_OF_DOMAIN, "particle %d (load order) is outside the safe region x/dx in [0.5, N-1.5)",
                idx);
  }
  if ((s = pipeline_on_load(h, &h->pb)) != NSF_OK) return s;
  h->loaded = true;
  return NSF_OK;
}

nsf_status nsf_mpm_load_stress_field(nsf_mpm* h, int32_t in_dim, int32_t width, int32_t n_hidden,
                                     int32_t out_dim, const uint16_t* W_bf16, const float* b,
                                     const float* X_ref, int32_t on_device) {
  if (!h) return NSF_ERR_INVALID_ARGUMENT;
  if (h->poisoned) return fail(h, NSF_ERR_CUDA, "handle poisoned");
  if (!(in_dim >= 4 && in_dim <= 16) || width != 128 || !(n_hidden >= 1 && n_hidden <= 8) || out_dim != 6)
    return fail(h, NSF_ERR_INVALID_ARGUMENT, "unsupported MLP shape (in<=16, width=128, 1<=hidden<=8, out=6)");
  if (!W_bf16 || !b) return fail(h, NSF_ERR_INVALID_ARGUMENT, "W and b are required");
  if (X_ref && !h->loaded) return fail(h, NSF_ERR_BAD_STATE, "load_particles before X_ref");
  CK(cudaStreamSynchronize(h->stream));
  invalidate_graph(h);
  h->mlp_loaded = false;   // until the new weights are in place
  MlpDev& M = h->mlp;
  M.in_dim = in_dim; M.width = width; M.n_hidden = n_hidden; M.out_dim = out_dim;
  int L = n_hidden + 1;
  int64_t wo = 0, bo = 0;
  for (int l = 0; l < L; ++l) {
    int in = l == 0 ? in_dim : width;
    int out = l == L - 1 ? out_dim : width;
    M.w_off[l] = wo; M.b_off[l] = bo;
    wo += (int64_t)in * out;
    bo += out;
  }
  M.w_off[L] = wo; M.b_off[L] = bo;
  nsf_status s;
  CK(cudaStreamSynchronize(h->stream));
  if ((s = alloc_into(h, &h->W, sizeof(uint16_t) * wo)) != NSF_OK) return s;
  if ((s = alloc_into(h, &h->b, sizeof(float) * bo)) != NSF_OK) return s;
  if ((s = to_device(h, W_bf16, sizeof(uint16_t) * wo, on_device, h->W)) != NSF_OK) return s;
  if ((s = to_device(h, b, sizeof(float) * bo, on_device, h->b)) != NSF_OK) return s;
  M.W = h->W;
  M.b = h->b;
  if (!h->mlp_ctr) {
    if ((s = alloc_into(h, &h->mlp_ctr, sizeof(unsigned int) * 4)) != NSF_OK) return s;
    CK(cudaMemsetAsync(h->mlp_ctr, 0, sizeof(unsigned int) * 4, h->stream));
  }
  M.ctr = h->mlp_ctr;
  if (X_ref) {
    int64_t n = h->n;
    if ((s = alloc_into(h, &h->X, sizeof(float) * 3 * h->pitch)) != NSF_OK) return s;
    // AoS n x 3 -> 3 planes via the pack/unpack helpers: stage then transpose on device
    if ((s = ensure_staging(h, sizeof(float) * 3 * n + 256)) != NSF_OK) return s;
    if ((s = to_device(h, X_ref, sizeof(float) * 3 * n, on_device, h->staging)) != NSF_OK) return s;
    pipeline_aos_to_planes(h->stream, n, (const float*)h->staging, 3, h->X, h->pitch);
    CK(cudaGetLastError());
  }
  CK(cudaStreamSynchronize(h->stream));
  h->mlp_loaded = true;
  pipeline_on_mlp(h, &h->pb);
  invalidate_graph(h);
  return NSF_OK;
}

nsf_status nsf_mpm_load_deformation_field(nsf_mpm* h, int32_t in_dim, int32_t width, int32_t n_hidden,
                                          int32_t out_dim, const uint16_t* W_bf16, const float* b,
                                          int32_t on_device) {
  if (!h) return NSF_ERR_INVALID_ARGUMENT;
  if (h->poisoned) return fail(h, NSF_ERR_CUDA, "handle poisoned");
  if (!(in_dim >= 4 && in_dim <= 16) || width != 128 || !(n_hidden >= 1 && n_hidden <= 4) || out_dim != 3)
    return fail(h, NSF_ERR_INVALID_ARGUMENT, "unsupported deformation field (in<=16, width=128, 1<=hidden<=4, out=3)");
  if (!W_bf16 || !b) return fail(h, NSF_ERR_INVALID_ARGUMENT, "W and b are required");
  if (!h->loaded) return fail(h, NSF_ERR_BAD_STATE, "load_particles first");
  h->gdef_loaded = false;   // until the new weights are in place
  MlpDev& M = h->gdef;
  M.in_dim = in_dim; M.width = width; M.n_hidden = n_hidden; M.out_dim = out_dim;
  const int L = n_hidden + 1;
  int64_t wo = 0, bo = 0;
  for (int l = 0; l < L; ++l) {
    const int in = l == 0 ? in_dim : width;
    const int out = l == L - 1 ? out_dim : width;
    M.w_off[l] = wo; M.b_off[l] = bo;
    wo += (int64_t)in * out;
    bo += out;
  }
  M.w_off[L] = wo; M.b_off[L] = bo;
  M.ctr = nullptr;
  if (gn_smem_bytes(M) > 227 * 1024) return fail(h, NSF_ERR_INVALID_ARGUMENT, "deformation field too large");
  nsf_status s;
  CK(cudaStreamSynchronize(h->stream));
  if ((s = alloc_into(h, &h->gW, sizeof(uint16_t) * wo)) != NSF_OK) return s;
  if ((s = alloc_into(h, &h->gb, sizeof(float) * bo)) != NSF_OK) return s;
  if ((s = to_device(h, W_bf16, sizeof(uint16_t) * wo, on_device, h->gW)) != NSF_OK) return s;
  if ((s = to_device(h, b, sizeof(float) * bo, on_device, h->gb)) != NSF_OK) return s;
  CK(cudaStreamSynchronize(h->stream));
  M.W = h->gW;
  M.b = h->gb;
  h->gdef_loaded = true;
  return NSF_OK;
}

nsf_status nsf_mpm_load_affine_field(nsf_mpm* h, int32_t in_dim, int32_t width, int32_t n_hidden,
                                     int32_t out_dim, const uint16_t* W_bf16, const float* b, int32_t on_device) {
  if (!h) return NSF_ERR_INVALID_ARGUMENT;
  if (h->poisoned) return fail(h, NSF_ERR_CUDA, "handle poisoned");
  if (!(in_dim >= 4 && in_dim <= 16) || width != 128 || !(n_hidden >= 1 && n_hidden <= 8) || out_dim != 9)
    return fail(h, NSF_ERR_INVALID_ARGUMENT, "unsupported affine field (in<=16, width=128, 1<=hidden<=8, out=9)");
  if (!W_bf16 || !b) return fail(h, NSF_ERR_INVALID_ARGUMENT, "W and b are required");
  h->ldef_loaded = false;   // until the new weights are in place
  MlpDev& M = h->ldef;
  M.in_dim = in_dim; M.width = width; M.n_hidden = n_hidden; M.out_dim = out_dim;
  const int L = n_hidden + 1;
  int64_t wo = 0, bo = 0;
  for (int l = 0; l < L; ++l) {
    const int in = l == 0 ? in_dim : width;
    const int out = l == L - 1 ? out_dim : width;
    M.w_off[l] = wo; M.b_off[l] = bo;
    wo += (int64_t)in * out;
    bo += out;
  }
  M.w_off[L] = wo; M.b_off[L] = bo;
  M.ctr = nullptr;
  nsf_status s;
  CK(cudaStreamSynchronize(h->stream));
  if ((s = alloc_into(h, &h->lW, sizeof(uint16_t) * wo)) != NSF_OK) return s;
  if ((s = alloc_into(h, &h->lb, sizeof(float) * bo)) != NSF_OK) return s;
  if ((s = to_device(h, W_bf16, sizeof(uint16_t) * wo, on_device, h->lW)) != NSF_OK) return s;
  if ((s = to_device(h, b, sizeof(float) * bo, on_device, h->lb)) != NSF_OK) return s;
  CK(cudaStreamSynchronize(h->stream));
  M.W = h->lW;
  M.b = h->lb;
  h->ldef_loaded = true;
  return NSF_OK;
}

static nsf_status inference_ready(nsf_mpm* h) {
  if (h->mat.model != NSF_NEURAL_STRESS || !h->loaded || !h->mlp_loaded || !h->latents_loaded || !h->X ||
      !h->gdef_loaded || !h->ldef_loaded)
    return fail(h, NSF_ERR_BAD_STATE,
                "needs the NSF model with load_stress_field(X_ref), set_latents, load_deformation_field, "
                "load_affine_field");
  if (h->gdef.in_dim != 3 + h->r || h->ldef.in_dim != 3 + h->r)
    return fail(h, NSF_ERR_INVALID_ARGUMENT, "g and l inputs must be 3 + r");
  return NSF_OK;
}

// x = g(X, z_n), v = (x - g(X, z_prev)) / dt, C = l(X, z_n) on the store
static nsf_status enqueue_infer(nsf_mpm* h) {
  if (h->n == 0) return NSF_OK;
  float* S = h->S[h->cur];
  const float* Xp = S + PXR * 32;   // the store's reference-position planes (follow the points)
  const int ns = h->mat.n_scenes, r = h->r;
  launch_nsf_mlp(h->stream, h->n, Xp, -1, h->scene_off, ns, h->zprev, nullptr, r, nullptr, h->gdef, 1.0f,
                 S + PV * 32, 0, 0);
  launch_nsf_mlp(h->stream, h->n, Xp, -1, h->scene_off, ns, h->z, h->dz, r, h->d_step, h->gdef, 1.0f, S + PX * 32,
                 0, 0);
  launch_backdiff(h->stream, h->n, S, (float)h->dt);
  launch_nsf_mlp(h->stream, h->n, Xp, -1, h->scene_off, ns, h->z, h->dz, r, h->d_step, h->ldef, 1.0f, S + PC * 32,
                 0, 0);
  CK(cudaGetLastError());
  return NSF_OK;
}

static nsf_status set_zprev(nsf_mpm* h, const float* z_prev, int32_t on_device) {
  const size_t m = (size_t)h->mat.n_scenes * h->r;
  nsf_status s;
  if ((s = alloc_into(h, &h->zprev, sizeof(float) * m)) != NSF_OK) return s;
  if (z_prev) return to_device(h, z_prev, sizeof(float) * m, on_device, h->zprev);
  launch_latent_at(h->stream, (int64_t)m, h->z, h->dz, h->host_step >= 1 ? h->host_step - 1 : 0, h->zprev);
  CK(cudaGetLastError());
  return NSF_OK;
}

nsf_status nsf_mpm_infer_state(nsf_mpm* h, const float* z_prev, int32_t on_device) {
  if (!h) return NSF_ERR_INVALID_ARGUMENT;
  if (h->poisoned) return fail(h, NSF_ERR_CUDA, "handle poisoned");
  nsf_status s;
  if ((s = inference_ready(h)) != NSF_OK) return s;
  if ((s = set_zprev(h, z_prev, on_device)) != NSF_OK) return s;
  return enqueue_infer(h);
}

static nsf_status build_set_impl(nsf_mpm* h, int64_t n_ref, const float* X_all, int32_t n_sample,
                                 const int32_t* sample_idx, const float* z_prev, int32_t zprev_on_device,
                                 int64_t* counts_out, int32_t on_device);

nsf_status nsf_mpm_build_integration_set(nsf_mpm* h, int64_t n_ref, const float* X_all, int32_t n_sample,
                                         const int32_t* sample_idx, const float* z_prev, int64_t* counts_out,
                                         int32_t on_device) {
  return build_set_impl(h, n_ref, X_all, n_sample, sample_idx, z_prev, on_device, counts_out, on_device);
}

static nsf_status build_set_impl(nsf_mpm* h, int64_t n_ref, const float* X_all, int32_t n_sample,
                                 const int32_t* sample_idx, const float* z_prev, int32_t zprev_on_device,
                                 int64_t* counts_out, int32_t on_device) {
  if (!h) return NSF_ERR_INVALID_ARGUMENT;
  if (h->poisoned) return fail(h, NSF_ERR_CUDA, "handle poisoned");
  nsf_status s;
  if ((s = inference_ready(h)) != NSF_OK) return s;
  const int ns = h->mat.n_scenes, r = h->r;
  if (n_ref < 1 || n_ref >= (int64_t(1) << 31) / (ns > 0 ? ns : 1) || !X_all || n_sample < 1 || n_sample > n_ref ||
      !sample_idx)
    return fail(h, NSF_ERR_INVALID_ARGUMENT, "1 <= n_sample <= n_ref, n_ref * n_scenes < 2^31, X_all and sample_idx");
  // sample indices: in range and distinct within a scene (checked on the host)
  std::vector<int32_t> sidx((size_t)ns * n_sample);
  if (on_device) {
    CK(cudaMemcpyAsync(sidx.data(), sample_idx, sizeof(int32_t) * sidx.size(), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
  }
  else memcpy(sidx.data(), sample_idx, sizeof(int32_t) * sidx.size());
  {
    std::vector<int32_t> seen((size_t)n_ref, -1);
    for (int sc = 0; sc < ns; ++sc)
      for (int q = 0; q < n_sample; ++q) {
        const int32_t i = sidx[(size_t)sc * n_sample + q];
        if (i < 0 || i >= n_ref || seen[i] == sc)
          return fail(h, NSF_ERR_INVALID_ARGUMENT, "sample_idx[%d][%d] out of range or repeated", sc, q);
        seen[i] = sc;
      }
  }
  CK(cudaStreamSynchronize(h->stream));
  const int64_t pitch_ref = ((n_ref + 127) / 128) * 128;
  const int64_t nodes = (int64_t)h->grid_res[0] * h->grid_res[1] * h->grid_res[2];
  const int64_t nblk = compact_blocks(n_ref);
  float *Xd = nullptr, *Xpl = nullptr, *xg = nullptr, *zc = nullptr, *Xnew = nullptr, *vzero = nullptr;
  int32_t *sid = nullptr, *cnt = nullptr, *base = nullptr, *list = nullptr;
  uint32_t* mask = nullptr;
  uint8_t *is_s = nullptr, *flag = nullptr;
  int64_t* offd = nullptr;
  int64_t* ctr = nullptr;   // [0] cursor, [1] sample base, [2..] per-scene counts
  auto cleanup = [&]() {
    for (void* p : {(void*)Xd, (void*)Xpl, (void*)xg, (void*)zc, (void*)Xnew, (void*)vzero, (void*)sid, (void*)cnt,
                    (void*)base, (void*)list, (void*)mask, (void*)is_s, (void*)flag, (void*)offd, (void*)ctr})
      dfree(h, p);
  };
#define TRY(expr) do { if ((s = (expr)) != NSF_OK) { cleanup(); return s; } } while (0)
#define TRYCU(expr) do { cudaError_t e_ = (expr); if (e_ != cudaSuccess) { cleanup(); return cuda_fail(h, e_, #expr); } } while (0)
  TRY(alloc_into(h, &Xd, sizeof(float) * 3 * n_ref));
  TRY(alloc_into(h, &Xpl, sizeof(float) * 3 * pitch_ref));
  TRY(alloc_into(h, &xg, sizeof(float) * 3 * n_ref));
  TRY(alloc_into(h, &zc, sizeof(float) * ns * r));
  TRY(alloc_into(h, &sid, sizeof(int32_t) * sidx.size()));
  TRY(alloc_into(h, &cnt, sizeof(int32_t) * nblk));
  TRY(alloc_into(h, &base, sizeof(int32_t) * nblk));
  TRY(alloc_into(h, &list, sizeof(int32_t) * (size_t)ns * n_ref));
  TRY(alloc_into(h, &mask, sizeof(uint32_t) * ((nodes + 31) / 32)));
  TRY(alloc_into(h, &is_s, (size_t)n_ref));
  TRY(alloc_into(h, &flag, (size_t)n_ref));
  TRY(alloc_into(h, &ctr, sizeof(int64_t) * (2 + ns)));
  TRY(to_device(h, X_all, sizeof(float) * 3 * n_ref, on_device, Xd));
  TRYCU(cudaMemcpyAsync(sid, sidx.data(), sizeof(int32_t) * sidx.size(), cudaMemcpyHostToDevice, h->stream));
  pipeline_aos_to_planes(h->stream, n_ref, Xd, 3, Xpl, pitch_ref);
  launch_latent_at(h->stream, (int64_t)ns * r, h->z, h->dz, h->host_step, zc);   // z_n of the next substep
  TRYCU(cudaMemsetAsync(is_s, 0, (size_t)n_ref, h->stream));
  TRY(reset_errors(h));
  std::vector<int64_t> off(ns + 1, 0), counts(ns);
  TRYCU(cudaMemsetAsync(ctr, 0, sizeof(int64_t) * (2 + ns), h->stream));
  // all scenes enqueued back to back; offsets are carried on the device (k_scene_scan)
  for (int sc = 0; sc < ns; ++sc) {
    const int32_t* si = sid + (size_t)sc * n_sample;
    // x = g(X_p, z_n(s)) for the whole reference body
    launch_nsf_mlp(h->stream, n_ref, Xpl, pitch_ref, nullptr, 1, zc + (size_t)sc * r, nullptr, r, nullptr, h->gdef,
                   1.0f, xg, 0, 1);
    TRYCU(cudaMemsetAsync(mask, 0, sizeof(uint32_t) * ((nodes + 31) / 32), h->stream));
    launch_mark_stencils(h->stream, n_sample, si, xg, mask, h->P, h->err);
    launch_set_samples(h->stream, n_sample, si, is_s, 1);
    launch_member_flags(h->stream, n_ref, xg, mask, is_s, flag, h->P);
    launch_set_samples(h->stream, n_sample, si, is_s, 0);
    launch_count_blocks(h->stream, n_ref, flag, cnt);
    launch_scene_scan(h->stream, nblk, cnt, n_sample, ctr, base, ctr + 2, sc, ctr + 1);
    launch_put_samples(h->stream, n_sample, si, ctr + 1, list);
    launch_compact(h->stream, n_ref, flag, base, list);
    TRYCU(cudaGetLastError());
  }
  TRYCU(cudaMemcpyAsync(counts.data(), ctr + 2, sizeof(int64_t) * ns, cudaMemcpyDeviceToHost, h->stream));
  TRYCU(cudaStreamSynchronize(h->stream));
  for (int sc = 0; sc < ns; ++sc) off[sc + 1] = off[sc] + counts[sc];
  TRYCU(cudaMemcpyAsync(h->err_host, h->err, sizeof(DevErr), cudaMemcpyDeviceToHost, h->stream));
  TRYCU(cudaStreamSynchronize(h->stream));
  if (h->err_host->bits & ERR_OUT_OF_DOMAIN) {
    reset_errors(h);
    cleanup();
    return fail(h, NSF_ERR_OUT_OF_DOMAIN, "a sample particle's stencil leaves the grid");
  }
  const int64_t n_new = off[ns];
  if (n_new >= (int64_t(1) << 31)) { cleanup(); return fail(h, NSF_ERR_INVALID_ARGUMENT, "integration set too large"); }
  TRY(alloc_into(h, &Xnew, sizeof(float) * 3 * n_new));
  TRY(alloc_into(h, &vzero, sizeof(float) * 3 * n_new));
  TRY(alloc_into(h, &offd, sizeof(int64_t) * (ns + 1)));
  launch_gather_rows3(h->stream, n_new, list, Xd, Xnew);
  TRYCU(cudaMemsetAsync(vzero, 0, sizeof(float) * 3 * n_new, h->stream));
  TRYCU(cudaMemcpyAsync(offd, off.data(), sizeof(int64_t) * (ns + 1), cudaMemcpyHostToDevice, h->stream));
  TRYCU(cudaStreamSynchronize(h->stream));
  // reload the points (placeholders x = X, v = 0), keeping the step counter (z_n = z + n dz)
  const int64_t step = h->host_step;
  TRY(nsf_mpm_load_particles(h, n_new, Xnew, vzero, nullptr, nullptr, offd, 1));
  h->host_step = step;
  TRYCU(cudaMemcpyAsync(h->d_step, &h->host_step, sizeof(int64_t), cudaMemcpyHostToDevice, h->stream));
  TRY(alloc_into(h, &h->X, sizeof(float) * 3 * h->pitch));
  pipeline_aos_to_planes(h->stream, n_new, Xnew, 3, h->X, h->pitch);
  pipeline_on_mlp(h, &h->pb);
  invalidate_graph(h);
  TRY(set_zprev(h, z_prev, zprev_on_device));
  TRY(enqueue_infer(h));
  TRYCU(cudaStreamSynchronize(h->stream));
  if (counts_out) memcpy(counts_out, counts.data(), sizeof(int64_t) * ns);
  cleanup();
#undef TRY
#undef TRYCU
  return NSF_OK;
}

nsf_status nsf_mpm_invert_latents(nsf_mpm* h, int32_t n_sample, int32_t n_iters, float* z_out, int32_t on_device) {
  if (!h) return NSF_ERR_INVALID_ARGUMENT;
  if (h->poisoned) return fail(h, NSF_ERR_CUDA, "handle poisoned");
  if (n_sample < 1 || n_iters < 1 || n_iters > 16) return fail(h, NSF_ERR_INVALID_ARGUMENT, "1 <= n_sample, 1 <= n_iters <= 16");
  if (h->mat.model != NSF_NEURAL_STRESS || !h->loaded || !h->mlp_loaded || !h->latents_loaded || !h->X ||
      !h->gdef_loaded)
    return fail(h, NSF_ERR_BAD_STATE, "needs the NSF model with load_stress_field, set_latents, load_deformation_field");
  if (h->gdef.in_dim != 3 + h->r) return fail(h, NSF_ERR_INVALID_ARGUMENT, "deformation field input must be 3 + r");
  const int ns = h->mat.n_scenes, r = h->r;
  const int nterm = r * (r + 1) / 2 + r;
  nsf_status s;
  const size_t need[3] = {sizeof(int32_t) * (size_t)ns * n_sample, sizeof(float) * (size_t)ns * r,
                          sizeof(double) * (size_t)ns * nterm};
  if (need[0] > h->inv_cap[0]) { if ((s = alloc_into(h, &h->inv_slots, need[0])) != NSF_OK) return s; h->inv_cap[0] = need[0]; }
  if (need[1] > h->inv_cap[1]) { if ((s = alloc_into(h, &h->inv_z, need[1])) != NSF_OK) return s; h->inv_cap[1] = need[1]; }
  if (need[2] > h->inv_cap[2]) { if ((s = alloc_into(h, &h->inv_acc, need[2])) != NSF_OK) return s; h->inv_cap[2] = need[2]; }
  launch_gn_invert(h->stream, h->n, h->ids[h->cur], h->scene_off, ns, n_sample, r, h->S[h->cur], h->z, h->dz,
                   h->d_step, h->gdef, n_iters, h->inv_slots, h->inv_z, h->inv_acc);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(h->z, h->inv_z, sizeof(float) * (size_t)ns * r, cudaMemcpyDeviceToDevice, h->stream));
  CK(cudaMemsetAsync(h->dz, 0, sizeof(float) * (size_t)ns * r, h->stream));
  if (z_out)
    CK(cudaMemcpyAsync(z_out, h->inv_z, sizeof(float) * (size_t)ns * r,
                       on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return NSF_OK;
}

// One latent-space time step of the reduced model (§5):
// (1) sample / integration particles and network inference at z_n (lines 251-254,
// 265-269), (2) one MPM substep on N (lines 255-256), (3) network inversion of
// Eq. (10) on S (lines 257-263): z_{n+1} becomes the handle's latent (dz = 0).  The
// previous call's z_n is kept on the device and serves as this call's z_{n-1}
// unless the caller passes z_prev.
nsf_status nsf_mpm_rom_step(nsf_mpm* h, int64_t n_ref, const float* X_all, int32_t n_sample,
                            const int32_t* sample_idx, const float* z_prev, int32_t gn_iters, float* z_out,
                            int64_t* counts_out, int32_t on_device) {
  if (!h) return NSF_ERR_INVALID_ARGUMENT;
  if (h->poisoned) return fail(h, NSF_ERR_CUDA, "handle poisoned");
  if (gn_iters < 1 || gn_iters > 16) return fail(h, NSF_ERR_INVALID_ARGUMENT, "1 <= gn_iters <= 16");
  nsf_status s;
  if ((s = inference_ready(h)) != NSF_OK) return s;
  const size_t zb = sizeof(float) * (size_t)h->mat.n_scenes * h->r;
  const float* zp = z_prev ? z_prev : (h->zrom_valid ? h->zrom : nullptr);
  if ((s = build_set_impl(h, n_ref, X_all, n_sample, sample_idx, zp, z_prev ? on_device : 1, counts_out,
                          on_device)) != NSF_OK)
    return s;
  if ((s = nsf_mpm_substep(h, 1)) != NSF_OK) return s;
  // z_n (the latent of this substep: z + n dz at n = step - 1) is the next call's z_{n-1}
  if (!h->zrom) {
    if ((s = alloc_into(h, &h->zrom, zb)) != NSF_OK) return s;
  }
  launch_latent_at(h->stream, (int64_t)h->mat.n_scenes * h->r, h->z, h->dz, h->host_step - 1, h->zrom);
  CK(cudaGetLastError());
  if ((s = nsf_mpm_invert_latents(h, n_sample, gn_iters, z_out, on_device)) != NSF_OK) return s;
  h->zrom_valid = true;
  return NSF_OK;
}

nsf_status nsf_mpm_set_latents(nsf_mpm* h, int32_t r, const float* z, const float* dz, int32_t on_device) {
  if (!h) return NSF_ERR_INVALID_ARGUMENT;
  if (h->poisoned) return fail(h, NSF_ERR_CUDA, "handle poisoned");
  if (r < 1 || r > 13 || !z) return fail(h, NSF_ERR_INVALID_ARGUMENT, "1 <= r <= 13 and z required");
  if (h->mlp_loaded && r + 3 != h->mlp.in_dim)
    return fail(h, NSF_ERR_INVALID_ARGUMENT, "r + 3 must equal the MLP input dimension");
  int ns = h->mat.n_scenes;
  nsf_status s;
  CK(cudaStreamSynchronize(h->stream));
  invalidate_graph(h);
  h->latents_loaded = false;   // until the new latents are in place
  if ((s = alloc_into(h, &h->z, sizeof(float) * ns * r)) != NSF_OK) return s;
  if ((s = alloc_into(h, &h->dz, sizeof(float) * ns * r)) != NSF_OK) return s;
  if ((s = to_device(h, z, sizeof(float) * ns * r, on_device, h->z)) != NSF_OK) return s;
  if (dz) { if ((s = to_device(h, dz, sizeof(float) * ns * r, on_device, h->dz)) != NSF_OK) return s; }
  else CK(cudaMemsetAsync(h->dz, 0, sizeof(float) * ns * r, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  h->r = r;
  h->latents_loaded = true;
  h->zrom_valid = false;
  invalidate_graph(h);
  return NSF_OK;
}

// NSF_WRITE_EVERY=1: every substep stores v, C, tau (A/B; read per call, so a test runs both)
static bool write_last_only() {
  const char* e = getenv("NSF_WRITE_EVERY");
  return !(e && e[0] == '1');
}

static nsf_status enqueue_substeps(nsf_mpm* h, int32_t n) {
  static const bool graph_env = [] { const char* e = getenv("NSF_GRAPH"); return !(e && e[0] == '0'); }();   // A/B
  const bool use_graph = graph_env && !h->profiling && pipeline_graphable(h, &h->pb);
  for (int i = 0; i < n; ++i) {
    // bit 2: a fused substep that is not the call's last does not store v, C, tau
    const int variant = pipeline_variant(h, &h->pb) | ((i + 1 < n && pipeline_fused(&h->pb) && write_last_only()) ? 4 : 0);
    if (variant < 0 || variant >= nsf_mpm::kVariants) return fail(h, NSF_ERR_CUDA, "substep variant out of range");
    if (!use_graph) {
      int next = pipeline_substep(h, &h->pb, h->cur, variant);
      if (next < 0) {
        h->poisoned = true;   // (earlier substeps of this call may not have stored v, C, tau)
        return fail(h, NSF_ERR_CUDA, "substep launch failed");
      }
      CK(cudaGetLastError());
      h->cur = next;
      pipeline_advance(h, &h->pb, variant, pipeline_launches_per_substep(h, &h->pb));
      continue;
    }
    const int c = h->cur;
    // a fused substep's graph is captured together with its sibling (stores v, C, tau /
    // does not), so a long call also prepares the graphs of the single-substep calls
    // that may follow it (and the reverse): no capture lands in a later timed region
    for (int sib = 0; sib < (pipeline_fused(&h->pb) ? 2 : 1); ++sib) {
      const int var = sib ? (variant ^ 4) : variant;
      if (h->graph[c][var]) continue;
      cudaGraph_t g;
      CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
      int next = pipeline_substep(h, &h->pb, c, var);
      cudaError_t ec = cudaStreamEndCapture(h->stream, &g);
      if (next < 0 || ec != cudaSuccess)
        return cuda_fail(h, ec == cudaSuccess ? cudaErrorUnknown : ec, "graph capture");
      CK(cudaGraphInstantiate(&h->graph[c][var], g, 0));
      cudaGraphDestroy(g);
      h->graph_next[c][var] = next;
      h->graph_launches[c][var] = pipeline_launches_per_substep(h, &h->pb);
    }
    CK(cudaGraphLaunch(h->graph[c][variant], h->stream));
    h->cur = h->graph_next[c][variant];
    pipeline_advance(h, &h->pb, variant, h->graph_launches[c][variant]);
  }
  return NSF_OK;
}

nsf_status nsf_mpm_substep(nsf_mpm* h, int32_t n) {
  if (!h) return NSF_ERR_INVALID_ARGUMENT;
  if (h->poisoned) return fail(h, NSF_ERR_CUDA, "handle poisoned");
  if (n < 0) return fail(h, NSF_ERR_INVALID_ARGUMENT, "n < 0");
  if (!h->loaded) return fail(h, NSF_ERR_BAD_STATE, "substep before load_particles");
  if (h->mat.model == NSF_NEURAL_STRESS && (!h->mlp_loaded || !h->latents_loaded || !h->X))
    return fail(h, NSF_ERR_BAD_STATE, "NSF model needs load_stress_field (with X_ref) and set_latents");
  if (n == 0) return NSF_OK;
  nsf_status s = enqueue_substeps(h, n);
  if (s == NSF_OK) h->host_step += n;
  return s;
}

nsf_status nsf_mpm_eval_stress_field(nsf_mpm* h, const float* z, int64_t m, const float* points,
                                     float* tau_out, int32_t on_device) {
  if (!h) return NSF_ERR_INVALID_ARGUMENT;
  if (h->poisoned) return fail(h, NSF_ERR_CUDA, "handle poisoned");
  if (!h->mlp_loaded) return fail(h, NSF_ERR_BAD_STATE, "load_stress_field first");
  if (m < 0 || (m > 0 && (!z || !points || !tau_out))) return fail(h, NSF_ERR_INVALID_ARGUMENT, "bad arguments");
  if (m == 0) return NSF_OK;
  int r = h->mlp.in_dim - 3;
  size_t bp = sizeof(float) * 3 * m, bt = sizeof(float) * 6 * m, bz = sizeof(float) * 16;
  size_t pplanes = sizeof(float) * 3 * m;
  nsf_status s;
  if ((s = ensure_staging(h, bp + bt + bz + pplanes + 1024)) != NSF_OK) return s;
  char* st = (char*)h->staging;
  float* dpts = (float*)st;
  float* dtau = (float*)(st + ((bp + 255) & ~size_t(255)));
  float* dz_ = (float*)((char*)dtau + ((bt + 255) & ~size_t(255)));
  float* dplanes = (float*)((char*)dz_ + 256);
  if ((s = to_device(h, points, bp, on_device, dpts)) != NSF_OK) return s;
  if ((s = to_device(h, z, sizeof(float) * r, on_device, dz_)) != NSF_OK) return s;
  pipeline_aos_to_planes(h->stream, m, dpts, 3, dplanes, m);
  pipeline_eval_mlp(h, &h->pb, m, dplanes, m, dz_, r, dtau);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(tau_out, dtau, bt, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return NSF_OK;
}

nsf_status nsf_mpm_read_state(nsf_mpm* h, uint32_t mask, float* const* dst, int32_t on_device) {
  if (!h) return NSF_ERR_INVALID_ARGUMENT;
  if (h->poisoned) return fail(h, NSF_ERR_CUDA, "handle poisoned");
  if (!h->loaded) return fail(h, NSF_ERR_BAD_STATE, "nothing loaded");
  if (mask == 0 || (mask & ~63u)) return fail(h, NSF_ERR_INVALID_ARGUMENT, "bad field mask");
  if (!dst) return fail(h, NSF_ERR_INVALID_ARGUMENT, "dst required");
  if ((mask & NSF_FIELD_F) && h->mat.model == NSF_NEURAL_STRESS)
    return fail(h, NSF_ERR_INVALID_ARGUMENT, "F is not tracked by the reduced (NSF) variant");
  nsf_status err_status = check_device_errors(h);
  if (h->poisoned) return err_status;
  const int planes[6] = {PX, PV, PC, PF, PT, PTY};
  const int comps[6] = {3, 3, 9, 9, 6, 1};
  int k = 0;
  int64_t n = h->n;
  for (int f = 0; f < 6; ++f) {
    if (!(mask & (1u << f))) continue;
    float* out = dst[k++];
    if (!out) return fail(h, NSF_ERR_INVALID_ARGUMENT, "dst[%d] is NULL", k - 1);
    if (n == 0) continue;
    size_t bytes = sizeof(float) * comps[f] * n;
    float* dout = out;
    nsf_status s;
    if (!on_device) {
      if ((s = ensure_staging(h, bytes)) != NSF_OK) return s;
      dout = (float*)h->staging;
    }
    launch_pack(h->stream, n, h->S[h->cur], h->pitch, h->ids[h->cur], planes[f], comps[f], dout);
    CK(cudaGetLastError());
    if (!on_device) CK(cudaMemcpyAsync(out, dout, bytes, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
  }
  return err_status;
}

nsf_status nsf_mpm_sync(nsf_mpm* h) {
  if (!h) return NSF_ERR_INVALID_ARGUMENT;
  if (h->poisoned) return fail(h, NSF_ERR_CUDA, "handle poisoned");
  CK(cudaStreamSynchronize(h->stream));
  resolve_profiling(h);
  return check_device_errors(h);
}

int64_t nsf_mpm_step_count(const nsf_mpm* h) { return h ? h->host_step : -1; }

int64_t nsf_mpm_inverted_count(nsf_mpm* h) {
  if (!h || h->poisoned) return -1;
  if (cudaMemcpyAsync(h->err_host, h->err, sizeof(DevErr), cudaMemcpyDeviceToHost, h->stream) != cudaSuccess ||
      cudaStreamSynchronize(h->stream) != cudaSuccess)
    return -1;
  return (int64_t)h->err_host->inverted;
}

const char* nsf_mpm_last_error(const nsf_mpm* h) { return h ? h->last_error.c_str() : "null handle"; }

void nsf_mpm_destroy(nsf_mpm* h) {
  if (!h) return;
  cudaStreamSynchronize(h->stream);
  invalidate_graph(h);
  for (auto& p : h->pending) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
  for (auto e : h->free_events) cudaEventDestroy(e);
  pipeline_destroy(h, &h->pb);
  while (!h->allocs.empty()) dfree(h, h->allocs.back().p);
  if (h->err_host) cudaFreeHost(h->err_host);
  if (h->own_stream) cudaStreamDestroy(h->own_stream);
  delete h;
}

nsf_status nsf_mpm_debug_bins(nsf_mpm* h, int32_t* counts, int32_t* perm, int32_t on_device) {
  if (!h) return NSF_ERR_INVALID_ARGUMENT;
  if (h->poisoned) return fail(h, NSF_ERR_CUDA, "handle poisoned");
  if (!h->loaded) return fail(h, NSF_ERR_BAD_STATE, "nothing loaded");
  int rc = pipeline_debug_bins(h, &h->pb, h->cur, counts, perm, on_device);
  if (rc != 0) return fail(h, NSF_ERR_CUDA, "debug_bins failed");
  CK(cudaStreamSynchronize(h->stream));
  return NSF_OK;
}

nsf_status nsf_mpm_debug_grid(nsf_mpm* h, int32_t stage, float* out, int32_t on_device) {
  if (!h) return NSF_ERR_INVALID_ARGUMENT;
  if (h->poisoned) return fail(h, NSF_ERR_CUDA, "handle poisoned");
  if (!h->loaded) return fail(h, NSF_ERR_BAD_STATE, "nothing loaded");
  if (stage < 0 || stage > 1 || !out) return fail(h, NSF_ERR_INVALID_ARGUMENT, "stage 0 or 1, out required");
  if (h->mat.model == NSF_NEURAL_STRESS && (!h->mlp_loaded || !h->latents_loaded || !h->X))
    return fail(h, NSF_ERR_BAD_STATE, "NSF model needs load_stress_field and set_latents");
  size_t bytes = sizeof(float) * 4 * h->total_nodes;
  float* dout = out;
  nsf_status s;
  if (!on_device) {
    if ((s = ensure_staging(h, bytes)) != NSF_OK) return s;
    dout = (float*)h->staging;
  }
  int rc = pipeline_debug_grid(h, &h->pb, h->cur, stage, dout);
  if (rc != 0) return fail(h, NSF_ERR_CUDA, "debug_grid failed");
  CK(cudaGetLastError());
  if (!on_device) CK(cudaMemcpyAsync(out, dout, bytes, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return NSF_OK;
}

nsf_status nsf_mpm_set_profiling(nsf_mpm* h, int32_t enable) {
  if (!h) return NSF_ERR_INVALID_ARGUMENT;
  resolve_profiling(h);
  h->profiling = enable != 0;
  if (enable) h->ktimes.clear();
  return NSF_OK;
}

int32_t nsf_mpm_kernel_times(nsf_mpm* h, const char** names, double* total_ms, int64_t* launches, int32_t max) {
  if (!h) return -1;
  resolve_profiling(h);
  int32_t k = 0;
  h->knames_storage.clear();
  for (auto& kv : h->ktimes) h->knames_storage.push_back(kv.first);
  for (auto& kv : h->ktimes) {
    if (k < max) {
      if (names) names[k] = h->knames_storage[k].c_str();
      if (total_ms) total_ms[k] = kv.second.first;
      if (launches) launches[k] = kv.second.second;
    }
    ++k;
  }
  return k;
}

nsf_status nsf_mpm_debug_stats(nsf_mpm* h, int64_t* out, int32_t n) {
  if (!h || !out || n < 1) return NSF_ERR_INVALID_ARGUMENT;
  const int k = stats_read(h->stream, out, n);
  if (k < 0) return cuda_fail(h, cudaGetLastError(), "debug_stats");
  if (k == 0) return fail(h, NSF_ERR_BAD_STATE, "work counters need the statistics build (-DNSF_STATS=1)");
  return NSF_OK;
}

int32_t nsf_mpm_launches_per_substep(nsf_mpm* h) {
  if (!h) return -1;
  return pipeline_launches_per_substep(h, &h->pb);
}

int64_t nsf_mpm_launch_count(const nsf_mpm* h) {
  if (!h) return -1;
  return pipeline_launch_total(const_cast<nsf_mpm*>(h), const_cast<PipelineBuffers*>(&h->pb));
}

#if NSF_CHECKED
// checked build only: a kernel whose NSF_CHECK fails, to show the checks trap
__global__ void k_checked_selftest(int v) { NSF_CHECK(v == 0); }
int32_t nsf_mpm_checked_selftest(int32_t fail) {
  k_checked_selftest<<<1, 1>>>(fail);
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 1;
}
#endif

}  // extern "C"

// ---- accessors used by the pipeline (pipeline.cu) -----------------------------
namespace nsf {
HandleView view(nsf_mpm* h) {
  HandleView v;
  v.P = &h->P;
  v.stream = h->stream;
  v.n = h->n;
  v.pitch = h->pitch;
  v.S[0] = h->S[0]; v.S[1] = h->S[1];
  v.ids[0] = h->ids[0]; v.ids[1] = h->ids[1];
  v.scene_off = h->scene_off;
  v.scene_off_host = h->scene_off_host.empty() ? nullptr : h->scene_off_host.data();
  v.n_scenes = h->mat.n_scenes;
  v.acc = h->acc;
  v.vel = h->vel;
  v.total_nodes = h->total_nodes;
  v.total_blocks = h->total_blocks;
  v.err = h->err;
  v.d_step = h->d_step;
  v.cur = h->cur;
  v.host_step = h->host_step;
  v.mlp = &h->mlp;
  v.X = h->X;
  v.z = h->z;
  v.dz = h->dz;
  v.r = h->r;
  v.model = h->mat.model;
  return v;
}
void set_cur(nsf_mpm* h, int cur) { h->cur = cur; }
void* pipeline_alloc(nsf_mpm* h, size_t bytes) { return dalloc(h, bytes); }
void pipeline_free(nsf_mpm* h, void* p) { dfree(h, p); }
}  // namespace nsf
