// Host-side launchers for the device kernels (internal; not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include "params.cuh"
#include <utility>

namespace nsf {
// launch with programmatic dependent launch (the kernel calls pdl_wait before it
// reads its predecessor's results)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = la;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
}  // namespace nsf

namespace nsf {

// kernels_basic.cu
void launch_unpack(cudaStream_t st, int64_t n, const float* x, const float* v, const float* C,
                   const float* F, float* S, int64_t pitch, int32_t* ids, const DevParams& P,
                   DevErr* err, int with_F);
void launch_pack(cudaStream_t st, int64_t n, const float* S, int64_t pitch, const int32_t* ids,
                 int plane0, int ncomp, float* out);
void launch_p2g_direct(cudaStream_t st, int64_t n, const float* S, int64_t pitch,
                       const int64_t* scene_off, int n_scenes, float4* acc, const DevParams& P);
void launch_g2p_direct(cudaStream_t st, int64_t n, float* S, int64_t pitch, const int64_t* scene_off,
                       int n_scenes, const float4* vel, const DevParams& P, DevErr* err, int64_t* d_step,
                       int with_F, const int32_t* ids);   // ids: load index of each slot (error reports)
void launch_grid_debug(cudaStream_t st, int stage, int64_t total_nodes, const float4* acc, float4* vel,
                       float* out, const DevParams& P, const int64_t* d_step);

// reduced (NSF) substep pieces (point_ops.cuh, kernels_basic.cu)
struct NsfP2G;
void launch_g2p_nsf(cudaStream_t st, int64_t n, float* S, const int64_t* scene_off, int n_scenes,
                    float4* acc0, float4* acc1, const DevParams& P, DevErr* err, int64_t* d_step, int* done,
                    const int32_t* ids);
void launch_nsf_reset_base(cudaStream_t st, int64_t n, float* S);

// kernels_nsf.cu -- neural stress field MLP
struct MlpDev {
  const uint16_t* W;    // bf16 bits, layer-major [out][in]
  const float* b;       // fp32 biases, layer-major
  int in_dim, width, n_hidden, out_dim;
  int64_t w_off[10];    // element offsets of each layer's weights
  int64_t b_off[10];
  unsigned int* ctr;    // [2] tile ticket + CTA completion counter of the tensor-core kernel (zero between
                        // launches), or nullptr for a static tile assignment
};
// tcgen05 tensor-core MLP (kernels_nsf_tc.cu): width 128, 2..4 hidden layers
bool nsf_mlp_tc_supported(const MlpDev& mlp);
void launch_nsf_mlp_tc(cudaStream_t st, int64_t n, const float* X, int64_t xpitch, const int64_t* scene_off,
                       int n_scenes, const float* z, const float* dz, int r, const int64_t* d_step,
                       const MlpDev& mlp, float stress_scale, float* tau_out, int aos_out, const NsfP2G* q);
// tau (AoSoA tau fields of the particle store, or AoS m x 6 if aos_out) = stress_scale * h(X, z_scene(p) + step*dz);
// dispatches to the tensor-core kernel when supported (NSF_MLP_SIMT=1 forces the CUDA-core kernel)
void launch_nsf_mlp(cudaStream_t st, int64_t n, const float* X /*3 planes, pitch*/, int64_t xpitch,
                    const int64_t* scene_off, int n_scenes, const float* z, const float* dz, int r,
                    const int64_t* d_step, const MlpDev& mlp, float stress_scale, float* tau_out,
                    int64_t tau_pitch, int aos_out, const NsfP2G* q = nullptr);
// ... with q: the same kernel then runs the P2G of each point with its tau

// kernels_inv.cu -- network inversion (Gauss-Newton over the deformation field)
size_t gn_smem_bytes(const MlpDev& g);
bool gn_tc_supported(const MlpDev& g, int r);
void launch_gn_tc(cudaStream_t st, int n_scenes, int n_sample, int r, const int32_t* slots, const float* S,
                  const float* zw, const MlpDev& g, double* accum);
void launch_gn_invert(cudaStream_t st, int64_t n, const int32_t* ids, const int64_t* scene_off, int n_scenes,
                      int n_sample, int r, const float* S, const float* z, const float* dz, const int64_t* d_step,
                      const MlpDev& g, int n_iters, int32_t* slots, float* zw, double* accum);

// kernels_infer.cu -- network inference and the integration set
void launch_latent_at(cudaStream_t st, int64_t m, const float* z, const float* dz, int64_t step, float* out);
void launch_backdiff(cudaStream_t st, int64_t n, float* S, float dt);
void launch_mark_stencils(cudaStream_t st, int n_sample, const int32_t* idx, const float* x, uint32_t* mask,
                          const DevParams& P, DevErr* err);
void launch_member_flags(cudaStream_t st, int64_t n_ref, const float* x, const uint32_t* mask,
                         const uint8_t* is_sample, uint8_t* flag, const DevParams& P);
void launch_set_samples(cudaStream_t st, int n_sample, const int32_t* idx, uint8_t* is_sample, uint8_t v);
int64_t compact_blocks(int64_t n);
void launch_count_blocks(cudaStream_t st, int64_t n, const uint8_t* flag, int32_t* cnt);
void launch_compact(cudaStream_t st, int64_t n, const uint8_t* flag, const int32_t* base, int32_t* out);
void launch_scene_scan(cudaStream_t st, int64_t nblk, const int32_t* cnt, int n_sample, int64_t* cursor,
                       int32_t* base, int64_t* scene_count, int scene, int64_t* sample_base);
void launch_put_samples(cudaStream_t st, int n_sample, const int32_t* idx, const int64_t* sample_base,
                        int32_t* list);
void launch_gather_rows3(cudaStream_t st, int64_t m, const int32_t* list, const float* X_all, float* X_new);

}  // namespace nsf
