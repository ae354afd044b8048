/*
 * nsf_mpm.h -- C ABI of the B200 (sm_100a) MLS-MPM substep library for
 * arXiv 2310.17790 "Neural Stress Fields for Reduced-order Elastoplasticity
 * and Fracture".  This header is the boundary: every entry point below is
 * implemented by CUDA kernels in paper_2310_17790_b200/csrc/ and nothing else.
 * No torch types cross it; pointers are plain host or device pointers.
 *
 * Citations are PAPER.md line numbers ("P:L") and SURVEY.md §8(c) readings
 * ("#k"); DESIGN.md lists every reading.
 *
 * What the library computes (one substep, §3.3):
 *   P2G   m_i = sum_p w_ip m_p ; m_i v_i = sum_p w_ip m_p (v_p + C_p (x_i - x_p))
 *         with the stress force of Eq. (6) folded into the momentum:
 *           MLS   (default, #1): - dt V0 (4/dx^2) w_ip tau_p (x_i - x_p)
 *           GRADW (literal Eq.(6)): - dt V0 tau_p grad(w_ip)
 *   grid  v_i = (m_i v_i)/m_i + dt g if m_i > 0, else 0 (#15); then the
 *         wall BCs (#11, #12) and the moving plate (#12).
 *   G2P   v_p = sum w v_i ; C_p = 4/dx^2 sum w v_i (x_i - x_p)^T ;
 *         x_p += dt v_p ; F_trial = (I + dt G) F_E ;
 *         F_E = returnMap(F_trial), tau = tau(F_E) (appendix).
 *   Reduced variant: tau_p = h(X_p, z_s(n)) from the neural stress
 *   field MLP (architecture P:498-500); no F, no SVD.
 *
 * Conventions
 *   Layouts   caller arrays are row-major AoS, float32: x, v as n x 3; C, F as
 *             n x 3 x 3 with C[p][a][b]; tau as n x 6 in Voigt order
 *             (xx, yy, zz, yz, xz, xy).  Grid node i = (i0,i1,i2) sits at i*dx
 *             (#8, #10); grid_res is nodes per axis and must be a multiple of 4.
 *   Ownership the handle owns all device memory (allocated through the optional
 *             allocator hook, else cudaMalloc).  The caller owns every buffer it
 *             passes; the library never keeps a caller pointer after a call.
 *   on_device 1: pointers are device pointers, valid and stream-ordered on the
 *             handle's stream; 0: host pointers (pinned or pageable).
 *   Synchrony nsf_mpm_substep only enqueues work and returns.  load_*,
 *             set_latents, eval_stress_field, read_state and the debug calls
 *             complete their own work (stream-ordered after earlier substeps)
 *             before returning.  nsf_mpm_sync blocks.
 *   Errors    every call returns nsf_status (0 = OK).  Argument checks happen at
 *             call time (NSF_ERR_INVALID_ARGUMENT).  Particles outside the safe
 *             region x/dx in [0.5, N - 1.5) are rejected at load with
 *             NSF_ERR_OUT_OF_DOMAIN (first index in last_error).  During
 *             substeps, out-of-domain and non-finite values set bits in a device
 *             error word (kernels clamp indices so memory stays in bounds); the
 *             next sync / read_state reports them.  A CUDA error poisons the
 *             handle: every later call returns NSF_ERR_CUDA.  Inverted F
 *             (det <= 0) is not an error (#21); it is counted.
 *   Threads   a handle is single-owner and not thread-safe; distinct handles are
 *             independent.
 */
#ifndef NSF_MPM_H
#define NSF_MPM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NSF_MPM_ABI_VERSION 5

typedef struct nsf_mpm nsf_mpm; /* opaque; owns all device state */

typedef enum {
  NSF_OK = 0,
  NSF_ERR_INVALID_ARGUMENT = 1,
  NSF_ERR_OUT_OF_DOMAIN = 2,
  NSF_ERR_NONFINITE = 3,
  NSF_ERR_CUDA = 4,
  NSF_ERR_OUT_OF_MEMORY = 5,
  NSF_ERR_BAD_STATE = 6
} nsf_status;

/* Constitutive model (PAPER.md appendix).  DP and VM use Hencky
 * (log-strain) elasticity (#5), with tau = U diag(2 mu eps + lambda sum eps) U^T
 * (#3).  NSF = reduced variant, stress from the neural stress field. */
typedef enum {
  NSF_FIXED_COROTATED = 0, /* tau = 2 mu (F - R) F^T + lambda (J-1) J I   (#2) */
  NSF_DRUCKER_PRAGER = 1,  /* sand return map */
  NSF_VON_MISES = 2,       /* perfect plasticity, radial return          (#4) */
  NSF_NEURAL_STRESS = 3,   /* tau = sigma_tau h(X, z) */
  NSF_HENCKY = 4,          /* the appendix's "StVK elasticity": Hencky, no return map (#3) */
  NSF_HERSCHEL_BULKLEY = 5 /* viscoplastic, h = 1 (#39): yield_stress = sigma_Y, viscosity
                              = eta; tau = kappa/2 (J^2-1) I + mu dev(bbar) (ABI 5)               */
} nsf_model;

/* Particle-grid transfer of P2G's momentum. */
typedef enum {
  NSF_TRANSFER_APIC = 0,   /* m_i v_i = sum w m_p (v_p + C_p (x_i - x_p)) */
  NSF_TRANSFER_PIC = 1,    /* m_i v_i = sum w m_p v_p (C_p still updated and used for F)  */
  NSF_TRANSFER_RPIC = 2    /* APIC with C_p = skew part of the G2P affine matrix (the
                              damping variant; F_trial still uses the full gradient) (ABI 5) */
} nsf_transfer;

/* Wall boundary condition on the nodes within bc_width of a face (#11, #12). */
typedef enum {
  NSF_BC_NONE = 0,
  NSF_BC_STICKY = 1, /* v_i = 0 */
  NSF_BC_SLIP = 2    /* zero the normal component if it points into the wall */
} nsf_bc;

typedef enum {
  NSF_FORCE_MLS = 0,  /* grad w -> (4/dx^2) w (x_i - x_p), F_trial = (I + dt C) F (#1) */
  NSF_FORCE_GRADW = 1 /* Eq. (6) and P:179 literally                                 */
} nsf_force_mode;

typedef struct {
  int32_t model;                /* nsf_model                                        */
  double E, nu, rho;            /* Pa, -, kg/m^3; E > 0, 0 <= nu < 0.5   */
  double friction_angle_deg;    /* DP phi_f in (0, 90)    */
  double yield_stress;          /* VM tau_Y >= 0 (Pa)    */
  double gravity[3];            /* m/s^2, y is up                          (#13)     */
  int32_t bc[6];                /* nsf_bc for faces -x,+x,-y,+y,-z,+z               */
  int32_t bc_width;             /* nodes (3 in every config)               (#11)     */
  int32_t plate_enabled;        /* moving rigid plate: nodes with y_i >= y_p(t_n)   */
  double plate_y0;              /*   y_p(t_n) = plate_y0 + plate_velocity[1] n dt   */
  double plate_velocity[3];     /*   get v_i = plate_velocity, after the walls (#12)*/
  int32_t force_mode;           /* nsf_force_mode                                   */
  int32_t deterministic;        /* 0: fastest (P2G float reductions in scheduling order);
                                   1: P2G reduced in 64-bit fixed point with integer atomics
                                   (units 2^-32 particle masses), so every substep is bitwise
                                   reproducible, independent of particle order and launch
                                   configuration; slower.  Other values: INVALID_ARGUMENT. */
  int32_t n_scenes;             /* >= 1; each scene owns a grid_res^3 grid          */
  double particle_volume;       /* V_p^0 (m^3); <= 0 -> dx^3/8 (8 ppc, #16); m = rho V0 */
  double stress_scale;          /* sigma_tau (Pa) multiplying the NSF output (#20)   */
  int32_t transfer;             /* nsf_transfer (ABI 2)                              */
  /* von Mises yield-stress evolution (ABI 3, readings #30-#32): with
   * either coefficient non-zero every particle carries its own tau_Y (starting at
   * yield_stress); after a projecting return map (delta_gamma > 0)
   *   tau_Y <- tau_Y + 2 mu hardening delta_gamma - softening ||eps - proj(eps)||_F
   * (the norm equals delta_gamma).  With softening > 0 a particle whose tau_Y reaches 0
   * is damaged: zero Lame parameters (tau = 0) and no return map from then on.
   * Both >= 0 and finite (else INVALID_ARGUMENT); ignored for other models. */
  double hardening;             /* xi                                                */
  double softening;             /* theta (1/Pa * Pa: tau_Y units per unit log strain) */
  double viscosity;             /* Herschel-Bulkley eta >= 0 (Pa s; ABI 5); the
                                   relaxation factor is 1 / (1 + eta / (2 mu dt))    */
} nsf_material;

/* read_state field mask; dst[k] is the k-th requested field in bit order. */
#define NSF_FIELD_X 1u   /* n x 3                                   */
#define NSF_FIELD_V 2u   /* n x 3                                   */
#define NSF_FIELD_C 4u   /* n x 3 x 3                               */
#define NSF_FIELD_F 8u   /* n x 3 x 3 (elastic F_E; not for NSF)     */
#define NSF_FIELD_TAU 16u /* n x 6 Voigt (stress used by the NEXT P2G) */
#define NSF_FIELD_TAU_Y 32u /* n x 1 per-particle von Mises yield stress (ABI 3) */

/* Work counters of the fused full-order kernel since the last call (statistics
 * build only, -DNSF_STATS=1; else NSF_ERR_BAD_STATE): out[0..n-1] = segments,
 * particles, staged P2G rows, listed (out-of-block) rows, inline scatters,
 * out-of-tile gathers, phase-1 passes, and the clock cycles (thread 0 of each CTA)
 * spent staging the velocity tile, in phase 1 and in phase 2, then out-of-block
 * particles.  Synchronizes the handle's stream; clears the counters.  (ABI 5) */
nsf_status nsf_mpm_debug_stats(nsf_mpm* h, int64_t* out, int32_t n);

/* Version of this header's ABI (NSF_MPM_ABI_VERSION). */
int32_t nsf_mpm_abi_version(void);

/* Create a simulator on the current CUDA device.  grid_res: nodes per axis
 * (each a multiple of 4, >= 2*bc_width + 3).  dx, dt > 0 (s, m).  dx should be
 * an exact power of two so B-spline bases are exact in fp32 (#10).  Returns
 * NSF_ERR_INVALID_ARGUMENT on a bad parameter (see nsf_material comments); for
 * NSF_NEURAL_STRESS also when an axis has more than 1024 nodes or a scene has
 * 2^31 nodes or more (the reduced G2P packs stencil bases in 10 bits per axis
 * and addresses a scene's nodes with 32-bit offsets). */
nsf_status nsf_mpm_create(const int32_t grid_res[3], double dx, double dt,
                          const nsf_material* material, nsf_mpm** out);

/* Stream for all later work (cudaStream_t; NULL = the non-blocking stream the handle
 * created for itself, which is also the default).  Cached CUDA graphs are dropped when the stream changes. */
nsf_status nsf_mpm_set_stream(nsf_mpm* h, void* cuda_stream);

/* Optional device allocator (e.g. torch's caching allocator), used for every
 * allocation made after this call.  alloc returns NULL on failure.  Returned
 * pointers must be 256-byte aligned (cudaMalloc's and torch's are): the kernels
 * make 256-bit accesses to grid node pairs and 128-byte particle tiles; every
 * allocation is checked, and a misaligned pointer is handed back to `release`
 * and fails the allocating call (NSF_ERR_INVALID_ARGUMENT from the load / create
 * calls, NSF_ERR_OUT_OF_MEMORY from internal scratch).  Each block is released
 * through the release function (and ctx) that was installed when it was
 * allocated, so the hook may be replaced or removed (alloc = release = NULL:
 * cudaMalloc again) at any time.  A call that fails part-way leaves the
 * affected state unloaded (BAD_STATE until it is loaded again), never a
 * handle that points at released memory. */
nsf_status nsf_mpm_set_allocator(nsf_mpm* h,
                                 void* (*alloc)(size_t bytes, void* stream, void* ctx),
                                 void (*release)(void* ptr, void* stream, void* ctx),
                                 void* ctx);

/* Load n particles (replaces any previous state, resets the step counter).
 * x, v: n x 3; C, F: n x 3 x 3 (NULL -> 0 / I).  tau^0 = tau(F^0) (#9).
 * scene_offsets: n_scenes + 1 monotone int64 with [0] = 0, [n_scenes] = n
 * (particles of scene s are [off[s], off[s+1])); NULL allowed if n_scenes = 1.
 * n = 0 is allowed (substeps are then no-ops).  Rejects out-of-domain
 * particles with NSF_ERR_OUT_OF_DOMAIN. */
nsf_status nsf_mpm_load_particles(nsf_mpm* h, int64_t n, const float* x, const float* v,
                                  const float* C, const float* F,
                                  const int64_t* scene_offsets, int32_t on_device);

/* Neural stress field h: in_dim = 3 + r inputs (X, z),
 * n_hidden hidden layers of `width` with ELU, out_dim = 6 (Voigt).  W_bf16:
 * bf16 bit patterns, layer-major, each layer row-major [out][in]; b: float32
 * biases, layer-major.  X_ref: n x 3 reference positions of the loaded
 * particles (same order as load_particles), or NULL to keep the previous ones.
 * Numerics (#20): layer-1 input fp32, hidden activations rounded to bf16 before
 * layers 2..L+1, fp32 accumulation, bias and ELU in fp32.
 * Supported: width = 128, 1 <= n_hidden <= 8, in_dim <= 16, out_dim = 6. */
nsf_status nsf_mpm_load_stress_field(nsf_mpm* h, int32_t in_dim, int32_t width,
                                     int32_t n_hidden, int32_t out_dim,
                                     const uint16_t* W_bf16, const float* b,
                                     const float* X_ref, int32_t on_device);

/* Latents: z is n_scenes x r; dz (n_scenes x r or NULL = 0) is the per-substep
 * drift, z_s(n) = z_s + n dz_s with n the handle's step counter (#26). */
nsf_status nsf_mpm_set_latents(nsf_mpm* h, int32_t r, const float* z, const float* dz,
                               int32_t on_device);

/* Neural deformation field g(X, z) -> x (architecture P:498-500), the
 * network that invert_latents inverts.  Same parameter layout and numerics as
 * load_stress_field; in_dim = 3 + r, out_dim = 3, width = 128, 1 <= n_hidden
 * <= 4.  INVALID_ARGUMENT otherwise; BAD_STATE before load_particles. */
nsf_status nsf_mpm_load_deformation_field(nsf_mpm* h, int32_t in_dim, int32_t width,
                                          int32_t n_hidden, int32_t out_dim,
                                          const uint16_t* W_bf16, const float* b,
                                          int32_t on_device);

/* Network inversion (Eq. (10)): per scene s, starting from the latent
 * the last substep used, z_s(n) = z_s + n dz_s, run n_iters Gauss-Newton
 * iterations (1 = the first-order Taylor variant) of
 *     min_z sum_{p in S_s} || g(X_p, z) - x_p ||^2
 * where S_s = the scene's first n_sample points in load order and x_p their
 * current positions.  Jacobians by forward mode on the GPU; normal equations
 * in fp64.  The handle's latents become z_s := z_hat_s, dz_s := 0 (the next
 * substeps use the inverted latent).  z_out (n_scenes x r, host or device per
 * on_device, or NULL) receives z_hat.  Requires the NSF model with
 * load_stress_field (X_ref), set_latents and load_deformation_field;
 * 1 <= n_sample, 1 <= n_iters <= 16.  A scene whose normal matrix is not
 * positive definite keeps its latent. */
nsf_status nsf_mpm_invert_latents(nsf_mpm* h, int32_t n_sample, int32_t n_iters, float* z_out,
                                  int32_t on_device);

/* Neural affine-velocity field l(X, z) -> C (9 outputs, row-major 3 x 3; PAPER.md
 * line 253) for infer_state (ABI 4).  Same parameter layout and numerics as
 * load_stress_field; in_dim = 3 + r, width = 128, 1 <= n_hidden <= 8, out_dim = 9.
 * INVALID_ARGUMENT otherwise.  Synchronous. */
nsf_status nsf_mpm_load_affine_field(nsf_mpm* h, int32_t in_dim, int32_t width, int32_t n_hidden,
                                     int32_t out_dim, const uint16_t* W_bf16, const float* b,
                                     int32_t on_device);

/* Network inference (ABI 4) for every current point p with
 * reference position X_p (load_stress_field's X_ref):
 *     x_p = g(X_p, z_n),  v_p = (g(X_p, z_n) - g(X_p, z_prev)) / dt,  C_p = l(X_p, z_n)
 * with z_n = z + n dz the latent of the next substep (n = the step counter) and
 * z_prev (n_scenes x r floats, host or device per on_device) the previous latent,
 * or NULL for z + (n-1) dz (n >= 1) resp. z_n (n = 0: particles at rest).
 * Overwrites x, v and C (tau comes from the stress field in the next substep).
 * Asynchronous.  BAD_STATE without the NSF model, load_stress_field with X_ref,
 * set_latents, load_deformation_field and load_affine_field; INVALID_ARGUMENT if g
 * or l does not take 3 + r inputs. */
nsf_status nsf_mpm_infer_state(nsf_mpm* h, const float* z_prev, int32_t on_device);

/* Sample and integration particles (ABI 4).  X_all: the
 * reference body (n_ref x 3, shared by all scenes); per scene s the sample particles
 * S_s = X_all[sample_idx[s * n_sample + q]], q < n_sample (distinct within a scene).
 * With x_p = g(X_p, z_n(s)) (z_n as in infer_state):
 *     I_s = nodes of the 27-node stencils (base = floor(x/dx - 1/2)) of the x_p, p in S_s
 *     N_s = { p : the stencil of x_p meets I_s }          (S_s is a subset of N_s)
 * The handle's points become, per scene, S_s in the given order followed by N_s \ S_s
 * in increasing index order (so invert_latents' "first n_sample points" are S_s),
 * with reference positions X_all[p] and infer_state(z_prev) applied; the step
 * counter and latents are kept.  counts_out (host, n_scenes) receives |N_s|; may be
 * NULL.  Synchronous; X_all, sample_idx and z_prev are host or device per on_device.
 * INVALID_ARGUMENT for bad sizes or indices, BAD_STATE as for infer_state,
 * OUT_OF_DOMAIN if a sample's stencil leaves the grid. */
nsf_status nsf_mpm_build_integration_set(nsf_mpm* h, int64_t n_ref, const float* X_all,
                                         int32_t n_sample, const int32_t* sample_idx,
                                         const float* z_prev, int64_t* counts_out,
                                         int32_t on_device);

/* One latent-space time step of the reduced model (§5; ABI 5):
 *   (1) build_integration_set(n_ref, X_all, n_sample, sample_idx) at z_n, with
 *       network inference of x, v, C on N; z_{n-1} = z_prev if given (n_scenes x r),
 *       else the z_n of the previous rom_step, else (first call after set_latents)
 *       the infer_state default,
 *   (2) one MPM substep on N (the sample particles' states are those of the
 *       full-order MPM, line 256),
 *   (3) invert_latents(n_sample, gn_iters): z_{n+1} from Eq. (10) on S.
 * z_out (n_scenes x r, host or device per on_device, or NULL) receives z_{n+1};
 * counts_out (host, n_scenes, or NULL) |N_s|.  Synchronous.  Errors as for the three
 * calls; 1 <= gn_iters <= 16. */
nsf_status nsf_mpm_rom_step(nsf_mpm* h, int64_t n_ref, const float* X_all, int32_t n_sample,
                            const int32_t* sample_idx, const float* z_prev, int32_t gn_iters, float* z_out,
                            int64_t* counts_out, int32_t on_device);

/* Enqueue n >= 0 substeps on the handle's stream (a cached CUDA graph of the
 * substep is replayed).  Asynchronous.  NSF_ERR_BAD_STATE before
 * load_particles, or for NSF without load_stress_field / set_latents.
 * The state every other call sees is that after the n-th substep.  On the
 * full-order MLS path, where G2P and the next P2G are one
 * kernel, v_p, C_p and tau_p of the first n - 1 substeps only feed that P2G and
 * stay in registers; the n-th substep stores them (x_p and F_E are stored by
 * every substep), so one call of n substeps moves less memory than n calls. */
nsf_status nsf_mpm_substep(nsf_mpm* h, int32_t n);

/* Evaluate tau = sigma_tau h(X, z) at m points (m x 3) for one latent z (r
 * floats) into tau_out (m x 6 Voigt).  Synchronous. */
nsf_status nsf_mpm_eval_stress_field(nsf_mpm* h, const float* z, int64_t m,
                                     const float* points, float* tau_out, int32_t on_device);

/* Copy the requested fields (mask of NSF_FIELD_*) of all particles, in the order
 * they were loaded, into dst[0..popcount(mask)-1].  Synchronous; reports
 * deferred device errors first. */
nsf_status nsf_mpm_read_state(nsf_mpm* h, uint32_t field_mask, float* const* dst,
                              int32_t on_device);

/* Block until all enqueued work is done; report deferred device errors
 * (NSF_ERR_OUT_OF_DOMAIN / NSF_ERR_NONFINITE with the smallest offending
 * particle index -- its position in the arrays passed to load_particles, not
 * its internal storage slot -- and the substep count in last_error). */
nsf_status nsf_mpm_sync(nsf_mpm* h);

/* Substeps enqueued since the last load (host counter). */
int64_t nsf_mpm_step_count(const nsf_mpm* h);

/* Number of particle updates that produced det F_E <= 0 since load (#21). */
int64_t nsf_mpm_inverted_count(nsf_mpm* h);

/* Human-readable description of the last error; valid until the next call. */
const char* nsf_mpm_last_error(const nsf_mpm* h);

/* Free everything (NULL-safe). */
void nsf_mpm_destroy(nsf_mpm* h);

/* ---- diagnostics (tests and bench; not on the hot path) -------------------- */

/* Binning of the current state: counts[b] = number of
 * particles whose base cell floor(x/dx - 1/2) lies in 4x4x4-cell block b
 * (b = (b0*NB1 + b1)*NB2 + b2 per scene, scenes concatenated, NB = grid_res/4),
 * and perm = a permutation of 0..n-1 (load order) grouping particles by block in
 * ascending block order.  counts has n_scenes*NB0*NB1*NB2 entries.  Either
 * output may be NULL.  Synchronous. */
nsf_status nsf_mpm_debug_bins(nsf_mpm* h, int32_t* counts, int32_t* perm, int32_t on_device);

/* Run P2G (stage 0) or P2G + grid update (stage 1) on the current state without
 * advancing it, and copy the dense grid, n_scenes x N0 x N1 x N2 x 4 floats in
 * natural node order: stage 0 (m_i, m_i v_i), stage 1 (v_i, m_i).  Synchronous. */
nsf_status nsf_mpm_debug_grid(nsf_mpm* h, int32_t stage, float* out, int32_t on_device);

/* Per-kernel timing with CUDA events on the handle's stream.  While enabled,
 * substeps are launched without a graph and every kernel launch is bracketed
 * by events.  nsf_mpm_kernel_times fills up to max entries (name, total ms,
 * launches) and returns the number of kernel kinds. */
nsf_status nsf_mpm_set_profiling(nsf_mpm* h, int32_t enable);
int32_t nsf_mpm_kernel_times(nsf_mpm* h, const char** names, double* total_ms,
                             int64_t* launches, int32_t max);

/* Number of kernel launches of the most recently enqueued substep. */
int32_t nsf_mpm_launches_per_substep(nsf_mpm* h);

/* Kernel launches enqueued by nsf_mpm_substep since the last load (the fused
 * pipeline adds a re-binning every 32 substeps, so this is not n x a constant). */
int64_t nsf_mpm_launch_count(const nsf_mpm* h);

#ifdef __cplusplus
}
#endif
#endif /* NSF_MPM_H */
