// Device-side parameters and grid indexing shared by every kernel.
// Layout:
//   grid  : 4x4x4-node blocks, each a contiguous 1 KB of float4; block id
//           b = (b0*NB1 + b1)*NB2 + b2, node (l0,l1,l2) in block at l0*16 + l1*4 + l2;
//           scenes are concatenated (scene s starts at s * nodes_per_scene).
//   particles: SoA component planes, float32, each plane `pitch` floats long.
#pragma once
#include <cstdint>
#include <cstdio>

// Device-side bounds checks of the checked build (libnsf_mpm_checked.so, built
// with -DNSF_CHECKED=1; tests/test_gpu_checked.py): every shared-memory slot,
// grid node, block id and list index the kernels write is asserted in range and a
// violation traps the kernel (the pool offers no compute-sanitizer).  Compiled out
// of the product library.
#ifndef NSF_CHECKED
#define NSF_CHECKED 0
#endif
// Programmatic dependent launch: a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization (launch_pdl, kernels.h) may be
// scheduled before its predecessor completes; pdl_wait() blocks until the
// predecessor's results are visible, pdl_launch_dependents() lets the successor
// be scheduled.  Both are no-ops for a normal launch.
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#endif
// Work counters of the statistics build (-DNSF_STATS=1, nsf_mpm_debug_stats):
// segments, particles, staged rows, listed, inline-scattered, out-of-tile gathers,
// phase-1 passes, and (thread 0 of each CTA, clock64) the cycles spent from the
// loop-top barrier to the staged tile, in phase 1 and in phase 2 of the fused kernel;
// per launch (globaltimer): the CTAs' summed idle time between their own exit and the
// last CTA's, the first-start-to-last-exit duration, and the CTA count.
#ifndef NSF_STATS
#define NSF_STATS 0
#endif
enum StatIdx : int { kStSegments, kStParticles, kStStaged, kStListed, kStInline, kStOutOfTile, kStPasses,
                     kStCycTile, kStCycPhase1, kStCycPhase2, kStOutOfBlock, kStCycP2Acc, kStCycP2Help,
                     kStTailNs, kStKernNs, kStCtas, kStCount = 16 };
#if NSF_STATS
extern __device__ unsigned long long g_nsf_stats[kStCount];
#define NSF_STAT_ADD(i, v) atomicAdd(&g_nsf_stats[(i)], (unsigned long long)(v))
#else
#define NSF_STAT_ADD(i, v) \
  do {                     \
  } while (0)
#endif

#if NSF_CHECKED
#define NSF_CHECK(cond)                                                                  \
  do {                                                                                   \
    if (!(cond)) {                                                                       \
      printf("NSF_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
             (int)blockIdx.x, (int)threadIdx.x);                                         \
      __trap();                                                                          \
    }                                                                                    \
  } while (0)
#else
#define NSF_CHECK(cond) \
  do {                  \
  } while (0)
#endif

namespace nsf {

constexpr int kBlock = 4;            // cells / nodes per block edge
constexpr int kBlockNodes = 64;      // 4^3

// Particle store layout (AoSoA): particles in tiles of 32; field k of particle p
// lives at S[pbase(p) + 32 k], pbase(p) = (p/32) * 32 * kPlanes + p % 32.  A warp
// touching 32 consecutive particles reads/writes 128 contiguous bytes per field,
// and all fields of one particle share one base address (immediate offsets).
// plane indices inside one particle buffer set
enum Plane : int {
  PX = 0,   // x0..x2
  PV = 3,   // v0..v2
  PC = 6,   // C00..C22 (row-major)
  PF = 15,  // F00..F22
  PT = 24,  // tau Voigt xx,yy,zz,yz,xz,xy
  // reduced (NSF) model, which has no F: plane PF holds the packed stencil base of
  // the last P2G, planes PXR..PXR+2 the reference position X (MLP input)
  PXR = PF + 1,
  PTY = 30,  // per-particle von Mises yield stress (hardening / softening); load value elsewhere
  kPlanes = 31
};

constexpr int kTileP = 32;
constexpr int kTileStride = kTileP * kPlanes;
__host__ __device__ __forceinline__ int64_t pbase(int64_t p) { return (p >> 5) * kTileStride + (p & 31); }

enum ErrBits : uint32_t { ERR_OUT_OF_DOMAIN = 1u, ERR_NONFINITE = 2u };

struct DevErr {
  uint32_t bits;
  int32_t first_index;   // atomicMin over offending particle ids
  int64_t step;          // substep at which the first error was seen (approximate)
  unsigned long long inverted;  // count of det F_E <= 0 updates
};

struct DevParams {
  int N[3];          // nodes per axis
  int NB[3];         // blocks per axis
  int nb_shift[3];   // log2 NB[a] when NB[a] is a power of two, else -1 (fast block decoding)
  int n_scenes;
  long long nodes_per_scene;
  long long blocks_per_scene;
  float dx, inv_dx, dt;
  float mass, V0;
  float mu, lam, alpha, tau_Y;
  float g[3];
  int bc[6];
  int bc_width;
  int plate_enabled;
  float plate_y0;
  float plate_v[3];
  int model;
  int force_mode;
  float mls_coef;    // dt V0 4/dx^2
  float gradw_coef;  // dt V0
  float stress_scale;
  int deterministic;  // 1: fixed-point P2G (kernels_det.cu), bitwise reproducible
  float mC;           // affine mass of P2G: m_p (APIC, RPIC) or 0 (PIC)
  int rpic;           // 1: G2P keeps the skew part of C_p (RPIC, reading #38)
  float kappa;        // bulk modulus E / (3 (1 - 2 nu)) (Herschel-Bulkley)
  float hb_yield;     // sqrt(2/3) sigma_Y (Herschel-Bulkley yield condition)
  float hb_relax;     // 1 / (1 + eta / (2 mu dt))
  int vm_hs;          // 1: von Mises with a per-particle yield stress (plane PTY, #30-#32)
  float vm_hard_k;    //   2 mu xi (hardening)
  float vm_soft;      //   theta (softening; tau_Y <= 0 is damage)
};

__host__ __device__ inline long long block_id(int b0, int b1, int b2, const DevParams& P) {
  return ((long long)b0 * P.NB[1] + b1) * P.NB[2] + b2;
}

__host__ __device__ inline long long node_index(int i, int j, int k, const DevParams& P) {
  return block_id(i >> 2, j >> 2, k >> 2, P) * kBlockNodes + ((i & 3) << 4) + ((j & 3) << 2) + (k & 3);
}

}  // namespace nsf
