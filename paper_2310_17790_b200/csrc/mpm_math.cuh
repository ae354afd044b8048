// Per-particle device math: quadratic B-spline stencil, rotation-safe 3x3 SVD,
// polar rotation, constitutive models and return maps (fp32, in registers).
//
// PAPER.md citations ("P:L"):
//   B-spline weights w_ip, degree b = 2 ............ P:165, P:180 (readings #7, #10)
//   fixed corotated tau = 2 mu (F-R) F^T + lambda (J-1) J I ... P:518 (#2)
//   Hencky tau = U diag(2 mu eps + lambda sum eps) U^T ...... P:524 (#3)
//   Drucker-Prager Z(Sigma) .......................... P:528-536 (#6)
//   von Mises Z(Sigma) .............................. P:538-545 (#4)
//   rotation-safe SVD, sigma >= 1e-4 before logs ..... reading #21
#pragma once
#include <cmath>
#include "params.cuh"

namespace nsf {

// ---------------------------------------------------------------------------
// Quadratic B-spline on one axis.  t = x * inv_dx is exact for power-of-two dx
// (#10), so base and f agree bit-for-bit with the fp64 oracle.
struct Axis {
  int base;
  float f;
  float w[3];
  float dw[3];   // d w / d x  (only used by GRADW)
};

// RPIC (reading #38): C <- (C - C^T) / 2, the rigid-rotation part
__device__ __forceinline__ void skew_part(float C[9]) {
  const float a = 0.5f * (C[1] - C[3]), b = 0.5f * (C[2] - C[6]), c = 0.5f * (C[5] - C[7]);
  C[0] = C[4] = C[8] = 0.0f;
  C[1] = a; C[3] = -a;
  C[2] = b; C[6] = -b;
  C[5] = c; C[7] = -c;
}

__device__ __forceinline__ Axis bspline_axis(float x, float inv_dx) {
  Axis a;
  float t = x * inv_dx;
  float b = floorf(t - 0.5f);
  a.base = (int)b;
  a.f = t - b;
  float f = a.f;
  float u = 1.5f - f, m = f - 1.0f, l = f - 0.5f;
  a.w[0] = 0.5f * u * u;
  a.w[1] = 0.75f - m * m;
  a.w[2] = 0.5f * l * l;
  a.dw[0] = -u * inv_dx;
  a.dw[1] = -2.0f * m * inv_dx;
  a.dw[2] = l * inv_dx;
  return a;
}

// ---------------------------------------------------------------------------
// small 3x3 helpers (row-major float[9])
__device__ __forceinline__ float det3(const float A[9]) {
  return A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) +
         A[2] * (A[3] * A[7] - A[4] * A[6]);
}

// One cyclic-Jacobi rotation zeroing S[p][q] of the symmetric S, accumulating V.
// (Classic two-sided Jacobi eigenvalue step on S = A^T A.)
__device__ __forceinline__ void jacobi_pq(float S[3][3], float V[3][3], int p, int q) {
  float apq = S[p][q];
  if (!(fabsf(apq) > 1e-18f)) return;
  float app = S[p][p], aqq = S[q][q];
  // t = tan(angle) = 2 apq sgn(d) / (|d| + sqrt(d^2 + 4 apq^2)), d = aqq - app (the
  // smaller root of t^2 + 2 theta t - 1 = 0, theta = d / (2 apq); overflow-free).
  // An approximate t still gives an exactly orthogonal (c, s); the sweep
  // absorbs the difference.
  const float d = aqq - app;
  const float h = fmaf(d, d, 4.0f * apq * apq);
  const float den = fabsf(d) + h * rsqrtf(h);
  float t = __fdividef(copysignf(2.0f, d) * apq, den);
  float c = rsqrtf(fmaf(t, t, 1.0f));
  float s = t * c;
  S[p][p] = app - t * apq;
  S[q][q] = aqq + t * apq;
  S[p][q] = 0.0f;
  S[q][p] = 0.0f;
  int r = 3 - p - q;
  float srp = S[r][p], srq = S[r][q];
  float nrp = c * srp - s * srq;
  float nrq = s * srp + c * srq;
  S[r][p] = nrp; S[p][r] = nrp;
  S[r][q] = nrq; S[q][r] = nrq;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    float vip = V[i][p], viq = V[i][q];
    V[i][p] = c * vip - s * viq;
    V[i][q] = s * vip + c * viq;
  }
}

// Givens rotation on rows (a, b) of B zeroing B[b][col]; the same row rotation
// is applied to Qt (so that Qt B = R at the end).
__device__ __forceinline__ void givens_rows(float B[3][3], float Qt[3][3], int a, int b, int col) {
  float x = B[a][col], y = B[b][col];
  float r2 = fmaf(x, x, y * y);
  float c = 1.0f, s = 0.0f;
  if (r2 > 1e-37f) {
    float ir = rsqrtf(r2);
    c = x * ir;
    s = y * ir;
  }
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    float ba = B[a][j], bb = B[b][j];
    B[a][j] = c * ba + s * bb;
    B[b][j] = -s * ba + c * bb;
    float qa = Qt[a][j], qb = Qt[b][j];
    Qt[a][j] = c * qa + s * qb;
    Qt[b][j] = -s * qa + c * qb;
  }
}

// Rotation-safe SVD A = U diag(sig) V^T, det U = det V = +1, sig sorted by
// decreasing magnitude with any reflection folded into sig[2] (reading #21).
// Jacobi eigen-decomposition of A^T A gives V; QR (Givens) of A V gives U, sig.
__device__ __forceinline__ void svd3(const float A[9], float U[3][3], float sig[3], float V[3][3]) {
  float S[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      S[i][j] = A[0 * 3 + i] * A[0 * 3 + j] + A[1 * 3 + i] * A[1 * 3 + j] + A[2 * 3 + i] * A[2 * 3 + j];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) V[i][j] = (i == j) ? 1.0f : 0.0f;

  for (int sweep = 0; sweep < 6; ++sweep) {
    float off = fabsf(S[0][1]) + fabsf(S[0][2]) + fabsf(S[1][2]);
    float dia = fabsf(S[0][0]) + fabsf(S[1][1]) + fabsf(S[2][2]);
    if (off <= 1e-9f * dia) break;
    jacobi_pq(S, V, 0, 1);
    jacobi_pq(S, V, 0, 2);
    jacobi_pq(S, V, 1, 2);
  }
  // B = A V
  float B[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      B[i][j] = A[i * 3 + 0] * V[0][j] + A[i * 3 + 1] * V[1][j] + A[i * 3 + 2] * V[2][j];
  // sort columns by decreasing norm; each swap negates one column so det V stays +1
  float n0 = B[0][0] * B[0][0] + B[1][0] * B[1][0] + B[2][0] * B[2][0];
  float n1 = B[0][1] * B[0][1] + B[1][1] * B[1][1] + B[2][1] * B[2][1];
  float n2 = B[0][2] * B[0][2] + B[1][2] * B[1][2] + B[2][2] * B[2][2];
  auto swapcol = [&](int a, int b) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      float t = B[i][a]; B[i][a] = -B[i][b]; B[i][b] = t;
      float u = V[i][a]; V[i][a] = -V[i][b]; V[i][b] = u;
    }
  };
  if (n0 < n1) { swapcol(0, 1); float t = n0; n0 = n1; n1 = t; }
  if (n0 < n2) { swapcol(0, 2); float t = n0; n0 = n2; n2 = t; }
  if (n1 < n2) { swapcol(1, 2); float t = n1; n1 = n2; n2 = t; }
  // QR of B by Givens: Qt B = R, U = Qt^T
  float Qt[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) Qt[i][j] = (i == j) ? 1.0f : 0.0f;
  givens_rows(B, Qt, 0, 1, 0);
  givens_rows(B, Qt, 0, 2, 0);
  givens_rows(B, Qt, 1, 2, 1);
  sig[0] = B[0][0];
  sig[1] = B[1][1];
  sig[2] = B[2][2];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) U[i][j] = Qt[j][i];
}

// ---------------------------------------------------------------------------
// constitutive update: F_trial -> (F_E, tau Voigt).  Returns det(F_E).
//   model 0: fixed corotated   1: Drucker-Prager + Hencky   2: von Mises + Hencky
// dg_out (optional): the von Mises delta_gamma where the map projects, else 0
// (the per-particle yield-stress update of P:545 uses it).
__device__ __forceinline__ float elastoplastic(const float Ft[9], int model, float mu, float lam,
                                               float alpha, float tau_Y, float FE[9], float tau[6],
                                               float* dg_out = nullptr) {
  float U[3][3], V[3][3], s[3];
  svd3(Ft, U, s, V);
  if (model == 0) {
    // R = U V^T ; tau = 2 mu (F - R) F^T + lambda (J - 1) J I
    float R[9], D[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        R[i * 3 + j] = U[i][0] * V[j][0] + U[i][1] * V[j][1] + U[i][2] * V[j][2];
        D[i * 3 + j] = Ft[i * 3 + j] - R[i * 3 + j];
      }
    float J = det3(Ft);
    float vol = lam * (J - 1.0f) * J;
    float T[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        T[i][j] = 2.0f * mu * (D[i * 3 + 0] * Ft[j * 3 + 0] + D[i * 3 + 1] * Ft[j * 3 + 1] +
                               D[i * 3 + 2] * Ft[j * 3 + 2]);
    tau[0] = T[0][0] + vol;
    tau[1] = T[1][1] + vol;
    tau[2] = T[2][2] + vol;
    tau[3] = 0.5f * (T[1][2] + T[2][1]);
    tau[4] = 0.5f * (T[0][2] + T[2][0]);
    tau[5] = 0.5f * (T[0][1] + T[1][0]);
#pragma unroll
    for (int k = 0; k < 9; ++k) FE[k] = Ft[k];
    return J;
  }
  // log-strain models (reading #21: clamp sigma >= 1e-4)
  const float kFloor = 1e-4f;
  bool clamped = (s[0] < kFloor) | (s[1] < kFloor) | (s[2] < kFloor);
  float sc[3] = {fmaxf(s[0], kFloor), fmaxf(s[1], kFloor), fmaxf(s[2], kFloor)};
  float e[3] = {logf(sc[0]), logf(sc[1]), logf(sc[2])};
  float tr = e[0] + e[1] + e[2];
  float eh[3] = {e[0] - tr * (1.0f / 3.0f), e[1] - tr * (1.0f / 3.0f), e[2] - tr * (1.0f / 3.0f)};
  float nrm = sqrtf(eh[0] * eh[0] + eh[1] * eh[1] + eh[2] * eh[2]);
  float dg;
  bool expand = false;
  if (model == 1) {
    expand = tr > 0.0f;
    dg = nrm + alpha * (3.0f * lam + 2.0f * mu) * tr / (2.0f * mu);
  } else {
    dg = nrm - tau_Y / (2.0f * mu);
  }
  if (dg_out) *dg_out = (model == 2 && dg > 0.0f) ? dg : 0.0f;
  float le[3];   // log Z
  bool elastic = false;
  if (expand) {
    le[0] = le[1] = le[2] = 0.0f;
  } else if (dg <= 0.0f) {
    le[0] = e[0]; le[1] = e[1]; le[2] = e[2];
    elastic = true;
  } else {
    float k = dg / nrm;
    le[0] = e[0] - k * eh[0];
    le[1] = e[1] - k * eh[1];
    le[2] = e[2] - k * eh[2];
  }
  float detFE;
  if (elastic && !clamped) {
#pragma unroll
    for (int k = 0; k < 9; ++k) FE[k] = Ft[k];
    detFE = det3(Ft);
  } else {
    float Z[3];
    if (elastic) { Z[0] = sc[0]; Z[1] = sc[1]; Z[2] = sc[2]; }
    else { Z[0] = expf(le[0]); Z[1] = expf(le[1]); Z[2] = expf(le[2]); }
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        FE[i * 3 + j] = U[i][0] * Z[0] * V[j][0] + U[i][1] * Z[1] * V[j][1] + U[i][2] * Z[2] * V[j][2];
    detFE = Z[0] * Z[1] * Z[2];
  }
  const float kLogFloor = -9.210340371976184f;   // log(1e-4)
  float l0 = fmaxf(le[0], kLogFloor), l1 = fmaxf(le[1], kLogFloor), l2 = fmaxf(le[2], kLogFloor);
  float sum = l0 + l1 + l2;
  float d0 = 2.0f * mu * l0 + lam * sum, d1 = 2.0f * mu * l1 + lam * sum, d2 = 2.0f * mu * l2 + lam * sum;
  // tau = U diag(d) U^T
  tau[0] = U[0][0] * U[0][0] * d0 + U[0][1] * U[0][1] * d1 + U[0][2] * U[0][2] * d2;
  tau[1] = U[1][0] * U[1][0] * d0 + U[1][1] * U[1][1] * d1 + U[1][2] * U[1][2] * d2;
  tau[2] = U[2][0] * U[2][0] * d0 + U[2][1] * U[2][1] * d1 + U[2][2] * U[2][2] * d2;
  tau[3] = U[1][0] * U[2][0] * d0 + U[1][1] * U[2][1] * d1 + U[1][2] * U[2][2] * d2;
  tau[4] = U[0][0] * U[2][0] * d0 + U[0][1] * U[2][1] * d1 + U[0][2] * U[2][2] * d2;
  tau[5] = U[0][0] * U[1][0] * d0 + U[0][1] * U[1][1] * d1 + U[0][2] * U[1][2] * d2;
  return detFE;
}

// ---------------------------------------------------------------------------
// Fast constitutive path (same results as elastoplastic() up to rounding).
// (vm_hs_update below wraps it for the per-particle yield stress of P:545.)
//
// Log-strain models (DP, VM): with F = U Sigma V^T, the left Cauchy-Green tensor
// b = F F^T = U Sigma^2 U^T, so a symmetric Jacobi eigen-decomposition of b gives
// U and sigma_i = sqrt(lambda_i) without the QR step; V is never formed:
// F_E = U diag(Z) V^T = U diag(Z/sigma) U^T F.  Fixed corotated: the polar
// rotation R = U V^T is the limit of the scaled Newton iteration
// R <- (g R + R^{-T}/g)/2, g = |det R|^{-1/3} (Higham), started at R = F.
// Both fall back to the rotation-safe SVD when det F <= 1e-6 or sigma < 1e-4
// (reading #21: inverted / degenerate F), so conventions stay identical.

#ifndef NSF_LOGSTRAIN_SERIES
#define NSF_LOGSTRAIN_SERIES 1   // eigen-free Hencky / return maps for ||F F^T - I||_F <= 0.3
#endif
#ifndef NSF_JACOBI_TOL2
#define NSF_JACOBI_TOL2 1e-13f   // (off-diagonal / ||A||)^2 stopping level of sym_eig3
#endif
// Symmetric 3x3 eigen-decomposition by cyclic Jacobi: A = V diag(A_ii) V^T.
// Stops once the off-diagonal mass is below 3e-7 of ||A||_F (fp32 round-off
// level for the small-strain matrices it is applied to, see elastoplastic_fast).
__device__ __forceinline__ void sym_eig3(float A[3][3], float V[3][3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) V[i][j] = (i == j) ? 1.0f : 0.0f;
  const float off0 = A[0][1] * A[0][1] + A[0][2] * A[0][2] + A[1][2] * A[1][2];
  const float tol2 = NSF_JACOBI_TOL2 * (A[0][0] * A[0][0] + A[1][1] * A[1][1] + A[2][2] * A[2][2] + 2.0f * off0);
  for (int sweep = 0; sweep < 6; ++sweep) {
    const float off = A[0][1] * A[0][1] + A[0][2] * A[0][2] + A[1][2] * A[1][2];
    if (off <= tol2) break;
    jacobi_pq(A, V, 0, 1);
    jacobi_pq(A, V, 0, 2);
    jacobi_pq(A, V, 1, 2);
  }
}

__device__ __forceinline__ bool polar_newton(const float F[9], float R[9]) {
#pragma unroll
  for (int k = 0; k < 9; ++k) R[k] = F[k];
  for (int it = 0; it < 12; ++it) {
    // cofactor matrix = det(R) R^{-T}
    float c[9];
    c[0] = R[4] * R[8] - R[5] * R[7];
    c[1] = R[5] * R[6] - R[3] * R[8];
    c[2] = R[3] * R[7] - R[4] * R[6];
    c[3] = R[2] * R[7] - R[1] * R[8];
    c[4] = R[0] * R[8] - R[2] * R[6];
    c[5] = R[1] * R[6] - R[0] * R[7];
    c[6] = R[1] * R[5] - R[2] * R[4];
    c[7] = R[2] * R[3] - R[0] * R[5];
    c[8] = R[0] * R[4] - R[1] * R[3];
    const float det = R[0] * c[0] + R[1] * c[1] + R[2] * c[2];
    if (!(det > 1e-12f)) return false;
    // g = det^{-1/3};  R' = (g R + cof/(g det)) / 2
    const float g = exp2f(-log2f(det) * (1.0f / 3.0f));
    const float a = 0.5f * g, b = 0.5f / (g * det);
    float diff = 0.0f;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const float r = a * R[k] + b * c[k];
      diff = fmaxf(diff, fabsf(r - R[k]));
      R[k] = r;
    }
    if (diff < 2e-7f) break;
  }
  return true;
}

// ---------------------------------------------------------------------------
// Eigen-free log-strain models for moderate strains.  All matrices below are
// functions of S = F F^T - I, hence symmetric and mutually commuting, so a
// product is stored by its 6 independent entries (xx, yy, zz, yz, xz, xy).
//   eps = 1/2 log(I + S) = atanh(Y) = Y + Y^3/3 + Y^5/5 + ..., Y = S (2I + S)^-1
// (|Y| <= 0.18 for ||S||_F <= 0.3: five terms leave < 1e-9 relative).  With
// F = V R and V = exp(eps): F_E = exp(eps_E - eps) F and
// tau = 2 mu eps_E + lambda tr(eps_E) I -- the same Hencky model and return
// maps as the eigen path (readings #3-#6), written as matrix
// functions.
struct Sym6 { float xx, yy, zz, yz, xz, xy; };

__device__ __forceinline__ Sym6 sym_mul(const Sym6& A, const Sym6& B) {
  Sym6 C;
  C.xx = fmaf(A.xx, B.xx, fmaf(A.xy, B.xy, A.xz * B.xz));
  C.yy = fmaf(A.xy, B.xy, fmaf(A.yy, B.yy, A.yz * B.yz));
  C.zz = fmaf(A.xz, B.xz, fmaf(A.yz, B.yz, A.zz * B.zz));
  C.yz = fmaf(A.xy, B.xz, fmaf(A.yy, B.yz, A.yz * B.zz));
  C.xz = fmaf(A.xx, B.xz, fmaf(A.xy, B.yz, A.xz * B.zz));
  C.xy = fmaf(A.xx, B.xy, fmaf(A.xy, B.yy, A.xz * B.yz));
  return C;
}

// C = A * B + c I
__device__ __forceinline__ Sym6 sym_mul_add_diag(const Sym6& A, const Sym6& B, float c) {
  Sym6 C = sym_mul(A, B);
  C.xx += c; C.yy += c; C.zz += c;
  return C;
}

__device__ __forceinline__ float sym_fro2(const Sym6& A) {
  return A.xx * A.xx + A.yy * A.yy + A.zz * A.zz + 2.0f * (A.yz * A.yz + A.xz * A.xz + A.xy * A.xy);
}

// C = s (A B) + c I
__device__ __forceinline__ Sym6 sym_mul_scale_add_diag(const Sym6& A, const Sym6& B, float s, float c) {
  const Sym6 M = sym_mul(A, B);
  return Sym6{fmaf(M.xx, s, c), fmaf(M.yy, s, c), fmaf(M.zz, s, c), M.yz * s, M.xz * s, M.xy * s};
}

// exp(A) for ||A||_F = a <= 0.2: Taylor polynomial of degree n in Horner form,
// n the smallest of 2, 3, 4, 6 whose remainder a^(n+1)/(n+1)! (times < 1.01)
// stays below 7e-9 -- under the fp32 resolution of the F_E = exp(A) F it feeds.
// The return-map increments of one substep are small, so n is mostly 2 or 3.
__device__ __forceinline__ Sym6 sym_exp_small(const Sym6& A, float a2) {
  const int n = a2 <= 9e-6f ? 2 : a2 <= 4e-4f ? 3 : a2 <= 3.6e-3f ? 4 : 6;
  // T = I + A/n; T <- I + (A T)/k for k = n-1 .. 1
  const float rn = n == 2 ? 0.5f : n == 3 ? 1.0f / 3.0f : n == 4 ? 0.25f : 1.0f / 6.0f;
  Sym6 T{fmaf(A.xx, rn, 1.0f), fmaf(A.yy, rn, 1.0f), fmaf(A.zz, rn, 1.0f), A.yz * rn, A.xz * rn, A.xy * rn};
#pragma unroll
  for (int k = 5; k >= 1; --k)
    if (k < n) T = sym_mul_scale_add_diag(A, T, 1.0f / (float)k, 1.0f);
  return T;
}

// Returns false (caller falls back to the eigen path) outside the series' range.
__device__ __forceinline__ bool elastoplastic_series(const float Ft[9], const Sym6& S, int model, float mu,
                                                     float lam, float alpha, float tau_Y, float FE[9], float tau[6],
                                                     float& detFE, float* dg_out = nullptr) {
  if (!(sym_fro2(S) <= 0.09f)) return false;
  // Y = S (2I + S)^-1
  const Sym6 M{2.0f + S.xx, 2.0f + S.yy, 2.0f + S.zz, S.yz, S.xz, S.xy};
  const float cxx = M.yy * M.zz - M.yz * M.yz, cyy = M.xx * M.zz - M.xz * M.xz, czz = M.xx * M.yy - M.xy * M.xy;
  const float cyz = M.xy * M.xz - M.xx * M.yz, cxz = M.xy * M.yz - M.yy * M.xz, cxy = M.xz * M.yz - M.zz * M.xy;
  const float rdet = 1.0f / (M.xx * cxx + M.xy * cxy + M.xz * cxz);
  const Sym6 Minv{cxx * rdet, cyy * rdet, czz * rdet, cyz * rdet, cxz * rdet, cxy * rdet};
  const Sym6 Y = sym_mul(S, Minv);
  const Sym6 Y2 = sym_mul(Y, Y);
  // eps = atanh(Y) = Y P, P = sum_{i<=m} Y2^i / (2i+1) (Horner); the remainder
  // ~ y^(2m+3)/(2m+3) stays below 5e-10 with m = 2 (y <= 0.06), 3 (y <= 0.12),
  // 4 (else; y <= 0.3/1.7 inside the range check), y = ||Y||_F
  const float y2 = Y2.xx + Y2.yy + Y2.zz;   // = ||Y||_F^2
  const int m = y2 <= 3.6e-3f ? 2 : y2 <= 1.44e-2f ? 3 : 4;
  const float r2m1 = m == 2 ? 0.2f : m == 3 ? 1.0f / 7.0f : 1.0f / 9.0f;
  const float r2m = m == 2 ? 1.0f / 3.0f : m == 3 ? 0.2f : 1.0f / 7.0f;
  Sym6 Pm{fmaf(Y2.xx, r2m1, r2m), fmaf(Y2.yy, r2m1, r2m), fmaf(Y2.zz, r2m1, r2m), Y2.yz * r2m1, Y2.xz * r2m1,
          Y2.xy * r2m1};
#pragma unroll
  for (int i = 2; i >= 0; --i)
    if (i <= m - 2) Pm = sym_mul_add_diag(Y2, Pm, 1.0f / (float)(2 * i + 1));
  const Sym6 E = sym_mul(Y, Pm);
  const float tr = E.xx + E.yy + E.zz;
  const Sym6 Eh{E.xx - tr * (1.0f / 3.0f), E.yy - tr * (1.0f / 3.0f), E.zz - tr * (1.0f / 3.0f), E.yz, E.xz, E.xy};
  const float nrm = sqrtf(sym_fro2(Eh));
  float dg;
  bool expand = false;
  if (model == 1) {   // Drucker-Prager
    expand = tr > 0.0f;
    dg = nrm + alpha * (3.0f * lam + 2.0f * mu) * tr / (2.0f * mu);
  } else {            // von Mises
    dg = nrm - tau_Y / (2.0f * mu);
  }
  if (dg_out) *dg_out = (model == 2 && dg > 0.0f) ? dg : 0.0f;
  Sym6 Ee = E;   // eps_E
  if (expand || dg > 0.0f) {
    // A = eps_E - eps: -eps (DP tip) or -(dg / |eps_hat|) eps_hat
    Sym6 A;
    if (expand) {
      A = Sym6{-E.xx, -E.yy, -E.zz, -E.yz, -E.xz, -E.xy};
    } else {
      const float k = dg / nrm;
      A = Sym6{-k * Eh.xx, -k * Eh.yy, -k * Eh.zz, -k * Eh.yz, -k * Eh.xz, -k * Eh.xy};
    }
    const float a2 = sym_fro2(A);
    if (!(a2 <= 0.04f)) return false;
    const Sym6 X = sym_exp_small(A, a2);
    const float Xm[9] = {X.xx, X.xy, X.xz, X.xy, X.yy, X.yz, X.xz, X.yz, X.zz};
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        FE[i * 3 + j] = Xm[i * 3 + 0] * Ft[0 * 3 + j] + Xm[i * 3 + 1] * Ft[1 * 3 + j] + Xm[i * 3 + 2] * Ft[2 * 3 + j];
    Ee = Sym6{E.xx + A.xx, E.yy + A.yy, E.zz + A.zz, E.yz + A.yz, E.xz + A.xz, E.xy + A.xy};
    detFE = det3(FE);
  } else {
#pragma unroll
    for (int k = 0; k < 9; ++k) FE[k] = Ft[k];
    detFE = det3(Ft);
  }
  const float lt = lam * (Ee.xx + Ee.yy + Ee.zz);
  tau[0] = 2.0f * mu * Ee.xx + lt;
  tau[1] = 2.0f * mu * Ee.yy + lt;
  tau[2] = 2.0f * mu * Ee.zz + lt;
  tau[3] = 2.0f * mu * Ee.yz;
  tau[4] = 2.0f * mu * Ee.xz;
  tau[5] = 2.0f * mu * Ee.xy;
  return true;
}

__device__ __forceinline__ float elastoplastic_fast(const float Ft[9], int model, float mu, float lam, float alpha,
                                                    float tau_Y, float FE[9], float tau[6], float* dg_out = nullptr) {
  const float J = det3(Ft);
  if (!(J > 1e-6f)) return elastoplastic(Ft, model, mu, lam, alpha, tau_Y, FE, tau, dg_out);
  if (model == 0) {
    float R[9];
    if (!polar_newton(Ft, R)) return elastoplastic(Ft, model, mu, lam, alpha, tau_Y, FE, tau, dg_out);
    float D[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) D[k] = Ft[k] - R[k];
    const float vol = lam * (J - 1.0f) * J;
    float T[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        T[i][j] = 2.0f * mu * (D[i * 3 + 0] * Ft[j * 3 + 0] + D[i * 3 + 1] * Ft[j * 3 + 1] + D[i * 3 + 2] * Ft[j * 3 + 2]);
    tau[0] = T[0][0] + vol;
    tau[1] = T[1][1] + vol;
    tau[2] = T[2][2] + vol;
    tau[3] = 0.5f * (T[1][2] + T[2][1]);
    tau[4] = 0.5f * (T[0][2] + T[2][0]);
    tau[5] = 0.5f * (T[0][1] + T[1][0]);
#pragma unroll
    for (int k = 0; k < 9; ++k) FE[k] = Ft[k];
    return J;
  }
  // S = b - I = F F^T - I, formed as H + H^T + H H^T with H = F - I (exact for
  // F near I) so that small strains keep their relative precision; b shares
  // S's eigenvectors and lambda_i(b) = 1 + lambda_i(S).
  float Hm[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) Hm[k] = Ft[k] - ((k & 3) == 0 ? 1.0f : 0.0f);
  float Bm[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = i; j < 3; ++j) {
      const float s = Hm[i * 3 + j] + Hm[j * 3 + i] +
                      (Hm[i * 3 + 0] * Hm[j * 3 + 0] + Hm[i * 3 + 1] * Hm[j * 3 + 1] + Hm[i * 3 + 2] * Hm[j * 3 + 2]);
      Bm[i][j] = s;
      Bm[j][i] = s;
    }
#if NSF_LOGSTRAIN_SERIES
  {
    float detS;
    const Sym6 S6{Bm[0][0], Bm[1][1], Bm[2][2], Bm[1][2], Bm[0][2], Bm[0][1]};
    if (elastoplastic_series(Ft, S6, model, mu, lam, alpha, tau_Y, FE, tau, detS, dg_out)) return detS;
  }
#endif
  float U[3][3];
  sym_eig3(Bm, U);
  // sigma_i^2 = 1 + lambda_i(S) carries an absolute error ~ eps ||S||, so log sigma
  // loses accuracy as sigma -> 0 (at sigma = 5e-5 the clamp decision of #21 is
  // lost entirely): below sigma = 1/4 the rotation-safe SVD decides instead
  const float kEigMin2 = 0.0625f;
  if (!(1.0f + Bm[0][0] > kEigMin2 && 1.0f + Bm[1][1] > kEigMin2 && 1.0f + Bm[2][2] > kEigMin2))
    return elastoplastic(Ft, model, mu, lam, alpha, tau_Y, FE, tau, dg_out);
  // eps = log sigma = log(lambda)/2
  const float e[3] = {0.5f * log1pf(Bm[0][0]), 0.5f * log1pf(Bm[1][1]), 0.5f * log1pf(Bm[2][2])};
  const float tr = e[0] + e[1] + e[2];
  const float eh[3] = {e[0] - tr * (1.0f / 3.0f), e[1] - tr * (1.0f / 3.0f), e[2] - tr * (1.0f / 3.0f)};
  const float nrm = sqrtf(eh[0] * eh[0] + eh[1] * eh[1] + eh[2] * eh[2]);
  float dg;
  bool expand = false;
  if (model == 1) {
    expand = tr > 0.0f;
    dg = nrm + alpha * (3.0f * lam + 2.0f * mu) * tr / (2.0f * mu);
  } else {
    dg = nrm - tau_Y / (2.0f * mu);
  }
  if (dg_out) *dg_out = (model == 2 && dg > 0.0f) ? dg : 0.0f;
  float le[3];
  bool elastic = false;
  if (expand) {
    le[0] = le[1] = le[2] = 0.0f;
  } else if (dg <= 0.0f) {
    le[0] = e[0]; le[1] = e[1]; le[2] = e[2];
    elastic = true;
  } else {
    const float k = dg / nrm;
    le[0] = e[0] - k * eh[0];
    le[1] = e[1] - k * eh[1];
    le[2] = e[2] - k * eh[2];
  }
  float detFE = J;
  if (elastic) {
#pragma unroll
    for (int k = 0; k < 9; ++k) FE[k] = Ft[k];
  } else {
    // F_E = U diag(Z/sigma) U^T F,  Z/sigma = exp(le - e)
    const float r0 = expf(le[0] - e[0]), r1 = expf(le[1] - e[1]), r2 = expf(le[2] - e[2]);
    float M[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) M[i][j] = U[i][0] * r0 * U[j][0] + U[i][1] * r1 * U[j][1] + U[i][2] * r2 * U[j][2];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        FE[i * 3 + j] = M[i][0] * Ft[0 * 3 + j] + M[i][1] * Ft[1 * 3 + j] + M[i][2] * Ft[2 * 3 + j];
    detFE = J * r0 * r1 * r2;
  }
  const float kLogFloor = -9.210340371976184f;   // log(1e-4)
  const float m0 = fmaxf(le[0], kLogFloor), m1 = fmaxf(le[1], kLogFloor), m2 = fmaxf(le[2], kLogFloor);
  const float sum = m0 + m1 + m2;
  const float d0 = 2.0f * mu * m0 + lam * sum, d1 = 2.0f * mu * m1 + lam * sum, d2 = 2.0f * mu * m2 + lam * sum;
  tau[0] = U[0][0] * U[0][0] * d0 + U[0][1] * U[0][1] * d1 + U[0][2] * U[0][2] * d2;
  tau[1] = U[1][0] * U[1][0] * d0 + U[1][1] * U[1][1] * d1 + U[1][2] * U[1][2] * d2;
  tau[2] = U[2][0] * U[2][0] * d0 + U[2][1] * U[2][1] * d1 + U[2][2] * U[2][2] * d2;
  tau[3] = U[1][0] * U[2][0] * d0 + U[1][1] * U[2][1] * d1 + U[1][2] * U[2][2] * d2;
  tau[4] = U[0][0] * U[2][0] * d0 + U[0][1] * U[2][1] * d1 + U[0][2] * U[2][2] * d2;
  tau[5] = U[0][0] * U[1][0] * d0 + U[0][1] * U[1][1] * d1 + U[0][2] * U[1][2] * d2;
  return detFE;
}

// Elastic stress of a given (admissible) F, used for tau^0 at load (reading #9).
// von Mises with a per-particle yield stress (readings #30-#32):
// the return map with tau_Y^n, then tau_Y^{n+1} = tau_Y^n + 2 mu xi dg - theta dg
// (||eps - proj(eps)||_F = dg for the radial return); with softening (theta > 0)
// tau_Y <= 0 is damage: Lame parameters zero (tau = 0) and no return map.
// tY is read and updated in place; returns det F_E.
__device__ __forceinline__ float vm_hs_update(const float Ft[9], float mu, float lam, float hard_k, float soft,
                                              float& tY, float FE[9], float tau[6]) {
  if (soft > 0.0f && !(tY > 0.0f)) {   // damaged
#pragma unroll
    for (int k = 0; k < 9; ++k) FE[k] = Ft[k];
#pragma unroll
    for (int k = 0; k < 6; ++k) tau[k] = 0.0f;
    tY = 0.0f;
    return det3(Ft);
  }
  float dg = 0.0f;
  const float J = elastoplastic_fast(Ft, 2, mu, lam, 0.0f, tY, FE, tau, &dg);
  float t1 = fmaf(hard_k, dg, tY) - soft * dg;
  t1 = t1 > 0.0f ? t1 : 0.0f;
  if (soft > 0.0f && !(t1 > 0.0f)) {
#pragma unroll
    for (int k = 0; k < 6; ++k) tau[k] = 0.0f;
  }
  tY = t1;
  return J;
}

// Herschel-Bulkley (Yue et al. 2015 with h = 1; reading #39), in the
// principal frame of F_trial = U diag(sigma) V^T (rotation-safe SVD):
//   bbar_i = |J|^(-2/3) sigma_i^2, s = mu dev(bbar), s^trial = ||s||;
//   if s^trial > yield (= sqrt(2/3) sigma_Y):
//     s <- s (s^trial - (s^trial - yield) relax) / s^trial, relax = 1 / (1 + eta / (2 mu dt)),
//     bbar_new = s / mu + I 1 with det(bbar_new) = 1 (Newton on the cubic from the trial
//     mean), F^E = U diag(sqrt(|J|^(2/3) bbar_new)) V^T (J and the rotation kept);
//   tau = kappa/2 (J^2 - 1) I + mu dev(bbar_E) = U diag(.) U^T.
// relax < 0: no return map (the elastic stress of F at load).  Returns det F^E.
__device__ __forceinline__ float hb_update(const float Ft[9], float mu, float kappa, float yield, float relax,
                                           float FE[9], float tau[6]) {
  float U[3][3], V[3][3], s[3];
  svd3(Ft, U, s, V);
  const float J = det3(Ft);   // from F itself: the product of the Jacobi singular values is biased low
  const float aJ = fabsf(J);
  float t[3] = {0.f, 0.f, 0.f};
  bool plastic = false;
  float sg[3] = {s[0], s[1], s[2]};
  if (aJ > 0.0f) {
    const float j23 = cbrtf(aJ * aJ), ij23 = 1.0f / j23;
    float bb[3] = {s[0] * s[0] * ij23, s[1] * s[1] * ij23, s[2] * s[2] * ij23};
    const float mean = (bb[0] + bb[1] + bb[2]) * (1.0f / 3.0f);
    // dev(bbar) from pairwise differences (s_i^2 - s_j^2 = (s_i - s_j)(s_i + s_j)): no
    // cancellation against the mean when the stretches are close
    const float q01 = (s[0] - s[1]) * (s[0] + s[1]), q02 = (s[0] - s[2]) * (s[0] + s[2]),
                q12 = (s[1] - s[2]) * (s[1] + s[2]);
    const float c3 = ij23 * (1.0f / 3.0f);
    float d[3] = {(q01 + q02) * c3, (q12 - q01) * c3, -(q02 + q12) * c3};
    const float st = mu * sqrtf(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    if (relax >= 0.0f && st > yield) {
      plastic = true;
      const float k = (st - (st - yield) * relax) / st;
      d[0] *= k; d[1] *= k; d[2] *= k;
      float I = mean;
#pragma unroll
      for (int it = 0; it < 4; ++it) {   // monotone Newton on prod(d_i + I) = 1
        const float a0 = d[0] + I, a1 = d[1] + I, a2 = d[2] + I;
        I -= (a0 * a1 * a2 - 1.0f) / (a1 * a2 + a0 * a2 + a0 * a1);
      }
      bb[0] = d[0] + I; bb[1] = d[1] + I; bb[2] = d[2] + I;
      sg[0] = sqrtf(j23 * bb[0]);
      sg[1] = sqrtf(j23 * bb[1]);
      sg[2] = J / (sg[0] * sg[1]);   // det F^E = J exactly up to one rounding (isochoric flow)
      // dev(bbar_E) = the relaxed deviator (bbar_E = d + I 1, det 1)
    }
    const float vol = 0.5f * kappa * (J * J - 1.0f);
    t[0] = vol + mu * d[0]; t[1] = vol + mu * d[1]; t[2] = vol + mu * d[2];
  } else {
    t[0] = t[1] = t[2] = -0.5f * kappa;
  }
  if (plastic) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        FE[i * 3 + j] = U[i][0] * sg[0] * V[j][0] + U[i][1] * sg[1] * V[j][1] + U[i][2] * sg[2] * V[j][2];
    // isochoric flow: det F^E = J (the fp32 U, V are orthogonal only to ~1e-7, with a
    // bias that would otherwise drift the volume substep after substep)
    const float c = cbrtf(J / det3(FE));
#pragma unroll
    for (int k = 0; k < 9; ++k) FE[k] *= c;
  } else {
#pragma unroll
    for (int k = 0; k < 9; ++k) FE[k] = Ft[k];
  }
  tau[0] = U[0][0] * U[0][0] * t[0] + U[0][1] * U[0][1] * t[1] + U[0][2] * U[0][2] * t[2];
  tau[1] = U[1][0] * U[1][0] * t[0] + U[1][1] * U[1][1] * t[1] + U[1][2] * U[1][2] * t[2];
  tau[2] = U[2][0] * U[2][0] * t[0] + U[2][1] * U[2][1] * t[1] + U[2][2] * U[2][2] * t[2];
  tau[3] = U[1][0] * U[2][0] * t[0] + U[1][1] * U[2][1] * t[1] + U[1][2] * U[2][2] * t[2];
  tau[4] = U[0][0] * U[2][0] * t[0] + U[0][1] * U[2][1] * t[1] + U[0][2] * U[2][2] * t[2];
  tau[5] = U[0][0] * U[1][0] * t[0] + U[0][1] * U[1][1] * t[1] + U[0][2] * U[1][2] * t[2];
  return J;
}

__device__ __forceinline__ void elastic_tau(const float F[9], int model, float mu, float lam, float tau[6],
                                            float kappa = 0.0f) {
  float FE[9];
  if (model == 5) {   // Herschel-Bulkley elasticity of F itself
    hb_update(F, mu, kappa, 0.0f, -1.0f, FE, tau);
    return;
  }
  // FC: same formula; DP/VM: Hencky of F itself (no return map at load)
  if (model == 0) {
    elastoplastic(F, 0, mu, lam, 0.0f, 0.0f, FE, tau);
  } else {
    // tau_Y = +inf -> von Mises never yields -> pure Hencky
    elastoplastic(F, 2, mu, lam, 0.0f, INFINITY, FE, tau);
  }
}

}  // namespace nsf
