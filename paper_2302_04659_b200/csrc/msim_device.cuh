// Device-side building blocks of the B200 MLS-MPM substep: fp32 3-vector /
// 3x3 math, the constitutive model on the displacement gradient, SDF
// primitives and the penalty law. Reference semantics are cited per function
// (paths relative to /root/reference/proj/include/msim/).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

// Rarely executed device paths (errors, volume SDF lookups, the global-memory
// scatter fallback). Inlined: out of line (variant build MSIM_OUTLINE_COLD)
// the k_particles launch took 1.24 ms instead of 0.98 ms (config D, 256 envs):
// a call site constrains the caller's register allocation even when cold.
#ifdef MSIM_OUTLINE_COLD
#define MSIM_COLD __noinline__
#else
#define MSIM_COLD __forceinline__
#endif

namespace msim_dev {

// Programmatic dependent launch (msim_internal.h launch_pdl): wait for the
// predecessor grid (complete, writes visible); allow the successor grid to be
// scheduled. Both are no-ops in a kernel launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---------------------------------------------------------------------------
// Small fp32 vector / matrix helpers (row-major 3x3 in registers).

struct f3 {
  float x, y, z;
};
__host__ __device__ __forceinline__ f3 mk3(float x, float y, float z) { return f3{x, y, z}; }
__host__ __device__ __forceinline__ f3 operator+(f3 a, f3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__host__ __device__ __forceinline__ f3 operator-(f3 a, f3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__host__ __device__ __forceinline__ f3 operator*(float s, f3 a) { return {s * a.x, s * a.y, s * a.z}; }
__host__ __device__ __forceinline__ float dot(f3 a, f3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__host__ __device__ __forceinline__ f3 cross(f3 a, f3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__host__ __device__ __forceinline__ float norm(f3 a) { return sqrtf(dot(a, a)); }
__host__ __device__ __forceinline__ float comp(f3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }

// y = M x, M row-major float[9]
__host__ __device__ __forceinline__ f3 matvec(const float* M, f3 x) {
  return {M[0] * x.x + M[1] * x.y + M[2] * x.z, M[3] * x.x + M[4] * x.y + M[5] * x.z,
          M[6] * x.x + M[7] * x.y + M[8] * x.z};
}
__host__ __device__ __forceinline__ f3 matTvec(const float* M, f3 x) {
  return {M[0] * x.x + M[3] * x.y + M[6] * x.z, M[1] * x.x + M[4] * x.y + M[7] * x.z,
          M[2] * x.x + M[5] * x.y + M[8] * x.z};
}

// ---------------------------------------------------------------------------
// Symmetric 3x3 eigen-decomposition by cyclic Jacobi, fp32.
// A = {a00, a11, a22, a01, a02, a12}; on return d = eigenvalues and V
// (row-major, columns = eigenvectors) with A = V diag(d) V^T.
// The solver runs on E = F F^T - I, whose entries are the (small) strains,
// so eigenvalues carry fp32 precision RELATIVE to the strain rather than
// relative to 1 (the cancellation that makes fp32 log(sigma) lossy).
__device__ __forceinline__ void jacobi_rotate(float& app, float& aqq, float& apq, float& arp,
                                              float& arq, float* V, int p, int q) {
  // tan of the rotation angle without the theta division:
  //   t = sign(tau) * 2 apq / (|tau| + sqrt(tau^2 + 4 apq^2)),  tau = aqq - app, sign(0) = +1
  // (the smaller root, |t| <= 1). MUFU reciprocal / rsqrt are enough: the
  // rotation stays orthogonal to rounding because c = rsqrt(1 + t^2), s = t c,
  // and any residual off-diagonal is removed by the next sweep.
  if (fabsf(apq) < 1e-18f) return;  // keeps 4 apq^2 a normal float
  const float tau = aqq - app;
  const float r2 = fmaf(tau, tau, 4.0f * apq * apq);
  const float r = r2 * rsqrtf(r2);  // MUFU sqrt approximation, r2 > 0
  const float t = __fdividef((tau < 0.0f ? -2.0f : 2.0f) * apq, fabsf(tau) + r);
  const float c = rsqrtf(fmaf(t, t, 1.0f));
  const float s = t * c;
  app -= t * apq;
  aqq += t * apq;
  apq = 0.0f;
  float rp = arp, rq = arq;
  arp = c * rp - s * rq;
  arq = s * rp + c * rq;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    float vp = V[r * 3 + p], vq = V[r * 3 + q];
    V[r * 3 + p] = c * vp - s * vq;
    V[r * 3 + q] = s * vp + c * vq;
  }
}

__device__ __forceinline__ void sym_eigen3(float a00, float a11, float a22, float a01, float a02,
                                           float a12, float* d, float* V) {
#pragma unroll
  for (int i = 0; i < 9; ++i) V[i] = (i % 4 == 0) ? 1.0f : 0.0f;
  // Stop once the off-diagonal is at fp32 rounding level of the matrix scale
  // (a tighter bound is never reached in fp32 and would force every sweep);
  // cyclic Jacobi converges quadratically, 3-4 sweeps in practice.
#pragma unroll 1
  for (int sweep = 0; sweep < 6; ++sweep) {
    float off = fabsf(a01) + fabsf(a02) + fabsf(a12);
    float scale = fabsf(a00) + fabsf(a11) + fabsf(a22) + off;
    if (off <= 2.5e-7f * scale || off == 0.0f) break;
    jacobi_rotate(a00, a11, a01, a02, a12, V, 0, 1);  // (p,q)=(0,1), r=2: a_rp=a02, a_rq=a12
    jacobi_rotate(a00, a22, a02, a01, a12, V, 0, 2);  // (0,2), r=1: a_rp=a01, a_rq=a12 (=a21)
    jacobi_rotate(a11, a22, a12, a01, a02, V, 1, 2);  // (1,2), r=0: a_rp=a10, a_rq=a20
  }
  d[0] = a00;
  d[1] = a11;
  d[2] = a22;
}

// ---------------------------------------------------------------------------
// Constitutive model on the displacement gradient G = F - I (stored state).

// model ids = MSIM_MODEL_* (include/msim_gpu.h)
constexpr int kModelVonMises = 0, kModelFixedCorotated = 1, kModelDruckerPrager = 2, kModelFluid = 3;

struct MatParams {
  float two_mu;       // 2 mu
  float lambda;
  float yield_thr;    // sqrt(2/3) * yield_stress (von Mises)
  float density;
  int model;
  float dp_alpha;     // Drucker-Prager cone: sqrt(2/3) 2 sin(phi) / (3 - sin(phi))
  float dp_k;         // (3 lambda + 2 mu) / (2 mu) * dp_alpha
  float bulk;         // fluid bulk modulus E / (3 (1 - 2 nu))
};

// det(I + G) without forming I + G (exact expansion).
__device__ __forceinline__ float det_I_plus(const float* G) {
  float tr = G[0] + G[4] + G[8];
  float m2 = (G[0] * G[4] - G[1] * G[3]) + (G[0] * G[8] - G[2] * G[6]) + (G[4] * G[8] - G[5] * G[7]);
  float dg = G[0] * (G[4] * G[8] - G[5] * G[7]) - G[1] * (G[3] * G[8] - G[5] * G[6]) +
             G[2] * (G[3] * G[7] - G[4] * G[6]);
  return 1.0f + tr + m2 + dg;
}

// Symmetric 3x3 {a00, a11, a22, a01, a02, a12}.
struct Sym {
  float a00, a11, a22, a01, a02, a12;
};
// A B for symmetric A, B that commute (polynomials of one matrix): the
// product is symmetric, so only its upper triangle is formed (18 FMA).
__device__ __forceinline__ Sym sym_mul(const Sym& A, const Sym& B) {
  return {A.a00 * B.a00 + A.a01 * B.a01 + A.a02 * B.a02, A.a01 * B.a01 + A.a11 * B.a11 + A.a12 * B.a12,
          A.a02 * B.a02 + A.a12 * B.a12 + A.a22 * B.a22, A.a00 * B.a01 + A.a01 * B.a11 + A.a02 * B.a12,
          A.a00 * B.a02 + A.a01 * B.a12 + A.a02 * B.a22, A.a01 * B.a02 + A.a11 * B.a12 + A.a12 * B.a22};
}
// A B + c I
__device__ __forceinline__ Sym sym_mul_add_id(const Sym& A, const Sym& B, float c) {
  Sym r = sym_mul(A, B);
  r.a00 += c;
  r.a11 += c;
  r.a22 += c;
  return r;
}
__device__ __forceinline__ Sym sym_scale_add_id(const Sym& A, float s, float c) {
  return {s * A.a00 + c, s * A.a11 + c, s * A.a22 + c, s * A.a01, s * A.a02, s * A.a12};
}
__device__ __forceinline__ float sym_norm2(const Sym& A) {
  return A.a00 * A.a00 + A.a11 * A.a11 + A.a22 * A.a22 + 2.0f * (A.a01 * A.a01 + A.a02 * A.a02 + A.a12 * A.a12);
}

// E = F F^T - I = G + G^T + G G^T
__device__ __forceinline__ Sym left_strain(const float* G) {
  return {2.0f * G[0] + (G[0] * G[0] + G[1] * G[1] + G[2] * G[2]),
          2.0f * G[4] + (G[3] * G[3] + G[4] * G[4] + G[5] * G[5]),
          2.0f * G[8] + (G[6] * G[6] + G[7] * G[7] + G[8] * G[8]),
          G[1] + G[3] + (G[0] * G[3] + G[1] * G[4] + G[2] * G[5]),
          G[2] + G[6] + (G[0] * G[6] + G[1] * G[7] + G[2] * G[8]),
          G[5] + G[7] + (G[3] * G[6] + G[4] * G[7] + G[5] * G[8])};
}

// Left principal frame of F = I + G: U (columns) and Hencky strains
// eps_i = log(sigma_i) = 0.5*log1p(e_i), e = eig(F F^T - I).
__device__ __forceinline__ void hencky_frame(const float* G, float* U, float* eps) {
  const Sym E = left_strain(G);
  float d[3];
#ifdef MSIM_ABLATE_EIGEN  // profiling-only build: frame = identity (wrong physics)
  d[0] = E.a00; d[1] = E.a11; d[2] = E.a22;
  for (int i = 0; i < 9; ++i) U[i] = (i % 4 == 0) ? 1.0f : 0.0f;
#else
  sym_eigen3(E.a00, E.a11, E.a22, E.a01, E.a02, E.a12, d, U);
#endif
#pragma unroll
  for (int i = 0; i < 3; ++i) eps[i] = 0.5f * log1pf(fmaxf(d[i], -0.99999994f));
}

// S = U diag(s) U^T  (symmetric, row-major out)
__device__ __forceinline__ void sym_from_frame(const float* U, const float* s, float* S) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = r; c < 3; ++c) {
      float v = U[r * 3 + 0] * s[0] * U[c * 3 + 0] + U[r * 3 + 1] * s[1] * U[c * 3 + 1] +
                U[r * 3 + 2] * s[2] * U[c * 3 + 2];
      S[r * 3 + c] = v;
      S[c * 3 + r] = v;
    }
}

// Large-strain path of hencky_strain: the principal frame by cyclic Jacobi.
// (Inlined: as a call it cost 60 % more kernel time.)
__device__ __forceinline__ Sym hencky_strain_jacobi(const float* G) {
  float U[9], e[3], S[9];
  hencky_frame(G, U, e);
  sym_from_frame(U, e, S);
  return {S[0], S[4], S[8], S[1], S[2], S[5]};
}

// Hencky strain TENSOR eps = 0.5 log(F F^T) = 0.5 log1p(E) in the spatial
// frame, i.e. U diag(log sigma) U^T, as a matrix function instead of an
// eigen-decomposition: with Z = E (2I + E)^-1 (eigenvalues z = e / (2 + e)),
//   0.5 log1p(e) = atanh(z) = z + z^3/3 + z^5/5 + ...,
// summed to z^11 by Horner in Z^2. Every factor is a polynomial in E, so all
// products commute and stay symmetric. For ||Z||_F <= 1/4 the truncation is
// below 2e-9 absolute (strains of |e| <~ 0.6, i.e. every elastic state of the
// clays, whose yield caps the deviatoric strain at 0.04-0.2); larger strains
// take the cyclic-Jacobi frame. Same function of F as the reference's
// SVD-based log(sigma) (mpm.hpp:152-161), to fp32 rounding relative to the strain.
__device__ __forceinline__ Sym hencky_strain(const float* G) {
  const Sym E = left_strain(G);
  const Sym B = {2.0f + E.a00, 2.0f + E.a11, 2.0f + E.a22, E.a01, E.a02, E.a12};
  const Sym Cf = {B.a11 * B.a22 - B.a12 * B.a12, B.a00 * B.a22 - B.a02 * B.a02, B.a00 * B.a11 - B.a01 * B.a01,
                  B.a02 * B.a12 - B.a01 * B.a22, B.a01 * B.a12 - B.a02 * B.a11, B.a01 * B.a02 - B.a00 * B.a12};
  const float inv_det = 1.0f / (B.a00 * Cf.a00 + B.a01 * Cf.a01 + B.a02 * Cf.a02);  // det B >= 1
  Sym Z = sym_mul(E, Cf);
  Z = sym_scale_add_id(Z, inv_det, 0.0f);
  const float nz2 = sym_norm2(Z);
#ifndef MSIM_ABLATE_EIGEN
  if (nz2 <= 0.0625f) {
#endif
    const Sym W = sym_mul(Z, Z);
    // |Z|_F <= 0.03 (the elastic strains of the firm clays): Z^9/9 and Z^11/11
    // are below 3e-15 and are dropped
    Sym q;
    if (nz2 > 9e-4f) {
      q = sym_scale_add_id(W, 1.0f / 11.0f, 1.0f / 9.0f);
      q = sym_mul_add_id(W, q, 1.0f / 7.0f);
      q = sym_mul_add_id(W, q, 1.0f / 5.0f);
    } else {
      q = sym_scale_add_id(W, 1.0f / 7.0f, 1.0f / 5.0f);
    }
    q = sym_mul_add_id(W, q, 1.0f / 3.0f);
    q = sym_mul_add_id(W, q, 1.0f);
    return sym_mul(Z, q);
#ifndef MSIM_ABLATE_EIGEN
  }
  return hencky_strain_jacobi(G);
#endif
}

// expm1 of a symmetric matrix: Taylor to M^7 / 7! on M / 2^s with
// ||M / 2^s||_F <= 1/4, then s doublings X <- X (2I + X), i.e.
// exp(2A) - I = (exp(A) - I)(exp(A) + I): no cancellation against I.
__device__ __forceinline__ Sym sym_expm1(Sym M) {
  const float n2 = sym_norm2(M);
  int s = 0;
  if (n2 > 0.0625f) {
    s = (int)ceilf(0.5f * log2f(n2 * 16.0f));
    const float sc = exp2f((float)-s);
    M = sym_scale_add_id(M, sc, 0.0f);
  }
  Sym q = sym_scale_add_id(M, 1.0f / 5040.0f, 1.0f / 720.0f);
  q = sym_mul_add_id(M, q, 1.0f / 120.0f);
  q = sym_mul_add_id(M, q, 1.0f / 24.0f);
  q = sym_mul_add_id(M, q, 1.0f / 6.0f);
  q = sym_mul_add_id(M, q, 0.5f);
  q = sym_mul_add_id(M, q, 1.0f);
  Sym X = sym_mul(M, q);
  for (int i = 0; i < s; ++i) {
    const Sym X2 = sym_mul(X, X);
    X = {2.0f * X.a00 + X2.a00, 2.0f * X.a11 + X2.a11, 2.0f * X.a22 + X2.a22,
         2.0f * X.a01 + X2.a01, 2.0f * X.a02 + X2.a02, 2.0f * X.a12 + X2.a12};
  }
  return X;
}

// Kirchhoff stress tau = 2 mu eps + lambda tr(eps) I (mpm.hpp:152-161: the
// principal-frame formula U diag(2 mu eps_i + lambda tr) U^T as a tensor).
__device__ __forceinline__ void kirchhoff_from_strain(const Sym& eps, const MatParams& m, float* tau) {
  const float lt = m.lambda * (eps.a00 + eps.a11 + eps.a22);
  tau[0] = m.two_mu * eps.a00 + lt;
  tau[4] = m.two_mu * eps.a11 + lt;
  tau[8] = m.two_mu * eps.a22 + lt;
  tau[1] = tau[3] = m.two_mu * eps.a01;
  tau[2] = tau[6] = m.two_mu * eps.a02;
  tau[5] = tau[7] = m.two_mu * eps.a12;
}

// Von Mises radial return (mpm.hpp:166-181) on the strain tensor: with
// dev = eps - tr(eps)/3 I and k = thr / (2 mu |dev|) < 1 the projected
// strain is eps + (k - 1) dev, and F' = exp((k - 1) dev) F (the reference's
// U diag(sigma') V^T), applied to G in place as G' = G + X + X G with
// X = expm1((k - 1) dev). eps is updated so the caller forms the next
// Kirchhoff stress without another decomposition. Returns true if yielded.
__device__ __forceinline__ bool von_mises_project_strain(float* G, Sym& eps, const MatParams& m) {
  const float mean = (eps.a00 + eps.a11 + eps.a22) * (1.0f / 3.0f);
  const Sym dev = {eps.a00 - mean, eps.a11 - mean, eps.a22 - mean, eps.a01, eps.a02, eps.a12};
  const float sdn = m.two_mu * sqrtf(sym_norm2(dev));
  if (sdn <= m.yield_thr) return false;
  const float km1 = m.yield_thr / sdn - 1.0f;
  const Sym M = sym_scale_add_id(dev, km1, 0.0f);
  eps = {eps.a00 + M.a00, eps.a11 + M.a11, eps.a22 + M.a22, eps.a01 + M.a01, eps.a02 + M.a02, eps.a12 + M.a12};
  const Sym X = sym_expm1(M);
  const float Xm[9] = {X.a00, X.a01, X.a02, X.a01, X.a11, X.a12, X.a02, X.a12, X.a22};
  float Gn[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      Gn[r * 3 + c] = G[r * 3 + c] + Xm[r * 3 + c] + Xm[r * 3 + 0] * G[0 * 3 + c] + Xm[r * 3 + 1] * G[1 * 3 + c] +
                      Xm[r * 3 + 2] * G[2 * 3 + c];
#pragma unroll
  for (int i = 0; i < 9; ++i) G[i] = Gn[i];
  return true;
}

// G' = G + X + X G (F' = (I + X) F) for a symmetric X
__device__ __forceinline__ void left_update(float* G, const Sym& X) {
  const float Xm[9] = {X.a00, X.a01, X.a02, X.a01, X.a11, X.a12, X.a02, X.a12, X.a22};
  float Gn[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      Gn[r * 3 + c] = G[r * 3 + c] + Xm[r * 3 + c] + Xm[r * 3 + 0] * G[0 * 3 + c] + Xm[r * 3 + 1] * G[1 * 3 + c] +
                      Xm[r * 3 + 2] * G[2 * 3 + c];
#pragma unroll
  for (int i = 0; i < 9; ++i) G[i] = Gn[i];
}

// ---- the north_star's other materials (oracle: msim_oracle.hpp) ----

// Drucker-Prager sand (Klar et al. 2016) on the Hencky strain tensor: tension
// (or a purely volumetric strain) projects to the cone tip (eps = 0, F = R),
// otherwise dgamma = |dev eps| + (3 lambda + 2 mu)/(2 mu) tr(eps) alpha > 0
// moves eps by -dgamma dev / |dev| (F' = exp(d eps) F as in the von Mises map);
// q accumulates the plastic strain.
__device__ __forceinline__ void drucker_prager_project_strain(float* G, Sym& eps, float& q, const MatParams& m) {
  const float tr = eps.a00 + eps.a11 + eps.a22;
  const float mean = tr * (1.0f / 3.0f);
  const Sym dev = {eps.a00 - mean, eps.a11 - mean, eps.a22 - mean, eps.a01, eps.a02, eps.a12};
  const float dn = sqrtf(sym_norm2(dev));
  Sym M;
  if (dn == 0.0f || tr > 0.0f) {
    q += sqrtf(sym_norm2(eps));
    M = sym_scale_add_id(eps, -1.0f, 0.0f);
  } else {
    const float dgamma = dn + m.dp_k * tr;
    if (dgamma <= 0.0f) return;
    q += dgamma;
    M = sym_scale_add_id(dev, -dgamma / dn, 0.0f);
  }
  eps = {eps.a00 + M.a00, eps.a11 + M.a11, eps.a22 + M.a22, eps.a01 + M.a01, eps.a02 + M.a02, eps.a12 + M.a12};
  left_update(G, sym_expm1(M));
}

// sqrt(I + E) - I = V - I (V = sqrt(F F^T), the left stretch) as a matrix
// function of E = F F^T - I: with Z = E (2I + E)^-1, I + E = (I + Z)(I - Z)^-1,
// so sqrt(I + E) = (I + Z)(I - Z^2)^-1/2 and
//   V - I = Z r + (r - I),  r = (I - Z^2)^-1/2 = sum_k C(2k, k) / 4^k Z^2k,
// summed to Z^12 (truncation < 1e-8 for |Z|_F <= 1/4); larger strains take the
// Jacobi frame, where sigma - 1 = e / (1 + sqrt(1 + e)).
__device__ __forceinline__ Sym left_stretch_m1(const float* G) {
  const Sym E = left_strain(G);
  const Sym B = {2.0f + E.a00, 2.0f + E.a11, 2.0f + E.a22, E.a01, E.a02, E.a12};
  const Sym Cf = {B.a11 * B.a22 - B.a12 * B.a12, B.a00 * B.a22 - B.a02 * B.a02, B.a00 * B.a11 - B.a01 * B.a01,
                  B.a02 * B.a12 - B.a01 * B.a22, B.a01 * B.a12 - B.a02 * B.a11, B.a01 * B.a02 - B.a00 * B.a12};
  const float inv_det = 1.0f / (B.a00 * Cf.a00 + B.a01 * Cf.a01 + B.a02 * Cf.a02);
  const Sym Z = sym_scale_add_id(sym_mul(E, Cf), inv_det, 0.0f);
  if (sym_norm2(Z) <= 0.0625f) {
    const Sym W = sym_mul(Z, Z);
    Sym r = sym_scale_add_id(W, 231.0f / 1024.0f, 63.0f / 256.0f);
    r = sym_mul_add_id(W, r, 35.0f / 128.0f);
    r = sym_mul_add_id(W, r, 5.0f / 16.0f);
    r = sym_mul_add_id(W, r, 3.0f / 8.0f);
    r = sym_mul_add_id(W, r, 0.5f);
    const Sym rm1 = sym_mul(W, r);  // r - I
    const Sym zr = sym_mul(Z, sym_scale_add_id(rm1, 1.0f, 1.0f));
    return {zr.a00 + rm1.a00, zr.a11 + rm1.a11, zr.a22 + rm1.a22, zr.a01 + rm1.a01, zr.a02 + rm1.a02,
            zr.a12 + rm1.a12};
  }
  float U[9], d[3], S[9];
  sym_eigen3(E.a00, E.a11, E.a22, E.a01, E.a02, E.a12, d, U);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const float e = fmaxf(d[i], -0.99999994f);
    d[i] = e / (1.0f + sqrtf(1.0f + e));
  }
  sym_from_frame(U, d, S);
  return {S[0], S[4], S[8], S[1], S[2], S[5]};
}

// Kirchhoff stress (as a symmetric tensor) of the stored state for P2G
// (mpm.hpp:235-237), by model: Hencky for von Mises and Drucker-Prager (from
// eps), fixed corotated 2 mu (E - (V - I)) + lambda (J - 1) J I (2 mu (F - R) F^T
// = 2 mu (F F^T - V)), fluid K (J - 1) J I with J = jp.
__device__ __forceinline__ Sym stress_of(int model, const float* G, const Sym& eps, float jp, const MatParams& m) {
  if (model == kModelFixedCorotated) {
    const Sym E = left_strain(G);
    const Sym S = left_stretch_m1(G);
    const float J = det_I_plus(G);
    const float p = m.lambda * (J - 1.0f) * J;
    return {m.two_mu * (E.a00 - S.a00) + p, m.two_mu * (E.a11 - S.a11) + p, m.two_mu * (E.a22 - S.a22) + p,
            m.two_mu * (E.a01 - S.a01), m.two_mu * (E.a02 - S.a02), m.two_mu * (E.a12 - S.a12)};
  }
  if (model == kModelFluid) {
    const float p = m.bulk * (jp - 1.0f) * jp;
    return {p, p, p, 0.f, 0.f, 0.f};
  }
  const float lt = m.lambda * (eps.a00 + eps.a11 + eps.a22);
  return {m.two_mu * eps.a00 + lt, m.two_mu * eps.a11 + lt, m.two_mu * eps.a22 + lt, m.two_mu * eps.a01,
          m.two_mu * eps.a02, m.two_mu * eps.a12};
}

// ---------------------------------------------------------------------------
// Quadratic B-spline weights (mpm.hpp:188-193), fx in [0.5, 1.5).
__device__ __forceinline__ void bspline_w(float fx, float* w) {
  float a = 1.5f - fx, b = fx - 1.0f, c = fx - 0.5f;
  w[0] = 0.5f * a * a;
  w[1] = 0.75f - b * b;
  w[2] = 0.5f * c * c;
}

// ---------------------------------------------------------------------------
// Colliders: one record per shape with its world<->local transform, body
// twist and contact parameters, written by the rigid-step kernel.
struct ShapeDev {
  float Rinv[9];   // world -> shape-local rotation (R^T)
  float tinv[3];   // world -> shape-local translation
  float R[9];      // shape-local -> world rotation (for gradients)
  float com[3];    // owning body's world COM
  float vlin[3];   // body linear velocity
  float vang[3];   // body angular velocity
  float p[4];      // geometry parameters (see msim_shape)
  float friction, k_n, k_t;
  int type;
  int body;        // body index within env (wrench slot)
  int vol_dims[3];
  float vol_origin[3];
  float vol_voxel;
  long long vol_off;  // offset into the volume sample pool
  // Conservative world-space bound of the region where phi can be < r_c:
  // bounded shapes: sphere (bnd[0..2] centre, bnd[3] radius, phi >= |x - c| - r);
  // planes (bplane): phi(x) = bnd[0..2] . x + bnd[3] exactly.
  float bnd[4];
  int bplane;
};

// Can any point of the box [lo, hi] be within r_c of the shape? (the bucket-
// level form of shape_may_touch; same bound, same relative margin)
__device__ __forceinline__ bool shape_may_touch_box(const ShapeDev& sh, f3 lo, f3 hi, float r_c) {
  const f3 c = 0.5f * (lo + hi), e = 0.5f * (hi - lo);
  const float margin = r_c + 1e-4f * (fabsf(c.x) + fabsf(c.y) + fabsf(c.z) + e.x + e.y + e.z + fabsf(sh.bnd[3])) + 1e-6f;
  if (sh.bplane)
    return sh.bnd[0] * c.x + sh.bnd[1] * c.y + sh.bnd[2] * c.z + sh.bnd[3] -
               (fabsf(sh.bnd[0]) * e.x + fabsf(sh.bnd[1]) * e.y + fabsf(sh.bnd[2]) * e.z) < margin;
  const float dx = fmaxf(fabsf(sh.bnd[0] - c.x) - e.x, 0.0f), dy = fmaxf(fabsf(sh.bnd[1] - c.y) - e.y, 0.0f),
              dz = fmaxf(fabsf(sh.bnd[2] - c.z) - e.z, 0.0f);
  return sqrtf(dx * dx + dy * dy + dz * dz) - sh.bnd[3] < margin;
}

// Can the point x be within r_c of the shape (phi < r_c)? A bound test of a
// few FMAs ahead of the SDF: a warp whose particles are all far from a
// collider skips its transform + SDF + gradient. Conservative by a relative
// margin (fp32 rounding of the bound vs the SDF).
__device__ __forceinline__ bool shape_may_touch(const ShapeDev& sh, f3 x, float r_c) {
  const float margin = r_c + 1e-4f * (fabsf(x.x) + fabsf(x.y) + fabsf(x.z) + fabsf(sh.bnd[3])) + 1e-6f;
  if (sh.bplane) return sh.bnd[0] * x.x + sh.bnd[1] * x.y + sh.bnd[2] * x.z + sh.bnd[3] < margin;
  const float dx = x.x - sh.bnd[0], dy = x.y - sh.bnd[1], dz = x.z - sh.bnd[2], rm = sh.bnd[3] + margin;
  return dx * dx + dy * dy + dz * dz < rm * rm;
}

// Trilinear SDF volume lookup with clamping (sdf.hpp:46-62), software
// interpolation (texture filtering would use 8-bit weights).
__device__ __forceinline__ float vol_at(const float* s, const ShapeDev& sh, int i, int j, int k) {
  return s[((long long)k * sh.vol_dims[1] + j) * sh.vol_dims[0] + i];
}
// Out of line: 7 calls per in-band particle would otherwise be inlined into the
// particle kernel (instruction-cache pressure); volumes are the rare shape type.
static __device__ MSIM_COLD float vol_interp(const float* pool, const ShapeDev& sh, f3 p) {
  const float* s = pool + sh.vol_off;
  float inv = 1.0f / sh.vol_voxel;
  f3 local = {(p.x - sh.vol_origin[0]) * inv, (p.y - sh.vol_origin[1]) * inv,
              (p.z - sh.vol_origin[2]) * inv};
  f3 cl = {fminf(fmaxf(local.x, 0.0f), sh.vol_dims[0] - 1.0f),
           fminf(fmaxf(local.y, 0.0f), sh.vol_dims[1] - 1.0f),
           fminf(fmaxf(local.z, 0.0f), sh.vol_dims[2] - 1.0f)};
  float outside = sh.vol_voxel * norm(local - cl);
  int i0 = min((int)cl.x, sh.vol_dims[0] - 2);
  int j0 = min((int)cl.y, sh.vol_dims[1] - 2);
  int k0 = min((int)cl.z, sh.vol_dims[2] - 2);
  float fx = cl.x - i0, fy = cl.y - j0, fz = cl.z - k0;
  float c00 = vol_at(s, sh, i0, j0, k0) * (1 - fx) + vol_at(s, sh, i0 + 1, j0, k0) * fx;
  float c10 = vol_at(s, sh, i0, j0 + 1, k0) * (1 - fx) + vol_at(s, sh, i0 + 1, j0 + 1, k0) * fx;
  float c01 = vol_at(s, sh, i0, j0, k0 + 1) * (1 - fx) + vol_at(s, sh, i0 + 1, j0, k0 + 1) * fx;
  float c11 = vol_at(s, sh, i0, j0 + 1, k0 + 1) * (1 - fx) + vol_at(s, sh, i0 + 1, j0 + 1, k0 + 1) * fx;
  float c0 = c00 * (1 - fy) + c10 * fy;
  float c1 = c01 * (1 - fy) + c11 * fy;
  return c0 * (1 - fz) + c1 * fz + outside;
}

// sdf_local (sdf.hpp:114-135)
__device__ __forceinline__ float sdf_local(const ShapeDev& sh, const float* pool, f3 p) {
  switch (sh.type) {
    case 0:
      return sh.p[0] * p.x + sh.p[1] * p.y + sh.p[2] * p.z - sh.p[3];
    case 1:
      return norm(p) - sh.p[0];
    case 2: {
      f3 q = {fabsf(p.x) - sh.p[0], fabsf(p.y) - sh.p[1], fabsf(p.z) - sh.p[2]};
      f3 qp = {fmaxf(q.x, 0.0f), fmaxf(q.y, 0.0f), fmaxf(q.z, 0.0f)};
      return norm(qp) + fminf(fmaxf(q.x, fmaxf(q.y, q.z)), 0.0f);
    }
    case 3: {
      f3 q = {p.x, p.y, p.z - fminf(fmaxf(p.z, -sh.p[0]), sh.p[0])};
      return norm(q) - sh.p[1];
    }
    default:
      return vol_interp(pool, sh, p);
  }
}

// sdf_gradient_local (sdf.hpp:139-179), tie-breaks toward +x.
__device__ __forceinline__ f3 sdf_grad_local(const ShapeDev& sh, const float* pool, f3 p) {
  const f3 tie = {1.0f, 0.0f, 0.0f};
  switch (sh.type) {
    case 0:
      return {sh.p[0], sh.p[1], sh.p[2]};
    case 1: {
      float n = norm(p);
      return n < 1e-12f ? tie : (1.0f / n) * p;
    }
    case 2: {
      f3 q = {fabsf(p.x) - sh.p[0], fabsf(p.y) - sh.p[1], fabsf(p.z) - sh.p[2]};
      f3 sg = {p.x < 0 ? -1.0f : 1.0f, p.y < 0 ? -1.0f : 1.0f, p.z < 0 ? -1.0f : 1.0f};
      f3 qp = {fmaxf(q.x, 0.0f), fmaxf(q.y, 0.0f), fmaxf(q.z, 0.0f)};
      float out = norm(qp);
      if (out > 1e-12f) return (1.0f / out) * f3{sg.x * qp.x, sg.y * qp.y, sg.z * qp.z};
      int ax = 0;
      float qa = q.x;
      if (q.y > qa) { ax = 1; qa = q.y; }
      if (q.z > qa) { ax = 2; }
      return ax == 0 ? f3{sg.x, 0, 0} : (ax == 1 ? f3{0, sg.y, 0} : f3{0, 0, sg.z});
    }
    case 3: {
      f3 q = {p.x, p.y, p.z - fminf(fmaxf(p.z, -sh.p[0]), sh.p[0])};
      float n = norm(q);
      return n < 1e-12f ? tie : (1.0f / n) * q;
    }
    default: {
      float h = 0.5f * sh.vol_voxel;
      f3 g;
      g.x = (vol_interp(pool, sh, p + f3{h, 0, 0}) - vol_interp(pool, sh, p - f3{h, 0, 0})) / (2 * h);
      g.y = (vol_interp(pool, sh, p + f3{0, h, 0}) - vol_interp(pool, sh, p - f3{0, h, 0})) / (2 * h);
      g.z = (vol_interp(pool, sh, p + f3{0, 0, h}) - vol_interp(pool, sh, p - f3{0, 0, h})) / (2 * h);
      float n = norm(g);
      return n < 1e-12f ? tie : (1.0f / n) * g;
    }
  }
}

// penalty_point_force (coupling.hpp:125-144). Returns false outside the band.
__device__ __forceinline__ bool penalty_force(const ShapeDev& sh, const float* pool, f3 x, f3 v,
                                              float r_c, float c_d, f3& f, float& pen) {
  f3 local = matvec(sh.Rinv, x) + f3{sh.tinv[0], sh.tinv[1], sh.tinv[2]};
  float phi = sdf_local(sh, pool, local);
  if (!(phi < r_c)) return false;
  f3 n = matvec(sh.R, sdf_grad_local(sh, pool, local));
  float depth = r_c - phi;
  f = (sh.k_n * depth) * n;
  f3 com = {sh.com[0], sh.com[1], sh.com[2]};
  f3 vb = f3{sh.vlin[0], sh.vlin[1], sh.vlin[2]} + cross(f3{sh.vang[0], sh.vang[1], sh.vang[2]}, x - com);
  f3 vrel = v - vb;
  float vn = dot(vrel, n);
  f = f + (-c_d * fminf(0.0f, vn)) * n;
  f3 vt = vrel - vn * n;
  float vtn = norm(vt);
  if (vtn > 1e-12f) {
    float cap = fminf(sh.friction * sh.k_n * depth, sh.k_t * vtn);
    f = f - (cap / vtn) * vt;
  }
  pen = fmaxf(0.0f, -phi);
  return true;
}

}  // namespace msim_dev
