// mpm_common.cuh -- MLS-MPM device helpers shared by the nvcc-compiled kernels
// (kernels.cu) and the NVRTC-specialised step kernels (step_kernels.cuh).
//
// Grid geometry: the grid is tiled into blocks of 4^3 cells (3D) or 8^2 cells (2D),
// 64 nodes each; a particle belongs to the block of its base cell
// base = floor(x/dx - 1/2) (Hu et al. 2018, cited P:561).  Its 3^d stencil lies in
// the block's (B+2)^d node tile.
#pragma once
#include "qmpm_device.cuh"

namespace qmpm {

constexpr unsigned FULL = 0xffffffffu;

template <int D>
struct Geo;
template <>
struct Geo<3> {
  static constexpr int B = 4;     // cells per block side
  static constexpr int LB = 2;    // log2(B)
  static constexpr int T = 6;     // tile side (nodes): B + 2
  static constexpr int TN = 216;  // tile nodes
};
template <>
struct Geo<2> {
  static constexpr int B = 8;
  static constexpr int LB = 3;
  static constexpr int T = 10;
  static constexpr int TN = 100;
};

template <int D, int MAT>
struct NS {
  static constexpr int value = 2 * D + (MAT == 1 ? 1 : D * D) + D * D;
};

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Block ids are z-major in 3D, id = (bz * nbx + bx) * nby + by (y-major in 2D), so a
// slab of z block planes [bz0, bz1) is the contiguous id range [bz0 P, bz1 P),
// P = nbx * nby: after the counting sort, particles that left a rank's slab are the
// sorted ranges below and above it.
// (3D: table-local ids, the table starting at block plane S.tab_bz0)
template <int D>
__device__ __forceinline__ void block_coords(uint32_t b, const SimDev& S, int bc[3]) {
  if (D == 3) {
    bc[1] = (int)(b % (uint32_t)S.nb[1]);
    const uint32_t r = b / (uint32_t)S.nb[1];
    bc[0] = (int)(r % (uint32_t)S.nb[0]);
    bc[2] = (int)(r / (uint32_t)S.nb[0]) + S.tab_bz0;
  } else {
    bc[1] = (int)(b % (uint32_t)S.nb[1]);
    bc[0] = (int)(b / (uint32_t)S.nb[1]);
    bc[2] = 0;
  }
}

template <int D>
__device__ __forceinline__ uint32_t block_id(const int c[3], const SimDev& S) {
  if (D == 3)
    return ((uint32_t)(c[2] - S.tab_bz0) * (uint32_t)S.nb[0] + (uint32_t)c[0]) * (uint32_t)S.nb[1] + (uint32_t)c[1];
  return (uint32_t)c[0] * (uint32_t)S.nb[1] + (uint32_t)c[1];
}

// node-in-block linear index (x-major)
template <int D>
__device__ __forceinline__ uint32_t local_node(const int l[3]) {
  if (D == 3) return (uint32_t)((l[0] * 4 + l[1]) * 4 + l[2]);
  return (uint32_t)(l[0] * 8 + l[1]);
}

// sort key of a particle from its (decoded) position: block id * 64 + the base cell's
// index inside its block (x-major).  The counting sort orders particles by this full
// key, so P2G finds each cell's particles as a contiguous range.
template <int D>
__device__ __forceinline__ uint32_t key_of(const float* x, const SimDev& S) {
  int c[3] = {0, 0, 0}, l[3] = {0, 0, 0};
#pragma unroll
  for (int a = 0; a < D; ++a) {
    float fx;
    bool o;
    const int b = base_fx(x[a], S.inv_dx, S.res[a], fx, o);
    c[a] = b >> Geo<D>::LB;
    l[a] = b & (Geo<D>::B - 1);
  }
  return (block_id<D>(c, S) << 6) | local_node<D>(l);
}

// key_of without the clamp; `oob` set when any axis is out of the domain (the caller
// then recomputes with key_of)
template <int D>
__device__ __forceinline__ uint32_t key_of_fast(const float* x, const SimDev& S, bool& oob) {
  int c[3] = {0, 0, 0}, l[3] = {0, 0, 0};
#pragma unroll
  for (int a = 0; a < D; ++a) {
    float fx;
    const int b = base_fx_fast(x[a], S.inv_dx, S.res[a], fx, oob);
    c[a] = b >> Geo<D>::LB;
    l[a] = b & (Geo<D>::B - 1);
  }
  return (block_id<D>(c, S) << 6) | local_node<D>(l);
}

// sort key from the base cell per axis (block id * 64 + cell in block)
template <int D>
__device__ __forceinline__ uint32_t key_from_base(const int b[3], const SimDev& S) {
  int c[3] = {0, 0, 0}, l[3] = {0, 0, 0};
#pragma unroll
  for (int a = 0; a < D; ++a) {
    c[a] = b[a] >> Geo<D>::LB;
    l[a] = b[a] & (Geo<D>::B - 1);
  }
  return (block_id<D>(c, S) << 6) | local_node<D>(l);
}

// z block plane of a full sort key (3D)
__device__ __forceinline__ int key_bz(uint32_t key, const SimDev& S) {
  return (int)((key >> 6) / ((uint32_t)S.nb[0] * (uint32_t)S.nb[1])) + S.tab_bz0;
}

// block plane bz of a particle relative to this rank's slab: 0 owned, -1 / +1 it left
// downwards / upwards, 2 it jumped further (an error: CFL keeps migration to one hop)
__device__ __forceinline__ int slab_side(int bz, const SimDev& S) {
  if (bz >= S.slab_bz0 && bz < S.slab_bz1) return 0;
  if (bz == S.slab_bz0 - 1 && S.slab_lo) return -1;
  if (bz == S.slab_bz1 && S.slab_hi) return 1;
  return 2;
}

// tile node t -> (global node coordinates) for a block with origin org
template <int D>
__device__ __forceinline__ void tile_node(int t, const int org[3], int node[3]) {
  using G = Geo<D>;
  if (D == 3) {
    node[2] = org[2] + t % G::T;
    node[1] = org[1] + (t / G::T) % G::T;
    node[0] = org[0] + t / (G::T * G::T);
  } else {
    node[1] = org[1] + t % G::T;
    node[0] = org[0] + t / G::T;
    node[2] = 0;
  }
}

// a harmless particle for the idle lanes of a partial warp (never stored)
template <int D, int MAT>
__device__ __forceinline__ void benign_state(float* s, const int org[3], float dx) {
  constexpr int NSV = NS<D, MAT>::value;
#pragma unroll
  for (int i = 0; i < NSV; ++i) s[i] = 0.0f;
#pragma unroll
  for (int a = 0; a < D; ++a) s[a] = (org[a] + 1.0f) * dx;
  if (MAT == 1) {
    s[2 * D] = 1.0f;
  } else {
#pragma unroll
    for (int a = 0; a < D; ++a) s[2 * D + a * D + a] = 1.0f;
  }
}

#ifndef QMPM_AB_VSQRT
#define QMPM_AB_VSQRT 1  // 3D fixed corotated through B - sqrt(B) instead of the Newton polar
#endif

// (F - R) F^T of the polar decomposition F = R S (det F > 0), in 3D without R:
// R F^T = R S R^T = V = sqrt(B), B = F F^T, so (F - R) F^T = B - V.  With E = B - I and
// mu_i its eigenvalues (closed form, trigonometric), sigma_i = sqrt(1 + mu_i), the
// matrix function G = V - I = g(E), g(mu) = sqrt(1 + mu) - 1, is the quadratic that
// interpolates g at the mu_i, G = a0 I + a1 E + a2 E^2, from the divided differences
//   g[mu_i, mu_j] = 1 / (sigma_i + sigma_j),
//   g[mu_1, mu_2, mu_3] = -1 / ((sigma_1 + sigma_2)(sigma_2 + sigma_3)(sigma_3 + sigma_1)),
// closed forms without cancellation, so B - V = E - G keeps its relative accuracy when
// the strain is small (no 1 - 1 differences anywhere).  Out: K = (F - R) F^T symmetric
// as {00, 11, 22, 01, 02, 12}.
__device__ __forceinline__ float sqrt_apx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_apx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// arccos on [-1, 1] to ~2e-8 absolute: acos(x) = sqrt(1 - x) P(x) for x >= 0 (the
// degree-7 fit of Abramowitz & Stegun 4.4.46), acos(-x) = pi - acos(x)
__device__ __forceinline__ float acos_apx(float r) {
  const float x = fabsf(r);
  float p = -0.0012624911f;
  p = fmaf(p, x, 0.0066700901f);
  p = fmaf(p, x, -0.0170881256f);
  p = fmaf(p, x, 0.0308918810f);
  p = fmaf(p, x, -0.0501743046f);
  p = fmaf(p, x, 0.0889789874f);
  p = fmaf(p, x, -0.2145988016f);
  p = fmaf(p, x, 1.5707963050f);
  const float a = sqrt_apx(1.0f - x) * p;
  return r < 0.0f ? 3.14159265f - a : a;
}

__device__ __forceinline__ void corot_kernel3(const float F[9], float K[6]) {
  float E[6];
  E[0] = fmaf(F[0], F[0], fmaf(F[1], F[1], fmaf(F[2], F[2], -1.0f)));
  E[1] = fmaf(F[3], F[3], fmaf(F[4], F[4], fmaf(F[5], F[5], -1.0f)));
  E[2] = fmaf(F[6], F[6], fmaf(F[7], F[7], fmaf(F[8], F[8], -1.0f)));
  E[3] = fmaf(F[0], F[3], fmaf(F[1], F[4], F[2] * F[5]));
  E[4] = fmaf(F[0], F[6], fmaf(F[1], F[7], F[2] * F[8]));
  E[5] = fmaf(F[3], F[6], fmaf(F[4], F[7], F[5] * F[8]));
  const float q = (E[0] + E[1] + E[2]) * (1.0f / 3.0f);
  const float d0 = E[0] - q, d1 = E[1] - q, d2 = E[2] - q;
  const float off2 = fmaf(E[3], E[3], fmaf(E[4], E[4], E[5] * E[5]));
  const float p2 = fmaf(d0, d0, fmaf(d1, d1, fmaf(d2, d2, 2.0f * off2))) * (1.0f / 6.0f);
  float m1 = q, m2 = q, m3 = q;
  if (p2 > 1e-20f) {  // (below: eigenvalue spread under fp32 resolution, all = q)
    const float ip = rsqrtf(p2), p = p2 * ip;
    const float detD = d0 * fmaf(d1, d2, -E[5] * E[5]) - E[3] * fmaf(E[3], d2, -E[5] * E[4]) +
                       E[4] * fmaf(E[3], E[5], -d1 * E[4]);
    const float r = fminf(fmaxf(((detD * ip) * ip) * ip * 0.5f, -1.0f), 1.0f);
    const float phi = acos_apx(r) * (1.0f / 3.0f);
    m1 = fmaf(2.0f * p, __cosf(phi), q);
    m3 = fmaf(2.0f * p, __cosf(phi + 2.09439510f), q);
    m2 = 3.0f * q - m1 - m3;
  }
  const float s1 = sqrt_apx(fmaxf(1.0f + m1, 1e-30f)), s2 = sqrt_apx(fmaxf(1.0f + m2, 1e-30f)),
              s3 = sqrt_apx(fmaxf(1.0f + m3, 1e-30f));
  const float s12 = s1 + s2, s23 = s2 + s3, s31 = s3 + s1;
  const float i12 = rcp_apx(s12);
  const float a2 = -rcp_apx(s12 * s23 * s31);
  const float a1 = fmaf(-(m1 + m2), a2, i12);
  const float a0 = fmaf(m1 * m2, a2, m1 * (rcp_apx(1.0f + s1) - i12));
  // E^2 (symmetric)
  const float Q[6] = {fmaf(E[0], E[0], fmaf(E[3], E[3], E[4] * E[4])), fmaf(E[1], E[1], fmaf(E[3], E[3], E[5] * E[5])),
                      fmaf(E[2], E[2], fmaf(E[4], E[4], E[5] * E[5])),
                      fmaf(E[0], E[3], fmaf(E[3], E[1], E[4] * E[5])),
                      fmaf(E[0], E[4], fmaf(E[3], E[5], E[4] * E[2])),
                      fmaf(E[3], E[4], fmaf(E[1], E[5], E[5] * E[2]))};
#pragma unroll
  for (int i = 0; i < 6; ++i) K[i] = E[i] - fmaf(a2, Q[i], (i < 3 ? a0 : 0.0f) + a1 * E[i]);
}

// the stress part of the affine momentum, -dt V_p 4/dx^2 P(F)F^T (Hu et al. 2018;
// DESIGN.md §2 Q15), from the decoded F (elastic) or J (fluid, diagonal only)
template <int D, int MAT>
__device__ __forceinline__ void stress_of(const float* s, const SimDev& S, float st[D * D]) {
  if (MAT == 1) {
    const float p = S.stress_scale * S.E * (s[2 * D] - 1.0f);
#pragma unroll
    for (int i = 0; i < D * D; ++i) st[i] = 0.0f;
#pragma unroll
    for (int a = 0; a < D; ++a) st[a * D + a] = p;
  } else if (D == 3 && QMPM_AB_VSQRT) {
    const float* F = s + 2 * D;
    float K[6];
    corot_kernel3(F, K);
    const float J = F[0] * (F[4] * F[8] - F[5] * F[7]) - F[1] * (F[3] * F[8] - F[5] * F[6]) +
                    F[2] * (F[3] * F[7] - F[4] * F[6]);
    const float two_mu = 2.0f * S.mu * S.stress_scale;
    const float diag = S.lambda * (J - 1.0f) * J * S.stress_scale;
    constexpr int SI[3][3] = {{0, 3, 4}, {3, 1, 5}, {4, 5, 2}};
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) st[a * D + b] = fmaf(two_mu, K[SI[a][b]], a == b ? diag : 0.0f);
  } else {
    const float* F = s + 2 * D;
    float R[D * D];
    float J;
    if (D == 3) {
      polar3(F, R);
      J = F[0] * (F[4] * F[8] - F[5] * F[7]) - F[1] * (F[3] * F[8] - F[5] * F[6]) +
          F[2] * (F[3] * F[7] - F[4] * F[6]);
    } else {
      polar2(F, R);
      J = F[0] * F[3] - F[1] * F[2];
    }
    const float two_mu = 2.0f * S.mu * S.stress_scale;
    const float diag = S.lambda * (J - 1.0f) * J * S.stress_scale;
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) {
        float acc = 0.0f;
#pragma unroll
        for (int k = 0; k < D; ++k) acc += (F[a * D + k] - R[a * D + k]) * F[b * D + k];
        st[a * D + b] = two_mu * acc + (a == b ? diag : 0.0f);
      }
  }
}

}  // namespace qmpm
