// adjoint.cu -- gradient tallies g_h of Algorithm 1 line 12 (Eq. 8,
// P:337; "Gradient Computation") on the GPU: the full-precision (fp32)
// MLS-MPM step (J-fluid or fixed-corotated elastic) on a dense grid, its adjoint, and
// the paper's bisection checkpointing.
// C ABI: include/qadjoint.h.  DESIGN.md §13.
//
// Forward (the same rules as the quantized step's, with fp32 state rows
// [n][ns] = x, v, J | F, C instead of records): P2G into a dense float4 grid (m, P) with
// atomics, grid update (v = P/m + dt g, separating walls), G2P.
// Adjoint of one step, lambda_t = (ds_{t+1}/ds_t)^T lambda_{t+1}, in three kernels:
//   g2p_bwd  gathers v_i, scatters the node adjoints W (lv' + 4/dx lC' (o - fx)) with
//            atomics, keeps the particle's partial (lx, lJ, d/dfx)
//   grid_bwd per node: lP = lv / m, lm = -lv . u / m (zero on wall-clamped components
//            and empty nodes)
//   p2g_bwd  gathers (lm, lP), finishes lambda_t (lv, lC, lJ from the stress, lx through
//            fx) and folds sum_p lambda^2 per scalar into the tallies (double atomics)
// Every derivative is the forward's as written: floor() is constant, clamps have zero
// derivative.  Both materials: the J-fluid (reading Q15) and the fixed-corotated
// elastic, whose stress adjoint differentiates the polar decomposition F = R S through
// skew(R^T dF) = (Omega S + S Omega)/2, Omega = R^T dR (oracle/adjoint.py states it).
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "qadjoint.h"
#include "qmpm_device.cuh"  // polar2 / polar3 (Newton-Higham), as the quantized step

namespace qmpm {
void set_thread_error(const char* msg);  // api.cu
}

struct AdjSim {
  int res[3];
  float dx, inv_dx, dt;
  float g[3];
  float m, k;  // particle mass; fluid stress factor -dt V_p 4/dx^2 E
  float scale, mu, la;  // elastic: -dt V_p 4/dx^2, Lame parameters
  int bound;
};

namespace {

qmpm_status afail(qmpm_status code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  qmpm::set_thread_error(buf);
  return code;
}

#define ACK(x)                                                                                   \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess) return afail(QMPM_ECUDA, "%s: %s", #x, cudaGetErrorString(e_));        \
  } while (0)

template <int D>
struct Stencil {
  int base[3];
  float fx[3], dfx[3];  // fx and d fx / d x (0 where the out-of-domain clamp holds)
  float w[3][3], dw[3][3];
};

// base / fx with the out-of-domain clamp (reading Q14) and the B-spline weights
template <int D>
__device__ __forceinline__ Stencil<D> stencil(const float* x, const AdjSim& S) {
  Stencil<D> st;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const float X = x[a] * S.inv_dx;
    int b = (int)floorf(X - 0.5f);
    bool oob = false;
    if (b < 0) b = 0, oob = true;
    if (b > S.res[a] - 3) b = S.res[a] - 3, oob = true;
    float f = X - (float)b;
    float df = S.inv_dx;
    if (oob && f < 0.5f) f = 0.5f, df = 0.0f;
    if (oob && f > 1.5f) f = 1.5f, df = 0.0f;
    st.base[a] = b;
    st.fx[a] = f;
    st.dfx[a] = df;
    st.w[a][0] = 0.5f * (1.5f - f) * (1.5f - f);
    st.w[a][1] = 0.75f - (f - 1.0f) * (f - 1.0f);
    st.w[a][2] = 0.5f * (f - 0.5f) * (f - 0.5f);
    st.dw[a][0] = -(1.5f - f);
    st.dw[a][1] = -2.0f * (f - 1.0f);
    st.dw[a][2] = f - 0.5f;
  }
  return st;
}

template <int D, bool EL>
constexpr int kNS = 2 * D + (EL ? D * D : 1) + D * D;
template <int D, bool EL>
constexpr int kCO = 2 * D + (EL ? D * D : 1);  // offset of C in a state row
template <int D>
constexpr int kNO = D == 3 ? 27 : 9;

template <int D>
__device__ __forceinline__ void offset_of(int q, int* o) {
  if (D == 3) {
    o[0] = q / 9, o[1] = (q / 3) % 3, o[2] = q % 3;
  } else {
    o[0] = q / 3, o[1] = q % 3, o[2] = 0;
  }
}

template <int D>
__device__ __forceinline__ long long node_of(const Stencil<D>& st, const int* o, const AdjSim& S) {
  const int i = st.base[0] + o[0], j = st.base[1] + o[1], k = D == 3 ? st.base[2] + o[2] : 0;
  return ((long long)i * S.res[1] + j) * (D == 3 ? S.res[2] : 1) + k;
}

template <int D>
__device__ __forceinline__ void weight(const Stencil<D>& st, const int* o, float& W, float* dW) {
  W = 1.0f;
#pragma unroll
  for (int a = 0; a < D; ++a) W *= st.w[a][o[a]];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    float p = st.dw[a][o[a]];
#pragma unroll
    for (int b = 0; b < D; ++b)
      if (b != a) p *= st.w[b][o[b]];
    dW[a] = p;
  }
}

// ---- fixed-corotated stress and its adjoint
template <int D>
__device__ __forceinline__ void cof(const float* F, float* c) {  // cofactor matrix = J F^{-T}
  if (D == 3) {
    c[0] = F[4] * F[8] - F[5] * F[7];
    c[1] = F[5] * F[6] - F[3] * F[8];
    c[2] = F[3] * F[7] - F[4] * F[6];
    c[3] = F[2] * F[7] - F[1] * F[8];
    c[4] = F[0] * F[8] - F[2] * F[6];
    c[5] = F[1] * F[6] - F[0] * F[7];
    c[6] = F[1] * F[5] - F[2] * F[4];
    c[7] = F[2] * F[3] - F[0] * F[5];
    c[8] = F[0] * F[4] - F[1] * F[3];
  } else {
    c[0] = F[3], c[1] = -F[2], c[2] = -F[1], c[3] = F[0];
  }
}

template <int D>
__device__ __forceinline__ void polarD(const float* F, float* R) {
  if constexpr (D == 3)
    qmpm::polar3(F, R);
  else
    qmpm::polar2(F, R);
}

// A_stress = scale (2 mu (F - R) F^T + la (J - 1) J I)
template <int D>
__device__ __forceinline__ void stress_el(const float* F, const AdjSim& S, float (*A)[D]) {
  float R[D * D], c[D * D];
  polarD<D>(F, R);
  cof<D>(F, c);
  float J = 0.0f;
#pragma unroll
  for (int b = 0; b < D; ++b) J += F[b] * c[b];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) {
      float acc = 0.0f;
#pragma unroll
      for (int e = 0; e < D; ++e) acc += (F[a * D + e] - R[a * D + e]) * F[b * D + e];
      A[a][b] = S.scale * (2.0f * S.mu * acc + (a == b ? S.la * (J - 1.0f) * J : 0.0f));
    }
}

// lF += d/dF of <lP, P F^T> (lP = dL/d(P F^T))
template <int D>
__device__ __forceinline__ void stress_el_adj(const float* F, const float (*lP)[D], const AdjSim& S, float* lF) {
  float R[D * D], c[D * D];
  polarD<D>(F, R);
  cof<D>(F, c);
  float J = 0.0f, trP = 0.0f;
#pragma unroll
  for (int b = 0; b < D; ++b) J += F[b] * c[b];
#pragma unroll
  for (int a = 0; a < D; ++a) trP += lP[a][a];
  float lR[D][D], Sm[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) {
      float pf = 0.0f, pt = 0.0f, rs = 0.0f;
#pragma unroll
      for (int e = 0; e < D; ++e) {
        pf += lP[a][e] * F[e * D + b];                          // (lP F)_ab
        pt += lP[e][a] * (F[e * D + b] - R[e * D + b]);         // (lP^T (F - R))_ab
        rs += R[e * D + a] * F[e * D + b];                      // (R^T F)_ab = S
      }
      lF[a * D + b] += 2.0f * S.mu * (pf + pt) + S.la * (2.0f * J - 1.0f) * trP * c[a * D + b];
      lR[a][b] = -2.0f * S.mu * pf;
      Sm[a][b] = rs;
    }
  // G = R^T lR, sk = skew(G)
  float sk[D][D];
  {
    float G[D][D];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) {
        float acc = 0.0f;
#pragma unroll
        for (int e = 0; e < D; ++e) acc += R[e * D + a] * lR[e][b];
        G[a][b] = acc;
      }
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) sk[a][b] = 0.5f * (G[a][b] - G[b][a]);
  }
  float X[D][D];
  if constexpr (D == 3) {
    // c = (tr S I - S)^{-1} axial(sk), X = [c]x; S symmetrised
    const float a0 = sk[2][1], a1 = sk[0][2], a2 = sk[1][0];
    const float tr = Sm[0][0] + Sm[1][1] + Sm[2][2];
    float K[9];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) K[a * 3 + b] = (a == b ? tr : 0.0f) - 0.5f * (Sm[a][b] + Sm[b][a]);
    float kc[9];
    cof<3>(K, kc);
    const float kd = K[0] * kc[0] + K[1] * kc[1] + K[2] * kc[2];
    // K^{-1} = cof(K)^T / det K (K symmetric: cof(K) symmetric)
    const float c0 = (kc[0] * a0 + kc[3] * a1 + kc[6] * a2) / kd;
    const float c1 = (kc[1] * a0 + kc[4] * a1 + kc[7] * a2) / kd;
    const float c2 = (kc[2] * a0 + kc[5] * a1 + kc[8] * a2) / kd;
    X[0][0] = 0.f, X[0][1] = -c2, X[0][2] = c1;
    X[1][0] = c2, X[1][1] = 0.f, X[1][2] = -c0;
    X[2][0] = -c1, X[2][1] = c0, X[2][2] = 0.f;
  } else {
    const float tr = Sm[0][0] + Sm[1][1];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) X[a][b] = sk[a][b] / tr;
  }
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) {
      float acc = 0.0f;
#pragma unroll
      for (int e = 0; e < D; ++e) acc += R[a * D + e] * X[e][b];
      lF[a * D + b] += 2.0f * acc;
    }
}

// ---- warp-aggregated scatter -----------------------------------------------------------
// Lanes whose particles share a base cell add into the same stencil nodes.  When every
// such group is a contiguous run of lanes (particles stored in spatial order, as the
// scenes' lattices are), the group's sums are formed with a segmented shuffle tree and
// only its first lane issues the atomics; otherwise every lane adds its own.  All 32
// lanes must call seg_of / seg_sum (invalid lanes pass a unique key and zeros).
struct Seg {
  bool ok;   // every group of the warp is contiguous
  bool head; // this lane issues the group's atomics
  int end;   // one past the group's last lane
};

__device__ __forceinline__ Seg seg_of(int key) {
  const unsigned peers = __match_any_sync(0xffffffffu, key);
  const int lane = threadIdx.x & 31, s0 = __ffs(peers) - 1, g = __popc(peers);
  const unsigned run = g == 32 ? 0xffffffffu : (((1u << g) - 1u) << s0);
  Seg r;
  r.ok = __all_sync(0xffffffffu, peers == run);
  r.head = lane == s0;
  r.end = s0 + g;
  return r;
}

__device__ __forceinline__ float seg_sum(float v, const Seg& sg) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const float o = __shfl_down_sync(0xffffffffu, v, off);
    if (lane + off < sg.end) v += o;
  }
  return v;
}

// ---------------------------------------------------------------- forward
// the affine matrix A = stress + m C of a state row (fluid: k (J - 1) I)
template <int D, bool EL>
__device__ __forceinline__ void affine(const float* st, const AdjSim& S, float (*A)[D]) {
  constexpr int CO = kCO<D, EL>;
  if constexpr (EL) {
    stress_el<D>(st + 2 * D, S, A);
  } else {
    const float sJ = S.k * (st[2 * D] - 1.0f);
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) A[a][b] = a == b ? sJ : 0.0f;
  }
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) A[a][b] += S.m * st[CO + a * D + b];
}

template <int D, bool EL>
__device__ __forceinline__ void p2g_fwd_body(uint64_t p, const float* __restrict__ s, uint64_t n, AdjSim S, float4* __restrict__ grid) {
  // every lane of the warp must call (warp-aggregated atomics); lanes past n add nothing
  constexpr int NS = kNS<D, EL>;
  const bool valid = p < n;
  const float* st = s + (valid ? p : 0) * NS;
  const Stencil<D> sc = stencil<D>(st, S);
  float A[D][D];
  affine<D, EL>(st, S, A);
  const int o0[3] = {0, 0, 0};
  const Seg sg = seg_of(valid ? (int)node_of<D>(sc, o0, S) : -1 - (int)(threadIdx.x & 31));
  for (int q = 0; q < kNO<D>; ++q) {
    int o[3];
    offset_of<D>(q, o);
    float W, dW[3];
    weight<D>(sc, o, W, dW);
    float dpos[D];
#pragma unroll
    for (int a = 0; a < D; ++a) dpos[a] = ((float)o[a] - sc.fx[a]) * S.dx;
    float vals[4] = {valid ? W * S.m : 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int a = 0; a < D; ++a) {
      float Ad = 0.0f;
#pragma unroll
      for (int b = 0; b < D; ++b) Ad += A[a][b] * dpos[b];
      vals[1 + a] = valid ? W * (S.m * st[D + a] + Ad) : 0.f;
    }
    float4* nd = grid + node_of<D>(sc, o, S);
    if (sg.ok) {
#pragma unroll
      for (int c = 0; c < D + 1; ++c) vals[c] = seg_sum(vals[c], sg);
    }
    if (valid && (!sg.ok || sg.head)) {
      atomicAdd(&nd->x, vals[0]);
      atomicAdd(&nd->y, vals[1]);
      atomicAdd(&nd->z, vals[2]);
      if (D == 3) atomicAdd(&nd->w, vals[3]);
    }
  }
}

template <int D, bool EL>
__global__ void k_p2g_fwd(const float* __restrict__ s, uint64_t n, AdjSim S, float4* __restrict__ grid) {
  p2g_fwd_body<D, EL>((uint64_t)blockIdx.x * blockDim.x + threadIdx.x, s, n, S, grid);
}

__device__ __forceinline__ float comp(const float4& v, int a) { return a == 0 ? v.y : (a == 1 ? v.z : v.w); }

// v = P/m + dt g, separating walls (reading Q13): gv = (m, vx, vy, vz).  The grids are
// zero at the start of every step (no memsets): the forward clears `grid` here once
// read (clear_grid), the adjoint step clears `lgrid` here (before g2p_bwd accumulates
// into it) and `grid` in k_grid_bwd, its last reader.
template <int D>
__device__ __forceinline__ void grid_fwd_body(uint64_t c, float4* __restrict__ grid, uint64_t nn, AdjSim S, float4* __restrict__ gv,
                           bool clear_grid, float4* __restrict__ clear_lgrid) {
  if (c >= nn) return;
  const float4 nd = grid[c];
  if (clear_grid) grid[c] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (clear_lgrid) clear_lgrid[c] = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 out = make_float4(nd.x, 0.f, 0.f, 0.f);
  if (nd.x > 0.0f) {
    const int nz = D == 3 ? S.res[2] : 1;
    const int ijk[3] = {(int)(c / ((uint64_t)S.res[1] * nz)), (int)((c / nz) % S.res[1]), (int)(c % nz)};
    float v[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int a = 0; a < D; ++a) {
      float va = comp(nd, a) / nd.x + S.dt * S.g[a];
      if (ijk[a] < S.bound && va < 0.0f) va = 0.0f;
      if (ijk[a] > S.res[a] - S.bound && va > 0.0f) va = 0.0f;
      v[a] = va;
    }
    out = make_float4(nd.x, v[0], v[1], v[2]);
  }
  gv[c] = out;
}

template <int D>
__global__ void k_grid_fwd(float4* __restrict__ grid, uint64_t nn, AdjSim S, float4* __restrict__ gv,
                           bool clear_grid, float4* __restrict__ clear_lgrid) {
  grid_fwd_body<D>((uint64_t)blockIdx.x * blockDim.x + threadIdx.x, grid, nn, S, gv, clear_grid, clear_lgrid);
}

// v' and C' of a particle from the updated grid
template <int D>
__device__ __forceinline__ void gather(const Stencil<D>& sc, const float4* __restrict__ gv, const AdjSim& S, float* v,
                                       float (*C)[D]) {
#pragma unroll
  for (int a = 0; a < D; ++a) {
    v[a] = 0.0f;
#pragma unroll
    for (int b = 0; b < D; ++b) C[a][b] = 0.0f;
  }
  for (int q = 0; q < kNO<D>; ++q) {
    int o[3];
    offset_of<D>(q, o);
    float W, dW[3];
    weight<D>(sc, o, W, dW);
    const float4 nd = gv[node_of<D>(sc, o, S)];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const float vi = comp(nd, a);
      v[a] += W * vi;
#pragma unroll
      for (int b = 0; b < D; ++b) C[a][b] += 4.0f * S.inv_dx * W * vi * ((float)o[b] - sc.fx[b]);
    }
  }
}

template <int D, bool EL>
__device__ __forceinline__ void g2p_fwd_body(uint64_t p, const float* __restrict__ s, uint64_t n, const float4* __restrict__ gv, AdjSim S,
                          float* __restrict__ out) {
  constexpr int NS = kNS<D, EL>, CO = kCO<D, EL>;
  if (p >= n) return;
  const float* st = s + p * NS;
  const Stencil<D> sc = stencil<D>(st, S);
  float v[D], C[D][D];
  gather<D>(sc, gv, S, v, C);
  float* o = out + p * NS;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    o[a] = st[a] + S.dt * v[a];
    o[D + a] = v[a];
  }
  if constexpr (EL) {  // F' = (I + dt C') F
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) {
        float acc = 0.0f;
#pragma unroll
        for (int e = 0; e < D; ++e) acc += ((a == e ? 1.0f : 0.0f) + S.dt * C[a][e]) * st[2 * D + e * D + b];
        o[2 * D + a * D + b] = acc;
      }
  } else {  // J' = J (1 + dt tr C')
    float tr = 0.0f;
#pragma unroll
    for (int a = 0; a < D; ++a) tr += C[a][a];
    o[2 * D] = st[2 * D] * (1.0f + S.dt * tr);
  }
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) o[CO + a * D + b] = C[a][b];
}

template <int D, bool EL>
__global__ void k_g2p_fwd(const float* __restrict__ s, uint64_t n, const float4* __restrict__ gv, AdjSim S,
                          float* __restrict__ out) {
  g2p_fwd_body<D, EL>((uint64_t)blockIdx.x * blockDim.x + threadIdx.x, s, n, gv, S, out);
}

// ---------------------------------------------------------------- adjoint
// sum_p lambda^2 per scalar into g: warp shuffles, then the 8 warps of the CTA through
// shared memory (double), then ONE double atomic per scalar per CTA (per-warp atomics on
// the ns addresses serialised: 14 us of a 57 us adjoint step at 80K particles).  Every
// thread of the CTA must call it.
template <int NS>
__device__ __forceinline__ void tally(const float* lam, bool valid, double* g) {
  __shared__ double part[8][NS];
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int h = 0; h < NS; ++h) {
    float q = valid ? lam[h] * lam[h] : 0.0f;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) q += __shfl_xor_sync(full, q, off);
    if (lane == 0) part[warp][h] = (double)q;
  }
  __syncthreads();
  if (threadIdx.x < NS) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w][threadIdx.x];
    if (t != 0.0) atomicAdd(g + threadIdx.x, t);
  }
}

// lambda_T = (0, m v_T, 0, 0), the kinetic energy z and the tally of lambda_T
template <int D, bool EL>
__device__ __forceinline__ void lambda_T_body(uint64_t p, const float* __restrict__ s, uint64_t n, AdjSim S, float* __restrict__ lam, double* g,
                           double* z) {
  constexpr int NS = kNS<D, EL>;
  const bool valid = p < n;
  float l[NS];
#pragma unroll
  for (int h = 0; h < NS; ++h) l[h] = 0.0f;
  float ke = 0.0f;
  if (valid) {
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const float va = s[p * NS + D + a];
      l[D + a] = S.m * va;
      ke += 0.5f * S.m * va * va;
    }
#pragma unroll
    for (int h = 0; h < NS; ++h) lam[p * NS + h] = l[h];
  }
  tally<NS>(l, valid, g);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) ke += __shfl_xor_sync(0xffffffffu, ke, off);
  if ((threadIdx.x & 31) == 0 && ke != 0.0f) atomicAdd(z, (double)ke);
}

template <int D, bool EL>
__global__ void k_lambda_T(const float* __restrict__ s, uint64_t n, AdjSim S, float* __restrict__ lam, double* g,
                           double* z) {
  lambda_T_body<D, EL>((uint64_t)blockIdx.x * blockDim.x + threadIdx.x, s, n, S, lam, g, z);
}

// G2P reverse: node adjoints lgrid.yzw += W (lv' + 4/dx lC' (o - fx)); particle partials:
// lam_t = (lx', 0, lJ' (1 + dt tr C') | (I + dt C')^T lF', 0) and lfx through G2P
template <int D, bool EL>
__device__ __forceinline__ void g2p_bwd_body(uint64_t p, const float* __restrict__ s, const float* __restrict__ lam1, uint64_t n,
                          const float4* __restrict__ gv, AdjSim S, float4* __restrict__ lgrid,
                          float* __restrict__ lam, float* __restrict__ lfx_out) {
  constexpr int NS = kNS<D, EL>, CO = kCO<D, EL>;
  // every lane of the warp must call (warp-aggregated atomics); lanes past n write nothing
  const bool valid = p < n;
  if (!valid) p = 0;
  const float* st = s + p * NS;
  const float* l1 = lam1 + p * NS;
  const Stencil<D> sc = stencil<D>(st, S);
  float vnew[D], Cn[D][D];
  gather<D>(sc, gv, S, vnew, Cn);  // forward recompute of C'
  float lv[D], lC[D][D];
  float* lo = lam + p * NS;
  float lw[NS];
#pragma unroll
  for (int h = 0; h < NS; ++h) lw[h] = 0.0f;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    lv[a] = l1[D + a] + S.dt * l1[a];
    lw[a] = l1[a];
#pragma unroll
    for (int b = 0; b < D; ++b) lC[a][b] = l1[CO + a * D + b];
  }
  if constexpr (EL) {
    // lF = (I + dt C')^T lF',  lC' += dt lF' F^T
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) {
        float acc = 0.0f, acc2 = 0.0f;
#pragma unroll
        for (int e = 0; e < D; ++e) {
          acc += ((e == a ? 1.0f : 0.0f) + S.dt * Cn[e][a]) * l1[2 * D + e * D + b];
          acc2 += l1[2 * D + a * D + e] * st[2 * D + b * D + e];
        }
        lw[2 * D + a * D + b] = acc;
        lC[a][b] += S.dt * acc2;
      }
  } else {
    float tr = 0.0f;
#pragma unroll
    for (int a = 0; a < D; ++a) tr += Cn[a][a];
    const float lJ1 = l1[2 * D];
    lw[2 * D] = lJ1 * (1.0f + S.dt * tr);
#pragma unroll
    for (int a = 0; a < D; ++a) lC[a][a] += lJ1 * st[2 * D] * S.dt;
  }
  float lfx[D];
#pragma unroll
  for (int a = 0; a < D; ++a) lfx[a] = 0.0f;
  const int o0[3] = {0, 0, 0};
  const Seg sg = seg_of(valid ? (int)node_of<D>(sc, o0, S) : -1 - (int)(threadIdx.x & 31));
  for (int q = 0; q < kNO<D>; ++q) {
    int o[3];
    offset_of<D>(q, o);
    float W, dW[3];
    weight<D>(sc, o, W, dW);
    const long long ni = node_of<D>(sc, o, S);
    const float4 nd = gv[ni];
    float dpc[D];
#pragma unroll
    for (int a = 0; a < D; ++a) dpc[a] = (float)o[a] - sc.fx[a];
    float lW = 0.0f, add[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const float vi = comp(nd, a);
      float Cd = 0.0f;
#pragma unroll
      for (int b = 0; b < D; ++b) Cd += lC[a][b] * dpc[b];
      add[a] = W * (lv[a] + 4.0f * S.inv_dx * Cd);
      lW += lv[a] * vi + 4.0f * S.inv_dx * vi * Cd;
    }
#pragma unroll
    for (int b = 0; b < D; ++b) {
      float s2 = 0.0f;
#pragma unroll
      for (int a = 0; a < D; ++a) s2 += lC[a][b] * comp(nd, a);
      lfx[b] += -4.0f * S.inv_dx * W * s2 + lW * dW[b];
    }
    if (!valid) add[0] = add[1] = add[2] = 0.0f;
    if (sg.ok) {
#pragma unroll
      for (int c = 0; c < D; ++c) add[c] = seg_sum(add[c], sg);
    }
    if (valid && (!sg.ok || sg.head)) {
      atomicAdd(&lgrid[ni].y, add[0]);
      atomicAdd(&lgrid[ni].z, add[1]);
      if (D == 3) atomicAdd(&lgrid[ni].w, add[2]);
    }
  }
  if (valid) {
#pragma unroll
    for (int h = 0; h < NS; ++h) lo[h] = lw[h];
#pragma unroll
    for (int a = 0; a < D; ++a) lfx_out[p * 3 + a] = lfx[a];
  }
}

template <int D, bool EL>
__global__ void k_g2p_bwd(const float* __restrict__ s, const float* __restrict__ lam1, uint64_t n,
                          const float4* __restrict__ gv, AdjSim S, float4* __restrict__ lgrid,
                          float* __restrict__ lam, float* __restrict__ lfx_out) {
  g2p_bwd_body<D, EL>((uint64_t)blockIdx.x * blockDim.x + threadIdx.x, s, lam1, n, gv, S, lgrid, lam, lfx_out);
}

// grid reverse: (0, lv) -> (lm, lP); lP = lv / m, lm = -lv . u / m, u = P / m; zero on
// wall-clamped components and on empty nodes
template <int D>
__device__ __forceinline__ void grid_bwd_body(uint64_t c, float4* __restrict__ grid, uint64_t nn, AdjSim S, float4* __restrict__ lgrid) {
  if (c >= nn) return;
  const float4 nd = grid[c];
  grid[c] = make_float4(0.f, 0.f, 0.f, 0.f);  // last reader of the step's grid
  const float4 lvn = lgrid[c];
  float4 out = make_float4(0.f, 0.f, 0.f, 0.f);
  if (nd.x > 0.0f) {
    const int nz = D == 3 ? S.res[2] : 1;
    const int ijk[3] = {(int)(c / ((uint64_t)S.res[1] * nz)), (int)((c / nz) % S.res[1]), (int)(c % nz)};
    float lP[3] = {0.f, 0.f, 0.f}, lm = 0.0f;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const float u = comp(nd, a) / nd.x;
      const float va = u + S.dt * S.g[a];
      const bool clamp = (ijk[a] < S.bound && va < 0.0f) || (ijk[a] > S.res[a] - S.bound && va > 0.0f);
      const float l = clamp ? 0.0f : comp(lvn, a);
      lP[a] = l / nd.x;
      lm -= l * u / nd.x;
    }
    out = make_float4(lm, lP[0], lP[1], lP[2]);
  }
  lgrid[c] = out;
}

template <int D>
__global__ void k_grid_bwd(float4* __restrict__ grid, uint64_t nn, AdjSim S, float4* __restrict__ lgrid) {
  grid_bwd_body<D>((uint64_t)blockIdx.x * blockDim.x + threadIdx.x, grid, nn, S, lgrid);
}

// P2G reverse: finishes lambda_t and tallies it
template <int D, bool EL>
__device__ __forceinline__ void p2g_bwd_body(uint64_t p, const float* __restrict__ s, uint64_t n, const float4* __restrict__ lgrid, AdjSim S,
                          const float* __restrict__ lfx_in, float* __restrict__ lam, double* __restrict__ g) {
  constexpr int NS = kNS<D, EL>, CO = kCO<D, EL>;
  const bool valid = p < n;
  float l[NS];
#pragma unroll
  for (int h = 0; h < NS; ++h) l[h] = 0.0f;
  if (valid) {
    const float* st = s + p * NS;
    const Stencil<D> sc = stencil<D>(st, S);
    float A[D][D], lA[D][D], lv[D], lfx[D];
    affine<D, EL>(st, S, A);
#pragma unroll
    for (int a = 0; a < D; ++a) {
      lv[a] = 0.0f;
      lfx[a] = lfx_in[p * 3 + a];
#pragma unroll
      for (int b = 0; b < D; ++b) lA[a][b] = 0.0f;
    }
    for (int q = 0; q < kNO<D>; ++q) {
      int o[3];
      offset_of<D>(q, o);
      float W, dW[3];
      weight<D>(sc, o, W, dW);
      const float4 ln = lgrid[node_of<D>(sc, o, S)];
      float dpos[D];
#pragma unroll
      for (int a = 0; a < D; ++a) dpos[a] = ((float)o[a] - sc.fx[a]) * S.dx;
      float lW = ln.x * S.m;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const float lPa = comp(ln, a);
        float Ad = 0.0f;
#pragma unroll
        for (int b = 0; b < D; ++b) Ad += A[a][b] * dpos[b];
        lW += lPa * (S.m * st[D + a] + Ad);
        lv[a] += W * S.m * lPa;
#pragma unroll
        for (int b = 0; b < D; ++b) lA[a][b] += W * lPa * dpos[b];
      }
#pragma unroll
      for (int b = 0; b < D; ++b) {
        float ld = 0.0f;
#pragma unroll
        for (int a = 0; a < D; ++a) ld += A[a][b] * comp(ln, a);
        lfx[b] += -S.dx * W * ld + lW * dW[b];
      }
    }
    const float* lo = lam + p * NS;
#pragma unroll
    for (int h = 0; h < NS; ++h) l[h] = lo[h];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      l[a] += sc.dfx[a] * lfx[a];
      l[D + a] = lv[a];
#pragma unroll
      for (int b = 0; b < D; ++b) l[CO + a * D + b] = S.m * lA[a][b];
    }
    if constexpr (EL) {
      float lP[D][D];
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = 0; b < D; ++b) lP[a][b] = S.scale * lA[a][b];
      stress_el_adj<D>(st + 2 * D, lP, S, l + 2 * D);
    } else {
      float trA = 0.0f;
#pragma unroll
      for (int a = 0; a < D; ++a) trA += lA[a][a];
      l[2 * D] += S.k * trA;
    }
    float* lw = lam + p * NS;
#pragma unroll
    for (int h = 0; h < NS; ++h) lw[h] = l[h];
  }
  if (g) tally<NS>(l, valid, g);
}

template <int D, bool EL>
__global__ void k_p2g_bwd(const float* __restrict__ s, uint64_t n, const float4* __restrict__ lgrid, AdjSim S,
                          const float* __restrict__ lfx_in, float* __restrict__ lam, double* __restrict__ g) {
  p2g_bwd_body<D, EL>((uint64_t)blockIdx.x * blockDim.x + threadIdx.x, s, n, lgrid, S, lfx_in, lam, g);
}

// ---- cooperative (single-launch) step chains (QADJ_COOP=1) ------------------------------
// k forward steps, or one adjoint step, in ONE cooperative launch with grid-wide barriers
// between the phases (the same device bodies as the separate kernels, so the same
// arithmetic).  Kept as an option: measured no faster (see qadj_create).
template <int D, bool EL>
__global__ void __launch_bounds__(256) k_forward_chain(const float* __restrict__ s0, float* __restrict__ a,
                                                       float* __restrict__ b, uint32_t k, uint64_t n, uint64_t nn,
                                                       AdjSim S, float4* __restrict__ grid, float4* __restrict__ gv) {
  cooperative_groups::grid_group G = cooperative_groups::this_grid();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const float* in = s0;
  for (uint32_t i = 0; i < k; ++i) {
    float* out = (i % 2 == 0) ? a : b;
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < n; base += stride)
      p2g_fwd_body<D, EL>(base + threadIdx.x, in, n, S, grid);
    G.sync();
    for (uint64_t c = t0; c < nn; c += stride) grid_fwd_body<D>(c, grid, nn, S, gv, true, nullptr);
    G.sync();
    for (uint64_t p = t0; p < n; p += stride) g2p_fwd_body<D, EL>(p, in, n, gv, S, out);
    G.sync();
    in = out;
  }
}

template <int D, bool EL>
__global__ void __launch_bounds__(256) k_adjoint_coop(const float* __restrict__ s, const float* __restrict__ lam1,
                                                      float* __restrict__ lam, double* __restrict__ g, uint64_t n,
                                                      uint64_t nn, AdjSim S, float4* __restrict__ grid,
                                                      float4* __restrict__ gv, float4* __restrict__ lgrid,
                                                      float* __restrict__ lfx) {
  cooperative_groups::grid_group G = cooperative_groups::this_grid();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < n; base += stride)
    p2g_fwd_body<D, EL>(base + threadIdx.x, s, n, S, grid);
  G.sync();
  for (uint64_t c = t0; c < nn; c += stride) grid_fwd_body<D>(c, grid, nn, S, gv, false, lgrid);
  G.sync();
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < n; base += stride)
    g2p_bwd_body<D, EL>(base + threadIdx.x, s, lam1, n, gv, S, lgrid, lam, lfx);
  G.sync();
  for (uint64_t c = t0; c < nn; c += stride) grid_bwd_body<D>(c, grid, nn, S, lgrid);
  G.sync();
  // block-uniform trip count: the tally's CTA barrier needs every thread
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < n; base += stride)
    p2g_bwd_body<D, EL>(base + threadIdx.x, s, n, lgrid, S, lfx, lam, g);
}

}  // namespace

// ---------------------------------------------------------------- runtime
struct qadj_ctx {
  int dim = 3;
  bool el = false;  // fixed-corotated elastic (else J-fluid)
  unsigned coop_fwd = 0, coop_adj = 0;  // co-resident grid sizes of the cooperative kernels (0: not used)
  uint64_t n = 0, nn = 0;
  int ns = 0;
  AdjSim S{};
  cudaStream_t stream = nullptr;
  float4 *grid = nullptr, *gv = nullptr, *lgrid = nullptr;
  float* lfx = nullptr;
  double* dacc = nullptr;  // [ns] tallies + [1] z
  std::vector<float*> pool;  // state / adjoint buffers [n][ns]
  uint64_t launches = 0;
};

namespace {

unsigned blocks(uint64_t n) { return (unsigned)((n + 255) / 256); }

template <int D, bool EL>
void forward_k(qadj_ctx* c, const float* in, float* out) {
  k_p2g_fwd<D, EL><<<blocks(c->n), 256, 0, c->stream>>>(in, c->n, c->S, c->grid);
  k_grid_fwd<D><<<blocks(c->nn), 256, 0, c->stream>>>(c->grid, c->nn, c->S, c->gv, true, nullptr);
  k_g2p_fwd<D, EL><<<blocks(c->n), 256, 0, c->stream>>>(in, c->n, c->gv, c->S, out);
}

template <int D, bool EL>
void adjoint_k(qadj_ctx* c, const float* s, const float* lam1, float* lam, double* g) {
  k_p2g_fwd<D, EL><<<blocks(c->n), 256, 0, c->stream>>>(s, c->n, c->S, c->grid);
  k_grid_fwd<D><<<blocks(c->nn), 256, 0, c->stream>>>(c->grid, c->nn, c->S, c->gv, false, c->lgrid);
  k_g2p_bwd<D, EL><<<blocks(c->n), 256, 0, c->stream>>>(s, lam1, c->n, c->gv, c->S, c->lgrid, lam, c->lfx);
  k_grid_bwd<D><<<blocks(c->nn), 256, 0, c->stream>>>(c->grid, c->nn, c->S, c->lgrid);
  k_p2g_bwd<D, EL><<<blocks(c->n), 256, 0, c->stream>>>(s, c->n, c->lgrid, c->S, c->lfx, lam, g);
}

qmpm_status forward_dev(qadj_ctx* c, const float* in, float* out);

template <int D, bool EL>
cudaError_t chain_k(qadj_ctx* c, const float* s0, float* a, float* b, uint32_t k) {
  void* args[] = {&s0, &a, &b, &k, &c->n, &c->nn, &c->S, &c->grid, &c->gv};
  return cudaLaunchCooperativeKernel((const void*)k_forward_chain<D, EL>, dim3(c->coop_fwd), dim3(256), args, 0,
                                     c->stream);
}

template <int D, bool EL>
cudaError_t adjoint_coop_k(qadj_ctx* c, const float* s, const float* lam1, float* lam, double* g) {
  void* args[] = {&s, &lam1, &lam, &g, &c->n, &c->nn, &c->S, &c->grid, &c->gv, &c->lgrid, &c->lfx};
  return cudaLaunchCooperativeKernel((const void*)k_adjoint_coop<D, EL>, dim3(c->coop_adj), dim3(256), args, 0,
                                     c->stream);
}

// k forward steps from s0 alternating into a, b (the last step lands in (k - 1) % 2 ? b : a)
qmpm_status forward_chain_dev(qadj_ctx* c, const float* s0, float* a, float* b, uint32_t k) {
  if (k == 0) return QMPM_OK;
  if (c->coop_fwd) {
    cudaError_t e;
    if (c->dim == 3)
      e = c->el ? chain_k<3, true>(c, s0, a, b, k) : chain_k<3, false>(c, s0, a, b, k);
    else
      e = c->el ? chain_k<2, true>(c, s0, a, b, k) : chain_k<2, false>(c, s0, a, b, k);
    c->launches += 1;
    ACK(e);
    return QMPM_OK;
  }
  const float* cur = s0;
  for (uint32_t i = 0; i < k; ++i) {
    float* dst = (i % 2 == 0) ? a : b;
    qmpm_status rc = forward_dev(c, cur, dst);
    if (rc) return rc;
    cur = dst;
  }
  return QMPM_OK;
}

qmpm_status forward_dev(qadj_ctx* c, const float* in, float* out) {
  if (c->dim == 3)
    c->el ? forward_k<3, true>(c, in, out) : forward_k<3, false>(c, in, out);
  else
    c->el ? forward_k<2, true>(c, in, out) : forward_k<2, false>(c, in, out);
  c->launches += 3;
  ACK(cudaGetLastError());
  return QMPM_OK;
}

// lambda_t from s_t and lambda_{t+1} (g nullable: device tallies to accumulate)
qmpm_status adjoint_dev(qadj_ctx* c, const float* s, const float* lam1, float* lam, double* g) {
  if (c->coop_adj) {
    cudaError_t e;
    if (c->dim == 3)
      e = c->el ? adjoint_coop_k<3, true>(c, s, lam1, lam, g) : adjoint_coop_k<3, false>(c, s, lam1, lam, g);
    else
      e = c->el ? adjoint_coop_k<2, true>(c, s, lam1, lam, g) : adjoint_coop_k<2, false>(c, s, lam1, lam, g);
    c->launches += 1;
    ACK(e);
    return QMPM_OK;
  }
  if (c->dim == 3)
    c->el ? adjoint_k<3, true>(c, s, lam1, lam, g) : adjoint_k<3, false>(c, s, lam1, lam, g);
  else
    c->el ? adjoint_k<2, true>(c, s, lam1, lam, g) : adjoint_k<2, false>(c, s, lam1, lam, g);
  c->launches += 5;
  ACK(cudaGetLastError());
  return QMPM_OK;
}

template <int D, bool EL>
void coop_sizes(qadj_ctx* c, int sms) {
  int bf = 0, ba = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bf, k_forward_chain<D, EL>, 256, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ba, k_adjoint_coop<D, EL>, 256, 0);
  cudaGetLastError();
  const uint64_t need = (std::max(c->n, c->nn) + 255) / 256;  // more CTAs than work only idles
  c->coop_fwd = (unsigned)std::min<uint64_t>((uint64_t)bf * sms, need);
  c->coop_adj = (unsigned)std::min<uint64_t>((uint64_t)ba * sms, need);
}

// a state-sized device buffer: from the free list, else a new pool buffer (kept by the ctx
// and handed to the next call's free list); `inuse` / `peak` count the call's buffers
qmpm_status get_buf(qadj_ctx* c, std::vector<float*>& freel, float** out, uint32_t* inuse = nullptr,
                    uint32_t* peak = nullptr) {
  if (inuse) {
    ++*inuse;
    if (peak && *inuse > *peak) *peak = *inuse;
  }
  if (!freel.empty()) {
    *out = freel.back();
    freel.pop_back();
    return QMPM_OK;
  }
  float* b = nullptr;
  if (cudaMalloc(&b, sizeof(float) * c->n * c->ns) != cudaSuccess) {
    cudaGetLastError();
    return afail(QMPM_ENOMEM, "qadj: cannot allocate a checkpoint (%zu bytes)", sizeof(float) * c->n * c->ns);
  }
  c->pool.push_back(b);
  *out = b;
  return QMPM_OK;
}

struct Bisect {
  qadj_ctx* c;
  std::vector<float*> freel;
  uint32_t resident = 0, max_resident = 0;
  uint32_t inuse = 0, peak = 0;  // state-sized buffers in use (checkpoints, adjoints, scratch)
  uint64_t fwd = 0, adj = 0;

  qmpm_status get(float** out) { return get_buf(c, freel, out, &inuse, &peak); }
  void put(float* b) {
    freel.push_back(b);
    --inuse;
  }

  // state at `to` from the state at `from` (k >= 1 steps) into a fresh buffer
  qmpm_status advance(const float* s, uint32_t k, float** out) {
    float *a = nullptr, *b = nullptr;
    qmpm_status rc = get(&a);
    if (!rc) rc = get(&b);
    if (rc) return rc;
    rc = forward_chain_dev(c, s, a, b, k);
    if (rc) return rc;
    fwd += k;
    float* last = ((k - 1) % 2 == 0) ? a : b;
    *out = last;
    put(last == a ? b : a);
    return QMPM_OK;
  }

  // lambda_lo (into lam_out) from the state at lo and lambda_hi
  qmpm_status back(uint32_t lo, uint32_t hi, const float* s_lo, const float* lam_hi, float* lam_out, double* g) {
    if (hi - lo == 1) {
      ++adj;
      return adjoint_dev(c, s_lo, lam_hi, lam_out, g);
    }
    const uint32_t mid = lo + (hi - lo) / 2;
    float* s_mid = nullptr;
    qmpm_status rc = advance(s_lo, mid - lo, &s_mid);
    if (rc) return rc;
    max_resident = std::max(max_resident, ++resident + 1);  // + s0
    float* lam_mid = nullptr;
    rc = get(&lam_mid);
    if (!rc) rc = back(mid, hi, s_mid, lam_hi, lam_mid, g);
    put(s_mid);
    --resident;
    if (!rc) rc = back(lo, mid, s_lo, lam_mid, lam_out, g);
    put(lam_mid);
    return rc;
  }
};

}  // namespace

extern "C" {

qmpm_status qadj_create(const qmpm_params* params, int32_t dim, int32_t material, uint64_t n, void* cuda_stream,
                        qadj_ctx** out) {
  if (!params || !out) return afail(QMPM_EINVAL, "NULL argument");
  *out = nullptr;
  if (dim != 2 && dim != 3) return afail(QMPM_EINVAL, "dim must be 2 or 3");
  if (material != QMPM_FLUID_J && material != QMPM_ELASTIC_FCR) return afail(QMPM_EINVAL, "qadj: unknown material");
  if (n == 0) return afail(QMPM_EINVAL, "n must be > 0");
  for (int a = 0; a < dim; ++a)
    if (params->grid_res[a] < 3) return afail(QMPM_EINVAL, "grid_res must be >= 3 per axis");
  qadj_ctx* c = new qadj_ctx();
  c->dim = dim;
  c->el = material == QMPM_ELASTIC_FCR;
  c->n = n;
  c->ns = 2 * dim + (c->el ? dim * dim : 1) + dim * dim;
  c->stream = (cudaStream_t)cuda_stream;
  AdjSim& S = c->S;
  for (int a = 0; a < 3; ++a) {
    S.res[a] = a < dim ? params->grid_res[a] : 1;
    S.g[a] = params->gravity[a];
  }
  S.dx = params->dx;
  S.inv_dx = 1.0f / params->dx;
  S.dt = params->dt;
  S.m = params->p_rho * params->p_vol;
  S.k = -params->dt * params->p_vol * 4.0f * S.inv_dx * S.inv_dx * params->E;
  S.scale = -params->dt * params->p_vol * 4.0f * S.inv_dx * S.inv_dx;
  S.mu = params->E / (2.0f * (1.0f + params->nu));
  S.la = params->E * params->nu / ((1.0f + params->nu) * (1.0f - 2.0f * params->nu));
  S.bound = params->bound;
  c->nn = (uint64_t)S.res[0] * S.res[1] * S.res[2];
  cudaError_t e = cudaMalloc(&c->grid, sizeof(float4) * c->nn);
  if (!e) e = cudaMalloc(&c->gv, sizeof(float4) * c->nn);
  if (!e) e = cudaMalloc(&c->lgrid, sizeof(float4) * c->nn);
  if (!e) e = cudaMalloc(&c->lfx, sizeof(float) * 3 * n);
  if (!e) e = cudaMalloc(&c->dacc, sizeof(double) * (c->ns + 1));
  if (!e) e = cudaMemsetAsync(c->grid, 0, sizeof(float4) * c->nn, c->stream);  // zero between steps from here on
  // QADJ_COOP=1: one cooperative launch per forward chain / adjoint step.  Measured, not
  // the default: at 80K particles (2D) a cooperative step costs what the separate
  // launches cost (29 us: the step is bound by its P2G atomics, not by launches), and at
  // 1M (3D) the grid-stride phases are 13 % slower than full-width launches.
  if (!e) {
    int dev = 0, coop = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const char* env = getenv("QADJ_COOP");
    const bool use = coop && env && atoi(env) != 0;
    if (use) {
      if (dim == 3)
        c->el ? coop_sizes<3, true>(c, sms) : coop_sizes<3, false>(c, sms);
      else
        c->el ? coop_sizes<2, true>(c, sms) : coop_sizes<2, false>(c, sms);
    }
  }
  if (!e) e = cudaStreamSynchronize(c->stream);
  if (e) {
    cudaGetLastError();
    qadj_destroy(c);
    return afail(QMPM_ENOMEM, "qadj_create: %s", cudaGetErrorString(e));
  }
  *out = c;
  return QMPM_OK;
}

qmpm_status qadj_destroy(qadj_ctx* c) {
  if (!c) return QMPM_OK;
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (void* p : {(void*)c->grid, (void*)c->gv, (void*)c->lgrid, (void*)c->lfx, (void*)c->dacc})
    if (p) cudaFree(p);
  for (float* p : c->pool) cudaFree(p);
  delete c;
  return QMPM_OK;
}

qmpm_status qadj_forward(qadj_ctx* c, const float* s_in, float* s_out) {
  if (!c || !s_in || !s_out) return afail(QMPM_EINVAL, "NULL argument");
  return forward_dev(c, s_in, s_out);
}

qmpm_status qadj_adjoint_step(qadj_ctx* c, const float* s_t, const float* lam_next, float* lam_t, double* g) {
  if (!c || !s_t || !lam_next || !lam_t) return afail(QMPM_EINVAL, "NULL argument");
  if (lam_t == lam_next) return afail(QMPM_EINVAL, "lam_t must not alias lam_next");
  return adjoint_dev(c, s_t, lam_next, lam_t, g);
}

qmpm_status qadj_gradient_tally(qadj_ctx* c, const float* s0, uint32_t T, double* g, double* z, float* lam0,
                                qadj_stats* stats) {
  if (!c || !s0 || !g) return afail(QMPM_EINVAL, "NULL argument");
  const size_t bytes = sizeof(float) * c->n * c->ns;
  Bisect B{c};
  B.freel = c->pool;  // every pool buffer is free between calls: reuse them
  float *s_first = nullptr, *lamT = nullptr, *lam_out = nullptr;
  qmpm_status rc = B.get(&s_first);
  if (rc) return rc;
  ACK(cudaMemcpyAsync(s_first, s0, bytes, cudaMemcpyDefault, c->stream));
  ACK(cudaMemsetAsync(c->dacc, 0, sizeof(double) * (c->ns + 1), c->stream));
  B.max_resident = 1;
  // s_T, lambda_T (and z, the tally of lambda_T)
  float* sT = s_first;
  if (T > 0) {
    rc = B.advance(s_first, T, &sT);
    if (rc) return rc;
    B.max_resident = 2;
  }
  rc = B.get(&lamT);
  if (rc) return rc;
  if (c->dim == 3 && c->el)
    k_lambda_T<3, true><<<blocks(c->n), 256, 0, c->stream>>>(sT, c->n, c->S, lamT, c->dacc, c->dacc + c->ns);
  else if (c->dim == 3)
    k_lambda_T<3, false><<<blocks(c->n), 256, 0, c->stream>>>(sT, c->n, c->S, lamT, c->dacc, c->dacc + c->ns);
  else if (c->el)
    k_lambda_T<2, true><<<blocks(c->n), 256, 0, c->stream>>>(sT, c->n, c->S, lamT, c->dacc, c->dacc + c->ns);
  else
    k_lambda_T<2, false><<<blocks(c->n), 256, 0, c->stream>>>(sT, c->n, c->S, lamT, c->dacc, c->dacc + c->ns);
  c->launches += 1;
  ACK(cudaGetLastError());
  if (T > 0) B.put(sT);
  float* lam_final = lamT;
  if (T > 0) {
    rc = B.get(&lam_out);
    if (rc) return rc;
    rc = B.back(0, T, s_first, lamT, lam_out, c->dacc);
    if (rc) return rc;
    lam_final = lam_out;
  }
  std::vector<double> h(c->ns + 1);
  ACK(cudaMemcpyAsync(h.data(), c->dacc, sizeof(double) * (c->ns + 1), cudaMemcpyDeviceToHost, c->stream));
  if (lam0) ACK(cudaMemcpyAsync(lam0, lam_final, bytes, cudaMemcpyDefault, c->stream));
  ACK(cudaStreamSynchronize(c->stream));
  for (int i = 0; i < c->ns; ++i) g[i] = h[i];
  if (z) *z = h[c->ns];
  if (stats) {
    stats->max_resident = B.max_resident;
    stats->peak_buffers = B.peak;
    stats->forward_steps = B.fwd;
    stats->adjoint_steps = B.adj;
  }
  return QMPM_OK;
}

qmpm_status qadj_launch_count(const qadj_ctx* c, uint64_t* launches) {
  if (!c || !launches) return afail(QMPM_EINVAL, "NULL argument");
  *launches = c->launches;
  return QMPM_OK;
}

}  // extern "C"
