// smoke_kernels.cuh -- the quantized Eulerian smoke step (P:574-579,
// P:954-957), NVRTC-specialised on two generated layout structs: SpecU (6 fields: the
// velocity of the two cells of a record, packing order cell0 x y z, cell1 x y z) and
// SpecP (2 fields: the pressure of the two cells).  DESIGN.md §12 readings S1-S8.
//
// Grid: collocated nx x ny x nz cells (S1); record r = (xr * ny + y) * nz + z holds cells
// x = 2 xr and 2 xr + 1 (S2), so consecutive threads (consecutive z) touch consecutive
// records.  Every kernel runs one thread per record (density: per cell) on a 3D grid:
// blockIdx.z = the x record (cell) plane, a 32 x 8 (z, y) tile per CTA, so no index
// division and the x-neighbour planes were just read by the previous CTAs (L2).  Lanes
// outside the domain stay to the end (encode_record's rare exact redo is a warp vote).
//
//   qsmoke_advect_u   u~ = A(q, u_vel, dt) [+ bdt rho e_y]: RK-3 backtrace (S4), trilinear
//                     clamped sampling (S3); q = u_vel, or 2 u_vel - u_refl (reflection, S8)
//   qsmoke_div        central-difference divergence, u = 0 outside (S5), fp32
//   qsmoke_jacobi     one Jacobi sweep with Neumann walls (S6), p re-encoded
//   qsmoke_project    u -= grad p (S7), wall-normal components zeroed, u re-encoded
//   qsmoke_advect_rho fp32 density advected by u, then the source box set to 1 (S8);
//                     optionally advances the device step counter (graph replay)
// All kernels march a CTA's (32 z x 8 y) record column along x (kXM planes per CTA):
// the stencils through a shared tile with a one-record halo, the advections through
// rings of decoded planes with a kH-cell halo (see below).
// Encodes are dithered with h = mix(record ^ salt) (reading Q5); salt comes from the host.
#pragma once
#include "codec_record.cuh"

#ifndef QSMOKE_JACOBI_MINB  // min resident CTAs per SM for the Jacobi sweep (tuning)
#define QSMOKE_JACOBI_MINB 6  // measured: 6 -> 0.542 ms, 1 -> 0.580, 7-8 -> 0.63 (612^3)
#endif
#ifndef QSMOKE_PROJECT_MINB  // min resident CTAs per SM for the projection (tuning)
#define QSMOKE_PROJECT_MINB 4  // measured at 612^3: 4 -> 0.92 ms, 1 -> 1.01, 5 -> 1.10
#endif
#ifndef QSMOKE_DIV_MINB  // min resident CTAs per SM for the divergence (tuning)
#define QSMOKE_DIV_MINB 8  // measured: 8 -> 0.63 ms, 1 or 6 -> 0.77
#endif
#ifndef QSMOKE_ADV_UNROLL  // 2: the two cells of a record interleaved; 1: one after the other
#define QSMOKE_ADV_UNROLL 2
#endif
constexpr int kAdvUnroll = QSMOKE_ADV_UNROLL;
#ifndef QSMOKE_ADV_MINB  // min resident CTAs per SM for the advection kernels (tuning)
#define QSMOKE_ADV_MINB 2
#endif

struct SmokeDev {
  int nx, ny, nz, nxr;     // cells per axis; records along x (nx / 2)
  float dx, inv_dx;        // cell size and its inverse
  float half_inv_dx, dx2;  // 1 / (2 dx), dx^2
  int lo[3], hi[3];        // density source box [lo, hi)
  unsigned long long n_rec;
};

// the dither salt of a store: a host value, or (graph replay) computed from the device
// step counter as step_salt(seed, 256 step + sub) -- the same value qmpm_encode derives
struct SaltSrc {
  uint32_t salt, sub, seed_lo, seed_hi;
  const unsigned long long* step;
};

namespace smoke {

using qmpm::sdec;

__device__ __forceinline__ unsigned long long rec_of(const SmokeDev& g, int xr, int y, int z) {
  return ((unsigned long long)xr * g.ny + y) * g.nz + z;
}

template <class SP>
__device__ __forceinline__ void ldrec(const uint32_t* __restrict__ base, unsigned long long r, uint32_t* w) {
#pragma unroll
  for (int q = 0; q < SP::W; ++q) w[q] = __ldg(base + r * SP::W + q);
  w[SP::W] = 0u;
}

// velocity of cells (x0, y, z) and (x0 + 1, y, z), 0 <= x0 <= nx - 2
__device__ __forceinline__ void u_pair(const uint32_t* __restrict__ U, const SmokeDev& g, int x0, int y, int z,
                                       float* a, float* b) {
  uint32_t w[SpecU::W + 1];
  ldrec<SpecU>(U, rec_of(g, x0 >> 1, y, z), w);
  if ((x0 & 1) == 0) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      a[c] = sdec<SpecU>(w, c);
      b[c] = sdec<SpecU>(w, 3 + c);
    }
  } else {
#pragma unroll
    for (int c = 0; c < 3; ++c) a[c] = sdec<SpecU>(w, 3 + c);
    ldrec<SpecU>(U, rec_of(g, (x0 >> 1) + 1, y, z), w);
#pragma unroll
    for (int c = 0; c < 3; ++c) b[c] = sdec<SpecU>(w, c);
  }
}

__device__ __forceinline__ void u_cell(const uint32_t* __restrict__ U, const SmokeDev& g, int x, int y, int z,
                                       float* u) {
  uint32_t w[SpecU::W + 1];
  ldrec<SpecU>(U, rec_of(g, x >> 1, y, z), w);
  if (x & 1) {
#pragma unroll
    for (int c = 0; c < 3; ++c) u[c] = sdec<SpecU>(w, 3 + c);
  } else {
#pragma unroll
    for (int c = 0; c < 3; ++c) u[c] = sdec<SpecU>(w, c);
  }
}

// S3: clamp to [0, n - 1], i0 = min(floor(p), n - 2), t = p - i0
__device__ __forceinline__ void corner(float p, int n, int& i0, float& t) {
  p = fminf(fmaxf(p, 0.0f), (float)(n - 1));
  i0 = min((int)floorf(p), n - 2);
  t = p - (float)i0;
}

// trilinear blend of the 8 corner values v[(dj * 2 + dk) * 2 + di][3] with weights t
// (S3); every sampling path uses this one arithmetic, so the shared-window and the
// global paths give identical results
__device__ __forceinline__ void trilerp(const float (*v)[3], float tx, float ty, float tz, float* out) {
#pragma unroll
  for (int c = 0; c < 3; ++c) out[c] = 0.0f;
#pragma unroll
  for (int dj = 0; dj < 2; ++dj) {
#pragma unroll
    for (int dk = 0; dk < 2; ++dk) {
      const float* a = v[(dj * 2 + dk) * 2];
      const float* b = v[(dj * 2 + dk) * 2 + 1];
      const float wyz = (dj ? ty : 1.0f - ty) * (dk ? tz : 1.0f - tz);
      const float wa = (1.0f - tx) * wyz, wb = tx * wyz;
#pragma unroll
      for (int c = 0; c < 3; ++c) out[c] = fmaf(wa, a[c], fmaf(wb, b[c], out[c]));
    }
  }
}

// the 8 corners of the cell block at (i, j, k) from the records in global memory
__device__ __forceinline__ void cube_global(const uint32_t* __restrict__ U, const SmokeDev& g, int i, int j, int k,
                                            float (*v)[3]) {
#pragma unroll
  for (int dj = 0; dj < 2; ++dj)
#pragma unroll
    for (int dk = 0; dk < 2; ++dk) u_pair(U, g, i, j + dj, k + dk, v[(dj * 2 + dk) * 2], v[(dj * 2 + dk) * 2 + 1]);
}

// sample of u (UR == NULL) or of 2 u - u_R (the reflection, S8) at p from global memory:
// the out-of-window path, not inlined so it costs the window path nothing
__device__ __noinline__ float3 sample_global(const uint32_t* __restrict__ U, const uint32_t* __restrict__ UR,
                                             const SmokeDev& g, float px, float py, float pz) {
  int i, j, k;
  float tx, ty, tz;
  corner(px, g.nx, i, tx);
  corner(py, g.ny, j, ty);
  corner(pz, g.nz, k, tz);
  float v[8][3], out[3];
  cube_global(U, g, i, j, k, v);
  if (UR) {
    float d[8][3];
    cube_global(UR, g, i, j, k, d);
#pragma unroll
    for (int e = 0; e < 8; ++e)
#pragma unroll
      for (int c = 0; c < 3; ++c) v[e][c] = 2.0f * v[e][c] - d[e][c];
  }
  trilerp(v, tx, ty, tz, out);
  return make_float3(out[0], out[1], out[2]);
}

// S4: RK-3 (Ralston) departure point of cell centre x, velocity in world units / dx;
// samp(p, out) samples the velocity
template <class Samp>
__device__ __forceinline__ void backtrace3(const SmokeDev& g, const float* x, const float* u0, float dt, Samp&& samp,
                                           float* xb) {
  const float s = dt * g.inv_dx;
  float k2[3], k3[3], p[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) p[c] = x[c] - 0.5f * s * u0[c];
  samp(p, k2);
#pragma unroll
  for (int c = 0; c < 3; ++c) p[c] = x[c] - 0.75f * s * k2[c];
  samp(p, k3);
#pragma unroll
  for (int c = 0; c < 3; ++c)
    xb[c] = x[c] - s * ((2.0f / 9.0f) * u0[c] + (1.0f / 3.0f) * k2[c] + (4.0f / 9.0f) * k3[c]);
}

__device__ __forceinline__ uint32_t salt_of(const SaltSrc& s) {
  return s.step ? qmpm::step_salt(s.seed_lo, s.seed_hi, (uint32_t)(*s.step * 256ull + s.sub)) : s.salt;
}

// pressure of cell (x, y, z)
__device__ __forceinline__ float p_at(const uint32_t* __restrict__ P, const SmokeDev& g, int x, int y, int z) {
  uint32_t w[SpecP::W + 1];
  ldrec<SpecP>(P, rec_of(g, x >> 1, y, z), w);
  return (x & 1) ? sdec<SpecP>(w, 1) : sdec<SpecP>(w, 0);
}

constexpr int kTZ = 32, kTY = 8;  // CTA tile (z, y); blockDim = (32, 8)

struct Here {
  int xr, y, z;
  bool valid;
  unsigned long long r;
};
__device__ __forceinline__ Here here(const SmokeDev& g) {
  Here h;
  h.z = blockIdx.x * kTZ + threadIdx.x;
  h.y = blockIdx.y * kTY + threadIdx.y;
  h.xr = blockIdx.z;
  h.valid = h.z < g.nz && h.y < g.ny;
  h.r = h.valid ? rec_of(g, h.xr, h.y, h.z) : 0ull;
  return h;
}

// the pressures of the 2 cells of record r and of their 6 neighbours each (Neumann: a
// neighbour outside the domain is the cell itself, S6): nb[c][0..5] = x-, x+, y-, y+, z-, z+
__device__ __forceinline__ void p_stencil(const uint32_t* __restrict__ P, const SmokeDev& g, const Here& h,
                                          float* pc, float (*nb)[6]) {
  uint32_t w[SpecP::W + 1];
  ldrec<SpecP>(P, h.r, w);
  pc[0] = sdec<SpecP>(w, 0);
  pc[1] = sdec<SpecP>(w, 1);
  nb[0][1] = pc[1];
  nb[1][0] = pc[0];
  nb[0][0] = h.xr > 0 ? p_at(P, g, 2 * h.xr - 1, h.y, h.z) : pc[0];
  nb[1][1] = h.xr + 1 < g.nxr ? p_at(P, g, 2 * h.xr + 2, h.y, h.z) : pc[1];
  const unsigned long long rn[4] = {h.y > 0 ? h.r - g.nz : h.r, h.y + 1 < g.ny ? h.r + g.nz : h.r,
                                    h.z > 0 ? h.r - 1 : h.r, h.z + 1 < g.nz ? h.r + 1 : h.r};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    ldrec<SpecP>(P, rn[q], w);
    nb[0][2 + q] = sdec<SpecP>(w, 0);
    nb[1][2 + q] = sdec<SpecP>(w, 1);
  }
}



// ---- x-marching plane tiles (jacobi, project, divergence) ----------------------------
// A CTA owns a (32 z, 8 y) column of records and marches kXM record planes along x.
// Per plane each record is decoded ONCE (by its owner) into a shared tile with a one-
// record halo in y and z (80 halo records per plane, decoded by warps 0-2); the x
// neighbours are the owner's previous / next records (registers, loaded one plane
// ahead).  Domain edges: halo / out-of-domain lanes load the CLAMPED record, which is
// the Neumann rule of S6 (an outside neighbour is the cell itself) -- the velocity
// march zeroes them instead (S5).
constexpr int kXM = 8;

struct March {
  int tz, ty, z, y, xs, xe;
  bool valid, has_halo;
  int hy, hz;                   // smem slot of this thread's halo record
  unsigned long long r0, hoff;  // in-plane offsets (clamped) of the own and halo record
  bool halo_outside;            // the halo record lies outside the domain
  unsigned long long plane;     // records per x plane (= cells per x plane)
};

__device__ __forceinline__ March march_setup(const SmokeDev& g) {
  March m;
  m.tz = threadIdx.x;
  m.ty = threadIdx.y;
  m.z = blockIdx.x * kTZ + m.tz;
  m.y = blockIdx.y * kTY + m.ty;
  m.xs = blockIdx.z * kXM;
  m.xe = min(m.xs + kXM, g.nxr);
  m.valid = m.z < g.nz && m.y < g.ny;
  m.plane = (unsigned long long)g.ny * g.nz;
  m.r0 = (unsigned long long)min(m.y, g.ny - 1) * g.nz + min(m.z, g.nz - 1);
  // halo: warp 0 -> row y0 - 1, warp 1 -> row y0 + 8, warp 2 lanes 0-7 -> column z0 - 1,
  // lanes 8-15 -> column z0 + 32
  const int y0 = blockIdx.y * kTY, z0 = blockIdx.x * kTZ;
  int hyg = 0, hzg = 0;
  m.has_halo = false;
  if (m.ty == 0 || m.ty == 1) {
    m.has_halo = true;
    hyg = m.ty == 0 ? y0 - 1 : y0 + kTY;
    hzg = z0 + m.tz;
    m.hy = m.ty == 0 ? 0 : kTY + 1;
    m.hz = m.tz + 1;
  } else if (m.ty == 2 && m.tz < 16) {
    m.has_halo = true;
    hyg = y0 + (m.tz & 7);
    hzg = m.tz < 8 ? z0 - 1 : z0 + kTZ;
    m.hy = (m.tz & 7) + 1;
    m.hz = m.tz < 8 ? 0 : kTZ + 1;
  } else {
    m.hy = m.hz = 0;
  }
  m.halo_outside = hyg < 0 || hyg >= g.ny || hzg < 0 || hzg >= g.nz;
  m.hoff = (unsigned long long)min(max(hyg, 0), g.ny - 1) * g.nz + min(max(hzg, 0), g.nz - 1);
  return m;
}

template <class SP>
__device__ __forceinline__ float2 dec2(const uint32_t* __restrict__ base, unsigned long long r) {
  uint32_t w[SP::W + 1];
  ldrec<SP>(base, r, w);
  return make_float2(sdec<SP>(w, 0), sdec<SP>(w, 1));
}

template <class SP>
__device__ __forceinline__ float2 dec2p(const uint32_t* __restrict__ q) {
  uint32_t w[SP::W + 1];
#pragma unroll
  for (int k = 0; k < SP::W; ++k) w[k] = __ldg(q + k);
  w[SP::W] = 0u;
  return make_float2(sdec<SP>(w, 0), sdec<SP>(w, 1));
}

// March the pressure field: for each record (xr, y, z) of the CTA's column calls
// f(m, xr, r, valid, pc, nb, d, wu) with r = the record index, the decoded pair pc, the
// Neumann neighbours nb[c][0..5] = x-, x+, y-, y+, z-, z+ of cell c, and (when the
// pointers are given) the two cells' divergence d[2] and the velocity record wu.  All
// threads call f (warp votes).  The own records are fetched two planes ahead and the
// div / velocity words at the top of the iteration, so their latency overlaps the tile
// exchange; addresses advance by one plane per iteration.
template <class F>
__device__ __forceinline__ void p_march(const uint32_t* __restrict__ P, const float* __restrict__ DIV,
                                        const uint32_t* __restrict__ U, const SmokeDev& g, F&& f) {
  constexpr int W = SpecP::W, WU = SpecU::W;
  __shared__ float2 tile[kTY + 2][kTZ + 2];
  const March m = march_setup(g);
  const unsigned long long pw = m.plane * W;
  unsigned long long r = (unsigned long long)m.xs * m.plane + m.r0;
  unsigned long long cell = 2ull * m.xs * m.plane + m.r0;
  const uint32_t* own = P + r * W;
  const uint32_t* halo = P + ((unsigned long long)m.xs * m.plane + m.hoff) * W;
  uint32_t wn[W + 1], wnn[W + 1];  // raw records xr + 1 and xr + 2
  wn[W] = wnn[W] = 0u;
  float2 prev = m.xs > 0 ? dec2p<SpecP>(own - pw) : make_float2(0.f, 0.f);
  float2 cur = dec2p<SpecP>(own);
#pragma unroll
  for (int k = 0; k < W; ++k) wn[k] = m.xs + 1 < g.nxr ? __ldg(own + pw + k) : 0u;
  for (int xr = m.xs; xr < m.xe; ++xr) {
    const bool has_next = xr + 1 < g.nxr;
#pragma unroll
    for (int k = 0; k < W; ++k) wnn[k] = xr + 2 < g.nxr ? __ldg(own + 2 * pw + k) : 0u;
    float d[2] = {0.f, 0.f};
    uint32_t wu[WU + 1];
    wu[WU] = 0u;
    if (DIV && m.valid) {
      d[0] = __ldg(DIV + cell);
      d[1] = __ldg(DIV + cell + m.plane);
    }
    if (U && m.valid) {
#pragma unroll
      for (int k = 0; k < WU; ++k) wu[k] = __ldg(U + r * WU + k);
    }
    float2 hv = make_float2(0.f, 0.f);
    if (m.has_halo) hv = dec2p<SpecP>(halo);
    __syncthreads();
    tile[m.ty + 1][m.tz + 1] = cur;
    if (m.has_halo) tile[m.hy][m.hz] = hv;
    __syncthreads();
    const float2 nxt = has_next ? make_float2(sdec<SpecP>(wn, 0), sdec<SpecP>(wn, 1)) : cur;
    const float2 ym = tile[m.ty][m.tz + 1], yp = tile[m.ty + 2][m.tz + 1];
    const float2 zm = tile[m.ty + 1][m.tz], zp = tile[m.ty + 1][m.tz + 2];
    float nb[2][6];
    nb[0][0] = xr > 0 ? prev.y : cur.x;
    nb[0][1] = cur.y;
    nb[1][0] = cur.x;
    nb[1][1] = has_next ? nxt.x : cur.y;
    nb[0][2] = ym.x;
    nb[1][2] = ym.y;
    nb[0][3] = yp.x;
    nb[1][3] = yp.y;
    nb[0][4] = zm.x;
    nb[1][4] = zm.y;
    nb[0][5] = zp.x;
    nb[1][5] = zp.y;
    const float pc[2] = {cur.x, cur.y};
    f(m, xr, r, m.valid, pc, nb, d, wu);
    prev = cur;
    cur = nxt;
#pragma unroll
    for (int k = 0; k < W; ++k) wn[k] = wnn[k];
    own += pw;
    halo += pw;
    r += m.plane;
    cell += 2 * m.plane;
  }
}

// ---- advection windows ---------------------------------------------------------------
// An advection CTA marches its (32 z x 8 y) record column along x like the stencils,
// keeping a ring of 3 record planes (xr - 1, xr, xr + 1 = cells 2xr - 2 .. 2xr + 3) of
// DECODED velocity with a kH-cell y/z halo in shared memory (float4 per cell), so the
// backtrace and the final sample read corners with LDS instead of re-decoding records
// (a corner pair outside the window -- a departure point more than ~2 cells away -- is
// decoded from global memory, with identical arithmetic).  The reflection's q = 2 u_h -
// u~ and the density get rings of their own.
constexpr int kH = 2;
constexpr int kWY = kTY + 2 * kH, kWZ = kTZ + 2 * kH;  // window tile (records)
constexpr int kRing = 3 * kWY * kWZ * 2;                // float4 cells per ring

struct Win {
  int xr, y0, z0;
  __device__ __forceinline__ bool has(int i, int j, int k) const {
    return i >= 2 * xr - 2 && i <= 2 * xr + 2 && j >= y0 - kH && j < y0 + kTY + kH - 1 && k >= z0 - kH &&
           k < z0 + kTZ + kH - 1;
  }
  // index of cell (i, j, k) in a ring (float4 units): [slot][cell parity][y][z], so a
  // warp's lanes (consecutive z) read consecutive 16-byte slots (no bank conflicts)
  __device__ __forceinline__ int at(int i, int j, int k) const {
    const int slot = ((i >> 1) + 3) % 3;
    return ((slot * 2 + (i & 1)) * kWY + (j - y0 + kH)) * kWZ + (k - z0 + kH);
  }
  // sample of ring R at p; out of the window: sample_global(U, UR) (identical arithmetic)
  __device__ __forceinline__ void sample(const SmokeDev& g, const float4* R, const uint32_t* U, const uint32_t* UR,
                                         const float* p, float* out) const {
    int i, j, k;
    float tx, ty, tz;
    corner(p[0], g.nx, i, tx);
    corner(p[1], g.ny, j, ty);
    corner(p[2], g.nz, k, tz);
    if (has(i, j, k)) {
      float v[8][3];
      cube(R, i, j, k, v);
      trilerp(v, tx, ty, tz, out);
    } else {
      const float3 r = sample_global(U, UR, g, p[0], p[1], p[2]);
      out[0] = r.x, out[1] = r.y, out[2] = r.z;
    }
  }
  // the 8 corners of the block at (i, j, k) from ring R (has(i, j, k) must hold)
  __device__ __forceinline__ void cube(const float4* R, int i, int j, int k, float (*v)[3]) const {
    const int a = at(i, j, k), b = at(i + 1, j, k);
#pragma unroll
    for (int dj = 0; dj < 2; ++dj)
#pragma unroll
      for (int dk = 0; dk < 2; ++dk) {
        const int o = dj * kWZ + dk;
        const float4 A = R[a + o], B = R[b + o];
        float* va = v[(dj * 2 + dk) * 2];
        float* vb = v[(dj * 2 + dk) * 2 + 1];
        va[0] = A.x, va[1] = A.y, va[2] = A.z, vb[0] = B.x, vb[1] = B.y, vb[2] = B.z;
      }
  }
};

// Ring fills are software-pipelined: the raw words of plane q are loaded into registers
// (each thread owns tile records t and t + 256 of the 12 x 36 window tile) one plane
// before they are decoded into the ring, so the loads overlap the previous plane's work.
constexpr int kFillPer = (kWY * kWZ + kTY * kTZ - 1) / (kTY * kTZ);  // 2

template <bool REFL, bool RHO>
struct Fill {
  uint32_t u[kFillPer][SpecU::W];
  uint32_t ur[REFL ? kFillPer : 1][SpecU::W];
  float d[RHO ? kFillPer : 1][2];
  bool ok[kFillPer];
};

template <bool REFL, bool RHO>
__device__ __forceinline__ void fill_load(const uint32_t* __restrict__ U, const uint32_t* __restrict__ UR,
                                          const float* __restrict__ D, const SmokeDev& g, const Win& w, int q,
                                          Fill<REFL, RHO>& F) {
  const unsigned long long plane = (unsigned long long)g.ny * g.nz;
#pragma unroll
  for (int e = 0; e < kFillPer; ++e) {
    const int t = threadIdx.y * kTZ + threadIdx.x + e * kTY * kTZ;
    const int jy = t / kWZ, kz = t - jy * kWZ;
    const int j = w.y0 - kH + jy, k = w.z0 - kH + kz;
    F.ok[e] = t < kWY * kWZ && q < g.nxr && j >= 0 && j < g.ny && k >= 0 && k < g.nz;
    if (!F.ok[e]) continue;
    const unsigned long long r = (unsigned long long)q * plane + (unsigned long long)j * g.nz + k;
#pragma unroll
    for (int c = 0; c < SpecU::W; ++c) F.u[e][c] = __ldg(U + r * SpecU::W + c);
    if (REFL) {
#pragma unroll
      for (int c = 0; c < SpecU::W; ++c) F.ur[e][c] = __ldg(UR + r * SpecU::W + c);
    }
    if (RHO) {
      const unsigned long long c = 2ull * q * plane + (unsigned long long)j * g.nz + k;
      F.d[e][0] = __ldg(D + c);
      F.d[e][1] = __ldg(D + c + plane);
    }
  }
}

template <bool REFL, bool RHO>
__device__ __forceinline__ void fill_store(const Fill<REFL, RHO>& F, int q, float4* ru, float4* rr, float* rd) {
  const int slot = (q + 3) % 3;
#pragma unroll
  for (int e = 0; e < kFillPer; ++e) {
    if (!F.ok[e]) continue;
    const int t = threadIdx.y * kTZ + threadIdx.x + e * kTY * kTZ;
    const int o = slot * 2 * kWY * kWZ + t;  // t = jy * kWZ + kz; cell 1 one plane further
    uint32_t wv[SpecU::W + 1];
#pragma unroll
    for (int c = 0; c < SpecU::W; ++c) wv[c] = F.u[e][c];
    wv[SpecU::W] = 0u;
    float u[6];
#pragma unroll
    for (int f = 0; f < 6; ++f) u[f] = sdec<SpecU>(wv, f);
    ru[o] = make_float4(u[0], u[1], u[2], 0.f);
    ru[o + kWY * kWZ] = make_float4(u[3], u[4], u[5], 0.f);
    if (REFL) {
#pragma unroll
      for (int c = 0; c < SpecU::W; ++c) wv[c] = F.ur[e][c];
      float a[6];
#pragma unroll
      for (int f = 0; f < 6; ++f) a[f] = 2.0f * u[f] - sdec<SpecU>(wv, f);
      rr[o] = make_float4(a[0], a[1], a[2], 0.f);
      rr[o + kWY * kWZ] = make_float4(a[3], a[4], a[5], 0.f);
    }
    if (RHO) {
      rd[o] = F.d[e][0];
      rd[o + kWY * kWZ] = F.d[e][1];
    }
  }
}

// march skeleton of the advection kernels: f(xr, y, z, r, valid, win) per record plane,
// once the ring holds planes xr - 1 .. xr + 1
// B (nullable): the buoyancy density, fetched for the thread's two cells one plane ahead
// and passed to f as bq
template <bool REFL, bool RHO, class F>
__device__ __forceinline__ void adv_march(const uint32_t* __restrict__ U, const uint32_t* __restrict__ UR,
                                          const float* __restrict__ D, const float* __restrict__ B, const SmokeDev& g,
                                          float4* ru, float4* rr, float* rd, F&& f) {
  Win w;
  w.y0 = blockIdx.y * kTY;
  w.z0 = blockIdx.x * kTZ;
  const int xs = blockIdx.z * kXM, xe = min(xs + kXM, g.nxr);
  const int y = w.y0 + threadIdx.y, z = w.z0 + threadIdx.x;
  const bool valid = y < g.ny && z < g.nz;
  Fill<REFL, RHO> fl;
  if (xs > 0) {
    fill_load(U, UR, D, g, w, xs - 1, fl);
    fill_store(fl, xs - 1, ru, rr, rd);
  }
  fill_load(U, UR, D, g, w, xs, fl);
  fill_store(fl, xs, ru, rr, rd);
  fill_load(U, UR, D, g, w, xs + 1, fl);  // q >= nxr loads nothing
  const unsigned long long cplane = (unsigned long long)g.ny * g.nz;
  const unsigned long long c0 = (unsigned long long)y * g.nz + z;
  float2 bq = make_float2(0.f, 0.f);
  if (B && valid) bq = make_float2(__ldg(B + 2ull * xs * cplane + c0), __ldg(B + (2ull * xs + 1) * cplane + c0));
  for (int xr = xs; xr < xe; ++xr) {
    w.xr = xr;
    fill_store(fl, xr + 1, ru, rr, rd);
    __syncthreads();
    if (xr + 1 < xe) fill_load(U, UR, D, g, w, xr + 2, fl);
    float2 bn = make_float2(0.f, 0.f);
    if (B && valid && xr + 1 < xe)
      bn = make_float2(__ldg(B + 2ull * (xr + 1) * cplane + c0), __ldg(B + (2ull * xr + 3) * cplane + c0));
    const unsigned long long r = valid ? ((unsigned long long)xr * g.ny + y) * g.nz + z : 0ull;
    f(xr, y, z, r, valid, w, bq);
    bq = bn;
    __syncthreads();
  }
}

// p_march with two records per thread (rows ty and ty + 8 of a 16-row tile): the loop,
// barrier, halo and address overheads are paid once per two records.  Same contract
// as p_march; f is called for the upper row, then the lower row.  blockDim = (32, 8),
// gridDim.y = ceil(ny / 16).
constexpr int kTY2 = 2 * kTY;

template <class F>
__device__ __forceinline__ void p_march2(const uint32_t* __restrict__ P, const float* __restrict__ DIV,
                                         const uint32_t* __restrict__ U, const SmokeDev& g, F&& f) {
  constexpr int W = SpecP::W, WU = SpecU::W;
  __shared__ float2 tile[kTY2 + 2][kTZ + 2];
  const int tz = threadIdx.x, ty = threadIdx.y;
  const int y0 = blockIdx.y * kTY2, z0 = blockIdx.x * kTZ;
  const int z = z0 + tz;
  const int xs = blockIdx.z * kXM, xe = min(xs + kXM, g.nxr);
  const unsigned long long plane = (unsigned long long)g.ny * g.nz, pw = plane * W;
  March m[2];  // per row: the fields the callbacks read (y, z, valid, r0, plane)
  unsigned long long r[2], cell[2];
  const uint32_t* own[2];
  float2 prev[2], cur[2];
  uint32_t wn[2][W + 1], wnn[2][W + 1];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    m[k].tz = tz;
    m[k].ty = ty + k * kTY;
    m[k].z = z;
    m[k].y = y0 + ty + k * kTY;
    m[k].xs = xs;
    m[k].xe = xe;
    m[k].valid = z < g.nz && m[k].y < g.ny;
    m[k].plane = plane;
    m[k].r0 = (unsigned long long)min(m[k].y, g.ny - 1) * g.nz + min(z, g.nz - 1);
    m[k].has_halo = false;
    r[k] = (unsigned long long)xs * plane + m[k].r0;
    cell[k] = 2ull * xs * plane + m[k].r0;
    own[k] = P + r[k] * W;
    prev[k] = xs > 0 ? dec2p<SpecP>(own[k] - pw) : make_float2(0.f, 0.f);
    cur[k] = dec2p<SpecP>(own[k]);
    wn[k][W] = wnn[k][W] = 0u;
#pragma unroll
    for (int q = 0; q < W; ++q) wn[k][q] = xs + 1 < g.nxr ? __ldg(own[k] + pw + q) : 0u;
  }
  // halo: warp 0 -> row y0 - 1, warp 1 -> row y0 + 16, warp 2 lanes 0-15 -> column z0 - 1,
  // warp 3 lanes 0-15 -> column z0 + 32 (rows y0 .. y0 + 15); clamped = Neumann (S6)
  bool has_halo = false;
  int hy = 0, hz = 0, hyg = 0, hzg = 0;
  if (ty == 0 || ty == 1) {
    has_halo = true;
    hyg = ty == 0 ? y0 - 1 : y0 + kTY2;
    hzg = z;
    hy = ty == 0 ? 0 : kTY2 + 1;
    hz = tz + 1;
  } else if ((ty == 2 || ty == 3) && tz < kTY2) {
    has_halo = true;
    hyg = y0 + tz;
    hzg = ty == 2 ? z0 - 1 : z0 + kTZ;
    hy = tz + 1;
    hz = ty == 2 ? 0 : kTZ + 1;
  }
  const unsigned long long hoff =
      (unsigned long long)min(max(hyg, 0), g.ny - 1) * g.nz + min(max(hzg, 0), g.nz - 1);
  const uint32_t* halo = P + ((unsigned long long)xs * plane + hoff) * W;
  for (int xr = xs; xr < xe; ++xr) {
    const bool has_next = xr + 1 < g.nxr;
    float d[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
    uint32_t wu[2][WU + 1];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
#pragma unroll
      for (int q = 0; q < W; ++q) wnn[k][q] = xr + 2 < g.nxr ? __ldg(own[k] + 2 * pw + q) : 0u;
      if (DIV && m[k].valid) {
        d[k][0] = __ldg(DIV + cell[k]);
        d[k][1] = __ldg(DIV + cell[k] + plane);
      }
      wu[k][WU] = 0u;
      if (U && m[k].valid) {
#pragma unroll
        for (int q = 0; q < WU; ++q) wu[k][q] = __ldg(U + r[k] * WU + q);
      }
    }
    float2 hv = make_float2(0.f, 0.f);
    if (has_halo) hv = dec2p<SpecP>(halo);
    __syncthreads();
    tile[ty + 1][tz + 1] = cur[0];
    tile[ty + kTY + 1][tz + 1] = cur[1];
    if (has_halo) tile[hy][hz] = hv;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int row = ty + k * kTY + 1;
      const float2 nxt = has_next ? make_float2(sdec<SpecP>(wn[k], 0), sdec<SpecP>(wn[k], 1)) : cur[k];
      const float2 ym = tile[row - 1][tz + 1], yp = tile[row + 1][tz + 1];
      const float2 zm = tile[row][tz], zp = tile[row][tz + 2];
      float nb[2][6];
      nb[0][0] = xr > 0 ? prev[k].y : cur[k].x;
      nb[0][1] = cur[k].y;
      nb[1][0] = cur[k].x;
      nb[1][1] = has_next ? nxt.x : cur[k].y;
      nb[0][2] = ym.x;
      nb[1][2] = ym.y;
      nb[0][3] = yp.x;
      nb[1][3] = yp.y;
      nb[0][4] = zm.x;
      nb[1][4] = zm.y;
      nb[0][5] = zp.x;
      nb[1][5] = zp.y;
      const float pc[2] = {cur[k].x, cur[k].y};
      f(m[k], xr, r[k], m[k].valid, pc, nb, d[k], wu[k]);
      prev[k] = cur[k];
      cur[k] = nxt;
#pragma unroll
      for (int q = 0; q < W; ++q) wn[k][q] = wnn[k][q];
      own[k] += pw;
      r[k] += plane;
      cell[k] += 2 * plane;
    }
    halo += pw;
  }
}
// ---- two Jacobi sweeps per launch (temporal blocking, S6) -----------------------------
// A CTA marches a (32 z x 16 y) record column along x (kXM2 planes) keeping three planes
// of the input pressure L0 (2-record y/z halo) and of the first sweep's pressure L1
// (1-record halo) decoded in shared memory.  Per plane: the next L0 plane is filled
// (raw words fetched a plane ahead), L1 is computed on the halo-extended plane and
// quantized exactly as the single sweep stores it (encode_record, then decode: the
// same dithered code, never written to memory), then the second sweep of the interior
// is encoded and stored.  Domain walls: every neighbour index is clamped into the
// domain (Neumann, S6), so halo slots outside it are never read.  The result is bit-
// identical to two qsmoke_jacobi launches (tests/test_gpu_smoke.py: graph vs chain).
constexpr int kXM2 = 16;
constexpr int kJY = 2 * kTY, kJZ = kTZ;             // interior tile (records)
constexpr int kL0Y = kJY + 4, kL0Z = kJZ + 4;       // L0 tile: 2-record halo
constexpr int kL1Y = kJY + 2, kL1Z = kJZ + 2;       // L1 tile: 1-record halo
constexpr int kL0N = kL0Y * kL0Z, kL1N = kL1Y * kL1Z;
constexpr int kL0Per = (kL0N + 255) / 256, kL1Per = (kL1N + 255) / 256;

struct Jac2 {
  int y0, z0;
  __device__ __forceinline__ int i0(int slot, int y, int z) const {
    return (slot * kL0Y + (y - y0 + 2)) * kL0Z + (z - z0 + 2);
  }
  __device__ __forceinline__ int i1(int slot, int y, int z) const {
    return (slot * kL1Y + (y - y0 + 1)) * kL1Z + (z - z0 + 1);
  }
};

// the single sweep's arithmetic (qsmoke_jacobi), both cells of a record at once
__device__ __forceinline__ float2 jacobi_pair(float xm0, float xp0, float xm1, float xp1, float2 ym, float2 yp,
                                              float2 zm, float2 zp, float d0, float d1, float dx2) {
  const float2 sx = __fadd2_rn(make_float2(xm0, xm1), make_float2(xp0, xp1));
  const float2 sy = __fadd2_rn(ym, yp);
  const float2 sz = __fadd2_rn(zm, zp);
  const float2 s2 = __fadd2_rn(__fadd2_rn(sx, sy), sz);
  return __fmul2_rn(__ffma2_rn(make_float2(-dx2, -dx2), make_float2(d0, d1), s2),
                    make_float2(1.0f / 6.0f, 1.0f / 6.0f));
}

}  // namespace smoke

extern "C" __global__ void __launch_bounds__(256)
    qsmoke_jacobi2(const uint32_t* __restrict__ P, const float* __restrict__ div, SmokeDev g, SaltSrc ss1,
                   SaltSrc ss2, uint32_t* __restrict__ out) {
  using namespace smoke;
  constexpr int W = SpecP::W;
  __shared__ float2 L0[3 * kL0N];
  __shared__ float2 L1[3 * kL1N];
  const int tid = threadIdx.y * kTZ + threadIdx.x;
  const int y0 = blockIdx.y * kJY, z0 = blockIdx.x * kJZ;
  const int xs = blockIdx.z * kXM2, xe = min(xs + kXM2, g.nxr);
  const unsigned long long plane = (unsigned long long)g.ny * g.nz;
  const uint32_t salt1 = salt_of(ss1), salt2 = salt_of(ss2);
  // per-thread constants (the (y, z) of each owned slot does not change along x)
  unsigned goff0[kL0Per];  // in-plane record offset of fill slot e (valid when in0 bit e)
  unsigned in0 = 0u;
#pragma unroll
  for (int e = 0; e < kL0Per; ++e) {
    const int t = tid + 256 * e;
    const int y = y0 - 2 + t / kL0Z, z = z0 - 2 + t % kL0Z;
    const bool ok = t < kL0N && y >= 0 && y < g.ny && z >= 0 && z < g.nz;
    in0 |= ok ? (1u << e) : 0u;
    goff0[e] = ok ? (unsigned)(y * g.nz + z) : 0u;
  }
  // sweep-1 slots: in-plane offset, L0 centre index and the clamped neighbour deltas
  unsigned goff1[kL1Per];
  int c1[kL1Per], dym[kL1Per], dyp[kL1Per], dzm[kL1Per], dzp[kL1Per];
  unsigned in1 = 0u;
#pragma unroll
  for (int e = 0; e < kL1Per; ++e) {
    const int t = tid + 256 * e;
    const int y = y0 - 1 + t / kL1Z, z = z0 - 1 + t % kL1Z;
    const bool ok = t < kL1N && y >= 0 && y < g.ny && z >= 0 && z < g.nz;
    in1 |= ok ? (1u << e) : 0u;
    goff1[e] = ok ? (unsigned)(y * g.nz + z) : 0u;
    c1[e] = (y - y0 + 2) * kL0Z + (z - z0 + 2);
    dym[e] = y > 0 ? -kL0Z : 0;
    dyp[e] = y + 1 < g.ny ? kL0Z : 0;
    dzm[e] = z > 0 ? -1 : 0;
    dzp[e] = z + 1 < g.nz ? 1 : 0;
  }
  // sweep-2 rows
  int c2[2], eym[2], eyp[2], ezm[2], ezp[2];
  unsigned goff2[2];
  bool in2[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int y = y0 + threadIdx.y + k * kTY, z = z0 + threadIdx.x;
    in2[k] = y < g.ny && z < g.nz;
    goff2[k] = in2[k] ? (unsigned)(y * g.nz + z) : 0u;
    c2[k] = (y - y0 + 1) * kL1Z + (z - z0 + 1);
    eym[k] = y > 0 ? -kL1Z : 0;
    eyp[k] = y + 1 < g.ny ? kL1Z : 0;
    ezm[k] = z > 0 ? -1 : 0;
    ezp[k] = z + 1 < g.nz ? 1 : 0;
  }
  uint32_t raw[kL0Per][W];
  auto fetch = [&](int q) {
    if (q < 0 || q >= g.nxr) return;
    const uint32_t* base = P + (unsigned long long)q * plane * W;
#pragma unroll
    for (int e = 0; e < kL0Per; ++e)
      if ((in0 >> e) & 1u) {
#pragma unroll
        for (int k = 0; k < W; ++k) raw[e][k] = __ldg(base + (unsigned long long)goff0[e] * W + k);
      }
  };
  auto store0 = [&](int q, int slot) {
    if (q < 0 || q >= g.nxr) return;
#pragma unroll
    for (int e = 0; e < kL0Per; ++e)
      if ((in0 >> e) & 1u) {
        uint32_t w[W + 1];
#pragma unroll
        for (int k = 0; k < W; ++k) w[k] = raw[e][k];
        w[W] = 0u;
        L0[slot * kL0N + tid + 256 * e] = make_float2(sdec<SpecP>(w, 0), sdec<SpecP>(w, 1));
      }
  };
  // first sweep on plane q: L0 slots (sm, s0, sp) = planes q - 1, q, q + 1; L1 slot t1
  auto sweep1 = [&](int q, int sm, int s0, int sp, int t1) {
    const bool qok = q >= 0 && q < g.nxr;
    const float* dq = div + 2ull * q * plane;
    const unsigned long long rq = (unsigned long long)q * plane;
#pragma unroll
    for (int e = 0; e < kL1Per; ++e) {
      const bool valid = qok && ((in1 >> e) & 1u);
      float v[2] = {0.f, 0.f};
      const unsigned long long r = rq + goff1[e];
      if (valid) {
        const float2* S0 = L0 + s0 * kL0N + c1[e];
        const float2 c = S0[0];
        const float xm0 = q > 0 ? L0[sm * kL0N + c1[e]].y : c.x;
        const float xp1 = q + 1 < g.nxr ? L0[sp * kL0N + c1[e]].x : c.y;
        const float2 rr = jacobi_pair(xm0, c.y, c.x, xp1, S0[dym[e]], S0[dyp[e]], S0[dzm[e]], S0[dzp[e]],
                                      __ldg(dq + goff1[e]), __ldg(dq + plane + goff1[e]), g.dx2);
        v[0] = rr.x;
        v[1] = rr.y;
      }
      const uint32_t hh = SpecP::DITHER ? qmpm::mix32((uint32_t)r ^ salt1) : 0u;
      uint32_t w[W + 1];
      qmpm::encode_record<SpecP>(v, hh, valid, w, nullptr);
      if (valid) L1[t1 * kL1N + tid + 256 * e] = make_float2(sdec<SpecP>(w, 0), sdec<SpecP>(w, 1));
    }
  };
  // ring slots rotate: plane q lives in slot (q - xs + 2) % 3 (no modulo in the loop)
  int a0 = 0, a1 = 1, a2 = 2;  // L0 slots of planes xs - 2, xs - 1, xs
  fetch(xs - 2);
  store0(xs - 2, a0);
  fetch(xs - 1);
  store0(xs - 1, a1);
  fetch(xs);
  store0(xs, a2);
  __syncthreads();
  int b0 = 0, b1 = 1, b2 = 2;  // L1 slots of planes xs - 1, xs, xs + 1
  sweep1(xs - 1, a0, a1, a2, b0);
  __syncthreads();
  fetch(xs + 1);
  store0(xs + 1, a0);  // plane xs - 2's slot: L0 slots now xs - 1 (a1), xs (a2), xs + 1 (a0)
  {
    const int t = a0;
    a0 = a1, a1 = a2, a2 = t;  // a0, a1, a2 = planes xs - 1, xs, xs + 1
  }
  __syncthreads();
  sweep1(xs, a0, a1, a2, b1);
  fetch(xs + 2);
  for (int xr = xs; xr < xe; ++xr) {
    // here: L0 slots a0, a1, a2 = planes xr - 1, xr, xr + 1; L1 slots b0, b1 = xr - 1, xr
    __syncthreads();
    store0(xr + 2, a0);  // plane xr - 1's slot
    {
      const int t = a0;
      a0 = a1, a1 = a2, a2 = t;  // planes xr, xr + 1, xr + 2
    }
    __syncthreads();
    fetch(xr + 3);
    sweep1(xr + 1, a0, a1, a2, b2);
    __syncthreads();
    const unsigned long long rq = (unsigned long long)xr * plane;
    const float* dq = div + 2ull * xr * plane;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      float v[2] = {0.f, 0.f};
      const unsigned long long r = rq + goff2[k];
      if (in2[k]) {
        const float2* S1 = L1 + b1 * kL1N + c2[k];
        const float2 c = S1[0];
        const float xm0 = xr > 0 ? L1[b0 * kL1N + c2[k]].y : c.x;
        const float xp1 = xr + 1 < g.nxr ? L1[b2 * kL1N + c2[k]].x : c.y;
        const float2 rr = jacobi_pair(xm0, c.y, c.x, xp1, S1[eym[k]], S1[eyp[k]], S1[ezm[k]], S1[ezp[k]],
                                      __ldg(dq + goff2[k]), __ldg(dq + plane + goff2[k]), g.dx2);
        v[0] = rr.x;
        v[1] = rr.y;
      }
      const uint32_t hh = SpecP::DITHER ? qmpm::mix32((uint32_t)r ^ salt2) : 0u;
      uint32_t o[W + 1];
      qmpm::encode_record<SpecP>(v, hh, in2[k], o, nullptr);
      if (in2[k]) qmpm::store_words<SpecP>(out + r * W, o);
    }
    const int t = b0;
    b0 = b1, b1 = b2, b2 = t;
  }
}

namespace smoke {
}  // namespace smoke

// ------------------------------------------------------------------ entry points
template <bool REFL>
__device__ __forceinline__ void advect_u_body(const uint32_t* __restrict__ uv, const uint32_t* __restrict__ ur,
                                              const float* __restrict__ rho, const SmokeDev& g, float dt, float bdt,
                                              const SaltSrc& ss, uint32_t* __restrict__ out, float* __restrict__ dbg) {
  constexpr int W = SpecU::W;
  extern __shared__ float4 smem_adv[];
  float4* ru = smem_adv;
  float4* rr = REFL ? smem_adv + smoke::kRing : nullptr;
  const uint32_t salt = smoke::salt_of(ss);
  smoke::adv_march<REFL, false>(uv, ur, nullptr, REFL ? nullptr : rho, g, ru, rr, nullptr,
                                [&](int xr, int y, int z, unsigned long long r, bool valid, const smoke::Win& w,
                                    float2 bq) {
    auto samp_u = [&](const float* p, float* o) { w.sample(g, ru, uv, nullptr, p, o); };
    float v[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (valid) {
#pragma unroll(kAdvUnroll)
      for (int c2 = 0; c2 < 2; ++c2) {
        const int x = 2 * xr + c2;
        const float xp[3] = {(float)x, (float)y, (float)z};
        const float4 U0 = ru[w.at(x, y, z)];
        const float u0[3] = {U0.x, U0.y, U0.z};
        float xb[3], q[3];
        smoke::backtrace3(g, xp, u0, dt, samp_u, xb);
        if (REFL)
          w.sample(g, rr, uv, ur, xb, q);
        else
          samp_u(xb, q);
        if (!REFL && rho) q[1] += bdt * (c2 == 0 ? bq.x : bq.y);
#pragma unroll
        for (int c = 0; c < 3; ++c) v[3 * c2 + c] = q[c];
      }
      if (dbg) {
#pragma unroll
        for (int f = 0; f < 6; ++f) dbg[r * 6 + f] = v[f];
      }
    }
    const uint32_t hh = SpecU::DITHER ? qmpm::mix32((uint32_t)r ^ salt) : 0u;
    uint32_t o[W + 1];
    qmpm::encode_record<SpecU>(v, hh, valid, o, nullptr);
    if (valid) qmpm::store_words<SpecU>(out + r * W, o);
  });
}

extern "C" __global__ void __launch_bounds__(256, QSMOKE_ADV_MINB)
    qsmoke_advect_u(const uint32_t* __restrict__ uv, const uint32_t* __restrict__ ur, const float* __restrict__ rho,
                    SmokeDev g, float dt, float bdt, SaltSrc ss, uint32_t* __restrict__ out, float* __restrict__ dbg) {
  advect_u_body<false>(uv, nullptr, rho, g, dt, bdt, ss, out, dbg);
}

// the reflection's advection (S8): q = 2 u_vel - u_refl sampled at the departure point
extern "C" __global__ void __launch_bounds__(256, QSMOKE_ADV_MINB)
    qsmoke_advect_refl(const uint32_t* __restrict__ uv, const uint32_t* __restrict__ ur, const float* __restrict__ rho,
                       SmokeDev g, float dt, float bdt, SaltSrc ss, uint32_t* __restrict__ out,
                       float* __restrict__ dbg) {
  advect_u_body<true>(uv, ur, nullptr, g, dt, 0.0f, ss, out, dbg);
}

// S5 on the x march: neighbours outside the domain are 0 (halo / x loads masked)
extern "C" __global__ void __launch_bounds__(256, QSMOKE_DIV_MINB)
    qsmoke_div(const uint32_t* __restrict__ U, SmokeDev g, float* __restrict__ div) {
  __shared__ float4 tile[smoke::kTY + 2][smoke::kTZ + 2];  // (uy0, uy1, uz0, uz1)
  const smoke::March m = smoke::march_setup(g);
  auto rec6 = [&](unsigned long long r, float* u) {
    uint32_t w[SpecU::W + 1];
    smoke::ldrec<SpecU>(U, r, w);
#pragma unroll
    for (int f = 0; f < 6; ++f) u[f] = qmpm::sdec<SpecU>(w, f);
  };
  float prev[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, cur[6], nxt[6];
  if (m.xs > 0) rec6((m.xs - 1) * m.plane + m.r0, prev);
  rec6(m.xs * m.plane + m.r0, cur);
  for (int xr = m.xs; xr < m.xe; ++xr) {
#pragma unroll
    for (int f = 0; f < 6; ++f) nxt[f] = 0.0f;
    if (xr + 1 < g.nxr) rec6((xr + 1) * m.plane + m.r0, nxt);
    float4 hv = make_float4(0.f, 0.f, 0.f, 0.f);
    if (m.has_halo && !m.halo_outside) {
      float h6[6];
      rec6(xr * m.plane + m.hoff, h6);
      hv = make_float4(h6[1], h6[4], h6[2], h6[5]);
    }
    __syncthreads();
    tile[m.ty + 1][m.tz + 1] = m.valid ? make_float4(cur[1], cur[4], cur[2], cur[5]) : make_float4(0.f, 0.f, 0.f, 0.f);
    if (m.has_halo) tile[m.hy][m.hz] = hv;
    __syncthreads();
    const float4 ym = tile[m.ty][m.tz + 1], yp = tile[m.ty + 2][m.tz + 1];
    const float4 zm = tile[m.ty + 1][m.tz], zp = tile[m.ty + 1][m.tz + 2];
    if (m.valid) {
      const float xm = xr > 0 ? prev[3] : 0.0f, xp = xr + 1 < g.nxr ? nxt[0] : 0.0f;
      const float d0 = ((cur[3] - xm) + (yp.x - ym.x) + (zp.z - zm.z)) * g.half_inv_dx;
      const float d1 = ((xp - cur[0]) + (yp.y - ym.y) + (zp.w - zm.w)) * g.half_inv_dx;
      const unsigned long long c = 2ull * xr * m.plane + m.r0;
      div[c] = d0;
      div[c + m.plane] = d1;
    }
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      prev[f] = cur[f];
      cur[f] = nxt[f];
    }
  }
}

extern "C" __global__ void __launch_bounds__(256, QSMOKE_JACOBI_MINB)
    qsmoke_jacobi(const uint32_t* __restrict__ P, const float* __restrict__ div, SmokeDev g, SaltSrc ss,
                  uint32_t* __restrict__ out, float* __restrict__ dbg) {
  constexpr int W = SpecP::W;
  const uint32_t salt = smoke::salt_of(ss);
  smoke::p_march2(P, div, nullptr, g, [&](const smoke::March& m, int xr, unsigned long long r, bool valid,
                                          const float* pc, const float (*nb)[6], const float* d, const uint32_t* wu) {
    float v[2] = {0.f, 0.f};
    if (valid) {
      // both cells at once in packed FP32x2 (FADD2 / FFMA2 / FMUL2)
      const float2 r2 = smoke::jacobi_pair(nb[0][0], nb[0][1], nb[1][0], nb[1][1], make_float2(nb[0][2], nb[1][2]),
                                           make_float2(nb[0][3], nb[1][3]), make_float2(nb[0][4], nb[1][4]),
                                           make_float2(nb[0][5], nb[1][5]), d[0], d[1], g.dx2);
      v[0] = r2.x;
      v[1] = r2.y;
      if (dbg) {
        dbg[2 * r] = v[0];
        dbg[2 * r + 1] = v[1];
      }
    }
    const uint32_t hh = SpecP::DITHER ? qmpm::mix32((uint32_t)r ^ salt) : 0u;
    uint32_t o[W + 1];
    qmpm::encode_record<SpecP>(v, hh, valid, o, nullptr);
    if (valid) qmpm::store_words<SpecP>(out + r * W, o);
  });
}

extern "C" __global__ void __launch_bounds__(256, QSMOKE_PROJECT_MINB)
    qsmoke_project(const uint32_t* __restrict__ U, const uint32_t* __restrict__ P, SmokeDev g, SaltSrc ss,
                   uint32_t* __restrict__ out, float* __restrict__ dbg) {
  constexpr int W = SpecU::W;
  const uint32_t salt = smoke::salt_of(ss);
  smoke::p_march2(P, nullptr, U, g, [&](const smoke::March& m, int xr, unsigned long long r, bool valid,
                                        const float* pc, const float (*nb)[6], const float* d, const uint32_t* wu) {
    float v[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (valid) {
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int a = 0; a < 3; ++a)
          v[3 * k + a] = qmpm::sdec<SpecU>(wu, 3 * k + a) - (nb[k][2 * a + 1] - nb[k][2 * a]) * g.half_inv_dx;
      // S7: wall-normal components zeroed in the boundary layer
      if (xr == 0) v[0] = 0.0f;
      if (xr + 1 == g.nxr) v[3] = 0.0f;
      if (m.y == 0 || m.y + 1 == g.ny) v[1] = v[4] = 0.0f;
      if (m.z == 0 || m.z + 1 == g.nz) v[2] = v[5] = 0.0f;
      if (dbg) {
#pragma unroll
        for (int f = 0; f < 6; ++f) dbg[r * 6 + f] = v[f];
      }
    }
    const uint32_t hh = SpecU::DITHER ? qmpm::mix32((uint32_t)r ^ salt) : 0u;
    uint32_t o[W + 1];
    qmpm::encode_record<SpecU>(v, hh, valid, o, nullptr);
    if (valid) qmpm::store_words<SpecU>(out + r * W, o);
  });
}

// density (S8): per record, backtrace on the velocity window, sample the density window
extern "C" __global__ void __launch_bounds__(256, QSMOKE_ADV_MINB)
    qsmoke_advect_rho(const float* __restrict__ rho, const uint32_t* __restrict__ U, SmokeDev g, float dt,
                      float* __restrict__ out, unsigned long long* __restrict__ tick) {
  extern __shared__ float4 smem_adv[];
  float4* ru = smem_adv;
  float* rd = reinterpret_cast<float*>(smem_adv + smoke::kRing);
  // the last kernel of a step advances the device step counter (nothing here reads it)
  if (tick && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0 && threadIdx.y == 0)
    *tick += 1ull;
  smoke::adv_march<false, true>(U, nullptr, rho, nullptr, g, ru, nullptr, rd,
                                [&](int xr, int y, int z, unsigned long long r, bool valid, const smoke::Win& w,
                                    float2) {
    if (!valid) return;
    auto samp_u = [&](const float* p, float* o) { w.sample(g, ru, U, nullptr, p, o); };
    const unsigned long long plane = (unsigned long long)g.ny * g.nz;
#pragma unroll(kAdvUnroll)
    for (int c2 = 0; c2 < 2; ++c2) {
      const int x = 2 * xr + c2;
      const unsigned long long c = (unsigned long long)x * plane + (unsigned long long)y * g.nz + z;
      float val;
      if (x >= g.lo[0] && x < g.hi[0] && y >= g.lo[1] && y < g.hi[1] && z >= g.lo[2] && z < g.hi[2]) {
        val = 1.0f;  // S8: the source box
      } else {
        const float xp[3] = {(float)x, (float)y, (float)z};
        const float4 U0 = ru[w.at(x, y, z)];
        const float u0[3] = {U0.x, U0.y, U0.z};
        float xb[3];
        smoke::backtrace3(g, xp, u0, dt, samp_u, xb);
        int i, j, k;
        float tx, ty, tz;
        smoke::corner(xb[0], g.nx, i, tx);
        smoke::corner(xb[1], g.ny, j, ty);
        smoke::corner(xb[2], g.nz, k, tz);
        float f8[8];
        if (w.has(i, j, k)) {
          const int a = w.at(i, j, k), b = w.at(i + 1, j, k);
#pragma unroll
          for (int dj = 0; dj < 2; ++dj)
#pragma unroll
            for (int dk = 0; dk < 2; ++dk) {
              f8[dj * 2 + dk] = rd[a + dj * smoke::kWZ + dk];
              f8[4 + dj * 2 + dk] = rd[b + dj * smoke::kWZ + dk];
            }
        } else {
#pragma unroll
          for (int di = 0; di < 2; ++di)
#pragma unroll
            for (int dj = 0; dj < 2; ++dj)
#pragma unroll
              for (int dk = 0; dk < 2; ++dk)
                f8[di * 4 + dj * 2 + dk] = __ldg(rho + ((unsigned long long)(i + di) * g.ny + (j + dj)) * g.nz + (k + dk));
        }
        val = 0.0f;
#pragma unroll
        for (int di = 0; di < 2; ++di)
#pragma unroll
          for (int dj = 0; dj < 2; ++dj)
#pragma unroll
            for (int dk = 0; dk < 2; ++dk) {
              const float wt = (di ? tx : 1.0f - tx) * (dj ? ty : 1.0f - ty) * (dk ? tz : 1.0f - tz);
              val = fmaf(wt, f8[di * 4 + dj * 2 + dk], val);
            }
      }
      out[c] = val;
    }
  });
}
