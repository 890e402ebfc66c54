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
// Encodes are dithered with h = mix(record ^ salt) (reading Q5); salt comes from the host.
#pragma once
#include "codec_record.cuh"

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

// trilinear sample of the velocity field at p (cell units)
__device__ __forceinline__ void sample_u(const uint32_t* __restrict__ U, const SmokeDev& g, const float* p, float* out) {
  int i, j, k;
  float tx, ty, tz;
  corner(p[0], g.nx, i, tx);
  corner(p[1], g.ny, j, ty);
  corner(p[2], g.nz, k, tz);
#pragma unroll
  for (int c = 0; c < 3; ++c) out[c] = 0.0f;
#pragma unroll
  for (int dj = 0; dj < 2; ++dj) {
#pragma unroll
    for (int dk = 0; dk < 2; ++dk) {
      float a[3], b[3];
      u_pair(U, g, i, j + dj, k + dk, a, b);
      const float wyz = (dj ? ty : 1.0f - ty) * (dk ? tz : 1.0f - tz);
      const float wa = (1.0f - tx) * wyz, wb = tx * wyz;
#pragma unroll
      for (int c = 0; c < 3; ++c) out[c] = fmaf(wa, a[c], fmaf(wb, b[c], out[c]));
    }
  }
}

__device__ __forceinline__ float sample_s(const float* __restrict__ f, const SmokeDev& g, const float* p) {
  int i, j, k;
  float tx, ty, tz;
  corner(p[0], g.nx, i, tx);
  corner(p[1], g.ny, j, ty);
  corner(p[2], g.nz, k, tz);
  float out = 0.0f;
#pragma unroll
  for (int di = 0; di < 2; ++di)
#pragma unroll
    for (int dj = 0; dj < 2; ++dj)
#pragma unroll
      for (int dk = 0; dk < 2; ++dk) {
        const float w = (di ? tx : 1.0f - tx) * (dj ? ty : 1.0f - ty) * (dk ? tz : 1.0f - tz);
        out = fmaf(w, __ldg(f + ((unsigned long long)(i + di) * g.ny + (j + dj)) * g.nz + (k + dk)), out);
      }
  return out;
}

// S4: RK-3 (Ralston) departure point of cell centre x, velocity in world units / dx
__device__ __forceinline__ void backtrace(const uint32_t* __restrict__ U, const SmokeDev& g, const float* x,
                                          const float* u0, float dt, float* xb) {
  const float s = dt * g.inv_dx;
  float k2[3], k3[3], p[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) p[c] = x[c] - 0.5f * s * u0[c];
  sample_u(U, g, p, k2);
#pragma unroll
  for (int c = 0; c < 3; ++c) p[c] = x[c] - 0.75f * s * k2[c];
  sample_u(U, g, p, k3);
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
}  // namespace smoke

// ------------------------------------------------------------------ entry points
extern "C" __global__ void __launch_bounds__(256)
    qsmoke_advect_u(const uint32_t* __restrict__ uv, const uint32_t* __restrict__ ur, const float* __restrict__ rho,
                    SmokeDev g, float dt, float bdt, SaltSrc ss, uint32_t* __restrict__ out, float* __restrict__ dbg) {
  constexpr int W = SpecU::W;
  const smoke::Here h = smoke::here(g);
  float v[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (h.valid) {
    uint32_t w[W + 1];
    smoke::ldrec<SpecU>(uv, h.r, w);
#pragma unroll
    for (int c2 = 0; c2 < 2; ++c2) {
      const float x[3] = {(float)(2 * h.xr + c2), (float)h.y, (float)h.z};
      float u0[3], xb[3], q[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) u0[c] = qmpm::sdec<SpecU>(w, 3 * c2 + c);
      smoke::backtrace(uv, g, x, u0, dt, xb);
      smoke::sample_u(uv, g, xb, q);
      if (ur) {  // reflection: sample 2 u_vel - u_refl (S8; trilinear sampling is linear)
        float qr[3];
        smoke::sample_u(ur, g, xb, qr);
#pragma unroll
        for (int c = 0; c < 3; ++c) q[c] = 2.0f * q[c] - qr[c];
      }
      if (rho) q[1] += bdt * __ldg(rho + ((unsigned long long)(2 * h.xr + c2) * g.ny + h.y) * g.nz + h.z);
#pragma unroll
      for (int c = 0; c < 3; ++c) v[3 * c2 + c] = q[c];
    }
    if (dbg) {
#pragma unroll
      for (int f = 0; f < 6; ++f) dbg[h.r * 6 + f] = v[f];
    }
  }
  const uint32_t hh = SpecU::DITHER ? qmpm::mix32((uint32_t)h.r ^ smoke::salt_of(ss)) : 0u;
  uint32_t o[W + 1];
  qmpm::encode_record<SpecU>(v, hh, h.valid, o, nullptr);
  if (h.valid) qmpm::store_words<SpecU>(out + h.r * W, o);
}

// S5 on the x march: neighbours outside the domain are 0 (halo / x loads masked)
extern "C" __global__ void __launch_bounds__(256)
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

extern "C" __global__ void __launch_bounds__(256)
    qsmoke_jacobi(const uint32_t* __restrict__ P, const float* __restrict__ div, SmokeDev g, SaltSrc ss,
                  uint32_t* __restrict__ out, float* __restrict__ dbg) {
  constexpr int W = SpecP::W;
  const uint32_t salt = smoke::salt_of(ss);
  smoke::p_march(P, div, nullptr, g, [&](const smoke::March& m, int xr, unsigned long long r, bool valid,
                                          const float* pc, const float (*nb)[6], const float* d, const uint32_t* wu) {
    float v[2] = {0.f, 0.f};
    if (valid) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const float s = ((nb[k][0] + nb[k][1]) + (nb[k][2] + nb[k][3])) + (nb[k][4] + nb[k][5]);
        v[k] = (s - g.dx2 * d[k]) * (1.0f / 6.0f);
      }
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

extern "C" __global__ void __launch_bounds__(256)
    qsmoke_project(const uint32_t* __restrict__ U, const uint32_t* __restrict__ P, SmokeDev g, SaltSrc ss,
                   uint32_t* __restrict__ out, float* __restrict__ dbg) {
  constexpr int W = SpecU::W;
  const uint32_t salt = smoke::salt_of(ss);
  smoke::p_march(P, nullptr, U, g, [&](const smoke::March& m, int xr, unsigned long long r, bool valid,
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

// one thread per CELL: blockIdx.z = the cell plane x
extern "C" __global__ void __launch_bounds__(256)
    qsmoke_advect_rho(const float* __restrict__ rho, const uint32_t* __restrict__ U, SmokeDev g, float dt,
                      float* __restrict__ out, unsigned long long* __restrict__ tick) {
  // the last kernel of a step advances the device step counter (nothing here reads it)
  if (tick && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0 && threadIdx.y == 0)
    *tick += 1ull;
  const int z = blockIdx.x * smoke::kTZ + threadIdx.x, y = blockIdx.y * smoke::kTY + threadIdx.y, x = blockIdx.z;
  if (z >= g.nz || y >= g.ny) return;
  const unsigned long long c = ((unsigned long long)x * g.ny + y) * g.nz + z;
  float val;
  if (x >= g.lo[0] && x < g.hi[0] && y >= g.lo[1] && y < g.hi[1] && z >= g.lo[2] && z < g.hi[2]) {
    val = 1.0f;  // S8: the source box
  } else {
    const float p[3] = {(float)x, (float)y, (float)z};
    float u0[3], xb[3];
    smoke::u_cell(U, g, x, y, z, u0);
    smoke::backtrace(U, g, p, u0, dt, xb);
    val = smoke::sample_s(rho, g, xb);
  }
  out[c] = val;
}
