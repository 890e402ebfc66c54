// smoke_kernels.cuh -- the quantized Eulerian smoke step (P:574-579,
// P:954-957), NVRTC-specialised on two generated layout structs: SpecU (6 fields: the
// velocity of the two cells of a record, packing order cell0 x y z, cell1 x y z) and
// SpecP (2 fields: the pressure of the two cells).  DESIGN.md §12 readings S1-S8.
//
// Grid: collocated nx x ny x nz cells (S1); record r = (xr * ny + y) * nz + z holds cells
// x = 2 xr and 2 xr + 1 (S2), so consecutive threads (consecutive z) touch consecutive
// records.  Every kernel runs one thread per record over a block-uniform grid-stride
// loop (encode_record's rare exact redo is a warp vote, so every lane reaches it).
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

__device__ __forceinline__ void rec_coords(const SmokeDev& g, unsigned long long r, int& xr, int& y, int& z) {
  z = (int)(r % g.nz);
  const unsigned long long q = r / g.nz;
  y = (int)(q % g.ny);
  xr = (int)(q / g.ny);
}

// neighbour pressure of cell (x, y, z) along the axes, Neumann walls (S6): outside -> self
__device__ __forceinline__ float p_at(const uint32_t* __restrict__ P, const SmokeDev& g, int x, int y, int z) {
  uint32_t w[SpecP::W + 1];
  ldrec<SpecP>(P, rec_of(g, x >> 1, y, z), w);
  return (x & 1) ? sdec<SpecP>(w, 1) : sdec<SpecP>(w, 0);
}

}  // namespace smoke

// ------------------------------------------------------------------ entry points
extern "C" __global__ void __launch_bounds__(256)
    qsmoke_advect_u(const uint32_t* __restrict__ uv, const uint32_t* __restrict__ ur, const float* __restrict__ rho,
                    SmokeDev g, float dt, float bdt, SaltSrc ss, uint32_t* __restrict__ out, float* __restrict__ dbg) {
  constexpr int W = SpecU::W;
  const uint32_t salt = smoke::salt_of(ss);
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long base = (unsigned long long)blockIdx.x * blockDim.x; base < g.n_rec; base += stride) {
    const unsigned long long r = base + threadIdx.x;
    const bool valid = r < g.n_rec;
    float v[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (valid) {
      int xr, y, z;
      smoke::rec_coords(g, r, xr, y, z);
      uint32_t w[W + 1];
      smoke::ldrec<SpecU>(uv, r, w);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float x[3] = {(float)(2 * xr + h), (float)y, (float)z};
        float u0[3], xb[3], q[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) u0[c] = qmpm::sdec<SpecU>(w, 3 * h + c);
        smoke::backtrace(uv, g, x, u0, dt, xb);
        smoke::sample_u(uv, g, xb, q);
        if (ur) {  // reflection: sample 2 u_vel - u_refl (S8; trilinear sampling is linear)
          float qr[3];
          smoke::sample_u(ur, g, xb, qr);
#pragma unroll
          for (int c = 0; c < 3; ++c) q[c] = 2.0f * q[c] - qr[c];
        }
        if (rho) q[1] += bdt * __ldg(rho + ((unsigned long long)(2 * xr + h) * g.ny + y) * g.nz + z);
#pragma unroll
        for (int c = 0; c < 3; ++c) v[3 * h + c] = q[c];
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
  }
}

extern "C" __global__ void __launch_bounds__(256)
    qsmoke_div(const uint32_t* __restrict__ U, SmokeDev g, float* __restrict__ div) {
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long r = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; r < g.n_rec; r += stride) {
    int xr, y, z;
    smoke::rec_coords(g, r, xr, y, z);
    float c0[3], c1[3], xm[3] = {0.f, 0.f, 0.f}, xp[3] = {0.f, 0.f, 0.f};
    smoke::u_pair(U, g, 2 * xr, y, z, c0, c1);
    if (xr > 0) smoke::u_cell(U, g, 2 * xr - 1, y, z, xm);
    if (xr + 1 < g.nxr) smoke::u_cell(U, g, 2 * xr + 2, y, z, xp);
    float ym0[3] = {0.f, 0.f, 0.f}, ym1[3] = {0.f, 0.f, 0.f}, yp0[3] = {0.f, 0.f, 0.f}, yp1[3] = {0.f, 0.f, 0.f};
    float zm0[3] = {0.f, 0.f, 0.f}, zm1[3] = {0.f, 0.f, 0.f}, zp0[3] = {0.f, 0.f, 0.f}, zp1[3] = {0.f, 0.f, 0.f};
    if (y > 0) smoke::u_pair(U, g, 2 * xr, y - 1, z, ym0, ym1);
    if (y + 1 < g.ny) smoke::u_pair(U, g, 2 * xr, y + 1, z, yp0, yp1);
    if (z > 0) smoke::u_pair(U, g, 2 * xr, y, z - 1, zm0, zm1);
    if (z + 1 < g.nz) smoke::u_pair(U, g, 2 * xr, y, z + 1, zp0, zp1);
    const float d0 = ((c1[0] - xm[0]) + (yp0[1] - ym0[1]) + (zp0[2] - zm0[2])) * g.half_inv_dx;
    const float d1 = ((xp[0] - c0[0]) + (yp1[1] - ym1[1]) + (zp1[2] - zm1[2])) * g.half_inv_dx;
    const unsigned long long c = ((unsigned long long)(2 * xr) * g.ny + y) * g.nz + z;
    div[c] = d0;
    div[c + (unsigned long long)g.ny * g.nz] = d1;
  }
}

extern "C" __global__ void __launch_bounds__(256)
    qsmoke_jacobi(const uint32_t* __restrict__ P, const float* __restrict__ div, SmokeDev g, SaltSrc ss,
                  uint32_t* __restrict__ out, float* __restrict__ dbg) {
  constexpr int W = SpecP::W;
  const uint32_t salt = smoke::salt_of(ss);
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  const unsigned long long plane = (unsigned long long)g.ny * g.nz;
  for (unsigned long long base = (unsigned long long)blockIdx.x * blockDim.x; base < g.n_rec; base += stride) {
    const unsigned long long r = base + threadIdx.x;
    const bool valid = r < g.n_rec;
    float v[2] = {0.f, 0.f};
    if (valid) {
      int xr, y, z;
      smoke::rec_coords(g, r, xr, y, z);
      uint32_t w[W + 1];
      smoke::ldrec<SpecP>(P, r, w);
      const float p0 = qmpm::sdec<SpecP>(w, 0), p1 = qmpm::sdec<SpecP>(w, 1);
      const float pxm = xr > 0 ? smoke::p_at(P, g, 2 * xr - 1, y, z) : p0;
      const float pxp = xr + 1 < g.nxr ? smoke::p_at(P, g, 2 * xr + 2, y, z) : p1;
      float ym0 = p0, ym1 = p1, yp0 = p0, yp1 = p1, zm0 = p0, zm1 = p1, zp0 = p0, zp1 = p1;
      if (y > 0) {
        smoke::ldrec<SpecP>(P, r - g.nz, w);
        ym0 = qmpm::sdec<SpecP>(w, 0);
        ym1 = qmpm::sdec<SpecP>(w, 1);
      }
      if (y + 1 < g.ny) {
        smoke::ldrec<SpecP>(P, r + g.nz, w);
        yp0 = qmpm::sdec<SpecP>(w, 0);
        yp1 = qmpm::sdec<SpecP>(w, 1);
      }
      if (z > 0) {
        smoke::ldrec<SpecP>(P, r - 1, w);
        zm0 = qmpm::sdec<SpecP>(w, 0);
        zm1 = qmpm::sdec<SpecP>(w, 1);
      }
      if (z + 1 < g.nz) {
        smoke::ldrec<SpecP>(P, r + 1, w);
        zp0 = qmpm::sdec<SpecP>(w, 0);
        zp1 = qmpm::sdec<SpecP>(w, 1);
      }
      const unsigned long long c = ((unsigned long long)(2 * xr) * g.ny + y) * g.nz + z;
      const float s0 = ((pxm + p1) + (ym0 + yp0)) + (zm0 + zp0);
      const float s1 = ((p0 + pxp) + (ym1 + yp1)) + (zm1 + zp1);
      v[0] = (s0 - g.dx2 * __ldg(div + c)) * (1.0f / 6.0f);
      v[1] = (s1 - g.dx2 * __ldg(div + c + plane)) * (1.0f / 6.0f);
      if (dbg) {
        dbg[2 * r] = v[0];
        dbg[2 * r + 1] = v[1];
      }
    }
    const uint32_t hh = SpecP::DITHER ? qmpm::mix32((uint32_t)r ^ salt) : 0u;
    uint32_t o[W + 1];
    qmpm::encode_record<SpecP>(v, hh, valid, o, nullptr);
    if (valid) qmpm::store_words<SpecP>(out + r * W, o);
  }
}

extern "C" __global__ void __launch_bounds__(256)
    qsmoke_project(const uint32_t* __restrict__ U, const uint32_t* __restrict__ P, SmokeDev g, SaltSrc ss,
                   uint32_t* __restrict__ out, float* __restrict__ dbg) {
  constexpr int W = SpecU::W;
  const uint32_t salt = smoke::salt_of(ss);
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long base = (unsigned long long)blockIdx.x * blockDim.x; base < g.n_rec; base += stride) {
    const unsigned long long r = base + threadIdx.x;
    const bool valid = r < g.n_rec;
    float v[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (valid) {
      int xr, y, z;
      smoke::rec_coords(g, r, xr, y, z);
      uint32_t w[SpecP::W + 1];
      smoke::ldrec<SpecP>(P, r, w);
      const float p0 = qmpm::sdec<SpecP>(w, 0), p1 = qmpm::sdec<SpecP>(w, 1);
      const float pxm = xr > 0 ? smoke::p_at(P, g, 2 * xr - 1, y, z) : p0;
      const float pxp = xr + 1 < g.nxr ? smoke::p_at(P, g, 2 * xr + 2, y, z) : p1;
      float ym0 = p0, ym1 = p1, yp0 = p0, yp1 = p1, zm0 = p0, zm1 = p1, zp0 = p0, zp1 = p1;
      if (y > 0) {
        smoke::ldrec<SpecP>(P, r - g.nz, w);
        ym0 = qmpm::sdec<SpecP>(w, 0);
        ym1 = qmpm::sdec<SpecP>(w, 1);
      }
      if (y + 1 < g.ny) {
        smoke::ldrec<SpecP>(P, r + g.nz, w);
        yp0 = qmpm::sdec<SpecP>(w, 0);
        yp1 = qmpm::sdec<SpecP>(w, 1);
      }
      if (z > 0) {
        smoke::ldrec<SpecP>(P, r - 1, w);
        zm0 = qmpm::sdec<SpecP>(w, 0);
        zm1 = qmpm::sdec<SpecP>(w, 1);
      }
      if (z + 1 < g.nz) {
        smoke::ldrec<SpecP>(P, r + 1, w);
        zp0 = qmpm::sdec<SpecP>(w, 0);
        zp1 = qmpm::sdec<SpecP>(w, 1);
      }
      const float gr[6] = {(p1 - pxm) * g.half_inv_dx, (yp0 - ym0) * g.half_inv_dx, (zp0 - zm0) * g.half_inv_dx,
                           (pxp - p0) * g.half_inv_dx, (yp1 - ym1) * g.half_inv_dx, (zp1 - zm1) * g.half_inv_dx};
      uint32_t wu[W + 1];
      smoke::ldrec<SpecU>(U, r, wu);
#pragma unroll
      for (int f = 0; f < 6; ++f) v[f] = qmpm::sdec<SpecU>(wu, f) - gr[f];
      // S7: wall-normal components zeroed in the boundary layer
      if (xr == 0) v[0] = 0.0f;
      if (xr + 1 == g.nxr) v[3] = 0.0f;
      if (y == 0 || y + 1 == g.ny) v[1] = v[4] = 0.0f;
      if (z == 0 || z + 1 == g.nz) v[2] = v[5] = 0.0f;
      if (dbg) {
#pragma unroll
        for (int f = 0; f < 6; ++f) dbg[r * 6 + f] = v[f];
      }
    }
    const uint32_t hh = SpecU::DITHER ? qmpm::mix32((uint32_t)r ^ salt) : 0u;
    uint32_t o[W + 1];
    qmpm::encode_record<SpecU>(v, hh, valid, o, nullptr);
    if (valid) qmpm::store_words<SpecU>(out + r * W, o);
  }
}

extern "C" __global__ void __launch_bounds__(256)
    qsmoke_advect_rho(const float* __restrict__ rho, const uint32_t* __restrict__ U, SmokeDev g, float dt,
                      float* __restrict__ out, unsigned long long* __restrict__ tick) {
  // the last kernel of a step advances the device step counter (nothing here reads it)
  if (tick && blockIdx.x == 0 && threadIdx.x == 0) *tick += 1ull;
  const unsigned long long n = 2ull * g.n_rec;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long c = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; c < n; c += stride) {
    const int z = (int)(c % g.nz);
    const int y = (int)((c / g.nz) % g.ny);
    const int x = (int)(c / ((unsigned long long)g.ny * g.nz));
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
}
