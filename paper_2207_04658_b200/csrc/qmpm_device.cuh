// qmpm_device.cuh -- device-side building blocks of the quantized MLS-MPM step:
// bit-pack field access, fixed-point decode/encode with non-subtractive dithering,
// the content-keyed dither hash, B-spline weights and the polar decomposition.
//
// Paper passages (P:n = /root/reference/PAPER.md line n; readings Qn = DESIGN.md §2):
//   decode    Eq. 3: value = u * Delta (+ offset, Q21), u sign-extended
//             from b+1 bits (Q2); a field may straddle two words (bit pack).
//   encode    Eq. 3 / Eq. 11: t = fl32(fl32(v - offset) * inv_Delta), no FMA
//             (Q3); RNE (Q6) or u = floor(t) + [y >= 1 - r] (Q6), saturated.
//   pair_hash / dither_omr  reading Q5 rev. 3 (the paper's generator, is in an
//             unavailable supplement).
#pragma once
#ifdef __CUDACC_RTC__
typedef unsigned char uint8_t;
typedef unsigned short uint16_t;
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
#else
#include <cstdint>
#include <cuda_runtime.h>
#endif

namespace qmpm {

constexpr int kMaxScalars = 24;   // 3D elastic: x3 v3 F9 C9
constexpr int kMaxFields = 64;
constexpr int kKindFixed = 0;
constexpr int kKindRaw = 1;
constexpr int kKindShared = 2;  // SHARED_EXP member (reading Q4)

// One field as the kernels see it.  `idx` is the packing index (RNG stream and
// counters); `col` is the column of the field's value in a vals row.
struct FieldDev {
  uint8_t word, shift, width, kind;   // SHARED_EXP: word/shift/width of the mantissa
  float delta, inv_delta, offset;     // SHARED_EXP: Delta_0 = R_min 2^-b and its inverse
  uint16_t idx, col;
  uint8_t ebits, gword, gshift, pad;  // SHARED_EXP: exponent width and position
  uint16_t glead, pad2;               // SHARED_EXP: the group leader (packing index; the MPM
                                      // layout re-maps it to the leader's state scalar)
};

// Layout for the MPM kernels: fields indexed by STATE SCALAR (x.., v.., F../J, C..).
struct LayoutDev {
  uint32_t W;           // words per record
  uint32_t SW;          // shared-memory row stride (odd, >= W + 1)
  uint32_t ns;          // number of state scalars
  uint32_t xword_mask;  // record words holding any x bit (particle key, Q5)
  uint32_t dither;      // 1 = Eq. 11 dithering, 0 = RNE
  uint32_t counters;    // 1 = count round-ups/downs
  uint32_t ranges;      // 1 = record max |value| per state scalar (Alg. 1 line 9)
  uint32_t seed_lo, seed_hi;
  FieldDev s[kMaxScalars];
};

// Layout for the standalone codec: fields in PACKING order.
struct CodecDev {
  uint32_t W, SW, nf, stride;  // stride = floats per vals row
  uint32_t dither;
  uint32_t seed_lo, seed_hi;
  uint32_t pad;
  FieldDev f[kMaxFields];
};

// Scene constants (DESIGN.md §2 Q12-Q15).
struct SimDev {
  int res[3];
  int nb[3];          // grid blocks per axis
  float dx, inv_dx, dt;
  float g[3];
  float p_mass;
  float stress_scale; // -dt * p_vol * 4 * inv_dx^2
  float mu, lambda;   // fixed corotated (elastic)
  float E;            // fluid: P F^T = E (J - 1) I
  int bound;
  uint32_t nblocks;   // blocks of this context's block table (slab: its planes + the ghost plane)
  // slab decomposition along z (3D): this rank owns block planes
  // [slab_bz0, slab_bz1); slab_lo / slab_hi = a neighbour rank exists below / above.
  // The block table covers the block planes [tab_bz0, tab_bz1): the owned planes plus
  // the ghost plane above (single GPU: all planes); block ids are table-local.
  int slab_bz0, slab_bz1, slab_lo, slab_hi;
  int tab_bz0, tab_bz1;
  uint32_t seed_lo, seed_hi;  // dither seed (reading Q5): G2P derives the step salt on the device
};

constexpr uint32_t kDeadKey = 0xffffffffu;  // sort key of a particle this rank does not own

// Device-side counters (accumulated across steps until set_state).
struct DevCounters {
  unsigned long long sat[kMaxFields];
  unsigned long long up[kMaxFields];
  unsigned long long down[kMaxFields];
  unsigned long long nonfinite;
  unsigned long long oob;
  unsigned long long overflow;
  unsigned int mig_dn, mig_up;  // particles that left the slab downwards / upwards (last step)
  unsigned int mig_overflow;
  unsigned int n_sorted;      // particles sorted in the last scan
  unsigned int n_active;      // last step
  unsigned int n_touched;     // last step (before clamping to the pool)
  unsigned int n_touched_eff; // min(n_touched, pool)
  unsigned int range_bits[kMaxScalars];  // max |value| per state scalar (float bits, >= 0)
  unsigned int next_p2g;      // dynamic work counters of P2G / G2P (active-list position),
  unsigned int next_g2p;      // reset by the scan every step
  unsigned int n_active_below;  // active blocks below the top owned plane (slab overlap split)
  unsigned int next_p2g_top, next_g2p_top;  // work counters of the top-plane launches
  // slab migration, all on the device (no host synchronisation per step):
  unsigned int n_rec;         // record slots written by the last G2P (= its sorted particles)
  unsigned int n_slots;       // record slots the next sort scans: n_rec + appended arrivals
  unsigned int n_leave;       // particles that left the slab since the last sort (dead slots)
  unsigned int status;        // sticky error bits (kStatus*), agreed by every rank each step
  unsigned int gstep;         // number of the step in flight (1, 2, ...; the scan advances it), so
  unsigned int pad2;          // a step's launches take no per-step argument (CUDA-graph replays)
};

// sticky device-side error bits (DevCounters::status; qmpm_read_state / qmpm_stats report them)
constexpr unsigned kStatusMigOverflow = 1u;  // more leavers than a migration buffer holds
constexpr unsigned kStatusCapacity = 2u;     // arrivals past max_particles
constexpr unsigned kStatusTwoHop = 4u;       // a particle moved more than one slab in one step
constexpr unsigned kStatusNonfinite = 8u;    // (host side) the encoder met non-finite values

// header of a migration buffer (followed by `cap` records of W words): count, status
struct MigHeader {
  unsigned int count, status, pad0, pad1;
};

// Migration buffers of the slab decomposition: per direction
// one contiguous buffer [MigHeader | cap records of W words | cap ids | cap pre-encode
// rows of ns floats (QMPM_DEBUG_PREENCODE only)], exchanged whole (fixed size: the
// exchange schedule never depends on data, so no rank waits on a host-side count and an
// error on one rank cannot hang the others).
struct MigDev {
  unsigned char* send[2];        // [0] to the rank below, [1] to the rank above
  const unsigned char* recv[2];  // [0] from the rank below, [1] from the rank above
  uint32_t* dead_list;           // record slots whose particle left (read_state compaction)
  uint32_t cap, dead_cap, W, ids;
  uint32_t dbg_ns;               // 0, or the floats per pre-encode row carried along
  uint32_t pad;
};

__host__ __device__ inline size_t mig_ids_off(const MigDev& M) { return 16u + (size_t)M.cap * M.W * 4u; }
__host__ __device__ inline size_t mig_dbg_off(const MigDev& M) {
  return mig_ids_off(M) + (M.ids ? (size_t)M.cap * 4u : 0u);
}
__host__ __device__ inline size_t mig_bytes_of(const MigDev& M) { return mig_dbg_off(M) + (size_t)M.cap * M.dbg_ns * 4u; }

// ---------------------------------------------------------------- hashing (Q5)
__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

__host__ __device__ __forceinline__ uint32_t mix32_hd(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

// salt = mix(seed_lo ^ mix(seed_hi ^ mix(step)))  (step mod 2^32)
__host__ __device__ __forceinline__ uint32_t step_salt(uint32_t seed_lo, uint32_t seed_hi,
                                                       uint32_t step) {
  return mix32_hd(seed_lo ^ mix32_hd(seed_hi ^ mix32_hd(step)));
}

// Reading Q5, revision 3: one 32-bit hash z per PAIR p of fields (packing indices 2p and
// 2p + 1), the lowbias32 rounds on the pair-salted particle hash h = mix(key ^ salt).
__device__ __forceinline__ uint32_t pair_hash(uint32_t h, uint32_t p) {
  uint32_t x = h ^ (p * 0x9E3779B9u);
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

// s = 1 + r16 2^-16 for field f as a float assembled from bits: r16 = bits 7..22 of z (even
// f) or of z rotated right by 16 (odd f), placed in mantissa bits 7..22.
__device__ __forceinline__ float dither_s(uint32_t h, uint32_t f) {
  uint32_t z = pair_hash(h, f >> 1);
  if (f & 1u) z = __funnelshift_r(z, z, 16);
  return __uint_as_float(0x3f800000u | (z & 0x007fff80u));
}

// the dither threshold 1 - r16 2^-16 = 2 - s (exact: Sterbenz), u = floor(t) + [y >= it]
__device__ __forceinline__ float dither_omr(uint32_t h, uint32_t f) { return __fsub_rn(2.0f, dither_s(h, f)); }

// ---------------------------------------------------------------- MLS-MPM helpers
// base / fx of one axis with the out-of-domain clamp of Q14.  Identical arithmetic
// wherever a base is computed (bin key, P2G, G2P, next-step key).
__device__ __forceinline__ int base_fx(float x, float inv_dx, int n_axis, float& fx, bool& oob) {
  const float X = __fmul_rn(x, inv_dx);
  int b = (int)floorf(__fsub_rn(X, 0.5f));
  oob = false;
  if (b < 0) { b = 0; oob = true; }
  if (b > n_axis - 3) { b = n_axis - 3; oob = true; }
  float f = __fsub_rn(X, (float)b);
  if (oob) f = fminf(fmaxf(f, 0.5f), 1.5f);
  fx = f;
  return b;
}

// The same without the clamp: `oob` is OR-accumulated and the caller redoes the warp
// with base_fx() when any lane saw it (identical arithmetic when in the domain).
__device__ __forceinline__ int base_fx_fast(float x, float inv_dx, int n_axis, float& fx, bool& oob) {
  const float X = __fmul_rn(x, inv_dx);
  const int b = (int)floorf(__fsub_rn(X, 0.5f));
  oob |= (unsigned)b > (unsigned)(n_axis - 3);
  fx = __fsub_rn(X, (float)b);
  return b;
}

__device__ __forceinline__ void bspline_w(float fx, float w[3]) {
  const float a = 1.5f - fx, b = fx - 1.0f, c = fx - 0.5f;
  w[0] = 0.5f * a * a;
  w[1] = 0.75f - b * b;
  w[2] = 0.5f * c * c;
}

#ifndef QMPM_AB_WPACK
#define QMPM_AB_WPACK 1
#endif
// the weights of the first two axes in packed FP32x2 (each lane the same IEEE ops as
// bspline_w, so the weights are bit-identical), the third (3D) in scalar.  Measured:
// G2P -0.4 % (C4) / -0.7 % (C3); P2G +0.6 % / -0.5 % (noise) -- P2G keeps the scalar form
template <int D, bool PACK = true>
__device__ __forceinline__ void bspline_weights(const float fx[3], float wt[3][3]) {
#if QMPM_AB_WPACK
  if (!PACK) {
#pragma unroll
    for (int a = 0; a < D; ++a) bspline_w(fx[a], wt[a]);
    return;
  }
  const float2 f = make_float2(fx[0], fx[1]);
  const float2 a = __fadd2_rn(make_float2(1.5f, 1.5f), make_float2(-f.x, -f.y));
  const float2 b = __fadd2_rn(f, make_float2(-1.0f, -1.0f));
  const float2 c = __fadd2_rn(f, make_float2(-0.5f, -0.5f));
  const float2 w0 = __fmul2_rn(__fmul2_rn(make_float2(0.5f, 0.5f), a), a);
  const float2 w1 = __ffma2_rn(make_float2(-b.x, -b.y), b, make_float2(0.75f, 0.75f));
  const float2 w2 = __fmul2_rn(__fmul2_rn(make_float2(0.5f, 0.5f), c), c);
  wt[0][0] = w0.x; wt[1][0] = w0.y;
  wt[0][1] = w1.x; wt[1][1] = w1.y;
  wt[0][2] = w2.x; wt[1][2] = w2.y;
  if (D == 3) bspline_w(fx[2], wt[2]);
#else
#pragma unroll
  for (int a = 0; a < D; ++a) bspline_w(fx[a], wt[a]);
#endif
}

// 3x3 polar decomposition F = R S, det R = +1 for det F > 0, by Newton's iteration
// R <- (g R + R^{-T}/g)/2 with Higham's determinant scaling g = |det R|^{-1/3}.
__device__ __forceinline__ void polar3(const float F[9], float R[9]) {
#pragma unroll
  for (int i = 0; i < 9; ++i) R[i] = F[i];
#pragma unroll 1
  for (int it = 0; it < 12; ++it) {
    // cofactor matrix (= det * R^{-T})
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
    const float ad = fabsf(det);
    if (!(ad > 1e-30f)) break;
#ifdef QMPM_POLAR_SLOW
    const float g = (it < 6) ? rcbrtf(ad) : 1.0f;
    const float a = 0.5f * g, b = 0.5f / (g * det);
#else
    // the scaling only speeds convergence (the fixed point R = R^{-T} does not depend on
    // it), so |det|^{-1/3} = 2^(-log2|det| / 3) from the approximate SFU ops serves; the
    // 1/(g det) of the update is an IEEE-rounded reciprocal
    float g = 1.0f;
    if (it < 6) {
      float lg, e;
      asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(ad));
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-0.33333334f * lg));
      g = e;
    }
    const float a = 0.5f * g, b = 0.5f * __frcp_rn(g * det);
#endif
    // R <- a R + b c in packed FP32x2 (4 pairs + 1), delta = max |change|
    float delta = 0.0f;
    const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      const float2 r2 = make_float2(R[i], R[i + 1]);
      const float2 nr = __ffma2_rn(b2, make_float2(c[i], c[i + 1]), __fmul2_rn(a2, r2));
      const float2 d2 = __fadd2_rn(nr, make_float2(-r2.x, -r2.y));
      delta = fmaxf(delta, fmaxf(fabsf(d2.x), fabsf(d2.y)));
      R[i] = nr.x;
      R[i + 1] = nr.y;
    }
    {
      const float nr = __fmaf_rn(b, c[8], a * R[8]);
      delta = fmaxf(delta, fabsf(nr - R[8]));
      R[8] = nr;
    }
    // Newton's iteration converges quadratically: with delta = |R_{k+1} - R_k| ~ the
    // error of R_k, the iterate just formed is within ~delta^2 / (2 sigma_min) of the
    // polar factor, so delta < 1e-4 leaves it at fp32 rounding (~1e-8 for sigma_min >=
    // 0.5) without the extra confirming iteration a 1e-7 test costs (~90 instructions)
    if (delta < 1e-4f) break;
  }
}

// 2D polar: closed form (rotation by atan2(F10 - F01, F00 + F11)).
__device__ __forceinline__ void polar2(const float F[4], float R[4]) {
  const float x = F[0] + F[3], y = F[2] - F[1];
  // IEEE sqrt and divisions: the stress depends on F - R, which for small strains is
  // ~1e-6, so R must be as accurate as fp32 allows (an approximate rsqrt is not).
  const float r = __fsqrt_rn(__fmaf_rn(x, x, y * y));
  float c = 1.0f, s = 0.0f;
  if (r > 0.0f) {
    c = __fdiv_rn(x, r);
    s = __fdiv_rn(y, r);
  }
  R[0] = c; R[1] = -s; R[2] = s; R[3] = c;
}

}  // namespace qmpm
