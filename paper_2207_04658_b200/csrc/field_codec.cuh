// field_codec.cuh -- compile-time bit-pack field access and the Eq. 3 / Eq. 11 codec,
// shared by the NVRTC-specialised step kernels (step_kernels.cuh) and the specialised
// standalone codec (codec_kernels.cuh).  `SP` is a generated layout struct: per scalar
// i its word, shift, width, kind, packing index idx (RNG stream and counters), Delta,
// 1/Delta and offset as constexpr functions, plus W and the DITHER flag.
//
//   sdec       Eq. 3 decode (sign-extended b+1 bits, reading Q2; offset Q21)
//   senc       exact encode: one fp32 multiply by 1/Delta, no FMA (Q3); round half to
//              even or u = floor(t) + [y >= 1 - r] (Eq. 11; Q6); saturating
//   senc_fast  the same without the clamp, flagging values that might saturate
//   sput       OR a field's bits into a register-resident record (may straddle a word)
//   senc_group a SHARED_EXP group (reading Q4): the smallest exponent E holding the
//              members' max |v|, members encoded with Delta_E = Delta_0 2^E (raised once
//              on a rounding overflow), E stored in front of the leader's mantissa
// SHARED_EXP entries also carry ebits (exponent width), gword/gshift (where the group's
// exponent sits) and glead (the Spec index of the group's leader); their word/shift is
// the mantissa's and delta/inv_delta are those of E = 0 (R_min 2^-b).
#pragma once
#include "qmpm_device.cuh"

namespace qmpm {

#ifndef QMPM_AB_SHFPACK
#define QMPM_AB_SHFPACK 1  // pack shifts as SHF (integer pipe): G2P -0.4 % (C4), -0.3 % (C3)
#endif
#ifndef QMPM_AB_SZEXT
#define QMPM_AB_SZEXT 1  // sign-extend decoded codes with szext (SASS SGXT, integer pipe)
#endif
// the low `width` bits of raw as a signed integer (two's complement, reading Q2).  The
// shift pair (raw << (32 - width)) >> (32 - width) puts its left shift on the FMA pipe
// (IMAD.SHL), the pipe that binds the step kernels; szext is one integer-pipe op.
__device__ __forceinline__ int sext_bits(uint32_t raw, int width) {
#if QMPM_AB_SZEXT
  if (width < 32) {
    int u;
    asm("szext.wrap.s32 %0, %1, %2;" : "=r"(u) : "r"(raw), "r"(width));
    return u;
  }
#endif
  return ((int)(raw << (32 - width))) >> (32 - width);
}

// value of state scalar i from a register-resident record w[0..W] (w[W] = 0)
template <class SP>
__device__ __forceinline__ float sdec(const uint32_t* w, const int i) {
  const int wd = SP::word(i), sh = SP::shift(i), wi = SP::width(i);
  const uint32_t raw = (sh + wi <= 32) ? (w[wd] >> sh) : __funnelshift_r(w[wd], w[wd + 1], sh);
  if (SP::kind(i) == kKindRaw) return __uint_as_float(raw);
  const int u = sext_bits(raw, wi);  // sign-extend b+1 bits (Q2)
  if (SP::kind(i) == kKindShared) {  // reading Q4: u * Delta_0 2^E, E = the group exponent
    const int gw = SP::gword(i), gs = SP::gshift(i), eb = SP::ebits(i);
    const uint32_t er = (gs + eb <= 32) ? (w[gw] >> gs) : __funnelshift_r(w[gw], w[gw + 1], gs);
    const uint32_t E = er & ((1u << eb) - 1u);
    return __fmul_rn(__int2float_rn(u), __int_as_float(__float_as_int(SP::delta(i)) + (int)(E << 23)));
  }
  float x = __fmul_rn(__int2float_rn(u), SP::delta(i));   // Eq. 3: u * Delta
  if (SP::offset(i) != 0.0f) x = __fadd_rn(x, SP::offset(i));
  return x;
}

struct EncFlags {
  bool up, down, sat, nonfinite;
};

// Eq. 3 / Eq. 11 encode of a fixed-point value of width wi with 1/Delta = inv and the
// given offset; returns the field's bits (width-masked).
template <bool DITHER>
__device__ __forceinline__ uint32_t senc_core(const int wi, const float offset, const float inv, float v, float omr,
                                              EncFlags& fl) {
  fl.up = fl.down = fl.sat = fl.nonfinite = false;
  if (!isfinite(v)) {
    fl.nonfinite = true;
    return 0u;
  }
  const float a = (offset != 0.0f) ? __fsub_rn(v, offset) : v;
  const float t = __fmul_rn(a, inv);  // one fp32 multiply, no FMA (Q3)
  const uint32_t mask = (wi == 32) ? 0xffffffffu : ((1u << wi) - 1u);
  if (wi <= 25) {
    // |codes| <= 2^24: clamping f to [-2^b - 2, 2^b] (exact floats) keeps every
    // saturation decision of the exact integer rule
    const float lo_f = -(float)(1 << (wi - 1)) - 2.0f, hi_f = (float)(1 << (wi - 1));
    const int lo = -(1 << (wi - 1)), hi = (1 << (wi - 1)) - 1;
    int u;
    if (DITHER) {
      const float f = floorf(t);
      const float y = __fsub_rn(t, f);  // exact
      fl.up = y >= omr;                 // u = floor(t + r), omr = 1 - r (Eq. 11, reading Q6)
      fl.down = !fl.up && y > 0.0f;
      u = __float2int_rz(fminf(fmaxf(f, lo_f), hi_f)) + (fl.up ? 1 : 0);
    } else {
      const float q = rintf(t);  // round half to even (Q6)
      fl.up = q > t;
      fl.down = q < t;
      u = __float2int_rz(fminf(fmaxf(q, lo_f), hi_f));
    }
    if (u > hi) { u = hi; fl.sat = true; }
    if (u < lo) { u = lo; fl.sat = true; }
    return (uint32_t)u & mask;
  } else {
    long long u;
    if (DITHER) {
      const float f = floorf(t);
      const float y = __fsub_rn(t, f);
      fl.up = y >= omr;
      fl.down = !fl.up && y > 0.0f;
      u = __float2ll_rz(fminf(fmaxf(f, -1099511627776.0f), 1099511627776.0f)) + (fl.up ? 1 : 0);
    } else {
      const float q = rintf(t);
      fl.up = q > t;
      fl.down = q < t;
      u = __float2ll_rz(fminf(fmaxf(q, -1099511627776.0f), 1099511627776.0f));
    }
    const long long hi = (1ll << (wi - 1)) - 1, lo = -(1ll << (wi - 1));
    if (u > hi) { u = hi; fl.sat = true; }
    if (u < lo) { u = lo; fl.sat = true; }
    return (uint32_t)u & mask;
  }
}

// Eq. 3 / Eq. 11 encode of FIXED or RAW entry i (SHARED_EXP entries: senc_group)
template <class SP>
__device__ __forceinline__ uint32_t senc(const int i, float v, float omr, EncFlags& fl) {
  if (SP::kind(i) == kKindRaw) {
    fl.up = fl.down = fl.sat = false;
    fl.nonfinite = !isfinite(v);
    return __float_as_uint(v);
  }
  return senc_core<SP::DITHER>(SP::width(i), SP::offset(i), SP::inv_delta(i), v, omr, fl);
}

template <class SP>
__device__ __forceinline__ void sput(uint32_t* w, const int i, uint32_t bits) {
  const int wd = SP::word(i), sh = SP::shift(i), wi = SP::width(i);
  // fields never overlap and `bits` holds no bit above the field's width, so the OR is
  // an ADD -- (bits << sh) + w is one LEA on the integer pipe instead of a shift the
  // compiler puts on the FMA pipe (IMAD.SHL) plus an OR
#if QMPM_AB_SZEXT && QMPM_AB_SHFPACK
  if (sh > 0 && sh + wi <= 32) {  // (a funnel shift with a zero low word: SHF, integer pipe)
    uint32_t r;
    asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(0u), "r"(bits), "r"(sh));
    w[wd] += r;
  } else {
    w[wd] += bits << sh;
  }
#elif QMPM_AB_SZEXT
  w[wd] += bits << sh;
#else
  w[wd] |= bits << sh;
#endif
  if (sh + wi > 32) w[wd + 1] |= bits >> (32 - sh);
}

// SHARED_EXP group led by Spec entry `lead` (reading Q4), values v[] indexed like the
// Spec: M = max |v| over the finite members; E = the smallest exponent in [0, 2^e - 1]
// with M < R_min 2^E (R_min = Delta_0 2^b, a power of two, so M / R_min is exact and
// E = floor(log2(M / R_min)) + 1 from the exponent bits); the members take the FIXED
// rule with 1/Delta_E = inv_delta 2^-E (exact); a saturating member raises E once
// (then |t| < 2^(b-1)).  Writes E and the member codes into w; fl[j] for each member j.
template <class SP>
__device__ __forceinline__ void senc_group(const int lead, const float* v, uint32_t h, uint32_t* w, EncFlags* fl) {
  constexpr int N = SP::NSPEC;
  const int eb = SP::ebits(lead);
  const uint32_t emax = (1u << eb) - 1u;
  float M = 0.0f;
#pragma unroll
  for (int j = 0; j < N; ++j)
    if (SP::kind(j) == kKindShared && SP::glead(j) == lead && isfinite(v[j])) M = fmaxf(M, fabsf(v[j]));
  // 1 / R_min = inv_delta(lead) 2^-b: exact powers of two
  const float inv_r = __int_as_float(__float_as_int(SP::inv_delta(lead)) - ((SP::width(lead) - 1) << 23));
  uint32_t E = 0u;
  const float y = __fmul_rn(M, inv_r);
  if (y >= 1.0f) E = min(emax, (uint32_t)(((__float_as_uint(y) >> 23) & 0xffu) - 127u + 1u));
  uint32_t code[N];
#pragma unroll 1
  for (int attempt = 0; attempt < 2; ++attempt) {
    bool sat = false;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      if (SP::kind(j) == kKindShared && SP::glead(j) == lead) {
        const float inv = __int_as_float(__float_as_int(SP::inv_delta(j)) - (int)(E << 23));
        const float omr = SP::DITHER ? dither_omr(h, SP::idx(j)) : 1.0f;
        code[j] = senc_core<SP::DITHER>(SP::width(j), 0.0f, inv, v[j], omr, fl[j]);
        sat |= fl[j].sat;
      }
    }
    if (!sat || E == emax) break;
    ++E;
  }
  {
    const int gw = SP::gword(lead), gs = SP::gshift(lead);
    w[gw] |= E << gs;
    if (gs + eb > 32) w[gw + 1] |= E >> (32 - gs);
  }
#pragma unroll
  for (int j = 0; j < N; ++j)
    if (SP::kind(j) == kKindShared && SP::glead(j) == lead) sput<SP>(w, j, code[j]);
}

// |t| below enc_lim(width) => floor/round(t) (+1) lies inside [-2^b, 2^b - 1]
__host__ __device__ constexpr float enc_lim(int wi) {
  return wi <= 1 ? 0.0f : (wi <= 25 ? (float)((1 << (wi - 1)) - 1) : (float)(1 << 24) * (float)(1 << (wi - 26)));
}

// content key of a record (reading Q5 rev. 3): k = (k ^ word) * 0x9E3779B1 over the words
// holding x (an odd multiply per word: a bijection of each word; the full mixing is the
// particle hash h = mix(key ^ salt) that follows)
template <class SP>
__device__ __forceinline__ uint32_t content_key(const uint32_t* w) {
  uint32_t k = 0;
#pragma unroll
  for (int q = 0; q < SP::W; ++q)
    if ((SP::XMASK >> q) & 1u) k = (k ^ w[q]) * 0x9E3779B1u;
  return k;
}

// Fast-path encode of state scalar i (Eq. 3 / Eq. 11, readings Q3, Q6): the code's
// bits WITHOUT the saturation clamp.  `flag` is raised (OR-accumulated) whenever the
// value might saturate or is not finite -- |t| >= 2^b - 1 or NaN -- and the caller then
// re-encodes the whole record with the exact senc() (rare).  up: u > t;  nz: the value
// is not on the grid (dither: down = nz - up) or, for RNE, dn: u < t.
template <class SP>
__device__ __forceinline__ uint32_t senc_fast(const int i, float v, float omr, bool& up, bool& nz, bool& flag) {
  if (SP::kind(i) == kKindRaw) {
    up = nz = false;
    flag |= !(fabsf(v) < __int_as_float(0x7f800000));
    return __float_as_uint(v);
  }
  const int wi = SP::width(i);
  const float a = (SP::offset(i) != 0.0f) ? __fsub_rn(v, SP::offset(i)) : v;
  const float t = __fmul_rn(a, SP::inv_delta(i));  // one fp32 multiply, no FMA (Q3)
  const uint32_t mask = (wi == 32) ? 0xffffffffu : ((1u << wi) - 1u);
  const float lim = enc_lim(wi);
  flag |= !(fabsf(t) < lim);
  int u;
  if (SP::DITHER) {
    const float f = floorf(t);
    const float y = __fsub_rn(t, f);  // exact
    up = y >= omr;  // u = floor(t + r) (Eq. 11, reading Q6)
    nz = y > 0.0f;
    u = __float2int_rz(f);
    if (up) ++u;
  } else {
    const float q = rintf(t);  // round half to even (Q6)
    up = q > t;
    nz = q < t;
    u = __float2int_rz(q);
  }
  return (uint32_t)u & mask;
}

// ---------------------------------------------------------------- dithered fast path
// Eq. 11 with readings Q3, Q5 rev. 3 and Q6 in packed FP32x2 (sm_100 FMUL2 /
// FADD2 / FFMA2: each lane is the IEEE-rounded scalar op), for FIXED entries of width
// <= 23 (|t| < 2^22 whenever the value cannot saturate):
//   t = fl(fl(v - offset) * 1/Delta)                (one multiply, no FMA: Q3)
//   s = fl_down(t + M) = M + floor(t), M = 1.5 2^23  (exact for |t| < 2^22; no F2I/FRND)
//   y = t - (s - M)                                  (exact)
//   d = y + (s_r - 2), s_r = 1 + r16 2^-16           (s_r - 2 = -(1 - r) exactly)
//   u = floor(t) + [y >= 1 - r] = bits(s) - bits(M) + 1 + (bits(d) >> 31)
// sign(d) is exact under round-to-nearest (d = +0 iff y = 1 - r: rounds up, Q6).
// `flag` as senc_fast (|t| >= 2^b - 1 or NaN: the caller re-encodes exactly); zi / zj are
// y == 0 (an on-grid value: counted as neither up nor down).
constexpr float kFloorMagic = 12582912.0f;  // 1.5 2^23
constexpr int kFloorMagicBits = 0x4b400000;

// -1 when the sign bit of d is set, else 0.  Kept as an opaque shr.s32: ptxas 12.9 fuses
// `(bits(d) >> 31) + bits(s)` with the later mask-and-shift of the bit pack into a LEA.HI
// sequence that drops the mask on the first lane of a pair (wrong words; reproduced by
// tools/pair_probe.py, measured on B200)
__device__ __forceinline__ int sign_mask(float d) {
  int r;
  asm("shr.s32 %0, %1, 31;" : "=r"(r) : "r"(__float_as_int(d)));
  return r;
}

template <class SP>
__host__ __device__ constexpr bool fast_ok(int i) {
  return SP::DITHER && SP::kind(i) == kKindFixed && SP::width(i) <= 23;
}

// 1: entry i opens a packed pair (i, i + 1) (i even); 2: i closes one; 0: i is encoded alone
template <class SP>
__host__ __device__ constexpr int pair_role(int i) {
  return (i % 2 == 0 && i + 1 < SP::NSPEC && fast_ok<SP>(i) && fast_ok<SP>(i + 1)) ? 1
         : (i % 2 == 1 && fast_ok<SP>(i - 1) && fast_ok<SP>(i)) ? 2
                                                                 : 0;
}

template <class SP>
__device__ __forceinline__ void senc_pair_fast(const int i, const int j, const float vi, const float vj,
                                               const float si, const float sj, int& ui, int& uj, int& sbi, int& sbj,
                                               bool& flag, bool& zi, bool& zj) {
  float2 a = make_float2(vi, vj);
  if (SP::offset(i) != 0.0f || SP::offset(j) != 0.0f)  // v - offset; adding -0 is the identity
    a = __fadd2_rn(a, make_float2(-SP::offset(i), -SP::offset(j)));
  const float2 t = __fmul2_rn(a, make_float2(SP::inv_delta(i), SP::inv_delta(j)));
  const float2 s = __fadd2_rd(t, make_float2(kFloorMagic, kFloorMagic));
  const float2 f = __fadd2_rn(s, make_float2(-kFloorMagic, -kFloorMagic));
  const float2 y = __ffma2_rn(f, make_float2(-1.0f, -1.0f), t);
  const float2 d = __fadd2_rn(y, __fadd2_rn(make_float2(si, sj), make_float2(-2.0f, -2.0f)));
  sbi = sign_mask(d.x);
  sbj = sign_mask(d.y);
  ui = __float_as_int(s.x) - (kFloorMagicBits - 1) + sbi;
  uj = __float_as_int(s.y) - (kFloorMagicBits - 1) + sbj;
  flag |= !(fabsf(t.x) < enc_lim(SP::width(i))) || !(fabsf(t.y) < enc_lim(SP::width(j)));
  zi = y.x == 0.0f;
  zj = y.y == 0.0f;
}

template <class SP>
__device__ __forceinline__ int senc1_fast(const int i, const float v, const float si, int& sb, bool& flag,
                                          bool& z) {
  const float a = (SP::offset(i) != 0.0f) ? __fsub_rn(v, SP::offset(i)) : v;
  const float t = __fmul_rn(a, SP::inv_delta(i));
  const float s = __fadd_rd(t, kFloorMagic);
  const float y = __fsub_rn(t, __fsub_rn(s, kFloorMagic));
  const float d = __fadd_rn(y, __fsub_rn(si, 2.0f));
  sb = sign_mask(d);
  flag |= !(fabsf(t) < enc_lim(SP::width(i)));
  z = y == 0.0f;
  return __float_as_int(s) - (kFloorMagicBits - 1) + sb;
}

// the integer code of FIXED entry i (sign-extended b+1 bits, reading Q2)
template <class SP>
__device__ __forceinline__ int scode(const uint32_t* w, const int i) {
  const int wd = SP::word(i), sh = SP::shift(i), wi = SP::width(i);
  const uint32_t raw = (sh + wi <= 32) ? (w[wd] >> sh) : __funnelshift_r(w[wd], w[wd + 1], sh);
  return sext_bits(raw, wi);
}

template <class SP>
__device__ __forceinline__ void sput_code(uint32_t* w, const int i, const int u) {
  const int wi = SP::width(i);
  sput<SP>(w, i, (uint32_t)u & ((wi == 32) ? 0xffffffffu : ((1u << wi) - 1u)));
}

}  // namespace qmpm
