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

// value of state scalar i from a register-resident record w[0..W] (w[W] = 0)
template <class SP>
__device__ __forceinline__ float sdec(const uint32_t* w, const int i) {
  const int wd = SP::word(i), sh = SP::shift(i), wi = SP::width(i);
  const uint32_t raw = (sh + wi <= 32) ? (w[wd] >> sh) : __funnelshift_r(w[wd], w[wd + 1], sh);
  if (SP::kind(i) == kKindRaw) return __uint_as_float(raw);
  const int u = ((int)(raw << (32 - wi))) >> (32 - wi);  // sign-extend b+1 bits (Q2)
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
__device__ __forceinline__ uint32_t senc_core(const int wi, const float offset, const float inv, float v, uint32_t r24,
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
      const float one_minus_r = __fmul_rn(__uint2float_rn(0x1000000u - r24), 0x1p-24f);  // exact
      fl.up = y >= one_minus_r;         // u = floor(t + r) (Eq. 11, reading Q6)
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
      const float one_minus_r = __fmul_rn(__uint2float_rn(0x1000000u - r24), 0x1p-24f);
      fl.up = y >= one_minus_r;
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
__device__ __forceinline__ uint32_t senc(const int i, float v, uint32_t r24, EncFlags& fl) {
  if (SP::kind(i) == kKindRaw) {
    fl.up = fl.down = fl.sat = false;
    fl.nonfinite = !isfinite(v);
    return __float_as_uint(v);
  }
  return senc_core<SP::DITHER>(SP::width(i), SP::offset(i), SP::inv_delta(i), v, r24, fl);
}

template <class SP>
__device__ __forceinline__ void sput(uint32_t* w, const int i, uint32_t bits) {
  const int wd = SP::word(i), sh = SP::shift(i), wi = SP::width(i);
  w[wd] |= bits << sh;
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
        const uint32_t r24 = SP::DITHER ? r24_of(h, SP::idx(j)) : 0u;
        code[j] = senc_core<SP::DITHER>(SP::width(j), 0.0f, inv, v[j], r24, fl[j]);
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

// content key of a record (reading Q5): k = mix(k ^ word) over the words holding x
template <class SP>
__device__ __forceinline__ uint32_t content_key(const uint32_t* w) {
  uint32_t k = 0;
#pragma unroll
  for (int q = 0; q < SP::W; ++q)
    if ((SP::XMASK >> q) & 1u) k = mix32(k ^ w[q]);
  return k;
}

// Fast-path encode of state scalar i (Eq. 3 / Eq. 11, readings Q3, Q6): the code's
// bits WITHOUT the saturation clamp.  `flag` is raised (OR-accumulated) whenever the
// value might saturate or is not finite -- |t| >= 2^b - 1 or NaN -- and the caller then
// re-encodes the whole record with the exact senc() (rare).  up: u > t;  nz: the value
// is not on the grid (dither: down = nz - up) or, for RNE, dn: u < t.
template <class SP>
__device__ __forceinline__ uint32_t senc_fast(const int i, float v, uint32_t r24, bool& up, bool& nz, bool& flag) {
  if (SP::kind(i) == kKindRaw) {
    up = nz = false;
    flag |= !(fabsf(v) < __int_as_float(0x7f800000));
    return __float_as_uint(v);
  }
  const int wi = SP::width(i);
  const float a = (SP::offset(i) != 0.0f) ? __fsub_rn(v, SP::offset(i)) : v;
  const float t = __fmul_rn(a, SP::inv_delta(i));  // one fp32 multiply, no FMA (Q3)
  const uint32_t mask = (wi == 32) ? 0xffffffffu : ((1u << wi) - 1u);
  // |t| below lim => floor/round(t) (+1) lies inside [-2^b, 2^b - 1]
  constexpr float lim_tab[33] = {0.f, 0.f, 1.f, 3.f, 7.f, 15.f, 31.f, 63.f, 127.f, 255.f, 511.f, 1023.f, 2047.f,
                                 4095.f, 8191.f, 16383.f, 32767.f, 65535.f, 131071.f, 262143.f, 524287.f,
                                 1048575.f, 2097151.f, 4194303.f, 8388607.f, 16777215.f, 0x1p24f, 0x1p25f,
                                 0x1p26f, 0x1p27f, 0x1p28f, 0x1p29f, 0x1p30f};
  const float lim = lim_tab[wi];
  flag |= !(fabsf(t) < lim);
  int u;
  if (SP::DITHER) {
    const float f = floorf(t);
    const float y = __fsub_rn(t, f);  // exact
    // 1 - r24 2^-24 = (2^24 - r24) 2^-24 is representable, so the fma is exact
    const float one_minus_r = __fmaf_rn(-0x1p-24f, __uint2float_rn(r24), 1.0f);
    up = y >= one_minus_r;  // u = floor(t + r) (Eq. 11, reading Q6)
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

}  // namespace qmpm
