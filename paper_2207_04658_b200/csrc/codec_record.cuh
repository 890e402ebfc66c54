// codec_record.cuh -- record-level codec templates on a generated layout struct SP
// (NF fields in packing order, W words, WV vector width, DITHER, COUNTERS): vector
// load/store of records and fp32 rows, and encode_record (Eq. 3 / Eq. 11 of a whole
// record: fast path + rare exact redo, or the exact rule with counters).  Shared by the
// standalone codec (codec_kernels.cuh) and the smoke kernels (smoke_kernels.cuh).
#pragma once
#include "field_codec.cuh"

namespace qmpm {

constexpr unsigned kCFull = 0xffffffffu;

// Vector widths: Spec::WV (words) and Spec::VV (vals) are 4, 2 or 1, chosen on the host
// from the row sizes AND the base pointers' alignment.
template <class SP>
__device__ __forceinline__ void load_words(const uint32_t* __restrict__ p, uint32_t* w) {
  constexpr int W = SP::W;
  if (SP::WV == 4) {
#pragma unroll
    for (int q = 0; q < W / 4; ++q) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(p) + q);
      w[4 * q] = v.x;
      w[4 * q + 1] = v.y;
      w[4 * q + 2] = v.z;
      w[4 * q + 3] = v.w;
    }
  } else if (SP::WV == 2) {
#pragma unroll
    for (int q = 0; q < W / 2; ++q) {
      const uint2 v = __ldg(reinterpret_cast<const uint2*>(p) + q);
      w[2 * q] = v.x;
      w[2 * q + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int q = 0; q < W; ++q) w[q] = __ldg(p + q);
  }
  w[W] = 0u;
}

template <class SP>
__device__ __forceinline__ void store_words(uint32_t* __restrict__ p, const uint32_t* w) {
  constexpr int W = SP::W;
  if (SP::WV == 4) {
#pragma unroll
    for (int q = 0; q < W / 4; ++q)
      reinterpret_cast<uint4*>(p)[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
  } else if (SP::WV == 2) {
#pragma unroll
    for (int q = 0; q < W / 2; ++q) reinterpret_cast<uint2*>(p)[q] = make_uint2(w[2 * q], w[2 * q + 1]);
  } else {
#pragma unroll
    for (int q = 0; q < W; ++q) p[q] = w[q];
  }
}

template <int ST, int VV>
__device__ __forceinline__ void load_row(const float* __restrict__ p, float* r) {
  if (VV == 4) {
#pragma unroll
    for (int q = 0; q < ST / 4; ++q) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(p) + q);
      r[4 * q] = v.x;
      r[4 * q + 1] = v.y;
      r[4 * q + 2] = v.z;
      r[4 * q + 3] = v.w;
    }
  } else if (VV == 2) {
#pragma unroll
    for (int q = 0; q < ST / 2; ++q) {
      const float2 v = __ldg(reinterpret_cast<const float2*>(p) + q);
      r[2 * q] = v.x;
      r[2 * q + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int q = 0; q < ST; ++q) r[q] = __ldg(p + q);
  }
}

template <int ST, int VV>
__device__ __forceinline__ void store_row(float* __restrict__ p, const float* r) {
  if (VV == 4) {
#pragma unroll
    for (int q = 0; q < ST / 4; ++q)
      reinterpret_cast<float4*>(p)[q] = make_float4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
  } else if (VV == 2) {
#pragma unroll
    for (int q = 0; q < ST / 2; ++q) reinterpret_cast<float2*>(p)[q] = make_float2(r[2 * q], r[2 * q + 1]);
  } else {
#pragma unroll
    for (int q = 0; q < ST; ++q) p[q] = r[q];
  }
}

// Encode the NF values v[] (packing order) of one record into w[0..W].  Exact saturating
// rule with counters (lane-ballots into counters[3][64]: sat, up, down); without
// counters the fast path with a rare exact redo for the warp (identical bits).
template <class SP>
__device__ __forceinline__ void encode_record(const float* v, uint32_t h, bool valid, uint32_t* w,
                                              unsigned long long* __restrict__ counters) {
  constexpr int NF = SP::NF, W = SP::W;
#pragma unroll
  for (int q = 0; q <= W; ++q) w[q] = 0u;
  if (SP::COUNTERS) {
    const int lane = threadIdx.x & 31;
    EncFlags fl[NF];
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      if (SP::kind(f) == kKindShared) {  // reading Q4: the whole group at its leader
        if (SP::glead(f) == f) senc_group<SP>(f, v, h, w, fl);
        continue;
      }
      const float omr = (SP::DITHER && SP::kind(f) == kKindFixed) ? dither_omr(h, SP::idx(f)) : 1.0f;
      sput<SP>(w, f, senc<SP>(f, v[f], omr, fl[f]));
    }
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      const unsigned bs = __ballot_sync(kCFull, valid && fl[f].sat);
      const unsigned bu = __ballot_sync(kCFull, valid && fl[f].up);
      const unsigned bd = __ballot_sync(kCFull, valid && fl[f].down);
      if (lane == 0) {
        if (bs) atomicAdd(&counters[SP::idx(f)], (unsigned long long)__popc(bs));
        if (bu) atomicAdd(&counters[64 + SP::idx(f)], (unsigned long long)__popc(bu));
        if (bd) atomicAdd(&counters[128 + SP::idx(f)], (unsigned long long)__popc(bd));
      }
    }
    return;
  }
  bool flag = false;
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    if (SP::kind(f) == kKindShared) {
      if (SP::glead(f) == f) {
        EncFlags gfl[NF];
        senc_group<SP>(f, v, h, w, gfl);
#pragma unroll
        for (int j = 0; j < NF; ++j)
          if (SP::kind(j) == kKindShared && SP::glead(j) == f) flag |= gfl[j].sat || gfl[j].nonfinite;
      }
      continue;
    }
    const float omr = (SP::DITHER && SP::kind(f) == kKindFixed) ? dither_omr(h, SP::idx(f)) : 1.0f;
    bool up, nz;
    sput<SP>(w, f, senc_fast<SP>(f, v[f], omr, up, nz, flag));
  }
  if (__any_sync(kCFull, valid && flag)) {  // rare: the exact saturating rule
#pragma unroll
    for (int q = 0; q <= W; ++q) w[q] = 0u;
    EncFlags fl[NF];
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      if (SP::kind(f) == kKindShared) {
        if (SP::glead(f) == f) senc_group<SP>(f, v, h, w, fl);
        continue;
      }
      const float omr = (SP::DITHER && SP::kind(f) == kKindFixed) ? dither_omr(h, SP::idx(f)) : 1.0f;
      sput<SP>(w, f, senc<SP>(f, v[f], omr, fl[f]));
    }
  }
}

}  // namespace qmpm
