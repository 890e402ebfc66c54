// codec_kernels.cuh -- the standalone codec (Eq. 3 / Eq. 11 + bit pack), specialised by
// NVRTC on a scheme's layout like the step kernels.  The generated preamble defines
// `struct Spec`: NF fields in PACKING order (word, shift, width, kind, idx = f, Delta,
// 1/Delta, offset), W words per record, STRIDE floats per vals row and col(f) = the
// column of field f in a row, DITHER (scheme dithers AND the caller passed keys) and
// COUNTERS (the caller passed counters).
//
//   qmpm_codec_encode   vals [n][STRIDE] fp32 -> records [n][W]
//   qmpm_codec_decode   records -> vals
//   qmpm_codec_matmul3  records of a 3x3 matrix (9 fields, row-major) -> decode,
//                       multiply by a constant 3x3 A, re-encode: the paper's "MatMul"
//                       task, fused so each matrix is read and written once
// One record per thread, grid-stride; records and rows move with vector loads/stores
// (a warp touches contiguous memory), so the kernels are HBM-bound.
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
      const uint32_t r24 = (SP::DITHER && SP::kind(f) == kKindFixed) ? r24_of(h, SP::idx(f)) : 0u;
      sput<SP>(w, f, senc<SP>(f, v[f], r24, fl[f]));
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
    const uint32_t r24 = (SP::DITHER && SP::kind(f) == kKindFixed) ? r24_of(h, SP::idx(f)) : 0u;
    bool up, nz;
    sput<SP>(w, f, senc_fast<SP>(f, v[f], r24, up, nz, flag));
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
      const uint32_t r24 = (SP::DITHER && SP::kind(f) == kKindFixed) ? r24_of(h, SP::idx(f)) : 0u;
      sput<SP>(w, f, senc<SP>(f, v[f], r24, fl[f]));
    }
  }
}

}  // namespace qmpm

// ------------------------------------------------------------------ entry points
// Each thread handles kU records per grid-stride iteration (record u*256 + tid of the
// CTA's chunk), issuing all kU loads before any compute so enough bytes are in flight
// to cover the HBM latency.
constexpr int kU = 4;

extern "C" __global__ void __launch_bounds__(256) qmpm_codec_encode(const float* __restrict__ vals,
                                                                    const uint32_t* __restrict__ keys, uint64_t n,
                                                                    uint32_t salt, uint32_t* __restrict__ words,
                                                                    unsigned long long* __restrict__ counters) {
  constexpr int NF = Spec::NF, W = Spec::W, ST = Spec::STRIDE;
  const uint64_t chunk = 256ull * kU;
  for (uint64_t c0 = (uint64_t)blockIdx.x * chunk; c0 < n; c0 += (uint64_t)gridDim.x * chunk) {
    float row[kU][ST];
    uint32_t key[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t i = c0 + u * 256 + threadIdx.x;
#pragma unroll
      for (int q = 0; q < ST; ++q) row[u][q] = 0.0f;
      key[u] = 0u;
      if (i < n) {
        qmpm::load_row<ST, Spec::VV>(vals + i * ST, row[u]);
        if (Spec::DITHER) key[u] = __ldg(keys + i);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t i = c0 + u * 256 + threadIdx.x;
      const bool valid = i < n;
      float v[NF];
#pragma unroll
      for (int f = 0; f < NF; ++f) v[f] = valid ? row[u][Spec::col(f)] : Spec::offset(f);
      const uint32_t h = Spec::DITHER ? qmpm::mix32(key[u] ^ salt) : 0u;
      uint32_t w[W + 1];
      qmpm::encode_record<Spec>(v, h, valid, w, counters);
      if (valid) qmpm::store_words<Spec>(words + i * W, w);
    }
  }
}

extern "C" __global__ void __launch_bounds__(256) qmpm_codec_decode(const uint32_t* __restrict__ words, uint64_t n,
                                                                    float* __restrict__ vals) {
  constexpr int NF = Spec::NF, W = Spec::W, ST = Spec::STRIDE;
  const uint64_t chunk = 256ull * kU;
  for (uint64_t c0 = (uint64_t)blockIdx.x * chunk; c0 < n; c0 += (uint64_t)gridDim.x * chunk) {
    uint32_t w[kU][W + 1];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t i = c0 + u * 256 + threadIdx.x;
      if (i < n) qmpm::load_words<Spec>(words + i * W, w[u]);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t i = c0 + u * 256 + threadIdx.x;
      if (i >= n) continue;
      float row[ST];
#pragma unroll
      for (int q = 0; q < ST; ++q) row[q] = 0.0f;
#pragma unroll
      for (int f = 0; f < NF; ++f) row[Spec::col(f)] = qmpm::sdec<Spec>(w[u], f);
      qmpm::store_row<ST, Spec::VV>(vals + i * ST, row);
    }
  }
}

// out = M A for each record's 3x3 matrix M (fields 0..8 = M row-major), fp32 with the
// products summed left to right without FMA: out[r][c] = (M[r][0] A[0][c] +
// M[r][1] A[1][c]) + M[r][2] A[2][c], then re-encoded (dithered with keys[i] when given).
struct QmpmMat3 {
  float a[9];
};
extern "C" __global__ void __launch_bounds__(256) qmpm_codec_matmul3(const uint32_t* __restrict__ in, uint64_t n,
                                                                     QmpmMat3 A, const uint32_t* __restrict__ keys,
                                                                     uint32_t salt, uint32_t* __restrict__ out) {
  constexpr int W = Spec::W;
  if constexpr (Spec::NF != 9) return;  // records must hold a 3x3 matrix (the host checks)
  const uint64_t chunk = 256ull * kU;
  for (uint64_t c0 = (uint64_t)blockIdx.x * chunk; c0 < n; c0 += (uint64_t)gridDim.x * chunk) {
    uint32_t wi[kU][W + 1], key[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t i = c0 + u * 256 + threadIdx.x;
#pragma unroll
      for (int q = 0; q <= W; ++q) wi[u][q] = 0u;
      key[u] = 0u;
      if (i < n) {
        qmpm::load_words<Spec>(in + i * W, wi[u]);
        if (Spec::DITHER) key[u] = __ldg(keys + i);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t i = c0 + u * 256 + threadIdx.x;
      const bool valid = i < n;
      float m[9], v[9];
#pragma unroll
      for (int f = 0; f < 9; ++f) m[f] = qmpm::sdec<Spec>(wi[u], f < Spec::NF ? f : 0);
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          v[3 * r + c] = __fadd_rn(__fadd_rn(__fmul_rn(m[3 * r], A.a[c]), __fmul_rn(m[3 * r + 1], A.a[3 + c])),
                                   __fmul_rn(m[3 * r + 2], A.a[6 + c]));
      const uint32_t h = Spec::DITHER ? qmpm::mix32(key[u] ^ salt) : 0u;
      uint32_t o[W + 1];
      qmpm::encode_record<Spec>(v, h, valid, o, nullptr);
      if (valid) qmpm::store_words<Spec>(out + i * W, o);
    }
  }
}
