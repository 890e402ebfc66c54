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
#include "codec_record.cuh"

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
