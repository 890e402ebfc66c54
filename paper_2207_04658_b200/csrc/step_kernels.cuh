// step_kernels.cuh -- the layout-specialised kernels of one quantized MLS-MPM step.
//
// Compiled at qmpm_create by NVRTC for sm_100a, after a generated preamble that
// defines `struct Spec` (the scheme's bit-pack layout as compile-time constants:
// per state scalar its word, shift, width, kind, Delta, 1/Delta, offset and packing
// index).  With the layout constant, every field access is a constant shift/mask on
// a record held in REGISTERS (bit pack load, Fig. bit_pack_operation), and
// the re-encode packs into registers (no read-modify-write of shared words).
//
//   qmpm_bin_count  a1        block key + histogram (first step after set_state/set_words)
//   qmpm_p2g        a2+a3     decode, stress, scatter into per-warp shared-memory tiles
//                             (lanes of one round have distinct base cells, so the
//                             tile RMW needs no atomics), red.global.add.v4.f32 flush
//   qmpm_g2p        a2+a5-a7  gather from a shared-memory tile, update, dithered encode,
//                             coalesced store in sorted order, next step's block key
#pragma once
#include "mpm_common.cuh"

namespace qmpm {

// ------------------------------------------------------------------ field access
// value of state scalar i from a register-resident record w[0..W] (w[W] = 0)
template <class SP>
__device__ __forceinline__ float sdec(const uint32_t* w, const int i) {
  const int wd = SP::word(i), sh = SP::shift(i), wi = SP::width(i);
  const uint32_t raw = (sh + wi <= 32) ? (w[wd] >> sh) : __funnelshift_r(w[wd], w[wd + 1], sh);
  if (SP::kind(i) == kKindRaw) return __uint_as_float(raw);
  const int u = ((int)(raw << (32 - wi))) >> (32 - wi);  // sign-extend b+1 bits (Q2)
  float x = __fmul_rn(__int2float_rn(u), SP::delta(i));   // Eq. 3: u * Delta
  if (SP::offset(i) != 0.0f) x = __fadd_rn(x, SP::offset(i));
  return x;
}

struct EncFlags {
  bool up, down, sat, nonfinite;
};

// Eq. 3 / Eq. 11 encode of state scalar i; returns the field's bits (width-masked).
template <class SP>
__device__ __forceinline__ uint32_t senc(const int i, float v, uint32_t r24, EncFlags& fl) {
  fl.up = fl.down = fl.sat = fl.nonfinite = false;
  if (SP::kind(i) == kKindRaw) {
    fl.nonfinite = !isfinite(v);
    return __float_as_uint(v);
  }
  const int wi = SP::width(i);
  if (!isfinite(v)) {
    fl.nonfinite = true;
    return 0u;
  }
  const float a = (SP::offset(i) != 0.0f) ? __fsub_rn(v, SP::offset(i)) : v;
  const float t = __fmul_rn(a, SP::inv_delta(i));  // one fp32 multiply, no FMA (Q3)
  const uint32_t mask = (wi == 32) ? 0xffffffffu : ((1u << wi) - 1u);
  if (wi <= 25) {
    // |codes| <= 2^24: clamping f to [-2^b - 2, 2^b] (exact floats) keeps every
    // saturation decision of the exact integer rule
    const float lo_f = -(float)(1 << (wi - 1)) - 2.0f, hi_f = (float)(1 << (wi - 1));
    const int lo = -(1 << (wi - 1)), hi = (1 << (wi - 1)) - 1;
    int u;
    if (SP::DITHER) {
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
    if (SP::DITHER) {
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

template <class SP>
__device__ __forceinline__ void sput(uint32_t* w, const int i, uint32_t bits) {
  const int wd = SP::word(i), sh = SP::shift(i), wi = SP::width(i);
  w[wd] |= bits << sh;
  if (sh + wi > 32) w[wd + 1] |= bits >> (32 - sh);
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

// ------------------------------------------------------------------ staging
// Warp-cooperative load of the warp's cnt records (record index of lane l in r_lane)
// into registers w[0..W] of their owner lane.  The words go global -> shared with
// cp.async (LDGSTS: no registers held while the W loads are in flight), then each
// lane reads its own conflict-free (odd-stride) row.  issue_records / take_records
// split the two halves so the next chunk's records can be in flight while the
// current chunk computes (double-buffered stage).
template <class SP>
__device__ __forceinline__ void issue_records(const uint32_t* __restrict__ rec, uint32_t r_lane, uint32_t cnt,
                                              uint32_t* wst, int lane) {
  constexpr int W = SP::W, SW = SP::SW;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(wst);
#pragma unroll
  for (int k = 0; k < W; ++k) {
    const uint32_t q = (uint32_t)(k * 32 + lane);
    const uint32_t l = q / W, o = q - l * W;
    const uint32_t r = __shfl_sync(FULL, r_lane, (int)(l & 31u));
    if (l < cnt) {
      const unsigned sa = sbase + 4u * (l * SW + o);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(rec + (size_t)r * W + o) : "memory");
    }
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

template <class SP>
__device__ __forceinline__ void take_records(const uint32_t* wst, int lane, uint32_t* w) {
  constexpr int W = SP::W, SW = SP::SW;
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncwarp();
#pragma unroll
  for (int k = 0; k < W; ++k) w[k] = wst[lane * SW + k];
  w[W] = 0u;
  __syncwarp();
}

template <class SP>
__device__ __forceinline__ void load_records(const uint32_t* __restrict__ rec, uint32_t r_lane, uint32_t cnt,
                                             uint32_t* wst, int lane, uint32_t* w) {
  issue_records<SP>(rec, r_lane, cnt, wst, lane);
  take_records<SP>(wst, lane, w);
}

// coalesced store of the warp's cnt records (lane l holds record l in w) to out[0..cnt*W)
template <class SP>
__device__ __forceinline__ void store_records(uint32_t* __restrict__ out, uint32_t cnt, uint32_t* wst, int lane,
                                              const uint32_t* w) {
  constexpr int W = SP::W, SW = SP::SW;
#pragma unroll
  for (int k = 0; k < W; ++k) wst[lane * SW + k] = w[k];
  __syncwarp();
#pragma unroll
  for (int k = 0; k < W; ++k) {
    const uint32_t q = (uint32_t)(k * 32 + lane);
    const uint32_t l = q / W, o = q - l * W;
    const uint32_t val = wst[l * SW + o];
    if (l < cnt) out[q] = val;
  }
  __syncwarp();
}

// ------------------------------------------------------------------ a1: bin count
template <class SP>
__device__ __forceinline__ void bin_count_body(const uint32_t* __restrict__ rec, uint32_t first, uint32_t n,
                                               const SimDev& S, uint32_t* __restrict__ key,
                                               uint32_t* __restrict__ block_count, int do_count) {
  constexpr int D = SP::D, W = SP::W;
  const uint32_t i = first + blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = i < first + n;
  uint32_t k = 0xffffffffu;
  if (valid) {
    uint32_t w[W + 1];
#pragma unroll
    for (int q = 0; q < W; ++q) w[q] = ((SP::XMASK >> q) & 1u) ? __ldg(rec + (size_t)i * W + q) : 0u;
    w[W] = 0u;
    float x[3];
#pragma unroll
    for (int a = 0; a < D; ++a) x[a] = sdec<SP>(w, a);
    const uint32_t full = key_of<D>(x, S);
    key[i] = full;
    k = full >> 6;
  }
  if (!do_count) return;
  const unsigned peers = __match_any_sync(FULL, k);
  if (valid && (threadIdx.x & 31) == (unsigned)(__ffs(peers) - 1)) atomicAdd(&block_count[k], __popc(peers));
}

// ------------------------------------------------------------------ cell ordering
// Within a block, particles are processed in (rank within base cell, cell) order:
// position = P[r] + #{cells c' < c holding more than r particles}, P[r] = number of
// particles of rank < r.  Consecutive lanes then have distinct base cells (except
// across a level boundary, which the match_any rounds below absorb), so the
// per-warp tile RMW of one stencil offset never collides.
constexpr int kOrderCap = 1024;   // particles ordered per batch
constexpr int kOrderLevels = 128; // ranks with a level mask (higher ranks go last)

struct OrderSmem {
  uint32_t p[kOrderCap];           // perm entries of the batch
  uint32_t q[kOrderCap];           // reordered
  uint16_t rank[kOrderCap];
  uint8_t cell[kOrderCap];
  unsigned cnt[64];
  unsigned long long mask[kOrderLevels];
  unsigned lvl[kOrderLevels + 1];  // exclusive prefix of level sizes
  unsigned over;
  unsigned maxc;
};

__device__ __forceinline__ void order_batch(uint32_t* __restrict__ perm, const uint8_t* __restrict__ cells,
                                            uint32_t nb, OrderSmem& o) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
  if (tid < 64) o.cnt[tid] = 0u;
  if (tid == 0) {
    o.over = 0u;
    o.maxc = 0u;
  }
  __syncthreads();
  for (uint32_t i0 = tid - lane; i0 < nb; i0 += nt) {  // warp-uniform trip count
    const uint32_t i = i0 + lane;
    const bool v = i < nb;
    const uint32_t p = v ? perm[i] : 0u;
    const uint32_t c = v ? (uint32_t)cells[i] : 64u + lane;
    const unsigned peers = __match_any_sync(FULL, c);
    const int leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (v && lane == leader) base = atomicAdd(&o.cnt[c], (unsigned)__popc(peers));
    base = __shfl_sync(FULL, base, leader);
    if (v) {
      o.p[i] = p;
      o.cell[i] = (uint8_t)c;
      o.rank[i] = (uint16_t)(base + __popc(peers & lanemask_lt()));
    }
  }
  __syncthreads();
  if (tid < 64) atomicMax(&o.maxc, o.cnt[tid]);
  __syncthreads();
  const unsigned levels = min(o.maxc, (unsigned)kOrderLevels);
  if (tid < 64) {
    const int half = tid >> 5;
    const unsigned c = o.cnt[tid];
    for (unsigned r = 0; r < levels; ++r) {
      const unsigned b = __ballot_sync(FULL, c > r);
      if (lane == 0) reinterpret_cast<unsigned*>(&o.mask[r])[half] = b;
    }
  }
  __syncthreads();
  if (tid < 32) {  // level prefix, one warp
    unsigned run = 0;
    for (unsigned r0 = 0; r0 < levels; r0 += 32) {
      const unsigned r = r0 + lane;
      const unsigned sz = r < levels ? (unsigned)__popcll(o.mask[r]) : 0u;
      unsigned inc = sz;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const unsigned t = __shfl_up_sync(FULL, inc, d);
        if (lane >= d) inc += t;
      }
      if (r < levels) o.lvl[r] = run + inc - sz;
      run += __shfl_sync(FULL, inc, 31);
    }
    if (lane == 0) o.lvl[levels] = run;
  }
  __syncthreads();
  for (uint32_t i = tid; i < nb; i += nt) {
    const unsigned r = o.rank[i], c = o.cell[i];
    uint32_t pos;
    if (r < levels)
      pos = o.lvl[r] + (uint32_t)__popcll(o.mask[r] & ((1ull << c) - 1ull));
    else
      pos = o.lvl[levels] + atomicAdd(&o.over, 1u);
    o.q[pos] = o.p[i];
    perm[pos] = o.p[i];
  }
  __syncthreads();
}

#ifndef QMPM_CELL_CAP
#define QMPM_CELL_CAP 256
#endif
// per-warp shared-memory footprint of the two step kernels (16-byte multiples)
template <class SP>
struct Smem {
  static constexpr int TN = Geo<SP::D>::TN;
  static constexpr int TILE = 16 * TN;
  static constexpr int STAGE = ((4 * 32 * SP::SW) + 15) / 16 * 16;
  static constexpr int PRM = 4 * 16 * 32;
  // P2G (2 warps per CTA): per warp one tile, two chunk stages and half of the
  // [16][kCellCap] parameter block; + the CTA's CellSmem (static)
  static constexpr int P2G_WARP = TILE + 2 * STAGE + 16 * 4 * QMPM_CELL_CAP / 2;
  static constexpr int G2P_WARP = TILE + 2 * STAGE + 32;  // double-buffered stage + 8 neighbour slots
};

// ------------------------------------------------------------------ a3: P2G
// phase 1 of the scatter: decode + stress of the lane's particle -> 16 parameters
// (cell, fx, Q, a_k) parked in shared memory: the momentum at stencil node o is
// m v + aff (o - fx) dx = Q + sum_k o_k a_k with a_k = dx aff[:,k], Q = m v - sum_k fx_k a_k.
template <class SP>
__device__ __forceinline__ void p2g_params(const uint32_t* w, bool valid, const int org[3], const SimDev& S,
                                           float* prm, int stride) {
  const int lane = threadIdx.x & 31;
  constexpr int D = SP::D, MAT = SP::MAT, NSV = SP::NS;
  float s[NSV];
  if (valid) {
#pragma unroll
    for (int i = 0; i < NSV; ++i) s[i] = sdec<SP>(w, i);
  } else {
    benign_state<D, MAT>(s, org, S.dx);
  }
  int lb[3] = {0, 0, 0};
  float fx[3] = {0.f, 0.f, 0.f};
#pragma unroll
  for (int a = 0; a < D; ++a) {
    bool o;
    lb[a] = base_fx(s[a], S.inv_dx, S.res[a], fx[a], o) - org[a];
  }
  float aff[D * D];
  affine_of<D, MAT>(s, S, aff);
  float Q[3] = {0.f, 0.f, 0.f};
#pragma unroll
  for (int a = 0; a < D; ++a) {
    Q[a] = S.p_mass * s[D + a];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const float akv = S.dx * aff[a * D + k];
      Q[a] -= fx[k] * akv;
      if (valid) prm[(7 + k * 3 + a) * stride + lane] = akv;
    }
  }
  if (!valid) return;
  prm[0 * stride + lane] = __int_as_float(D == 3 ? (lb[0] * 4 + lb[1]) * 4 + lb[2] : lb[0] * 8 + lb[1]);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    prm[(1 + a) * stride + lane] = fx[a];
    prm[(4 + a) * stride + lane] = Q[a];
  }
}

// One CTA of 2 warps (64 lanes = the 64 base cells of a block) per active block,
// grid-stride.  Per batch of <= kCellCap particles of the block:
//   1. counting sort by base cell (cells[] from the scatter, warp-aggregated ranks);
//   2. phase 1: both warps stage records (cp.async, the next chunk in flight) and park
//      16 parameters per particle in shared memory (structure of arrays);
//   3. phase 2: lane c OWNS cell c: it loops over its cell's particles accumulating
//      one stencil layer (fixed ox: 3^(d-1) nodes x 4 channels) in registers, then
//      read-modify-writes those nodes of its warp's private tile.  Lanes own distinct
//      cells, so one layer's RMW never collides; __syncwarp orders successive nodes.
//      The shared-memory RMW count drops from 27 per particle to 27 per cell.
// The two warp tiles are summed and flushed with red.global.add.v4.f32.
#ifndef QMPM_CELL_CAP
#define QMPM_CELL_CAP 256
#endif
constexpr int kCellCap = QMPM_CELL_CAP;  // particles per P2G batch

struct CellSmem {
  uint32_t p[kCellCap];   // perm entries of the batch
  uint32_t q[kCellCap];   // sorted by cell
  uint16_t pos[kCellCap];
  uint8_t cell[kCellCap];
  uint32_t cnt[64];
  uint32_t cstart[65];
};

template <class SP>
__device__ __forceinline__ void p2g_body(const uint32_t* __restrict__ rec, uint32_t* __restrict__ perm,
                                         const uint8_t* __restrict__ cells,
                                         const uint32_t* __restrict__ block_start,
                                         const uint32_t* __restrict__ active_list,
                                         const DevCounters* __restrict__ dc,
                                         const uint32_t* __restrict__ block_slot, float4* __restrict__ mp,
                                         const SimDev& S) {
  constexpr int D = SP::D;
  using G = Geo<D>;
  using SM = Smem<SP>;
  constexpr int SWW = 32 * SP::SW;  // words per chunk stage
  extern __shared__ float4 smem4[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float4* tiles = smem4;                                                            // [2][TN]
  float* prm = reinterpret_cast<float*>(tiles + 2 * G::TN);                         // [16][kCellCap]
  uint32_t* stage = reinterpret_cast<uint32_t*>(prm + 16 * kCellCap);               // [2 warps][2][SWW]
  uint32_t* wst = stage + warp * 2 * SWW;
  float4* tile = tiles + warp * G::TN;
  __shared__ CellSmem cs;
  const uint32_t n_active = dc->n_active;

  for (uint32_t ab = blockIdx.x; ab < n_active; ab += gridDim.x) {
    const uint32_t b = active_list[ab];
    const uint32_t start = block_start[b], end = block_start[b + 1];
    int bc[3];
    block_coords<D>(b, S, bc);
    const int org[3] = {bc[0] * G::B, bc[1] * G::B, bc[2] * G::B};
    for (int t = tid; t < 2 * G::TN; t += 64) tiles[t] = make_float4(0.f, 0.f, 0.f, 0.f);

    // batches are strided samples of the block (element i of batch bi is block
    // particle bi + i * nbatch), so every batch spans all cells even when the block's
    // particles arrive grouped by cell
    const uint32_t n_blk = end - start;
    const uint32_t nbatch = (n_blk + kCellCap - 1) / kCellCap;
    for (uint32_t bi = 0; bi < nbatch; ++bi) {
      const uint32_t nb = (n_blk - bi + nbatch - 1) / nbatch;
      // ---- 1. counting sort of the batch by base cell
      cs.cnt[tid] = 0u;
      __syncthreads();
      for (uint32_t i0 = warp * 32; i0 < nb; i0 += 64) {
        const uint32_t i = i0 + lane;
        const bool v = i < nb;
        const uint32_t gi = start + bi + i * nbatch;
        const uint32_t c = v ? (uint32_t)cells[gi] : 64u + lane;
        const unsigned peers = __match_any_sync(FULL, c);
        const int leader = __ffs(peers) - 1;
        uint32_t base = 0;
        if (v && lane == leader) base = atomicAdd(&cs.cnt[c], (unsigned)__popc(peers));
        base = __shfl_sync(FULL, base, leader);
        if (v) {
          cs.p[i] = perm[gi];
          cs.cell[i] = (uint8_t)c;
          cs.pos[i] = (uint16_t)(base + __popc(peers & lanemask_lt()));
        }
      }
      __syncthreads();
      if (warp == 0) {  // exclusive scan of the 64 cell counts
        const uint32_t c0 = cs.cnt[lane], c1 = cs.cnt[lane + 32];
        uint32_t i0 = c0, i1 = c1;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t t0 = __shfl_up_sync(FULL, i0, d), t1 = __shfl_up_sync(FULL, i1, d);
          if (lane >= d) {
            i0 += t0;
            i1 += t1;
          }
        }
        const uint32_t tot0 = __shfl_sync(FULL, i0, 31);
        cs.cstart[lane] = i0 - c0;
        cs.cstart[lane + 32] = tot0 + i1 - c1;
        if (lane == 31) cs.cstart[64] = tot0 + i1;
      }
      __syncthreads();
      for (uint32_t i = tid; i < nb; i += 64) {
        const uint32_t q = cs.cstart[cs.cell[i]] + cs.pos[i];
        cs.q[q] = cs.p[i];
      }
      __syncthreads();
      // ---- 2. phase 1: parameters of every particle of the batch
      {
        int buf = 0;
        uint32_t j0 = warp * 32;
        if (j0 < nb) {
          const uint32_t c0 = min(32u, nb - j0);
          issue_records<SP>(rec, cs.q[j0 + ((uint32_t)lane < c0 ? lane : 0)], c0, wst, lane);
        }
        for (; j0 < nb; j0 += 64) {
          const uint32_t cnt = min(32u, nb - j0);
          const bool valid = (uint32_t)lane < cnt;
          uint32_t w[SP::W + 1];
          take_records<SP>(wst + buf * SWW, lane, w);
          const uint32_t jn = j0 + 64;
          if (jn < nb) {
            const uint32_t cn = min(32u, nb - jn);
            issue_records<SP>(rec, cs.q[jn + ((uint32_t)lane < cn ? lane : 0)], cn, wst + (buf ^ 1) * SWW, lane);
          }
          buf ^= 1;
          p2g_params<SP>(w, valid, org, S, prm + j0, kCellCap);
        }
      }
      __syncthreads();
      // ---- 3. phase 2: lane `tid` owns base cell `tid`
      {
        const int c = tid;
        const uint32_t k0 = cs.cstart[c], k1 = cs.cstart[c + 1];
        const unsigned has = __ballot_sync(FULL, k1 > k0);
        int lb[3];
        if (D == 3) {
          lb[0] = (c >> 4) & 3;
          lb[1] = (c >> 2) & 3;
          lb[2] = c & 3;
        } else {
          lb[0] = (c >> 3) & 7;
          lb[1] = c & 7;
          lb[2] = 0;
        }
        const int base_idx = D == 3 ? (lb[0] * G::T + lb[1]) * G::T + lb[2] : lb[0] * G::T + lb[1];
        const uint32_t kmax = __reduce_max_sync(FULL, k1 - k0);
        if (has) {
#pragma unroll 1
          for (int ox = 0; ox < 3; ++ox) {
            constexpr int NL = D == 3 ? 9 : 3;  // nodes of one layer
            float am[NL], ax[NL], ay[NL], az[NL];
#pragma unroll
            for (int q = 0; q < NL; ++q) am[q] = ax[q] = ay[q] = az[q] = 0.0f;
            for (uint32_t k = 0; k < kmax; ++k) {
              if (k0 + k < k1) {
                const uint32_t pi = k0 + k;
                const float fx0 = prm[1 * kCellCap + pi], fx1 = prm[2 * kCellCap + pi];
                float wq[3], wy[3], wz[3] = {1.f, 0.f, 0.f};
                bspline_w(fx0, wq);
                bspline_w(fx1, wy);
                if (D == 3) bspline_w(prm[3 * kCellCap + pi], wz);
                const float wxo = wq[ox];
                float M[3];
#pragma unroll
                for (int a = 0; a < 3; ++a) M[a] = prm[(4 + a) * kCellCap + pi] + ox * prm[(7 + a) * kCellCap + pi];
                float a1[3], a2[3];
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                  a1[a] = prm[(10 + a) * kCellCap + pi];
                  a2[a] = prm[(13 + a) * kCellCap + pi];
                }
#pragma unroll
                for (int oy = 0; oy < 3; ++oy) {
                  const float wxy = wxo * wy[oy];
                  float My[3] = {M[0] + oy * a1[0], M[1] + oy * a1[1], M[2] + oy * a1[2]};
#pragma unroll
                  for (int oz = 0; oz < (D == 3 ? 3 : 1); ++oz) {
                    const int q = D == 3 ? oy * 3 + oz : oy;
                    const float ww = D == 3 ? wxy * wz[oz] : wxy;
                    am[q] += ww;
                    ax[q] = fmaf(ww, My[0], ax[q]);
                    ay[q] = fmaf(ww, My[1], ay[q]);
                    az[q] = fmaf(ww, My[2], az[q]);
                    if (D == 3) {
                      My[0] += a2[0];
                      My[1] += a2[1];
                      My[2] += a2[2];
                    }
                  }
                }
              }
            }
            // one RMW per node of the layer (m = p_mass * sum w)
#pragma unroll
            for (int q = 0; q < NL; ++q) {
              const int oy = D == 3 ? q / 3 : q, oz = D == 3 ? q % 3 : 0;
              const int idx = base_idx + (D == 3 ? (ox * G::T + oy) * G::T + oz : ox * G::T + oy);
              if (k1 > k0) {
                float4 t = tile[idx];
                t.x = fmaf(am[q], S.p_mass, t.x);
                t.y += ax[q];
                t.z += ay[q];
                t.w += az[q];
                tile[idx] = t;
              }
              __syncwarp();
            }
          }
        }
      }
      __syncthreads();  // parameters and sort arrays are reused by the next batch
    }
    // flush: sum the two warp tiles, one vector reduction per non-empty node
    for (int t = tid; t < G::TN; t += 64) {
      const float4 a = tiles[t], o = tiles[G::TN + t];
      const float4 acc = make_float4(a.x + o.x, a.y + o.y, a.z + o.z, a.w + o.w);
      if (acc.x != 0.0f) {
        int node[3];
        tile_node<D>(t, org, node);
        int nbk[3], ln[3];
#pragma unroll
        for (int a2 = 0; a2 < 3; ++a2) {
          nbk[a2] = node[a2] >> G::LB;
          ln[a2] = node[a2] & (G::B - 1);
        }
        const uint32_t slot = block_slot[block_id<D>(nbk, S)];
        if (slot != 0xffffffffu) atomicAdd(&mp[(size_t)slot * 64 + local_node<D>(ln)], acc);
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ a5-a7: G2P + encode
// One WARP per active block: stage the block's (B+2)^d velocity tile, then gather,
// update, dither + pack in registers, store in sorted order, emit next step's key.
template <class SP>
__device__ __forceinline__ void g2p_body(const uint32_t* __restrict__ rec_in, uint32_t* __restrict__ rec_out,
                                         const uint32_t* __restrict__ perm, const uint32_t* __restrict__ ids_in,
                                         uint32_t* __restrict__ ids_out, float* __restrict__ dbg,
                                         uint32_t* __restrict__ key_out, uint32_t* __restrict__ block_count,
                                         const uint32_t* __restrict__ block_start,
                                         const uint32_t* __restrict__ active_list, DevCounters* __restrict__ dc,
                                         const uint32_t* __restrict__ block_slot, const float4* __restrict__ gv,
                                         const SimDev& S, uint32_t salt) {
  constexpr int D = SP::D, MAT = SP::MAT, NSV = SP::NS, WARPS = SP::G2P_WARPS, W = SP::W;
  constexpr int CO = 2 * D + (MAT == 1 ? 1 : D * D);
  using G = Geo<D>;
  using SM = Smem<SP>;
  extern __shared__ float4 smem4[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  char* wbase = reinterpret_cast<char*>(smem4) + warp * SM::G2P_WARP;
  float4* tile = reinterpret_cast<float4*>(wbase);
  uint32_t* wst = reinterpret_cast<uint32_t*>(wbase + SM::TILE);
  uint32_t* nslot = reinterpret_cast<uint32_t*>(wbase + SM::TILE + 2 * SM::STAGE);  // [4] / [8] neighbour slots
  // per-lane counters: lane f accumulates field-scalar f's round-ups / downs / saturations
  unsigned c_up = 0, c_down = 0, c_sat = 0, c_nf = 0, c_oob = 0;
  const uint32_t n_active = dc->n_active;
  const float four_inv_dx = 4.0f * S.inv_dx;

  for (uint32_t ab = blockIdx.x * WARPS + warp; ab < n_active; ab += gridDim.x * WARPS) {
    const uint32_t b = active_list[ab];
    const uint32_t start = block_start[b], end = block_start[b + 1];
    int bc[3];
    block_coords<D>(b, S, bc);
    const int org[3] = {bc[0] * G::B, bc[1] * G::B, bc[2] * G::B};
    // slots of the block and its +x/+y(/+z) neighbours, then the velocity tile
    if (lane < (1 << D)) {
      int nbk[3] = {bc[0] + (lane & 1), bc[1] + ((lane >> 1) & 1), D == 3 ? bc[2] + ((lane >> 2) & 1) : 0};
      uint32_t sl = 0xffffffffu;
      if (nbk[0] < S.nb[0] && nbk[1] < S.nb[1] && nbk[2] < S.nb[2]) sl = block_slot[block_id<D>(nbk, S)];
      nslot[lane] = sl;
    }
    __syncwarp();
    for (int t = lane; t < G::TN; t += 32) {
      int node[3];
      tile_node<D>(t, org, node);
      int sel = 0, ln[3] = {0, 0, 0};
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const int hi = (node[a] - org[a]) >= G::B;
        sel |= hi << a;
        ln[a] = node[a] & (G::B - 1);
      }
      const uint32_t slot = nslot[sel];
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (slot != 0xffffffffu) v = gv[(size_t)slot * 64 + local_node<D>(ln)];
      tile[t] = v;
    }
    __syncwarp();

    int buf = 0;
    uint32_t r_next = 0;
    if (start < end) {
      const uint32_t c0 = min(32u, end - start);
      r_next = perm[start + ((uint32_t)lane < c0 ? lane : 0)];
      issue_records<SP>(rec_in, r_next, c0, wst, lane);
    }
    for (uint32_t j0 = start; j0 < end; j0 += 32) {
      const uint32_t cnt = min(32u, end - j0);
      const bool valid = (uint32_t)lane < cnt;
      const uint32_t r = r_next;
      uint32_t* cur = wst + buf * 32 * SP::SW;
      uint32_t w[W + 1];
      take_records<SP>(cur, lane, w);
      {  // the next chunk's records go in flight while this one computes
        const uint32_t jn = j0 + 32;
        if (jn < end) {
          const uint32_t cn = min(32u, end - jn);
          r_next = perm[jn + ((uint32_t)lane < cn ? lane : 0)];
          issue_records<SP>(rec_in, r_next, cn, wst + (buf ^ 1) * 32 * SP::SW, lane);
        }
        buf ^= 1;
      }
      const uint32_t h = mix32(content_key<SP>(w) ^ salt);
      float s[NSV];
      if (valid) {
#pragma unroll
        for (int i = 0; i < NSV; ++i) s[i] = 0.0f;
#pragma unroll
        for (int i = 0; i < D; ++i) s[i] = sdec<SP>(w, i);
#pragma unroll
        for (int i = 2 * D; i < CO; ++i) s[i] = sdec<SP>(w, i);
      } else {
        benign_state<D, MAT>(s, org, S.dx);
      }
      int lb[3] = {0, 0, 0};
      float fx[3] = {0.f, 0.f, 0.f}, wt[3][3];
      bool oob_any = false;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        bool o;
        lb[a] = base_fx(s[a], S.inv_dx, S.res[a], fx[a], o) - org[a];
        oob_any |= o;
        bspline_w(fx[a], wt[a]);
      }
      // gather: v' = sum w v_i;  C' = 4/dx sum w v_i (x) (i - fx) = 4/dx (T - v' fx^T)
      float Sv[3] = {0.f, 0.f, 0.f}, T[3][3] = {{0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}};
      const int base_idx = D == 3 ? (lb[0] * G::T + lb[1]) * G::T + lb[2] : lb[0] * G::T + lb[1];
      if (D == 3) {
#pragma unroll
        for (int ox = 0; ox < 3; ++ox)
#pragma unroll
          for (int oy = 0; oy < 3; ++oy) {
            const float wxy = wt[0][ox] * wt[1][oy];
            const int idx = base_idx + (ox * G::T + oy) * G::T;
            const float4 g0 = tile[idx], g1 = tile[idx + 1], g2 = tile[idx + 2];
            const float g[3][3] = {{g0.x, g0.y, g0.z}, {g1.x, g1.y, g1.z}, {g2.x, g2.y, g2.z}};
#pragma unroll
            for (int a = 0; a < 3; ++a) {
              const float u0 = wt[2][0] * g[0][a], u1 = wt[2][1] * g[1][a], u2 = wt[2][2] * g[2][a];
              const float sz = u0 + u1 + u2;
              const float tz = u1 + 2.0f * u2;
              Sv[a] = fmaf(wxy, sz, Sv[a]);
              T[a][2] = fmaf(wxy, tz, T[a][2]);
              if (ox) T[a][0] = fmaf(wxy * ox, sz, T[a][0]);
              if (oy) T[a][1] = fmaf(wxy * oy, sz, T[a][1]);
            }
          }
      } else {
#pragma unroll
        for (int ox = 0; ox < 3; ++ox) {
          const int idx = base_idx + ox * G::T;
          const float4 g0 = tile[idx], g1 = tile[idx + 1], g2 = tile[idx + 2];
          const float g[3][2] = {{g0.x, g0.y}, {g1.x, g1.y}, {g2.x, g2.y}};
#pragma unroll
          for (int a = 0; a < 2; ++a) {
            const float u0 = wt[1][0] * g[0][a], u1 = wt[1][1] * g[1][a], u2 = wt[1][2] * g[2][a];
            const float sy = u0 + u1 + u2;
            const float ty = u1 + 2.0f * u2;
            Sv[a] = fmaf(wt[0][ox], sy, Sv[a]);
            T[a][1] = fmaf(wt[0][ox], ty, T[a][1]);
            if (ox) T[a][0] = fmaf(wt[0][ox] * ox, sy, T[a][0]);
          }
        }
      }
      float Cn[D * D];
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int k = 0; k < D; ++k) Cn[a * D + k] = four_inv_dx * (T[a][k] - Sv[a] * fx[k]);
      float o[NSV];
#pragma unroll
      for (int a = 0; a < D; ++a) {
        o[a] = s[a] + S.dt * Sv[a];
        o[D + a] = Sv[a];
      }
      if (MAT == 1) {
        float tr = 0.f;
#pragma unroll
        for (int a = 0; a < D; ++a) tr += Cn[a * D + a];
        o[2 * D] = s[2 * D] * (1.0f + S.dt * tr);
      } else {
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
          for (int k = 0; k < D; ++k) {
            float acc = s[2 * D + a * D + k];
#pragma unroll
            for (int m = 0; m < D; ++m) acc = fmaf(S.dt * Cn[a * D + m], s[2 * D + m * D + k], acc);
            o[2 * D + a * D + k] = acc;
          }
      }
#pragma unroll
      for (int i = 0; i < D * D; ++i) o[CO + i] = Cn[i];
      const uint32_t j = j0 + lane;
      if (dbg != nullptr && valid) {
#pragma unroll
        for (int i = 0; i < NSV; ++i) dbg[(size_t)j * NSV + i] = o[i];
      }
      // dithered encode into registers (Eq. 11; reading Q5, Q6)
      uint32_t ow[W + 1];
#pragma unroll
      for (int q = 0; q <= W; ++q) ow[q] = 0u;
      bool any_flag = false;
#pragma unroll
      for (int i = 0; i < NSV; ++i) {
        const uint32_t r24 = (SP::DITHER && SP::kind(i) == kKindFixed) ? r24_of(h, SP::idx(i)) : 0u;
        EncFlags fl;
        const uint32_t bits = senc<SP>(i, o[i], r24, fl);
        sput<SP>(ow, i, bits);
        if (SP::COUNTERS && SP::kind(i) == kKindFixed) {
          const unsigned bu = __ballot_sync(FULL, valid && fl.up);
          const unsigned bd = __ballot_sync(FULL, valid && fl.down);
          if (lane == i) {
            c_up += __popc(bu);
            c_down += __popc(bd);
          }
        }
        if (valid && (fl.sat || fl.nonfinite)) any_flag = true;
      }
      if (__any_sync(FULL, any_flag)) {  // rare: recount saturations / non-finite
#pragma unroll
        for (int i = 0; i < NSV; ++i) {
          EncFlags fl;
          const uint32_t r24 = (SP::DITHER && SP::kind(i) == kKindFixed) ? r24_of(h, SP::idx(i)) : 0u;
          senc<SP>(i, o[i], r24, fl);
          const unsigned bs = __ballot_sync(FULL, valid && fl.sat);
          const unsigned bn = __ballot_sync(FULL, valid && fl.nonfinite);
          if (lane == i) c_sat += __popc(bs);
          if (lane == 0) c_nf += __popc(bn);
        }
      }
      {
        const unsigned bo = __ballot_sync(FULL, valid && oob_any);
        if (lane == 0) c_oob += __popc(bo);
      }
      // next step's sort key from the re-decoded (quantized) x
      float xq[3];
#pragma unroll
      for (int a = 0; a < D; ++a) xq[a] = sdec<SP>(ow, a);
      const uint32_t nkey = key_of<D>(xq, S);
      if (valid) key_out[j] = nkey;
      const uint32_t nk = valid ? (nkey >> 6) : 0xffffffffu;
      const unsigned kp = __match_any_sync(FULL, nk);
      if (valid && lane == __ffs(kp) - 1) atomicAdd(&block_count[nk], (unsigned)__popc(kp));
      if (ids_out != nullptr && valid) ids_out[j] = ids_in[r];
      store_records<SP>(rec_out + (size_t)j0 * W, cnt, cur, lane, ow);
    }
    __syncwarp();
  }
  // flush this thread's counters (lane i holds scalar i's counts)
  if (lane < NSV) {
    int fi = 0;
#pragma unroll
    for (int i = 0; i < NSV; ++i)
      if (lane == i) fi = SP::idx(i);
    if (c_up) atomicAdd(&dc->up[fi], (unsigned long long)c_up);
    if (c_down) atomicAdd(&dc->down[fi], (unsigned long long)c_down);
    if (c_sat) atomicAdd(&dc->sat[fi], (unsigned long long)c_sat);
  }
  if (c_nf) atomicAdd(&dc->nonfinite, (unsigned long long)c_nf);
  if (c_oob) atomicAdd(&dc->oob, (unsigned long long)c_oob);
}

}  // namespace qmpm

// ------------------------------------------------------------------ entry points
// per-warp shared-memory bytes of P2G and G2P, read by the host after loading the module
extern "C" __device__ const unsigned qmpm_smem_per_warp[2] = {(unsigned)qmpm::Smem<Spec>::P2G_WARP,
                                                             (unsigned)qmpm::Smem<Spec>::G2P_WARP};
extern "C" __global__ void __launch_bounds__(256) qmpm_bin_count(const uint32_t* rec, uint32_t first, uint32_t n,
                                                                 qmpm::SimDev S, uint32_t* key, uint32_t* block_count,
                                                                 int do_count) {
  qmpm::bin_count_body<Spec>(rec, first, n, S, key, block_count, do_count);
}

extern "C" __global__ void __launch_bounds__(64, Spec::P2G_MINB)
    qmpm_p2g(const uint32_t* rec, uint32_t* perm, const uint8_t* cells, const uint32_t* block_start,
             const uint32_t* active_list, const qmpm::DevCounters* dc, const uint32_t* block_slot, float4* mp,
             qmpm::SimDev S) {
  qmpm::p2g_body<Spec>(rec, perm, cells, block_start, active_list, dc, block_slot, mp, S);
}

extern "C" __global__ void __launch_bounds__(Spec::G2P_WARPS * 32, Spec::G2P_MINB)
    qmpm_g2p(const uint32_t* rec_in, uint32_t* rec_out, const uint32_t* perm, const uint32_t* ids_in,
             uint32_t* ids_out, float* dbg, uint32_t* key_out, uint32_t* block_count, const uint32_t* block_start,
             const uint32_t* active_list, qmpm::DevCounters* dc, const uint32_t* block_slot, const float4* gv,
             qmpm::SimDev S, uint32_t salt) {
  qmpm::g2p_body<Spec>(rec_in, rec_out, perm, ids_in, ids_out, dbg, key_out, block_count, block_start, active_list,
                       dc, block_slot, gv, S, salt);
}
