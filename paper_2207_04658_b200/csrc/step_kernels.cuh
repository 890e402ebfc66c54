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
//   qmpm_p2g        a2+a3     balanced per-cell segments; a lane accumulates its segment's
//                             3^d stencil in registers; one tile RMW per node per
//                             segment (no atomics), red.global.add.v4.f32 flush
//   qmpm_g2p        a2+a5-a7  gather from a shared-memory tile, update, dithered encode,
//                             coalesced store in sorted order, next step's block key
#pragma once
#include "field_codec.cuh"
#include "mpm_common.cuh"

namespace qmpm {

// ------------------------------------------------------------------ slab migration
// (MigDev / MigHeader: qmpm_device.cuh)
__device__ __forceinline__ MigHeader* mig_hdr(unsigned char* b) { return reinterpret_cast<MigHeader*>(b); }
__device__ __forceinline__ const MigHeader* mig_hdr(const unsigned char* b) {
  return reinterpret_cast<const MigHeader*>(b);
}
__device__ __forceinline__ size_t mig_rec_off() { return sizeof(MigHeader); }

// a particle whose base block plane lies outside this rank's slab: its record (and id)
// go to the neighbour's send buffer; `slot` (nullable) is remembered as a dead slot
template <int W>
__device__ __forceinline__ void mig_push(const MigDev& M, DevCounters* dc, int side, const uint32_t* rec,
                                         uint32_t id, uint32_t slot, const float* dbg_row) {
  if (side != -1 && side != 1) {
    atomicOr(&dc->status, kStatusTwoHop);
    return;
  }
  unsigned char* buf = side > 0 ? M.send[1] : M.send[0];  // (no dynamic index into the param)
  const uint32_t k = atomicAdd(&mig_hdr(buf)->count, 1u);
  if (k >= M.cap) {
    atomicOr(&dc->status, kStatusMigOverflow);
    return;
  }
  uint32_t* dst = reinterpret_cast<uint32_t*>(buf + mig_rec_off()) + (size_t)k * W;
#pragma unroll
  for (int q = 0; q < W; ++q) dst[q] = rec[q];
  if (M.ids) reinterpret_cast<uint32_t*>(buf + mig_ids_off(M))[k] = id;
  if (M.dbg_ns && dbg_row) {
    float* dd = reinterpret_cast<float*>(buf + mig_dbg_off(M)) + (size_t)k * M.dbg_ns;
    for (uint32_t q = 0; q < M.dbg_ns; ++q) dd[q] = dbg_row[q];
  }
  const uint32_t dk = atomicAdd(&dc->n_leave, 1u);
  if (dk < M.dead_cap) M.dead_list[dk] = slot;
}

// ------------------------------------------------------------------ a1: bin count
// keys (+ histograms) of records [first, first + n); on a slab rank a record whose base
// lies in a neighbour's slab is routed to it (first step after set_state: reading of
// qmpm_create_slab, particles may start in an adjacent slab)
template <class SP>
__device__ __forceinline__ void bin_count_body(const uint32_t* __restrict__ rec, const uint32_t* __restrict__ ids,
                                               uint32_t first, uint32_t n, const SimDev& S,
                                               uint32_t* __restrict__ key, uint32_t* __restrict__ block_count,
                                               uint32_t* __restrict__ cell_count, int do_count, MigDev M,
                                               DevCounters* dc) {
  constexpr int D = SP::D, W = SP::W;
  const uint32_t i = first + blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = i < first + n;
  uint32_t k = 0xffffffffu, full = kDeadKey;
  if (valid) {
    uint32_t w[W + 1];
#pragma unroll
    for (int q = 0; q < W; ++q) w[q] = __ldg(rec + (size_t)i * W + q);
    w[W] = 0u;
    float x[3];
#pragma unroll
    for (int a = 0; a < D; ++a) x[a] = sdec<SP>(w, a);
    int bsv[3] = {0, 0, 0};
#pragma unroll
    for (int a = 0; a < D; ++a) {
      float fx;
      bool o;
      bsv[a] = base_fx(x[a], S.inv_dx, S.res[a], fx, o);
    }
    const int side = (SP::SLAB && D == 3) ? slab_side(bsv[2] >> 2, S) : 0;
    if (side == 0) {
      full = key_from_base<D>(bsv, S);
      k = full >> 6;
    } else {
      mig_push<W>(M, dc, side, w, ids ? ids[i] : 0u, i, nullptr);
    }
    key[i] = full;
  }
  if (!do_count) return;
  const unsigned peers = __match_any_sync(FULL, k);
  if (k != 0xffffffffu && (threadIdx.x & 31) == (unsigned)(__ffs(peers) - 1)) atomicAdd(&block_count[k], __popc(peers));
  const unsigned cp = __match_any_sync(FULL, full);
  if (full != kDeadKey && (threadIdx.x & 31) == (unsigned)(__ffs(cp) - 1)) atomicAdd(&cell_count[full], __popc(cp));
}

// Arrivals from the two neighbours (their headers give the counts) are appended at the
// record slots [n_rec, n_rec + arrivals) with their keys and histogram counts; n_slots
// (the sort's slot range) becomes n_rec + arrivals.  The statuses the neighbours sent
// are folded into this rank's sticky status.
template <class SP>
__device__ __forceinline__ void append_body(uint32_t* __restrict__ rec, uint32_t* __restrict__ ids, float* __restrict__ dbg,
                                            uint64_t cap, const SimDev& S, uint32_t* __restrict__ key,
                                            uint32_t* __restrict__ block_count, uint32_t* __restrict__ cell_count,
                                            MigDev M, DevCounters* dc) {
  constexpr int D = SP::D, W = SP::W;
  const MigHeader* h0 = mig_hdr(M.recv[0]);
  const MigHeader* h1 = mig_hdr(M.recv[1]);
  const uint32_t c0 = min(h0->count, M.cap), c1 = min(h1->count, M.cap);
  const uint32_t n0 = dc->n_rec;
  const uint32_t arr = c0 + c1;
  const uint32_t fit = (uint64_t)n0 + arr > cap ? (uint32_t)(cap - n0) : arr;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    dc->n_slots = n0 + fit;
    const unsigned st = h0->status | h1->status | ((h0->count > M.cap || h1->count > M.cap) ? kStatusMigOverflow : 0u) |
                        (fit < arr ? kStatusCapacity : 0u);
    if (st) atomicOr(&dc->status, st);
  }
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < ((fit + 31u) & ~31u); t += gridDim.x * blockDim.x) {
    const bool valid = t < fit;
    uint32_t k = 0xffffffffu, full = kDeadKey;
    if (valid) {
      const int dir = t < c0 ? 0 : 1;
      const uint32_t q = dir ? t - c0 : t;
      const unsigned char* rb = dir ? M.recv[1] : M.recv[0];  // (no dynamic index into the param)
      const uint32_t* src = reinterpret_cast<const uint32_t*>(rb + mig_rec_off()) + (size_t)q * W;
      uint32_t w[W + 1];
#pragma unroll
      for (int e = 0; e < W; ++e) w[e] = src[e];
      w[W] = 0u;
      const uint32_t slot = n0 + t;
#pragma unroll
      for (int e = 0; e < W; ++e) rec[(size_t)slot * W + e] = w[e];
      if (ids) ids[slot] = reinterpret_cast<const uint32_t*>(rb + mig_ids_off(M))[q];
      if (dbg && M.dbg_ns) {
        const float* sd = reinterpret_cast<const float*>(rb + mig_dbg_off(M)) + (size_t)q * M.dbg_ns;
        for (uint32_t e = 0; e < M.dbg_ns; ++e) dbg[(size_t)slot * M.dbg_ns + e] = sd[e];
      }
      float x[3];
      int bsv[3] = {0, 0, 0};
#pragma unroll
      for (int a = 0; a < D; ++a) {
        x[a] = sdec<SP>(w, a);
        float fx;
        bool o;
        bsv[a] = base_fx(x[a], S.inv_dx, S.res[a], fx, o);
      }
      if (slab_side(bsv[2] >> 2, S) == 0) {
        full = key_from_base<D>(bsv, S);
        k = full >> 6;
      } else {
        atomicOr(&dc->status, kStatusTwoHop);  // (CFL: one hop per step)
      }
      key[slot] = full;
    }
    const unsigned peers = __match_any_sync(FULL, k);
    if (k != 0xffffffffu && (threadIdx.x & 31) == (unsigned)(__ffs(peers) - 1)) atomicAdd(&block_count[k], __popc(peers));
    const unsigned cp = __match_any_sync(FULL, full);
    if (full != kDeadKey && (threadIdx.x & 31) == (unsigned)(__ffs(cp) - 1)) atomicAdd(&cell_count[full], __popc(cp));
  }
}

// per-warp shared-memory footprint of the two step kernels (16-byte multiples)
template <class SP>
struct Smem {
  static constexpr int TN = Geo<SP::D>::TN;
  static constexpr int TILE = 16 * TN;
  // velocity tile + 8 neighbour slots + double-buffered record stage + tile node table
  static constexpr int STAGE = TILE + 32;
  static constexpr int TNODE = STAGE + (2 * 32 * 4 * SP::W + 15) / 16 * 16;
  static constexpr int G2P_WARP = TNODE + (2 * TN + 15) / 16 * 16;
};

// tile node t -> which of the 2^d blocks a (B+2)^d tile spans it lies in (bit a: the +a
// neighbour) and its node inside that block: u16 (sel << 6 | node), the same for every
// block, built once per warp
template <int D>
__device__ __forceinline__ void build_tile_nodes(uint16_t* tn, int lane) {
  using G = Geo<D>;
  for (int t = lane; t < G::TN; t += 32) {
    int node[3];
    const int zero[3] = {0, 0, 0};
    tile_node<D>(t, zero, node);
    int sel = 0, ln[3] = {0, 0, 0};
#pragma unroll
    for (int a = 0; a < D; ++a) {
      sel |= (node[a] >= G::B) << a;
      ln[a] = node[a] & (G::B - 1);
    }
    tn[t] = (uint16_t)((sel << 6) | (int)local_node<D>(ln));
  }
}

// Per-lane asynchronous copy of record r (W words) into shared memory (cp.async, no
// registers held while in flight; 16-byte granules when the record size allows).
// The caller commits the group and waits with cp_async_wait<N>.
template <class SP>
__device__ __forceinline__ void record_async(const uint32_t* __restrict__ rec, uint32_t r, uint32_t* dst) {
  constexpr int W = SP::W;
  const uint32_t* src = rec + (size_t)r * W;
  const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  if (W % 4 == 0) {
#pragma unroll
    for (int q = 0; q < W / 4; ++q)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa + 16u * q), "l"(src + 4 * q) : "memory");
  } else if (W % 2 == 0) {
#pragma unroll
    for (int q = 0; q < W / 2; ++q)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa + 8u * q), "l"(src + 2 * q) : "memory");
  } else {
#pragma unroll
    for (int q = 0; q < W; ++q)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa + 4u * q), "l"(src + q) : "memory");
  }
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// read a record this thread staged (row of W words, 16/8-byte aligned as staged)
template <class SP>
__device__ __forceinline__ void read_staged(const uint32_t* row, uint32_t* w) {
  constexpr int W = SP::W;
  if (W % 4 == 0) {
#pragma unroll
    for (int q = 0; q < W / 4; ++q) {
      const uint4 v = reinterpret_cast<const uint4*>(row)[q];
      w[4 * q] = v.x;
      w[4 * q + 1] = v.y;
      w[4 * q + 2] = v.z;
      w[4 * q + 3] = v.w;
    }
  } else if (W % 2 == 0) {
#pragma unroll
    for (int q = 0; q < W / 2; ++q) {
      const uint2 v = reinterpret_cast<const uint2*>(row)[q];
      w[2 * q] = v.x;
      w[2 * q + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int q = 0; q < W; ++q) w[q] = row[q];
  }
  w[W] = 0u;
}

// ------------------------------------------------------------------ a3: P2G
// One WARP per active block (taken dynamically from a work counter; the warps of a CTA
// are independent, so there is no CTA barrier and no tail).  The global counting sort
// orders particles by (block, base cell) and its cursors leave each cell's start in
// cell_count, so the block's 64 cell ranges are known without a local sort.
//   1. segment table: cell c is cut into full segments of L particles (listed
//      level-major: all first segments in cell order, then all second segments, ...)
//      and one tail segment (the tails sorted by length); group g = entries
//      [32 g, 32 g + 32), one segment per lane: lanes get near-equal work whatever the
//      cells' occupancy;
//   2. a lane walks its segment: records stream through a per-lane 3-slot cp.async ring
//      (two in flight), decode, stress and affine momentum, and it accumulates all 3^d
//      stencil nodes x (m, p) in REGISTERS -- no shared-memory traffic per particle;
//   3. per group, one read-modify-write per stencil node per lane into the warp's
//      private tile: lanes holding distinct cells touch distinct nodes for a fixed
//      offset; lanes sharing a cell (a group straddling two levels) take turns;
//   4. the tile is flushed with one red.global.add.v4.f32 per non-empty node.
// Momentum at stencil node o of a particle: m v + aff (o - fx) dx = Q + sum_k o_k a_k,
// a_k = dx aff[:, k], Q = m v - sum_k fx_k a_k (Hu et al. 2018 APIC/MLS form).
#ifndef QMPM_SEG_L
#define QMPM_SEG_L 48
#endif
// A/B switches of micro-optimisations (tools/ab_step.py; defaults = the measured winners)
#ifndef QMPM_AB_P2G_PF
#define QMPM_AB_P2G_PF 0  // (measured at C4: 6.92 with vs 7.22 ms without before IDX_FIRST; after it 6.24 without vs 6.28-6.33 with)
#endif
#ifndef QMPM_AB_CNT_LOP3
#define QMPM_AB_CNT_LOP3 0  // (measured: 9.996 vs 10.132 ms G2P at C4 -- the shift-add form wins)
#endif
#ifndef QMPM_AB_TILE_PACK
#define QMPM_AB_TILE_PACK 0  // P2G: tile (m, p_z, p_x, p_y) with packed node updates (measured slower:
                              // C4 P2G 6.54 vs 6.25 ms, C3 10.79 vs 10.60 -- the per-node RMW chain is latency-bound)
#endif
#ifndef QMPM_AB_DPACK
#define QMPM_AB_DPACK 0  // P2G: decode scaling of same-Delta scalar pairs as FMUL2 (A/B variant)
#endif
#ifndef QMPM_AB_P2G_NEXT
#define QMPM_AB_P2G_NEXT 0  // P2G: claim the next block one block ahead (measured: C3 P2G 10.60 vs
                            // 10.66 ms, 8 ppc 9.01 vs 9.06, C4 6.44 vs 6.33-6.38 -- noise-level, off)
#endif
#ifndef QMPM_AB_CNT_NEG
#define QMPM_AB_CNT_NEG 0  // G2P round counters: count not-up from 255 down (one LEA per field);
                           // 2: fluid specs only (measured within noise: C4 G2P 9.645 vs 9.72-9.74 ms on
                           // one box, 9.78-9.86 vs 9.75 on another; C3 11.41 vs 11.34)
#endif
#ifndef QMPM_AB_P2G_PACK
#define QMPM_AB_P2G_PACK 1  // P2G: packed weight products and node momenta (3D)
#endif
#ifndef QMPM_AB_G2P_IDX_FIRST
#define QMPM_AB_G2P_IDX_FIRST 0  // G2P: the chunk-after-next's indices load before the next chunk's copies
#endif
#ifndef QMPM_AB_IDX_FIRST
#define QMPM_AB_IDX_FIRST 1  // P2G: the next record index loads before the current record's copy (C4 P2G 6.90 -> 6.39 ms)
#endif
#ifndef QMPM_AB_BCNT
#define QMPM_AB_BCNT 1  // G2P: the next step's count of the current block summed per block
#endif
#ifndef QMPM_AB_ZPACK
#define QMPM_AB_ZPACK 1  // (measured: G2P 10.13 vs 10.23 ms at C4 with the round counters)
#endif
#ifndef QMPM_SEG_LMIN
#define QMPM_SEG_LMIN 48
#endif
// particles per P2G segment (one lane, one group): n_blk / 128 clamped to [kSegLmin, kSegL]
// (QMPM_SEG_LMIN < QMPM_SEG_L shortens the segments of sparse blocks so every lane gets
// work; measured on B200: at C4 (~72 ppc) P2G takes 7.15 / 7.07 / 6.99 ms with segments
// of 16 / 24 / 32 particles and 6.85 vs 6.92 with 48 vs 32 (paired A/B on one state,
// tools/ab_step.py) -- fewer per-group tile updates; at 8 ppc every cell is one
// tail segment whatever the length, and a floor of 8 was 2.5 % slower there than 16)
constexpr int kSegL = QMPM_SEG_L;
constexpr int kSegLmin = QMPM_SEG_LMIN < QMPM_SEG_L ? QMPM_SEG_LMIN : QMPM_SEG_L;
constexpr int kSegLev = 32;        // segments per cell at most (the last one takes the rest)

// per-warp shared-memory layout of P2G (byte offsets; 16-byte aligned parts first)
template <class SP>
struct P2GLayout {
  static constexpr int TN = Geo<SP::D>::TN;
  static constexpr int TILE = 0;                               // float4[TN]
  static constexpr int RING = TILE + 16 * TN;                  // u32[3][32][W]
  static constexpr int START = RING + 3 * 32 * 4 * SP::W;      // u32[65]
  static constexpr int LSTART = START + 4 * 68;                // u32[kSegLev]
  static constexpr int SEG = LSTART + 4 * kSegLev;             // u16[64 * kSegLev]
  static constexpr int NS = SEG + 2 * 64 * kSegLev;            // u8[64]
  static constexpr int NSLOT = (NS + 64 + 15) / 16 * 16;       // u32[8] the 2^d blocks a tile spans
  static constexpr int TNODE = NSLOT + 32;                     // u16[TN] tile node -> (block << 6 | node)
  static constexpr int BYTES = (TNODE + 2 * TN + 15) / 16 * 16;
};

template <class SP>
__device__ __forceinline__ void p2g_body(const uint32_t* __restrict__ rec, const uint32_t* __restrict__ perm,
                                         uint32_t* __restrict__ cell_count,
                                         const uint32_t* __restrict__ block_start,
                                         const uint32_t* __restrict__ active_list, DevCounters* __restrict__ dc,
                                         const uint32_t* __restrict__ block_slot, float4* __restrict__ mp,
                                         const SimDev& S, int part) {
  constexpr int D = SP::D, MAT = SP::MAT, NSV = SP::NS, W = SP::W;
  constexpr int NN = D == 3 ? 27 : 9;  // stencil nodes
  // the warp tile as (m, p_z, p_x, p_y) (3D, packed accumulators): one FFMA2 + one FADD2
  // per node update instead of four scalar ops
  constexpr bool kTP = QMPM_AB_TILE_PACK && D == 3 && QMPM_AB_P2G_PACK;
  using G = Geo<D>;
  using LY = P2GLayout<SP>;
  extern __shared__ float4 smem4[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  char* wb = reinterpret_cast<char*>(smem4) + warp * LY::BYTES;
  float4* tile = reinterpret_cast<float4*>(wb + LY::TILE);
  uint32_t* ring = reinterpret_cast<uint32_t*>(wb + LY::RING) + lane * W;  // slot q at ring + q * 32 * W
  uint32_t* s_start = reinterpret_cast<uint32_t*>(wb + LY::START);
  uint32_t* s_lstart = reinterpret_cast<uint32_t*>(wb + LY::LSTART);
  uint16_t* s_seg = reinterpret_cast<uint16_t*>(wb + LY::SEG);
  uint8_t* s_ns = reinterpret_cast<uint8_t*>(wb + LY::NS);
  uint32_t* s_nslot = reinterpret_cast<uint32_t*>(wb + LY::NSLOT);
  uint16_t* s_tnode = reinterpret_cast<uint16_t*>(wb + LY::TNODE);
  build_tile_nodes<D>(s_tnode, lane);  // (for the flush)
  // part 0: every active block; 1: the blocks below the slab's top block plane; 2: the
  // top plane only (whose partial sums reach the ghost plane: launched first so the
  // exchange overlaps part 1)
  const uint32_t lo = part == 2 ? dc->n_active_below : 0u;
  const uint32_t hi = part == 1 ? dc->n_active_below : dc->n_active;
  unsigned* ctr = part == 2 ? &dc->next_p2g_top : &dc->next_p2g;
  if (part != 2 && blockIdx.x == 0 && threadIdx.x == 0) {
    // the sort has consumed the slots [0, n_slots): G2P writes the n_sorted particles
    dc->n_rec = dc->n_slots = dc->n_sorted;
    dc->n_leave = 0u;
  }
#if QMPM_AB_P2G_NEXT
  // the next block is claimed while this one runs and its id loaded before this one's
  // flush, so the dependent chain counter -> active_list -> block_start / cell_count
  // is not all exposed at each block start (at 8 ppc blocks are short)
  uint32_t nx_ab = 0, nx_claim = 0;
  if (lane == 0) nx_ab = lo + atomicAdd(ctr, 1u);
  nx_ab = __shfl_sync(FULL, nx_ab, 0);
  uint32_t nx_b = nx_ab < hi ? active_list[nx_ab] : 0u;
#endif
  for (;;) {  // blocks are taken dynamically (a work counter): no tail from uneven blocks
#if QMPM_AB_P2G_NEXT
    const uint32_t ab = nx_ab;
    if (ab >= hi) break;
    const uint32_t b = nx_b;
    if (lane == 0) nx_claim = lo + atomicAdd(ctr, 1u);  // (consumed before the flush)
#else
    uint32_t ab = 0;
    if (lane == 0) ab = lo + atomicAdd(ctr, 1u);
    ab = __shfl_sync(FULL, ab, 0);
    if (ab >= hi) break;
    const uint32_t b = active_list[ab];
#endif
    const uint32_t start = block_start[b], end = block_start[b + 1];
    int bc[3];
    block_coords<D>(b, S, bc);
    const int org[3] = {bc[0] * G::B, bc[1] * G::B, bc[2] * G::B};
    for (int t = lane; t < G::TN; t += 32) tile[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (lane < (1 << D)) {  // slots of the block and its +x/+y(/+z) neighbours (flush)
      const int nbk[3] = {bc[0] + (lane & 1), bc[1] + ((lane >> 1) & 1), D == 3 ? bc[2] + ((lane >> 2) & 1) : 0};
      uint32_t sl = 0xffffffffu;
      if (nbk[0] < S.nb[0] && nbk[1] < S.nb[1] && (D == 2 || nbk[2] < S.tab_bz1)) sl = block_slot[block_id<D>(nbk, S)];
      s_nslot[lane] = sl;
    }
    // cell starts (the scatter left them in cell_count); zeroed for the next step
    uint32_t* cc = cell_count + (size_t)b * 64;
    const uint32_t st0 = cc[lane] - start, st1 = cc[lane + 32] - start;
    cc[lane] = 0u;
    cc[lane + 32] = 0u;
    s_start[lane] = st0;
    s_start[lane + 32] = st1;
    if (lane == 0) s_start[64] = end - start;
    __syncwarp();
    // ---- 1. segment table (lane handles cells lane and lane + 32).  Cell c has
    // nf_c = min(n_c / L, kSegLev - 1) FULL segments of L particles and, if anything is
    // left, one TAIL segment.  Full segments come first, level-major (all first
    // segments in cell order, then all second segments, ...): those groups run exactly
    // L iterations.  Tails follow, sorted by length (longest first, then cell order),
    // so each tail group's lanes have similar lengths.  A cell appears at most once per
    // level and once among the tails, so only the group straddling two sections can
    // hold a cell twice (the flush serialises those lanes).
    const uint32_t nc0 = s_start[lane + 1] - st0, nc1 = s_start[lane + 33] - st1;
    const uint32_t L = min((uint32_t)kSegL, max((uint32_t)kSegLmin, (end - start + 127) / 128));
    const uint32_t nf0 = min(nc0 / L, (uint32_t)kSegLev - 1u), nf1 = min(nc1 / L, (uint32_t)kSegLev - 1u);
    const uint32_t tl0 = nc0 - nf0 * L, tl1 = nc1 - nf1 * L;  // tail lengths (0: none)
    s_ns[lane] = (uint8_t)nf0;
    s_ns[lane + 32] = (uint8_t)nf1;
    const uint32_t nlev = __reduce_max_sync(FULL, max(nf0, nf1));
    uint32_t sz = 0;  // lane l: size of level l
    for (uint32_t l = 0; l < nlev; ++l) {
      const unsigned m0 = __ballot_sync(FULL, nf0 > l), m1 = __ballot_sync(FULL, nf1 > l);
      if ((uint32_t)lane == l) sz = __popc(m0) + __popc(m1);
    }
    uint32_t inc = sz;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t t = __shfl_up_sync(FULL, inc, d);
      if (lane >= d) inc += t;
    }
    s_lstart[lane] = inc - sz;
    const uint32_t nfull = __shfl_sync(FULL, inc, 31);
    __syncwarp();
    for (uint32_t l = 0; l < nlev; ++l) {
      const unsigned m0 = __ballot_sync(FULL, nf0 > l), m1 = __ballot_sync(FULL, nf1 > l);
      const uint32_t ls = s_lstart[l];
      if (nf0 > l) s_seg[ls + __popc(m0 & lanemask_lt())] = (uint16_t)((lane << 8) | l);
      if (nf1 > l) s_seg[ls + __popc(m0) + __popc(m1 & lanemask_lt())] = (uint16_t)(((lane + 32) << 8) | l);
    }
    uint32_t nseg = nfull;
    {  // tails, by key = min(length, L) descending, ties in cell order
      const uint32_t k0 = min(tl0, L), k1 = min(tl1, L);
      uint32_t above = 0;
      // (from the longest tail present: at 8 ppc the tails are short and a loop from L
      // was 10 % of the kernel's instructions)
      for (uint32_t v = __reduce_max_sync(FULL, max(k0, k1)); v >= 1u; --v) {
        const unsigned b0 = __ballot_sync(FULL, k0 == v), b1 = __ballot_sync(FULL, k1 == v);
        if (k0 == v) s_seg[nfull + above + __popc(b0 & lanemask_lt())] = (uint16_t)((lane << 8) | nf0);
        if (k1 == v)
          s_seg[nfull + above + __popc(b0) + __popc(b1 & lanemask_lt())] = (uint16_t)(((lane + 32) << 8) | nf1);
        above += __popc(b0) + __popc(b1);
      }
      nseg += above;
    }
    __syncwarp();
    const uint32_t ngroups = (nseg + 31) / 32;
    const uint32_t* pidx = perm + start;  // the block's record indices in (cell) order
    // particle range [k, e) of segment entry i (empty past the table): level l < nf_c is
    // a full segment, l == nf_c the tail
    auto seg_range = [&](uint32_t i, uint32_t& k, uint32_t& e, int& c) {
      if (i < nseg) {
        const uint32_t v = s_seg[i];
        c = (int)(v >> 8);
        const uint32_t l = v & 255u;
        k = s_start[c] + l * L;
        e = (l == (uint32_t)s_ns[c]) ? s_start[c + 1] : k + L;
      } else {
        k = e = 0u;
        c = 0;
      }
    };
    // ---- 2. the fetch cursor walks this lane's segments of all groups ahead of the
    // compute: fidx = pidx[fk] is loaded one fetch ahead, and the next segment's first
    // index (nidx) a whole segment ahead (it starts a new cache line)
    uint32_t fk, fe, fidx = 0u, nk, ne, nidx = 0u, fg = 1;
    int fslot = 0, slot = 0;
    {
      int c_;
      seg_range(lane, fk, fe, c_);
      if (fk < fe) fidx = __ldg(pidx + fk);
      seg_range(32 + lane, nk, ne, c_);
      if (nk < ne) nidx = __ldg(pidx + nk);
    }
    auto fetch = [&]() {
      if (fk < fe) {
#if QMPM_AB_IDX_FIRST
        const uint32_t cur = fidx;  // (the next index's load goes out before this copy)
#else
        record_async<SP>(rec, fidx, ring + fslot * 32 * W);
        fslot = fslot == 2 ? 0 : fslot + 1;
#endif
        if (++fk == fe) {
          fk = nk;
          fe = ne;
          fidx = nidx;
          fg += 1;
          int c_;
          seg_range(fg * 32 + lane, nk, ne, c_);
          if (nk < ne) {
            nidx = __ldg(pidx + nk);
            // the next segment's indices (contiguous, <= L): into L1 a segment ahead, so the
            // one-ahead index loads of its particles hit (ncu: the index latency was the top
            // stall of the loop; records bypass L1 with cp.async.cg)
#if QMPM_AB_P2G_PF
            asm volatile("prefetch.global.L1 [%0];" ::"l"(pidx + nk + 1));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(pidx + ne - 1));
#if QMPM_AB_P2G_PF == 2
            // (a 48-index segment can straddle three 128-byte lines)
            if (ne - nk > 32u) asm volatile("prefetch.global.L1 [%0];" ::"l"(pidx + nk + 24));
#endif
#endif
          }
        } else {
          fidx = __ldg(pidx + fk);
#if QMPM_AB_P2G_PF == 3
          asm volatile("prefetch.global.L1 [%0];" ::"l"(pidx + fk + 8));
#elif QMPM_AB_P2G_PF == 4
          // the segment's next 128-byte index line, 8 particles before it is needed
          if ((((unsigned long long)(pidx + fk + 8)) & 127ull) < 4ull && fk + 8 < fe)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(pidx + fk + 8));
#endif
        }
#if QMPM_AB_IDX_FIRST
        record_async<SP>(rec, cur, ring + fslot * 32 * W);
        fslot = fslot == 2 ? 0 : fslot + 1;
#endif
      }
      cp_async_commit();
    };
    fetch();
    fetch();
#pragma unroll 1
    for (uint32_t g = 0; g < ngroups; ++g) {
      uint32_t k0, k1;
      int c;
      seg_range(g * 32 + lane, k0, k1, c);
      // node accumulators as fp32 pairs for the packed FFMA2/FADD2 (sm_100): axy = (p_x,
      // p_y), azm = (p_z, sum w); each lane of a pair is the same IEEE op as scalar code
      float2 axy[NN], azm[NN];
#pragma unroll
      for (int q = 0; q < NN; ++q) axy[q] = azm[q] = make_float2(0.0f, 0.0f);
#pragma unroll 1
      for (uint32_t k = k0; k < k1; ++k) {
        fetch();
        cp_async_wait<2>();
        uint32_t w[W + 1];
        read_staged<SP>(ring + slot * 32 * W, w);
        slot = slot == 2 ? 0 : slot + 1;
        // Decode what P2G needs.  Its values are never re-encoded, so a FIXED field's Eq. 3
        // scaling u * Delta is folded into its consumer's constant (one multiply by
        // Delta * p_mass (* dx) instead of two or three), and fx / the base cell come from
        // the integer x codes (exact, as in G2P's next-step key, Spec::XK)
        constexpr int CO = 2 * D + (MAT == 1 ? 1 : D * D);  // first C scalar
        float s[NSV];
#pragma unroll
        for (int i = 0; i < NSV; ++i)
          if (i >= 2 * D && i < CO) s[i] = sdec<SP>(w, i);  // F or J: the stress
        float fx[3] = {0.f, 0.f, 0.f};
        {
          bool oob = false;
          if (SP::XK > 0) {
#pragma unroll
            for (int a = 0; a < D; ++a) {
              const int u = scode<SP>(w, a);
              const int bs = (u - (1 << (SP::XK - 1))) >> SP::XK;
              oob |= (unsigned)bs > (unsigned)(S.res[a] - 3);
              fx[a] = __fmul_rn(__int2float_rn(u - (bs << SP::XK)), __int_as_float((127 - SP::XK) << 23));
            }
          } else {
#pragma unroll
            for (int a = 0; a < D; ++a) base_fx_fast(sdec<SP>(w, a), S.inv_dx, S.res[a], fx[a], oob);
          }
          if (oob) {  // rare (per lane, no warp vote in this divergent loop): reading Q14's clamp
#pragma unroll
            for (int a = 0; a < D; ++a) {
              bool o;
              base_fx(sdec<SP>(w, a), S.inv_dx, S.res[a], fx[a], o);
            }
          }
        }
        auto folds = [](int i) { return SP::kind(i) == kKindFixed && SP::offset(i) == 0.0f; };
        const float pm = S.p_mass, pmdx = S.p_mass * S.dx;
        float st[D * D];
        stress_of<D, MAT>(s, S, st);  // -dt V_p 4/dx^2 P F^T
        float Q[3] = {0.f, 0.f, 0.f}, A[3][3];
        // m_p v and m_p dx C, decoded with the scaling folded; consecutive scalars with the
        // same Delta scale as one FMUL2 pair (the FMA pipe binds; each lane the same op)
        float mv[3], mcv[D * D];
        {
          auto scaled = [&](int i, float m) {
            return folds(i) ? __int2float_rn(scode<SP>(w, i)) * (SP::delta(i) * m) : m * sdec<SP>(w, i);
          };
          auto pair_ok = [&](int i) {
            return QMPM_AB_DPACK && folds(i) && folds(i + 1) && SP::delta(i) == SP::delta(i + 1);
          };
#pragma unroll
          for (int q = 0; q < D; q += 2) {
            if (q + 1 < D && pair_ok(D + q)) {
              const float sc = SP::delta(D + q) * pm;
              const float2 r = __fmul2_rn(make_float2(__int2float_rn(scode<SP>(w, D + q)),
                                                      __int2float_rn(scode<SP>(w, D + q + 1))), make_float2(sc, sc));
              mv[q] = r.x;
              mv[q + 1] = r.y;
            } else {
              mv[q] = scaled(D + q, pm);
              if (q + 1 < D) mv[q + 1] = scaled(D + q + 1, pm);
            }
          }
#pragma unroll
          for (int q = 0; q < D * D; q += 2) {
            if (q + 1 < D * D && pair_ok(CO + q)) {
              const float sc = SP::delta(CO + q) * pmdx;
              const float2 r = __fmul2_rn(make_float2(__int2float_rn(scode<SP>(w, CO + q)),
                                                      __int2float_rn(scode<SP>(w, CO + q + 1))), make_float2(sc, sc));
              mcv[q] = r.x;
              mcv[q + 1] = r.y;
            } else {
              mcv[q] = scaled(CO + q, pmdx);
              if (q + 1 < D * D) mcv[q + 1] = scaled(CO + q + 1, pmdx);
            }
          }
        }
#pragma unroll
        for (int a = 0; a < D; ++a) {
          // m_p v
          Q[a] = mv[a];
#pragma unroll
          for (int k2 = 0; k2 < D; ++k2) {
            // A[k][a] = dx (stress + m_p C)[a][k] (the APIC/MLS affine momentum)
            const float mc = mcv[a * D + k2];
            A[k2][a] = (MAT == 1 && a != k2) ? mc : fmaf(S.dx, st[a * D + k2], mc);
            Q[a] = fmaf(-fx[k2], A[k2][a], Q[a]);
          }
        }
        float wt[3][3];
        bspline_weights<D, false>(fx, wt);
        if (D == 3 && QMPM_AB_P2G_PACK) {
          // the same sums with the weight products in FMUL2 pairs and each node's momentum
          // per unit weight built by packed adds of A's columns (row, then column, then
          // node: Q + ox A_x + oy A_y + oz A_z)
          // (TILE_PACK: the z pair is (1, M_z), so azm accumulates (sum w, p_z) -- the
          // order of the tile's (m, p_z) pair)
          const float2 a0xy = make_float2(A[0][0], A[0][1]), a0z0 = kTP ? make_float2(0.0f, A[0][2]) : make_float2(A[0][2], 0.0f);
          const float2 a1xy = make_float2(A[1][0], A[1][1]), a1z0 = kTP ? make_float2(0.0f, A[1][2]) : make_float2(A[1][2], 0.0f);
          const float2 a2xy = make_float2(A[2][0], A[2][1]), a2z0 = kTP ? make_float2(0.0f, A[2][2]) : make_float2(A[2][2], 0.0f);
          const float2 wy01 = make_float2(wt[1][0], wt[1][1]), wz01 = make_float2(wt[2][0], wt[2][1]);
          float2 rxy = make_float2(Q[0], Q[1]), rz1 = kTP ? make_float2(1.0f, Q[2]) : make_float2(Q[2], 1.0f);
#pragma unroll
          for (int ox = 0; ox < 3; ++ox) {
            const float2 wxy01 = __fmul2_rn(make_float2(wt[0][ox], wt[0][ox]), wy01);
            const float wxy2 = wt[0][ox] * wt[1][2];
            float2 mxy = rxy, mz1 = rz1;
#pragma unroll
            for (int oy = 0; oy < 3; ++oy) {
              const float wxy = oy == 0 ? wxy01.x : (oy == 1 ? wxy01.y : wxy2);
              const float2 ww01 = __fmul2_rn(make_float2(wxy, wxy), wz01);
              const float ww2 = wxy * wt[2][2];
              float2 nxy = mxy, nz1 = mz1;
#pragma unroll
              for (int oz = 0; oz < 3; ++oz) {
                const int q = (ox * 3 + oy) * 3 + oz;
                const float ww = oz == 0 ? ww01.x : (oz == 1 ? ww01.y : ww2);
                const float2 w2 = make_float2(ww, ww);
                axy[q] = __ffma2_rn(w2, nxy, axy[q]);
                azm[q] = __ffma2_rn(w2, nz1, azm[q]);  // .y: sum w + ww * 1 (exact product)
                if (oz < 2) {
                  nxy = __fadd2_rn(nxy, a2xy);
                  nz1 = __fadd2_rn(nz1, a2z0);
                }
              }
              if (oy < 2) {
                mxy = __fadd2_rn(mxy, a1xy);
                mz1 = __fadd2_rn(mz1, a1z0);
              }
            }
            if (ox < 2) {
              rxy = __fadd2_rn(rxy, a0xy);
              rz1 = __fadd2_rn(rz1, a0z0);
            }
          }
        } else if (D == 3) {
          const float2 a2xy = make_float2(A[2][0], A[2][1]), a2z0 = make_float2(A[2][2], 0.0f);
#pragma unroll
          for (int ox = 0; ox < 3; ++ox) {
#pragma unroll
            for (int oy = 0; oy < 3; ++oy) {
              const float wxy = wt[0][ox] * wt[1][oy];
              // (M_x, M_y), (M_z, 1): momentum per unit weight at node (ox, oy, 0)
              float2 mxy = make_float2(Q[0] + (float)ox * A[0][0] + (float)oy * A[1][0],
                                       Q[1] + (float)ox * A[0][1] + (float)oy * A[1][1]);
              float2 mz1 = make_float2(Q[2] + (float)ox * A[0][2] + (float)oy * A[1][2], 1.0f);
#pragma unroll
              for (int oz = 0; oz < 3; ++oz) {
                const int q = (ox * 3 + oy) * 3 + oz;
                const float ww = wxy * wt[2][oz];
                const float2 w2 = make_float2(ww, ww);
                axy[q] = __ffma2_rn(w2, mxy, axy[q]);
                azm[q] = __ffma2_rn(w2, mz1, azm[q]);  // .y: sum w + ww * 1 (exact product)
                if (oz < 2) {
                  mxy = __fadd2_rn(mxy, a2xy);
                  mz1 = __fadd2_rn(mz1, a2z0);
                }
              }
            }
          }
        } else {
          const float2 a1xy = make_float2(A[1][0], A[1][1]);
#pragma unroll
          for (int ox = 0; ox < 3; ++ox) {
            float2 mxy = make_float2(Q[0] + (float)ox * A[0][0], Q[1] + (float)ox * A[0][1]);
#pragma unroll
            for (int oy = 0; oy < 3; ++oy) {
              const int q = ox * 3 + oy;
              const float ww = wt[0][ox] * wt[1][oy];
              const float2 w2 = make_float2(ww, ww);
              axy[q] = __ffma2_rn(w2, mxy, axy[q]);
              azm[q].y += ww;
              if (oy < 2) mxy = __fadd2_rn(mxy, a1xy);
            }
          }
        }
      }
      // ---- 3. one RMW per stencil node of the segment's cell (m = p_mass * sum w)
      const bool mine = k1 > k0;
      int lc[3];
      if (D == 3) {
        lc[0] = (c >> 4) & 3;
        lc[1] = (c >> 2) & 3;
        lc[2] = c & 3;
      } else {
        lc[0] = (c >> 3) & 7;
        lc[1] = c & 7;
        lc[2] = 0;
      }
      const int base_idx = D == 3 ? (lc[0] * G::T + lc[1]) * G::T + lc[2] : lc[0] * G::T + lc[1];
      const unsigned peers = __match_any_sync(FULL, mine ? (unsigned)c : 64u + lane);
      const int occ = __popc(peers & lanemask_lt());
      const int nocc = (int)__reduce_max_sync(FULL, (unsigned)__popc(peers));
#pragma unroll 1
      for (int o = 0; o < nocc; ++o) {
#pragma unroll
        for (int q = 0; q < NN; ++q) {
          const int ox = D == 3 ? q / 9 : q / 3, oy = D == 3 ? (q / 3) % 3 : q % 3, oz = D == 3 ? q % 3 : 0;
          const int idx = base_idx + (D == 3 ? (ox * G::T + oy) * G::T + oz : ox * G::T + oy);
          if (mine && occ == o) {
            float4 t = tile[idx];
            if (kTP) {  // tile (m, p_z, p_x, p_y): (m, p_z) += (sum w, p_z) * (m_p, 1); (p_x, p_y) += axy
              const float2 mz = __ffma2_rn(azm[q], make_float2(S.p_mass, 1.0f), make_float2(t.x, t.y));
              const float2 xy = __fadd2_rn(make_float2(t.z, t.w), axy[q]);
              t = make_float4(mz.x, mz.y, xy.x, xy.y);
            } else {
              t.x = fmaf(azm[q].y, S.p_mass, t.x);
              t.y += axy[q].x;
              t.z += axy[q].y;
              t.w += azm[q].x;
            }
            tile[idx] = t;
          }
          __syncwarp();
        }
      }
    }
#if QMPM_AB_P2G_NEXT
    nx_ab = __shfl_sync(FULL, nx_claim, 0);
    nx_b = nx_ab < hi ? active_list[nx_ab] : 0u;
#endif
    cp_async_wait<0>();
    __syncwarp();
    // ---- 4. flush: one vector reduction per non-empty node
    for (int t = lane; t < G::TN; t += 32) {
      const float4 acc = tile[t];
      if (acc.x != 0.0f) {
        const uint32_t e = s_tnode[t];
        const uint32_t slot = s_nslot[e >> 6];
        if (slot != 0xffffffffu)
          atomicAdd(&mp[(size_t)slot * 64 + (e & 63u)], kTP ? make_float4(acc.x, acc.z, acc.w, acc.y) : acc);
      }
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ a5-a7: G2P + encode
// per-lane round counters packed 4 per register (byte i%4 of word i/4 counts state
// scalar i), flushed into 32-bit per-lane totals (lane i holds scalar i) before a byte can
// overflow.  Dithered: pu counts round-ups and pz on-grid values (down = all - up - on
// grid, with the idle lanes of partial chunks counted as on-grid); RNE: pu ups, pz downs.
template <class SP>
struct RoundCounters {
  static constexpr int NP = (SP::NS + 3) / 4;
  // QMPM_AB_CNT_NEG: pu's bytes start at 255 and count DOWN once per chunk in which the
  // scalar did not round up, so the fast encode adds its sign mask sb (0 up, -1 not)
  // shifted into place -- one LEA per field; no byte reaches 0 within the 255 chunks
  // between flushes, so no borrow crosses bytes
  static constexpr bool NEG = QMPM_AB_CNT_NEG == 2 ? SP::MAT == 1 : QMPM_AB_CNT_NEG != 0;
  static constexpr uint32_t PU0 = NEG ? 0xffffffffu : 0u;
  uint32_t pu[NP], pz[NP];
  uint32_t n_since;  // chunks (per lane) since the last flush, warp-uniform
  unsigned c_up, c_z;
  unsigned long long c_n;  // lane-particles counted (dithered: the "all" of down)
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      pu[k] = PU0;
      pz[k] = 0u;
    }
    n_since = 0u;
    c_up = c_z = 0u;
    c_n = 0ull;
  }
  // the fast encode's up flag of scalar i as its sign mask sb (0: rounded up, -1: not)
  __device__ __forceinline__ void count_sb(int i, int sb) {
    if (NEG)
      pu[i / 4] += (uint32_t)sb << (8 * (i % 4));
    else
      pu[i / 4] += (1u + (uint32_t)sb) << (8 * (i % 4));
  }
  // exact flags of scalar i: dithered counts on-grid (neither), RNE counts downs
  __device__ __forceinline__ void count(int i, bool up, bool down) {
    count_sb(i, up ? 0 : -1);
    if (SP::DITHER ? (!up && !down) : down) pz[i / 4] += 1u << (8 * (i % 4));
  }
  __device__ __forceinline__ void flush(int lane) {
#pragma unroll
    for (int i = 0; i < SP::NS; ++i) {
      if (SP::kind(i) == kKindRaw) continue;
      unsigned tu = __reduce_add_sync(FULL, (pu[i / 4] >> (8 * (i % 4))) & 255u);
      if (NEG) tu -= 32u * (255u - n_since);  // sum over lanes of n_since - (255 - byte)
      const unsigned tz = __reduce_add_sync(FULL, (pz[i / 4] >> (8 * (i % 4))) & 255u);
      if (lane == i) {
        c_up += tu;
        c_z += tz;
      }
    }
    c_n += 32ull * n_since;
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      pu[k] = PU0;
      pz[k] = 0u;
    }
    n_since = 0u;
  }
  // (up, down) of this lane's scalar after the last flush
  __device__ __forceinline__ unsigned long long downs() const {
    return SP::DITHER ? c_n - c_up - c_z : (unsigned long long)c_z;
  }
};

// One WARP per active block: stage the block's (B+2)^d velocity tile, then per chunk of
// 32 particles (P2G's cell order, so lanes mostly share a cell and the tile reads
// broadcast): gather, update, dither + pack in registers, store in that order, emit
// the next step's block key.  Records move with per-lane vector loads/stores; the next
// chunk's records are in flight while the current one computes.
template <class SP>
__device__ __forceinline__ void g2p_body(const uint32_t* __restrict__ rec_in, uint32_t* __restrict__ rec_out,
                                         const uint32_t* __restrict__ perm, const uint32_t* __restrict__ ids_in,
                                         uint32_t* __restrict__ ids_out, float* __restrict__ dbg,
                                         uint32_t* __restrict__ key_out, uint32_t* __restrict__ block_count,
                                         uint32_t* __restrict__ cell_count, const uint32_t* __restrict__ block_start,
                                         const uint32_t* __restrict__ active_list, DevCounters* __restrict__ dc,
                                         const uint32_t* __restrict__ block_slot, const float4* __restrict__ gv,
                                         const SimDev& S, const MigDev& M, int part) {
  constexpr int D = SP::D, MAT = SP::MAT, NSV = SP::NS, W = SP::W;
  constexpr int CO = 2 * D + (MAT == 1 ? 1 : D * D);
  using G = Geo<D>;
  using SM = Smem<SP>;
  extern __shared__ float4 smem4[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  char* wbase = reinterpret_cast<char*>(smem4) + warp * SM::G2P_WARP;
  float4* tile = reinterpret_cast<float4*>(wbase);
  uint32_t* nslot = reinterpret_cast<uint32_t*>(wbase + SM::TILE);  // [4] / [8] neighbour slots
  uint32_t* wring = reinterpret_cast<uint32_t*>(wbase + SM::STAGE);  // [2][32][W] record stage
  uint16_t* s_tnode = reinterpret_cast<uint16_t*>(wbase + SM::TNODE);
  build_tile_nodes<D>(s_tnode, lane);
  RoundCounters<SP> rc;
  rc.init();
  unsigned rmax = 0u;  // range recording (float bits of max |value|, lane i: scalar i)
  unsigned c_sat = 0, c_nf = 0, c_oob = 0;
  const float four_inv_dx = 4.0f * S.inv_dx;
  // the step's dither salt (reading Q5): steps numbered 1, 2, ... (Q20), advanced by the scan
  const uint32_t salt = step_salt(S.seed_lo, S.seed_hi, dc->gstep);
  // part 0: every active block; 1: below the top block plane; 2: the top plane (the one
  // reading the ghost plane's velocities: launched after the velocity exchange)
  const uint32_t lo = part == 2 ? dc->n_active_below : 0u;
  const uint32_t hi = part == 1 ? dc->n_active_below : dc->n_active;
  unsigned* ctr = part == 2 ? &dc->next_g2p_top : &dc->next_g2p;

  for (;;) {  // blocks are taken dynamically (a work counter): no tail from uneven blocks
    uint32_t ab = 0;
    if (lane == 0) ab = lo + atomicAdd(ctr, 1u);
    ab = __shfl_sync(FULL, ab, 0);
    if (ab >= hi) break;
    const uint32_t b = active_list[ab];
    const uint32_t start = block_start[b], end = block_start[b + 1];
    int bc[3];
    block_coords<D>(b, S, bc);
    const int org[3] = {bc[0] * G::B, bc[1] * G::B, bc[2] * G::B};
    // first chunk's records in flight while the tile is staged
    uint32_t r_next = 0, r_after = 0;  // record indices of the next chunk and the one after
    if ((uint32_t)lane < end - start) {
      r_next = perm[start + lane];
      record_async<SP>(rec_in, r_next, wring + lane * W);
    }
    if (start + 32 + lane < end) r_after = perm[start + 32 + lane];
    cp_async_commit();
    int buf = 0;
    // slots of the block and its +x/+y(/+z) neighbours, then the velocity tile
    if (lane < (1 << D)) {
      int nbk[3] = {bc[0] + (lane & 1), bc[1] + ((lane >> 1) & 1), D == 3 ? bc[2] + ((lane >> 2) & 1) : 0};
      uint32_t sl = 0xffffffffu;
      if (nbk[0] < S.nb[0] && nbk[1] < S.nb[1] && (D == 2 || nbk[2] < S.tab_bz1)) sl = block_slot[block_id<D>(nbk, S)];
      nslot[lane] = sl;
    }
    __syncwarp();
    {  // all of the lane's tile loads in flight at once, then the shared stores
      constexpr int TPL = (G::TN + 31) / 32;
      float4 v[TPL];
#pragma unroll
      for (int u = 0; u < TPL; ++u) {
        const int t = lane + 32 * u;
        v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (t < G::TN) {
          const uint32_t e = s_tnode[t];
          const uint32_t slot = nslot[e >> 6];
          if (slot != 0xffffffffu) v[u] = gv[(size_t)slot * 64 + (e & 63u)];
        }
      }
#pragma unroll
      for (int u = 0; u < TPL; ++u)
        if (lane + 32 * u < G::TN) tile[lane + 32 * u] = v[u];
    }
    __syncwarp();

    unsigned stay = 0;  // (QMPM_AB_BCNT) particles of this chunk loop staying in block b
    for (uint32_t j0 = start; j0 < end; j0 += 32) {
      const uint32_t cnt = min(32u, end - j0);
      const bool valid = (uint32_t)lane < cnt;
      const uint32_t r = r_next;
      {  // the next chunk's records go in flight while this one computes
        const uint32_t jn = j0 + 32 + lane;
#if QMPM_AB_G2P_IDX_FIRST
        const uint32_t ra = r_after;
        if (jn + 32 < end) r_after = perm[jn + 32];  // (issued before the copies, as in P2G)
        if (jn < end) {
          r_next = ra;
          record_async<SP>(rec_in, r_next, wring + ((buf ^ 1) * 32 + lane) * W);
        }
        cp_async_commit();
#else
        if (jn < end) {
          r_next = r_after;
          record_async<SP>(rec_in, r_next, wring + ((buf ^ 1) * 32 + lane) * W);
        }
        cp_async_commit();
        if (jn + 32 < end) r_after = perm[jn + 32];
#endif
      }
      cp_async_wait<1>();
      uint32_t w[W + 1];
      read_staged<SP>(wring + (buf * 32 + lane) * W, w);
      buf ^= 1;
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
      for (int a = 0; a < D; ++a) lb[a] = base_fx_fast(s[a], S.inv_dx, S.res[a], fx[a], oob_any) - org[a];
      if (__any_sync(FULL, oob_any)) {  // rare: the clamped rule of reading Q14
#pragma unroll
        for (int a = 0; a < D; ++a) {
          bool o;
          lb[a] = base_fx(s[a], S.inv_dx, S.res[a], fx[a], o) - org[a];
        }
      }
      bspline_weights<D>(fx, wt);
      // gather: v' = sum w v_i;  C' = 4/dx sum w v_i (x) (i - fx) = 4/dx (T - v' fx^T),
      // T[a][k] = sum w v_i,a o_k, reduced axis by axis (z, then y, then x)
      float Sv[3] = {0.f, 0.f, 0.f}, T[3][3] = {{0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}};
      const int base_idx = D == 3 ? (lb[0] * G::T + lb[1]) * G::T + lb[2] : lb[0] * G::T + lb[1];
      if (D == 3) {
#if QMPM_AB_ZPACK
        // packed FP32x2 (sm_100 FFMA2 / FMUL2; each lane is the IEEE op the scalar form does):
        // (v_x, v_y) of a node as one pair through every level; v_z, which would waste half
        // a pair, carries its two z-moments instead: (sum_oz w v_z, sum_oz w oz v_z) with the
        // weight pairs (w0, 0), (w1, w1), (w2, 2 w2), then (S, T_z) pairs up the y and x levels
        const float wz0 = wt[2][0], wz1 = wt[2][1], wz2 = wt[2][2], wz2x2 = 2.0f * wt[2][2];
        const float2 wzp0 = make_float2(wz0, 0.0f), wzp1 = make_float2(wz1, wz1), wzp2 = make_float2(wz2, wz2x2);
        float2 sv = make_float2(0.f, 0.f), tx = sv, tyy = sv, tzz = sv;
        float2 svz = sv;  // (sum w v_z, T[2][2])
        float tyz = 0.f, txz = 0.f;
#pragma unroll
        for (int ox = 0; ox < 3; ++ox) {
          float2 sy = make_float2(0.f, 0.f), ty = sy, tzy = sy, syz = sy;
          float tyzo = 0.f;
#pragma unroll
          for (int oy = 0; oy < 3; ++oy) {
            const int idx = base_idx + (ox * G::T + oy) * G::T;
            const float4 g0 = tile[idx], g1 = tile[idx + 1], g2 = tile[idx + 2];
            const float wy = wt[1][oy], wyo = wt[1][oy] * oy;
            const float2 a0 = make_float2(g0.x, g0.y), a1 = make_float2(g1.x, g1.y), a2 = make_float2(g2.x, g2.y);
            const float2 p1 = __fmul2_rn(make_float2(wz1, wz1), a1);
            const float2 tz = __ffma2_rn(make_float2(wz2x2, wz2x2), a2, p1);  // sum_oz w oz g
            const float2 sz = __ffma2_rn(make_float2(wz0, wz0), a0,
                                         __ffma2_rn(make_float2(wz2, wz2), a2, p1));  // sum_oz w g
            sy = __ffma2_rn(make_float2(wy, wy), sz, sy);
            tzy = __ffma2_rn(make_float2(wy, wy), tz, tzy);
            if (oy) ty = __ffma2_rn(make_float2(wyo, wyo), sz, ty);
            const float2 z = __ffma2_rn(wzp2, make_float2(g2.z, g2.z),
                                        __ffma2_rn(wzp1, make_float2(g1.z, g1.z),
                                                   __fmul2_rn(wzp0, make_float2(g0.z, g0.z))));
            syz = __ffma2_rn(make_float2(wy, wy), z, syz);
            if (oy) tyzo = fmaf(wyo, z.x, tyzo);
          }
          const float wx = wt[0][ox], wxo = wt[0][ox] * ox;
          sv = __ffma2_rn(make_float2(wx, wx), sy, sv);
          tyy = __ffma2_rn(make_float2(wx, wx), ty, tyy);
          tzz = __ffma2_rn(make_float2(wx, wx), tzy, tzz);
          if (ox) tx = __ffma2_rn(make_float2(wxo, wxo), sy, tx);
          svz = __ffma2_rn(make_float2(wx, wx), syz, svz);
          tyz = fmaf(wx, tyzo, tyz);
          if (ox) txz = fmaf(wxo, syz.x, txz);
        }
        Sv[0] = sv.x;
        Sv[1] = sv.y;
        Sv[2] = svz.x;
        T[0][0] = tx.x;
        T[1][0] = tx.y;
        T[2][0] = txz;
        T[0][1] = tyy.x;
        T[1][1] = tyy.y;
        T[2][1] = tyz;
        T[0][2] = tzz.x;
        T[1][2] = tzz.y;
        T[2][2] = svz.y;
#else
        // packed FP32x2 (sm_100 FFMA2 / FMUL2): pair 0 = (v_x, v_y), pair 1 = (v_z, 0) of a
        // node; each lane is the same IEEE op the scalar form does
        const float wz0 = wt[2][0], wz1 = wt[2][1], wz2 = wt[2][2], wz2x2 = 2.0f * wt[2][2];
        float2 sv[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        float2 tx[2] = {sv[0], sv[0]}, tyy[2] = {sv[0], sv[0]}, tzz[2] = {sv[0], sv[0]};
#pragma unroll
        for (int ox = 0; ox < 3; ++ox) {
          float2 sy[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)}, ty[2] = {sy[0], sy[0]},
                 tzy[2] = {sy[0], sy[0]};
#pragma unroll
          for (int oy = 0; oy < 3; ++oy) {
            const int idx = base_idx + (ox * G::T + oy) * G::T;
            const float4 g0 = tile[idx], g1 = tile[idx + 1], g2 = tile[idx + 2];
            const float2 ga[3][2] = {{make_float2(g0.x, g0.y), make_float2(g0.z, g0.w)},
                                     {make_float2(g1.x, g1.y), make_float2(g1.z, g1.w)},
                                     {make_float2(g2.x, g2.y), make_float2(g2.z, g2.w)}};
            const float wy = wt[1][oy], wyo = wt[1][oy] * oy;
#pragma unroll
            for (int pp = 0; pp < 2; ++pp) {
              const float2 p1 = __fmul2_rn(make_float2(wz1, wz1), ga[1][pp]);
              const float2 tz = __ffma2_rn(make_float2(wz2x2, wz2x2), ga[2][pp], p1);  // sum_oz w oz g
              const float2 sz = __ffma2_rn(make_float2(wz0, wz0), ga[0][pp],
                                           __ffma2_rn(make_float2(wz2, wz2), ga[2][pp], p1));  // sum_oz w g
              sy[pp] = __ffma2_rn(make_float2(wy, wy), sz, sy[pp]);
              tzy[pp] = __ffma2_rn(make_float2(wy, wy), tz, tzy[pp]);
              if (oy) ty[pp] = __ffma2_rn(make_float2(wyo, wyo), sz, ty[pp]);
            }
          }
          const float wx = wt[0][ox], wxo = wt[0][ox] * ox;
#pragma unroll
          for (int pp = 0; pp < 2; ++pp) {
            sv[pp] = __ffma2_rn(make_float2(wx, wx), sy[pp], sv[pp]);
            tyy[pp] = __ffma2_rn(make_float2(wx, wx), ty[pp], tyy[pp]);
            tzz[pp] = __ffma2_rn(make_float2(wx, wx), tzy[pp], tzz[pp]);
            if (ox) tx[pp] = __ffma2_rn(make_float2(wxo, wxo), sy[pp], tx[pp]);
          }
        }
        Sv[0] = sv[0].x;
        Sv[1] = sv[0].y;
        Sv[2] = sv[1].x;
        T[0][0] = tx[0].x;
        T[1][0] = tx[0].y;
        T[2][0] = tx[1].x;
        T[0][1] = tyy[0].x;
        T[1][1] = tyy[0].y;
        T[2][1] = tyy[1].x;
        T[0][2] = tzz[0].x;
        T[1][2] = tzz[0].y;
        T[2][2] = tzz[1].x;
#endif
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
      // dithered encode into registers (Eq. 11; reading Q5, Q6).  Idle lanes of a partial
      // chunk encode their fields' offsets (t = 0: on the grid, counted neither up nor
      // down), so the round counters need no per-field lane predicate.
      if (cnt < 32u && !valid) {
#pragma unroll
        for (int i = 0; i < NSV; ++i) o[i] = SP::kind(i) == kKindFixed ? SP::offset(i) : 0.0f;  // (shared: 0)
      }
      uint32_t ow[W + 1];
#pragma unroll
      for (int q = 0; q <= W; ++q) ow[q] = 0u;
      bool flag = false;
      int xc[3] = {0, 0, 0};  // x codes (next step's key)
      uint32_t pu_save[RoundCounters<SP>::NP], pz_save[RoundCounters<SP>::NP];
      if (SP::COUNTERS) {
#pragma unroll
        for (int k = 0; k < RoundCounters<SP>::NP; ++k) {
          pu_save[k] = rc.pu[k];
          pz_save[k] = rc.pz[k];
        }
      }
#pragma unroll
      for (int i = 0; i < NSV; ++i) {
        const int role = pair_role<SP>(i);
        if (role == 2) continue;
        if (role == 1) {  // packed pair (i, i + 1), one pair hash when they share one (Q5 rev. 3)
          int ui, uj, sbi, sbj;
          bool zi, zj;
          senc_pair_fast<SP>(i, i + 1, o[i], o[i + 1], dither_s(h, SP::idx(i)), dither_s(h, SP::idx(i + 1)), ui, uj,
                             sbi, sbj, flag, zi, zj);
          sput_code<SP>(ow, i, ui);
          sput_code<SP>(ow, i + 1, uj);
          if (i < D) xc[i] = ui;
          if (i + 1 < D) xc[i + 1] = uj;
          if (SP::COUNTERS) {
            // + 1 in the bytes of i and i + 1 (one counter register: i is even) that rounded
            // up (sb == 0): two LOP3 and an add on the integer pipe (the FMA pipe binds)
            if (QMPM_AB_CNT_LOP3 && !RoundCounters<SP>::NEG) {
              const uint32_t ci = 0xffu << (8 * (i % 4));
              const uint32_t bij = (1u << (8 * (i % 4))) | (1u << (8 * ((i + 1) % 4)));
              rc.pu[i / 4] += ((~(uint32_t)sbi & ci) | (~(uint32_t)sbj & ~ci)) & bij;
            } else {
              rc.count_sb(i, sbi);
              rc.count_sb(i + 1, sbj);
            }
            if (zi) rc.pz[i / 4] += 1u << (8 * (i % 4));
            if (zj) rc.pz[(i + 1) / 4] += 1u << (8 * ((i + 1) % 4));
          }
          continue;
        }
        if (fast_ok<SP>(i)) {
          int sb;
          bool z;
          const int u = senc1_fast<SP>(i, o[i], dither_s(h, SP::idx(i)), sb, flag, z);
          sput_code<SP>(ow, i, u);
          if (i < D) xc[i] = u;
          if (SP::COUNTERS) {
            rc.count_sb(i, sb);
            if (z) rc.pz[i / 4] += 1u << (8 * (i % 4));
          }
          continue;
        }
        if (SP::kind(i) == kKindShared) {  // reading Q4: the whole group at its leader
          if (SP::glead(i) == i) {
            EncFlags gfl[NSV];
            senc_group<SP>(i, o, h, ow, gfl);
#pragma unroll
            for (int j = 0; j < NSV; ++j) {
              if (SP::kind(j) != kKindShared || SP::glead(j) != i) continue;
              flag |= gfl[j].sat || gfl[j].nonfinite;
              if (SP::COUNTERS) rc.count(j, gfl[j].up, gfl[j].down);
            }
          }
          continue;
        }
        const float omr = (SP::DITHER && SP::kind(i) == kKindFixed) ? dither_omr(h, SP::idx(i)) : 1.0f;
        bool up, nz;
        sput<SP>(ow, i, senc_fast<SP>(i, o[i], omr, up, nz, flag));
        if (i < D && SP::kind(i) == kKindFixed) xc[i] = scode<SP>(ow, i);
        if (SP::COUNTERS && SP::kind(i) == kKindFixed) rc.count(i, up, SP::DITHER ? (nz && !up) : nz);
      }
      if (__any_sync(FULL, valid && flag)) {  // rare: exact re-encode with saturation / non-finite
#pragma unroll
        for (int q = 0; q <= W; ++q) ow[q] = 0u;
        EncFlags fl[NSV];
#pragma unroll
        for (int i = 0; i < NSV; ++i) {
          if (SP::kind(i) == kKindShared) {
            if (SP::glead(i) == i) senc_group<SP>(i, o, h, ow, fl);
            continue;
          }
          const float omr = (SP::DITHER && SP::kind(i) == kKindFixed) ? dither_omr(h, SP::idx(i)) : 1.0f;
          sput<SP>(ow, i, senc<SP>(i, o[i], omr, fl[i]));
        }
        if (SP::COUNTERS) {  // the exact rule's counts replace the fast pass's
#pragma unroll
          for (int k = 0; k < RoundCounters<SP>::NP; ++k) {
            rc.pu[k] = pu_save[k];
            rc.pz[k] = pz_save[k];
          }
#pragma unroll
          for (int i = 0; i < NSV; ++i)
            if (SP::kind(i) != kKindRaw) rc.count(i, fl[i].up, fl[i].down);
        }
#pragma unroll
        for (int i = 0; i < D; ++i)
          if (SP::kind(i) == kKindFixed) xc[i] = scode<SP>(ow, i);
#pragma unroll
        for (int i = 0; i < NSV; ++i) {
          const unsigned bs = __ballot_sync(FULL, valid && fl[i].sat);
          const unsigned bn = __ballot_sync(FULL, valid && fl[i].nonfinite);
          if (lane == i) c_sat += __popc(bs);
          if (lane == 0) c_nf += __popc(bn);
        }
      }
      if (SP::COUNTERS && ++rc.n_since == 255u) rc.flush(lane);
      if (SP::RANGES) {  // Alg. 1 line 9: max |value| of s_{t+1} per state scalar (lane i keeps scalar i)
#pragma unroll
        for (int i = 0; i < NSV; ++i) {
          const unsigned m = __reduce_max_sync(FULL, valid ? (__float_as_uint(o[i]) & 0x7fffffffu) : 0u);
          if (lane == i) rmax = max(rmax, m);
        }
      }
      {
        const unsigned bo = __ballot_sync(FULL, valid && oob_any);
        if (lane == 0) c_oob += __popc(bo);
      }
      // next step's sort key: from the integer x codes when x = u Delta and x / dx are exact
      // powers-of-two scalings (Spec::XK = log2(dx / Delta) > 0: base = floor(u 2^-XK - 1/2),
      // bit-identical to floor(fl(fl(u Delta) / dx) - 1/2)), else from the re-decoded x
      uint32_t nkey;
      bool leave = false;
      {
        int bsv[3] = {0, 0, 0};
        bool koob = false;
        if (SP::XK > 0) {
#pragma unroll
          for (int a = 0; a < D; ++a) {
            bsv[a] = (xc[a] - (1 << (SP::XK - 1))) >> SP::XK;
            koob |= (unsigned)bsv[a] > (unsigned)(S.res[a] - 3);
          }
        } else {
          float xq[3];
#pragma unroll
          for (int a = 0; a < D; ++a) {
            xq[a] = sdec<SP>(ow, a);
            float fq;
            bsv[a] = base_fx_fast(xq[a], S.inv_dx, S.res[a], fq, koob);
          }
        }
        if (__any_sync(FULL, valid && koob)) {  // rare: clamped base (Q14)
          float xq[3];
#pragma unroll
          for (int a = 0; a < D; ++a) {
            xq[a] = sdec<SP>(ow, a);
            float fq;
            bool o;
            bsv[a] = base_fx(xq[a], S.inv_dx, S.res[a], fq, o);
          }
        }
        // slab ranks: a particle whose new base block plane is a neighbour's leaves
        int side = 0;
        if (SP::SLAB && D == 3) side = slab_side(bsv[2] >> G::LB, S);  // (compiled out on one GPU)
        leave = valid && side != 0;
        nkey = side == 0 ? key_from_base<D>(bsv, S) : kDeadKey;
        if (SP::SLAB && __any_sync(FULL, leave) && leave)
          mig_push<W>(M, dc, side, ow, ids_out != nullptr ? ids_in[r] : 0u, j,
                   dbg != nullptr ? dbg + (size_t)j * NSV : nullptr);
      }
      if (valid) key_out[j] = nkey;
      {  // next step's histograms, one atomic per distinct key of the warp
        const bool cnt_it = valid && !leave;
#if QMPM_AB_BCNT
        // most particles stay in their block: those are summed over the block's chunks
        // (one atomic per block below), the others count themselves
        const bool same = cnt_it && (nkey >> 6) == b;
        stay += (unsigned)__popc(__ballot_sync(FULL, same));
        if (cnt_it && !same) atomicAdd(&block_count[nkey >> 6], 1u);
#else
        const uint32_t nk = cnt_it ? (nkey >> 6) : 0xffffffffu;
        const unsigned kp = __match_any_sync(FULL, nk);
        if (cnt_it && lane == __ffs(kp) - 1) atomicAdd(&block_count[nk], (unsigned)__popc(kp));
#endif
        const unsigned cp = __match_any_sync(FULL, cnt_it ? nkey : kDeadKey);
        if (cnt_it && lane == __ffs(cp) - 1) atomicAdd(&cell_count[nkey], (unsigned)__popc(cp));
      }
      if (valid) {
        if (ids_out != nullptr) ids_out[j] = ids_in[r];
        uint32_t* op = rec_out + (size_t)j * W;
        if (W % 4 == 0) {
#pragma unroll
          for (int q = 0; q < W / 4; ++q)
            reinterpret_cast<uint4*>(op)[q] = make_uint4(ow[4 * q], ow[4 * q + 1], ow[4 * q + 2], ow[4 * q + 3]);
        } else if (W % 2 == 0) {
#pragma unroll
          for (int q = 0; q < W / 2; ++q) reinterpret_cast<uint2*>(op)[q] = make_uint2(ow[2 * q], ow[2 * q + 1]);
        } else {
#pragma unroll
          for (int q = 0; q < W; ++q) op[q] = ow[q];
        }
      }
    }
    if (QMPM_AB_BCNT && lane == 0 && stay != 0u) atomicAdd(&block_count[b], stay);
    __syncwarp();
  }
  if (SP::COUNTERS) rc.flush(lane);
  // flush this thread's counters (lane i holds scalar i's counts)
  if (lane < NSV) {
    int fi = 0;
    bool raw = false;
#pragma unroll
    for (int i = 0; i < NSV; ++i)
      if (lane == i) {
        fi = SP::idx(i);
        raw = SP::kind(i) == kKindRaw;
      }
    const unsigned long long c_dn = (SP::COUNTERS && !raw) ? rc.downs() : 0ull;
    if (rc.c_up) atomicAdd(&dc->up[fi], (unsigned long long)rc.c_up);
    if (c_dn) atomicAdd(&dc->down[fi], c_dn);
    if (c_sat) atomicAdd(&dc->sat[fi], (unsigned long long)c_sat);
  }
  if (c_nf) atomicAdd(&dc->nonfinite, (unsigned long long)c_nf);
  if (c_oob) atomicAdd(&dc->oob, (unsigned long long)c_oob);
  if (SP::RANGES && lane < NSV && rmax) atomicMax(&dc->range_bits[lane], rmax);
}

}  // namespace qmpm

// ------------------------------------------------------------------ entry points
// per-warp shared-memory bytes of P2G and G2P, read by the host after loading the module
extern "C" __device__ const unsigned qmpm_smem_per_warp[2] = {(unsigned)qmpm::P2GLayout<Spec>::BYTES,
                                                             (unsigned)qmpm::Smem<Spec>::G2P_WARP};
extern "C" __global__ void __launch_bounds__(256) qmpm_bin_count(const uint32_t* rec, const uint32_t* ids, uint32_t first,
                                                                 uint32_t n, qmpm::SimDev S, uint32_t* key,
                                                                 uint32_t* block_count, uint32_t* cell_count,
                                                                 int do_count, qmpm::MigDev M, qmpm::DevCounters* dc) {
  qmpm::bin_count_body<Spec>(rec, ids, first, n, S, key, block_count, cell_count, do_count, M, dc);
}

extern "C" __global__ void __launch_bounds__(256) qmpm_append(uint32_t* rec, uint32_t* ids, float* dbg, uint64_t cap,
                                                              qmpm::SimDev S, uint32_t* key, uint32_t* block_count,
                                                              uint32_t* cell_count, qmpm::MigDev M,
                                                              qmpm::DevCounters* dc) {
  qmpm::append_body<Spec>(rec, ids, dbg, cap, S, key, block_count, cell_count, M, dc);
}

extern "C" __global__ void __launch_bounds__(Spec::P2G_WARPS * 32, Spec::P2G_MINB)
    qmpm_p2g(const uint32_t* rec, const uint32_t* perm, uint32_t* cell_count, const uint32_t* block_start,
             const uint32_t* active_list, qmpm::DevCounters* dc, const uint32_t* block_slot, float4* mp,
             qmpm::SimDev S, int part) {
  qmpm::p2g_body<Spec>(rec, perm, cell_count, block_start, active_list, dc, block_slot, mp, S, part);
}

extern "C" __global__ void __launch_bounds__(Spec::G2P_WARPS * 32, Spec::G2P_MINB)
    qmpm_g2p(const uint32_t* rec_in, uint32_t* rec_out, const uint32_t* perm, const uint32_t* ids_in,
             uint32_t* ids_out, float* dbg, uint32_t* key_out, uint32_t* block_count, uint32_t* cell_count,
             const uint32_t* block_start, const uint32_t* active_list, qmpm::DevCounters* dc,
             const uint32_t* block_slot, const float4* gv, qmpm::SimDev S, qmpm::MigDev M, int part) {
  qmpm::g2p_body<Spec>(rec_in, rec_out, perm, ids_in, ids_out, dbg, key_out, block_count, cell_count, block_start,
                       active_list, dc, block_slot, gv, S, M, part);
}
