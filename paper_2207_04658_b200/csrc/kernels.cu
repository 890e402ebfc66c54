// kernels.cu -- sm_100a kernels of one quantized MLS-MPM step.
//
//   k_bin_count    a1  block key of every record + per-block histogram (first step only;
//                      afterwards G2P computes next step's keys from the re-encoded x)
//   k_scan_*       a1  exclusive scan over the dense block table: particle offsets,
//                      active-block list, touched-block (pool slot) assignment
//   k_bin_scatter  a1  counting-sort scatter: perm[sorted slot] = record index
//   k_p2g          a2+a3  decode records (warp-cooperative coalesced staging), stress,
//                      scatter into per-warp conflict-free shared-memory tiles,
//                      flush with red.global.add.v4.f32
//   k_grid_update  a4  v = p/m + dt g, separating walls; clears (m, p) for next step
//   k_g2p          a2+a5+a6+a7  gather from a shared-memory tile, update x, v, C, F|J,
//                      dithered encode + pack into thread-owned rows (no RMW on
//                      global words), coalesced store in sorted order, next
//                      step's block key + histogram
//
// The MLS-MPM arithmetic follows Hu et al. 2018 (cited P:561) as restated in
// DESIGN.md §2; codec arithmetic is in qmpm_device.cuh.
#include <cuda_runtime.h>

#include "qmpm_device.cuh"
#include "qmpm_launch.h"

namespace qmpm {

constexpr unsigned FULL = 0xffffffffu;

template <int D>
struct Geo;
template <>
struct Geo<3> {
  static constexpr int B = 4;     // cells per block side
  static constexpr int LB = 2;    // log2(B)
  static constexpr int T = 6;     // tile side (nodes): B + 2
  static constexpr int TN = 216;  // tile nodes
  static constexpr int NN = 27;   // stencil nodes
};
template <>
struct Geo<2> {
  static constexpr int B = 8;
  static constexpr int LB = 3;
  static constexpr int T = 10;
  static constexpr int TN = 100;
  static constexpr int NN = 9;
};

template <int D, int MAT>
struct NS {
  static constexpr int value = 2 * D + (MAT == 1 ? 1 : D * D) + D * D;
};

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <int D>
__device__ __forceinline__ void block_coords(uint32_t b, const SimDev& S, int bc[3]) {
  if (D == 3) {
    bc[2] = (int)(b % (uint32_t)S.nb[2]);
    const uint32_t r = b / (uint32_t)S.nb[2];
    bc[1] = (int)(r % (uint32_t)S.nb[1]);
    bc[0] = (int)(r / (uint32_t)S.nb[1]);
  } else {
    bc[1] = (int)(b % (uint32_t)S.nb[1]);
    bc[0] = (int)(b / (uint32_t)S.nb[1]);
    bc[2] = 0;
  }
}

template <int D>
__device__ __forceinline__ uint32_t block_id(const int c[3], const SimDev& S) {
  if (D == 3) return ((uint32_t)c[0] * (uint32_t)S.nb[1] + (uint32_t)c[1]) * (uint32_t)S.nb[2] + (uint32_t)c[2];
  return (uint32_t)c[0] * (uint32_t)S.nb[1] + (uint32_t)c[1];
}

// node-in-block linear index (x-major) and block-local node coordinates
template <int D>
__device__ __forceinline__ uint32_t local_node(const int l[3]) {
  if (D == 3) return (uint32_t)((l[0] * 4 + l[1]) * 4 + l[2]);
  return (uint32_t)(l[0] * 8 + l[1]);
}

// block key of a particle from its (decoded) position
template <int D>
__device__ __forceinline__ uint32_t key_of(const float* x, const SimDev& S) {
  int c[3] = {0, 0, 0};
#pragma unroll
  for (int a = 0; a < D; ++a) {
    float fx;
    bool o;
    c[a] = base_fx(x[a], S.inv_dx, S.res[a], fx, o) >> Geo<D>::LB;
  }
  return block_id<D>(c, S);
}

// ============================================================== a1: binning
template <int D>
__global__ void k_bin_count(const uint32_t* __restrict__ rec, uint32_t n, LayoutDev L, SimDev S,
                            uint32_t* __restrict__ key, uint32_t* __restrict__ block_count) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = i < n;
  uint32_t k = 0xffffffffu;
  if (valid) {
    const uint32_t* row = rec + (size_t)i * L.W;
    float x[3];
#pragma unroll
    for (int a = 0; a < D; ++a) x[a] = decode_field(row, L.s[a]);
    k = key_of<D>(x, S);
    key[i] = k;
  }
  const unsigned peers = __match_any_sync(FULL, k);
  if (valid && (threadIdx.x & 31) == (unsigned)(__ffs(peers) - 1)) atomicAdd(&block_count[k], __popc(peers));
}

// per-block (count, active, touched); touched = any of the blocks b - {0,1}^D holds particles
template <int D>
__device__ __forceinline__ void block_flags(uint32_t b, const uint32_t* __restrict__ count,
                                            const SimDev& S, uint32_t& c, uint32_t& act,
                                            uint32_t& touched) {
  if (b >= S.nblocks) {
    c = act = touched = 0;
    return;
  }
  c = count[b];
  act = c > 0;
  touched = act;
  int bc[3];
  block_coords<D>(b, S, bc);
#pragma unroll
  for (int dl = 1; dl < (1 << D); ++dl) {
    int nc[3] = {bc[0] - (dl & 1), bc[1] - ((dl >> 1) & 1), D == 3 ? bc[2] - ((dl >> 2) & 1) : 0};
    if (nc[0] < 0 || nc[1] < 0 || nc[2] < 0) continue;
    touched |= count[block_id<D>(nc, S)] > 0;
  }
}

constexpr int kScanThreads = 256;
constexpr int kScanPer = kScanTile / kScanThreads;  // 4

// block-wide exclusive scan of a uint3 (returns exclusive prefix, writes total)
__device__ __forceinline__ uint3 block_exclusive_scan3(uint3 v, uint3& total) {
  __shared__ uint3 s_warp[32];
  __shared__ uint3 s_total;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint3 inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t a = __shfl_up_sync(FULL, inc.x, o), b = __shfl_up_sync(FULL, inc.y, o),
                   c = __shfl_up_sync(FULL, inc.z, o);
    if (lane >= o) {
      inc.x += a;
      inc.y += b;
      inc.z += c;
    }
  }
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  if (warp == 0) {
    uint3 w = lane < nw ? s_warp[lane] : make_uint3(0, 0, 0);
    uint3 wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t a = __shfl_up_sync(FULL, wi.x, o), b = __shfl_up_sync(FULL, wi.y, o),
                     c = __shfl_up_sync(FULL, wi.z, o);
      if (lane >= o) {
        wi.x += a;
        wi.y += b;
        wi.z += c;
      }
    }
    if (lane < nw) s_warp[lane] = make_uint3(wi.x - w.x, wi.y - w.y, wi.z - w.z);
    if (lane == nw - 1) s_total = wi;
  }
  __syncthreads();
  const uint3 wo = s_warp[warp];
  total = s_total;
  __syncthreads();
  return make_uint3(wo.x + inc.x - v.x, wo.y + inc.y - v.y, wo.z + inc.z - v.z);
}

template <int D>
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const uint32_t* __restrict__ count, SimDev S,
                                                              uint4* __restrict__ tile_sums) {
  const uint32_t b0 = blockIdx.x * kScanTile + threadIdx.x * kScanPer;
  uint3 v = make_uint3(0, 0, 0);
#pragma unroll
  for (int q = 0; q < kScanPer; ++q) {
    uint32_t c, a, t;
    block_flags<D>(b0 + q, count, S, c, a, t);
    v.x += c;
    v.y += a;
    v.z += t;
  }
  uint3 total;
  block_exclusive_scan3(v, total);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = make_uint4(total.x, total.y, total.z, 0);
}

// one CTA: exclusive scan over tiles, totals -> counters, blockStart[nblocks] = n
__global__ void __launch_bounds__(1024) k_scan_tiles(const uint4* __restrict__ tile_sums, uint32_t ntiles,
                                                     uint4* __restrict__ tile_off, DevCounters* dc,
                                                     uint32_t* __restrict__ block_start, uint32_t nblocks,
                                                     uint32_t pool) {
  const uint32_t per = (ntiles + blockDim.x - 1) / blockDim.x;
  const uint32_t t0 = threadIdx.x * per;
  uint3 v = make_uint3(0, 0, 0);
  for (uint32_t t = t0; t < t0 + per && t < ntiles; ++t) {
    const uint4 s = tile_sums[t];
    v.x += s.x;
    v.y += s.y;
    v.z += s.z;
  }
  uint3 total;
  uint3 ex = block_exclusive_scan3(v, total);
  for (uint32_t t = t0; t < t0 + per && t < ntiles; ++t) {
    tile_off[t] = make_uint4(ex.x, ex.y, ex.z, 0);
    const uint4 s = tile_sums[t];
    ex.x += s.x;
    ex.y += s.y;
    ex.z += s.z;
  }
  if (threadIdx.x == 0) {
    dc->n_active = total.y;
    dc->n_touched = total.z;
    dc->n_touched_eff = total.z < pool ? total.z : pool;
    if (total.z > pool) dc->overflow += 1ull;
    block_start[nblocks] = total.x;
  }
}

template <int D>
__global__ void __launch_bounds__(kScanThreads) k_scan_apply(const uint32_t* __restrict__ count, SimDev S,
                                                             const uint4* __restrict__ tile_off,
                                                             uint32_t* __restrict__ block_start,
                                                             uint32_t* __restrict__ block_slot,
                                                             uint32_t* __restrict__ active_list,
                                                             uint32_t* __restrict__ touched_list,
                                                             uint32_t pool) {
  const uint32_t b0 = blockIdx.x * kScanTile + threadIdx.x * kScanPer;
  uint32_t c[kScanPer], a[kScanPer], t[kScanPer];
  uint3 v = make_uint3(0, 0, 0);
#pragma unroll
  for (int q = 0; q < kScanPer; ++q) {
    block_flags<D>(b0 + q, count, S, c[q], a[q], t[q]);
    v.x += c[q];
    v.y += a[q];
    v.z += t[q];
  }
  uint3 total;
  uint3 ex = block_exclusive_scan3(v, total);
  const uint4 to = tile_off[blockIdx.x];
  ex.x += to.x;
  ex.y += to.y;
  ex.z += to.z;
#pragma unroll
  for (int q = 0; q < kScanPer; ++q) {
    const uint32_t b = b0 + q;
    if (b < S.nblocks) {
      block_start[b] = ex.x;
      if (a[q]) active_list[ex.y] = b;
      uint32_t slot = 0xffffffffu;
      if (t[q] && ex.z < pool) {
        slot = ex.z;
        touched_list[slot] = b;
      }
      block_slot[b] = slot;
    }
    ex.x += c[q];
    ex.y += a[q];
    ex.z += t[q];
  }
}

__global__ void k_bin_scatter(const uint32_t* __restrict__ key, uint32_t n,
                              const uint32_t* __restrict__ block_start, uint32_t* __restrict__ block_count,
                              uint32_t* __restrict__ perm) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = i < n;
  const uint32_t k = valid ? key[i] : 0xffffffffu;
  const unsigned peers = __match_any_sync(FULL, k);
  const int leader = __ffs(peers) - 1;
  const int rank = __popc(peers & lanemask_lt());
  uint32_t old = 0;
  if (valid && (int)(threadIdx.x & 31) == leader) old = atomicSub(&block_count[k], (uint32_t)__popc(peers));
  old = __shfl_sync(FULL, old, leader);
  if (valid) perm[block_start[k] + old - 1 - rank] = i;
}

// ============================================================== staging
// Warp-cooperative load of the warp's `cnt` records (record index r_lane held by
// lane l) into rows wst[l * SW + w]; coalesced when the records are contiguous.
__device__ __forceinline__ void stage_load(const uint32_t* __restrict__ rec, uint32_t r_lane, uint32_t cnt,
                                           uint32_t W, uint32_t SW, uint32_t* wst, int lane) {
  const uint32_t total = cnt * W;
  uint32_t l = (uint32_t)lane / W, w = (uint32_t)lane % W;
  const uint32_t dl = 32u / W, dw = 32u % W;
  for (uint32_t q0 = 0; q0 < total; q0 += 32) {
    const uint32_t r = __shfl_sync(FULL, r_lane, (int)(l & 31u));
    if (q0 + lane < total) wst[l * SW + w] = __ldg(rec + (size_t)r * W + w);
    l += dl;
    w += dw;
    if (w >= W) {
      w -= W;
      l += 1;
    }
  }
  if ((uint32_t)lane < cnt) wst[lane * SW + W] = 0u;  // spare word for straddle reads
}

__device__ __forceinline__ void stage_store(uint32_t* __restrict__ out, uint32_t cnt, uint32_t W, uint32_t SW,
                                            const uint32_t* wst, int lane) {
  const uint32_t total = cnt * W;
  uint32_t l = (uint32_t)lane / W, w = (uint32_t)lane % W;
  const uint32_t dl = 32u / W, dw = 32u % W;
  for (uint32_t q = lane; q < total; q += 32) {
    out[q] = wst[l * SW + w];
    l += dl;
    w += dw;
    if (w >= W) {
      w -= W;
      l += 1;
    }
  }
}

// a harmless particle for the idle lanes of a partial warp (never stored)
template <int D, int MAT>
__device__ __forceinline__ void benign_state(float* s, const int org[3], float dx) {
  constexpr int NSV = NS<D, MAT>::value;
#pragma unroll
  for (int i = 0; i < NSV; ++i) s[i] = 0.0f;
#pragma unroll
  for (int a = 0; a < D; ++a) s[a] = (org[a] + 1.0f) * dx;
  if (MAT == 1) {
    s[2 * D] = 1.0f;
  } else {
#pragma unroll
    for (int a = 0; a < D; ++a) s[2 * D + a * D + a] = 1.0f;
  }
}

// ============================================================== stress
template <int D, int MAT>
__device__ __forceinline__ void affine_of(const float* s, const SimDev& S, float aff[D * D]) {
  constexpr int CO = 2 * D + (MAT == 1 ? 1 : D * D);  // offset of C
  if (MAT == 1) {
    const float J = s[2 * D];
    const float p = S.stress_scale * S.E * (J - 1.0f);
#pragma unroll
    for (int i = 0; i < D * D; ++i) aff[i] = S.p_mass * s[CO + i];
#pragma unroll
    for (int a = 0; a < D; ++a) aff[a * D + a] += p;
  } else {
    const float* F = s + 2 * D;
    float R[D * D];
    float J;
    if (D == 3) {
      polar3(F, R);
      J = F[0] * (F[4] * F[8] - F[5] * F[7]) - F[1] * (F[3] * F[8] - F[5] * F[6]) +
          F[2] * (F[3] * F[7] - F[4] * F[6]);
    } else {
      polar2(F, R);
      J = F[0] * F[3] - F[1] * F[2];
    }
    const float two_mu = 2.0f * S.mu * S.stress_scale;
    const float diag = S.lambda * (J - 1.0f) * J * S.stress_scale;
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) {
        float acc = 0.0f;
#pragma unroll
        for (int k = 0; k < D; ++k) acc += (F[a * D + k] - R[a * D + k]) * F[b * D + k];
        aff[a * D + b] = two_mu * acc + S.p_mass * s[CO + a * D + b] + (a == b ? diag : 0.0f);
      }
  }
}

// ============================================================== a3: P2G
template <int D, int MAT, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_p2g(const uint32_t* __restrict__ rec,
                                                    const uint32_t* __restrict__ perm,
                                                    const uint32_t* __restrict__ block_start,
                                                    const uint32_t* __restrict__ active_list,
                                                    const DevCounters* __restrict__ dc,
                                                    const uint32_t* __restrict__ block_slot,
                                                    float4* __restrict__ mp, LayoutDev L, SimDev S) {
  using G = Geo<D>;
  constexpr int NSV = NS<D, MAT>::value;
  extern __shared__ float4 smem4[];
  float4* tiles = smem4;                                        // [WARPS][TN]
  uint32_t* stage = reinterpret_cast<uint32_t*>(tiles + WARPS * G::TN);  // [WARPS][32][SW]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float4* tile = tiles + warp * G::TN;
  uint32_t* wst = stage + warp * 32 * L.SW;
  const uint32_t n_active = dc->n_active;

  for (uint32_t ab = blockIdx.x; ab < n_active; ab += gridDim.x) {
    const uint32_t b = active_list[ab];
    const uint32_t start = block_start[b], end = block_start[b + 1];
    int bc[3];
    block_coords<D>(b, S, bc);
    const int org[3] = {bc[0] * G::B, bc[1] * G::B, bc[2] * G::B};
    for (int t = threadIdx.x; t < WARPS * G::TN; t += blockDim.x) tiles[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();

    for (uint32_t j0 = start + warp * 32; j0 < end; j0 += WARPS * 32) {
      const uint32_t cnt = min(32u, end - j0);
      const bool valid = (uint32_t)lane < cnt;
      const uint32_t r = perm[j0 + (valid ? lane : 0)];
      stage_load(rec, r, cnt, L.W, L.SW, wst, lane);
      __syncwarp();
      const uint32_t* row = wst + lane * L.SW;
      float s[NSV];
      if (valid) {
#pragma unroll
        for (int i = 0; i < NSV; ++i) s[i] = decode_field(row, L.s[i]);
      } else {
        benign_state<D, MAT>(s, org, S.dx);
      }
      int lb[3] = {0, 0, 0};
      float fx[3] = {0.f, 0.f, 0.f}, w[3][3];
#pragma unroll
      for (int a = 0; a < D; ++a) {
        bool o;
        lb[a] = base_fx(s[a], S.inv_dx, S.res[a], fx[a], o) - org[a];
        bspline_w(fx[a], w[a]);
      }
      float aff[D * D];
      affine_of<D, MAT>(s, S, aff);
      // momentum at node o: m v + aff (o - fx) dx = Q + sum_k o_k a_k,  a_k = dx aff[:,k]
      float ak[3][3], Q[3];
#pragma unroll
      for (int a = 0; a < D; ++a) {
        Q[a] = S.p_mass * s[D + a];
#pragma unroll
        for (int k = 0; k < D; ++k) {
          ak[k][a] = S.dx * aff[a * D + k];
          Q[a] -= fx[k] * ak[k][a];
        }
      }
      // conflict rounds: lanes of one round have distinct base cells, so the RMW
      // of one stencil offset touches distinct tile nodes (no shared-memory atomics)
      const int cell = valid ? (D == 3 ? (lb[0] * 4 + lb[1]) * 4 + lb[2] : lb[0] * 8 + lb[1]) : -1 - lane;
      const unsigned peers = __match_any_sync(FULL, cell);
      const int rank = __popc(peers & lanemask_lt());
      const int rounds = __reduce_max_sync(FULL, (unsigned)__popc(peers));
      const int base_idx = D == 3 ? (lb[0] * G::T + lb[1]) * G::T + lb[2] : lb[0] * G::T + lb[1];
      for (int rr = 0; rr < rounds; ++rr) {
        const bool mine = valid && rank == rr;
        const unsigned m = __ballot_sync(FULL, mine);
        if (mine) {
#pragma unroll
          for (int ox = 0; ox < 3; ++ox) {
#pragma unroll
            for (int oy = 0; oy < 3; ++oy) {
              const float wxy = w[0][ox] * w[1][oy];
              if (D == 3) {
#pragma unroll
                for (int oz = 0; oz < 3; ++oz) {
                  const float wt = wxy * w[2][oz];
                  const int idx = base_idx + (ox * G::T + oy) * G::T + oz;
                  float4 t = tile[idx];
                  t.x += wt * S.p_mass;
                  t.y += wt * (Q[0] + ox * ak[0][0] + oy * ak[1][0] + oz * ak[2][0]);
                  t.z += wt * (Q[1] + ox * ak[0][1] + oy * ak[1][1] + oz * ak[2][1]);
                  t.w += wt * (Q[2] + ox * ak[0][2] + oy * ak[1][2] + oz * ak[2][2]);
                  tile[idx] = t;
                  __syncwarp(m);
                }
              } else {
                const int idx = base_idx + ox * G::T + oy;
                float4 t = tile[idx];
                t.x += wxy * S.p_mass;
                t.y += wxy * (Q[0] + ox * ak[0][0] + oy * ak[1][0]);
                t.z += wxy * (Q[1] + ox * ak[0][1] + oy * ak[1][1]);
                tile[idx] = t;
                __syncwarp(m);
              }
            }
          }
        }
        __syncwarp();
      }
    }
    __syncthreads();
    // flush: sum the warp tiles, one vector reduction per non-empty node
    for (int t = threadIdx.x; t < G::TN; t += blockDim.x) {
      float4 acc = tiles[t];
#pragma unroll
      for (int wv = 1; wv < WARPS; ++wv) {
        const float4 o = tiles[wv * G::TN + t];
        acc.x += o.x;
        acc.y += o.y;
        acc.z += o.z;
        acc.w += o.w;
      }
      if (acc.x != 0.0f) {
        int tc[3];
        if (D == 3) {
          tc[2] = t % G::T;
          tc[1] = (t / G::T) % G::T;
          tc[0] = t / (G::T * G::T);
        } else {
          tc[1] = t % G::T;
          tc[0] = t / G::T;
          tc[2] = 0;
        }
        int nb[3], ln[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const int node = (a < D ? org[a] : 0) + tc[a];
          nb[a] = node >> G::LB;
          ln[a] = node & (G::B - 1);
        }
        const uint32_t slot = block_slot[block_id<D>(nb, S)];
        if (slot != 0xffffffffu) atomicAdd(&mp[(size_t)slot * 64 + local_node<D>(ln)], acc);
      }
    }
    __syncthreads();
  }
}

// ============================================================== a4: grid update
template <int D>
__global__ void k_grid_update(float4* __restrict__ mp, float4* __restrict__ gv,
                              const uint32_t* __restrict__ touched_list, const DevCounters* __restrict__ dc,
                              SimDev S) {
  using G = Geo<D>;
  const uint32_t nn = dc->n_touched_eff * 64u;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nn; t += gridDim.x * blockDim.x) {
    const uint32_t slot = t >> 6, ln = t & 63u;
    int bc[3];
    block_coords<D>(touched_list[slot], S, bc);
    int node[3];
    if (D == 3) {
      node[0] = bc[0] * G::B + (int)(ln >> 4);
      node[1] = bc[1] * G::B + (int)((ln >> 2) & 3);
      node[2] = bc[2] * G::B + (int)(ln & 3);
    } else {
      node[0] = bc[0] * G::B + (int)(ln >> 3);
      node[1] = bc[1] * G::B + (int)(ln & 7);
      node[2] = 0;
    }
    const float4 q = mp[t];
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
    if (q.x > 0.0f) {
      float v[3] = {q.y / q.x, q.z / q.x, q.w / q.x};
#pragma unroll
      for (int a = 0; a < D; ++a) {
        v[a] += S.dt * S.g[a];
        if (node[a] < S.bound && v[a] < 0.0f) v[a] = 0.0f;
        if (node[a] > S.res[a] - S.bound && v[a] > 0.0f) v[a] = 0.0f;
      }
      o = make_float4(v[0], v[1], D == 3 ? v[2] : 0.0f, 0.0f);
    }
    gv[t] = o;
    mp[t] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// ============================================================== a5-a7: G2P + encode
template <int D, int MAT, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_g2p(const uint32_t* __restrict__ rec_in,
                                                    uint32_t* __restrict__ rec_out,
                                                    const uint32_t* __restrict__ perm,
                                                    const uint32_t* __restrict__ ids_in,
                                                    uint32_t* __restrict__ ids_out,
                                                    float* __restrict__ dbg,
                                                    uint32_t* __restrict__ key_out,
                                                    uint32_t* __restrict__ block_count,
                                                    const uint32_t* __restrict__ block_start,
                                                    const uint32_t* __restrict__ active_list,
                                                    DevCounters* __restrict__ dc,
                                                    const uint32_t* __restrict__ block_slot,
                                                    const float4* __restrict__ gv, LayoutDev L, SimDev S,
                                                    uint32_t salt) {
  using G = Geo<D>;
  constexpr int NSV = NS<D, MAT>::value;
  constexpr int CO = 2 * D + (MAT == 1 ? 1 : D * D);
  extern __shared__ float4 smem4[];
  float4* tile = smem4;                                            // [TN]
  uint32_t* stage = reinterpret_cast<uint32_t*>(tile + G::TN);     // [WARPS][32][SW]
  __shared__ unsigned s_up[kMaxScalars], s_down[kMaxScalars], s_sat[kMaxScalars];
  __shared__ unsigned s_nonfinite, s_oob;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* wst = stage + warp * 32 * L.SW;
  for (int i = threadIdx.x; i < kMaxScalars; i += blockDim.x) s_up[i] = s_down[i] = s_sat[i] = 0u;
  if (threadIdx.x == 0) s_nonfinite = s_oob = 0u;
  const uint32_t n_active = dc->n_active;
  const float four_inv_dx = 4.0f * S.inv_dx;

  for (uint32_t ab = blockIdx.x; ab < n_active; ab += gridDim.x) {
    const uint32_t b = active_list[ab];
    const uint32_t start = block_start[b], end = block_start[b + 1];
    int bc[3];
    block_coords<D>(b, S, bc);
    const int org[3] = {bc[0] * G::B, bc[1] * G::B, bc[2] * G::B};
    __syncthreads();  // previous tile fully consumed
    for (int t = threadIdx.x; t < G::TN; t += blockDim.x) {
      int tc[3];
      if (D == 3) {
        tc[2] = t % G::T;
        tc[1] = (t / G::T) % G::T;
        tc[0] = t / (G::T * G::T);
      } else {
        tc[1] = t % G::T;
        tc[0] = t / G::T;
        tc[2] = 0;
      }
      int nb[3], ln[3];
      bool inside = true;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const int node = (a < D ? org[a] : 0) + tc[a];
        if (a < D && node >= S.res[a]) inside = false;
        nb[a] = node >> G::LB;
        ln[a] = node & (G::B - 1);
      }
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (inside) {
        const uint32_t slot = block_slot[block_id<D>(nb, S)];
        if (slot != 0xffffffffu) v = gv[(size_t)slot * 64 + local_node<D>(ln)];
      }
      tile[t] = v;
    }
    __syncthreads();

    for (uint32_t j0 = start + warp * 32; j0 < end; j0 += WARPS * 32) {
      const uint32_t cnt = min(32u, end - j0);
      const bool valid = (uint32_t)lane < cnt;
      const uint32_t r = perm[j0 + (valid ? lane : 0)];
      stage_load(rec_in, r, cnt, L.W, L.SW, wst, lane);
      __syncwarp();
      uint32_t* row = wst + lane * L.SW;
      // content key of the INPUT record (reading Q5)
      uint32_t key = 0;
      for (uint32_t m = L.xword_mask; m; m &= m - 1) key = mix32(key ^ row[__ffs(m) - 1]);
      const uint32_t h = mix32(key ^ salt);
      // decode x and F | J (v and C are overwritten)
      float s[NSV];
      if (valid) {
#pragma unroll
        for (int i = 0; i < NSV; ++i) s[i] = 0.0f;
#pragma unroll
        for (int i = 0; i < D; ++i) s[i] = decode_field(row, L.s[i]);
#pragma unroll
        for (int i = 2 * D; i < CO; ++i) s[i] = decode_field(row, L.s[i]);
      } else {
        benign_state<D, MAT>(s, org, S.dx);
      }
      int lb[3] = {0, 0, 0};
      float fx[3] = {0.f, 0.f, 0.f}, w[3][3];
      bool oob_any = false;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        bool o;
        lb[a] = base_fx(s[a], S.inv_dx, S.res[a], fx[a], o) - org[a];
        oob_any |= o;
        bspline_w(fx[a], w[a]);
      }
      // gather: v' = sum w v_i;  C' = 4/dx sum w v_i (i - fx) = 4/dx (T - S fx^T)
      float Sv[3] = {0.f, 0.f, 0.f}, T[3][3] = {{0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}};
      const int base_idx = D == 3 ? (lb[0] * G::T + lb[1]) * G::T + lb[2] : lb[0] * G::T + lb[1];
      if (D == 3) {
#pragma unroll
        for (int ox = 0; ox < 3; ++ox)
#pragma unroll
          for (int oy = 0; oy < 3; ++oy) {
            const float wxy = w[0][ox] * w[1][oy];
            const int idx = base_idx + (ox * G::T + oy) * G::T;
            const float4 g0 = tile[idx], g1 = tile[idx + 1], g2 = tile[idx + 2];
            const float g[3][3] = {{g0.x, g0.y, g0.z}, {g1.x, g1.y, g1.z}, {g2.x, g2.y, g2.z}};
#pragma unroll
            for (int a = 0; a < 3; ++a) {
              const float u0 = w[2][0] * g[0][a], u1 = w[2][1] * g[1][a], u2 = w[2][2] * g[2][a];
              const float sz = u0 + u1 + u2;
              const float tz = u1 + 2.0f * u2;
              Sv[a] += wxy * sz;
              T[a][2] += wxy * tz;
              if (ox) T[a][0] += (wxy * ox) * sz;
              if (oy) T[a][1] += (wxy * oy) * sz;
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
            const float u0 = w[1][0] * g[0][a], u1 = w[1][1] * g[1][a], u2 = w[1][2] * g[2][a];
            const float sy = u0 + u1 + u2;
            const float ty = u1 + 2.0f * u2;
            Sv[a] += w[0][ox] * sy;
            T[a][1] += w[0][ox] * ty;
            if (ox) T[a][0] += (w[0][ox] * ox) * sy;
          }
        }
      }
      float Cn[D * D];
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int k = 0; k < D; ++k) Cn[a * D + k] = four_inv_dx * (T[a][k] - Sv[a] * fx[k]);
      // new state, scalar order
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
            for (int m = 0; m < D; ++m) acc += S.dt * Cn[a * D + m] * s[2 * D + m * D + k];
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
      // encode into the thread-owned row (Eq. 11 dithering, reading Q5/Q6)
      __syncwarp();
      for (uint32_t q = 0; q <= L.W; ++q) row[q] = 0u;
      const bool dither = L.dither != 0;
#pragma unroll
      for (int i = 0; i < NSV; ++i) {
        const FieldDev& f = L.s[i];
        EncStat st;
        const uint32_t r24 = (dither && f.kind == kKindFixed) ? r24_of(h, f.idx) : 0u;
        const uint32_t bits = encode_field(o[i], f, dither, r24, st);
        put_field(row, f, bits);
        if (L.counters) {
          const unsigned bu = __ballot_sync(FULL, valid && st.up);
          const unsigned bd = __ballot_sync(FULL, valid && st.down);
          if (lane == 0) {
            if (bu) atomicAdd(&s_up[i], (unsigned)__popc(bu));
            if (bd) atomicAdd(&s_down[i], (unsigned)__popc(bd));
          }
        }
        if (__any_sync(FULL, valid && (st.sat | st.nonfinite))) {
          const unsigned bs = __ballot_sync(FULL, valid && st.sat);
          const unsigned bn = __ballot_sync(FULL, valid && st.nonfinite);
          if (lane == 0) {
            if (bs) atomicAdd(&s_sat[i], (unsigned)__popc(bs));
            if (bn) atomicAdd(&s_nonfinite, (unsigned)__popc(bn));
          }
        }
      }
      {
        const unsigned bo = __ballot_sync(FULL, valid && oob_any);
        if (lane == 0 && bo) atomicAdd(&s_oob, (unsigned)__popc(bo));
      }
      // next step's block key from the re-decoded (quantized) x
      float xq[3];
#pragma unroll
      for (int a = 0; a < D; ++a) xq[a] = decode_field(row, L.s[a]);
      const uint32_t nk = valid ? key_of<D>(xq, S) : 0xffffffffu;
      if (valid) key_out[j] = nk;
      const unsigned kp = __match_any_sync(FULL, nk);
      if (valid && lane == __ffs(kp) - 1) atomicAdd(&block_count[nk], (unsigned)__popc(kp));
      if (ids_out != nullptr && valid) ids_out[j] = ids_in[r];
      __syncwarp();
      stage_store(rec_out + (size_t)j0 * L.W, cnt, L.W, L.SW, wst, lane);
      __syncwarp();
    }
  }
  __syncthreads();
  // flush the CTA's counters (map scalar -> packing index)
  for (int i = threadIdx.x; i < NSV; i += blockDim.x) {
    const int fi = L.s[i].idx;
    if (s_up[i]) atomicAdd(&dc->up[fi], (unsigned long long)s_up[i]);
    if (s_down[i]) atomicAdd(&dc->down[fi], (unsigned long long)s_down[i]);
    if (s_sat[i]) atomicAdd(&dc->sat[fi], (unsigned long long)s_sat[i]);
  }
  if (threadIdx.x == 0) {
    if (s_nonfinite) atomicAdd(&dc->nonfinite, (unsigned long long)s_nonfinite);
    if (s_oob) atomicAdd(&dc->oob, (unsigned long long)s_oob);
  }
}

// ============================================================== standalone codec
constexpr int kCodecThreads = 128;

__global__ void __launch_bounds__(kCodecThreads) k_encode(const float* __restrict__ vals,
                                                          const uint32_t* __restrict__ keys, uint64_t n,
                                                          CodecDev C, uint32_t salt,
                                                          uint32_t* __restrict__ words,
                                                          unsigned long long* __restrict__ counters) {
  extern __shared__ uint32_t sm[];
  float* vst = reinterpret_cast<float*>(sm);         // [128][stride]
  uint32_t* wst = sm + kCodecThreads * C.stride;     // [128][SW]
  __shared__ unsigned s_cnt[3][kMaxFields];
  for (int i = threadIdx.x; i < 3 * kMaxFields; i += blockDim.x) (&s_cnt[0][0])[i] = 0u;
  const uint64_t row0 = (uint64_t)blockIdx.x * kCodecThreads;
  const uint32_t cnt = (uint32_t)min((uint64_t)kCodecThreads, n - row0);
  for (uint32_t q = threadIdx.x; q < cnt * C.stride; q += blockDim.x) vst[q] = vals[row0 * C.stride + q];
  __syncthreads();
  const uint32_t tid = threadIdx.x;
  if (tid < cnt) {
    uint32_t* row = wst + tid * C.SW;
    for (uint32_t q = 0; q <= C.W; ++q) row[q] = 0u;
    const bool dither = keys != nullptr && C.dither;
    const uint32_t h = dither ? mix32(keys[row0 + tid] ^ salt) : 0u;
    for (uint32_t fi = 0; fi < C.nf; ++fi) {
      const FieldDev& f = C.f[fi];
      EncStat st;
      const uint32_t r24 = (dither && f.kind == kKindFixed) ? r24_of(h, fi) : 0u;
      const uint32_t bits = encode_field(vst[tid * C.stride + f.col], f, dither, r24, st);
      put_field(row, f, bits);
      if (counters) {
        if (st.sat) atomicAdd(&s_cnt[0][fi], 1u);
        if (st.up) atomicAdd(&s_cnt[1][fi], 1u);
        if (st.down) atomicAdd(&s_cnt[2][fi], 1u);
      }
    }
  }
  __syncthreads();
  for (uint32_t q = threadIdx.x; q < cnt * C.W; q += blockDim.x)
    words[row0 * C.W + q] = wst[(q / C.W) * C.SW + q % C.W];
  if (counters) {
    for (uint32_t i = threadIdx.x; i < 3 * C.nf; i += blockDim.x) {
      const uint32_t k = i / C.nf, fi = i % C.nf;
      if (s_cnt[k][fi]) atomicAdd(&counters[k * kMaxFields + fi], (unsigned long long)s_cnt[k][fi]);
    }
  }
}

__global__ void __launch_bounds__(kCodecThreads) k_decode(const uint32_t* __restrict__ words, uint64_t n,
                                                          CodecDev C, float* __restrict__ vals) {
  extern __shared__ uint32_t sm[];
  float* vst = reinterpret_cast<float*>(sm);
  uint32_t* wst = sm + kCodecThreads * C.stride;
  const uint64_t row0 = (uint64_t)blockIdx.x * kCodecThreads;
  const uint32_t cnt = (uint32_t)min((uint64_t)kCodecThreads, n - row0);
  for (uint32_t q = threadIdx.x; q < cnt * C.W; q += blockDim.x)
    wst[(q / C.W) * C.SW + q % C.W] = words[row0 * C.W + q];
  __syncthreads();
  const uint32_t tid = threadIdx.x;
  if (tid < cnt) {
    uint32_t* row = wst + tid * C.SW;
    row[C.W] = 0u;
    for (uint32_t fi = 0; fi < C.nf; ++fi) vst[tid * C.stride + C.f[fi].col] = decode_field(row, C.f[fi]);
  }
  __syncthreads();
  for (uint32_t q = threadIdx.x; q < cnt * C.stride; q += blockDim.x) vals[row0 * C.stride + q] = vst[q];
}

__global__ void k_iota(uint32_t* ids, uint32_t n, uint32_t first) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) ids[i] = first + i;
}

// ============================================================== launchers
constexpr int kP2GWarps = 4;
constexpr int kG2PWarps = 4;

template <int D, int MAT>
static size_t p2g_smem(const LayoutDev& L) {
  return sizeof(float4) * kP2GWarps * Geo<D>::TN + sizeof(uint32_t) * kP2GWarps * 32 * L.SW;
}
template <int D, int MAT>
static size_t g2p_smem(const LayoutDev& L) {
  return sizeof(float4) * Geo<D>::TN + sizeof(uint32_t) * kG2PWarps * 32 * L.SW;
}

template <int D, int MAT>
static cudaError_t setup_dm(const LayoutDev& L, LaunchCfg& cfg) {
  int dev;
  cudaError_t e = cudaGetDevice(&dev);
  if (e) return e;
  e = cudaDeviceGetAttribute(&cfg.num_sms, cudaDevAttrMultiProcessorCount, dev);
  if (e) return e;
  cfg.p2g_smem = p2g_smem<D, MAT>(L);
  cfg.g2p_smem = g2p_smem<D, MAT>(L);
  e = cudaFuncSetAttribute(k_p2g<D, MAT, kP2GWarps>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.p2g_smem);
  if (e) return e;
  e = cudaFuncSetAttribute(k_g2p<D, MAT, kG2PWarps>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.g2p_smem);
  if (e) return e;
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_p2g<D, MAT, kP2GWarps>, kP2GWarps * 32, cfg.p2g_smem);
  if (e) return e;
  cfg.p2g_ctas = cfg.num_sms * (occ > 0 ? occ : 1);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_g2p<D, MAT, kG2PWarps>, kG2PWarps * 32, cfg.g2p_smem);
  if (e) return e;
  cfg.g2p_ctas = cfg.num_sms * (occ > 0 ? occ : 1);
  return cudaSuccess;
}

cudaError_t setup_kernels(int dim, int material, const LayoutDev& L, LaunchCfg& cfg) {
  if (dim == 3 && material == 0) return setup_dm<3, 0>(L, cfg);
  if (dim == 3 && material == 1) return setup_dm<3, 1>(L, cfg);
  if (dim == 2 && material == 0) return setup_dm<2, 0>(L, cfg);
  return setup_dm<2, 1>(L, cfg);
}

cudaError_t launch_bin_count(int dim, const uint32_t* rec, uint32_t n, const LayoutDev& L, const SimDev& S,
                             uint32_t* key, uint32_t* block_count, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const int th = 256;
  const unsigned blocks = (n + th - 1) / th;
  if (dim == 3)
    k_bin_count<3><<<blocks, th, 0, st>>>(rec, n, L, S, key, block_count);
  else
    k_bin_count<2><<<blocks, th, 0, st>>>(rec, n, L, S, key, block_count);
  return cudaGetLastError();
}

template <int D, int MAT>
static cudaError_t step_dm(const StepBuffers& B, const LayoutDev& L, const SimDev& S, uint32_t salt,
                           const LaunchCfg& cfg, cudaStream_t st, KernelHook hook, void* user) {
  auto H = [&](int k, int b) {
    if (hook) hook(user, k, b);
  };
  H(KScanReduce, 1);
  k_scan_reduce<D><<<B.ntiles, kScanThreads, 0, st>>>(B.block_count, S, B.tile_sums);
  H(KScanReduce, 0);
  H(KScanTiles, 1);
  k_scan_tiles<<<1, 1024, 0, st>>>(B.tile_sums, B.ntiles, B.tile_off, B.dc, B.block_start, S.nblocks, B.pool);
  H(KScanTiles, 0);
  H(KScanApply, 1);
  k_scan_apply<D><<<B.ntiles, kScanThreads, 0, st>>>(B.block_count, S, B.tile_off, B.block_start, B.block_slot,
                                                     B.active_list, B.touched_list, B.pool);
  H(KScanApply, 0);
  if (B.n) {
    H(KBinScatter, 1);
    k_bin_scatter<<<(B.n + 255) / 256, 256, 0, st>>>(B.key, B.n, B.block_start, B.block_count, B.perm);
    H(KBinScatter, 0);
  }
  H(KP2G, 1);
  k_p2g<D, MAT, kP2GWarps><<<cfg.p2g_ctas, kP2GWarps * 32, cfg.p2g_smem, st>>>(
      B.rec_in, B.perm, B.block_start, B.active_list, B.dc, B.block_slot, B.mp, L, S);
  H(KP2G, 0);
  H(KGridUpdate, 1);
  k_grid_update<D><<<cfg.num_sms * 8, 256, 0, st>>>(B.mp, B.gv, B.touched_list, B.dc, S);
  H(KGridUpdate, 0);
  H(KG2P, 1);
  k_g2p<D, MAT, kG2PWarps><<<cfg.g2p_ctas, kG2PWarps * 32, cfg.g2p_smem, st>>>(
      B.rec_in, B.rec_out, B.perm, B.ids_in, B.ids_out, B.dbg, B.key, B.block_count, B.block_start,
      B.active_list, B.dc, B.block_slot, B.gv, L, S, salt);
  H(KG2P, 0);
  return cudaGetLastError();
}

cudaError_t launch_step(int dim, int material, const StepBuffers& B, const LayoutDev& L, const SimDev& S,
                        uint32_t salt, const LaunchCfg& cfg, cudaStream_t st, KernelHook hook, void* user) {
  if (dim == 3 && material == 0) return step_dm<3, 0>(B, L, S, salt, cfg, st, hook, user);
  if (dim == 3 && material == 1) return step_dm<3, 1>(B, L, S, salt, cfg, st, hook, user);
  if (dim == 2 && material == 0) return step_dm<2, 0>(B, L, S, salt, cfg, st, hook, user);
  return step_dm<2, 1>(B, L, S, salt, cfg, st, hook, user);
}

static size_t codec_smem(const CodecDev& C) {
  return sizeof(uint32_t) * kCodecThreads * (C.stride + C.SW);
}

cudaError_t launch_encode(const CodecDev& C, uint64_t n, const float* vals, const uint32_t* keys, uint32_t salt,
                          uint32_t* words, unsigned long long* counters, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const size_t sm = codec_smem(C);
  cudaError_t e = cudaFuncSetAttribute(k_encode, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e) return e;
  const uint64_t blocks = (n + kCodecThreads - 1) / kCodecThreads;
  k_encode<<<(unsigned)blocks, kCodecThreads, sm, st>>>(vals, keys, n, C, salt, words, counters);
  return cudaGetLastError();
}

cudaError_t launch_decode(const CodecDev& C, uint64_t n, const uint32_t* words, float* vals, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const size_t sm = codec_smem(C);
  cudaError_t e = cudaFuncSetAttribute(k_decode, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e) return e;
  const uint64_t blocks = (n + kCodecThreads - 1) / kCodecThreads;
  k_decode<<<(unsigned)blocks, kCodecThreads, sm, st>>>(words, n, C, vals);
  return cudaGetLastError();
}

cudaError_t launch_iota(uint32_t* ids, uint32_t n, uint32_t first, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_iota<<<(n + 255) / 256, 256, 0, st>>>(ids, n, first);
  return cudaGetLastError();
}

}  // namespace qmpm
