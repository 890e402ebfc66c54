// kernels.cu -- the layout-independent kernels of one quantized MLS-MPM step
// and the standalone codec.  The layout-dependent
// kernels (bin count, P2G, G2P + encode) are NVRTC-specialised: step_kernels.cuh.
//
//   k_scan_*       a1  exclusive scan over the dense block table: particle offsets,
//                      active-block list, touched-block (pool slot) assignment
//   k_cell_scan    a1  per active block: cell counts -> cell cursors (end positions)
//   k_bin_scatter  a1  counting-sort scatter by (block, cell): perm[sorted slot] = record index
//   k_grid_update  a4  v = p/m + dt g, separating walls; clears (m, p) for next step
// (the standalone codec is NVRTC-specialised too: codec_kernels.cuh)
#include <algorithm>

#include <cuda_runtime.h>

#include "jit.h"
#include "mpm_common.cuh"
#include "qmpm_launch.h"

namespace qmpm {

// ============================================================== a1: binning
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
  // a slab's bottom block plane receives the lower neighbour's ghost contributions
  if (D == 3 && S.slab_lo && bc[2] == S.slab_bz0) touched = 1;
#pragma unroll
  for (int dl = 1; dl < (1 << D); ++dl) {
    int nc[3] = {bc[0] - (dl & 1), bc[1] - ((dl >> 1) & 1), D == 3 ? bc[2] - ((dl >> 2) & 1) : 0};
    if (nc[0] < 0 || nc[1] < 0 || (D == 3 && nc[2] < S.tab_bz0)) continue;
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
    dc->gstep += 1u;  // the step this sort starts (G2P's dither salt)
    dc->n_active = total.y;
    dc->next_p2g = 0u;
    dc->next_g2p = 0u;
    dc->n_touched = total.z;
    dc->n_touched_eff = total.z < pool ? total.z : pool;
    dc->n_sorted = total.x;
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
                                                             uint32_t pool, DevCounters* __restrict__ dc) {
  // slab ranks: active blocks below the top owned block plane (the overlap split of P2G/G2P)
  const uint32_t top_first = D == 3 ? (uint32_t)(S.slab_bz1 - 1 - S.tab_bz0) * (uint32_t)S.nb[0] * (uint32_t)S.nb[1]
                                    : 0xffffffffu;
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
    if (b == top_first) dc->n_active_below = ex.y;
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

// Cell-level cursors of the counting sort by (block, base cell): one warp per active
// block turns the 64 cell counts (accumulated by G2P / bin_count) into END positions
// block_start[b] + inclusive prefix; the scatter's atomicSub leaves each at its cell's
// START, which P2G reads (and zeroes for the next step's counts).  The block's count
// has been consumed by the scan: it is zeroed here for the next step's histogram.
__device__ __forceinline__ void cell_scan_block(uint32_t b, uint32_t lane, uint32_t* __restrict__ cell_count,
                                                uint32_t* __restrict__ block_count,
                                                const uint32_t* __restrict__ block_start) {
  uint32_t* cc = cell_count + (size_t)b * 64;
  const uint32_t c0 = cc[lane], c1 = cc[lane + 32];
  uint32_t i0 = c0, i1 = c1;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t0 = __shfl_up_sync(FULL, i0, d), t1 = __shfl_up_sync(FULL, i1, d);
    if ((int)lane >= d) {
      i0 += t0;
      i1 += t1;
    }
  }
  const uint32_t base = block_start[b];
  const uint32_t tot0 = __shfl_sync(FULL, i0, 31);
  cc[lane] = base + i0;
  cc[lane + 32] = base + tot0 + i1;
  if (lane == 0) block_count[b] = 0u;
}

__global__ void k_cell_scan(uint32_t* __restrict__ cell_count, uint32_t* __restrict__ block_count,
                            const uint32_t* __restrict__ block_start, const uint32_t* __restrict__ active_list,
                            const DevCounters* __restrict__ dc) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  const uint32_t n_active = dc->n_active;
  for (uint32_t ab = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; ab < n_active; ab += warps)
    cell_scan_block(active_list[ab], lane, cell_count, block_count, block_start);
}

// The whole sort front (scan_reduce + scan_tiles + scan_apply + cell_scan) in ONE CTA
// when the block table fits one scan tile (nblocks <= kScanTile, e.g. C1's 2D 128^2
// grid): the same arithmetic in the same order, three launches fewer per step (C1 is
// launch-bound).  The tile offset of the single tile is 0.
template <int D>
__global__ void __launch_bounds__(kScanThreads) k_sort_small(uint32_t* __restrict__ count, SimDev S,
                                                             uint32_t* __restrict__ block_start,
                                                             uint32_t* __restrict__ block_slot,
                                                             uint32_t* __restrict__ active_list,
                                                             uint32_t* __restrict__ touched_list, uint32_t pool,
                                                             DevCounters* __restrict__ dc,
                                                             uint32_t* __restrict__ cell_count) {
  const uint32_t top_first = D == 3 ? (uint32_t)(S.slab_bz1 - 1 - S.tab_bz0) * (uint32_t)S.nb[0] * (uint32_t)S.nb[1]
                                    : 0xffffffffu;
  const uint32_t b0 = threadIdx.x * kScanPer;
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
  uint3 ex = block_exclusive_scan3(v, total);  // (ends with a barrier: every count read)
  if (threadIdx.x == 0) {  // k_scan_tiles' counters
    dc->gstep += 1u;
    dc->n_active = total.y;
    dc->next_p2g = 0u;
    dc->next_g2p = 0u;
    dc->n_touched = total.z;
    dc->n_touched_eff = total.z < pool ? total.z : pool;
    dc->n_sorted = total.x;
    if (total.z > pool) dc->overflow += 1ull;
    block_start[S.nblocks] = total.x;
  }
#pragma unroll
  for (int q = 0; q < kScanPer; ++q) {  // k_scan_apply
    const uint32_t b = b0 + q;
    if (b == top_first) dc->n_active_below = ex.y;
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
  __syncthreads();  // block_start / active_list visible to the CTA
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t ab = threadIdx.x >> 5; ab < total.y; ab += kScanThreads / 32)  // k_cell_scan
    cell_scan_block(active_list[ab], lane, cell_count, count, block_start);
}

// Counting-sort scatter by the full key (block, base cell): perm[pos] = record slot,
// pos from a warp-aggregated atomicSub on the key's cell cursor; dead keys (particles a
// slab rank no longer owns) are skipped.  The slot count comes from the device
// (DevCounters::n_slots: it includes a slab's appended arrivals, never synchronised to
// the host).  kBinItems particles per thread in flight (strided by the CTA size, so loads
// stay coalesced): the per-particle chain key -> atomic -> store is latency-bound.
// (Measured at C4, 0.91 ms: 2 or 8 items per thread and 4 or 16 CTAs per SM all within
// noise of this configuration.)
constexpr int kBinItems = 4;

// Grid of a grid-stride (or work-counter) kernel: per_sm CTAs per SM, but no more than
// `work` items at `per_cta` items per CTA need -- the device-side counts are not known
// on the host (no per-step sync), the capacity / block count / pool bound them.  Small
// problems (C1: 8K particles) then launch tens of CTAs instead of ~1,200 idle ones.
inline unsigned grid_for(int num_sms, int per_sm, uint64_t work, uint64_t per_cta = 256) {
  const uint64_t need = (work + per_cta - 1) / per_cta;
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)num_sms * per_sm, need));
}
// active blocks are at most the blocks of the table and at most the particles
inline uint64_t max_active(const StepBuffers& B, const SimDev& S) {
  return std::min<uint64_t>((uint64_t)S.nblocks, (uint64_t)B.cap);
}
__global__ void __launch_bounds__(256) k_bin_scatter(const uint32_t* __restrict__ key, const DevCounters* __restrict__ dc,
                                                      uint32_t* __restrict__ cell_count, uint32_t* __restrict__ perm) {
  const uint32_t n = dc->n_slots;
  const uint32_t stride = gridDim.x * blockDim.x * kBinItems;
  for (uint32_t i0 = blockIdx.x * (blockDim.x * kBinItems) + threadIdx.x; i0 - threadIdx.x < n; i0 += stride) {
    uint32_t k[kBinItems], old[kBinItems];
    unsigned peers[kBinItems];
#pragma unroll
    for (int u = 0; u < kBinItems; ++u) {
      const uint32_t i = i0 + u * blockDim.x;
      k[u] = i < n ? __ldg(key + i) : kDeadKey;
    }
#pragma unroll
    for (int u = 0; u < kBinItems; ++u) {
      peers[u] = __match_any_sync(FULL, k[u]);
      const int leader = __ffs(peers[u]) - 1;
      old[u] = 0;
      if (k[u] != kDeadKey && (int)(threadIdx.x & 31) == leader)
        old[u] = atomicSub(&cell_count[k[u]], (uint32_t)__popc(peers[u]));
    }
#pragma unroll
    for (int u = 0; u < kBinItems; ++u) {
      const int leader = __ffs(peers[u]) - 1;
      const uint32_t top = __shfl_sync(FULL, old[u], leader);
      if (k[u] != kDeadKey) perm[top - 1 - __popc(peers[u] & lanemask_lt())] = i0 + u * blockDim.x;
    }
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

// ============================================================== slab exchange (a8)
// Dense copy of one z block plane of a float4 node array (all nbx * nby blocks,
// 64 nodes each; blocks without a pool slot read as zero).
__global__ void k_plane_pack(const float4* __restrict__ src, const uint32_t* __restrict__ block_slot, SimDev S,
                             int bz, float4* __restrict__ buf) {
  const uint32_t P = (uint32_t)S.nb[0] * (uint32_t)S.nb[1];
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < P * 64u; t += gridDim.x * blockDim.x) {
    const uint32_t pb = t >> 6;
    const int c[3] = {(int)(pb / (uint32_t)S.nb[1]), (int)(pb % (uint32_t)S.nb[1]), bz};
    const uint32_t slot = block_slot[block_id<3>(c, S)];
    buf[t] = slot != 0xffffffffu ? src[(size_t)slot * 64 + (t & 63u)] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// add (halo reduce of P2G partial sums) or store (velocity halo) a packed plane
__global__ void k_plane_unpack(float4* __restrict__ dst, const uint32_t* __restrict__ block_slot, SimDev S, int bz,
                               const float4* __restrict__ buf, int add) {
  const uint32_t P = (uint32_t)S.nb[0] * (uint32_t)S.nb[1];
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < P * 64u; t += gridDim.x * blockDim.x) {
    const uint32_t pb = t >> 6;
    const int c[3] = {(int)(pb / (uint32_t)S.nb[1]), (int)(pb % (uint32_t)S.nb[1]), bz};
    const uint32_t slot = block_slot[block_id<3>(c, S)];
    if (slot == 0xffffffffu) continue;
    const float4 v = buf[t];
    float4& d = dst[(size_t)slot * 64 + (t & 63u)];
    if (add) {
      d.x += v.x;
      d.y += v.y;
      d.z += v.z;
      d.w += v.w;
    } else {
      d = v;
    }
  }
}

__global__ void k_iota(uint32_t* ids, uint32_t n, uint32_t first) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) ids[i] = first + i;
}

// ============================================================== launchers
namespace {
struct Hk {
  KernelHook hook;
  void* user;
  void operator()(int k, int b) const {
    if (hook) hook(user, k, b);
  }
};
}  // namespace

template <int D>
static cudaError_t sort_d(const StepBuffers& B, const SimDev& S, cudaStream_t st, Hk H) {
  if (B.ntiles == 1) {  // one scan tile: the fused single-CTA front (timed as scan_reduce)
    H(KScanReduce, 1);
    k_sort_small<D><<<1, kScanThreads, 0, st>>>(B.block_count, S, B.block_start, B.block_slot, B.active_list,
                                                B.touched_list, B.pool, B.dc, B.cell_count);
    H(KScanReduce, 0);
  } else {
  H(KScanReduce, 1);
  k_scan_reduce<D><<<B.ntiles, kScanThreads, 0, st>>>(B.block_count, S, B.tile_sums);
  H(KScanReduce, 0);
  H(KScanTiles, 1);
  k_scan_tiles<<<1, 1024, 0, st>>>(B.tile_sums, B.ntiles, B.tile_off, B.dc, B.block_start, S.nblocks, B.pool);
  H(KScanTiles, 0);
  H(KScanApply, 1);
  k_scan_apply<D><<<B.ntiles, kScanThreads, 0, st>>>(B.block_count, S, B.tile_off, B.block_start, B.block_slot,
                                                     B.active_list, B.touched_list, B.pool, B.dc);
  H(KScanApply, 0);
  H(KCellScan, 1);
  k_cell_scan<<<grid_for(B.num_sms, 8, 32ull * max_active(B, S)), 256, 0, st>>>(B.cell_count, B.block_count,
                                                                                  B.block_start, B.active_list, B.dc);
  H(KCellScan, 0);
  }
  H(KBinScatter, 1);
  k_bin_scatter<<<grid_for(B.num_sms, 8, (uint64_t)B.cap, 256 * kBinItems), 256, 0, st>>>(B.key, B.dc, B.cell_count,
                                                                                           B.perm);
  H(KBinScatter, 0);
  return cudaGetLastError();
}

int step_launches(const StepBuffers& B) { return B.ntiles == 1 ? 5 : 8; }

cudaError_t launch_sort(int dim, const StepBuffers& B, const SimDev& S, cudaStream_t st, KernelHook hook, void* user) {
  return dim == 3 ? sort_d<3>(B, S, st, Hk{hook, user}) : sort_d<2>(B, S, st, Hk{hook, user});
}

cudaError_t launch_p2g(const StepBuffers& B, const SimDev& S, const StepJit& J, int part, cudaStream_t st,
                       KernelHook hook, void* user) {
  Hk H{hook, user};
  H(KP2G, 1);
  SimDev Sv = S;
  int pv = part;
  void* args[] = {(void*)&B.rec_in,      (void*)&B.perm, (void*)&B.cell_count, (void*)&B.block_start,
                  (void*)&B.active_list, (void*)&B.dc,   (void*)&B.block_slot, (void*)&B.mp,
                  (void*)&Sv,            (void*)&pv};
  cudaError_t e = jit_launch(J.p2g, std::min<unsigned>(J.p2g_ctas, grid_for(1, 1 << 30, max_active(B, S), J.p2g_threads / 32)),
                             J.p2g_threads, J.p2g_smem, st, args);
  H(KP2G, 0);
  return e;
}

cudaError_t launch_grid_update(int dim, const StepBuffers& B, const SimDev& S, const StepJit& J, cudaStream_t st,
                               KernelHook hook, void* user) {
  Hk H{hook, user};
  H(KGridUpdate, 1);
  if (dim == 3)
    k_grid_update<3><<<grid_for(J.num_sms, 8, 64ull * B.pool), 256, 0, st>>>(B.mp, B.gv, B.touched_list, B.dc, S);
  else
    k_grid_update<2><<<grid_for(J.num_sms, 8, 64ull * B.pool), 256, 0, st>>>(B.mp, B.gv, B.touched_list, B.dc, S);
  H(KGridUpdate, 0);
  return cudaGetLastError();
}

cudaError_t launch_g2p(const StepBuffers& B, const SimDev& S, const MigDev& M, const StepJit& J, int part,
                       cudaStream_t st, KernelHook hook, void* user) {
  Hk H{hook, user};
  H(KG2P, 1);
  SimDev Sv = S;
  MigDev Mv = M;
  int pv = part;
  void* args[] = {(void*)&B.rec_in, (void*)&B.rec_out, (void*)&B.perm, (void*)&B.ids_in, (void*)&B.ids_out,
                  (void*)&B.dbg, (void*)&B.key, (void*)&B.block_count, (void*)&B.cell_count, (void*)&B.block_start,
                  (void*)&B.active_list, (void*)&B.dc, (void*)&B.block_slot, (void*)&B.gv, (void*)&Sv,
                  (void*)&Mv, (void*)&pv};
  cudaError_t e = jit_launch(J.g2p, std::min<unsigned>(J.g2p_ctas, grid_for(1, 1 << 30, max_active(B, S), J.g2p_threads / 32)),
                             J.g2p_threads, J.g2p_smem, st, args);
  H(KG2P, 0);
  return e;
}

cudaError_t launch_step(int dim, const StepBuffers& B, const SimDev& S, const MigDev& M, const StepJit& J,
                        cudaStream_t st, KernelHook hook, void* user) {
  cudaError_t e = launch_sort(dim, B, S, st, hook, user);
  if (!e) e = launch_p2g(B, S, J, 0, st, hook, user);
  if (!e) e = launch_grid_update(dim, B, S, J, st, hook, user);
  if (!e) e = launch_g2p(B, S, M, J, 0, st, hook, user);
  return e;
}

cudaError_t launch_bin_count(const uint32_t* rec, const uint32_t* ids, uint32_t first, uint32_t n, const SimDev& S,
                             uint32_t* key, uint32_t* block_count, uint32_t* cell_count, int do_count,
                             const MigDev& M, DevCounters* dc, const StepJit& J, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  SimDev Sv = S;
  MigDev Mv = M;
  void* args[] = {(void*)&rec, (void*)&ids, (void*)&first, (void*)&n, (void*)&Sv, (void*)&key,
                  (void*)&block_count, (void*)&cell_count, (void*)&do_count, (void*)&Mv, (void*)&dc};
  return jit_launch(J.bin_count, (n + 255) / 256, 256, 0, st, args);
}

cudaError_t launch_append(uint32_t* rec, uint32_t* ids, float* dbg, uint64_t cap, const SimDev& S, uint32_t* key,
                          uint32_t* block_count, uint32_t* cell_count, const MigDev& M, DevCounters* dc,
                          const StepJit& J, cudaStream_t st) {
  SimDev Sv = S;
  MigDev Mv = M;
  uint64_t capv = cap;
  void* args[] = {(void*)&rec, (void*)&ids, (void*)&dbg, (void*)&capv, (void*)&Sv, (void*)&key,
                  (void*)&block_count, (void*)&cell_count, (void*)&Mv, (void*)&dc};
  return jit_launch(J.append, (unsigned)std::min<uint64_t>((2ull * M.cap + 255) / 256, (uint64_t)J.num_sms * 8), 256,
                    0, st, args);
}

cudaError_t launch_plane(float4* nodes, const uint32_t* block_slot, const SimDev& S, int bz, float4* buf, int mode,
                         int num_sms, cudaStream_t st) {
  if (mode == 0)
    k_plane_pack<<<num_sms * 4, 256, 0, st>>>(nodes, block_slot, S, bz, buf);
  else
    k_plane_unpack<<<num_sms * 4, 256, 0, st>>>(nodes, block_slot, S, bz, buf, mode == 1);
  return cudaGetLastError();
}

// read_state of a slab context: the live record slots (every slot of [0, n_slots) not in
// the sorted dead list) in slot order: out[i] = the i-th live slot
__global__ void k_live_slots(const uint32_t* __restrict__ dead_sorted, uint32_t n_dead, uint32_t n_slots,
                             uint32_t* __restrict__ out) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n_slots; s += gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = n_dead;  // dead slots below s
    while (lo < hi) {
      const uint32_t mid = (lo + hi) / 2;
      if (dead_sorted[mid] < s) lo = mid + 1; else hi = mid;
    }
    if (lo < n_dead && dead_sorted[lo] == s) continue;
    out[s - lo] = s;
  }
}

__global__ void k_gather_rows(const uint32_t* __restrict__ src, const uint32_t* __restrict__ slots, uint32_t n,
                              uint32_t row, uint32_t* __restrict__ dst) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < (uint64_t)n * row;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = t / row, q = t - i * row;
    dst[t] = src[(uint64_t)slots[i] * row + q];
  }
}

cudaError_t launch_live_slots(const uint32_t* dead_sorted, uint32_t n_dead, uint32_t n_slots, uint32_t* out,
                              int num_sms, cudaStream_t st) {
  if (n_slots == 0) return cudaSuccess;
  k_live_slots<<<num_sms * 8, 256, 0, st>>>(dead_sorted, n_dead, n_slots, out);
  return cudaGetLastError();
}

cudaError_t launch_gather_rows(const uint32_t* src, const uint32_t* slots, uint32_t n, uint32_t row, uint32_t* dst,
                               int num_sms, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_gather_rows<<<num_sms * 8, 256, 0, st>>>(src, slots, n, row, dst);
  return cudaGetLastError();
}

// qmpm_set_state / append_state: non-finite input values (an error value; the
// encoder stores code 0) are counted into DevCounters::nonfinite
__global__ void k_count_nonfinite(const float* __restrict__ v, uint64_t n, unsigned long long* __restrict__ out) {
  unsigned c = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    c += !isfinite(v[i]);
  c = __reduce_add_sync(FULL, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

cudaError_t launch_count_nonfinite(const float* vals, uint64_t n, unsigned long long* out, int num_sms,
                                   cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_count_nonfinite<<<num_sms * 4, 256, 0, st>>>(vals, n, out);
  return cudaGetLastError();
}

cudaError_t launch_iota(uint32_t* ids, uint32_t n, uint32_t first, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_iota<<<(n + 255) / 256, 256, 0, st>>>(ids, n, first);
  return cudaGetLastError();
}

}  // namespace qmpm
