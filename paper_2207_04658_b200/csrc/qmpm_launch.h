// qmpm_launch.h -- host-side launchers of the qmpm kernels (kernels.cu), used by
// the runtime (api.cu).  Internal; not part of the C ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include <cuda.h>

#include "qmpm_device.cuh"

namespace qmpm {

struct StepBuffers {
  const uint32_t* rec_in;
  uint32_t* rec_out;
  const uint32_t* ids_in;  // nullable
  uint32_t* ids_out;       // nullable
  uint32_t* key;           // [n] block key of each record in rec_in order (in), rec_out order (out)
  uint32_t* perm;          // [n] sorted slot -> rec_in index, sorted by (block, base cell)
  uint32_t* cell_count;    // [nblocks * 64] per (block, cell): next step's counts (G2P) ->
                           // cursors (k_cell_scan) -> cell starts (scatter) -> 0 (P2G)
  uint32_t* block_count;   // [nblocks]
  uint32_t* block_start;   // [nblocks + 1]
  uint32_t* block_slot;    // [nblocks]
  uint32_t* active_list;   // [nblocks]
  uint32_t* touched_list;  // [pool]
  uint4* tile_sums;        // [ntiles]
  uint4* tile_off;         // [ntiles]
  float4* mp;              // [pool * 64]  (m, p) -- zero between steps
  float4* gv;              // [pool * 64]  (v, 0)
  DevCounters* dc;
  float* dbg;              // nullable [n][ns]
  uint32_t n;
  uint32_t cap;             // particle capacity (an upper bound of the device-side counts)
  uint32_t pool;
  uint32_t ntiles;
  int num_sms;
};

constexpr int kScanTile = 1024;  // grid blocks per scan tile

// kernel ids for profiling (order = qmpm_kernel_name)
enum KernelId {
  KBinCount = 0,
  KScanReduce,
  KScanTiles,
  KScanApply,
  KCellScan,
  KBinScatter,
  KP2G,
  KGridUpdate,
  KG2P,
  KNumKernels
};

// the NVRTC-specialised kernels of one layout and their launch configuration
struct StepJit {
  CUfunction bin_count, p2g, g2p, append;
  int num_sms;
  unsigned p2g_ctas, g2p_ctas, p2g_threads, g2p_threads;
  size_t p2g_smem, g2p_smem;
};

// one hook per kernel so the runtime can bracket launches with events
typedef void (*KernelHook)(void* user, int kernel_id, int begin);

// kernels launch_step launches per step (a one-tile block table fuses the sort front)
int step_launches(const StepBuffers& B);
// whole step (single GPU)
cudaError_t launch_step(int dim, const StepBuffers& B, const SimDev& S, const MigDev& M, const StepJit& J,
                        cudaStream_t st, KernelHook hook, void* user);
// the step's phases, for the slab decomposition (exchanges in between); part: 0 all
// active blocks, 1 those below the top owned block plane, 2 the top plane
cudaError_t launch_sort(int dim, const StepBuffers& B, const SimDev& S, cudaStream_t st, KernelHook hook, void* user);
cudaError_t launch_p2g(const StepBuffers& B, const SimDev& S, const StepJit& J, int part, cudaStream_t st,
                       KernelHook hook, void* user);
cudaError_t launch_grid_update(int dim, const StepBuffers& B, const SimDev& S, const StepJit& J, cudaStream_t st,
                               KernelHook hook, void* user);
cudaError_t launch_g2p(const StepBuffers& B, const SimDev& S, const MigDev& M, const StepJit& J, int part,
                       cudaStream_t st, KernelHook hook, void* user);
// keys (+ optional histogram) of records [first, first + n); slab: routes out-of-slab records
cudaError_t launch_bin_count(const uint32_t* rec, const uint32_t* ids, uint32_t first, uint32_t n, const SimDev& S,
                             uint32_t* key, uint32_t* block_count, uint32_t* cell_count, int do_count,
                             const MigDev& M, DevCounters* dc, const StepJit& J, cudaStream_t st);
// append the arrivals of the received migration buffers (keys + histograms)
cudaError_t launch_append(uint32_t* rec, uint32_t* ids, float* dbg, uint64_t cap, const SimDev& S, uint32_t* key,
                          uint32_t* block_count, uint32_t* cell_count, const MigDev& M, DevCounters* dc,
                          const StepJit& J, cudaStream_t st);
// mode 0: pack plane bz of `nodes` into buf; 1: add buf into the plane; 2: store buf into the plane
cudaError_t launch_plane(float4* nodes, const uint32_t* block_slot, const SimDev& S, int bz, float4* buf, int mode,
                         int num_sms, cudaStream_t st);
// read_state compaction of a slab context
cudaError_t launch_live_slots(const uint32_t* dead_sorted, uint32_t n_dead, uint32_t n_slots, uint32_t* out,
                              int num_sms, cudaStream_t st);
cudaError_t launch_gather_rows(const uint32_t* src, const uint32_t* slots, uint32_t n, uint32_t row, uint32_t* dst,
                               int num_sms, cudaStream_t st);

cudaError_t launch_iota(uint32_t* ids, uint32_t n, uint32_t first, cudaStream_t st);
cudaError_t launch_count_nonfinite(const float* vals, uint64_t n, unsigned long long* out, int num_sms,
                                   cudaStream_t st);

}  // namespace qmpm
