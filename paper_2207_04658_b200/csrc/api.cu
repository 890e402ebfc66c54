// api.cu -- host runtime and C ABI of libqmpm (include/qmpm.h).
//
// Owns the device pools of one simulation context: ping-pong packed records
// (records are physically re-sorted by grid block every step: G2P writes record j
// of the sorted order), the block table of the counting sort, the grid-block pool
// and the device counters.  Everything is enqueued on the ctx stream; qmpm_step
// allocates nothing.
#include <algorithm>
#include <cstddef>
#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "comm.h"
#include "jit.h"
#include "qmpm.h"
#include "qmpm_launch.h"

using namespace qmpm;

namespace {

thread_local std::string g_err;

struct EvPair {
  int kernel;
  cudaEvent_t a, b;
};

}  // namespace

struct qmpm_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  qmpm_params P{};
  int dim = 3, material = 0, ns = 0;
  uint32_t W = 0, nf = 0;
  uint64_t seed = 0;
  LayoutDev L{};
  SimDev S{};
  CodecDev C{};  // state codec: vals in scalar order
  StepJit jit{};
  std::string jit_src;
  int jit_regs_p2g = 0, jit_regs_g2p = 0;
  uint64_t cap = 0, n = 0, step = 0;
  uint32_t* rec[2] = {nullptr, nullptr};
  int cur = 0;
  uint32_t* ids[2] = {nullptr, nullptr};
  uint32_t* key = nullptr;
  uint32_t* perm = nullptr;
  uint32_t* cell_count = nullptr;  // [nblocks * 64]
  uint32_t *block_count = nullptr, *block_start = nullptr, *block_slot = nullptr;
  uint32_t *active_list = nullptr, *touched_list = nullptr;
  uint4 *tile_sums = nullptr, *tile_off = nullptr;
  uint32_t ntiles = 0;
  uint64_t pool = 0;
  float4 *mp = nullptr, *gv = nullptr;
  DevCounters* dc = nullptr;
  float* dbg = nullptr;
  bool dbg_valid = false;
  bool binned = false;
  bool prof = false;
  std::vector<EvPair> pending;
  std::vector<cudaEvent_t> free_events;
  double ms[KNumKernels] = {0};
  uint64_t launches[KNumKernels] = {0};
  uint64_t launches_total = 0;
  std::string err;
  // slab decomposition
  bool slab = false;
  int nranks = 1, rank = 0;
  uint64_t mig_cap = 0;
  unsigned char* mig_buf[4] = {nullptr, nullptr, nullptr, nullptr};  // send down, send up, recv down, recv up
  size_t mig_bytes = 0;      // one migration buffer: header + records (+ ids), exchanged whole
  uint32_t* dead_list = nullptr;
  uint32_t dead_cap = 0;
  float4* plane_send = nullptr;
  float4* plane_recv = nullptr;
  size_t plane_elems = 0;
  cudaStream_t comm = nullptr;       // NCCL exchanges overlapping the interior P2G / G2P
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  uint32_t sticky = 0;               // device status seen by the last synchronising call
  NcclComm* nccl = nullptr;
  // single GPU: the step as a CUDA graph per ping-pong parity (QMPM_NO_GRAPH=1: launches)
  bool use_graphs = true;
  cudaGraphExec_t graph[2] = {nullptr, nullptr};
};

// kernels one single-GPU step launches (sort: 5, P2G, grid update, G2P)

namespace qmpm {
// the thread-local message qmpm_last_error(NULL) returns (used by solver.cu too)
void set_thread_error(const char* msg) { g_err = msg; }
}  // namespace qmpm

namespace {

qmpm_status fail(qmpm_ctx* ctx, qmpm_status code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  if (ctx) ctx->err = buf;
  return code;
}

#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? QMPM_ENOMEM : QMPM_ECUDA, "%s: %s (%s:%d)", \
                  #call, cudaGetErrorString(e_), __FILE__, __LINE__);                         \
  } while (0)

int n_scalars(int dim, int material) { return 2 * dim + (material == QMPM_FLUID_J ? 1 : dim * dim) + dim * dim; }

// state-scalar index of (attr, comp), or -1 if not part of this material's state
int scalar_of(int attr, int comp, int d, int material) {
  switch (attr) {
    case QMPM_X: return comp < d ? comp : -1;
    case QMPM_V: return comp < d ? d + comp : -1;
    case QMPM_F: return (material == QMPM_ELASTIC_FCR && comp < d * d) ? 2 * d + comp : -1;
    case QMPM_J: return (material == QMPM_FLUID_J && comp == 0) ? 2 * d : -1;
    case QMPM_C: return comp < d * d ? 2 * d + (material == QMPM_FLUID_J ? 1 : d * d) + comp : -1;
    default: return -1;
  }
}

// SHARED_EXP groups (reading Q4): maximal runs of consecutive SHARED_EXP fields with equal
// group ids; the first (the leader) stores the exponent in front of its mantissa.
bool group_first(const qmpm_scheme* s, uint32_t i) {
  const qmpm_field* f = s->fields;
  return f[i].kind == QMPM_SHARED_EXP &&
         (i == 0 || f[i - 1].kind != QMPM_SHARED_EXP || f[i - 1].group != f[i].group);
}
uint32_t group_start(const qmpm_scheme* s, uint32_t i) {
  while (!group_first(s, i)) --i;
  return i;
}

uint32_t field_width(const qmpm_field& f) { return f.kind == QMPM_RAW_F32 ? 32u : (uint32_t)f.frac_bits + 1u; }
uint32_t field_width_in(const qmpm_scheme* s, uint32_t i) {
  return field_width(s->fields[i]) + (group_first(s, i) ? s->fields[i].exp_bits : 0u);
}

// bit-pack layout: contiguous, LSB-first, in declaration order; layout_policy 1
// keeps every field inside one word (the bit struct's rule)
qmpm_status layout_of(qmpm_ctx* ctx, const qmpm_scheme* s, std::vector<uint32_t>& offs, uint32_t& W,
                      uint32_t& bits) {
  if (!s || !s->fields) return fail(ctx, QMPM_EINVAL, "scheme or scheme->fields is NULL");
  if (s->n_fields == 0 || s->n_fields > QMPM_MAX_FIELDS)
    return fail(ctx, QMPM_ELAYOUT, "n_fields=%u out of [1, %d]", s->n_fields, QMPM_MAX_FIELDS);
  if (s->layout_policy > 1) return fail(ctx, QMPM_ELAYOUT, "layout_policy %u not supported", s->layout_policy);
  offs.resize(s->n_fields);
  uint32_t total = 0;
  for (uint32_t i = 0; i < s->n_fields; ++i) {
    const qmpm_field& f = s->fields[i];
    if (f.kind != QMPM_FIXED && f.kind != QMPM_RAW_F32 && f.kind != QMPM_SHARED_EXP)
      return fail(ctx, QMPM_ELAYOUT, "field %u: bad kind %u", i, f.kind);
    if (f.kind == QMPM_SHARED_EXP) {  // members share b, e and R_min (a power of two); no offset
      const qmpm_field& g = s->fields[group_start(s, i)];
      int ex = 0;
      const bool pow2 = f.range > 0.0f && std::isfinite(f.range) && std::frexp(f.range, &ex) == 0.5f;
      if (f.exp_bits < 1 || f.exp_bits > 8 || f.frac_bits != g.frac_bits || f.exp_bits != g.exp_bits ||
          f.range != g.range || !pow2 || f.offset != 0.0f || (uint32_t)f.frac_bits + 1u > 24u)
        return fail(ctx, QMPM_ELAYOUT,
                    "field %u: SHARED_EXP members need equal frac_bits (<= 23), exp_bits (1..8) and a power-of-two "
                    "range, and no offset", i);
      // Delta_0 2^E must stay a normal float for E in [0, 2^e - 1]
      const int lo = (ex - 1) - (int)f.frac_bits, hi = lo + (1 << f.exp_bits) - 1;
      if (lo < -120 || hi > 120) return fail(ctx, QMPM_ELAYOUT, "field %u: SHARED_EXP range out of bounds", i);
    }
    if (f.kind == QMPM_FIXED) {
      if ((uint32_t)f.frac_bits + 1u > 32u) return fail(ctx, QMPM_ELAYOUT, "field %u: width %u > 32", i, f.frac_bits + 1u);
      if (!(f.range > 0.0f) || !std::isfinite(f.range)) return fail(ctx, QMPM_ELAYOUT, "field %u: range must be > 0", i);
      if (!std::isfinite(f.offset)) return fail(ctx, QMPM_ELAYOUT, "field %u: offset not finite", i);
    }
    const uint32_t w = field_width_in(s, i);
    // policy 1 (bit struct): a field that would straddle starts at the next word
    if (s->layout_policy == 1 && (total % 32) + w > 32) total = (total + 31) / 32 * 32;
    offs[i] = total;
    total += w;
  }
  bits = total;
  W = (total + 31) / 32;
  return QMPM_OK;
}

// `off` = the field's first bit; `lead_off` = its group leader's first bit (SHARED_EXP)
FieldDev field_dev(const qmpm_field& f, uint32_t off, uint16_t idx, uint16_t col, bool lead = false,
                   uint32_t lead_off = 0, uint16_t lead_idx = 0) {
  FieldDev d{};
  if (f.kind == QMPM_SHARED_EXP) off += lead ? f.exp_bits : 0u;  // the mantissa follows the exponent
  d.word = (uint8_t)(off / 32);
  d.shift = (uint8_t)(off % 32);
  d.width = (uint8_t)field_width(f);
  d.kind = f.kind == QMPM_RAW_F32 ? kKindRaw : (f.kind == QMPM_SHARED_EXP ? kKindShared : kKindFixed);
  if (f.kind == QMPM_SHARED_EXP) {
    d.ebits = f.exp_bits;
    d.gword = (uint8_t)(lead_off / 32);
    d.gshift = (uint8_t)(lead_off % 32);
    d.glead = lead_idx;
  }
  if (f.kind == QMPM_FIXED || f.kind == QMPM_SHARED_EXP) {
    d.delta = (float)std::ldexp((double)f.range, -(int)f.frac_bits);             // exact
    d.inv_delta = (float)(std::ldexp(1.0, (int)f.frac_bits) / (double)f.range);  // one rounding (Q3)
    d.offset = f.offset;
  } else {
    d.delta = 1.0f;
    d.inv_delta = 1.0f;
    d.offset = 0.0f;
  }
  d.idx = idx;
  d.col = col;
  return d;
}

uint32_t stage_stride(uint32_t W) { return (W % 2 == 0) ? W + 1 : W + 2; }

qmpm_status codec_of(qmpm_ctx* ctx, const qmpm_scheme* s, CodecDev& C) {
  std::vector<uint32_t> offs;
  uint32_t W, bits;
  qmpm_status rc = layout_of(ctx, s, offs, W, bits);
  if (rc) return rc;
  memset(&C, 0, sizeof(C));
  C.W = W;
  C.SW = stage_stride(W);
  C.nf = s->n_fields;
  C.stride = s->n_fields;
  C.dither = s->rounding == QMPM_DITHER;
  C.seed_lo = (uint32_t)(s->dither_seed & 0xffffffffu);
  C.seed_hi = (uint32_t)(s->dither_seed >> 32);
  for (uint32_t i = 0; i < s->n_fields; ++i) {
    const uint32_t g = s->fields[i].kind == QMPM_SHARED_EXP ? group_start(s, i) : i;
    C.f[i] = field_dev(s->fields[i], offs[i], (uint16_t)i, (uint16_t)i, g == i, offs[g], (uint16_t)g);
  }
  return QMPM_OK;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

void hook_fn(void* user, int kernel, int begin) {
  qmpm_ctx* ctx = (qmpm_ctx*)user;
  ctx->launches_total += begin ? 1 : 0;
  if (!ctx->prof) return;
  cudaEvent_t ev;
  if (ctx->free_events.empty()) {
    cudaEventCreate(&ev);
  } else {
    ev = ctx->free_events.back();
    ctx->free_events.pop_back();
  }
  cudaEventRecord(ev, ctx->stream);
  if (begin) {
    ctx->pending.push_back(EvPair{kernel, ev, nullptr});
  } else {
    ctx->pending.back().b = ev;
  }
}

qmpm_status harvest(qmpm_ctx* ctx) {
  CK(cudaStreamSynchronize(ctx->stream));
  for (auto& p : ctx->pending) {
    if (p.b) {
      float ms = 0;
      cudaEventElapsedTime(&ms, p.a, p.b);
      ctx->ms[p.kernel] += ms;
      ctx->launches[p.kernel] += 1;
      ctx->free_events.push_back(p.b);
    }
    ctx->free_events.push_back(p.a);
  }
  ctx->pending.clear();
  return QMPM_OK;
}

qmpm_status copy_in(qmpm_ctx* ctx, void* dst, const void* src, size_t bytes) {
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->stream));
  return QMPM_OK;
}

MigDev mig_of(const qmpm_ctx* ctx) {
  MigDev M{};
  M.send[0] = ctx->mig_buf[0];
  M.send[1] = ctx->mig_buf[1];
  M.recv[0] = ctx->mig_buf[2];
  M.recv[1] = ctx->mig_buf[3];
  M.dead_list = ctx->dead_list;
  M.cap = (uint32_t)ctx->mig_cap;
  M.dead_cap = ctx->dead_cap;
  M.W = ctx->W;
  M.ids = ctx->ids[0] != nullptr;
  M.dbg_ns = ctx->dbg ? (uint32_t)ctx->ns : 0u;
  return M;
}

// the record slot counters of a freshly set state: n_rec = n_slots = n, nothing dead
qmpm_status set_slot_counts(qmpm_ctx* ctx) {
  // n_rec, n_slots, n_leave, status, gstep (the scan advances gstep to this step's number)
  const uint32_t v[5] = {(uint32_t)ctx->n, (uint32_t)ctx->n, 0u, 0u, (uint32_t)ctx->step};
  static_assert(offsetof(DevCounters, n_slots) == offsetof(DevCounters, n_rec) + 4, "layout");
  static_assert(offsetof(DevCounters, n_leave) == offsetof(DevCounters, n_rec) + 8, "layout");
  static_assert(offsetof(DevCounters, gstep) == offsetof(DevCounters, n_rec) + 16, "layout");
  CK(cudaMemcpyAsync(&ctx->dc->n_rec, v, sizeof(v), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));  // (v is on the stack)
  return QMPM_OK;
}

qmpm_status clear_send_headers(qmpm_ctx* ctx) {
  for (int d = 0; d < 2; ++d) CK(cudaMemsetAsync(ctx->mig_buf[d], 0, sizeof(MigHeader), ctx->stream));
  return QMPM_OK;
}

// keys and histograms of a freshly set state; a slab rank routes the records whose base
// lies in a neighbour's slab into the send buffers (exchanged before the first sort)
qmpm_status rebin(qmpm_ctx* ctx) {
  qmpm_status rc = set_slot_counts(ctx);
  if (rc) return rc;
  CK(cudaMemsetAsync(ctx->block_count, 0, sizeof(uint32_t) * ctx->S.nblocks, ctx->stream));
  CK(cudaMemsetAsync(ctx->cell_count, 0, sizeof(uint32_t) * 64 * (size_t)ctx->S.nblocks, ctx->stream));
  if (ctx->slab && (rc = clear_send_headers(ctx))) return rc;
  hook_fn(ctx, KBinCount, 1);
  CK(launch_bin_count(ctx->rec[ctx->cur], ctx->ids[ctx->cur], 0u, (uint32_t)ctx->n, ctx->S, ctx->key,
                      ctx->block_count, ctx->cell_count, 1, mig_of(ctx), ctx->dc, ctx->jit, ctx->stream));
  hook_fn(ctx, KBinCount, 0);
  ctx->binned = true;
  return QMPM_OK;
}

qmpm_status reset_counters(qmpm_ctx* ctx) {
  CK(cudaMemsetAsync(ctx->dc, 0, sizeof(DevCounters), ctx->stream));
  ctx->sticky = 0;
  return QMPM_OK;
}

// The standalone codec through its NVRTC-specialised kernels (codec_kernels.cuh).
// op 0: vals -> words (keys: nullable => RNE), op 1: words -> vals, op 2: matmul3.
qmpm_status codec_run(qmpm_ctx* ctx, const CodecDev& C, int op, uint64_t n, const float* vals_in, float* vals_out,
                      const uint32_t* keys, uint32_t salt, const uint32_t* words_in, uint32_t* words_out,
                      unsigned long long* counters, const float* mat, cudaStream_t st) {
  if (n == 0) return QMPM_OK;
  auto vec = [](uint32_t count, const void* p) {
    const uintptr_t a = (uintptr_t)p;
    if (count % 4 == 0 && a % 16 == 0) return 4;
    if (count % 2 == 0 && a % 8 == 0) return 2;
    return 1;
  };
  const void* wp = op == 0 ? (const void*)words_out : (const void*)words_in;
  int wv = vec(C.W, wp);
  if (op == 2) wv = std::min(wv, vec(C.W, words_out));
  const void* vp = op == 0 ? (const void*)vals_in : (const void*)vals_out;
  const int vv = op == 2 ? 1 : vec(C.stride, vp);
  const bool dither = C.dither && keys != nullptr && op != 1;
  const bool counters_on = counters != nullptr && op == 0;
  CodecJit J;
  std::string err;
  cudaError_t e = jit_codec(codec_spec_source(C, dither, counters_on, wv, vv), J, err);
  if (e) return fail(ctx, QMPM_ECUDA, "codec specialisation failed: %s", err.c_str());
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t want = (n + 255) / 256;
  const unsigned grid = (unsigned)std::min<uint64_t>(want, (uint64_t)sms * 8);
  if (op == 0) {
    void* args[] = {(void*)&vals_in, (void*)&keys, (void*)&n, (void*)&salt, (void*)&words_out, (void*)&counters};
    e = jit_launch(J.encode, grid, 256, 0, st, args);
  } else if (op == 1) {
    void* args[] = {(void*)&words_in, (void*)&n, (void*)&vals_out};
    e = jit_launch(J.decode, grid, 256, 0, st, args);
  } else {
    struct {
      float a[9];
    } A;
    for (int i = 0; i < 9; ++i) A.a[i] = mat[i];
    void* args[] = {(void*)&words_in, (void*)&n, (void*)&A, (void*)&keys, (void*)&salt, (void*)&words_out};
    e = jit_launch(J.matmul3, grid, 256, 0, st, args);
  }
  if (e) return fail(ctx, QMPM_ECUDA, "codec kernel launch failed");
  return QMPM_OK;
}

// encode n scalar-order rows (host or device) into records [first, first+n) at step 0
qmpm_status encode_rows(qmpm_ctx* ctx, uint64_t first, uint64_t n, const float* vals) {
  if (n == 0) return QMPM_OK;
  const float* dv = vals;
  float* tmp = nullptr;
  if (!is_device_ptr(vals)) {
    CK(cudaMallocAsync((void**)&tmp, sizeof(float) * ctx->ns * n, ctx->stream));
    CK(cudaMemcpyAsync(tmp, vals, sizeof(float) * ctx->ns * n, cudaMemcpyDefault, ctx->stream));
    dv = tmp;
  }
  ctx->launches_total += 2;
  CK(launch_count_nonfinite(dv, n * (uint64_t)ctx->ns, &ctx->dc->nonfinite, ctx->jit.num_sms, ctx->stream));
  qmpm_status rc = codec_run(ctx, ctx->C, 0, n, dv, nullptr, nullptr, 0u, nullptr, ctx->rec[ctx->cur] + first * ctx->W,
                             (unsigned long long*)ctx->dc, nullptr, ctx->stream);
  if (rc) return rc;
  if (ctx->ids[ctx->cur]) {
    ctx->launches_total += 1;
    CK(launch_iota(ctx->ids[ctx->cur] + first, (uint32_t)n, (uint32_t)first, ctx->stream));
  }
  if (tmp) CK(cudaFreeAsync(tmp, ctx->stream));
  return QMPM_OK;
}

}  // namespace

namespace qmpm {
// the scheme -> CodecDev translation of the standalone codec, for smoke.cu
qmpm_status codec_dev_of(const qmpm_scheme* s, CodecDev& C) { return codec_of(nullptr, s, C); }
}  // namespace qmpm

extern "C" {

int qmpm_abi_version(void) { return QMPM_ABI_VERSION; }

const char* qmpm_last_error(const qmpm_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

const char* qmpm_kernel_name(int i) {
  static const char* names[KNumKernels] = {"bin_count", "scan_reduce", "scan_tiles",  "scan_apply", "cell_scan",
                                           "bin_scatter", "p2g",       "grid_update", "g2p"};
  return (i >= 0 && i < KNumKernels) ? names[i] : "";
}

uint64_t qmpm_launch_count(const qmpm_ctx* ctx) { return ctx ? ctx->launches_total : 0; }

qmpm_status qmpm_layout(const qmpm_scheme* scheme, uint32_t* words_per_particle, uint32_t* bits_used,
                        uint32_t* bit_offsets) {
  qmpm_ctx* ctx = nullptr;
  std::vector<uint32_t> offs;
  uint32_t W, bits;
  qmpm_status rc = layout_of(ctx, scheme, offs, W, bits);
  if (rc) return rc;
  if (words_per_particle) *words_per_particle = W;
  if (bits_used) *bits_used = bits;
  if (bit_offsets)
    for (size_t i = 0; i < offs.size(); ++i) bit_offsets[i] = offs[i];
  return QMPM_OK;
}

qmpm_status qmpm_destroy(qmpm_ctx* ctx) {
  if (!ctx) return QMPM_OK;
  cudaStreamSynchronize(ctx->stream);
  void* ptrs[] = {ctx->rec[0], ctx->rec[1], ctx->ids[0], ctx->ids[1], ctx->key, ctx->perm, ctx->cell_count,
                  ctx->block_count, ctx->block_start, ctx->block_slot, ctx->active_list, ctx->touched_list,
                  ctx->tile_sums, ctx->tile_off, ctx->mp, ctx->gv, ctx->dc, ctx->dbg};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  void* sptrs[] = {ctx->mig_buf[0], ctx->mig_buf[1], ctx->mig_buf[2], ctx->mig_buf[3], ctx->dead_list,
                   ctx->plane_send, ctx->plane_recv};
  for (void* p : sptrs)
    if (p) cudaFree(p);
  for (auto e : ctx->ev)
    if (e) cudaEventDestroy(e);
  for (auto g : ctx->graph)
    if (g) cudaGraphExecDestroy(g);
  if (ctx->comm) cudaStreamDestroy(ctx->comm);
  if (ctx->nccl) nccl_destroy(ctx->nccl);
  for (auto& p : ctx->pending) {
    cudaEventDestroy(p.a);
    if (p.b) cudaEventDestroy(p.b);
  }
  for (auto e : ctx->free_events) cudaEventDestroy(e);
  delete ctx;
  return QMPM_OK;
}

}  // extern "C"

namespace {
// qmpm_create, and qmpm_create_slab with `slab` set: the block table then covers the
// rank's own block planes plus the ghost plane above (table-local block ids)
// (Re)allocate a slab ctx's migration buffers for `cap` particles per direction.
static cudaError_t alloc_migration(qmpm_ctx* ctx, uint64_t cap) {
  for (int b = 0; b < 4; ++b)
    if (ctx->mig_buf[b]) {
      cudaFree(ctx->mig_buf[b]);
      ctx->mig_buf[b] = nullptr;
    }
  if (ctx->dead_list) {
    cudaFree(ctx->dead_list);
    ctx->dead_list = nullptr;
  }
  ctx->mig_cap = cap;
  ctx->dead_cap = (uint32_t)std::min<uint64_t>(2 * ctx->mig_cap, 0xffffffffull);
  ctx->mig_bytes = mig_bytes_of(mig_of(ctx));
  cudaError_t e = cudaSuccess;
  for (int b = 0; b < 4 && !e; ++b) e = cudaMalloc((void**)&ctx->mig_buf[b], ctx->mig_bytes);
  if (!e) e = cudaMalloc((void**)&ctx->dead_list, sizeof(uint32_t) * ctx->dead_cap);
  for (int b = 0; b < 4 && !e; ++b) e = cudaMemsetAsync(ctx->mig_buf[b], 0, sizeof(MigHeader), ctx->stream);
  if (!e) e = cudaStreamSynchronize(ctx->stream);
  return e;
}

qmpm_status create_impl(const qmpm_params* params, const qmpm_scheme* scheme, void* cuda_stream,
                        const qmpm_slab* slab, qmpm_ctx** out) {
  qmpm_ctx* ctx = nullptr;
  if (!params || !scheme || !out) return fail(ctx, QMPM_EINVAL, "NULL argument to qmpm_create");
  *out = nullptr;
  const int d = (int)scheme->dim;
  if (d != 2 && d != 3) return fail(ctx, QMPM_EINVAL, "dim must be 2 or 3 (got %d)", d);
  if (scheme->material != QMPM_ELASTIC_FCR && scheme->material != QMPM_FLUID_J)
    return fail(ctx, QMPM_EINVAL, "bad material %u", scheme->material);
  if (scheme->rounding != QMPM_RNE && scheme->rounding != QMPM_DITHER)
    return fail(ctx, QMPM_EINVAL, "bad rounding %u", scheme->rounding);
  std::vector<uint32_t> offs;
  uint32_t W, bits;
  qmpm_status rc = layout_of(ctx, scheme, offs, W, bits);
  if (rc) return rc;
  const int ns = n_scalars(d, (int)scheme->material);
  if ((int)scheme->n_fields != ns)
    return fail(ctx, QMPM_ELAYOUT, "scheme has %u fields; dim %d material %u needs exactly %d", scheme->n_fields, d,
                scheme->material, ns);
  std::vector<int> seen(ns, -1);
  for (uint32_t i = 0; i < scheme->n_fields; ++i) {
    const qmpm_field& f = scheme->fields[i];
    const int s = scalar_of(f.attr, f.comp, d, (int)scheme->material);
    if (s < 0) return fail(ctx, QMPM_ELAYOUT, "field %u: attr %u comp %u not in the state", i, f.attr, f.comp);
    if (seen[s] >= 0) return fail(ctx, QMPM_ELAYOUT, "fields %d and %u store the same scalar", seen[s], i);
    seen[s] = (int)i;
  }
  const qmpm_params& P = *params;
  for (int a = 0; a < d; ++a)
    if (P.grid_res[a] < 4 || P.grid_res[a] > (1 << 20))
      return fail(ctx, QMPM_EINVAL, "grid_res[%d]=%d out of range", a, P.grid_res[a]);
  if (!(P.dx > 0) || !(P.dt > 0) || !(P.p_rho > 0) || !(P.p_vol > 0))
    return fail(ctx, QMPM_EINVAL, "dx, dt, p_rho, p_vol must be > 0");
  if (P.max_particles >= 0xffffffffull) return fail(ctx, QMPM_EINVAL, "max_particles must be < 2^32 - 1");
  if (scheme->material == QMPM_ELASTIC_FCR && !(P.nu > -1.0f && P.nu < 0.5f))
    return fail(ctx, QMPM_EINVAL, "nu must be in (-1, 0.5)");

  ctx = new qmpm_ctx();
  ctx->stream = (cudaStream_t)cuda_stream;
  ctx->P = P;
  ctx->dim = d;
  ctx->material = (int)scheme->material;
  ctx->ns = ns;
  ctx->W = W;
  ctx->nf = scheme->n_fields;
  ctx->seed = scheme->dither_seed;
  ctx->cap = P.max_particles;
  cudaGetDevice(&ctx->device);
  {
    const char* ng = getenv("QMPM_NO_GRAPH");
    ctx->use_graphs = !(ng && *ng && *ng != '0');
  }

  // MPM layout (fields by state scalar) and the state codec (vals in scalar order)
  LayoutDev& L = ctx->L;
  L.W = W;
  L.SW = stage_stride(W);
  L.ns = (uint32_t)ns;
  L.dither = scheme->rounding == QMPM_DITHER;
  L.counters = (P.flags & QMPM_NO_ROUND_COUNTERS) ? 0u : 1u;
  L.ranges = (P.flags & QMPM_RECORD_RANGES) ? 1u : 0u;
  L.seed_lo = (uint32_t)(scheme->dither_seed & 0xffffffffu);
  L.seed_hi = (uint32_t)(scheme->dither_seed >> 32);
  L.xword_mask = 0;
  CodecDev& C = ctx->C;
  memset(&C, 0, sizeof(C));
  C.W = W;
  C.SW = L.SW;
  C.nf = scheme->n_fields;
  C.stride = (uint32_t)ns;
  C.dither = 0;
  for (uint32_t i = 0; i < scheme->n_fields; ++i) {
    const qmpm_field& f = scheme->fields[i];
    const int s = scalar_of(f.attr, f.comp, d, (int)scheme->material);
    const uint32_t g = f.kind == QMPM_SHARED_EXP ? group_start(scheme, i) : i;
    const qmpm_field& fg = scheme->fields[g];
    const int sg = scalar_of(fg.attr, fg.comp, d, (int)scheme->material);
    // the MPM layout indexes by state scalar: its group leader is the leader's scalar
    L.s[s] = field_dev(f, offs[i], (uint16_t)i, (uint16_t)s, g == i, offs[g], (uint16_t)sg);
    C.f[i] = field_dev(f, offs[i], (uint16_t)i, (uint16_t)s, g == i, offs[g], (uint16_t)g);
    if (f.attr == QMPM_X) {
      const uint32_t w0 = offs[i] / 32, w1 = (offs[i] + field_width_in(scheme, i) - 1) / 32;
      for (uint32_t w = w0; w <= w1; ++w) L.xword_mask |= 1u << w;
    }
  }

  // scene constants
  SimDev& S = ctx->S;
  const int B = d == 3 ? 4 : 8;
  uint64_t nblocks = 1;
  for (int a = 0; a < 3; ++a) {
    S.res[a] = a < d ? P.grid_res[a] : 1;
    S.nb[a] = a < d ? (P.grid_res[a] + B - 1) / B : 1;
    S.g[a] = a < d ? P.gravity[a] : 0.0f;
  }
  S.slab_bz0 = 0;
  S.slab_bz1 = S.nb[2];
  S.slab_lo = 0;
  S.slab_hi = 0;
  if (slab) {
    S.slab_bz0 = slab->z0 / 4;
    S.slab_bz1 = (slab->z1 + 3) / 4;
    S.slab_lo = slab->rank > 0;
    S.slab_hi = slab->rank + 1 < slab->nranks;
  }
  S.tab_bz0 = S.slab_bz0;
  S.tab_bz1 = std::min(S.slab_bz1 + (S.slab_hi ? 1 : 0), S.nb[2]);
  nblocks = (uint64_t)S.nb[0] * S.nb[1] * (uint64_t)(d == 3 ? S.tab_bz1 - S.tab_bz0 : 1);
  if (nblocks >= 0xffffffffull) {
    qmpm_destroy(ctx);
    return fail(nullptr, QMPM_EINVAL, "grid has too many blocks");
  }
  S.nblocks = (uint32_t)nblocks;
  S.dx = P.dx;
  S.inv_dx = (float)(1.0 / (double)P.dx);
  S.dt = P.dt;
  S.p_mass = (float)((double)P.p_rho * (double)P.p_vol);
  S.stress_scale = (float)(-(double)P.dt * (double)P.p_vol * 4.0 / ((double)P.dx * (double)P.dx));
  S.mu = (float)((double)P.E / (2.0 * (1.0 + (double)P.nu)));
  S.lambda = (float)((double)P.E * (double)P.nu / ((1.0 + (double)P.nu) * (1.0 - 2.0 * (double)P.nu)));
  S.E = P.E;
  S.bound = P.bound;
  S.seed_lo = L.seed_lo;
  S.seed_hi = L.seed_hi;

  ctx->ntiles = (uint32_t)((nblocks + kScanTile - 1) / kScanTile);
  ctx->pool = P.pool_blocks ? P.pool_blocks : std::min<uint64_t>(nblocks, 4096 + P.max_particles / 256);
  if (ctx->pool > nblocks) ctx->pool = nblocks;

  const size_t cap = (size_t)ctx->cap;
#define ALLOC(ptr, bytes)                                                                     \
  do {                                                                                        \
    cudaError_t e_ = cudaMalloc((void**)&(ptr), (bytes) ? (bytes) : 16);                      \
    if (e_ != cudaSuccess) {                                                                  \
      cudaGetLastError();                                                                     \
      qmpm_destroy(ctx);                                                                      \
      return fail(nullptr, QMPM_ENOMEM, "cudaMalloc(%s, %zu bytes): %s", #ptr, (size_t)(bytes), \
                  cudaGetErrorString(e_));                                                    \
    }                                                                                         \
  } while (0)
  ALLOC(ctx->rec[0], sizeof(uint32_t) * (cap * W + 1));
  ALLOC(ctx->rec[1], sizeof(uint32_t) * (cap * W + 1));
  if (P.flags & QMPM_TRACK_IDS) {
    ALLOC(ctx->ids[0], sizeof(uint32_t) * cap);
    ALLOC(ctx->ids[1], sizeof(uint32_t) * cap);
  }
  ALLOC(ctx->key, sizeof(uint32_t) * cap);
  ALLOC(ctx->perm, sizeof(uint32_t) * cap);
  ALLOC(ctx->cell_count, sizeof(uint32_t) * 64 * nblocks);
  ALLOC(ctx->block_count, sizeof(uint32_t) * nblocks);
  ALLOC(ctx->block_start, sizeof(uint32_t) * (nblocks + 1));
  ALLOC(ctx->block_slot, sizeof(uint32_t) * nblocks);
  ALLOC(ctx->active_list, sizeof(uint32_t) * nblocks);
  ALLOC(ctx->touched_list, sizeof(uint32_t) * ctx->pool);
  ALLOC(ctx->tile_sums, sizeof(uint4) * ctx->ntiles);
  ALLOC(ctx->tile_off, sizeof(uint4) * ctx->ntiles);
  ALLOC(ctx->mp, sizeof(float4) * 64 * ctx->pool);
  ALLOC(ctx->gv, sizeof(float4) * 64 * ctx->pool);
  ALLOC(ctx->dc, sizeof(DevCounters));
  if (P.flags & QMPM_DEBUG_PREENCODE) ALLOC(ctx->dbg, sizeof(float) * cap * ns);
#undef ALLOC
  cudaError_t e = cudaMemsetAsync(ctx->mp, 0, sizeof(float4) * 64 * ctx->pool, ctx->stream);
  if (!e) e = cudaMemsetAsync(ctx->block_count, 0, sizeof(uint32_t) * nblocks, ctx->stream);
  if (!e) e = cudaMemsetAsync(ctx->cell_count, 0, sizeof(uint32_t) * 64 * nblocks, ctx->stream);
  if (!e) e = cudaMemsetAsync(ctx->dc, 0, sizeof(DevCounters), ctx->stream);
  if (!e) e = cudaMemsetAsync(ctx->rec[0], 0, sizeof(uint32_t) * (cap * W + 1), ctx->stream);
  if (!e) e = cudaMemsetAsync(ctx->rec[1], 0, sizeof(uint32_t) * (cap * W + 1), ctx->stream);
  if (!e) e = cudaStreamSynchronize(ctx->stream);
  if (e) {
    qmpm_destroy(ctx);
    return fail(nullptr, QMPM_ECUDA, "qmpm_create: %s", cudaGetErrorString(e));
  }
  // specialise the step kernels on this layout (NVRTC, sm_100a)
  {
    constexpr int kP2GWarps = 2, kG2PWarps = 4;  // P2G: 64 lanes = the 64 cells of a block
    // minimum resident CTAs per SM the kernels are compiled for (register cap);
    // QMPM_P2G_MINB / QMPM_G2P_MINB override the defaults for tuning runs
    auto env_int = [](const char* name, int dflt) {
      const char* v = getenv(name);
      return (v && *v) ? atoi(v) : dflt;
    };
    // (3D elastic G2P holds F and C: 3 CTAs x 168 registers beat 4 x 128 with spills;
    // P2G: 6 CTAs x 168 registers -- at 5 ptxas also stops at 168 but spills 20 bytes
    // (measured equal, 7.33 ms at C4), at 7 it spills heavily (14.7 ms))
    const int kP2GMinBlocks = env_int("QMPM_P2G_MINB", 6),
              kG2PMinBlocks = env_int("QMPM_G2P_MINB", (d == 3 && ctx->material == QMPM_ELASTIC_FCR) ? 3 : 4);
    const int xk = env_int("QMPM_FLOAT_KEY", 0) ? 0 : integer_key_shift(d, ctx->L, S.inv_dx);
    ctx->jit_src = spec_source(d, ctx->material, ctx->L, kP2GWarps, kG2PWarps, kP2GMinBlocks, kG2PMinBlocks, xk,
                               slab != nullptr && slab->nranks > 1);
    JitModule m;
    std::string jerr;
    e = jit_get(ctx->jit_src, m, jerr);
    if (e) {
      qmpm_destroy(ctx);
      return fail(nullptr, QMPM_ECUDA, "kernel specialisation failed: %s", jerr.c_str());
    }
    StepJit& J = ctx->jit;
    J.bin_count = m.bin_count;
    J.p2g = m.p2g;
    J.g2p = m.g2p;
    J.append = m.append;
    ctx->jit_regs_p2g = m.regs_p2g;
    ctx->jit_regs_g2p = m.regs_g2p;
    cudaDeviceGetAttribute(&J.num_sms, cudaDevAttrMultiProcessorCount, ctx->device);
    J.p2g_threads = kP2GWarps * 32;
    J.g2p_threads = kG2PWarps * 32;
    J.p2g_smem = (size_t)m.smem_warp_p2g * kP2GWarps;
    J.g2p_smem = (size_t)m.smem_warp_g2p * kG2PWarps;
    e = jit_set_smem(J.p2g, J.p2g_smem);
    if (!e) e = jit_set_smem(J.g2p, J.g2p_smem);
    if (e) {
      qmpm_destroy(ctx);
      return fail(nullptr, QMPM_ECUDA, "cannot set dynamic shared memory of the step kernels");
    }
    J.p2g_ctas = (unsigned)(J.num_sms * jit_occupancy(J.p2g, (int)J.p2g_threads, J.p2g_smem));
    J.g2p_ctas = (unsigned)(J.num_sms * jit_occupancy(J.g2p, (int)J.g2p_threads, J.g2p_smem));
  }
  if (slab) {
    ctx->slab = true;
    ctx->nranks = slab->nranks;
    ctx->rank = slab->rank;
    // steady state at C4: ~1.5M particles per cell plane, a few % cross a slab face per
    // step; the first step may route up to half a plane (particles loaded by position)
    ctx->mig_cap = slab->migrate_capacity ? slab->migrate_capacity
                                          : std::max<uint64_t>(65536, std::min<uint64_t>(ctx->cap / 256, 1u << 22));
    ctx->plane_elems = (size_t)S.nb[0] * S.nb[1] * 64;
    cudaError_t e2 = alloc_migration(ctx, ctx->mig_cap);
    if (!e2) e2 = cudaMalloc((void**)&ctx->plane_send, sizeof(float4) * ctx->plane_elems);
    if (!e2) e2 = cudaMalloc((void**)&ctx->plane_recv, sizeof(float4) * ctx->plane_elems);
    if (!e2) e2 = cudaMemsetAsync(ctx->plane_recv, 0, sizeof(float4) * ctx->plane_elems, ctx->stream);
    if (!e2) e2 = cudaStreamCreateWithFlags(&ctx->comm, cudaStreamNonBlocking);
    for (int b = 0; b < 4 && !e2; ++b) e2 = cudaEventCreateWithFlags(&ctx->ev[b], cudaEventDisableTiming);
    if (!e2) e2 = cudaStreamSynchronize(ctx->stream);
    if (e2) {
      cudaGetLastError();
      qmpm_destroy(ctx);
      return fail(nullptr, e2 == cudaErrorMemoryAllocation ? QMPM_ENOMEM : QMPM_ECUDA, "qmpm_create_slab: %s",
                  cudaGetErrorString(e2));
    }
  }
  *out = ctx;
  return QMPM_OK;
}
}  // namespace

extern "C" {

qmpm_status qmpm_create(const qmpm_params* params, const qmpm_scheme* scheme, void* cuda_stream, qmpm_ctx** out) {
  return create_impl(params, scheme, cuda_stream, nullptr, out);
}

qmpm_status qmpm_set_state(qmpm_ctx* ctx, uint64_t n, const float* vals) {
  if (!ctx) return fail(ctx, QMPM_EINVAL, "NULL ctx");
  if (n > ctx->cap) return fail(ctx, QMPM_ECAPACITY, "n=%llu > max_particles=%llu", (unsigned long long)n,
                                (unsigned long long)ctx->cap);
  if (n && !vals) return fail(ctx, QMPM_EINVAL, "vals is NULL");
  qmpm_status rc = reset_counters(ctx);
  if (rc) return rc;
  ctx->cur = 0;
  ctx->n = 0;
  ctx->step = 0;
  ctx->dbg_valid = false;
  rc = encode_rows(ctx, 0, n, vals);
  if (rc) return rc;
  ctx->n = n;
  ctx->binned = false;
  return set_slot_counts(ctx);
}

qmpm_status qmpm_append_state(qmpm_ctx* ctx, uint64_t n, const float* vals) {
  if (!ctx) return fail(ctx, QMPM_EINVAL, "NULL ctx");
  if (ctx->n + n > ctx->cap) return fail(ctx, QMPM_ECAPACITY, "append past max_particles");
  if (n && !vals) return fail(ctx, QMPM_EINVAL, "vals is NULL");
  qmpm_status rc = encode_rows(ctx, ctx->n, n, vals);
  if (rc) return rc;
  ctx->n += n;
  ctx->binned = false;
  ctx->dbg_valid = false;
  return set_slot_counts(ctx);
}

qmpm_status qmpm_set_words(qmpm_ctx* ctx, uint64_t n, const uint32_t* words, uint64_t step) {
  if (!ctx) return fail(ctx, QMPM_EINVAL, "NULL ctx");
  if (n > ctx->cap) return fail(ctx, QMPM_ECAPACITY, "n > max_particles");
  if (n && !words) return fail(ctx, QMPM_EINVAL, "words is NULL");
  qmpm_status rc = reset_counters(ctx);
  if (rc) return rc;
  ctx->cur = 0;
  if (n) {
    rc = copy_in(ctx, ctx->rec[0], words, sizeof(uint32_t) * ctx->W * n);
    if (rc) return rc;
  }
  if (ctx->ids[0]) {
    ctx->launches_total += 1;
    CK(launch_iota(ctx->ids[0], (uint32_t)n, 0u, ctx->stream));
  }
  ctx->n = n;
  ctx->step = step;
  ctx->binned = false;
  ctx->dbg_valid = false;
  return set_slot_counts(ctx);
}

}  // extern "C"

namespace {

StepBuffers buffers(qmpm_ctx* ctx, uint64_t n) {
  StepBuffers B{};
  B.rec_in = ctx->rec[ctx->cur];
  B.rec_out = ctx->rec[ctx->cur ^ 1];
  B.ids_in = ctx->ids[ctx->cur];
  B.ids_out = ctx->ids[ctx->cur ^ 1];
  B.key = ctx->key;
  B.perm = ctx->perm;
  B.cell_count = ctx->cell_count;
  B.num_sms = ctx->jit.num_sms;
  B.block_count = ctx->block_count;
  B.block_start = ctx->block_start;
  B.block_slot = ctx->block_slot;
  B.active_list = ctx->active_list;
  B.touched_list = ctx->touched_list;
  B.tile_sums = ctx->tile_sums;
  B.tile_off = ctx->tile_off;
  B.mp = ctx->mp;
  B.gv = ctx->gv;
  B.dc = ctx->dc;
  B.dbg = ctx->dbg;
  B.n = (uint32_t)n;
  B.cap = (uint32_t)std::min<uint64_t>(ctx->cap, 0xffffffffull);
  B.pool = (uint32_t)ctx->pool;
  B.ntiles = ctx->ntiles;
  return B;
}

void finish_step(qmpm_ctx* ctx) {
  ctx->cur ^= 1;
  ctx->step += 1;
  ctx->dbg_valid = ctx->dbg != nullptr;
}

// ---------------------------------------------------------------- slab phases
// One slab step, every size fixed so the exchange schedule never depends
// on data and the host never waits for the device:
//   sort                                   (slots [0, n_slots): owned + arrived particles)
//   P2G top block plane -> pack ghost plane -> [ghost exchange, comm stream]
//   P2G interior (overlaps the exchange) -> add the lower rank's ghost plane
//   grid update -> pack bottom plane velocities -> [velocity exchange, comm stream]
//   G2P interior (overlaps the exchange) -> store the upper rank's velocities -> G2P top
//     (particles whose new base lies in a neighbour's slab are copied to a send buffer)
//   [migration exchange + status all-reduce] -> append the arrivals (keys, histograms)
// The first step after set_state / set_words routes the records loaded outside the slab
// the same way (bin_count + migration) before its sort.

// transport of one exchange kind between the z-neighbours
enum XKind { XGhost = 0, XVel = 1, XMig = 2 };

qmpm_status nccl_x(qmpm_ctx* ctx, XKind k, cudaStream_t st) {
  std::string err;
  const size_t pb = ctx->plane_elems * sizeof(float4);
  P2P x{};
  if (k == XGhost) {  // partial sums of the ghost plane go up
    x = P2P{nullptr, 0, ctx->plane_send, ctx->S.slab_hi ? pb : 0, ctx->plane_recv, ctx->S.slab_lo ? pb : 0, nullptr, 0};
  } else if (k == XVel) {  // bottom plane velocities go down
    x = P2P{ctx->plane_send, ctx->S.slab_lo ? pb : 0, nullptr, 0, nullptr, 0, ctx->plane_recv, ctx->S.slab_hi ? pb : 0};
  } else {
    const size_t mb = ctx->mig_bytes;
    x = P2P{ctx->mig_buf[0], ctx->S.slab_lo ? mb : 0, ctx->mig_buf[1], ctx->S.slab_hi ? mb : 0,
            ctx->mig_buf[2], ctx->S.slab_lo ? mb : 0, ctx->mig_buf[3], ctx->S.slab_hi ? mb : 0};
  }
  if (!nccl_exchange(ctx->nccl, x, st, err)) return fail(ctx, QMPM_ENCCL, "%s", err.c_str());
  if (k == XMig && !nccl_allreduce_max_u32(ctx->nccl, &ctx->dc->status, st, err))
    return fail(ctx, QMPM_ENCCL, "%s", err.c_str());
  return QMPM_OK;
}

qmpm_status append_arrivals(qmpm_ctx* ctx) {
  if (!ctx->S.slab_lo) CK(cudaMemsetAsync(ctx->mig_buf[2], 0, sizeof(MigHeader), ctx->stream));
  if (!ctx->S.slab_hi) CK(cudaMemsetAsync(ctx->mig_buf[3], 0, sizeof(MigHeader), ctx->stream));
  ctx->launches_total += 1;
  CK(launch_append(ctx->rec[ctx->cur], ctx->ids[ctx->cur], ctx->dbg, ctx->cap, ctx->S, ctx->key, ctx->block_count,
                   ctx->cell_count, mig_of(ctx), ctx->dc, ctx->jit, ctx->stream));
  return QMPM_OK;
}

// the per-rank phases of one step; `x(kind, stream)` performs one exchange for this rank
// (NCCL), or is null for the in-process group (its driver copies between the phases)
struct SlabPhases {
  qmpm_ctx* ctx;
  // (first step) keys, routing of out-of-slab records
  qmpm_status pre() {
    if (ctx->binned) return QMPM_OK;
    return rebin(ctx);
  }
  qmpm_status sort() {
    StepBuffers B = buffers(ctx, ctx->n);
    CK(launch_sort(ctx->dim, B, ctx->S, ctx->stream, hook_fn, ctx));
    return QMPM_OK;
  }
  // P2G; with `overlap` the top plane first, its ghost plane handed to the exchange
  qmpm_status p2g(bool overlap) {
    StepBuffers B = buffers(ctx, ctx->n);
    if (!overlap) {
      CK(launch_p2g(B, ctx->S, ctx->jit, 0, ctx->stream, hook_fn, ctx));
      if (ctx->S.slab_hi) {
        ctx->launches_total += 1;
        CK(launch_plane(ctx->mp, ctx->block_slot, ctx->S, ctx->S.slab_bz1, ctx->plane_send, 0, ctx->jit.num_sms, ctx->stream));
      }
      return QMPM_OK;
    }
    CK(launch_p2g(B, ctx->S, ctx->jit, 2, ctx->stream, hook_fn, ctx));
    if (ctx->S.slab_hi) {
      ctx->launches_total += 1;
      CK(launch_plane(ctx->mp, ctx->block_slot, ctx->S, ctx->S.slab_bz1, ctx->plane_send, 0, ctx->jit.num_sms, ctx->stream));
    }
    CK(cudaEventRecord(ctx->ev[0], ctx->stream));
    CK(cudaStreamWaitEvent(ctx->comm, ctx->ev[0], 0));
    qmpm_status rc = nccl_x(ctx, XGhost, ctx->comm);
    if (rc) return rc;
    CK(cudaEventRecord(ctx->ev[1], ctx->comm));
    CK(launch_p2g(B, ctx->S, ctx->jit, 1, ctx->stream, hook_fn, ctx));
    CK(cudaStreamWaitEvent(ctx->stream, ctx->ev[1], 0));
    return QMPM_OK;
  }
  qmpm_status grid() {
    StepBuffers B = buffers(ctx, ctx->n);
    if (ctx->S.slab_lo) {
      ctx->launches_total += 1;
      CK(launch_plane(ctx->mp, ctx->block_slot, ctx->S, ctx->S.slab_bz0, ctx->plane_recv, 1, ctx->jit.num_sms, ctx->stream));
    }
    CK(launch_grid_update(ctx->dim, B, ctx->S, ctx->jit, ctx->stream, hook_fn, ctx));
    if (ctx->S.slab_lo) {
      ctx->launches_total += 1;
      CK(launch_plane(ctx->gv, ctx->block_slot, ctx->S, ctx->S.slab_bz0, ctx->plane_send, 0, ctx->jit.num_sms, ctx->stream));
    }
    return QMPM_OK;
  }
  qmpm_status g2p(bool overlap) {
    StepBuffers B = buffers(ctx, ctx->n);
    qmpm_status rc = clear_send_headers(ctx);
    if (rc) return rc;
    auto store_ghost = [&]() -> qmpm_status {
      if (ctx->S.slab_hi) {
        ctx->launches_total += 1;
        CK(launch_plane(ctx->gv, ctx->block_slot, ctx->S, ctx->S.slab_bz1, ctx->plane_recv, 2, ctx->jit.num_sms, ctx->stream));
      }
      return QMPM_OK;
    };
    if (!overlap) {
      if ((rc = store_ghost())) return rc;
      CK(launch_g2p(B, ctx->S, mig_of(ctx), ctx->jit, 0, ctx->stream, hook_fn, ctx));
      return QMPM_OK;
    }
    CK(cudaEventRecord(ctx->ev[2], ctx->stream));
    CK(cudaStreamWaitEvent(ctx->comm, ctx->ev[2], 0));
    if ((rc = nccl_x(ctx, XVel, ctx->comm))) return rc;
    CK(cudaEventRecord(ctx->ev[3], ctx->comm));
    CK(launch_g2p(B, ctx->S, mig_of(ctx), ctx->jit, 1, ctx->stream, hook_fn, ctx));
    CK(cudaStreamWaitEvent(ctx->stream, ctx->ev[3], 0));
    if ((rc = store_ghost())) return rc;
    CK(launch_g2p(B, ctx->S, mig_of(ctx), ctx->jit, 2, ctx->stream, hook_fn, ctx));
    return QMPM_OK;
  }
};

// one slab step with NCCL exchanges (one process per GPU), no host synchronisation
qmpm_status slab_step_nccl(qmpm_ctx* ctx) {
  SlabPhases ph{ctx};
  qmpm_status rc;
  if (!ctx->binned) {
    if ((rc = ph.pre())) return rc;
    if ((rc = nccl_x(ctx, XMig, ctx->stream))) return rc;
    if ((rc = append_arrivals(ctx))) return rc;
  }
  if ((rc = ph.sort())) return rc;
  if ((rc = ph.p2g(true))) return rc;
  if ((rc = ph.grid())) return rc;
  if ((rc = ph.g2p(true))) return rc;
  finish_step(ctx);
  if ((rc = nccl_x(ctx, XMig, ctx->stream))) return rc;
  return append_arrivals(ctx);
}

// sticky device status -> error code (the ctx stays in error until set_state / set_words)
qmpm_status status_error(qmpm_ctx* ctx, uint32_t st) {
  if (st & kStatusTwoHop)
    return fail(ctx, QMPM_EDOMAIN, "a particle moved more than one slab in one step (CFL violated)");
  if (st & kStatusMigOverflow)
    return fail(ctx, QMPM_ECAPACITY, "slab migration buffer overflow (capacity %llu per direction)",
                (unsigned long long)ctx->mig_cap);
  if (st & kStatusCapacity) return fail(ctx, QMPM_ECAPACITY, "arrivals exceed max_particles");
  if (st & kStatusNonfinite)
    return fail(ctx, QMPM_ENONFINITE, "non-finite values were encoded (as code 0; S:42): see qmpm_stats.nonfinite");
  return QMPM_OK;
}

}  // namespace

extern "C" {

qmpm_status qmpm_step(qmpm_ctx* ctx, uint32_t n_steps) {
  if (!ctx) return fail(ctx, QMPM_EINVAL, "NULL ctx");
  if (ctx->sticky) return fail(ctx, QMPM_ESTATE, "the ctx is in error (%u): set_state or set_words first", ctx->sticky);
  if (ctx->slab && ctx->nranks > 1) {
    if (!ctx->nccl) return fail(ctx, QMPM_ESTATE, "slab ctx: call qmpm_connect_nccl or use qmpm_step_group");
    for (uint32_t t = 0; t < n_steps; ++t) {
      qmpm_status rc = slab_step_nccl(ctx);
      if (rc) return rc;
    }
    return QMPM_OK;
  }
  for (uint32_t t = 0; t < n_steps; ++t) {
    if (!ctx->binned) {
      qmpm_status rc = rebin(ctx);
      if (rc) return rc;
    }
    if (!ctx->prof && ctx->use_graphs && ctx->stream != nullptr && ctx->stream != cudaStreamLegacy &&
        ctx->stream != cudaStreamPerThread) {
      // one CUDA-graph launch per step: the step's launches take no per-step argument
      // (the dither salt comes from the device step counter), so one graph per ping-pong
      // parity replays for the ctx's lifetime
      cudaGraphExec_t& g = ctx->graph[ctx->cur];
      if (!g) {
        StepBuffers B = buffers(ctx, ctx->n);
        cudaGraph_t graph = nullptr;
        CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
        cudaError_t e = launch_step(ctx->dim, B, ctx->S, mig_of(ctx), ctx->jit, ctx->stream, nullptr, nullptr);
        cudaError_t e2 = cudaStreamEndCapture(ctx->stream, &graph);
        if (!e) e = e2;
        if (!e) e = cudaGraphInstantiate(&g, graph, 0);
        if (graph) cudaGraphDestroy(graph);
        if (e) {  // (e.g. a stream already being captured by the caller): plain launches
          cudaGetLastError();
          g = nullptr;
          ctx->use_graphs = false;
          StepBuffers B2 = buffers(ctx, ctx->n);
          CK(launch_step(ctx->dim, B2, ctx->S, mig_of(ctx), ctx->jit, ctx->stream, hook_fn, ctx));
          finish_step(ctx);
          continue;
        }
      }
      CK(cudaGraphLaunch(g, ctx->stream));
      ctx->launches_total += (uint64_t)step_launches(buffers(ctx, ctx->n));
    } else {
      StepBuffers B = buffers(ctx, ctx->n);
      CK(launch_step(ctx->dim, B, ctx->S, mig_of(ctx), ctx->jit, ctx->stream, hook_fn, ctx));
    }
    finish_step(ctx);
  }
  return QMPM_OK;
}

// in-process transport: the same phases, the exchanges as device copies between the ctxs
qmpm_status qmpm_step_group(qmpm_ctx* const* ctxs, int n, uint32_t n_steps) {
  qmpm_ctx* ctx = nullptr;
  if (!ctxs || n < 1) return fail(ctx, QMPM_EINVAL, "empty group");
  for (int r = 0; r < n; ++r) {
    if (!ctxs[r] || !ctxs[r]->slab || ctxs[r]->nranks != n || ctxs[r]->rank != r)
      return fail(ctx, QMPM_EINVAL, "qmpm_step_group: ctxs[%d] must be the slab ctx of rank %d of %d", r, r, n);
    if (ctxs[r]->stream != ctxs[0]->stream) return fail(ctx, QMPM_EINVAL, "qmpm_step_group: one stream for all ctxs");
    if ((ctxs[r]->ids[0] != nullptr) != (ctxs[0]->ids[0] != nullptr) || ctxs[r]->W != ctxs[0]->W)
      return fail(ctx, QMPM_EINVAL, "qmpm_step_group: ctxs differ in scheme or flags");
    if (ctxs[r]->sticky) return fail(ctxs[r], QMPM_ESTATE, "ctx %d is in error", r);
  }
  {  // one migration capacity for the group (as qmpm_connect_nccl agrees on over NCCL)
    uint64_t mc = 0;
    for (int r = 0; r < n; ++r) mc = std::max<uint64_t>(mc, ctxs[r]->mig_cap);
    for (int r = 0; r < n; ++r)
      if (ctxs[r]->mig_cap != mc) {
        const cudaError_t e = alloc_migration(ctxs[r], mc);
        if (e) return fail(ctxs[r], e == cudaErrorMemoryAllocation ? QMPM_ENOMEM : QMPM_ECUDA, "qmpm_step_group: %s",
                           cudaGetErrorString(e));
      }
  }
  cudaStream_t st = ctxs[0]->stream;
  auto copy = [&](void* dst, const void* src, size_t bytes) -> qmpm_status {
    if (cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return fail(ctx, QMPM_ECUDA, "step_group copy failed");
    return QMPM_OK;
  };
  auto migrate = [&]() -> qmpm_status {
    qmpm_status rc;
    for (int r = 0; r < n; ++r) {
      if (r > 0 && (rc = copy(ctxs[r]->mig_buf[2], ctxs[r - 1]->mig_buf[1], ctxs[r]->mig_bytes))) return rc;
      if (r + 1 < n && (rc = copy(ctxs[r]->mig_buf[3], ctxs[r + 1]->mig_buf[0], ctxs[r]->mig_bytes))) return rc;
    }
    for (int r = 0; r < n; ++r)
      if ((rc = append_arrivals(ctxs[r]))) return rc;
    return QMPM_OK;
  };
  for (uint32_t t = 0; t < n_steps; ++t) {
    qmpm_status rc;
    bool pre = false;
    for (int r = 0; r < n; ++r) {
      pre |= !ctxs[r]->binned;
      if ((rc = SlabPhases{ctxs[r]}.pre())) return rc;
    }
    if (pre && (rc = migrate())) return rc;
    for (int r = 0; r < n; ++r) {
      SlabPhases ph{ctxs[r]};
      if ((rc = ph.sort()) || (rc = ph.p2g(false))) return rc;
    }
    for (int r = 0; r + 1 < n; ++r)
      if ((rc = copy(ctxs[r + 1]->plane_recv, ctxs[r]->plane_send, ctxs[r]->plane_elems * sizeof(float4)))) return rc;
    for (int r = 0; r < n; ++r)
      if ((rc = SlabPhases{ctxs[r]}.grid())) return rc;
    for (int r = 1; r < n; ++r)
      if ((rc = copy(ctxs[r - 1]->plane_recv, ctxs[r]->plane_send, ctxs[r]->plane_elems * sizeof(float4)))) return rc;
    for (int r = 0; r < n; ++r) {
      if ((rc = SlabPhases{ctxs[r]}.g2p(false))) return rc;
      finish_step(ctxs[r]);
    }
    if ((rc = migrate())) return rc;
  }
  return QMPM_OK;
}

qmpm_status qmpm_get_unique_id(uint8_t id[128]) {
  qmpm_ctx* ctx = nullptr;
  std::string err;
  if (!id) return fail(ctx, QMPM_EINVAL, "NULL id");
  if (!nccl_unique_id(id, err)) return fail(ctx, QMPM_ENCCL, "%s", err.c_str());
  return QMPM_OK;
}

qmpm_status qmpm_connect_nccl(qmpm_ctx* ctx, const uint8_t id[128]) {
  if (!ctx || !id) return fail(ctx, QMPM_EINVAL, "NULL argument");
  if (!ctx->slab) return fail(ctx, QMPM_ESTATE, "qmpm_connect_nccl needs a slab ctx (qmpm_create_slab)");
  std::string err;
  ctx->nccl = nccl_connect(id, ctx->nranks, ctx->rank, err);
  if (!ctx->nccl) return fail(ctx, QMPM_ENCCL, "%s", err.c_str());
  // The migration exchanges are fixed-size (no host sync per step), so every rank must
  // post buffers of ONE capacity.  The default capacity follows each rank's own particle
  // capacity, which differs between slabs: agree on the largest over the ranks (one
  // all-reduce, here only) and re-size this rank's buffers to it.
  {
    unsigned int* d = nullptr;
    unsigned int v = (unsigned int)std::min<uint64_t>(ctx->mig_cap, 0xffffffffull);
    cudaError_t e = cudaMalloc((void**)&d, sizeof(unsigned int));
    if (!e) e = cudaMemcpyAsync(d, &v, sizeof(v), cudaMemcpyHostToDevice, ctx->stream);
    if (e) {
      if (d) cudaFree(d);
      return fail(ctx, QMPM_ECUDA, "qmpm_connect_nccl: %s", cudaGetErrorString(e));
    }
    if (!nccl_allreduce_max_u32(ctx->nccl, d, ctx->stream, err)) {
      cudaFree(d);
      return fail(ctx, QMPM_ENCCL, "%s", err.c_str());
    }
    e = cudaMemcpyAsync(&v, d, sizeof(v), cudaMemcpyDeviceToHost, ctx->stream);
    if (!e) e = cudaStreamSynchronize(ctx->stream);
    cudaFree(d);
    if (!e && (uint64_t)v != ctx->mig_cap) e = alloc_migration(ctx, v);
    if (e)
      return fail(ctx, e == cudaErrorMemoryAllocation ? QMPM_ENOMEM : QMPM_ECUDA, "qmpm_connect_nccl: %s",
                  cudaGetErrorString(e));
  }
  return QMPM_OK;
}

qmpm_status qmpm_create_dist(const qmpm_params* params, const qmpm_scheme* scheme, void* cuda_stream, int nranks,
                             int rank, const uint8_t id[128], const int32_t* slab_cuts, qmpm_ctx** out) {
  if (!slab_cuts || !id || !out) return fail(nullptr, QMPM_EINVAL, "NULL argument to qmpm_create_dist");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(nullptr, QMPM_EINVAL, "bad rank %d of %d", rank, nranks);
  for (int r = 0; r < nranks; ++r)
    if (slab_cuts[r] >= slab_cuts[r + 1]) return fail(nullptr, QMPM_EINVAL, "slab_cuts must increase");
  if (!params || slab_cuts[0] != 0 || slab_cuts[nranks] != params->grid_res[2])
    return fail(nullptr, QMPM_EINVAL, "slab_cuts must span [0, grid_res[2]]");
  qmpm_slab slab{};
  slab.nranks = nranks;
  slab.rank = rank;
  slab.z0 = slab_cuts[rank];
  slab.z1 = slab_cuts[rank + 1];
  qmpm_ctx* ctx = nullptr;
  qmpm_status rc = qmpm_create_slab(params, scheme, cuda_stream, &slab, &ctx);
  if (rc) return rc;
  rc = qmpm_connect_nccl(ctx, id);
  if (rc) {
    qmpm_destroy(ctx);
    return rc;
  }
  *out = ctx;
  return QMPM_OK;
}

qmpm_status qmpm_create_slab(const qmpm_params* params, const qmpm_scheme* scheme, void* cuda_stream,
                             const qmpm_slab* slab, qmpm_ctx** out) {
  qmpm_ctx* ctx = nullptr;
  if (!slab || !out) return fail(ctx, QMPM_EINVAL, "NULL argument to qmpm_create_slab");
  if (!scheme || scheme->dim != 3) return fail(ctx, QMPM_EINVAL, "slab decomposition is 3D (z slabs)");
  if (slab->nranks < 1 || slab->rank < 0 || slab->rank >= slab->nranks)
    return fail(ctx, QMPM_EINVAL, "bad rank %d of %d", slab->rank, slab->nranks);
  if (!params) return fail(ctx, QMPM_EINVAL, "NULL params");
  const int nz = params->grid_res[2];
  if (slab->z0 < 0 || slab->z1 > nz || slab->z0 >= slab->z1 || slab->z0 % 4 != 0 || (slab->z1 % 4 != 0 && slab->z1 != nz))
    return fail(ctx, QMPM_EINVAL, "slab [%d, %d) must be non-empty, inside [0, %d) and on 4-cell block planes",
                slab->z0, slab->z1, nz);
  return create_impl(params, scheme, cuda_stream, slab, out);
}

qmpm_status qmpm_set_ids(qmpm_ctx* ctx, uint64_t n, const uint32_t* ids) {
  if (!ctx) return fail(ctx, QMPM_EINVAL, "NULL ctx");
  if (!ctx->ids[ctx->cur]) return fail(ctx, QMPM_ESTATE, "qmpm_set_ids needs QMPM_TRACK_IDS");
  if (n != ctx->n) return fail(ctx, QMPM_EINVAL, "n=%llu but the ctx holds %llu particles", (unsigned long long)n,
                               (unsigned long long)ctx->n);
  if (n && !ids) return fail(ctx, QMPM_EINVAL, "ids is NULL");
  if (n) CK(cudaMemcpyAsync(ctx->ids[ctx->cur], ids, sizeof(uint32_t) * n, cudaMemcpyDefault, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return QMPM_OK;
}

}  // extern "C"

namespace {

// synchronise and read the device counters; the sticky status becomes the ctx's
qmpm_status sync_counters(qmpm_ctx* ctx, DevCounters& h) {
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaMemcpy(&h, ctx->dc, sizeof(h), cudaMemcpyDeviceToHost));
  ctx->sticky |= h.status | (h.nonfinite ? kStatusNonfinite : 0u);
  return QMPM_OK;
}

// The live record slots: [0, n_slots) minus the slots whose particle left the slab (their
// records stay until the next sort).  Without leavers the identity (`slots` = null);
// else the i-th live slot in slot order, written to ctx->perm (scratch between steps).
qmpm_status live_slots(qmpm_ctx* ctx, const DevCounters& h, const uint32_t** slots, uint64_t* n) {
  *slots = nullptr;
  *n = h.n_slots;
  if (h.n_leave == 0) return QMPM_OK;
  const uint32_t nd = std::min(h.n_leave, ctx->dead_cap);
  std::vector<uint32_t> dead(nd);
  CK(cudaMemcpy(dead.data(), ctx->dead_list, sizeof(uint32_t) * nd, cudaMemcpyDeviceToHost));
  std::sort(dead.begin(), dead.end());
  uint32_t* d_dead = nullptr;
  CK(cudaMalloc((void**)&d_dead, sizeof(uint32_t) * std::max<uint32_t>(nd, 1u)));
  cudaError_t e = cudaMemcpy(d_dead, dead.data(), sizeof(uint32_t) * nd, cudaMemcpyHostToDevice);
  if (!e) e = launch_live_slots(d_dead, nd, h.n_slots, ctx->perm, ctx->jit.num_sms, ctx->stream);
  if (!e) e = cudaStreamSynchronize(ctx->stream);
  cudaFree(d_dead);
  if (e) return fail(ctx, QMPM_ECUDA, "read_state compaction: %s", cudaGetErrorString(e));
  *slots = ctx->perm;
  *n = (uint64_t)h.n_slots - nd;
  return QMPM_OK;
}

// rows [n][row] of `src` at the live slots (identity when slots == null) -> dst (any memory)
qmpm_status gather_rows(qmpm_ctx* ctx, const uint32_t* src, const uint32_t* slots, uint64_t n, uint32_t row,
                        uint32_t* scratch, void* dst) {
  if (!n) return QMPM_OK;
  if (!slots) {
    CK(cudaMemcpyAsync(dst, src, sizeof(uint32_t) * row * n, cudaMemcpyDefault, ctx->stream));
    return QMPM_OK;
  }
  CK(launch_gather_rows(src, slots, (uint32_t)n, row, scratch, ctx->jit.num_sms, ctx->stream));
  CK(cudaMemcpyAsync(dst, scratch, sizeof(uint32_t) * row * n, cudaMemcpyDefault, ctx->stream));
  return QMPM_OK;
}

}  // namespace

extern "C" {

qmpm_status qmpm_read_state(qmpm_ctx* ctx, float* vals, uint32_t* words, uint32_t* ids, uint64_t capacity,
                            uint64_t* n_out) {
  if (!ctx) return fail(ctx, QMPM_EINVAL, "NULL ctx");
  DevCounters h;
  qmpm_status rc = sync_counters(ctx, h);
  if (rc) return rc;
  const uint32_t* slots = nullptr;
  uint64_t n = 0;
  if ((rc = live_slots(ctx, h, &slots, &n))) return rc;
  if (n_out) *n_out = n;
  if (capacity < n) return fail(ctx, QMPM_ECAPACITY, "capacity %llu < n %llu", (unsigned long long)capacity,
                                (unsigned long long)n);
  if (ids && !ctx->ids[ctx->cur]) return fail(ctx, QMPM_ESTATE, "ids requested without QMPM_TRACK_IDS");
  // the live records, gathered into the other ping-pong buffer (free between steps)
  const uint32_t* rec = ctx->rec[ctx->cur];
  if (slots && n) {
    CK(launch_gather_rows(rec, slots, (uint32_t)n, ctx->W, ctx->rec[ctx->cur ^ 1], ctx->jit.num_sms, ctx->stream));
    rec = ctx->rec[ctx->cur ^ 1];
  }
  if (vals && n) {
    float* dv = vals;
    float* tmp = nullptr;
    if (!is_device_ptr(vals)) {
      CK(cudaMallocAsync((void**)&tmp, sizeof(float) * ctx->ns * n, ctx->stream));
      dv = tmp;
    }
    ctx->launches_total += 1;
    rc = codec_run(ctx, ctx->C, 1, n, nullptr, dv, nullptr, 0u, rec, nullptr, nullptr, nullptr, ctx->stream);
    if (rc) return rc;
    if (tmp) {
      CK(cudaMemcpyAsync(vals, tmp, sizeof(float) * ctx->ns * n, cudaMemcpyDefault, ctx->stream));
      CK(cudaFreeAsync(tmp, ctx->stream));
    }
  }
  if (words && n) CK(cudaMemcpyAsync(words, rec, sizeof(uint32_t) * ctx->W * n, cudaMemcpyDefault, ctx->stream));
  if (ids && n && (rc = gather_rows(ctx, ctx->ids[ctx->cur], slots, n, 1, ctx->ids[ctx->cur ^ 1], ids))) return rc;
  CK(cudaStreamSynchronize(ctx->stream));
  if (h.overflow) return fail(ctx, QMPM_ECAPACITY, "grid pool overflow in %llu step(s): raise pool_blocks",
                              (unsigned long long)h.overflow);
  return status_error(ctx, ctx->sticky);
}

qmpm_status qmpm_read_debug(qmpm_ctx* ctx, float* pre, uint64_t capacity, uint64_t* n_out) {
  if (!ctx) return fail(ctx, QMPM_EINVAL, "NULL ctx");
  if (!ctx->dbg) return fail(ctx, QMPM_ESTATE, "QMPM_DEBUG_PREENCODE not set");
  if (!ctx->dbg_valid) return fail(ctx, QMPM_ESTATE, "no step taken since the state was set");
  DevCounters h;
  qmpm_status rc = sync_counters(ctx, h);
  if (rc) return rc;
  const uint32_t* slots = nullptr;
  uint64_t n = 0;
  if ((rc = live_slots(ctx, h, &slots, &n))) return rc;
  if (n_out) *n_out = n;
  if (capacity < n) return fail(ctx, QMPM_ECAPACITY, "capacity < n");
  uint32_t* scratch = nullptr;
  if (slots && n) CK(cudaMallocAsync((void**)&scratch, sizeof(float) * ctx->ns * n, ctx->stream));
  rc = gather_rows(ctx, reinterpret_cast<const uint32_t*>(ctx->dbg), slots, n, (uint32_t)ctx->ns, scratch, pre);
  if (scratch) CK(cudaFreeAsync(scratch, ctx->stream));
  if (rc) return rc;
  CK(cudaStreamSynchronize(ctx->stream));
  return QMPM_OK;
}

qmpm_status qmpm_read_ranges(qmpm_ctx* ctx, float* max_abs, int reset) {
  if (!ctx || !max_abs) return fail(ctx, QMPM_EINVAL, "NULL argument to qmpm_read_ranges");
  if (!ctx->L.ranges) return fail(ctx, QMPM_ESTATE, "qmpm_read_ranges needs params.flags |= QMPM_RECORD_RANGES");
  uint32_t bits[kMaxScalars];
  CK(cudaMemcpyAsync(bits, ctx->dc->range_bits, sizeof(bits), cudaMemcpyDeviceToHost, ctx->stream));
  if (reset) CK(cudaMemsetAsync(ctx->dc->range_bits, 0, sizeof(bits), ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < ctx->ns; ++i) memcpy(&max_abs[i], &bits[i], sizeof(float));
  return QMPM_OK;
}

qmpm_status qmpm_stats(qmpm_ctx* ctx, qmpm_stats_t* out) {
  if (!ctx || !out) return fail(ctx, QMPM_EINVAL, "NULL argument");
  DevCounters h;
  qmpm_status rc = sync_counters(ctx, h);
  if (rc) return rc;
  memset(out, 0, sizeof(*out));
  out->step = ctx->step;
  out->n_particles = (uint64_t)h.n_slots - std::min(h.n_leave, h.n_slots);  // live particles on this rank
  for (int i = 0; i < QMPM_MAX_FIELDS; ++i) {
    out->saturations[i] = h.sat[i];
    out->round_up[i] = h.up[i];
    out->round_down[i] = h.down[i];
  }
  out->nonfinite = h.nonfinite;
  out->out_of_domain = h.oob;
  out->active_blocks = h.n_active;
  out->touched_blocks = h.n_touched;
  out->pool_overflow = h.overflow;
  return status_error(ctx, ctx->sticky);
}

qmpm_status qmpm_encode(const qmpm_scheme* scheme, uint64_t n, const float* vals, const uint32_t* keys, uint64_t step,
                        uint32_t* words, uint64_t* counters, void* cuda_stream) {
  qmpm_ctx* ctx = nullptr;
  CodecDev C;
  qmpm_status rc = codec_of(ctx, scheme, C);
  if (rc) return rc;
  if (n && (!vals || !words)) return fail(ctx, QMPM_EINVAL, "NULL vals/words");
  const uint32_t salt = step_salt(C.seed_lo, C.seed_hi, (uint32_t)step);
  return codec_run(ctx, C, 0, n, vals, nullptr, keys, salt, nullptr, words, (unsigned long long*)counters, nullptr,
                   (cudaStream_t)cuda_stream);
}

qmpm_status qmpm_codec_matmul3(const qmpm_scheme* scheme, uint64_t n, const uint32_t* words_in, const float* a,
                               const uint32_t* keys, uint64_t step, uint32_t* words_out, void* cuda_stream) {
  qmpm_ctx* ctx = nullptr;
  CodecDev C;
  qmpm_status rc = codec_of(ctx, scheme, C);
  if (rc) return rc;
  if (C.nf != 9) return fail(ctx, QMPM_ELAYOUT, "qmpm_codec_matmul3 needs a scheme of 9 fields (got %u)", C.nf);
  if (n && (!words_in || !words_out || !a)) return fail(ctx, QMPM_EINVAL, "NULL words/matrix");
  const uint32_t salt = step_salt(C.seed_lo, C.seed_hi, (uint32_t)step);
  return codec_run(ctx, C, 2, n, nullptr, nullptr, keys, salt, words_in, words_out, nullptr, a,
                   (cudaStream_t)cuda_stream);
}

qmpm_status qmpm_decode(const qmpm_scheme* scheme, uint64_t n, const uint32_t* words, float* vals, void* cuda_stream) {
  qmpm_ctx* ctx = nullptr;
  CodecDev C;
  qmpm_status rc = codec_of(ctx, scheme, C);
  if (rc) return rc;
  if (n && (!vals || !words)) return fail(ctx, QMPM_EINVAL, "NULL vals/words");
  return codec_run(ctx, C, 1, n, nullptr, vals, nullptr, 0u, words, nullptr, nullptr, nullptr,
                   (cudaStream_t)cuda_stream);
}

qmpm_status qmpm_set_profiling(qmpm_ctx* ctx, int enabled) {
  if (!ctx) return fail(ctx, QMPM_EINVAL, "NULL ctx");
  qmpm_status rc = harvest(ctx);
  if (rc) return rc;
  ctx->prof = enabled != 0;
  for (int k = 0; k < KNumKernels; ++k) {
    ctx->ms[k] = 0;
    ctx->launches[k] = 0;
  }
  return QMPM_OK;
}

qmpm_status qmpm_kernel_times(qmpm_ctx* ctx, double* ms, uint64_t* launches) {
  if (!ctx) return fail(ctx, QMPM_EINVAL, "NULL ctx");
  qmpm_status rc = harvest(ctx);
  if (rc) return rc;
  for (int k = 0; k < KNumKernels; ++k) {
    if (ms) ms[k] = ctx->ms[k];
    if (launches) launches[k] = ctx->launches[k];
  }
  return QMPM_OK;
}

}  // extern "C"
