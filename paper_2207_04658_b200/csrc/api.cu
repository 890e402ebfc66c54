// api.cu -- host runtime and C ABI of libqmpm (include/qmpm.h).
//
// Owns the device pools of one simulation context: ping-pong packed records
// (records are physically re-sorted by grid block every step: G2P writes record j
// of the sorted order), the block table of the counting sort, the grid-block pool
// and the device counters.  Everything is enqueued on the ctx stream; qmpm_step
// allocates nothing.
#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

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
  uint8_t* cells = nullptr;
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
};

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

uint32_t field_width(const qmpm_field& f) { return f.kind == QMPM_RAW_F32 ? 32u : (uint32_t)f.frac_bits + 1u; }

// bit-pack layout: contiguous, LSB-first, in declaration order
qmpm_status layout_of(qmpm_ctx* ctx, const qmpm_scheme* s, std::vector<uint32_t>& offs, uint32_t& W,
                      uint32_t& bits) {
  if (!s || !s->fields) return fail(ctx, QMPM_EINVAL, "scheme or scheme->fields is NULL");
  if (s->n_fields == 0 || s->n_fields > QMPM_MAX_FIELDS)
    return fail(ctx, QMPM_ELAYOUT, "n_fields=%u out of [1, %d]", s->n_fields, QMPM_MAX_FIELDS);
  if (s->layout_policy != 0) return fail(ctx, QMPM_ELAYOUT, "layout_policy %u not supported", s->layout_policy);
  offs.resize(s->n_fields);
  uint32_t total = 0;
  for (uint32_t i = 0; i < s->n_fields; ++i) {
    const qmpm_field& f = s->fields[i];
    if (f.kind == QMPM_SHARED_EXP) return fail(ctx, QMPM_ELAYOUT, "field %u: SHARED_EXP is not supported", i);
    if (f.kind != QMPM_FIXED && f.kind != QMPM_RAW_F32) return fail(ctx, QMPM_ELAYOUT, "field %u: bad kind %u", i, f.kind);
    if (f.kind == QMPM_FIXED) {
      if ((uint32_t)f.frac_bits + 1u > 32u) return fail(ctx, QMPM_ELAYOUT, "field %u: width %u > 32", i, f.frac_bits + 1u);
      if (!(f.range > 0.0f) || !std::isfinite(f.range)) return fail(ctx, QMPM_ELAYOUT, "field %u: range must be > 0", i);
      if (!std::isfinite(f.offset)) return fail(ctx, QMPM_ELAYOUT, "field %u: offset not finite", i);
    }
    offs[i] = total;
    total += field_width(f);
  }
  bits = total;
  W = (total + 31) / 32;
  return QMPM_OK;
}

FieldDev field_dev(const qmpm_field& f, uint32_t off, uint16_t idx, uint16_t col) {
  FieldDev d{};
  d.word = (uint8_t)(off / 32);
  d.shift = (uint8_t)(off % 32);
  d.width = (uint8_t)field_width(f);
  d.kind = f.kind == QMPM_RAW_F32 ? kKindRaw : kKindFixed;
  if (f.kind == QMPM_FIXED) {
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
  for (uint32_t i = 0; i < s->n_fields; ++i) C.f[i] = field_dev(s->fields[i], offs[i], (uint16_t)i, (uint16_t)i);
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

qmpm_status rebin(qmpm_ctx* ctx) {
  CK(cudaMemsetAsync(ctx->block_count, 0, sizeof(uint32_t) * ctx->S.nblocks, ctx->stream));
  hook_fn(ctx, KBinCount, 1);
  CK(launch_bin_count(ctx->rec[ctx->cur], 0u, (uint32_t)ctx->n, ctx->S, ctx->key, ctx->block_count, 1, ctx->jit,
                      ctx->stream));
  hook_fn(ctx, KBinCount, 0);
  ctx->binned = true;
  return QMPM_OK;
}

qmpm_status reset_counters(qmpm_ctx* ctx) {
  CK(cudaMemsetAsync(ctx->dc, 0, sizeof(DevCounters), ctx->stream));
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
  ctx->launches_total += 1;
  CK(launch_encode(ctx->C, n, dv, nullptr, 0u, ctx->rec[ctx->cur] + first * ctx->W,
                   (unsigned long long*)ctx->dc, ctx->stream));
  if (ctx->ids[ctx->cur]) {
    ctx->launches_total += 1;
    CK(launch_iota(ctx->ids[ctx->cur] + first, (uint32_t)n, (uint32_t)first, ctx->stream));
  }
  if (tmp) CK(cudaFreeAsync(tmp, ctx->stream));
  return QMPM_OK;
}

}  // namespace

extern "C" {

int qmpm_abi_version(void) { return QMPM_ABI_VERSION; }

const char* qmpm_last_error(const qmpm_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

const char* qmpm_kernel_name(int i) {
  static const char* names[KNumKernels] = {"bin_count", "scan_reduce", "scan_tiles", "scan_apply",
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
  void* ptrs[] = {ctx->rec[0], ctx->rec[1], ctx->ids[0], ctx->ids[1], ctx->key, ctx->perm, ctx->cells,
                  ctx->block_count, ctx->block_start, ctx->block_slot, ctx->active_list, ctx->touched_list,
                  ctx->tile_sums, ctx->tile_off, ctx->mp, ctx->gv, ctx->dc, ctx->dbg};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (auto& p : ctx->pending) {
    cudaEventDestroy(p.a);
    if (p.b) cudaEventDestroy(p.b);
  }
  for (auto e : ctx->free_events) cudaEventDestroy(e);
  delete ctx;
  return QMPM_OK;
}

qmpm_status qmpm_create(const qmpm_params* params, const qmpm_scheme* scheme, void* cuda_stream, qmpm_ctx** out) {
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

  // MPM layout (fields by state scalar) and the state codec (vals in scalar order)
  LayoutDev& L = ctx->L;
  L.W = W;
  L.SW = stage_stride(W);
  L.ns = (uint32_t)ns;
  L.dither = scheme->rounding == QMPM_DITHER;
  L.counters = (P.flags & QMPM_NO_ROUND_COUNTERS) ? 0u : 1u;
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
    L.s[s] = field_dev(f, offs[i], (uint16_t)i, (uint16_t)s);
    C.f[i] = field_dev(f, offs[i], (uint16_t)i, (uint16_t)s);
    if (f.attr == QMPM_X) {
      const uint32_t w0 = offs[i] / 32, w1 = (offs[i] + field_width(f) - 1) / 32;
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
    nblocks *= (uint64_t)S.nb[a];
    S.g[a] = a < d ? P.gravity[a] : 0.0f;
  }
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
  ALLOC(ctx->cells, cap);
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
    constexpr int kP2GWarps = 4, kG2PWarps = 4;
    // minimum resident CTAs per SM the kernels are compiled for (register cap);
    // QMPM_P2G_MINB / QMPM_G2P_MINB override the defaults for tuning runs
    auto env_int = [](const char* name, int dflt) {
      const char* v = getenv(name);
      return (v && *v) ? atoi(v) : dflt;
    };
    const int kP2GMinBlocks = env_int("QMPM_P2G_MINB", 3), kG2PMinBlocks = env_int("QMPM_G2P_MINB", 4);
    ctx->jit_src = spec_source(d, ctx->material, ctx->L, kP2GWarps, kG2PWarps, kP2GMinBlocks, kG2PMinBlocks);
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
  *out = ctx;
  return QMPM_OK;
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
  return QMPM_OK;
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
  return QMPM_OK;
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
  return QMPM_OK;
}

qmpm_status qmpm_step(qmpm_ctx* ctx, uint32_t n_steps) {
  if (!ctx) return fail(ctx, QMPM_EINVAL, "NULL ctx");
  for (uint32_t t = 0; t < n_steps; ++t) {
    if (!ctx->binned) {
      qmpm_status rc = rebin(ctx);
      if (rc) return rc;
    }
    StepBuffers B{};
    B.rec_in = ctx->rec[ctx->cur];
    B.rec_out = ctx->rec[ctx->cur ^ 1];
    B.ids_in = ctx->ids[ctx->cur];
    B.ids_out = ctx->ids[ctx->cur ^ 1];
    B.key = ctx->key;
    B.perm = ctx->perm;
    B.cells = ctx->cells;
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
    B.n = (uint32_t)ctx->n;
    B.pool = (uint32_t)ctx->pool;
    B.ntiles = ctx->ntiles;
    const uint64_t t_step = ctx->step + 1;  // steps are numbered 1, 2, ... (Q20)
    const uint32_t salt = step_salt(ctx->L.seed_lo, ctx->L.seed_hi, (uint32_t)t_step);
    CK(launch_step(ctx->dim, B, ctx->S, salt, ctx->jit, ctx->stream, hook_fn, ctx));
    ctx->cur ^= 1;
    ctx->step = t_step;
    ctx->dbg_valid = ctx->dbg != nullptr;
  }
  return QMPM_OK;
}

qmpm_status qmpm_read_state(qmpm_ctx* ctx, float* vals, uint32_t* words, uint32_t* ids, uint64_t capacity,
                            uint64_t* n_out) {
  if (!ctx) return fail(ctx, QMPM_EINVAL, "NULL ctx");
  const uint64_t n = ctx->n;
  if (n_out) *n_out = n;
  if (capacity < n) return fail(ctx, QMPM_ECAPACITY, "capacity %llu < n %llu", (unsigned long long)capacity,
                                (unsigned long long)n);
  if (ids && !ctx->ids[ctx->cur]) return fail(ctx, QMPM_ESTATE, "ids requested without QMPM_TRACK_IDS");
  if (vals && n) {
    float* dv = vals;
    float* tmp = nullptr;
    if (!is_device_ptr(vals)) {
      CK(cudaMallocAsync((void**)&tmp, sizeof(float) * ctx->ns * n, ctx->stream));
      dv = tmp;
    }
    ctx->launches_total += 1;
    CK(launch_decode(ctx->C, n, ctx->rec[ctx->cur], dv, ctx->stream));
    if (tmp) {
      CK(cudaMemcpyAsync(vals, tmp, sizeof(float) * ctx->ns * n, cudaMemcpyDefault, ctx->stream));
      CK(cudaFreeAsync(tmp, ctx->stream));
    }
  }
  if (words && n) CK(cudaMemcpyAsync(words, ctx->rec[ctx->cur], sizeof(uint32_t) * ctx->W * n, cudaMemcpyDefault, ctx->stream));
  if (ids && n) CK(cudaMemcpyAsync(ids, ctx->ids[ctx->cur], sizeof(uint32_t) * n, cudaMemcpyDefault, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  DevCounters h;
  CK(cudaMemcpy(&h, ctx->dc, sizeof(h), cudaMemcpyDeviceToHost));
  if (h.overflow) return fail(ctx, QMPM_ECAPACITY, "grid pool overflow in %llu step(s): raise pool_blocks",
                              (unsigned long long)h.overflow);
  return QMPM_OK;
}

qmpm_status qmpm_read_debug(qmpm_ctx* ctx, float* pre, uint64_t capacity, uint64_t* n_out) {
  if (!ctx) return fail(ctx, QMPM_EINVAL, "NULL ctx");
  if (!ctx->dbg) return fail(ctx, QMPM_ESTATE, "QMPM_DEBUG_PREENCODE not set");
  if (!ctx->dbg_valid) return fail(ctx, QMPM_ESTATE, "no step taken since the state was set");
  const uint64_t n = ctx->n;
  if (n_out) *n_out = n;
  if (capacity < n) return fail(ctx, QMPM_ECAPACITY, "capacity < n");
  if (n) CK(cudaMemcpyAsync(pre, ctx->dbg, sizeof(float) * ctx->ns * n, cudaMemcpyDefault, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return QMPM_OK;
}

qmpm_status qmpm_stats(qmpm_ctx* ctx, qmpm_stats_t* out) {
  if (!ctx || !out) return fail(ctx, QMPM_EINVAL, "NULL argument");
  CK(cudaStreamSynchronize(ctx->stream));
  DevCounters h;
  CK(cudaMemcpy(&h, ctx->dc, sizeof(h), cudaMemcpyDeviceToHost));
  memset(out, 0, sizeof(*out));
  out->step = ctx->step;
  out->n_particles = ctx->n;
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
  return QMPM_OK;
}

qmpm_status qmpm_encode(const qmpm_scheme* scheme, uint64_t n, const float* vals, const uint32_t* keys, uint64_t step,
                        uint32_t* words, uint64_t* counters, void* cuda_stream) {
  qmpm_ctx* ctx = nullptr;
  CodecDev C;
  qmpm_status rc = codec_of(ctx, scheme, C);
  if (rc) return rc;
  if (n && (!vals || !words)) return fail(ctx, QMPM_EINVAL, "NULL vals/words");
  const uint32_t salt = step_salt(C.seed_lo, C.seed_hi, (uint32_t)step);
  CK(launch_encode(C, n, vals, keys, salt, words, (unsigned long long*)counters, (cudaStream_t)cuda_stream));
  return QMPM_OK;
}

qmpm_status qmpm_decode(const qmpm_scheme* scheme, uint64_t n, const uint32_t* words, float* vals, void* cuda_stream) {
  qmpm_ctx* ctx = nullptr;
  CodecDev C;
  qmpm_status rc = codec_of(ctx, scheme, C);
  if (rc) return rc;
  if (n && (!vals || !words)) return fail(ctx, QMPM_EINVAL, "NULL vals/words");
  CK(launch_decode(C, n, words, vals, (cudaStream_t)cuda_stream));
  return QMPM_OK;
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
