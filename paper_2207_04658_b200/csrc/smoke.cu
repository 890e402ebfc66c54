// smoke.cu -- host runtime and C ABI of the quantized smoke step (include/qsmoke.h).
//
// A ctx owns the NVRTC-specialised kernels for one (velocity, pressure) scheme pair,
// the state (velocity and pressure records, fp32 density) and the step's scratch
// (u~, u_h, u', a second pressure buffer, div, a second density buffer, the device step
// counter).  qsmoke_step replays a captured CUDA graph of one step (2 iters + 7 kernels);
// the dither salts come from the device step counter, so one graph serves every step;
// two graphs (by density parity) avoid a copy of the ping-ponged density.
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "jit.h"
#include "qsmoke.h"

using namespace qmpm;

namespace qmpm {
qmpm_status codec_dev_of(const qmpm_scheme* s, CodecDev& C);  // api.cu
void set_thread_error(const char* msg);                        // api.cu
}  // namespace qmpm

// must match smoke_kernels.cuh
struct SmokeDev {
  int nx, ny, nz, nxr;
  float dx, inv_dx;
  float half_inv_dx, dx2;
  int lo[3], hi[3];
  unsigned long long n_rec;
};
struct SaltSrc {
  uint32_t salt, sub, seed_lo, seed_hi;
  const unsigned long long* step;
};

struct qsmoke_ctx {
  qsmoke_params P{};
  CodecDev U{}, Pc{};
  SmokeJit k{};
  SmokeDev g{};
  cudaStream_t stream = nullptr, cap = nullptr;
  uint64_t n_rec = 0, n_cells = 0, launches = 0, step = 0;
  uint32_t *u = nullptr, *ut = nullptr, *uh = nullptr, *up = nullptr, *p[2] = {nullptr, nullptr};
  float *div = nullptr, *rho[2] = {nullptr, nullptr};
  int rcur = 0;  // which density buffer holds the state
  // two Jacobi sweeps per launch (qsmoke_jacobi2, temporal blocking): bit-identical but
  // measured SLOWER (1.93 ms per two sweeps at 612^3 vs 2 x 0.54 ms: the halo-extended
  // first sweep and three barriers per plane cost more issue slots than the halved DRAM
  // traffic saves -- the single sweep is issue-bound); QSMOKE_FUSE=1 enables
  bool fuse2 = false;
  unsigned long long* dstep = nullptr;
  cudaGraphExec_t graph[2] = {nullptr, nullptr};
};

namespace {

qmpm_status sfail(qmpm_status code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  set_thread_error(buf);
  return code;
}

#define SCK(x)                                                                                     \
  do {                                                                                             \
    cudaError_t e_ = (x);                                                                          \
    if (e_ != cudaSuccess) return sfail(QMPM_ECUDA, "%s: %s", #x, cudaGetErrorString(e_));          \
  } while (0)

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

int vec_width(uint32_t W) { return W % 4 == 0 ? 4 : (W % 2 == 0 ? 2 : 1); }

SaltSrc host_salt(const CodecDev& C, uint64_t dstep) {
  SaltSrc s{};
  s.salt = step_salt(C.seed_lo, C.seed_hi, (uint32_t)dstep);
  return s;
}

SaltSrc dev_salt(const qsmoke_ctx* c, const CodecDev& C, uint32_t sub) {
  SaltSrc s{};
  s.sub = sub;
  s.seed_lo = C.seed_lo;
  s.seed_hi = C.seed_hi;
  s.step = c->dstep;
  return s;
}

// every kernel: (32 z, 8 y) record tiles, blockIdx.z = a march of kXM = 8 record planes
// (smoke_kernels.cuh); the advections take dynamic shared memory for their rings of
// 3 planes x (8 + 2 kH) x (32 + 2 kH) records x 2 cells (kH = 2): float4 velocity,
// float4 reflected field, float density
constexpr size_t kRingCells = 3 * (8 + 4) * (32 + 4) * 2;
constexpr size_t kSmemAdvect = kRingCells * 16, kSmemReflect = 2 * kRingCells * 16,
                 kSmemDensity = kRingCells * 16 + kRingCells * 4;
qmpm_status launch(qsmoke_ctx* c, CUfunction f, cudaStream_t st, void** args, size_t smem = 0, int rows = 8,
                   int planes = 8) {
  const dim3 grid((c->g.nz + 31) / 32, (c->g.ny + rows - 1) / rows, (c->g.nxr + planes - 1) / planes);
  c->launches += 1;
  SCK(jit_launch3(f, grid, dim3(32, 8, 1), smem, st, args));
  return QMPM_OK;
}

qmpm_status advect_u(qsmoke_ctx* c, cudaStream_t st, const uint32_t* uv, const uint32_t* ur, const float* rho,
                     float dt, float bdt, SaltSrc ss, uint32_t* out, float* dbg) {
  void* a[] = {&uv, &ur, &rho, &c->g, &dt, &bdt, &ss, &out, &dbg};
  return ur ? launch(c, c->k.advect_refl, st, a, kSmemReflect) : launch(c, c->k.advect_u, st, a, kSmemAdvect);
}
qmpm_status divergence(qsmoke_ctx* c, cudaStream_t st, const uint32_t* u, float* div) {
  void* a[] = {&u, &c->g, &div};
  return launch(c, c->k.div, st, a);
}
qmpm_status jacobi(qsmoke_ctx* c, cudaStream_t st, const uint32_t* pin, const float* div, SaltSrc ss, uint32_t* pout,
                   float* dbg) {
  void* a[] = {&pin, &div, &c->g, &ss, &pout, &dbg};
  return launch(c, c->k.jacobi, st, a, 0, 16);  // two rows per thread (p_march2)
}
// two sweeps in one launch (qsmoke_jacobi2: 16 planes per CTA, 16-row tiles)
qmpm_status jacobi2(qsmoke_ctx* c, cudaStream_t st, const uint32_t* pin, const float* div, SaltSrc s1, SaltSrc s2,
                    uint32_t* pout) {
  void* a[] = {&pin, &div, &c->g, &s1, &s2, &pout};
  return launch(c, c->k.jacobi2, st, a, 0, 16, 16);
}
qmpm_status project(qsmoke_ctx* c, cudaStream_t st, const uint32_t* u, const uint32_t* p, SaltSrc ss, uint32_t* out,
                    float* dbg) {
  void* a[] = {&u, &p, &c->g, &ss, &out, &dbg};
  return launch(c, c->k.project, st, a, 0, 16);
}
qmpm_status advect_rho(qsmoke_ctx* c, cudaStream_t st, const float* rin, const uint32_t* u, float dt, float* rout,
                       unsigned long long* tick) {
  void* a[] = {&rin, &u, &c->g, &dt, &rout, &tick};
  return launch(c, c->k.advect_rho, st, a, kSmemDensity);
}

// one projection (S6-S7) of u_in into u_out; subs: sub0 = the velocity store,
// sub0 + 1 + k = Jacobi sweep k.  Pressure ends in p[0] (even sweep count per step).
qmpm_status projection(qsmoke_ctx* c, cudaStream_t st, const uint32_t* u_in, uint32_t sub0, uint32_t* u_out) {
  qmpm_status rc = divergence(c, st, u_in, c->div);
  if (rc) return rc;
  int cur = 0;
  for (int k = 0; k < c->P.jacobi_iters;) {
    if (k + 1 < c->P.jacobi_iters && c->fuse2) {  // sweeps k, k + 1 in one launch
      rc = jacobi2(c, st, c->p[cur], c->div, dev_salt(c, c->Pc, sub0 + 1 + k), dev_salt(c, c->Pc, sub0 + 2 + k),
                   c->p[cur ^ 1]);
      k += 2;
    } else {
      rc = jacobi(c, st, c->p[cur], c->div, dev_salt(c, c->Pc, sub0 + 1 + k), c->p[cur ^ 1], nullptr);
      k += 1;
    }
    if (rc) return rc;
    cur ^= 1;
  }
  if (cur) {  // odd sweep count: bring the pressure back to p[0]
    SCK(cudaMemcpyAsync(c->p[0], c->p[1], sizeof(uint32_t) * c->Pc.W * c->n_rec, cudaMemcpyDeviceToDevice, st));
  }
  return project(c, st, u_in, c->p[0], dev_salt(c, c->U, sub0), u_out, nullptr);
}

// one step of S8 from density buffer `par`, enqueued on st (captured into graph[par])
qmpm_status enqueue_step(qsmoke_ctx* c, cudaStream_t st, int par) {
  const float dt = c->P.dt, half = 0.5f * c->P.dt, bdt = 0.5f * c->P.dt * c->P.buoyancy;
  qmpm_status rc = advect_u(c, st, c->u, nullptr, c->rho[par], half, bdt, dev_salt(c, c->U, 0), c->ut, nullptr);
  if (!rc) rc = projection(c, st, c->ut, 1, c->uh);
  if (!rc) rc = advect_u(c, st, c->uh, c->ut, nullptr, half, 0.0f, dev_salt(c, c->U, 100), c->up, nullptr);
  if (!rc) rc = projection(c, st, c->up, 101, c->u);
  if (!rc) rc = advect_rho(c, st, c->rho[par], c->u, dt, c->rho[par ^ 1], c->dstep);
  return rc;
}

qmpm_status build_graphs(qsmoke_ctx* c) {
  for (int par = 0; par < 2; ++par) {
    cudaGraph_t g = nullptr;
    const uint64_t l0 = c->launches;
    SCK(cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeThreadLocal));
    qmpm_status rc = enqueue_step(c, c->cap, par);
    cudaError_t e = cudaStreamEndCapture(c->cap, &g);
    c->launches = l0;  // captured, not launched
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (e != cudaSuccess) return sfail(QMPM_ECUDA, "graph capture: %s", cudaGetErrorString(e));
    e = cudaGraphInstantiate(&c->graph[par], g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return sfail(QMPM_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
  }
  return QMPM_OK;
}

void release(qsmoke_ctx* c) {
  for (auto& g : c->graph)
    if (g) cudaGraphExecDestroy(g);
  for (void* p : {(void*)c->u, (void*)c->ut, (void*)c->uh, (void*)c->up, (void*)c->p[0], (void*)c->p[1],
                  (void*)c->div, (void*)c->rho[0], (void*)c->rho[1], (void*)c->dstep})
    if (p) cudaFree(p);
  if (c->cap) cudaStreamDestroy(c->cap);
  delete c;
}

qmpm_status copy_any(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  SCK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st));
  return QMPM_OK;
}

}  // namespace

extern "C" {

qmpm_status qsmoke_create(const qsmoke_params* params, const qmpm_scheme* u_scheme, const qmpm_scheme* p_scheme,
                          void* cuda_stream, qsmoke_ctx** out) {
  if (!params || !u_scheme || !p_scheme || !out) return sfail(QMPM_EINVAL, "NULL argument");
  *out = nullptr;
  const qsmoke_params& P = *params;
  if (P.res[0] < 2 || P.res[0] % 2 || P.res[1] < 2 || P.res[2] < 2)
    return sfail(QMPM_EINVAL, "res must be nx even >= 2, ny, nz >= 2 (got %d %d %d)", P.res[0], P.res[1], P.res[2]);
  if (!(P.dx > 0.0f) || !(P.dt >= 0.0f)) return sfail(QMPM_EINVAL, "dx must be > 0 and dt >= 0");
  if (P.jacobi_iters < 0 || P.jacobi_iters > 98) return sfail(QMPM_EINVAL, "jacobi_iters must be in 0..98");
  if (P.res[0] > 65535 || P.res[1] > 65535 * 8) return sfail(QMPM_EINVAL, "res too large for the launch grid");
  if (u_scheme->n_fields != 6) return sfail(QMPM_ELAYOUT, "velocity scheme needs 6 fields (got %u)", u_scheme->n_fields);
  if (p_scheme->n_fields != 2) return sfail(QMPM_ELAYOUT, "pressure scheme needs 2 fields (got %u)", p_scheme->n_fields);
  qsmoke_ctx* c = new qsmoke_ctx();
  c->P = P;
  qmpm_status rc = codec_dev_of(u_scheme, c->U);
  if (!rc) rc = codec_dev_of(p_scheme, c->Pc);
  if (rc) {
    delete c;
    return rc;
  }
  if (getenv("QSMOKE_FUSE") && atoi(getenv("QSMOKE_FUSE")) != 0) c->fuse2 = true;
  for (uint32_t i = 0; i < p_scheme->n_fields; ++i)
    if (p_scheme->fields[i].kind == QMPM_SHARED_EXP) c->fuse2 = false;
  std::string err;
  const std::string src = smoke_spec_source(c->U, c->Pc, vec_width(c->U.W), vec_width(c->Pc.W));
  if (jit_smoke(src, c->k, err) != cudaSuccess) {
    delete c;
    return sfail(QMPM_ECUDA, "%s", err.c_str());
  }
  if (jit_set_smem(c->k.advect_u, kSmemAdvect) != cudaSuccess ||
      jit_set_smem(c->k.advect_refl, kSmemReflect) != cudaSuccess ||
      jit_set_smem(c->k.advect_rho, kSmemDensity) != cudaSuccess) {
    delete c;
    return sfail(QMPM_ECUDA, "cannot enable %zu bytes of shared memory for the advection kernels", kSmemReflect);
  }
  c->stream = (cudaStream_t)cuda_stream;
  c->n_rec = (uint64_t)(P.res[0] / 2) * P.res[1] * P.res[2];
  c->n_cells = 2 * c->n_rec;
  SmokeDev& g = c->g;
  g.nx = P.res[0];
  g.ny = P.res[1];
  g.nz = P.res[2];
  g.nxr = P.res[0] / 2;
  g.dx = P.dx;
  g.inv_dx = 1.0f / P.dx;
  g.half_inv_dx = 0.5f / P.dx;
  g.dx2 = P.dx * P.dx;
  for (int a = 0; a < 3; ++a) {
    g.lo[a] = P.source_lo[a];
    g.hi[a] = P.source_hi[a];
  }
  g.n_rec = c->n_rec;
  const size_t bu = sizeof(uint32_t) * c->U.W * c->n_rec, bp = sizeof(uint32_t) * c->Pc.W * c->n_rec,
               bf = sizeof(float) * c->n_cells;
  cudaError_t e = cudaSuccess;
  for (uint32_t** p : {&c->u, &c->ut, &c->uh, &c->up})
    if (!e) e = cudaMalloc(p, bu);
  for (uint32_t** p : {&c->p[0], &c->p[1]})
    if (!e) e = cudaMalloc(p, bp);
  for (float** p : {&c->div, &c->rho[0], &c->rho[1]})
    if (!e) e = cudaMalloc(p, bf);
  if (!e) e = cudaMalloc(&c->dstep, sizeof(unsigned long long));
  if (!e) e = cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking);
  if (e) {
    release(c);
    cudaGetLastError();
    return sfail(e == cudaErrorMemoryAllocation ? QMPM_ENOMEM : QMPM_ECUDA, "qsmoke_create: %s",
                 cudaGetErrorString(e));
  }
  if (!e) e = cudaMemsetAsync(c->u, 0, bu, c->stream);
  if (!e) e = cudaMemsetAsync(c->p[0], 0, bp, c->stream);
  if (!e) e = cudaMemsetAsync(c->rho[0], 0, bf, c->stream);
  if (!e) e = cudaMemsetAsync(c->dstep, 0, sizeof(unsigned long long), c->stream);
  if (!e) e = cudaStreamSynchronize(c->stream);
  if (e) {
    release(c);
    return sfail(QMPM_ECUDA, "qsmoke_create: %s", cudaGetErrorString(e));
  }
  rc = build_graphs(c);
  if (rc) {
    release(c);
    return rc;
  }
  *out = c;
  return QMPM_OK;
}

qmpm_status qsmoke_destroy(qsmoke_ctx* ctx) {
  if (!ctx) return QMPM_OK;
  cudaStreamSynchronize(ctx->stream);
  release(ctx);
  return QMPM_OK;
}

qmpm_status qsmoke_layout(const qsmoke_ctx* ctx, uint32_t* words_u, uint32_t* words_p, uint64_t* n_records) {
  if (!ctx) return sfail(QMPM_EINVAL, "NULL ctx");
  if (words_u) *words_u = ctx->U.W;
  if (words_p) *words_p = ctx->Pc.W;
  if (n_records) *n_records = ctx->n_rec;
  return QMPM_OK;
}

qmpm_status qsmoke_advect_velocity(qsmoke_ctx* ctx, const uint32_t* u_vel, const uint32_t* u_refl, const float* rho,
                                   float dt, float bdt, uint64_t dstep, uint32_t* u_out, float* dbg) {
  if (!ctx || !u_vel || !u_out) return sfail(QMPM_EINVAL, "NULL ctx/u_vel/u_out");
  if (!aligned16(u_vel) || !aligned16(u_refl) || !aligned16(u_out)) return sfail(QMPM_EINVAL, "records must be 16-byte aligned");
  return advect_u(ctx, ctx->stream, u_vel, u_refl, rho, dt, bdt, host_salt(ctx->U, dstep), u_out, dbg);
}

qmpm_status qsmoke_divergence(qsmoke_ctx* ctx, const uint32_t* u, float* div) {
  if (!ctx || !u || !div) return sfail(QMPM_EINVAL, "NULL ctx/u/div");
  return divergence(ctx, ctx->stream, u, div);
}

qmpm_status qsmoke_jacobi(qsmoke_ctx* ctx, const uint32_t* p_in, const float* div, uint64_t dstep, uint32_t* p_out,
                          float* dbg) {
  if (!ctx || !p_in || !div || !p_out) return sfail(QMPM_EINVAL, "NULL ctx/p_in/div/p_out");
  if (!aligned16(p_out)) return sfail(QMPM_EINVAL, "records must be 16-byte aligned");
  return jacobi(ctx, ctx->stream, p_in, div, host_salt(ctx->Pc, dstep), p_out, dbg);
}

qmpm_status qsmoke_project(qsmoke_ctx* ctx, const uint32_t* u_in, const uint32_t* p, uint64_t dstep, uint32_t* u_out,
                           float* dbg) {
  if (!ctx || !u_in || !p || !u_out) return sfail(QMPM_EINVAL, "NULL ctx/u_in/p/u_out");
  if (!aligned16(u_out)) return sfail(QMPM_EINVAL, "records must be 16-byte aligned");
  return project(ctx, ctx->stream, u_in, p, host_salt(ctx->U, dstep), u_out, dbg);
}

qmpm_status qsmoke_advect_density(qsmoke_ctx* ctx, const float* rho_in, const uint32_t* u, float dt, float* rho_out) {
  if (!ctx || !rho_in || !u || !rho_out) return sfail(QMPM_EINVAL, "NULL ctx/rho_in/u/rho_out");
  return advect_rho(ctx, ctx->stream, rho_in, u, dt, rho_out, nullptr);
}

qmpm_status qsmoke_set_state(qsmoke_ctx* ctx, const uint32_t* u_words, const uint32_t* p_words, const float* rho,
                             uint64_t step) {
  if (!ctx || !u_words || !p_words || !rho) return sfail(QMPM_EINVAL, "NULL ctx/state");
  ctx->rcur = 0;
  ctx->step = step;
  qmpm_status rc = copy_any(ctx->u, u_words, sizeof(uint32_t) * ctx->U.W * ctx->n_rec, ctx->stream);
  if (!rc) rc = copy_any(ctx->p[0], p_words, sizeof(uint32_t) * ctx->Pc.W * ctx->n_rec, ctx->stream);
  if (!rc) rc = copy_any(ctx->rho[0], rho, sizeof(float) * ctx->n_cells, ctx->stream);
  if (!rc) rc = copy_any(ctx->dstep, &ctx->step, sizeof(unsigned long long), ctx->stream);
  if (rc) return rc;
  SCK(cudaStreamSynchronize(ctx->stream));  // the step value is a host local's copy
  return QMPM_OK;
}

qmpm_status qsmoke_get_state(qsmoke_ctx* ctx, uint32_t* u_words, uint32_t* p_words, float* rho) {
  if (!ctx) return sfail(QMPM_EINVAL, "NULL ctx");
  qmpm_status rc = QMPM_OK;
  if (u_words) rc = copy_any(u_words, ctx->u, sizeof(uint32_t) * ctx->U.W * ctx->n_rec, ctx->stream);
  if (!rc && p_words) rc = copy_any(p_words, ctx->p[0], sizeof(uint32_t) * ctx->Pc.W * ctx->n_rec, ctx->stream);
  if (!rc && rho) rc = copy_any(rho, ctx->rho[ctx->rcur], sizeof(float) * ctx->n_cells, ctx->stream);
  if (rc) return rc;
  SCK(cudaStreamSynchronize(ctx->stream));
  return QMPM_OK;
}

qmpm_status qsmoke_step(qsmoke_ctx* ctx, uint64_t n_steps) {
  if (!ctx) return sfail(QMPM_EINVAL, "NULL ctx");
  const uint64_t sweeps = ctx->fuse2 ? (uint64_t)(ctx->P.jacobi_iters / 2 + ctx->P.jacobi_iters % 2)
                                     : (uint64_t)ctx->P.jacobi_iters;
  const uint64_t per_step = 2ull * sweeps + 7;
  for (uint64_t s = 0; s < n_steps; ++s) {
    SCK(cudaGraphLaunch(ctx->graph[ctx->rcur], ctx->stream));
    ctx->rcur ^= 1;
    ctx->step += 1;
    ctx->launches += per_step;
  }
  return QMPM_OK;
}

qmpm_status qsmoke_launch_count(const qsmoke_ctx* ctx, uint64_t* launches) {
  if (!ctx || !launches) return sfail(QMPM_EINVAL, "NULL argument");
  *launches = ctx->launches;
  return QMPM_OK;
}

}  // extern "C"
