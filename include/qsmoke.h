/*
 * qsmoke.h -- C ABI of the quantized Eulerian smoke step in libqmpm (SURVEY §8(f) row
 * f4): the paper's second simulator, "an Eulerian fluid solver with advection-
 * reflection (Zehnder et al. 2018) ... semi-Lagrangian advection with RK-3 path
 * integration ... Poisson's equation by 64 Jacobi iterations ... quantized pressure
 * and velocity".  The paper says nothing more; the readings
 * S1-S8 fix the discretisation:
 *   S1 collocated nx x ny x nz cells, dx per cell, velocity in world units per second;
 *   S2 records of two cells along x: record r = (xr * ny + y) * nz + z holds cells
 *      x = 2 xr, 2 xr + 1; a velocity record packs 6 fields (cell0 ux uy uz, cell1
 *      ux uy uz), a pressure record 2 (cell0 p, cell1 p), in the given schemes'
 *      bit-pack layouts (qmpm.h); density is an fp32 array [nx][ny][nz];
 *   S3 trilinear sampling with positions clamped to [0, n - 1];
 *   S4 RK-3 (Ralston) backtrace; S5 central-difference divergence, u = 0 outside;
 *   S6 Jacobi sweeps p <- (sum of 6 neighbours - dx^2 div) / 6, Neumann walls;
 *   S7 u -= grad p (central differences, Neumann), wall-normal u zeroed at the walls;
 *   S8 the step: u~ = A(u, u, dt/2) + dt/2 b rho e_y; u_h = P(u~); u' = A(2 u_h - u~,
 *      u_h, dt/2); u = P(u'); rho = A(rho, u, dt), rho = 1 in the source box.
 * Every store of velocity or pressure is encoded with its scheme, dithered (Eq. 11)
 * with key = record index and the dither step index `dstep` (salt as in qmpm_encode).
 * qsmoke_step uses dstep = 256 step + sub, sub = 0 (first advection), 1 (first
 * projection's velocity), 2 + k (its Jacobi sweep k), 100, 101, 102 + k (second half).
 *
 * Conventions: as qmpm.h (status codes, qmpm_last_error, caller-owned pointers).  All
 * array arguments of the sub-step calls are DEVICE pointers on the ctx's device,
 * 16-byte aligned, sized for n_records = nx/2 * ny * nz records (velocity W_u words,
 * pressure W_p words each) or nx*ny*nz floats; work goes to the ctx stream; inputs and
 * outputs must not overlap.  dbg (nullable, device) receives the values before encoding
 * ([n_records][6] or [n_records][2] fp32).
 */
#ifndef QSMOKE_H
#define QSMOKE_H
#include "qmpm.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct qsmoke_ctx qsmoke_ctx; /* opaque: the specialised kernels + the state */

typedef struct {
    int32_t res[3];       /* nx (even, >= 2), ny, nz (>= 2) */
    float dx, dt;         /* cell size, time step */
    float buoyancy;       /* b: dt/2 b rho is added to u_y in the first advection */
    int32_t source_lo[3]; /* density source box [lo, hi) in cells */
    int32_t source_hi[3];
    int32_t jacobi_iters; /* Jacobi sweeps per projection (64); 0..98 */
    int32_t pad;
} qsmoke_params;

/* Create a ctx on the current device: validates the schemes (velocity: 6 fields,
 * pressure: 2 fields; FIXED / RAW_F32 / SHARED_EXP as qmpm.h), compiles the kernels
 * for their layouts (NVRTC, cached per process) and allocates the state (velocity,
 * pressure and density) plus the step's scratch, all zero.  QMPM_EINVAL for bad
 * params, QMPM_ELAYOUT for a bad scheme. */
qmpm_status qsmoke_create(const qsmoke_params* params, const qmpm_scheme* u_scheme, const qmpm_scheme* p_scheme,
                          void* cuda_stream, qsmoke_ctx** out);
qmpm_status qsmoke_destroy(qsmoke_ctx* ctx); /* synchronizes; NULL is a no-op */
/* Words per velocity / pressure record and the number of records (S2). */
qmpm_status qsmoke_layout(const qsmoke_ctx* ctx, uint32_t* words_u, uint32_t* words_p, uint64_t* n_records);

/* S3-S4 (+ S8 buoyancy): u_out = encode(A(q, u_vel, dt) [+ bdt rho e_y]), q = u_vel, or
 * 2 u_vel - u_refl when u_refl != NULL (the reflection, S8); rho nullable (no
 * buoyancy), bdt = dt/2 b in qsmoke_step. */
qmpm_status qsmoke_advect_velocity(qsmoke_ctx* ctx, const uint32_t* u_vel, const uint32_t* u_refl, const float* rho,
                                   float dt, float bdt, uint64_t dstep, uint32_t* u_out, float* dbg);
/* S5: div [nx][ny][nz] fp32 of the decoded velocity. */
qmpm_status qsmoke_divergence(qsmoke_ctx* ctx, const uint32_t* u, float* div);
/* S6: one Jacobi sweep p_out = encode(J(p_in, div)). */
qmpm_status qsmoke_jacobi(qsmoke_ctx* ctx, const uint32_t* p_in, const float* div, uint64_t dstep, uint32_t* p_out,
                          float* dbg);
/* S7: u_out = encode(walls(u_in - grad p)). */
qmpm_status qsmoke_project(qsmoke_ctx* ctx, const uint32_t* u_in, const uint32_t* p, uint64_t dstep, uint32_t* u_out,
                           float* dbg);
/* S8 last line: rho_out = A(rho_in, u, dt), then 1 in the source box (fp32). */
qmpm_status qsmoke_advect_density(qsmoke_ctx* ctx, const float* rho_in, const uint32_t* u, float dt, float* rho_out);

/* The ctx-owned state: set (host or device arrays, copied; sets the step counter),
 * get (host or device destinations; synchronizes). */
qmpm_status qsmoke_set_state(qsmoke_ctx* ctx, const uint32_t* u_words, const uint32_t* p_words, const float* rho,
                             uint64_t step);
qmpm_status qsmoke_get_state(qsmoke_ctx* ctx, uint32_t* u_words, uint32_t* p_words, float* rho);
/* n_steps steps of S8 on the ctx state (2 jacobi_iters + 7 kernels per step, replayed
 * from a CUDA graph); asynchronous on the ctx stream. */
qmpm_status qsmoke_step(qsmoke_ctx* ctx, uint64_t n_steps);
/* Kernels this ctx launched (all entry points), for the bench's claim. */
qmpm_status qsmoke_launch_count(const qsmoke_ctx* ctx, uint64_t* launches);

#ifdef __cplusplus
}
#endif
#endif
