/*
 * qadjoint.h -- C ABI of the gradient tallies in libqmpm:
 * Algorithm 1 line 12 -- "back propagation and accumulate gradients in g
 * according to Eq. 8" -- on the full-precision simulation (the scheme is
 * linearised at the fp32 run), with the paper's bisection checkpointing.
 *
 *   z   = KE(s_T) = 1/2 m_p sum_p |v_{T,p}|^2             (the evaluation function)
 *   g_h = sum_{t=0..T} sum_p (dz / ds_{t,p,h})^2           (Eq. 8)
 * with one type h per state scalar (x_a, v_a, J | F_ab, C_ab: the order of qmpm.h's state rows).
 * The g_h feed qmpm_solve_error_bounded / qmpm_solve_memory_bounded (qmpm.h).
 *
 * Scope: both materials (QMPM_FLUID_J, reading Q15; QMPM_ELASTIC_FCR, whose
 * adjoint differentiates the polar decomposition), 2D and 3D; the step is the MLS-MPM
 * step of qmpm.h in fp32 on a dense grid of grid_res nodes (16 B per node, 3 grids),
 * state rows fp32 [n][ns] in qmpm.h's scalar order, ns = 2d + 1 + d^2 (fluid) or
 * 2d + 2d^2 (elastic).  DESIGN.md §13.
 *
 * Conventions as qmpm.h.  Device pointers unless marked "host or device"; work goes to
 * the ctx stream; qadj_gradient_tally synchronizes.
 */
#ifndef QADJOINT_H
#define QADJOINT_H
#include "qmpm.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct qadj_ctx qadj_ctx; /* opaque: dense grids + the checkpoint pool */

typedef struct {
    uint32_t max_resident;  /* forward checkpoints held at once by the bisection (s0 included): O(log T) */
    uint32_t peak_buffers;  /* state-sized device buffers in use at once: checkpoints + the
                               adjoints of each recursion level + 2 scratch, ~2 log2 T + 4 */
    uint64_t forward_steps; /* forward steps run (T the first time, then the re-runs): O(T log T) */
    uint64_t adjoint_steps; /* T */
} qadj_stats;

/* A ctx for n particles of dimension dim (2 | 3) and material (QMPM_ELASTIC_FCR |
 * QMPM_FLUID_J); params as qmpm_create's (grid_res, dx, dt, gravity, p_rho, p_vol, E,
 * nu, bound; flags and capacities ignored).  QMPM_EINVAL for bad sizes or an unknown
 * material, QMPM_ENOMEM. */
qmpm_status qadj_create(const qmpm_params* params, int32_t dim, int32_t material, uint64_t n, void* cuda_stream,
                        qadj_ctx** out);
qmpm_status qadj_destroy(qadj_ctx* ctx); /* synchronizes; NULL is a no-op */

/* One fp32 step s_out = F(s_in) (P2G -> grid update -> G2P); s_in != s_out. */
qmpm_status qadj_forward(qadj_ctx* ctx, const float* s_in, float* s_out);
/* One adjoint step lam_t = (d s_{t+1} / d s_t)^T lam_next; when g != NULL
 * (device, ns doubles) sum_p lam_t^2 per scalar is added to it.  lam_t != lam_next. */
qmpm_status qadj_adjoint_step(qadj_ctx* ctx, const float* s_t, const float* lam_next, float* lam_t, double* g);
/* Algorithm 1 lines 8-12 from s0 (host or device [n][ns]): T forward steps, z = KE(s_T),
 * back-propagation with bisection checkpointing, the tallies g (host, ns doubles).  z
 * (host, nullable) receives KE(s_T); lam0 (host or device [n][ns], nullable) dz/ds_0;
 * stats (nullable) the checkpointing counts. */
qmpm_status qadj_gradient_tally(qadj_ctx* ctx, const float* s0, uint32_t T, double* g, double* z, float* lam0,
                                qadj_stats* stats);
/* Kernels this ctx launched, for the bench's claim. */
qmpm_status qadj_launch_count(const qadj_ctx* ctx, uint64_t* launches);

#ifdef __cplusplus
}
#endif
#endif
