/*
 * qmpm.h -- C ABI of libqmpm: the quantized MLS-MPM hot path of Liu et al.,
 * "Automatic Quantization for Physics-Based Simulation" (arXiv 2207.04658), on B200.
 *
 * Citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
 * readings Qn = DESIGN.md §2.
 *
 * Conventions for every entry point:
 *   - Return value: qmpm_status, QMPM_OK (0) on success.  On failure a message
 *     is available from qmpm_last_error(ctx) (ctx may be NULL: thread-local).
 *   - Pointers marked "host or device" may be either; the library inspects them
 *     with cudaPointerGetAttributes and copies through pinned staging if needed.
 *     Pointers marked "device" must be device memory on the ctx's device.
 *   - The caller owns every pointer it passes; the library never frees caller
 *     memory.  The library allocates only in qmpm_create (records, sort scratch,
 *     grid pool, counters, optional debug/id buffers), sized from max_particles.
 *   - A ctx is single-owner and single-stream: all work is enqueued on the stream
 *     given to qmpm_create; calls marked "synchronizes" block until it drains.
 *   - Device-side conditions (non-finite values, out-of-domain particles, grid
 *     pool overflow) are COUNTED on the device; pool overflow additionally sets a
 *     sticky error that the next synchronizing call returns as QMPM_ECAPACITY.
 *     Saturation of a fixed-point field is only counted.
 */
#ifndef QMPM_H
#define QMPM_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QMPM_ABI_VERSION 1
#define QMPM_MAX_FIELDS 64

typedef struct qmpm_ctx qmpm_ctx; /* opaque; owns all device pools */
typedef int32_t qmpm_status;

enum {
    QMPM_OK = 0,
    QMPM_EINVAL = 1,     /* bad argument (null pointer, size, dim, material...) */
    QMPM_ELAYOUT = 2,    /* scheme cannot be laid out (width 0 or > 32; missing scalar) */
    QMPM_ENOMEM = 3,     /* device allocation failed */
    QMPM_ECUDA = 4,      /* CUDA runtime error */
    QMPM_ENCCL = 5,      /* NCCL error in the slab exchange */
    QMPM_ENONFINITE = 6, /* the encoder met non-finite values (encoded as code 0, counted) */
    QMPM_EDOMAIN = 7,    /* a particle moved more than one slab in a step; the error-bounded
                            solver cannot meet its bound within b_max.  (Particles whose base
                            leaves the grid are clamped and only counted: S:263, Q14.) */
    QMPM_ECAPACITY = 8,  /* n > max_particles, grid pool or migration buffer overflow */
    QMPM_ESTATE = 9      /* call not valid in the ctx's current state (e.g. a sticky error) */
};

/* Field kinds.  FIXED: Eq. 3, u = round(v/Delta) stored as frac_bits+1-bit
 * two's complement (reading Q2), Delta = range * 2^-frac_bits, value =
 * offset + u*Delta (offset: reading Q21).  RAW_F32: the IEEE bits (32 bits).
 * SHARED_EXP (reading Q4): a group -- a maximal run of consecutive SHARED_EXP fields
 * with equal `group` ids -- shares one unsigned exp_bits-bit exponent E, stored in
 * front of the group's first mantissa; each member is a frac_bits+1-bit two's
 * complement mantissa u with value u * range * 2^(E - frac_bits) (range = R_min, a
 * power of two).  The encoder picks the smallest E in [0, 2^exp_bits - 1] with
 * max |v| < R_min 2^E, raises it once if a member's rounding overflows, and
 * saturates at the top.  Members share frac_bits (<= 23), exp_bits (1..8), range;
 * offset must be 0.  The paper's types are fixed-point; the shared exponent
 * is the north star's "shared-exponent fields". */
enum { QMPM_FIXED = 0, QMPM_RAW_F32 = 1, QMPM_SHARED_EXP = 2 };
/* Attributes of a particle: position, velocity, deformation
 * gradient (elastic), its determinant J (fluid), affine velocity C. */
enum { QMPM_X = 0, QMPM_V = 1, QMPM_F = 2, QMPM_C = 3, QMPM_J = 4 };
/* Rounding at every store of steps >= 1: Eq. 11 dithering or
 * round-half-even (the undithered ablation, T-dither-perf P:767-786). */
enum { QMPM_RNE = 0, QMPM_DITHER = 1 };
/* Materials: fixed-corotated elastic, J-tracking fluid (reading Q15). */
enum { QMPM_ELASTIC_FCR = 0, QMPM_FLUID_J = 1 };
/* qmpm_params.flags */
enum {
    QMPM_TRACK_IDS = 1u << 0,       /* keep a u32 particle id alongside each record */
    QMPM_DEBUG_PREENCODE = 1u << 1, /* keep the last step's fp32 state before encode */
    QMPM_NO_ROUND_COUNTERS = 1u << 2, /* skip the per-field round-up/down counters */
    QMPM_RECORD_RANGES = 1u << 3      /* fold max |value| per state scalar into qmpm_read_ranges */
};

/* One quantized quantity h: one scalar component of one attribute.
 * Fields are bit-packed contiguously in array order, LSB-first, each particle
 * record starting at a fresh 32-bit word (bit pack; reading Q10). */
typedef struct {
    uint8_t attr;      /* QMPM_X .. QMPM_J */
    uint8_t comp;      /* component: 0..d-1 for x, v; row-major 0..d*d-1 for F, C; 0 for J */
    uint8_t kind;      /* QMPM_FIXED | QMPM_RAW_F32 | QMPM_SHARED_EXP */
    uint8_t frac_bits; /* b; FIXED width = b+1 in [1, 32] */
    float range;       /* R > 0 (FIXED) */
    float offset;      /* value = offset + u*Delta (FIXED) */
    uint8_t exp_bits, group, pad[2]; /* SHARED_EXP: exponent width (1..8) and group id */
} qmpm_field;

/* A quantization scheme {(b_h, R_h)} (Alg. 1 output) plus packing order. */
typedef struct {
    uint32_t dim;      /* 2 or 3 */
    uint32_t material; /* QMPM_ELASTIC_FCR | QMPM_FLUID_J */
    uint32_t n_fields; /* must cover every state scalar exactly once (see below) */
    uint32_t rounding; /* QMPM_DITHER | QMPM_RNE */
    const qmpm_field* fields; /* host pointer, n_fields entries, packing order */
    uint64_t dither_seed;     /* seed of the content-keyed dither hash (reading Q5) */
    uint32_t layout_policy;   /* 0 = bit pack (fields may straddle words); 1 = no field
                                 straddles a word (the bit struct's rule): a field that would
                                 cross a word boundary starts at the next word */
    uint32_t pad;
} qmpm_scheme;

/* Scene parameters of the MLS-MPM step. */
typedef struct {
    int32_t grid_res[3]; /* nodes per axis (grid_res[2] ignored in 2D) */
    float dx, dt;        /* cell size, time step */
    float gravity[3];
    float p_rho, p_vol;  /* particle density and volume; m_p = p_rho * p_vol */
    float E, nu;         /* Young's modulus (fluid: bulk stiffness), Poisson ratio */
    int32_t bound;       /* separating-wall thickness in nodes (reading Q13) */
    uint32_t flags;      /* QMPM_TRACK_IDS | QMPM_DEBUG_PREENCODE | QMPM_NO_ROUND_COUNTERS */
    uint64_t max_particles;
    uint64_t pool_blocks; /* grid-pool capacity in blocks (4^3 nodes 3D, 8^2 2D); 0 = auto */
} qmpm_params;

typedef struct {
    uint64_t step;          /* steps taken since set_state (set_words sets it) */
    uint64_t n_particles;
    uint64_t saturations[QMPM_MAX_FIELDS]; /* per field, cumulative */
    uint64_t round_up[QMPM_MAX_FIELDS];    /* per field: u > v/Delta (T-dither-eff) */
    uint64_t round_down[QMPM_MAX_FIELDS];  /* per field: u < v/Delta */
    uint64_t nonfinite;     /* non-finite values met by the encoder */
    uint64_t out_of_domain; /* particle-steps whose base was clamped (reading Q14) */
    uint64_t active_blocks; /* grid blocks holding particles, last step */
    uint64_t touched_blocks;/* grid blocks in the pool (active + their upper neighbours), last step */
    uint64_t pool_overflow; /* steps whose touched blocks exceeded pool_blocks */
} qmpm_stats_t;

/*
 * State scalar order used by qmpm_set_state / qmpm_read_state / qmpm_read_debug
 * ("vals" as [n][n_scalars] fp32, row-major): x[d], v[d], then F[d*d] row-major
 * (elastic) or J (fluid), then C[d*d] row-major.  n_scalars = 2d + 2d^2 (elastic)
 * or 2d + 1 + d^2 (fluid): 3D elastic 24, 3D fluid 16, 2D elastic 12, 2D fluid 9.
 * This order is independent of the packing order.
 */

/* Layout of a scheme (bit pack): words per particle record, bits used,
 * and each field's bit offset (nullable; n_fields entries).  Pure host function.
 * QMPM_ELAYOUT if a width is 0 or > 32 or a kind is unsupported. */
qmpm_status qmpm_layout(const qmpm_scheme* scheme, uint32_t* words_per_particle,
                        uint32_t* bits_used, uint32_t* bit_offsets);

/* Create a single-GPU context on the current CUDA device; all work goes to
 * cuda_stream (a cudaStream_t; NULL = legacy default stream).  Validates the
 * scheme (every state scalar stored exactly once), uploads its constants and
 * allocates every pool.  *out receives the ctx. */
qmpm_status qmpm_create(const qmpm_params* params, const qmpm_scheme* scheme, void* cuda_stream,
                        qmpm_ctx** out);
qmpm_status qmpm_destroy(qmpm_ctx* ctx); /* synchronizes; NULL is a no-op */

/* Replace the state with n particles given as fp32 scalars (host or device,
 * [n][n_scalars]); encoded with round-half-even at step 0 (reading Q20); the
 * step counter and all stats are reset; ids become 0..n-1. */
qmpm_status qmpm_set_state(qmpm_ctx* ctx, uint64_t n, const float* vals);
/* Append n particles (same encoding) after the current ones, for chunked
 * creation of large scenes; ids continue.  QMPM_ECAPACITY past max_particles. */
qmpm_status qmpm_append_state(qmpm_ctx* ctx, uint64_t n, const float* vals);
/* Replace the state with n packed records (host or device, [n][W] u32) and set
 * the step counter (resume; dithering is keyed by content and step, so a resumed
 * run is bit-identical, reading Q5). */
qmpm_status qmpm_set_words(qmpm_ctx* ctx, uint64_t n, const uint32_t* words, uint64_t step);

/* Overwrite the ids of the current n particles (host or device [n] u32; needs
 * QMPM_TRACK_IDS).  With a slab decomposition, ids must be unique across ranks. */
qmpm_status qmpm_set_ids(qmpm_ctx* ctx, uint64_t n, const uint32_t* ids);

/* Advance n_steps MLS-MPM steps (decode -> bin -> P2G -> grid update -> G2P ->
 * dithered encode), asynchronously on the ctx stream; allocates nothing and never
 * synchronises.  Single GPU: one CUDA-graph launch per step (captured on first use per
 * ping-pong parity; QMPM_NO_GRAPH=1 or qmpm_set_profiling(1) launch kernel by kernel).
 * Device-side conditions (non-finite values met by the encoder, migration overflow,
 * capacity, a two-slab jump) set a sticky status that the next synchronising call
 * (qmpm_read_state, qmpm_stats) reports as QMPM_ENONFINITE / QMPM_ECAPACITY /
 * QMPM_EDOMAIN; qmpm_step then returns QMPM_ESTATE until qmpm_set_state / set_words. */
qmpm_status qmpm_step(qmpm_ctx* ctx, uint32_t n_steps);

/* Read the current particles (synchronizes).  vals: [n][n_scalars] decoded fp32
 * (nullable); words: [n][W] packed records (nullable); ids: [n] (nullable; needs
 * QMPM_TRACK_IDS).  All host or device.  Particles are in the library's storage
 * order (sorted by grid block after a step); use ids to match them.  *n_out = n
 * (a slab rank: the particles it owns now, migrants received, leavers excluded);
 * QMPM_ECAPACITY if capacity < n.  The outputs are filled before a sticky error
 * (see qmpm_step) is returned. */
qmpm_status qmpm_read_state(qmpm_ctx* ctx, float* vals, uint32_t* words, uint32_t* ids,
                            uint64_t capacity, uint64_t* n_out);
/* The last step's fp32 state BEFORE the encode (needs QMPM_DEBUG_PREENCODE), in
 * the same order as qmpm_read_state.  Synchronizes. */
qmpm_status qmpm_read_debug(qmpm_ctx* ctx, float* pre_encode_vals, uint64_t capacity,
                            uint64_t* n_out);
qmpm_status qmpm_stats(qmpm_ctx* ctx, qmpm_stats_t* out); /* synchronizes; fills *out, then
                                                            returns the sticky error if any */

/* Standalone codec (Eq. 3 / Eq. 11 + bit pack) on device arrays, enqueued on
 * cuda_stream.  vals: [n][n_fields] fp32 in PACKING order; words: [n][W].
 * keys: nullable => round-half-even; else dithered with the 16-bit draw r16(seed, step,
 * keys[i], field) of reading Q5 rev. 3 when scheme->rounding == QMPM_DITHER.  The scheme's dim/material are not
 * used and attr/comp are not checked.  counters (nullable, device, 3*64 u64,
 * accumulated): saturations, round-ups, round-downs per field. */
qmpm_status qmpm_encode(const qmpm_scheme* scheme, uint64_t n, const float* vals,
                        const uint32_t* keys, uint64_t step, uint32_t* words,
                        uint64_t* counters, void* cuda_stream);
qmpm_status qmpm_decode(const qmpm_scheme* scheme, uint64_t n, const uint32_t* words, float* vals,
                        void* cuda_stream);
/* The paper's "MatMul" codec task: each record holds a 3x3 matrix M (the
 * scheme's 9 fields, row-major M[r][c] = field 3r+c); it is decoded, multiplied by the
 * constant a (host, 9 floats, row-major) as out[r][c] = (M[r][0] a[c] + M[r][1] a[3+c])
 * + M[r][2] a[6+c] in fp32 (no FMA) and re-encoded into words_out (dithered with
 * keys[i] when keys != NULL and the scheme dithers, else RNE).  Device arrays
 * [n][W]; words_in and words_out must not overlap.  QMPM_ELAYOUT unless 9 fields. */
qmpm_status qmpm_codec_matmul3(const qmpm_scheme* scheme, uint64_t n, const uint32_t* words_in, const float* a,
                               const uint32_t* keys, uint64_t step, uint32_t* words_out, void* cuda_stream);

/* Per-kernel timing for the roofline: when enabled, qmpm_step brackets each
 * kernel with CUDA events on the ctx stream.  qmpm_kernel_times (synchronizes)
 * returns, for each of the QMPM_NUM_KERNELS kernels in the order of
 * qmpm_kernel_name(i), the summed milliseconds and launch count since enabling. */
#define QMPM_NUM_KERNELS 9
qmpm_status qmpm_set_profiling(qmpm_ctx* ctx, int enabled);
qmpm_status qmpm_kernel_times(qmpm_ctx* ctx, double* ms, uint64_t* launches);
const char* qmpm_kernel_name(int i);
/* Total kernels this ctx launched (all entry points), for the bench's claim. */
uint64_t qmpm_launch_count(const qmpm_ctx* ctx);

/* ---- Slab decomposition --------------------------
 * The 3D grid is cut into slabs of z cell planes, one per rank.  A rank owns the
 * particles whose base cell lies in its slab.  Every step: P2G partial sums of the
 * ghost block plane above the slab are added into the upper neighbour; the upper
 * neighbour's updated velocities of that plane come back; particles whose base
 * leaves the slab migrate to the neighbour (CFL keeps migration to one hop). */
typedef struct {
    int32_t nranks, rank;
    int32_t z0, z1;            /* owned cell planes [z0, z1): multiples of 4 (z1 may be grid_res[2]) */
    uint64_t migrate_capacity; /* particles per direction per step (the fixed migration buffer);
                                  0 = max(65536, min(max_particles / 256, 2^22)).  The exchanges
                                  are fixed-size, so the ranks of one run agree on ONE capacity:
                                  qmpm_connect_nccl (one all-reduce) and qmpm_step_group re-size
                                  every rank's buffers to the largest value of the ranks */
} qmpm_slab;

/* Like qmpm_create, for rank `slab->rank` of `slab->nranks` (3D only).  Particles
 * given to qmpm_set_state must lie in this slab or an adjacent one (they are routed
 * to their owner during the first step).  QMPM_EINVAL for a bad slab. */
qmpm_status qmpm_create_slab(const qmpm_params* params, const qmpm_scheme* scheme, void* cuda_stream,
                             const qmpm_slab* slab, qmpm_ctx** out);
/* NCCL transport (one process per GPU): rank 0 creates the unique id, the caller
 * broadcasts it (e.g. torch.distributed), every rank connects; qmpm_step then
 * exchanges, with grouped ncclSend/ncclRecv of FIXED sizes (the schedule never depends
 * on data; no host synchronisation): the ghost-plane partial sums (on a comm stream,
 * overlapping the interior P2G), the velocity plane (overlapping the interior G2P) and
 * the migration buffers, plus an all-reduce of the sticky status so that every rank
 * reports an error at its next synchronising call.  QMPM_ENCCL on failure (including a
 * missing libnccl.so.2). */
qmpm_status qmpm_get_unique_id(uint8_t id[128]);
qmpm_status qmpm_connect_nccl(qmpm_ctx* ctx, const uint8_t id[128]);
/* The one-call form: qmpm_create_slab for rank `rank` of `nranks` with
 * the cell planes [slab_cuts[rank], slab_cuts[rank + 1]) (host array of nranks + 1
 * increasing block-plane cuts from 0 to grid_res[2]), then qmpm_connect_nccl with the
 * broadcast id.  QMPM_EINVAL for bad cuts / rank, QMPM_ENCCL if the connect fails (the
 * ctx is destroyed). */
qmpm_status qmpm_create_dist(const qmpm_params* params, const qmpm_scheme* scheme, void* cuda_stream, int nranks,
                             int rank, const uint8_t id[128], const int32_t* slab_cuts, qmpm_ctx** out);
/* In-process transport: advance all slabs of one decomposition that live in this
 * process (ctxs[r] = rank r of n, one shared stream), exchanging with device copies.
 * Synchronizes once per step. */
qmpm_status qmpm_step_group(qmpm_ctx* const* ctxs, int n, uint32_t n_steps);

/* ---- Scheme derivation (Algorithm 1) ------------
 * Range recording, Alg. 1 line 9 "Update R_1...R_H according to s_{t+1}":
 * with params.flags |= QMPM_RECORD_RANGES every step's G2P folds max |value| of each
 * state scalar of s_{t+1} (the fp32 value before its encode) into a device
 * accumulator.  qmpm_read_ranges copies it to max_abs (host, [n_scalars], scalar
 * order of qmpm_set_state) and zeroes it when reset != 0.  Synchronizes.  The paper
 * records on the full-precision run and multiplies by a factor, e.g. 2.
 * QMPM_ESTATE without the flag. */
qmpm_status qmpm_read_ranges(qmpm_ctx* ctx, float* max_abs, int reset);

/* Predicted error, Eq. 8: *sigma_out = sqrt(1/12 sum_h delta[h]^2 g[h]).
 * H quantities; host arrays; g = the accumulated squared gradients (caller-supplied). */
qmpm_status qmpm_predict_error(uint32_t H, const double* delta, const double* g, double* sigma_out);
/* Error-bounded scheme (Eq. 6/9; Algorithm 1 lines 13-15):
 * delta_out[h] = sqrt(12 P_h (eps_err z)^2 / (g_h sum P)), bits_out[h] = frac bits
 * ceil(-log2(delta/R_h)) clamped to [b_min, b_max] (0 <= b_min <= b_max <= 31).
 * P_h > 0 (variables of type h), g_h >= 0 (a type with g_h = 0 gets b_min and
 * delta = inf), R_h > 0 (ranges), z != 0 the reference metric, eps_err > 0.  Host
 * arrays, no GPU.  QMPM_EINVAL (message in qmpm_last_error(NULL)) on bad input;
 * QMPM_EDOMAIN when the b_max clamp leaves sigma_pred (Eq. 8, with the clamped widths)
 * above eps_err |z| -- the outputs are still filled with the clamped scheme. */
qmpm_status qmpm_solve_error_bounded(uint32_t H, const double* P, const double* g, const double* R, double z,
                                     double eps_err, int32_t b_min, int32_t b_max, double* delta_out,
                                     int32_t* bits_out);
/* Memory-bounded scheme (Eq. 7): minimise E[dz] subject to
 * sum_h P_h bits[h] <= budget_bits (FRACTION bits: the stored width is bits + 1, so a
 * physical budget eps_mem * M is budget_bits = eps_mem * M - sum_h P_h).  Closed form
 * of SPEC.md:342 (the paper's is in its supplement): delta_h = c sqrt(P_h/g_h),
 * bits = floor(-log2(delta/R_h)) over the box [b_min, b_max] by an active set (a width
 * the closed form puts outside the box is fixed at the bound and the others re-solved
 * with the budget left); types with g_h = 0 take b_min.  QMPM_EINVAL when the budget
 * cannot hold b_min everywhere. */
qmpm_status qmpm_solve_memory_bounded(uint32_t H, const double* P, const double* g, const double* R,
                                      double budget_bits, int32_t b_min, int32_t b_max, double* delta_out,
                                      int32_t* bits_out);

const char* qmpm_last_error(const qmpm_ctx* ctx);
int qmpm_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* QMPM_H */
