/*
 * oracle.h -- CPU oracle for the quantized MLS-MPM hot path of
 * Liu et al., "Automatic Quantization for Physics-Based Simulation" (arXiv 2207.04658).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2207_04658_b200/, libqmpm.so) never links, includes or calls it, and
 * this file includes nothing from include/qmpm.h or the CUDA sources.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (the paper's LaTeX source),
 * "S:n" = SPEC.md line n, "SURVEY §8(c)" = /root/repo/SURVEY.md section 8(c),
 * whose readings (Q1..Q22) are restated in DESIGN.md.
 *
 * Parity pins: every function below is pinned by tests/test_oracle_*.py against
 * worked examples, closed forms, invariants or brute force.  The 100-step
 * aggregates are "parity unpinned" beyond those invariants.
 */
#ifndef QMPM_ORACLE_H
#define QMPM_ORACLE_H
#include <stdint.h>

#define ORACLE_MAX_FIELDS 64
#define ORACLE_FIXED 0u
#define ORACLE_RAW_F32 1u
#define ORACLE_SHARED_EXP 2u
#define ORACLE_RNE 0u
#define ORACLE_DITHER 1u
#define ORACLE_ELASTIC 0u
#define ORACLE_FLUID 1u

/* counters[] layout (uint64): [0,64) saturations per field, [64,128) round-ups,
 * [128,192) round-downs, [192] non-finite values, [193] out-of-domain particles. */
#define ORACLE_NCOUNTERS 194

/* A quantization scheme {(b_h, R_h)} (Alg. 1 output) plus packing order
 * (bit pack) and the dither seed (Eq. 11). */
typedef struct {
    uint32_t n_fields;
    uint32_t kind[ORACLE_MAX_FIELDS];      /* ORACLE_FIXED or ORACLE_RAW_F32 */
    uint32_t frac_bits[ORACLE_MAX_FIELDS]; /* b; stored width b+1 (two's complement) */
    float range[ORACLE_MAX_FIELDS];        /* R; Delta = R * 2^-b (Eq. 3) */
    float offset[ORACLE_MAX_FIELDS];       /* value = offset + u*Delta (reading Q21) */
    uint32_t scalar[ORACLE_MAX_FIELDS];    /* which state scalar the field stores */
    uint32_t rounding;                     /* ORACLE_RNE or ORACLE_DITHER */
    uint32_t layout_policy;                /* 0 bit pack; 1 no field straddles a word (bit struct) */
    uint64_t dither_seed;
    /* SHARED_EXP (reading Q4): consecutive fields with the same group id share one
     * exp_bits-bit exponent E stored in front of the group's first mantissa; member
     * values are u * Delta_E, Delta_E = range * 2^(E - b) (range = R_min, a power of 2). */
    uint32_t exp_bits[ORACLE_MAX_FIELDS];
    uint32_t group[ORACLE_MAX_FIELDS];
} oracle_scheme;

/* MLS-MPM scene parameters (reading SURVEY §8(c) C-mpm). */
typedef struct {
    int32_t dim, material;
    int32_t grid_res[3];
    int32_t bound;
    double dx, dt;
    double gravity[3];
    double p_rho, p_vol, E, nu;
} oracle_sim;

/* ---- codec (Eq. 3, Eq. 11, bit pack P:542-549) ---- */
uint32_t oracle_mix32(uint32_t x);
uint32_t oracle_pair_hash(uint64_t seed, uint64_t step, uint32_t key, uint32_t pair);
uint32_t oracle_r16(uint64_t seed, uint64_t step, uint32_t key, uint32_t field);
void oracle_r16_batch(uint64_t seed, uint64_t step, uint64_t n, const uint32_t* keys, uint32_t field,
                      uint32_t* out);
int oracle_layout(const oracle_scheme* s, uint32_t* offsets, uint32_t* words, uint32_t* bits);
uint32_t oracle_get_bits(const uint32_t* rec, uint32_t offset, uint32_t width);
void oracle_put_bits(uint32_t* rec, uint32_t offset, uint32_t width, uint32_t value);
int64_t oracle_encode_value(float v, uint32_t frac_bits, float range, float offset, int dithered,
                            uint32_t r16, uint64_t* sat, uint64_t* up, uint64_t* down,
                            uint64_t* nonfinite);
float oracle_decode_value(int32_t u, uint32_t frac_bits, float range, float offset);
/* vals[n][n_fields] in packing order; keys nullable => RNE regardless of s->rounding */
int oracle_encode(const oracle_scheme* s, uint64_t n, const float* vals, const uint32_t* keys,
                  uint64_t step, uint32_t* words, uint64_t* counters);
int oracle_decode(const oracle_scheme* s, uint64_t n, const uint32_t* words, float* vals);
/* particle dither key: fold of the record words holding any x bit (reading Q5) */
uint32_t oracle_particle_key(const oracle_scheme* s, int dim, const uint32_t* rec);

/* ---- state in scalar order: x[d], v[d], F[d*d] | J, C[d*d] ---- */
int oracle_n_scalars(int dim, int material);
int oracle_decode_state(const oracle_scheme* s, int dim, int material, uint64_t n,
                        const uint32_t* words, float* state);
int oracle_encode_state(const oracle_scheme* s, int dim, int material, uint64_t n,
                        const float* state, uint64_t step, const uint32_t* keys,
                        uint32_t* words, uint64_t* counters);

/* ---- MLS-MPM pieces, fp64 ("truth") and fp32 ("tight comparator") ----
 * Grid is a dense box: node (i,j,k) lives at ((i-o0)*g1 + (j-o1))*g2 + (k-o2),
 * 4 values per node: (m, p_x, p_y, p_z) after P2G; (m, v_x, v_y, v_z) after update.
 * In 2D g2 = 1, o2 = 0 and the 4th value is unused. */
void oracle_p2g_f64(const oracle_sim* sim, uint64_t n, const double* state, const int32_t* origin,
                    const int32_t* gsize, double* grid, uint64_t* oob);
void oracle_grid_update_f64(const oracle_sim* sim, const int32_t* origin, const int32_t* gsize,
                            double* grid);
void oracle_g2p_f64(const oracle_sim* sim, uint64_t n, const double* state_in,
                    const int32_t* origin, const int32_t* gsize, const double* grid,
                    double* state_out);
void oracle_polar_f64(int dim, const double* F, double* R);
int oracle_step_f64(const oracle_sim* sim, const oracle_scheme* s, uint64_t n,
                    const uint32_t* words_in, uint64_t step, double* pre_encode,
                    uint32_t* words_out, uint64_t* counters);
int oracle_step_f32(const oracle_sim* sim, const oracle_scheme* s, uint64_t n,
                    const uint32_t* words_in, uint64_t step, float* pre_encode,
                    uint32_t* words_out, uint64_t* counters);
/* same as step, but P2G/G2P only computed for the particles listed in `sample`
 * (n_sample indices); every particle still contributes to the grid.  Output rows
 * follow `sample` order.  For full-size sampled parity. */
int oracle_step_sampled_f64(const oracle_sim* sim, const oracle_scheme* s, uint64_t n,
                            const uint32_t* words_in, uint64_t step, uint64_t n_sample,
                            const uint64_t* sample, double* pre_encode, uint32_t* words_out);
/* run n_steps full steps (fp64), words in/out may alias */
int oracle_run_f64(const oracle_sim* sim, const oracle_scheme* s, uint64_t n, uint32_t* words,
                   uint64_t first_step, uint32_t n_steps, uint64_t* counters);
/* the same step / run with the particle and node loops on n_threads OpenMP threads
 * (<= 0: all); P2G sums ordered by 4-cell x slab (deterministic, thread-count free) */
int oracle_step_omp_f64(const oracle_sim* sim, const oracle_scheme* s, uint64_t n, const uint32_t* words_in,
                        uint64_t step, double* pre_encode, uint32_t* words_out, uint64_t* counters,
                        int n_threads);
int oracle_run_omp_f64(const oracle_sim* sim, const oracle_scheme* s, uint64_t n, uint32_t* words,
                       uint64_t first_step, uint32_t n_steps, uint64_t* counters, int n_threads);
int oracle_num_threads(void);

#endif
