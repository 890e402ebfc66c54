/*
 * codec.c -- oracle codec: bit-pack layout, fixed-point encode/decode with and
 * without dithering, and the counter-based dither RNG.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Compiled with -ffp-contract=off so
 * that every float operation below is a single correctly-rounded IEEE op.
 *
 * Readings of the paper used here (all listed in DESIGN.md "Readings"):
 *   - Eq. 3: u = round(v/Delta), v' = u*Delta, Delta = 2^-b R.
 *     Stored as b+1-bit two's complement (reading Q2), saturating.
 *     t = v/Delta is computed as ONE fp32 multiply by a host-rounded 1/Delta,
 *     no FMA (reading Q3).  Undithered ties round half to even (reading Q6).
 *   - Eq. 11: u = floor(v/Delta + xi) rounded, xi ~ U(-1/2,1/2); evaluated
 *     exactly as u = f + [y >= 1 - r], f = floor(t), y = t - f, r = r16 * 2^-16,
 *     which is floor(t + r) in real arithmetic (reading Q6), so P(up) = y to within
 *     2^-16.
 *   - Bit pack (Fig. bit_pack_operation): fields placed
 *     contiguously in declaration order, LSB-first, records word-aligned
 *     (reading Q10); a field may straddle two words.
 *   - RNG (P:811's generator is in an unavailable supplement): lowbias32 hash,
 *     keyed by (seed, step, particle content key, field) -- reading Q5.
 */
#include "oracle.h"
#include <math.h>
#include <string.h>

/* The public "lowbias32" integer hash (reading Q5). */
uint32_t oracle_mix32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

/* 16-bit uniform integer for (seed, step, particle key, field index): reading Q5,
 * revision 3 (one 32-bit hash per PAIR of fields, f = 2p and f = 2p + 1):
 *   salt = mix(seed_lo ^ mix(seed_hi ^ mix(step)))   (step taken mod 2^32)
 *   h    = mix(key ^ salt)
 *   z    = x ^ (x >> 16),  x = ((h ^ p * 0x9E3779B9) * 0x7feb352d ^ ...) -- written out
 *          below: the lowbias32 rounds on the pair-salted particle hash
 *   even field: r16 = bits 7..22 of z;  odd field: r16 = bits 7..22 of z rotated right
 *   by 16 (= bits 23..31 and 0..6 of z).
 * Each step is a bijection of h and the two fields of a pair take disjoint bits of z, so
 * for a uniform h every r16 is exactly uniform and the pair is exactly jointly uniform. */
uint32_t oracle_pair_hash(uint64_t seed, uint64_t step, uint32_t key, uint32_t pair) {
    uint32_t seed_lo = (uint32_t)(seed & 0xffffffffu);
    uint32_t seed_hi = (uint32_t)(seed >> 32);
    uint32_t salt = oracle_mix32(seed_lo ^ oracle_mix32(seed_hi ^ oracle_mix32((uint32_t)step)));
    uint32_t h = oracle_mix32(key ^ salt);
    uint32_t x = h ^ (pair * 0x9E3779B9u);
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

uint32_t oracle_r16(uint64_t seed, uint64_t step, uint32_t key, uint32_t field) {
    uint32_t z = oracle_pair_hash(seed, step, key, field >> 1);
    if (field & 1u) z = (z >> 16) | (z << 16); /* rotate right by 16 */
    return (z >> 7) & 0xffffu;
}

void oracle_r16_batch(uint64_t seed, uint64_t step, uint64_t n, const uint32_t* keys, uint32_t field,
                      uint32_t* out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = oracle_r16(seed, step, keys[i], field);
}

/* SHARED_EXP groups (reading Q4): a maximal run of consecutive SHARED_EXP fields with
 * equal group ids.  The first member stores the group exponent in front of its
 * mantissa. */
static int group_first(const oracle_scheme* s, uint32_t f) {
    return s->kind[f] == ORACLE_SHARED_EXP &&
           (f == 0 || s->kind[f - 1] != ORACLE_SHARED_EXP || s->group[f - 1] != s->group[f]);
}
static uint32_t group_start(const oracle_scheme* s, uint32_t f) {
    while (!group_first(s, f)) --f;
    return f;
}
static uint32_t group_last(const oracle_scheme* s, uint32_t f) {
    while (f + 1 < s->n_fields && s->kind[f + 1] == ORACLE_SHARED_EXP && !group_first(s, f + 1)) ++f;
    return f;
}

static uint32_t field_width(const oracle_scheme* s, uint32_t f) {
    if (s->kind[f] == ORACLE_RAW_F32) return 32;
    if (s->kind[f] == ORACLE_SHARED_EXP) return s->frac_bits[f] + 1 + (group_first(s, f) ? s->exp_bits[f] : 0);
    return s->frac_bits[f] + 1;
}

static int is_pow2(float r) {
    int e;
    return r > 0.0f && isfinite(r) && frexpf(r, &e) == 0.5f;
}

/* Layout: offset_k = sum_{j<k} width_j; W = ceil(total/32).
 * Returns 0, or -1 if a width is 0 or > 32 or the field count is bad. */
int oracle_layout(const oracle_scheme* s, uint32_t* offsets, uint32_t* words, uint32_t* bits) {
    if (s->n_fields == 0 || s->n_fields > ORACLE_MAX_FIELDS) return -1;
    uint32_t total = 0;
    for (uint32_t f = 0; f < s->n_fields; ++f) {
        if (s->kind[f] != ORACLE_FIXED && s->kind[f] != ORACLE_RAW_F32 && s->kind[f] != ORACLE_SHARED_EXP) return -1;
        if (s->kind[f] == ORACLE_SHARED_EXP) { /* members share b, e and R_min; e in 1..8 */
            uint32_t g0 = group_start(s, f);
            if (s->exp_bits[f] < 1 || s->exp_bits[f] > 8 || s->frac_bits[f] != s->frac_bits[g0] ||
                s->exp_bits[f] != s->exp_bits[g0] || s->range[f] != s->range[g0] || !is_pow2(s->range[f]) ||
                s->offset[f] != 0.0f)
                return -1;
        }
        uint32_t w = field_width(s, f);
        if (w == 0 || w > 32) return -1;
        /* layout policy 1, the bit struct's rule ("it does not allow custom data
         * types to span across two physical words"): a field that would straddle starts
         * at the next word (Fig. bit_struct: three 17-bit fields take 3 words) */
        if (s->layout_policy == 1 && (total % 32) + w > 32) total = (total + 31) / 32 * 32;
        if (s->layout_policy > 1) return -1;
        if (offsets) offsets[f] = total;
        total += w;
    }
    if (bits) *bits = total;
    if (words) *words = (total + 31) / 32;
    return 0;
}

/* Bit i of a record is bit (i mod 32) of word floor(i/32) (LSB-first).
 * Written one bit at a time so the rule can be checked by eye. */
uint32_t oracle_get_bits(const uint32_t* rec, uint32_t offset, uint32_t width) {
    uint32_t v = 0;
    for (uint32_t j = 0; j < width; ++j) {
        uint32_t i = offset + j;
        uint32_t bit = (rec[i / 32] >> (i % 32)) & 1u;
        v |= bit << j;
    }
    return v;
}

void oracle_put_bits(uint32_t* rec, uint32_t offset, uint32_t width, uint32_t value) {
    for (uint32_t j = 0; j < width; ++j) {
        uint32_t i = offset + j;
        uint32_t bit = (value >> j) & 1u;
        rec[i / 32] = (rec[i / 32] & ~(1u << (i % 32))) | (bit << (i % 32));
    }
}

/* Delta = fl32(R * 2^-b) (exact: power-of-two scaling), 1/Delta = fl32(2^b / R). */
static float delta_of(uint32_t b, float range) { return (float)ldexp((double)range, -(int)b); }
static float inv_delta_of(uint32_t b, float range) {
    return (float)(ldexp(1.0, (int)b) / (double)range);
}

/* Eq. 3 / Eq. 11 encode of one fp32 value.  Returns the saturated integer code u.
 * Counters: sat when clamped; up when u > t, down when u < t (T-dither-eff,
 * P:735-738; values exactly on the grid count as neither); nonfinite => u = 0. */
int64_t oracle_encode_value(float v, uint32_t frac_bits, float range, float offset, int dithered,
                            uint32_t r16, uint64_t* sat, uint64_t* up, uint64_t* down,
                            uint64_t* nonfinite) {
    if (!isfinite(v)) {
        if (nonfinite) (*nonfinite)++;
        return 0;
    }
    float inv_delta = inv_delta_of(frac_bits, range);
    float a = (offset != 0.0f) ? (v - offset) : v; /* fp32 subtract */
    float t = a * inv_delta;                        /* fp32 multiply, no FMA (Q3) */
    double ud;
    if (dithered) {
        float f = floorf(t);
        float y = t - f;                                       /* exact */
        float one_minus_r = (float)(65536u - r16) * 0x1p-16f; /* exact */
        int is_up = (y >= one_minus_r);
        ud = (double)f + (double)is_up;
        if (is_up) {
            if (up) (*up)++;
        } else if (y > 0.0f) {
            if (down) (*down)++;
        }
    } else {
        float rr = rintf(t); /* round half to even in the default FP environment */
        if (rr > t && up) (*up)++;
        if (rr < t && down) (*down)++;
        ud = (double)rr;
    }
    double lo = -ldexp(1.0, (int)frac_bits);
    double hi = ldexp(1.0, (int)frac_bits) - 1.0;
    if (ud < lo) {
        ud = lo;
        if (sat) (*sat)++;
    } else if (ud > hi) {
        ud = hi;
        if (sat) (*sat)++;
    }
    return (int64_t)ud;
}

/* phi^{-1}(u) = u * Delta (Eq. 3), then + offset (reading Q21), each fp32-rounded. */
float oracle_decode_value(int32_t u, uint32_t frac_bits, float range, float offset) {
    float d = delta_of(frac_bits, range);
    float x = (float)u * d;
    if (offset != 0.0f) x = x + offset;
    return x;
}

static int32_t sign_extend(uint32_t raw, uint32_t width) {
    if (width == 32) return (int32_t)raw;
    uint32_t sign = 1u << (width - 1);
    if (raw & sign) return (int32_t)(raw | ~((sign << 1) - 1u));
    return (int32_t)raw;
}

/* One SHARED_EXP group [f0, f1] of a record (reading Q4).  M = max |v| over the finite
 * members; E = the smallest exponent in [0, 2^e - 1] with M < R_min 2^E; the members
 * are encoded by the FIXED rule with range R_min 2^E (Delta_E = R_min 2^(E - b), exact);
 * if a member's code would saturate and E < 2^e - 1, E is raised by one and the group
 * re-encoded.  At E = 2^e - 1 codes saturate (counted). */
static void encode_group(const oracle_scheme* s, const uint32_t* offsets, uint32_t f0, uint32_t f1,
                         const float* vals, int dithered, uint32_t key, uint64_t step, uint32_t* rec,
                         uint64_t* counters) {
    uint32_t b = s->frac_bits[f0], e = s->exp_bits[f0], emax = (1u << e) - 1u;
    float R = s->range[f0];
    float M = 0.0f;
    for (uint32_t f = f0; f <= f1; ++f)
        if (isfinite(vals[f]) && fabsf(vals[f]) > M) M = fabsf(vals[f]);
    uint32_t E = 0;
    while (E < emax && !(M < ldexpf(R, (int)E))) ++E;
    for (;;) {
        uint64_t sat = 0;
        for (uint32_t f = f0; f <= f1; ++f) {
            uint32_t r16 = dithered ? oracle_r16(s->dither_seed, step, key, f) : 0;
            oracle_encode_value(vals[f], b, ldexpf(R, (int)E), 0.0f, dithered, r16, &sat, 0, 0, 0);
        }
        if (sat == 0 || E == emax) break;
        ++E;
    }
    oracle_put_bits(rec, offsets[f0], e, E);
    for (uint32_t f = f0; f <= f1; ++f) {
        uint32_t r16 = dithered ? oracle_r16(s->dither_seed, step, key, f) : 0;
        int64_t u = oracle_encode_value(vals[f], b, ldexpf(R, (int)E), 0.0f, dithered, r16,
                                        counters ? &counters[f] : 0, counters ? &counters[64 + f] : 0,
                                        counters ? &counters[128 + f] : 0, counters ? &counters[192] : 0);
        uint32_t width = b + 1, mask = (width == 32) ? 0xffffffffu : ((1u << width) - 1u);
        oracle_put_bits(rec, offsets[f] + (f == f0 ? e : 0), width, (uint32_t)u & mask);
    }
}

static void encode_record(const oracle_scheme* s, const uint32_t* offsets, uint32_t W,
                          const float* vals /* packing order */, int dithered, uint32_t key,
                          uint64_t step, uint32_t* rec, uint64_t* counters) {
    for (uint32_t w = 0; w < W; ++w) rec[w] = 0;
    for (uint32_t f = 0; f < s->n_fields; ++f) {
        float v = vals[f];
        if (s->kind[f] == ORACLE_SHARED_EXP) {
            if (group_first(s, f)) encode_group(s, offsets, f, group_last(s, f), vals, dithered, key, step, rec,
                                                counters);
            continue;
        }
        if (s->kind[f] == ORACLE_RAW_F32) {
            if (!isfinite(v) && counters) counters[192]++;
            uint32_t bits;
            memcpy(&bits, &v, 4);
            oracle_put_bits(rec, offsets[f], 32, bits);
            continue;
        }
        uint32_t r16 = dithered ? oracle_r16(s->dither_seed, step, key, f) : 0;
        int64_t u = oracle_encode_value(v, s->frac_bits[f], s->range[f], s->offset[f], dithered,
                                        r16, counters ? &counters[f] : 0,
                                        counters ? &counters[64 + f] : 0,
                                        counters ? &counters[128 + f] : 0,
                                        counters ? &counters[192] : 0);
        uint32_t width = s->frac_bits[f] + 1;
        uint32_t mask = (width == 32) ? 0xffffffffu : ((1u << width) - 1u);
        oracle_put_bits(rec, offsets[f], width, (uint32_t)u & mask);
    }
}

int oracle_encode(const oracle_scheme* s, uint64_t n, const float* vals, const uint32_t* keys,
                  uint64_t step, uint32_t* words, uint64_t* counters) {
    uint32_t offsets[ORACLE_MAX_FIELDS], W, bits;
    if (oracle_layout(s, offsets, &W, &bits)) return -1;
    int dithered = (keys != 0) && (s->rounding == ORACLE_DITHER);
    for (uint64_t i = 0; i < n; ++i)
        encode_record(s, offsets, W, vals + i * s->n_fields, dithered, keys ? keys[i] : 0, step,
                      words + i * W, counters);
    return 0;
}

static float decode_field(const oracle_scheme* s, const uint32_t* offsets, const uint32_t* rec,
                          uint32_t f) {
    if (s->kind[f] == ORACLE_SHARED_EXP) { /* reading Q4: u * R_min 2^(E - b) */
        uint32_t g0 = group_start(s, f), e = s->exp_bits[f], width = s->frac_bits[f] + 1;
        uint32_t E = oracle_get_bits(rec, offsets[g0], e);
        int32_t u = sign_extend(oracle_get_bits(rec, offsets[f] + (f == g0 ? e : 0), width), width);
        return oracle_decode_value(u, s->frac_bits[f], ldexpf(s->range[f], (int)E), 0.0f);
    }
    if (s->kind[f] == ORACLE_RAW_F32) {
        uint32_t bits = oracle_get_bits(rec, offsets[f], 32);
        float v;
        memcpy(&v, &bits, 4);
        return v;
    }
    uint32_t width = s->frac_bits[f] + 1;
    int32_t u = sign_extend(oracle_get_bits(rec, offsets[f], width), width);
    return oracle_decode_value(u, s->frac_bits[f], s->range[f], s->offset[f]);
}

int oracle_decode(const oracle_scheme* s, uint64_t n, const uint32_t* words, float* vals) {
    uint32_t offsets[ORACLE_MAX_FIELDS], W, bits;
    if (oracle_layout(s, offsets, &W, &bits)) return -1;
    for (uint64_t i = 0; i < n; ++i)
        for (uint32_t f = 0; f < s->n_fields; ++f)
            vals[i * s->n_fields + f] = decode_field(s, offsets, words + i * W, f);
    return 0;
}

int oracle_n_scalars(int dim, int material) {
    return material == ORACLE_FLUID ? 2 * dim + 1 + dim * dim : 2 * dim + 2 * dim * dim;
}

/* Particle key (reading Q5): k = 0; for each record word holding any bit of an
 * x field (scalars 0..dim-1), in ascending word order: k = (k ^ word) * 0x9E3779B1 (rev. 3;
 * an odd multiply per word, the particle hash mix(key ^ salt) does the mixing). */
uint32_t oracle_particle_key(const oracle_scheme* s, int dim, const uint32_t* rec) {
    uint32_t offsets[ORACLE_MAX_FIELDS], W, bits;
    if (oracle_layout(s, offsets, &W, &bits)) return 0;
    uint32_t k = 0;
    for (uint32_t w = 0; w < W; ++w) {
        int holds_x = 0;
        for (uint32_t f = 0; f < s->n_fields; ++f) {
            if (s->scalar[f] >= (uint32_t)dim) continue;
            uint32_t first = offsets[f] / 32, last = (offsets[f] + field_width(s, f) - 1) / 32;
            if (w >= first && w <= last) holds_x = 1;
        }
        if (holds_x) k = (k ^ rec[w]) * 0x9E3779B1u; /* reading Q5 rev. 3: multiply-xor fold */
    }
    return k;
}

/* scheme must store every state scalar exactly once */
static int check_scalars(const oracle_scheme* s, int ns) {
    if ((int)s->n_fields != ns) return -1;
    int seen[ORACLE_MAX_FIELDS] = {0};
    for (uint32_t f = 0; f < s->n_fields; ++f) {
        if ((int)s->scalar[f] >= ns) return -1;
        if (seen[s->scalar[f]]++) return -1;
    }
    return 0;
}

int oracle_decode_state(const oracle_scheme* s, int dim, int material, uint64_t n,
                        const uint32_t* words, float* state) {
    uint32_t offsets[ORACLE_MAX_FIELDS], W, bits;
    int ns = oracle_n_scalars(dim, material);
    if (oracle_layout(s, offsets, &W, &bits) || check_scalars(s, ns)) return -1;
    for (uint64_t i = 0; i < n; ++i)
        for (uint32_t f = 0; f < s->n_fields; ++f)
            state[i * ns + s->scalar[f]] = decode_field(s, offsets, words + i * W, f);
    return 0;
}

/* keys nullable => RNE (used for set_state, step 0, reading Q20) */
int oracle_encode_state(const oracle_scheme* s, int dim, int material, uint64_t n,
                        const float* state, uint64_t step, const uint32_t* keys,
                        uint32_t* words, uint64_t* counters) {
    uint32_t offsets[ORACLE_MAX_FIELDS], W, bits;
    int ns = oracle_n_scalars(dim, material);
    if (oracle_layout(s, offsets, &W, &bits) || check_scalars(s, ns)) return -1;
    int dithered = (keys != 0) && (s->rounding == ORACLE_DITHER);
    float vals[ORACLE_MAX_FIELDS];
    for (uint64_t i = 0; i < n; ++i) {
        for (uint32_t f = 0; f < s->n_fields; ++f) vals[f] = state[i * ns + s->scalar[f]];
        encode_record(s, offsets, W, vals, dithered, keys ? keys[i] : 0, step, words + i * W,
                      counters);
    }
    return 0;
}
