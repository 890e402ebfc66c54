/*
 * mpm.c -- oracle MLS-MPM: fp64 and fp32 instantiations of mpm_impl.h, the
 * polar decomposition, a sampled full-size step and a multi-step driver.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).
 */
#include "oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* Polar decomposition F = R S with det R = +1 (fixed corotated).
 * 2D: closed form R = rotation by atan2(F10 - F01, F00 + F11).
 * 3D: SVD via cyclic Jacobi eigen-decomposition of F^T F = V diag(s^2) V^T,
 *     U_i = F v_i / s_i, R = U V^T; if det R < 0 the column of the smallest
 *     singular value is flipped (the rotation-variant SVD).  Library-equivalent;
 *     pinned by tests (R^T R = I, det R = 1, R^T F symmetric). */
void oracle_polar_f64(int dim, const double* F, double* R) {
    if (dim == 2) {
        double x = F[0] + F[3], y = F[2] - F[1];
        double r = sqrt(x * x + y * y);
        double c = 1.0, s = 0.0;
        if (r > 0) { c = x / r; s = y / r; }
        R[0] = c; R[1] = -s; R[2] = s; R[3] = c;
        return;
    }
    double A[3][3], V[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double acc = 0;
            for (int k = 0; k < 3; ++k) acc += F[k * 3 + i] * F[k * 3 + j];
            A[i][j] = acc;
        }
    for (int sweep = 0; sweep < 64; ++sweep) {
        double off = fabs(A[0][1]) + fabs(A[0][2]) + fabs(A[1][2]);
        double diag = fabs(A[0][0]) + fabs(A[1][1]) + fabs(A[2][2]);
        if (off <= 1e-300 || off <= 1e-17 * diag) break;
        for (int p = 0; p < 2; ++p)
            for (int q = p + 1; q < 3; ++q) {
                if (A[p][q] == 0.0) continue;
                double theta = (A[q][q] - A[p][p]) / (2.0 * A[p][q]);
                double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < 3; ++k) { /* A <- A J */
                    double akp = A[k][p], akq = A[k][q];
                    A[k][p] = c * akp - s * akq;
                    A[k][q] = s * akp + c * akq;
                }
                for (int k = 0; k < 3; ++k) { /* A <- J^T A */
                    double apk = A[p][k], aqk = A[q][k];
                    A[p][k] = c * apk - s * aqk;
                    A[q][k] = s * apk + c * aqk;
                }
                for (int k = 0; k < 3; ++k) { /* V <- V J */
                    double vkp = V[k][p], vkq = V[k][q];
                    V[k][p] = c * vkp - s * vkq;
                    V[k][q] = s * vkp + c * vkq;
                }
            }
    }
    /* sort eigenpairs by eigenvalue, descending */
    int idx[3] = {0, 1, 2};
    for (int i = 0; i < 3; ++i)
        for (int j = i + 1; j < 3; ++j)
            if (A[idx[j]][idx[j]] > A[idx[i]][idx[i]]) { int t = idx[i]; idx[i] = idx[j]; idx[j] = t; }
    double sig[3], v[3][3], u[3][3];
    for (int c = 0; c < 3; ++c) {
        double l = A[idx[c]][idx[c]];
        sig[c] = sqrt(l > 0 ? l : 0);
        for (int k = 0; k < 3; ++k) v[c][k] = V[k][idx[c]];
    }
    for (int c = 0; c < 3; ++c) {
        if (c < 2 || sig[2] > 1e-12 * sig[0]) {
            for (int k = 0; k < 3; ++k) {
                double acc = 0;
                for (int m = 0; m < 3; ++m) acc += F[k * 3 + m] * v[c][m];
                u[c][k] = sig[c] > 0 ? acc / sig[c] : (k == c ? 1.0 : 0.0);
            }
        } else { /* degenerate: complete the basis */
            u[2][0] = u[0][1] * u[1][2] - u[0][2] * u[1][1];
            u[2][1] = u[0][2] * u[1][0] - u[0][0] * u[1][2];
            u[2][2] = u[0][0] * u[1][1] - u[0][1] * u[1][0];
        }
    }
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            R[i * 3 + j] = u[0][i] * v[0][j] + u[1][i] * v[1][j] + u[2][i] * v[2][j];
    double detR = R[0] * (R[4] * R[8] - R[5] * R[7]) - R[1] * (R[3] * R[8] - R[5] * R[6]) +
                  R[2] * (R[3] * R[7] - R[4] * R[6]);
    if (detR < 0)
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) R[i * 3 + j] -= 2.0 * u[2][i] * v[2][j];
}

#define REAL double
#define SUF(name) name##_f64
#include "mpm_impl.h"
#undef REAL
#undef SUF

#define REAL float
#define SUF(name) name##_f32
#include "mpm_impl.h"
#undef REAL
#undef SUF

int oracle_run_f64(const oracle_sim* sim, const oracle_scheme* s, uint64_t n, uint32_t* words,
                   uint64_t first_step, uint32_t n_steps, uint64_t* counters) {
    uint32_t W, bits;
    if (oracle_layout(s, 0, &W, &bits)) return -1;
    uint32_t* tmp = (uint32_t*)malloc(sizeof(uint32_t) * W * (n ? n : 1));
    if (!tmp) return -2;
    for (uint32_t t = 0; t < n_steps; ++t) {
        int rc = oracle_step_f64(sim, s, n, words, first_step + t, 0, tmp, counters);
        if (rc) { free(tmp); return rc; }
        memcpy(words, tmp, sizeof(uint32_t) * W * n);
    }
    free(tmp);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Sampled step for full-size parity: the same arithmetic as oracle_step_f64,
 * restricted to the grid nodes the sampled particles read.  A node's value only
 * depends on particles whose base lies within 2 cells of it, so only particles
 * whose base is within 2 cells of a sample's base are scattered.              */

typedef struct { uint64_t* keys; double* vals; uint64_t cap; } hmap;

static uint64_t hkey(int i, int j, int k) {
    return ((uint64_t)(uint32_t)(i + 1024) << 42) | ((uint64_t)(uint32_t)(j + 1024) << 21) |
           (uint64_t)(uint32_t)(k + 1024);
}
static uint64_t hslot(const hmap* h, uint64_t key) {
    uint64_t x = key * 0x9E3779B97F4A7C15ull;
    uint64_t s = (x >> 17) & (h->cap - 1);
    while (h->keys[s] != ~0ull && h->keys[s] != key) s = (s + 1) & (h->cap - 1);
    return s;
}
static double* hget(hmap* h, uint64_t key, int insert) {
    uint64_t s = hslot(h, key);
    if (h->keys[s] == ~0ull) {
        if (!insert) return 0;
        h->keys[s] = key;
    }
    return h->vals ? h->vals + 4 * s : (double*)h->keys; /* non-null marker for sets */
}
static int hinit(hmap* h, uint64_t n, int with_vals) {
    h->cap = 1;
    while (h->cap < 2 * n + 16) h->cap <<= 1;
    h->keys = (uint64_t*)malloc(sizeof(uint64_t) * h->cap);
    h->vals = with_vals ? (double*)calloc(h->cap * 4, sizeof(double)) : 0;
    if (!h->keys || (with_vals && !h->vals)) return -1;
    memset(h->keys, 0xff, sizeof(uint64_t) * h->cap);
    return 0;
}
static void hfree(hmap* h) { free(h->keys); free(h->vals); }

int oracle_step_sampled_f64(const oracle_sim* sim, const oracle_scheme* s, uint64_t n,
                            const uint32_t* words_in, uint64_t step, uint64_t n_sample,
                            const uint64_t* sample, double* pre_encode, uint32_t* words_out) {
    int d = sim->dim, ns = oracle_n_scalars(d, sim->material);
    uint32_t W, bits;
    if (oracle_layout(s, 0, &W, &bits)) return -1;
    double inv_dx = 1.0 / sim->dx;
    int span = (d == 3) ? 5 : 1;
    hmap cells, nodes;
    if (hinit(&cells, n_sample * 125, 0) || hinit(&nodes, n_sample * 27, 1)) return -2;
    float dec[64];
    double st[64];
    for (uint64_t q = 0; q < n_sample; ++q) {
        if (oracle_decode_state(s, d, sim->material, 1, words_in + sample[q] * W, dec)) return -1;
        int b[3] = {0, 0, 0};
        double f;
        for (int a = 0; a < d; ++a) base_fx_f64((double)dec[a], inv_dx, sim->grid_res[a], &b[a], &f);
        for (int i = -2; i <= 2; ++i)
            for (int j = -2; j <= 2; ++j)
                for (int k = 0; k < span; ++k)
                    hget(&cells, hkey(b[0] + i, b[1] + j, d == 3 ? b[2] + k - 2 : 0), 1);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                for (int k = 0; k < (d == 3 ? 3 : 1); ++k)
                    hget(&nodes, hkey(b[0] + i, b[1] + j, d == 3 ? b[2] + k : 0), 1);
    }
    /* scatter every particle whose base is an interesting cell; the filter
     * decodes only the x fields (same decode as oracle_decode_state) */
    uint32_t offsets[ORACLE_MAX_FIELDS], xf[3] = {0, 0, 0};
    oracle_layout(s, offsets, 0, 0);
    for (uint32_t f = 0; f < s->n_fields; ++f)
        if (s->scalar[f] < (uint32_t)d) xf[s->scalar[f]] = f;
    for (uint64_t p = 0; p < n; ++p) {
        const uint32_t* rec = words_in + p * W;
        int b[3] = {0, 0, 0};
        double f;
        for (int a = 0; a < d; ++a) {
            uint32_t fi = xf[a];
            float xa;
            if (s->kind[fi] == ORACLE_RAW_F32) {
                uint32_t raw = oracle_get_bits(rec, offsets[fi], 32);
                memcpy(&xa, &raw, 4);
            } else {
                uint32_t wdt = s->frac_bits[fi] + 1;
                uint32_t raw = oracle_get_bits(rec, offsets[fi], wdt);
                int32_t u = (wdt < 32 && (raw >> (wdt - 1)) & 1u) ? (int32_t)(raw | ~((1u << wdt) - 1u))
                                                                  : (int32_t)raw;
                xa = oracle_decode_value(u, s->frac_bits[fi], s->range[fi], s->offset[fi]);
            }
            base_fx_f64((double)xa, inv_dx, sim->grid_res[a], &b[a], &f);
        }
        if (!hget(&cells, hkey(b[0], b[1], d == 3 ? b[2] : 0), 0)) continue;
        if (oracle_decode_state(s, d, sim->material, 1, rec, dec)) return -1;
        for (int a = 0; a < ns; ++a) st[a] = (double)dec[a];
        /* P2G into a private 3^d box, then add the box into the node map */
        int32_t origin[3] = {b[0], b[1], d == 3 ? b[2] : 0};
        int32_t gsize[3] = {3, 3, d == 3 ? 3 : 1};
        double box[27 * 4];
        memset(box, 0, sizeof(box));
        p2g_one_f64(sim, st, origin, gsize, box);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                for (int k = 0; k < gsize[2]; ++k) {
                    double* nd = hget(&nodes, hkey(b[0] + i, b[1] + j, origin[2] + k), 0);
                    if (!nd) continue;
                    const double* src = box + 4 * ((i * 3 + j) * gsize[2] + k);
                    for (int c = 0; c < 4; ++c) nd[c] += src[c];
                }
    }
    for (uint64_t sl = 0; sl < nodes.cap; ++sl) {
        if (nodes.keys[sl] == ~0ull) continue;
        uint64_t key = nodes.keys[sl];
        int ijk[3] = {(int)((key >> 42) & 0x1fffff) - 1024, (int)((key >> 21) & 0x1fffff) - 1024,
                      (int)(key & 0x1fffff) - 1024};
        update_node_f64(sim, ijk, nodes.vals + 4 * sl);
    }
    /* G2P + encode of the samples */
    for (uint64_t q = 0; q < n_sample; ++q) {
        const uint32_t* rec = words_in + sample[q] * W;
        oracle_decode_state(s, d, sim->material, 1, rec, dec);
        for (int a = 0; a < ns; ++a) st[a] = (double)dec[a];
        int b[3] = {0, 0, 0};
        double f;
        for (int a = 0; a < d; ++a) base_fx_f64(st[a], inv_dx, sim->grid_res[a], &b[a], &f);
        int32_t origin[3] = {b[0], b[1], d == 3 ? b[2] : 0};
        int32_t gsize[3] = {3, 3, d == 3 ? 3 : 1};
        double box[27 * 4];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                for (int k = 0; k < gsize[2]; ++k) {
                    double* nd = hget(&nodes, hkey(b[0] + i, b[1] + j, origin[2] + k), 0);
                    memcpy(box + 4 * ((i * 3 + j) * gsize[2] + k), nd, 4 * sizeof(double));
                }
        double out[64];
        g2p_one_f64(sim, st, origin, gsize, box, out);
        if (pre_encode) memcpy(pre_encode + q * ns, out, sizeof(double) * ns);
        float o32[64];
        for (int a = 0; a < ns; ++a) o32[a] = (float)out[a];
        uint32_t key = oracle_particle_key(s, d, rec);
        if (words_out) oracle_encode_state(s, d, sim->material, 1, o32, step, &key, words_out + q * W, 0);
    }
    hfree(&cells);
    hfree(&nodes);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* The same step as oracle_step_f64 with its particle and node loops spread over
 * OpenMP threads (the oracle on all host cores).  Nothing of the
 * arithmetic changes; only the order of the P2G sums: particles are bucketed by the
 * 4-cell x slab of their base cell, even slabs are scattered in parallel (their
 * stencils, 6 node planes wide, never overlap), then odd slabs; inside a slab in
 * particle order.  The order does not depend on the thread count, so the result is
 * deterministic.  Counters are summed over per-thread copies (integers).            */
#ifdef _OPENMP
#include <omp.h>
#endif

int oracle_step_omp_f64(const oracle_sim* sim, const oracle_scheme* s, uint64_t n, const uint32_t* words_in,
                        uint64_t step, double* pre_encode, uint32_t* words_out, uint64_t* counters,
                        int n_threads) {
    int d = sim->dim, ns = oracle_n_scalars(d, sim->material);
    uint32_t W, bits;
    if (oracle_layout(s, 0, &W, &bits)) return -1;
#ifdef _OPENMP
    if (n_threads <= 0) n_threads = omp_get_max_threads();
#else
    n_threads = 1;
#endif
    uint64_t nn = n ? n : 1;
    float* dec = (float*)malloc(sizeof(float) * ns * nn);
    double* st = (double*)malloc(sizeof(double) * ns * nn);
    double* out = (double*)malloc(sizeof(double) * ns * nn);
    uint32_t* keys = (uint32_t*)malloc(sizeof(uint32_t) * nn);
    int32_t* bx = (int32_t*)malloc(sizeof(int32_t) * nn);
    if (!dec || !st || !out || !keys || !bx) return -2;
    int err = 0;
    double inv_dx = 1.0 / sim->dx;
#pragma omp parallel num_threads(n_threads) reduction(| : err)
    {
#ifdef _OPENMP
        int t = omp_get_thread_num(), nt = omp_get_num_threads();
#else
        int t = 0, nt = 1;
#endif
        uint64_t lo = n * (uint64_t)t / (uint64_t)nt, hi = n * (uint64_t)(t + 1) / (uint64_t)nt;
        if (hi > lo) err |= oracle_decode_state(s, d, sim->material, hi - lo, words_in + lo * W, dec + lo * ns) != 0;
        for (uint64_t p = lo; p < hi; ++p) {
            for (int a = 0; a < ns; ++a) st[p * ns + a] = (double)dec[p * ns + a];
            keys[p] = oracle_particle_key(s, d, words_in + p * W);
            int b;
            double f;
            base_fx_f64(st[p * ns], inv_dx, sim->grid_res[0], &b, &f);
            bx[p] = b;
        }
    }
    if (err) return -1;
    int32_t origin[3], gsize[3];
    stencil_box_f64(sim, n, st, origin, gsize);
    long cells = (long)gsize[0] * gsize[1] * gsize[2];
    double* grid = (double*)calloc((size_t)cells * 4, sizeof(double));
    if (!grid) return -2;
    /* bucket particles by 4-cell x slab (counting sort, particle order kept) */
    int nslab = (gsize[0] + 3) / 4 + 1;
    uint64_t* start = (uint64_t*)calloc((size_t)nslab + 1, sizeof(uint64_t));
    uint64_t* order = (uint64_t*)malloc(sizeof(uint64_t) * nn);
    if (!start || !order) return -2;
    for (uint64_t p = 0; p < n; ++p) start[(bx[p] - origin[0]) / 4 + 1]++;
    for (int q = 0; q < nslab; ++q) start[q + 1] += start[q];
    {
        uint64_t* cur = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)nslab);
        memcpy(cur, start, sizeof(uint64_t) * (size_t)nslab);
        for (uint64_t p = 0; p < n; ++p) order[cur[(bx[p] - origin[0]) / 4]++] = p;
        free(cur);
    }
    uint64_t oob = 0;
    for (int parity = 0; parity < 2; ++parity) {
#pragma omp parallel for num_threads(n_threads) schedule(dynamic, 1) reduction(+ : oob)
        for (int q = parity; q < nslab; q += 2)
            for (uint64_t k = start[q]; k < start[q + 1]; ++k)
                oob += (uint64_t)p2g_one_f64(sim, st + order[k] * ns, origin, gsize, grid);
    }
#pragma omp parallel for num_threads(n_threads) schedule(static)
    for (long c = 0; c < cells; ++c) {
        long li = c / ((long)gsize[1] * gsize[2]), lj = (c / gsize[2]) % gsize[1], lk = c % gsize[2];
        int ijk[3] = {origin[0] + (int)li, origin[1] + (int)lj, origin[2] + (int)lk};
        update_node_f64(sim, ijk, grid + 4 * c);
    }
#pragma omp parallel for num_threads(n_threads) schedule(static)
    for (int64_t p = 0; p < (int64_t)n; ++p) g2p_one_f64(sim, st + p * ns, origin, gsize, grid, out + p * ns);
    if (counters) counters[193] += oob;
    if (pre_encode) memcpy(pre_encode, out, sizeof(double) * ns * n);
    uint64_t* tc = (uint64_t*)calloc((size_t)n_threads * ORACLE_NCOUNTERS, sizeof(uint64_t));
    if (!tc) return -2;
#pragma omp parallel num_threads(n_threads) reduction(| : err)
    {
#ifdef _OPENMP
        int t = omp_get_thread_num(), nt = omp_get_num_threads();
#else
        int t = 0, nt = 1;
#endif
        uint64_t lo = n * (uint64_t)t / (uint64_t)nt, hi = n * (uint64_t)(t + 1) / (uint64_t)nt;
        for (uint64_t i = lo * ns; i < hi * ns; ++i) dec[i] = (float)out[i];
        if (hi > lo)
            err |= oracle_encode_state(s, d, sim->material, hi - lo, dec + lo * ns, step, keys + lo,
                                       words_out + lo * W, counters ? tc + (size_t)t * ORACLE_NCOUNTERS : 0) != 0;
    }
    if (counters)
        for (int t = 0; t < n_threads; ++t)
            for (int c = 0; c < ORACLE_NCOUNTERS; ++c) counters[c] += tc[(size_t)t * ORACLE_NCOUNTERS + c];
    free(tc);
    free(grid);
    free(start);
    free(order);
    free(dec);
    free(st);
    free(out);
    free(keys);
    free(bx);
    return err ? -1 : 0;
}

int oracle_run_omp_f64(const oracle_sim* sim, const oracle_scheme* s, uint64_t n, uint32_t* words,
                       uint64_t first_step, uint32_t n_steps, uint64_t* counters, int n_threads) {
    uint32_t W, bits;
    if (oracle_layout(s, 0, &W, &bits)) return -1;
    uint32_t* tmp = (uint32_t*)malloc(sizeof(uint32_t) * W * (n ? n : 1));
    if (!tmp) return -2;
    for (uint32_t t = 0; t < n_steps; ++t) {
        int rc = oracle_step_omp_f64(sim, s, n, words, first_step + t, 0, tmp, counters, n_threads);
        if (rc) { free(tmp); return rc; }
        memcpy(words, tmp, sizeof(uint32_t) * W * n);
    }
    free(tmp);
    return 0;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
