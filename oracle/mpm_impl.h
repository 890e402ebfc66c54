/*
 * mpm_impl.h -- oracle MLS-MPM step, instantiated twice by mpm.c:
 *   REAL=double, SUF(name)=name##_f64   (the "truth")
 *   REAL=float,  SUF(name)=name##_f32   (the tight fp32 comparator)
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * The paper names MLS-MPM (Hu et al. 2018) and J-tracking fluid
 * (Tampubolon 2017) but gives no internals; per S:260 the internals
 * follow the cited method's public reference programs (reading SURVEY §8(c) C-mpm):
 *   P2G:  base = floor(x/dx - 0.5), fx = x/dx - base,
 *         w = (0.5(1.5-fx)^2, 0.75-(fx-1)^2, 0.5(fx-0.5)^2),
 *         stress = -dt * V_p * 4/dx^2 * P(F)F^T, affine = stress + m_p C,
 *         m_i += w m_p,  p_i += w (m_p v_p + affine (x_i - x_p)).
 *   Grid: v = p/m + dt g; separating walls within `bound` nodes (reading Q13).
 *   G2P:  v' = sum w v_i,  C' = 4/dx sum w v_i (x) (i - fx),  x' = x + dt v',
 *         F' = (I + dt C') F  (elastic, reading Q11)  |  J' = J (1 + dt tr C')  (fluid).
 * Elastic P(F)F^T = 2mu (F - R) F^T + lambda (J-1) J I (fixed corotated);
 * fluid P(F)F^T = E (J-1) I (reading Q15).
 * Out-of-domain particles (base outside [0, n-3]) are counted and clamped (Q14).
 * No blocking, fusion or reordering: every loop is the textbook one.
 */

static void SUF(mat_mul)(int d, const REAL* A, const REAL* B, REAL* out) {
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) {
            REAL acc = 0;
            for (int k = 0; k < d; ++k) acc += A[i * d + k] * B[k * d + j];
            out[i * d + j] = acc;
        }
}

static REAL SUF(det)(int d, const REAL* F) {
    if (d == 2) return F[0] * F[3] - F[1] * F[2];
    return F[0] * (F[4] * F[8] - F[5] * F[7]) - F[1] * (F[3] * F[8] - F[5] * F[6]) +
           F[2] * (F[3] * F[7] - F[4] * F[6]);
}

/* base/fx of one axis, with the out-of-domain clamp of reading Q14 */
static int SUF(base_fx)(REAL x, REAL inv_dx, int n_axis, int* base, REAL* fx) {
    REAL X = x * inv_dx;
    long b = (long)floor((double)(X - (REAL)0.5));
    int oob = 0;
    if (b < 0) { b = 0; oob = 1; }
    if (b > n_axis - 3) { b = n_axis - 3; oob = 1; }
    REAL f = X - (REAL)b;
    if (oob) {
        if (f < (REAL)0.5) f = (REAL)0.5;
        if (f > (REAL)1.5) f = (REAL)1.5;
    }
    *base = (int)b;
    *fx = f;
    return oob;
}

/* quadratic B-spline weights at offsets 0,1,2 (Hu et al. 2018) */
static void SUF(weights)(REAL fx, REAL* w) {
    w[0] = (REAL)0.5 * ((REAL)1.5 - fx) * ((REAL)1.5 - fx);
    w[1] = (REAL)0.75 - (fx - (REAL)1.0) * (fx - (REAL)1.0);
    w[2] = (REAL)0.5 * (fx - (REAL)0.5) * (fx - (REAL)0.5);
}

static long SUF(node_index)(const int32_t* origin, const int32_t* gsize, int i, int j, int k) {
    int li = i - origin[0], lj = j - origin[1], lk = k - origin[2];
    if (li < 0 || lj < 0 || lk < 0 || li >= gsize[0] || lj >= gsize[1] || lk >= gsize[2])
        return -1;
    return ((long)li * gsize[1] + lj) * gsize[2] + lk;
}

/* stress contribution of one particle: out = -dt * V_p * 4 * inv_dx^2 * P(F)F^T */
static void SUF(stress)(const oracle_sim* sim, const REAL* st, REAL* out) {
    int d = sim->dim;
    REAL dt = (REAL)sim->dt, inv_dx = (REAL)1 / (REAL)sim->dx;
    REAL p_vol = (REAL)sim->p_vol, E = (REAL)sim->E, nu = (REAL)sim->nu;
    REAL PFt[9] = {0};
    if (sim->material == ORACLE_FLUID) {
        REAL J = st[2 * d];
        for (int a = 0; a < d; ++a) PFt[a * d + a] = E * (J - (REAL)1);
    } else {
        const REAL* F = st + 2 * d;
        REAL mu = E / ((REAL)2 * ((REAL)1 + nu));
        REAL la = E * nu / (((REAL)1 + nu) * ((REAL)1 - (REAL)2 * nu));
        REAL J = SUF(det)(d, F);
        double Fd[9] = {0}, Rd[9] = {0};
        for (int a = 0; a < d * d; ++a) Fd[a] = (double)F[a];
        oracle_polar_f64(d, Fd, Rd);
        REAL FmR[9] = {0}, Ft[9] = {0};
        for (int a = 0; a < d; ++a)
            for (int b = 0; b < d; ++b) {
                FmR[a * d + b] = F[a * d + b] - (REAL)Rd[a * d + b];
                Ft[a * d + b] = F[b * d + a];
            }
        SUF(mat_mul)(d, FmR, Ft, PFt);
        for (int a = 0; a < d * d; ++a) PFt[a] = (REAL)2 * mu * PFt[a];
        for (int a = 0; a < d; ++a) PFt[a * d + a] += la * (J - (REAL)1) * J;
    }
    REAL scale = -dt * p_vol * (REAL)4 * inv_dx * inv_dx;
    for (int a = 0; a < d * d; ++a) out[a] = scale * PFt[a];
}

/* P2G of particle p into the box grid (m, p_x, p_y, p_z per node) */
static int SUF(p2g_one)(const oracle_sim* sim, const REAL* st, const int32_t* origin,
                        const int32_t* gsize, REAL* grid) {
    int d = sim->dim;
    REAL dx = (REAL)sim->dx, inv_dx = (REAL)1 / dx;
    REAL p_mass = (REAL)(sim->p_rho * sim->p_vol);
    int base[3] = {0, 0, 0};
    REAL fx[3] = {0, 0, 0}, w[3][3];
    int oob = 0;
    for (int a = 0; a < d; ++a) {
        oob |= SUF(base_fx)(st[a], inv_dx, sim->grid_res[a], &base[a], &fx[a]);
        SUF(weights)(fx[a], w[a]);
    }
    REAL affine[9];
    SUF(stress)(sim, st, affine);
    const REAL* C = st + (sim->material == ORACLE_FLUID ? 2 * d + 1 : 2 * d + d * d);
    for (int a = 0; a < d * d; ++a) affine[a] += p_mass * C[a];
    const REAL* v = st + d;
    int nz = (d == 3) ? 3 : 1;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            for (int k = 0; k < nz; ++k) {
                int o[3] = {i, j, k};
                REAL weight = 1, dpos[3];
                for (int a = 0; a < d; ++a) {
                    weight *= w[a][o[a]];
                    dpos[a] = ((REAL)o[a] - fx[a]) * dx;
                }
                long idx = SUF(node_index)(origin, gsize, base[0] + i, base[1] + j,
                                           d == 3 ? base[2] + k : 0);
                if (idx < 0) continue;
                REAL* node = grid + 4 * idx;
                node[0] += weight * p_mass;
                for (int a = 0; a < d; ++a) {
                    REAL Ad = 0;
                    for (int b = 0; b < d; ++b) Ad += affine[a * d + b] * dpos[b];
                    node[1 + a] += weight * (p_mass * v[a] + Ad);
                }
            }
    return oob;
}

void SUF(oracle_p2g)(const oracle_sim* sim, uint64_t n, const REAL* state, const int32_t* origin,
                     const int32_t* gsize, REAL* grid, uint64_t* oob) {
    int ns = oracle_n_scalars(sim->dim, sim->material);
    for (uint64_t p = 0; p < n; ++p) {
        int o = SUF(p2g_one)(sim, state + p * ns, origin, gsize, grid);
        if (o && oob) (*oob)++;
    }
}

/* grid update of one node: v = p/m + dt g, then separating walls (reading Q13) */
static void SUF(update_node)(const oracle_sim* sim, const int* ijk, REAL* node) {
    int d = sim->dim;
    REAL m = node[0];
    if (!(m > 0)) {
        node[1] = node[2] = node[3] = 0;
        return;
    }
    for (int a = 0; a < d; ++a) {
        REAL va = node[1 + a] / m;
        va += (REAL)sim->dt * (REAL)sim->gravity[a];
        if (ijk[a] < sim->bound && va < 0) va = 0;
        if (ijk[a] > sim->grid_res[a] - sim->bound && va > 0) va = 0;
        node[1 + a] = va;
    }
}

void SUF(oracle_grid_update)(const oracle_sim* sim, const int32_t* origin, const int32_t* gsize,
                             REAL* grid) {
    for (int li = 0; li < gsize[0]; ++li)
        for (int lj = 0; lj < gsize[1]; ++lj)
            for (int lk = 0; lk < gsize[2]; ++lk) {
                int ijk[3] = {origin[0] + li, origin[1] + lj, origin[2] + lk};
                long idx = ((long)li * gsize[1] + lj) * gsize[2] + lk;
                SUF(update_node)(sim, ijk, grid + 4 * idx);
            }
}

static void SUF(g2p_one)(const oracle_sim* sim, const REAL* st, const int32_t* origin,
                         const int32_t* gsize, const REAL* grid, REAL* out) {
    int d = sim->dim;
    int ns = oracle_n_scalars(d, sim->material);
    REAL dt = (REAL)sim->dt, inv_dx = (REAL)1 / (REAL)sim->dx;
    int base[3] = {0, 0, 0};
    REAL fx[3] = {0, 0, 0}, w[3][3];
    for (int a = 0; a < d; ++a) {
        SUF(base_fx)(st[a], inv_dx, sim->grid_res[a], &base[a], &fx[a]);
        SUF(weights)(fx[a], w[a]);
    }
    REAL new_v[3] = {0, 0, 0}, new_C[9] = {0};
    int nz = (d == 3) ? 3 : 1;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            for (int k = 0; k < nz; ++k) {
                int o[3] = {i, j, k};
                REAL weight = 1, dpos[3];
                for (int a = 0; a < d; ++a) {
                    weight *= w[a][o[a]];
                    dpos[a] = (REAL)o[a] - fx[a];
                }
                long idx = SUF(node_index)(origin, gsize, base[0] + i, base[1] + j,
                                           d == 3 ? base[2] + k : 0);
                const REAL* node = grid + 4 * idx; /* caller's box covers every stencil */
                for (int a = 0; a < d; ++a) {
                    new_v[a] += weight * node[1 + a];
                    for (int b = 0; b < d; ++b)
                        new_C[a * d + b] += (REAL)4 * inv_dx * weight * node[1 + a] * dpos[b];
                }
            }
    for (int a = 0; a < ns; ++a) out[a] = st[a];
    for (int a = 0; a < d; ++a) {
        out[a] = st[a] + dt * new_v[a];
        out[d + a] = new_v[a];
    }
    if (sim->material == ORACLE_FLUID) {
        REAL tr = 0;
        for (int a = 0; a < d; ++a) tr += new_C[a * d + a];
        out[2 * d] = st[2 * d] * ((REAL)1 + dt * tr);
        for (int a = 0; a < d * d; ++a) out[2 * d + 1 + a] = new_C[a];
    } else {
        REAL G[9] = {0};
        for (int a = 0; a < d; ++a)
            for (int b = 0; b < d; ++b) G[a * d + b] = (a == b ? (REAL)1 : (REAL)0) + dt * new_C[a * d + b];
        SUF(mat_mul)(d, G, st + 2 * d, out + 2 * d);
        for (int a = 0; a < d * d; ++a) out[2 * d + d * d + a] = new_C[a];
    }
}

void SUF(oracle_g2p)(const oracle_sim* sim, uint64_t n, const REAL* state_in,
                     const int32_t* origin, const int32_t* gsize, const REAL* grid,
                     REAL* state_out) {
    int ns = oracle_n_scalars(sim->dim, sim->material);
    for (uint64_t p = 0; p < n; ++p)
        SUF(g2p_one)(sim, state_in + p * ns, origin, gsize, grid, state_out + p * ns);
}

/* bounding box of all stencils (base .. base+2 per axis) */
static void SUF(stencil_box)(const oracle_sim* sim, uint64_t n, const REAL* state,
                             int32_t* origin, int32_t* gsize) {
    int d = sim->dim, ns = oracle_n_scalars(d, sim->material);
    REAL inv_dx = (REAL)1 / (REAL)sim->dx;
    int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int a = 0; a < 3; ++a) { lo[a] = 1 << 30; hi[a] = -(1 << 30); }
    for (uint64_t p = 0; p < n; ++p)
        for (int a = 0; a < d; ++a) {
            int b;
            REAL f;
            SUF(base_fx)(state[p * ns + a], inv_dx, sim->grid_res[a], &b, &f);
            if (b < lo[a]) lo[a] = b;
            if (b + 2 > hi[a]) hi[a] = b + 2;
        }
    for (int a = 0; a < 3; ++a) {
        if (a >= d || n == 0) { origin[a] = 0; gsize[a] = 1; continue; }
        origin[a] = lo[a];
        gsize[a] = hi[a] - lo[a] + 1;
    }
}

/* One quantized step (Eq. 1): decode -> F -> encode with dither at step t. */
int SUF(oracle_step)(const oracle_sim* sim, const oracle_scheme* s, uint64_t n,
                     const uint32_t* words_in, uint64_t step, REAL* pre_encode,
                     uint32_t* words_out, uint64_t* counters) {
    int d = sim->dim, ns = oracle_n_scalars(d, sim->material);
    uint32_t W, bits;
    if (oracle_layout(s, 0, &W, &bits)) return -1;
    float* dec = (float*)malloc(sizeof(float) * ns * (n ? n : 1));
    REAL* st = (REAL*)malloc(sizeof(REAL) * ns * (n ? n : 1));
    REAL* out = (REAL*)malloc(sizeof(REAL) * ns * (n ? n : 1));
    uint32_t* keys = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    if (!dec || !st || !out || !keys) return -2;
    if (oracle_decode_state(s, d, sim->material, n, words_in, dec)) return -1;
    for (uint64_t i = 0; i < n * ns; ++i) st[i] = (REAL)dec[i];
    for (uint64_t p = 0; p < n; ++p) keys[p] = oracle_particle_key(s, d, words_in + p * W);
    int32_t origin[3], gsize[3];
    SUF(stencil_box)(sim, n, st, origin, gsize);
    long cells = (long)gsize[0] * gsize[1] * gsize[2];
    REAL* grid = (REAL*)calloc((size_t)cells * 4, sizeof(REAL));
    if (!grid) return -2;
    uint64_t oob = 0;
    SUF(oracle_p2g)(sim, n, st, origin, gsize, grid, &oob);
    SUF(oracle_grid_update)(sim, origin, gsize, grid);
    SUF(oracle_g2p)(sim, n, st, origin, gsize, grid, out);
    if (counters) counters[193] += oob;
    if (pre_encode) memcpy(pre_encode, out, sizeof(REAL) * ns * n);
    /* the encode takes the fp32 value (both sides decide codes in fp32) */
    for (uint64_t i = 0; i < n * ns; ++i) dec[i] = (float)out[i];
    int rc = oracle_encode_state(s, d, sim->material, n, dec, step, keys, words_out, counters);
    free(grid);
    free(dec);
    free(st);
    free(out);
    free(keys);
    return rc;
}
