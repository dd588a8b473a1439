/* oracle_body.h -- the per-REAL body of the CPU oracle; included twice by
 * wave_oracle.c (REAL = float, then REAL = double).  TEST INFRASTRUCTURE ONLY.
 *
 * Every function follows the cited passage literally: one plain triple loop
 * per time step over the whole (local) extended domain, the PML/inner choice
 * made per point ("a single kernel ... contains
 * conditionals"; SPEC.md L176-179 reference_propagate), no blocking, no
 * fusion, no reordering of the arithmetic.
 */

/* One sweep (one application of Eq. 2's left-hand side at every point):
 *   PAPER.md L237-240 (Eq. 2), L243-249 (Eq. 3), L259-262 (Alg. 1 lines 2-3);
 *   SPEC.md L140-157 (step_inner / step_pml), L376 (accumulation order).
 * u_pad   : u^n   padded [nz+8][ny+8][nx+8], zero pad = Dirichlet fringe
 *           (SPEC.md L81); in z the pad holds the neighbour slab's planes
 *           (ghosts) when the grid is a z-slab of a larger one.
 * up_pad  : u^{n-1} on entry, u^{n+1} on exit (same layout).
 * vdt2    : dense [nz][ny][nx] fp (V*dt)^2 values.
 */
static REAL SFX(eta_star)(const oracle_geom *g, const struct SFX(consts) *K, const REAL *eta_arr,
                          int64_t i, int64_t j, int64_t kg);

static void SFX(sweep)(const oracle_geom *g, const struct SFX(consts) *K,
                       const REAL *u, REAL *up, const REAL *vdt2, const REAL *eta_arr)
{
    const int64_t nx = g->nx, ny = g->ny, nz = g->nz;
    const int64_t sy = nx + 2 * R, sz = (ny + 2 * R) * sy;
    int64_t k;
#pragma omp parallel for schedule(static)
    for (k = 0; k < nz; ++k) {
        const int64_t kg = k + g->z_offset;          /* global z of this plane */
        for (int64_t j = 0; j < ny; ++j) {
            for (int64_t i = 0; i < nx; ++i) {
                const int64_t p = pidx(g, i, j, k);
                const int64_t q = (k * ny + j) * nx + i;
                const REAL uc = u[p];

                /* Eq. 3: c_xyz*u + sum_m c_am*(u(+m) + u(-m)),
                 * pair sum first, axes x, y, z, m = 1..4. */
                REAL L = K->c0 * uc;
                for (int m = 1; m <= R; ++m) L = L + K->cx[m] * (u[p + m] + u[p - m]);
                for (int m = 1; m <= R; ++m) L = L + K->cy[m] * (u[p + m * sy] + u[p - m * sy]);
                for (int m = 1; m <= R; ++m) L = L + K->cz[m] * (u[p + m * sz] + u[p - m * sz]);

                const int64_t d = dist3(g, i, j, kg);
                REAL un;
                if (d == 0) {
                    /* inner region: u_next = 2u - u_prev + dt^2 V^2 Lap(u) */
                    un = ((REAL)2 * uc - up[p]) + vdt2[q] * L;
                } else {
                    /* PML region, SPEC.md L152 (formula), L197 + DESIGN.md R2/R3 (eta profile):
                     * u_next = [2u - (1 - eta dt) u_prev + dt^2 V^2 (Lap(u) + sum_a d_a eta d_a u)]
                     *          / (1 + eta dt),  d_a f = (f(+1) - f(-1)) / (2 h_a).
                     * eta is read on the 7-point star. */
                    REAL gsum = 0;
                    gsum = gsum + ((SFX(eta_star)(g, K, eta_arr, i + 1, j, kg) - SFX(eta_star)(g, K, eta_arr, i - 1, j, kg)) * K->i2h[0])
                                * ((u[p + 1] - u[p - 1]) * K->i2h[0]);
                    gsum = gsum + ((SFX(eta_star)(g, K, eta_arr, i, j + 1, kg) - SFX(eta_star)(g, K, eta_arr, i, j - 1, kg)) * K->i2h[1])
                                * ((u[p + sy] - u[p - sy]) * K->i2h[1]);
                    gsum = gsum + ((SFX(eta_star)(g, K, eta_arr, i, j, kg + 1) - SFX(eta_star)(g, K, eta_arr, i, j, kg - 1)) * K->i2h[2])
                                * ((u[p + sz] - u[p - sz]) * K->i2h[2]);
                    REAL A = K->A[d], B = K->B[d];
                    if (eta_arr) {
                        /* stored eta (R16): A = 1 - eta dt, B = 1 + eta dt from
                         * this point's stored value, computed in fp64, rounded once */
                        const double e = (double)eta_arr[q], dt = (double)g->dt;
                        A = (REAL)(K->round32 ? fp32_round(1.0 - e * dt) : 1.0 - e * dt);
                        B = (REAL)(K->round32 ? fp32_round(1.0 + e * dt) : 1.0 + e * dt);
                    }
                    un = (((REAL)2 * uc - A * up[p]) + vdt2[q] * (L + gsum)) / B;
                }
                up[p] = un;
            }
        }
    }
}

/* eta on the 7-point star: the stored field (user-supplied eta, SURVEY.md
 * §8(f) rank 3; dense [nz][ny][nx] of this single-slab grid) or the profile
 * eta_{d(q)}; 0 outside the domain either way. */
static REAL SFX(eta_star)(const oracle_geom *g, const struct SFX(consts) *K, const REAL *eta_arr,
                          int64_t i, int64_t j, int64_t kg)
{
    if (!eta_arr) return SFX(eta_at)(g, K, i, j, kg);
    if (!inside(g, i, j, kg)) return 0;
    return eta_arr[((kg - g->z_offset) * g->ny + j) * g->nx + i];
}

/* Source injection, PAPER.md L263 (Alg. 1 "u^n = u^n + f^n") with the Eq. 2
 * right-hand-side scaling dt^2 V^2, applied
 * after the sweep.  inc = fp(vdt2[src] * w[n]). */
static void SFX(inject)(const oracle_geom *g, REAL *up, const REAL *vdt2,
                        int64_t si, int64_t sj, int64_t sk, float wn, int round32)
{
    const int64_t k = sk - g->z_offset;
    if (k < 0 || k >= g->nz) return;                 /* source owned by another slab */
    const REAL vs = vdt2[(k * g->ny + sj) * g->nx + si];
    const double inc64 = (double)vs * (double)wn;
    const REAL inc = (REAL)(round32 ? fp32_round(inc64) : inc64);
    const int64_t p = pidx(g, si, sj, k);
    up[p] = up[p] + inc;
}

static int SFX(all_finite)(const oracle_geom *g, const REAL *u)
{
    int ok = 1;
    for (int64_t k = 0; k < g->nz; ++k)
        for (int64_t j = 0; j < g->ny; ++j)
            for (int64_t i = 0; i < g->nx; ++i)
                if (!isfinite((double)u[pidx(g, i, j, k)])) ok = 0;
    return ok;
}

/* ---- exported entry points (C ABI) -------------------------------------- */

/* One time step of Algorithm 1 on a (possibly slab) padded grid:
 * sweep, then inject w[n] if the source lies in this slab. */
EXPORT int SFX(oracle_step)(const oracle_geom *g, int round32, const REAL *u_pad,
                            REAL *up_pad, const REAL *vdt2, int64_t si, int64_t sj,
                            int64_t sk, float wn)
{
    struct SFX(consts) K;
    if (SFX(make_consts)(g, round32, &K)) return ORACLE_ERR_CONFIG;
    SFX(sweep)(g, &K, u_pad, up_pad, vdt2, NULL);
    SFX(inject)(g, up_pad, vdt2, si, sj, sk, wn, round32);
    SFX(free_consts)(&K);
    return ORACLE_OK;
}

/* Algorithm 1 for T steps on a single (non-slab) grid: PAPER.md L255-267,
 * SPEC.md L176-184 (reference_propagate).  u, up: dense [nz][ny][nx], in:
 * u^0, u^{-1} ("u^0 := 0" is the all-zero input); out: u^T,
 * u^{T-1}.  Non-finite check every `check_every` steps (0 = only at the end):
 * returns ORACLE_ERR_UNSTABLE and the step count in *fail_step. */
/* eta_in: NULL (the eta_max (d/w)^2 profile) or a user-supplied eta field,
 * dense [nz][ny][nx] fp32, >= 0 (stored-eta variant, R16). */
EXPORT int SFX(oracle_propagate_eta)(const oracle_geom *g, int round32, const float *V,
                                     const float *eta_in, const float *wavelet, int64_t T, int64_t si,
                                     int64_t sj, int64_t sk, REAL *u, REAL *up, int64_t check_every,
                                     int64_t *fail_step)
{
    struct SFX(consts) K;
    if (g->z_offset != 0 || g->nz_global != g->nz) return ORACLE_ERR_CONFIG;
    if (SFX(make_consts)(g, round32, &K)) return ORACLE_ERR_CONFIG;
    const int64_t n = g->nx * g->ny * g->nz;
    REAL *eta_arr = NULL;
    if (eta_in) {
        eta_arr = (REAL *)malloc(sizeof(REAL) * n);
        if (!eta_arr) { SFX(free_consts)(&K); return ORACLE_ERR_ALLOC; }
        for (int64_t q = 0; q < n; ++q) eta_arr[q] = (REAL)eta_in[q];
    }
    const int64_t np = (g->nx + 2 * R) * (g->ny + 2 * R) * (g->nz + 2 * R);
    REAL *vdt2 = (REAL *)malloc(sizeof(REAL) * n);
    REAL *a = (REAL *)calloc(np, sizeof(REAL));
    REAL *b = (REAL *)calloc(np, sizeof(REAL));
    if (!vdt2 || !a || !b) {
        free(vdt2); free(a); free(b); free(eta_arr); SFX(free_consts)(&K);
        return ORACLE_ERR_ALLOC;
    }
    SFX(vdt2_fill)(V, n, g->dt, round32, vdt2);
    for (int64_t k = 0; k < g->nz; ++k)
        for (int64_t j = 0; j < g->ny; ++j)
            for (int64_t i = 0; i < g->nx; ++i) {
                a[pidx(g, i, j, k)] = u[(k * g->ny + j) * g->nx + i];
                b[pidx(g, i, j, k)] = up[(k * g->ny + j) * g->nx + i];
            }
    REAL *cur = a, *prev = b;
    int status = ORACLE_OK;
    if (fail_step) *fail_step = -1;
    for (int64_t s = 0; s < T; ++s) {
        SFX(sweep)(g, &K, cur, prev, vdt2, eta_arr);            /* prev <- u^{s+1} */
        SFX(inject)(g, prev, vdt2, si, sj, sk, wavelet[s], round32); /* + f^{s+1}   */
        REAL *t = cur; cur = prev; prev = t;                    /* role swap        */
        if ((check_every > 0 && (s + 1) % check_every == 0) || s + 1 == T) {
            if (!SFX(all_finite)(g, cur)) {
                status = ORACLE_ERR_UNSTABLE;
                if (fail_step) *fail_step = s + 1;
                break;
            }
        }
    }
    for (int64_t k = 0; k < g->nz; ++k)
        for (int64_t j = 0; j < g->ny; ++j)
            for (int64_t i = 0; i < g->nx; ++i) {
                u[(k * g->ny + j) * g->nx + i] = cur[pidx(g, i, j, k)];
                up[(k * g->ny + j) * g->nx + i] = prev[pidx(g, i, j, k)];
            }
    free(vdt2); free(a); free(b); free(eta_arr);
    SFX(free_consts)(&K);
    return status;
}

EXPORT int SFX(oracle_propagate)(const oracle_geom *g, int round32, const float *V,
                                 const float *wavelet, int64_t T, int64_t si, int64_t sj,
                                 int64_t sk, REAL *u, REAL *up, int64_t check_every,
                                 int64_t *fail_step)
{
    return SFX(oracle_propagate_eta)(g, round32, V, NULL, wavelet, T, si, sj, sk, u, up, check_every,
                                     fail_step);
}

/* The fp constants the oracle uses (for the pins in tests/): c[13] =
 * {c_xyz, c_x1..4, c_y1..4, c_z1..4}, eta/A/B[w+1], inv2h[3]. */
EXPORT int SFX(oracle_constants)(const oracle_geom *g, int round32, REAL *c13,
                                 REAL *eta, REAL *A, REAL *B, REAL *inv2h)
{
    struct SFX(consts) K;
    if (SFX(make_consts)(g, round32, &K)) return ORACLE_ERR_CONFIG;
    c13[0] = K.c0;
    for (int m = 1; m <= R; ++m) { c13[m] = K.cx[m]; c13[4 + m] = K.cy[m]; c13[8 + m] = K.cz[m]; }
    for (int d = 0; d <= g->w; ++d) { eta[d] = K.eta[d]; A[d] = K.A[d]; B[d] = K.B[d]; }
    for (int a = 0; a < 3; ++a) inv2h[a] = K.i2h[a];
    SFX(free_consts)(&K);
    return ORACLE_OK;
}

EXPORT void SFX(oracle_vdt2)(const float *V, int64_t n, float dt, int round32, REAL *out)
{
    SFX(vdt2_fill)(V, n, dt, round32, out);
}
