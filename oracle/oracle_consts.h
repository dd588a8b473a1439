/* oracle_consts.h -- per-REAL constant setup for the oracle (SURVEY.md §8(c)
 * step 2; R8 "compute every constant in fp64, round once").
 * Included twice by wave_oracle.c.  TEST INFRASTRUCTURE ONLY.
 *
 * round32 = 1: every constant is computed in fp64 and rounded once to fp32
 *              (the parity configuration, used by both REAL = float and the
 *              "fp64 arithmetic on fp32 constants" diagnostic);
 * round32 = 0: constants kept in fp64 (the fp64 reference).
 */

static int SFX(make_consts)(const oracle_geom *g, int round32, struct SFX(consts) *K)
{
    if (g->nx < 1 || g->ny < 1 || g->nz < 1 || g->w < 0) return 1;
    if (!(g->hx > 0 && g->hy > 0 && g->hz > 0)) return 1;
    double (*rnd)(double) = round32 ? fp32_round : NULL;
    K->round32 = round32;
#define RND(x) (rnd ? rnd(x) : (x))
    const double ih2[3] = { 1.0 / (g->hx * g->hx), 1.0 / (g->hy * g->hy), 1.0 / (g->hz * g->hz) };
    /* c_xyz = w0 (1/hx^2 + 1/hy^2 + 1/hz^2)  (SPEC.md L125 with per-axis h, R1) */
    K->c0 = (REAL)RND(W8[0] * (ih2[0] + ih2[1] + ih2[2]));
    K->cx[0] = K->cy[0] = K->cz[0] = 0;
    for (int m = 1; m <= R; ++m) {                    /* c_am = w_m / h_a^2 */
        K->cx[m] = (REAL)RND(W8[m] * ih2[0]);
        K->cy[m] = (REAL)RND(W8[m] * ih2[1]);
        K->cz[m] = (REAL)RND(W8[m] * ih2[2]);
    }
    K->i2h[0] = (REAL)RND(1.0 / (2.0 * g->hx));       /* 1/(2 h_a) */
    K->i2h[1] = (REAL)RND(1.0 / (2.0 * g->hy));
    K->i2h[2] = (REAL)RND(1.0 / (2.0 * g->hz));
    const int w = g->w;
    K->eta = (REAL *)malloc(sizeof(REAL) * (w + 1));
    K->A = (REAL *)malloc(sizeof(REAL) * (w + 1));
    K->B = (REAL *)malloc(sizeof(REAL) * (w + 1));
    const double dt = (double)g->dt;
    for (int d = 0; d <= w; ++d) {
        /* eta_d = eta_max (d/w)^2 (R2), A_d = 1 - eta_d dt, B_d = 1 + eta_d dt */
        const double r = w > 0 ? (double)d / (double)w : 0.0;
        const double eta = g->eta_max * r * r;
        K->eta[d] = (REAL)RND(eta);
        K->A[d] = (REAL)RND(1.0 - eta * dt);
        K->B[d] = (REAL)RND(1.0 + eta * dt);
    }
#undef RND
    return 0;
}

static void SFX(free_consts)(struct SFX(consts) *K)
{
    free(K->eta); free(K->A); free(K->B);
}

/* eta on the 7-point star: eta_{d(q)} inside the domain, 0 outside
 * (SPEC.md L32/L81 zero pad, R4). */
static inline REAL SFX(eta_at)(const oracle_geom *g, const struct SFX(consts) *K,
                               int64_t i, int64_t j, int64_t kg)
{
    if (!inside(g, i, j, kg)) return 0;
    return K->eta[dist3(g, i, j, kg)];
}

/* vdt2 = (V dt)^2 computed in fp64, rounded once when round32. */
static void SFX(vdt2_fill)(const float *V, int64_t n, float dt, int round32, REAL *out)
{
    for (int64_t i = 0; i < n; ++i) {
        const double a = (double)V[i] * (double)dt;
        out[i] = (REAL)(round32 ? fp32_round(a * a) : a * a);
    }
}
