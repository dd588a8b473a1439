/* wave_oracle.c -- CPU ORACLE for the 25-point acoustic wave step.
 *
 * TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product
 * (paper_2009_04619_b200/) never links, imports or calls it, and shares no
 * code, header, table or constant generator with it.
 *
 * What it computes (plain definition, evaluated literally):
 *   PAPER.md L232-240  Eq. 1-2: u^{n+1} - Q u^n + u^{n-1} = dt^2 V^2 f^n,
 *                      Q = 2 + dt^2 V^2 Lap
 *   PAPER.md L241-251  Eq. 3: 25-point star Laplacian, radius 4
 *   PAPER.md L255-267  Algorithm 1 (time loop, u^0 := 0, source after sweep)
 *   PAPER.md L269-275  inner region: 25-pt on u; PML region: 7-pt star on eta
 *   SPEC.md  L122-184  make_coeffs_order8, laplacian25, step_inner, step_pml,
 *                      inject_source, reference_propagate
 * with the readings of DESIGN.md §3 (R1..R12): eta = eta_max (d/w)^2 with d
 * the integer Chebyshev distance to the inner box, eta = 0 outside the
 * domain, constants computed in fp64 and rounded once to fp32 (round32=1).
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fPIC -shared (never -ffast-math:
 * the PML division must stay a true IEEE division, R9).
 *
 * Parity pins: see tests/test_oracle_*.py (closed forms, invariants, brute
 * force).  The PML formula itself is SPEC's stand-in (PAPER.md gives only
 * its footprint): "parity unpinned against the paper" for the PML update's
 * exact form -- it is pinned against closed forms of that stand-in
 * (linear-ramp probe, constant state, eta=0 reduction), see DESIGN.md §3.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define EXPORT __attribute__((visibility("default")))
#define R 4                       /* stencil radius */

enum { ORACLE_OK = 0, ORACLE_ERR_CONFIG = 1, ORACLE_ERR_UNSTABLE = 2, ORACLE_ERR_ALLOC = 5 };

typedef struct {
    int64_t nx, ny, nz;           /* local extents; nz = planes of this z-slab */
    int32_t w;                    /* PML width (cells) */
    double hx, hy, hz;            /* spacing (m) */
    float dt;                     /* time step (s), the fp32 value used */
    double eta_max;               /* 1/s */
    int64_t nz_global, z_offset;  /* slab position in the global grid */
} oracle_geom;

/* 8th-order central second-derivative weights: centre, m=1..4. */
static const double W8[R + 1] = { -205.0 / 72.0, 8.0 / 5.0, -1.0 / 5.0, 8.0 / 315.0, -1.0 / 560.0 };

/* Padded linear index, SPEC.md L31 (pad = R on every side, x innermost). */
static inline int64_t pidx(const oracle_geom *g, int64_t i, int64_t j, int64_t k)
{
    return ((k + R) * (g->ny + 2 * R) + (j + R)) * (g->nx + 2 * R) + (i + R);
}

/* Distance (cells) to the inner box along one axis: 0 inside [w, n-w),
 * 1 for the first PML cell, w for the outermost (R3). */
static inline int64_t dist1(int64_t i, int64_t n, int64_t w)
{
    int64_t d = 0;
    if (w - i > d) d = w - i;
    if (i - (n - w - 1) > d) d = i - (n - w - 1);
    return d;
}

/* Chebyshev distance to the inner box (global coordinates). */
static inline int64_t dist3(const oracle_geom *g, int64_t i, int64_t j, int64_t kg)
{
    int64_t d = dist1(i, g->nx, g->w);
    int64_t e = dist1(j, g->ny, g->w);
    int64_t f = dist1(kg, g->nz_global, g->w);
    if (e > d) d = e;
    if (f > d) d = f;
    return d;
}

static inline int inside(const oracle_geom *g, int64_t i, int64_t j, int64_t kg)
{
    return i >= 0 && i < g->nx && j >= 0 && j < g->ny && kg >= 0 && kg < g->nz_global;
}

static double fp32_round(double x) { return (double)(float)x; }

/* ---------------- instantiate for float ---------------- */
#define REAL float
#define SFX(name) name##_f32
struct consts_f32 { float c0, cx[R + 1], cy[R + 1], cz[R + 1], i2h[3]; float *eta, *A, *B; int round32; };
#include "oracle_consts.h"
#include "oracle_body.h"
#undef REAL
#undef SFX

/* ---------------- instantiate for double ---------------- */
#define REAL double
#define SFX(name) name##_f64
struct consts_f64 { double c0, cx[R + 1], cy[R + 1], cz[R + 1], i2h[3]; double *eta, *A, *B; int round32; };
#include "oracle_consts.h"
#include "oracle_body.h"
#undef REAL
#undef SFX

/* dt rule: dt = 0.4 h_min / Vmax, Vmax the fp32 max of V. */
EXPORT float oracle_dt_auto(double hx, double hy, double hz, const float *V, int64_t n)
{
    float vmax = 0.0f;
    for (int64_t i = 0; i < n; ++i) if (V[i] > vmax) vmax = V[i];
    double h = hx;
    if (hy < h) h = hy;
    if (hz < h) h = hz;
    return (float)(0.4 * h / (double)vmax);
}

EXPORT void oracle_set_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

EXPORT int oracle_get_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
