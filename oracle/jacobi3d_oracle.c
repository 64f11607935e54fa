/*
 * oracle/jacobi3d_oracle.c -- CPU ORACLE FOR THE OVERDECOMPOSED JACOBI3D HOT PATH.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or execute this code.  The
 * product path (paper_2605_12734_b200/) never links, imports or calls it, and
 * this file shares no code, header, table or constant generator with it.
 *
 * What it computes (§5 "jacobi2d": "applies the Jacobi iterative
 * method on a 2D grid ... run for 100 iterations without convergence checks";
 * lifted to 3D per SURVEY.md §8(c) reading R1): the plain, UNDECOMPOSED Jacobi
 * iteration on the padded global grid.  Overdecomposition (blocks, ODF, GPUs) is
 * an execution strategy for this same iteration, so the oracle never sees it
 * ("bit-exact ... serial reference Jacobi on the full grid").
 *
 * Readings:
 *   R2  arithmetic mean of the 7 stencil points (centre included)
 *   R3  multiply by K = fl(1/7) written as a hex literal, not a division by 7
 *   R4  fixed left-to-right order ((((((c + x-) + x+) + y-) + y+) + z-) + z+) * K
 *   R6  Dirichlet: the 1-cell shell of the padded array keeps U0's values forever
 *   R7  nx,ny,nz count the UPDATED (interior) points; the shell is extra
 *   R8  IEEE binary64, round-to-nearest-even
 *   R12 exactly n sweeps, n = 0 is the identity
 *
 * Layout: padded array of (nz+2)*(ny+2)*(nx+2) doubles, x fastest,
 *   p(i,j,k) = (k*(ny+2) + j)*(nx+2) + i,  i in [0,nx+1], j in [0,ny+1], k in [0,nz+1].
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math (-fopenmp for the _omp variant).
 * The sum-then-scale update has no a*b+c pattern, so contraction cannot alter it;
 * -ffp-contract=off is kept anyway so the claim does not depend on the compiler.
 *
 * Pins (tests/test_oracle_pins.py, all -m "not gpu"): constant field (P1), linear
 * field (P2), the 4^3 hand cases (P3, tests/golden/p3_cube4.txt), eigenmode
 * closed form (P4), rounding-error bound against exact rationals (P5), numpy
 * second oracle (P6), CPU blockwise partition invariance (P7), light cone (P8),
 * identity/determinism/restart (P9), OpenMP == serial (P10), max principle (P12),
 * SURVEY C1 regression constants (tests/golden/c1_regression.txt).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* fl(1/7): the binary64 nearest to 1/7 (relative error exactly -2^-54). Reading R3. */
static const double ORACLE_K = 0x1.2492492492492p-3;

/* One Jacobi sweep A -> B over the interior, in k, j, i order (any order gives the
 * same bits: each point reads only iteration-t values). */
static void sweep(int64_t nx, int64_t ny, int64_t nz, const double *A, double *B,
                  int64_t k_lo, int64_t k_hi)
{
    const int64_t sy = nx + 2;              /* stride between y-neighbours */
    const int64_t sz = (nx + 2) * (ny + 2); /* stride between z-neighbours */
    for (int64_t k = k_lo; k <= k_hi; ++k)
        for (int64_t j = 1; j <= ny; ++j)
            for (int64_t i = 1; i <= nx; ++i) {
                const int64_t p = (k * (ny + 2) + j) * (nx + 2) + i;
                double s = A[p];          /* centre */
                s = s + A[p - 1];         /* x- */
                s = s + A[p + 1];         /* x+ */
                s = s + A[p - sy];        /* y- */
                s = s + A[p + sy];        /* y+ */
                s = s + A[p - sz];        /* z- */
                s = s + A[p + sz];        /* z+ */
                B[p] = s * ORACLE_K;
            }
}

/* Returns 0 on success, -1 on bad arguments, -2 on allocation failure.
 * u0 and out are host arrays of padded size; they may alias.  *loop_seconds (if
 * non-NULL) receives the wall time of the iteration loop alone (the bench's
 * single-threaded CPU baseline, SURVEY §8(d.4) mode (a)); timing only. */
static double now_s(void);
int oracle_jacobi3d_timed(int64_t nx, int64_t ny, int64_t nz, const double *u0, int64_t n,
                          double *out, double *loop_seconds)
{
    if (nx < 1 || ny < 1 || nz < 1 || n < 0 || !u0 || !out) return -1;
    const size_t cells = (size_t)(nx + 2) * (size_t)(ny + 2) * (size_t)(nz + 2);
    double *A = (double *)malloc(cells * sizeof(double));
    double *B = (double *)malloc(cells * sizeof(double));
    if (!A || !B) { free(A); free(B); return -2; }
    memcpy(A, u0, cells * sizeof(double));
    memcpy(B, u0, cells * sizeof(double)); /* shell identical in both, never written */
    const double t0 = now_s();
    for (int64_t it = 0; it < n; ++it) {
        sweep(nx, ny, nz, A, B, 1, nz);
        double *t = A; A = B; B = t;
    }
    if (loop_seconds) *loop_seconds = now_s() - t0;
    memcpy(out, A, cells * sizeof(double));
    free(A); free(B);
    return 0;
}

int oracle_jacobi3d(int64_t nx, int64_t ny, int64_t nz, const double *u0, int64_t n,
                    double *out)
{
    return oracle_jacobi3d_timed(nx, ny, nz, u0, n, out, 0);
}

/* Same iteration with the k-loop split over OpenMP threads.
 * Per-point arithmetic is unchanged, so the result is bit-identical to the serial
 * oracle.  nthreads <= 0 means the OpenMP default.  Returns the thread count used
 * (>=1) or a negative error as above. */
#include <time.h>
static double now_s(void)
{
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

int oracle_jacobi3d_omp_timed(int64_t nx, int64_t ny, int64_t nz, const double *u0, int64_t n,
                              double *out, int nthreads, double *loop_seconds);

int oracle_jacobi3d_omp(int64_t nx, int64_t ny, int64_t nz, const double *u0, int64_t n,
                        double *out, int nthreads)
{
    return oracle_jacobi3d_omp_timed(nx, ny, nz, u0, n, out, nthreads, 0);
}

/* As oracle_jacobi3d_omp; *loop_seconds (if non-NULL) receives the wall time of the
 * iteration loop alone (monotonic clock), for the bench's CPU baseline. */
int oracle_jacobi3d_omp_timed(int64_t nx, int64_t ny, int64_t nz, const double *u0, int64_t n,
                              double *out, int nthreads, double *loop_seconds)
{
    if (nx < 1 || ny < 1 || nz < 1 || n < 0 || !u0 || !out) return -1;
    const size_t cells = (size_t)(nx + 2) * (size_t)(ny + 2) * (size_t)(nz + 2);
    double *A = (double *)malloc(cells * sizeof(double));
    double *B = (double *)malloc(cells * sizeof(double));
    if (!A || !B) { free(A); free(B); return -2; }
    int used = 1;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
    {
#pragma omp single
        used = omp_get_num_threads();
    }
#endif
    memcpy(A, u0, cells * sizeof(double));
    memcpy(B, u0, cells * sizeof(double));
    const double t0 = now_s();
    for (int64_t it = 0; it < n; ++it) {
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
        for (int64_t k = 1; k <= nz; ++k) sweep(nx, ny, nz, A, B, k, k);
        double *t = A; A = B; B = t;
    }
    if (loop_seconds) *loop_seconds = now_s() - t0;
    memcpy(out, A, cells * sizeof(double));
    free(A); free(B);
    return used;
}

/* Reporting helpers. Not part of the method. */

/* Left-to-right sum over the interior in k, j, i order. */
double oracle_checksum(int64_t nx, int64_t ny, int64_t nz, const double *u)
{
    double s = 0.0;
    for (int64_t k = 1; k <= nz; ++k)
        for (int64_t j = 1; j <= ny; ++j)
            for (int64_t i = 1; i <= nx; ++i) s = s + u[(k * (ny + 2) + j) * (nx + 2) + i];
    return s;
}

/* H = sum_q bits(u_q) * (2q+1) mod 2^64 over the interior, q = interior index in
 * k, j, i order. */
uint64_t oracle_bithash(int64_t nx, int64_t ny, int64_t nz, const double *u)
{
    uint64_t h = 0, q = 0;
    for (int64_t k = 1; k <= nz; ++k)
        for (int64_t j = 1; j <= ny; ++j)
            for (int64_t i = 1; i <= nx; ++i, ++q) {
                uint64_t b;
                memcpy(&b, &u[(k * (ny + 2) + j) * (nx + 2) + i], sizeof b);
                h += b * (2u * q + 1u);
            }
    return h;
}

/* ------------------------------------------------------------------ Jacobi2D
 * the paper's own stencil app, "applies the Jacobi iterative
 * method on a 2D grid".  SPEC.md:474 fixes the update as a "5-point
 * average into a double-buffered tile" with "fixed borders (outer halo = initial
 * boundary values)".  Readings (DESIGN.md §2, 2-D column): mean of the 5 points,
 * x fl(1/5) = 0x1.999999999999ap-3, fixed order ((((c + x-) + x+) + y-) + y+).
 * Padded array (ny+2)*(nx+2), x fastest, p(i,j) = j*(nx+2) + i. */
static const double ORACLE_K5 = 0x1.999999999999ap-3;

static void sweep2d(int64_t nx, int64_t ny, const double *A, double *B, int64_t j_lo, int64_t j_hi)
{
    const int64_t sy = nx + 2;
    for (int64_t j = j_lo; j <= j_hi; ++j)
        for (int64_t i = 1; i <= nx; ++i) {
            const int64_t p = j * (nx + 2) + i;
            double s = A[p];       /* centre */
            s = s + A[p - 1];      /* x- */
            s = s + A[p + 1];      /* x+ */
            s = s + A[p - sy];     /* y- */
            s = s + A[p + sy];     /* y+ */
            B[p] = s * ORACLE_K5;
        }
}

int oracle_jacobi2d_omp_timed(int64_t nx, int64_t ny, const double *u0, int64_t n, double *out, int nthreads,
                              double *loop_seconds);

int oracle_jacobi2d_omp(int64_t nx, int64_t ny, const double *u0, int64_t n, double *out, int nthreads)
{
    return oracle_jacobi2d_omp_timed(nx, ny, u0, n, out, nthreads, 0);
}

/* As oracle_jacobi2d_omp; *loop_seconds (if non-NULL) = wall time of the iteration
 * loop alone (for the bench's CPU baseline). */
int oracle_jacobi2d_omp_timed(int64_t nx, int64_t ny, const double *u0, int64_t n, double *out, int nthreads,
                              double *loop_seconds)
{
    if (nx < 1 || ny < 1 || n < 0 || !u0 || !out) return -1;
    const size_t cells = (size_t)(nx + 2) * (size_t)(ny + 2);
    double *A = (double *)malloc(cells * sizeof(double));
    double *B = (double *)malloc(cells * sizeof(double));
    if (!A || !B) { free(A); free(B); return -2; }
    int used = 1;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
    {
#pragma omp single
        used = omp_get_num_threads();
    }
#endif
    memcpy(A, u0, cells * sizeof(double));
    memcpy(B, u0, cells * sizeof(double));
    const double t0 = now_s();
    for (int64_t it = 0; it < n; ++it) {
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
        for (int64_t j = 1; j <= ny; ++j) sweep2d(nx, ny, A, B, j, j);
        double *t = A; A = B; B = t;
    }
    if (loop_seconds) *loop_seconds = now_s() - t0;
    memcpy(out, A, cells * sizeof(double));
    free(A); free(B);
    return used;
}

int oracle_jacobi2d(int64_t nx, int64_t ny, const double *u0, int64_t n, double *out)
{
    if (nx < 1 || ny < 1 || n < 0 || !u0 || !out) return -1;
    const size_t cells = (size_t)(nx + 2) * (size_t)(ny + 2);
    double *A = (double *)malloc(cells * sizeof(double));
    double *B = (double *)malloc(cells * sizeof(double));
    if (!A || !B) { free(A); free(B); return -2; }
    memcpy(A, u0, cells * sizeof(double));
    memcpy(B, u0, cells * sizeof(double));
    for (int64_t it = 0; it < n; ++it) {
        sweep2d(nx, ny, A, B, 1, ny);
        double *t = A; A = B; B = t;
    }
    memcpy(out, A, cells * sizeof(double));
    free(A); free(B);
    return 0;
}

int oracle_has_openmp(void)
{
#ifdef _OPENMP
    return 1;
#else
    return 0;
#endif
}
