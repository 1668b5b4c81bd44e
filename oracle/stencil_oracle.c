/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle for the Minimod acoustic stencil and
 * the fixed-order matmul.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker / the timed CPU baseline.  The
 * product path (paper_2506_02486_b200) never links or calls it.
 *
 * Independent restatement of the reference algorithm:
 *   - per-point update order: reference/pkg/src/diomp/kernels/reference.py:14-31
 *     and kernels/_core.pyx:9-32 (acc = center*u; x taps t=1..R; y taps; z taps;
 *     u_next = (2*u - u_prev) + acc), no FMA contraction (the reference builds
 *     with -ffp-contract=off, pkg/setup.py:22) -- this file must be compiled
 *     with -ffp-contract=off as well (oracle/Makefile does).
 *   - driver: reference/pkg/src/diomp/apps/stencil.py:70-136 (zero fields,
 *     per-step update with u_next aliasing u_prev, point source += amp at the
 *     global centre after the update, buffer swap).
 *
 * Parity pin: tests/golden/stencil_golden.json holds sha256 checksums produced
 * by importing the reference package itself (tests/golden/make_golden.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline size_t at(long i, long j, long k, long NY, long NZ)
{
    return ((size_t)i * (size_t)NY + (size_t)j) * (size_t)NZ + (size_t)k;
}

/* One update of the interior of (NX, NY, NZ) arrays (ghost width r). */
void oracle_stencil_update(double *u_next, const double *u_cur, const double *u_prev,
                           long NX, long NY, long NZ, double center,
                           const double *wx, const double *wy, const double *wz, int r)
{
    for (long i = r; i < NX - r; ++i)
        for (long j = r; j < NY - r; ++j)
            for (long k = r; k < NZ - r; ++k) {
                double u = u_cur[at(i, j, k, NY, NZ)];
                double acc = center * u;
                for (int t = 1; t <= r; ++t)
                    acc = acc + wx[t] * (u_cur[at(i + t, j, k, NY, NZ)] +
                                         u_cur[at(i - t, j, k, NY, NZ)]);
                for (int t = 1; t <= r; ++t)
                    acc = acc + wy[t] * (u_cur[at(i, j + t, k, NY, NZ)] +
                                         u_cur[at(i, j - t, k, NY, NZ)]);
                for (int t = 1; t <= r; ++t)
                    acc = acc + wz[t] * (u_cur[at(i, j, k + t, NY, NZ)] +
                                         u_cur[at(i, j, k - t, NY, NZ)]);
                u_next[at(i, j, k, NY, NZ)] = 2.0 * u - u_prev[at(i, j, k, NY, NZ)] + acc;
            }
}

/*
 * Single-slab run of the driver (the reference proves the result independent
 * of the slab count, selftest.py:466-470).  w[0..r] are the scaled weights of
 * stencil.py:61-67 (computed by the Python caller so the dt arithmetic is
 * Python's own); center = 3*w[0].  field_out receives the (nx, ny, nz)
 * interior in C order (x slowest).  Returns 0, or -1 on allocation failure.
 */
int oracle_stencil_run(long nx, long ny, long nz, long steps, int r,
                       const double *w, double amp, double *field_out)
{
    long NX = nx + 2 * r, NY = ny + 2 * r, NZ = nz + 2 * r;
    size_t n = (size_t)NX * NY * NZ;
    double *a = calloc(n, sizeof(double));
    double *b = calloc(n, sizeof(double));
    if (!a || !b) { free(a); free(b); return -1; }
    double center = 3.0 * w[0];
    size_t src = at(nx / 2 + r, ny / 2 + r, nz / 2 + r, NY, NZ);
    double *prev = a, *cur = b;
    for (long s = 0; s < steps; ++s) {
        oracle_stencil_update(prev, cur, prev, NX, NY, NZ, center, w, w, w, r);
        if (amp != 0.0)
            prev[src] += amp;
        double *t = prev; prev = cur; cur = t;
    }
    for (long i = 0; i < nx; ++i)
        for (long j = 0; j < ny; ++j)
            memcpy(field_out + ((size_t)i * ny + j) * nz, cur + at(i + r, j + r, r, NY, NZ),
                   (size_t)nz * sizeof(double));
    free(a);
    free(b);
    return 0;
}

/*
 * Fixed-order matmul oracle (kernels/reference.py:34-37, _core.pyx:35-46):
 * c[i,j] = left fold over k of a[i,k]*b[k,j], no FMA.
 */
void oracle_matmul_f64(const double *a, const double *b, double *c, long n, long kk, long m)
{
    for (long i = 0; i < n; ++i)
        for (long j = 0; j < m; ++j) {
            double acc = 0.0;
            for (long k = 0; k < kk; ++k)
                acc = acc + a[i * kk + k] * b[k * m + j];
            c[i * m + j] = acc;
        }
}
