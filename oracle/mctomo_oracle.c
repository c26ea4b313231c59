/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Not part of the product path.
 *
 * Plain-C fp64 restatement of the reference's operators for the hot path
 * (arxiv 2410.10503 package `mctomo`, /root/reference/pkg/src/mctomo):
 *   - Joseph parallel-beam ray transform A and its exact transpose A^*
 *     (projector.py:126-217), computing the traversal weights on the fly instead
 *     of materialising the 48*A*B*n-byte tables, in the reference's own
 *     arithmetic order (separate multiply/add, compiled with
 *     -ffp-contract=off) and, single-threaded, in the reference's own scatter
 *     order (rows group then cols group, table order, projector.py:209-217);
 *   - the bilinear inverse-mapping warp D and its transpose (motion.py:132-194),
 *     plus the dense-field restatement src = p + phi(p) (not in the reference;
 *     SURVEY.md §8a row a9).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library, and only as the checker / the timed CPU baseline.
 * Multi-threaded calls (nthreads > 1) partition the work with private
 * accumulators reduced in a fixed order: deterministic, equal to the
 * single-thread result up to fp64 summation order.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_RIGID 1
#define ORC_DILATATION 2
#define ORC_DENSE 3

int orc_version(void) { return 1; }

/* One Joseph sample of ray (a, j) at dominant index k (projector.py:134-176).
 * Returns the clipped flat tap indices and their weights (already scaled by
 * the step, zero when the tap is outside the grid). */
static inline void joseph_sample(int rows, int cols, int rows_dom, double cs, double sn,
                                 double s_j, int k, long *f0, long *f1, double *w0, double *w1) {
    double cont, step;
    long lim;
    if (rows_dom) {
        double u = (double)k - (rows - 1) / 2.0;  /* projector.py:137 */
        double v = (s_j + u * sn) / cs;           /* :141 */
        cont = v + (cols - 1) / 2.0;              /* :142 */
        step = 1.0 / fabs(cs);                    /* :143 */
        lim = cols;
    } else {
        double v = (double)k - (cols - 1) / 2.0;  /* :148 */
        double u = (v * cs - s_j) / sn;           /* :152 */
        cont = u + (rows - 1) / 2.0;              /* :153 */
        step = 1.0 / sn;                          /* :154 */
        lim = rows;
    }
    double fl = floor(cont);                      /* :161 */
    long i0 = (long)fl;
    double frac = cont - fl;                      /* :162 */
    long i1 = i0 + 1;
    *w0 = (i0 >= 0 && i0 < lim) ? (1.0 - frac) * step : 0.0;  /* :165 */
    *w1 = (i1 >= 0 && i1 < lim) ? frac * step : 0.0;          /* :166 */
    long i0c = i0 < 0 ? 0 : (i0 > lim - 1 ? lim - 1 : i0);    /* :167-168 */
    long i1c = i1 < 0 ? 0 : (i1 > lim - 1 ? lim - 1 : i1);
    if (rows_dom) {                               /* :169-172 */
        *f0 = (long)k * cols + i0c;
        *f1 = (long)k * cols + i1c;
    } else {                                      /* :173-176 */
        *f0 = i0c * cols + k;
        *f1 = i1c * cols + k;
    }
}

static inline double bin_center(int B, double sp, int j) {
    /* Geometry.bin_centers (projector.py:75-79) */
    return ((double)j - (B - 1) / 2.0) * sp;
}

/* A: sino[a, j] = sum_k w0 x[f0] + sum_k w1 x[f1]  (projector.py:201-207). */
void orc_ray_forward(int rows, int cols, int A, int B, double sp, const double *cos_a,
                     const double *sin_a, const uint8_t *rows_dom, const double *x, double *sino,
                     int nthreads) {
#ifdef _OPENMP
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(dynamic, 4) num_threads(nthreads)
#endif
    for (long aj = 0; aj < (long)A * B; ++aj) {
        int a = (int)(aj / B), j = (int)(aj % B);
        int rd = rows_dom[a];
        int nmaj = rd ? rows : cols;
        double s_j = bin_center(B, sp, j);
        double acc0 = 0.0, acc1 = 0.0;
        for (int k = 0; k < nmaj; ++k) {
            long f0, f1;
            double w0, w1;
            joseph_sample(rows, cols, rd, cos_a[a], sin_a[a], s_j, k, &f0, &f1, &w0, &w1);
            acc0 += x[f0] * w0;
            acc1 += x[f1] * w1;
        }
        sino[aj] = acc0 + acc1;
    }
}

/* A^*: exact transpose, scatter (projector.py:209-217).  nthreads == 1
 * reproduces the reference's bincount order: rows group, then cols group,
 * each in (angle, bin, tap0 samples, tap1 samples) table order. */
void orc_ray_adjoint(int rows, int cols, int A, int B, double sp, const double *cos_a,
                     const double *sin_a, const uint8_t *rows_dom, const double *y, double *img,
                     int nthreads) {
    const long n = (long)rows * cols;
    if (nthreads < 1) nthreads = 1;
    int nt = nthreads;
    double *priv = (double *)calloc((size_t)nt * 2 * n, sizeof(double));
#ifdef _OPENMP
#pragma omp parallel num_threads(nt)
#endif
    {
        int t = 0;
#ifdef _OPENMP
        t = omp_get_thread_num();
#endif
        for (int grp = 0; grp < 2; ++grp) {
            double *acc = priv + ((size_t)t * 2 + grp) * n;
            int want_rows = (grp == 0);
            /* contiguous angle partition per thread keeps the per-thread order
             * identical to the table order restricted to its angles */
            int a_lo = (int)((long)A * t / nt), a_hi = (int)((long)A * (t + 1) / nt);
            for (int a = a_lo; a < a_hi; ++a) {
                if ((rows_dom[a] != 0) != want_rows) continue;
                int nmaj = want_rows ? rows : cols;
                for (int j = 0; j < B; ++j) {
                    double s_j = bin_center(B, sp, j);
                    double yv = y[(long)a * B + j];
                    for (int tap = 0; tap < 2; ++tap) {
                        for (int k = 0; k < nmaj; ++k) {
                            long f0, f1;
                            double w0, w1;
                            joseph_sample(rows, cols, want_rows, cos_a[a], sin_a[a], s_j, k, &f0,
                                          &f1, &w0, &w1);
                            if (tap == 0)
                                acc[f0] += yv * w0;
                            else
                                acc[f1] += yv * w1;
                        }
                    }
                }
            }
        }
    }
    /* fixed-order reduction: per group over threads, then rows + cols */
    for (long p = 0; p < n; ++p) {
        double r = 0.0, c = 0.0;
        for (int t = 0; t < nt; ++t) {
            r += priv[((size_t)t * 2 + 0) * n + p];
            c += priv[((size_t)t * 2 + 1) * n + p];
        }
        img[p] = (0.0 + r) + c;
    }
    free(priv);
}

/* ------------------------------------------------------------------ warps */
/* Source position and the 4 bilinear taps of output pixel (r, c):
 * motion.py:132-176 (rigid / dilatation), dense restatement src = p + phi. */
static inline void warp_taps(int kind, int rows, int cols, double cs, double sn, double tr,
                             double tc, double scale, const float *phi, int r, int c, long flat[4],
                             double w[4]) {
    double src_r, src_c;
    if (kind == ORC_DENSE) {
        long p = (long)r * cols + c;
        src_r = (double)r + (double)phi[p];
        src_c = (double)c + (double)phi[(long)rows * cols + p];
    } else {
        double u = (double)r - (rows - 1) / 2.0; /* motion.py:135-137 */
        double v = (double)c - (cols - 1) / 2.0;
        double su, sv;
        if (kind == ORC_RIGID) {
            double du = u - tr, dv = v - tc;    /* :148-149 */
            su = cs * du + sn * dv;             /* :150 */
            sv = -sn * du + cs * dv;            /* :151 */
        } else {
            su = u / scale;                     /* :153 */
            sv = v / scale;                     /* :154 */
        }
        src_r = su + (rows - 1) / 2.0;          /* :155 */
        src_c = sv + (cols - 1) / 2.0;          /* :156 */
    }
    double r0f = floor(src_r), c0f = floor(src_c);
    double fr = src_r - r0f, fc = src_c - c0f;  /* :157-160 */
    double ww[4] = {(1.0 - fr) * (1.0 - fc), (1.0 - fr) * fc, fr * (1.0 - fc), fr * fc};
    static const int DR[4] = {0, 0, 1, 1}, DC[4] = {0, 1, 0, 1};
    for (int k = 0; k < 4; ++k) {
        double rr = r0f + DR[k], cc = c0f + DC[k];
        int valid = rr >= 0 && rr < rows && cc >= 0 && cc < cols;
        long ri = rr < 0 ? 0 : (rr > rows - 1 ? rows - 1 : (long)rr);
        long ci = cc < 0 ? 0 : (cc > cols - 1 ? cols - 1 : (long)cc);
        flat[k] = ri * cols + ci;                 /* :172 */
        w[k] = valid ? ww[k] : 0.0;               /* :173 */
    }
}

/* D: out[p] = sum_k w[k,p] x[flat[k,p]]  (motion.py:178-183) */
void orc_warp_forward(int kind, int rows, int cols, double cs, double sn, double tr, double tc,
                      double scale, const float *phi, const double *x, double *out) {
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) {
            long flat[4];
            double w[4];
            warp_taps(kind, rows, cols, cs, sn, tr, tc, scale, phi, r, c, flat, w);
            double acc = 0.0;
            for (int k = 0; k < 4; ++k) acc += x[flat[k]] * w[k];
            out[(long)r * cols + c] = acc;
        }
}

/* D^*: bincount scatter in tap-major order (motion.py:185-194) */
void orc_warp_adjoint(int kind, int rows, int cols, double cs, double sn, double tr, double tc,
                      double scale, const float *phi, const double *y, double *out) {
    const long n = (long)rows * cols;
    memset(out, 0, sizeof(double) * n);
    for (int k = 0; k < 4; ++k)
        for (int r = 0; r < rows; ++r)
            for (int c = 0; c < cols; ++c) {
                long flat[4];
                double w[4];
                warp_taps(kind, rows, cols, cs, sn, tr, tc, scale, phi, r, c, flat, w);
                long p = (long)r * cols + c;
                out[flat[k]] += w[k] * y[p];
            }
}
