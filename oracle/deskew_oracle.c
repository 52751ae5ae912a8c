/*
 * CPU ORACLE (test infrastructure only) -- plain C restatement of the
 * reference's deskew + projection path, for parity checks at sizes where the
 * numpy oracle (deskew_oracle.py) is too slow.  Only tests/, smoke() and
 * bench.py's CPU-baseline leg load it; the product never does.
 *
 * Follows (reference file:line):
 *   spans            ss/geometry.py:124-126, 236-255   (snapped ceil/floor, eps = 1e-9)
 *   canvas formula   ss/pipeline.py:229-236  j = u - i*s; j0 = clip(floor j, 0, H-1);
 *                    j1 = min(j0+1, H-1); f = j - j0; rint((1-f)*a + f*b)
 *   npinterp formula ss/phantom.py:396-400 -> numpy arr_interp: j = max{k: xp[k] <= x},
 *                    xp[k] = i*s + k; slope = (fp[j+1]-fp[j]) / (xp[j+1]-xp[j]);
 *                    v = slope*(x - xp[j]) + fp[j]; edge / node cases -> fp[.];
 *                    then rint + clip (ss/phantom.py:402)
 *   nearest          ss/pipeline.py:283-287, ss/phantom.py:393-394
 *
 * Compile with -ffp-contract=off: every product and sum must be rounded on
 * its own, exactly like numpy's element-wise float64 ops.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EPS 1e-9

enum { INTERP_NEAREST = 0, INTERP_LINEAR = 1 };
enum { FORMULA_CANVAS = 0, FORMULA_NPINTERP = 1 };
enum { REDUCE_MAX = 0, REDUCE_SUM = 1 };

static void span_of(int64_t i, double s, int64_t h, int interp, int64_t *lo, int64_t *hi) {
    double off = (double)i * s;
    if (interp == INTERP_NEAREST) {
        *lo = (int64_t)floor(off + 0.5);
        *hi = *lo + h - 1;
    } else {
        *lo = (int64_t)ceil(off - EPS);
        *hi = (int64_t)floor(((off + (double)h) - 1.0) + EPS);
    }
}

static inline uint16_t round_u16(double v) {
    double r = rint(v); /* default rounding mode: half to even, like np.rint */
    if (r < 0.0) r = 0.0;
    if (r > 65535.0) r = 65535.0;
    return (uint16_t)r;
}

/* Values that global slice i contributes to canvas row u (u within its span). */
static void row_values(const uint16_t *px, int64_t h, int64_t w, int64_t i, double s,
                       int interp, int formula, int64_t lo, int64_t u, uint16_t *out) {
    if (interp == INTERP_NEAREST) {
        memcpy(out, px + (u - lo) * w, (size_t)w * sizeof(uint16_t));
        return;
    }
    if (formula == FORMULA_CANVAS) {
        double off = (double)i * s;
        double j = (double)u - off;
        int64_t j0 = (int64_t)floor(j);
        if (j0 < 0) j0 = 0;
        if (j0 > h - 1) j0 = h - 1;
        int64_t j1 = j0 + 1 < h - 1 ? j0 + 1 : h - 1;
        double f = j - (double)j0;
        double w0 = 1.0 - f;
        const uint16_t *a = px + j0 * w, *b = px + j1 * w;
        for (int64_t x = 0; x < w; ++x) {
            double va = w0 * (double)a[x];
            double vb = f * (double)b[x];
            out[x] = round_u16(va + vb);
        }
        return;
    }
    /* np.interp restatement */
    double off = (double)i * s;
    double x = (double)u;
    if (h == 1) {
        memcpy(out, px, (size_t)w * sizeof(uint16_t));
        return;
    }
    /* xp[k] = off + k (float + int -> float64) */
    int64_t k = (int64_t)floor(x - off);
    if (k < -1) k = -1;
    if (k > h - 1) k = h - 1;
    while (k + 1 <= h - 1 && off + (double)(k + 1) <= x) ++k;
    while (k >= 0 && off + (double)k > x) --k;
    const double xp_last = off + (double)(h - 1);
    int64_t src = -1;
    if (k < 0) src = 0;                     /* x < xp[0]  -> left value fp[0]   */
    else if (x > xp_last) src = h - 1;      /* x > xp[-1] -> right value fp[-1] */
    else if (k == h - 1) src = h - 1;       /* x == xp[-1]                      */
    else if (off + (double)k == x) src = k; /* exactly on a node                */
    if (src >= 0) {
        memcpy(out, px + src * w, (size_t)w * sizeof(uint16_t));
        return;
    }
    const double xk = off + (double)k, xk1 = off + (double)(k + 1);
    const double dx = xk1 - xk, t = x - xk;
    const uint16_t *a = px + k * w, *b = px + (k + 1) * w;
    for (int64_t c = 0; c < w; ++c) {
        double slope = ((double)b[c] - (double)a[c]) / dx;
        double v = slope * t;
        v = v + (double)a[c];
        out[c] = round_u16(v);
    }
}

/*
 * stack: n frames (h, w) uint16; global slice index of frame k is first + k.
 * Canvas rows u_begin .. u_begin + u_count - 1.
 * vol (n, u_count, w) uint16, may be NULL.
 * xy (u_count, w), xz (n, w), yz (n, u_count): uint32, may be NULL; zero-filled here.
 * Returns 0 on success, 1 on allocation failure.
 */
int oracle_deskew(const uint16_t *stack, int64_t n, int64_t h, int64_t w, int64_t first,
                  double s, int interp, int formula, int64_t u_begin, int64_t u_count,
                  uint16_t *vol, uint32_t *xy, uint32_t *xz, uint32_t *yz, int reduce) {
    if (xy) memset(xy, 0, (size_t)(u_count * w) * sizeof(uint32_t));
    if (xz) memset(xz, 0, (size_t)(n * w) * sizeof(uint32_t));
    if (yz) memset(yz, 0, (size_t)(n * u_count) * sizeof(uint32_t));
    if (vol) memset(vol, 0, (size_t)(n * u_count * w) * sizeof(uint16_t));
    int64_t *los = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *his = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    if (!los || !his) { free(los); free(his); return 1; }
    for (int64_t k = 0; k < n; ++k) span_of(first + k, s, h, interp, &los[k], &his[k]);
    int fail = 0;
#pragma omp parallel
    {
        uint16_t *row = (uint16_t *)malloc((size_t)w * sizeof(uint16_t));
        uint32_t *xz_local = xz ? (uint32_t *)calloc((size_t)(n * w), sizeof(uint32_t)) : NULL;
        if (!row || (xz && !xz_local)) {
#pragma omp atomic write
            fail = 1;
        } else {
#pragma omp for schedule(dynamic, 4)
            for (int64_t r = 0; r < u_count; ++r) {
                int64_t u = u_begin + r;
                uint32_t *xyr = xy ? xy + r * w : NULL;
                for (int64_t k = 0; k < n; ++k) {
                    if (u < los[k] || u > his[k]) continue;
                    row_values(stack + k * h * w, h, w, first + k, s, interp, formula, los[k], u, row);
                    if (vol) memcpy(vol + (k * u_count + r) * w, row, (size_t)w * sizeof(uint16_t));
                    uint32_t acc = 0;
                    for (int64_t x = 0; x < w; ++x) {
                        uint32_t v = row[x];
                        if (reduce == REDUCE_MAX) {
                            if (xyr && v > xyr[x]) xyr[x] = v;
                            if (xz_local && v > xz_local[k * w + x]) xz_local[k * w + x] = v;
                            if (v > acc) acc = v;
                        } else {
                            if (xyr) xyr[x] += v;
                            if (xz_local) xz_local[k * w + x] += v;
                            acc += v;
                        }
                    }
                    if (yz) yz[k * u_count + r] = acc;
                }
            }
            if (xz) {
#pragma omp critical
                for (int64_t e = 0; e < n * w; ++e) {
                    if (reduce == REDUCE_MAX) { if (xz_local[e] > xz[e]) xz[e] = xz_local[e]; }
                    else xz[e] += xz_local[e];
                }
            }
        }
        free(row);
        free(xz_local);
    }
    free(los);
    free(his);
    return fail;
}

/* ss/pipeline.py:434-457 restated: 1-D row lerp, rint; identity at scale 1. */
int oracle_warp(const uint16_t *proj, int64_t rows, int64_t cols, double scale, uint16_t *out,
                int64_t out_rows) {
    if (scale == 1.0) {
        memcpy(out, proj, (size_t)(rows * cols) * sizeof(uint16_t));
        return 0;
    }
    for (int64_t m = 0; m < out_rows; ++m) {
        double mm = (double)m / scale;
        if (mm < 0.0) mm = 0.0;
        if (mm > (double)(rows - 1)) mm = (double)(rows - 1);
        int64_t m0 = (int64_t)floor(mm);
        int64_t m1 = m0 + 1 < rows - 1 ? m0 + 1 : rows - 1;
        double f = mm - (double)m0;
        double w0 = 1.0 - f;
        for (int64_t c = 0; c < cols; ++c) {
            double va = w0 * (double)proj[m0 * cols + c];
            double vb = f * (double)proj[m1 * cols + c];
            out[m * cols + c] = round_u16(va + vb);
        }
    }
    return 0;
}
