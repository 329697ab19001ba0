/*
 * TEST INFRASTRUCTURE (oracle/, see oracle/__init__.py): a C restatement of the
 * reference's emulated binary16 Householder reduction, so the CPU oracle can run the
 * level QR at config-3 shapes (6144 x 2048) in seconds instead of the hour the
 * numpy emulation takes.  Never linked into or called by the product package.
 *
 * Follows, operation for operation:
 *   householder_reduce   src/dense.py:108-161  (the loop over pivot columns)
 *   _HalfOps             src/precision.py:118-150 (every scalar op rounded to binary16)
 *   _pairwise_sum        src/precision.py:106-115 (level-by-level adjacent pairs, an odd
 *                                                  trailing element carried to the end)
 * numpy's float16 ufuncs compute each op in binary32 and round the result to
 * binary16 (round to nearest even); the helpers below do exactly that, one explicit
 * cast per op, compiled with -ffp-contract=off so nothing is fused.
 * Pinned bitwise against the reference's R (tests/golden/qr16_golden.json).
 *
 * w: d x n COLUMN-major binary16 working matrix (the already prescaled, rounded
 * sketch), overwritten with R in its upper triangle (alpha on the diagonal, exact
 * zeros below).  Returns 0, or 1 / 2 / 3 for the three RankDeficient triggers
 * (zero pivot column, vanished reflector, tau out of range) with *fail_col set.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef _Float16 h16;

static inline h16 hadd(h16 a, h16 b) { return (h16)((float)a + (float)b); }
static inline h16 hsub(h16 a, h16 b) { return (h16)((float)a - (float)b); }
static inline h16 hmul(h16 a, h16 b) { return (h16)((float)a * (float)b); }
static inline h16 hdiv(h16 a, h16 b) { return (h16)((float)a / (float)b); }
static inline h16 hsqrt(h16 a) { return (h16)sqrtf((float)a); }

/* _pairwise_sum over x[0..L), in place */
static h16 tree(h16 *x, int64_t L) {
    while (L > 1) {
        const int64_t p = L / 2;
        for (int64_t k = 0; k < p; ++k) x[k] = hadd(x[2 * k], x[2 * k + 1]);
        if (L & 1) x[p] = x[L - 1];
        L = p + (L & 1);
    }
    return x[0];
}

int oracle_householder16(uint16_t *w_bits, int64_t d, int64_t n, uint16_t *taus_bits, int *fail_col) {
    h16 *w = (h16 *)w_bits;
    h16 *x = (h16 *)malloc((size_t)d * sizeof(h16));
    h16 *buf = (h16 *)malloc((size_t)d * sizeof(h16));
    int rc = 0;
    *fail_col = -1;
    for (int64_t j = 0; j < n && rc == 0; ++j) {
        const int64_t L = d - j;
        h16 *col = w + j * d + j;
        memcpy(x, col, (size_t)L * sizeof(h16));                     /* x = w[j:, j].copy() */
        for (int64_t i = 0; i < L; ++i) buf[i] = hmul(x[i], x[i]);
        const h16 nrm = hsqrt(tree(buf, L));                          /* sqrt(dot(x, x)) */
        if ((float)nrm == 0.0f) { rc = 1; *fail_col = (int)j; break; }
        const h16 alpha = ((float)x[0] >= 0.0f) ? (h16)(-(float)nrm) : nrm;
        x[0] = hsub(x[0], alpha);                                     /* v = x, v[0] = x0 - alpha */
        for (int64_t i = 0; i < L; ++i) buf[i] = hmul(x[i], x[i]);
        const h16 vtv = tree(buf, L);
        if ((float)vtv == 0.0f) { rc = 2; *fail_col = (int)j; break; }
        const h16 tau = hdiv((h16)2.0f, vtv);
        if (!isfinite((float)tau)) { rc = 3; *fail_col = (int)j; break; }
        if (taus_bits) ((h16 *)taus_bits)[j] = tau;
        /* t = tau * tree(v o w[j:, c]);  w[j:, c] -= v * t   (columns independent) */
#pragma omp parallel
        {
            h16 *p = (h16 *)malloc((size_t)L * sizeof(h16));
#pragma omp for schedule(static)
            for (int64_t c = j + 1; c < n; ++c) {
                h16 *wc = w + c * d + j;
                for (int64_t i = 0; i < L; ++i) p[i] = hmul(x[i], wc[i]);
                const h16 t = hmul(tau, tree(p, L));
                for (int64_t i = 0; i < L; ++i) wc[i] = hsub(wc[i], hmul(x[i], t));
            }
            free(p);
        }
        col[0] = alpha;                                               /* w[j, j] = alpha */
        for (int64_t i = 1; i < L; ++i) col[i] = (h16)0.0f;          /* w[j+1:, j] = 0 */
    }
    free(x);
    free(buf);
    return rc;
}
