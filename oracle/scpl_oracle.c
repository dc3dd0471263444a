/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle for the buffered SCPL path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * legs may load this library, and only as the checker.  The product path
 * (paper_1903_03180_b200 + libscpl.so) never links or calls it.
 *
 * This file restates, in plain C, the two pieces of third-party arithmetic the
 * reference path leans on (they live in numpy 2.3.5 / scipy-openblas 0.3.30,
 * not under /root/reference):
 *
 *   1. to_luma (pkg/src/vidcarve/energy.py:35-36): `rgb.astype(f64) @ [.299,
 *      .587, .114]` then `np.rint`.  OpenBLAS's dgemv kernel evaluates the
 *      3-term dot product as fma(b, .114, fma(r, .299, g * .587)); pinned against
 *      the reference over all 2^24 RGB triples (tests/golden/luma_table.sha256).
 *   2. numpy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
 *      pairwise_sum_DOUBLE, PW_BLOCKSIZE 128), which is what `.mean()` in
 *      _asde_from_sums (pkg/src/vidcarve/buffering.py:174-176) reduces with.
 *
 * Compile with -ffp-contract=off: every +,* below must round on its own.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>

/* energy.py:35-36 -- BT.601 luma via the OpenBLAS dgemv evaluation order */
void oracle_luma(const uint8_t *rgb, size_t npx, uint8_t *out) {
    for (size_t p = 0; p < npx; ++p) {
        double r = rgb[3 * p], g = rgb[3 * p + 1], b = rgb[3 * p + 2];
        double acc = g * 0.587;
        acc = fma(r, 0.299, acc);
        acc = fma(b, 0.114, acc);
        out[p] = (uint8_t)nearbyint(acc); /* default rounding: ties to even == np.rint */
    }
}

/* numpy pairwise_sum_DOUBLE restated: blocks of <= 128 with 8 accumulators,
 * recursive halving rounded down to a multiple of 8. */
double oracle_pairwise_sum(const double *a, long n) {
    if (n < 8) {
        double s = 0.0;
        for (long i = 0; i < n; ++i) s += a[i];
        return s;
    }
    if (n <= 128) {
        double acc[8];
        for (int k = 0; k < 8; ++k) acc[k] = a[k];
        long i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int k = 0; k < 8; ++k) acc[k] += a[i + k];
        double s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
        for (; i < n; ++i) s += a[i];
        return s;
    }
    long half = n / 2;
    half -= half % 8;
    double left = oracle_pairwise_sum(a, half);
    double right = oracle_pairwise_sum(a + half, n - half);
    return left + right;
}

/* buffering.py:174-176 -- ASDE of a candidate buffer of n maps from its
 * per-pixel sums S and sums of squares Q (N pixels, row-major).  `work` is
 * caller scratch of N doubles. */
double oracle_asde(const double *S, const double *Q, long N, int n, double *work) {
    double dn = (double)n;
    for (long p = 0; p < N; ++p) {
        double m = S[p] / dn;
        double var = Q[p] / dn - m * m;
        work[p] = sqrt(var >= 0.0 ? var : 0.0);
    }
    return (0.0 + oracle_pairwise_sum(work, N)) / (double)N;
}

/* energy.py:40-59 -- edge-replicated 3x3 Sobel, |Gx|+|Gy| clamped to 255, in
 * integers (the reference's float64 values are integer-valued, hence exact). */
void oracle_sobel(const uint8_t *luma, int h, int w, uint8_t *out) {
    for (int i = 0; i < h; ++i) {
        int im = i > 0 ? i - 1 : 0, ip = i < h - 1 ? i + 1 : h - 1;
        for (int j = 0; j < w; ++j) {
            int jm = j > 0 ? j - 1 : 0, jp = j < w - 1 ? j + 1 : w - 1;
#define L(r, c) ((int)luma[(size_t)(r) * w + (c)])
            int gx = (L(im, jp) + 2 * L(i, jp) + L(ip, jp)) - (L(im, jm) + 2 * L(i, jm) + L(ip, jm));
            int gy = (L(ip, jm) + 2 * L(ip, j) + L(ip, jp)) - (L(im, jm) + 2 * L(im, j) + L(im, jp));
#undef L
            int g = (gx < 0 ? -gx : gx) + (gy < 0 ? -gy : gy);
            out[(size_t)i * w + j] = (uint8_t)(g > 255 ? 255 : g);
        }
    }
}
