/*
 * CPU oracle helpers in plain C -- TEST INFRASTRUCTURE ONLY.
 *
 * These restate the parts of the reference (`temo` 0.1.0) whose floating-point
 * results depend on BLAS/LAPACK kernels rather than on NumPy ufuncs, so that the
 * oracle does not depend on which OpenBLAS core the host CPU selects:
 *
 *   orc_associate   nsga3.py:96-116   (dgemm Fp@W.T as an FMA chain)
 *   orc_lu_solve    nsga3.py:86       (np.linalg.solve -> getrf/getrs, App. A4)
 *   orc_hv_block    hype.py:77-84     (dominates @ weight -> dgemv_t order, App. A7)
 *
 * Build: gcc -O2 -fPIC -shared -ffp-contract=off -fno-fast-math oracle.c -lm
 * (no FMA contraction: every fused multiply-add below is an explicit fma()).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <float.h>

#define ORC_BIG DBL_MAX

/* NumPy add.reduce over a short contiguous last axis:
 * sequential for m < 8; eight strided accumulators combined pairwise for m >= 8,
 * followed by a sequential tail. */
static double np_lastaxis_sum(const double *v, int m)
{
    if (m < 8) {
        double s = v[0];
        for (int k = 1; k < m; ++k) s = s + v[k];
        return s;
    }
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = v[j];
    int i = 8;
    for (; i + 8 <= m; i += 8)
        for (int j = 0; j < 8; ++j) r[j] = r[j] + v[i + j];
    double s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < m; ++i) s = s + v[i];
    return s;
}

static double row_norm(const double *x, int m)
{
    double sq[64];
    for (int k = 0; k < m; ++k) sq[k] = x[k] * x[k];
    return sqrt(np_lastaxis_sum(sq, m));
}

/* nsga3.associate (nsga3.py:96-116) for rows [0, N). */
void orc_associate(const double *Fp, int64_t N, int m, const double *W, int64_t R,
                   int64_t *pi_out, double *dist_out)
{
    for (int64_t i = 0; i < N; ++i) {
        const double *f = Fp + i * m;
        double nf = row_norm(f, m);
        int64_t best = 0;
        double best_d = 0.0;
        if (nf == 0.0) {
            best = 0;  /* D[norm_f == 0] = 0 -> first index */
            best_d = 0.0;
        } else {
            for (int64_t r = 0; r < R; ++r) {
                const double *w = W + r * m;
                double nw = row_norm(w, m);
                double dot = f[0] * w[0];
                for (int k = 1; k < m; ++k) dot = fma(f[k], w[k], dot);
                double c = dot / (nf * nw);
                double t = 1.0 - c * c;
                if (t < 0.0) t = 0.0;         /* np.clip(., 0, None); NaN passes */
                double d = nf * sqrt(t);
                if (isnan(d)) d = ORC_BIG;    /* np.where(isnan(D), BIG, D) */
                if (r == 0 || d < best_d) { best = r; best_d = d; }
            }
        }
        if (isnan(nf)) best_d = NAN;          /* dist[nan_row] = nan */
        pi_out[i] = best;
        dist_out[i] = best_d;
    }
}

/* np.linalg.solve(E, ones(m)) for m <= 16, bit for bit with NumPy's OpenBLAS 0.3.30
 * (scipy-openblas64, SkylakeX kernels; LAPACK dgesv = getrf_single + getrs_N_single):
 *
 * getf2 (unblocked, column j):  pivots of earlier columns applied to column j; for rows
 *   i < j: b_i -= ddot(L[i, :i], b[:i]) with the strided ddot_k order (4-unrolled pairs,
 *   t1 += fma(y0, x0, y2 x2), t2 += fma(y1, x1, y3 x3), tail fma chain into t1, t1 + t2);
 *   rows i >= j: b_i -= L[i, :j] b[:j] with dgemv_n: rows of the leading (rows & ~3) block
 *   take 4-column groups (acc = a1 x1; fma a0 x0; fma a2 x2; fma a3 x3; y -= acc), then a
 *   2-column group (y -= fma(a0, x0, a1 x1)), then 1 column (y -= round(a0 x0)); the last
 *   (rows & 3) rows take one fma chain over all columns; first max |b| pivot; rows j and jp
 *   swapped over columns 0..j; L column scaled by 1/pivot.
 * getrf_single: blocking = ceil(mn/2 / 2) * 2 (GEMM_UNROLL_N = 2); <= 4 -> getf2 on the
 *   whole matrix, else panels of `blocking` columns: getf2 on the panel, the panel's pivots
 *   on the trailing columns, a unit-lower TRSM in row blocks of 16/8/4/2/1 (GEMM update
 *   from the solved rows as an fma chain from 0, then an in-block fma solve), the trailing
 *   GEMM update (fma chain from 0 over the panel, one subtraction), and finally the later
 *   pivots applied to earlier panels.
 * getrs (nrhs = 1): laswp, unit-lower axpy substitution, upper substitution with true
 *   division.
 * Derived by calling the library's own kernels (ddot_k_SKYLAKEX, dgemv_n_SKYLAKEX,
 * scipy_dgesv_64_) on random inputs; checked against np.linalg.solve for m = 2..16.
 * Returns 0, or 1 on an exactly zero pivot. */
#define ORC_LDA 16

static double orc_ddot_strided(const double *x, const double *y, int n)  /* x: row of L, y: b */
{
    double t1 = 0.0, t2 = 0.0;
    int i = 0;
    for (; i + 4 <= n; i += 4) {
        t1 = t1 + fma(y[i], x[i], y[i + 2] * x[i + 2]);
        t2 = t2 + fma(y[i + 1], x[i + 1], y[i + 3] * x[i + 3]);
    }
    for (; i < n; ++i) t1 = fma(y[i], x[i], t1);
    return t1 + t2;
}

static double orc_gemv_row(const double *a, const double *x, int c, double y, int block_row)
{
    if (!block_row) {
        double t = 0.0;
        for (int k = 0; k < c; ++k) t = fma(a[k], x[k], t);
        return y - t;
    }
    int k = 0;
    for (; k + 4 <= c; k += 4) {
        double t = a[k + 1] * x[k + 1];
        t = fma(a[k], x[k], t);
        t = fma(a[k + 2], x[k + 2], t);
        t = fma(a[k + 3], x[k + 3], t);
        y = y - t;
    }
    if (c - k >= 2) {
        y = y - fma(a[k], x[k], a[k + 1] * x[k + 1]);
        k += 2;
    }
    if (c - k == 1) y = y + a[k] * (-x[k]);
    return y;
}

/* getf2 on rows [r0, m) x columns [c0, c0 + nc) of a (row-major, lda 16); ipiv absolute */
static int orc_getf2(double a[][ORC_LDA], int m, int r0, int c0, int nc, int *ipiv)
{
    const int rows = m - r0;
    double b[16], lrow[16];
    for (int jj = 0; jj < nc; ++jj) {
        const int j = c0 + jj;
        for (int i = 0; i < rows; ++i) b[i] = a[r0 + i][j];
        for (int i = 0; i < jj; ++i) {
            const int jp = ipiv[c0 + i] - r0;
            if (jp != i) { double t = b[i]; b[i] = b[jp]; b[jp] = t; }
        }
        for (int i = 1; i < jj; ++i) {
            for (int k = 0; k < i; ++k) lrow[k] = a[r0 + i][c0 + k];
            b[i] = b[i] - orc_ddot_strided(lrow, b, i);
        }
        const int rr = rows - jj;
        if (jj > 0)
            for (int ii = 0; ii < rr; ++ii) {
                const int i = jj + ii;
                for (int k = 0; k < jj; ++k) lrow[k] = a[r0 + i][c0 + k];
                b[i] = orc_gemv_row(lrow, b, jj, b[i], ii < (rr & ~3));
            }
        int jp = jj;
        double amax = fabs(b[jj]);
        for (int i = jj + 1; i < rows; ++i)
            if (fabs(b[i]) > amax) { amax = fabs(b[i]); jp = i; }
        ipiv[c0 + jj] = r0 + jp;
        for (int i = 0; i < rows; ++i) a[r0 + i][j] = b[i];
        if (b[jp] == 0.0) return 1;
        const double rcp = 1.0 / b[jp];
        if (jp != jj)
            for (int k = c0; k <= j; ++k) { double t = a[r0 + jj][k]; a[r0 + jj][k] = a[r0 + jp][k]; a[r0 + jp][k] = t; }
        for (int i = jj + 1; i < rows; ++i) a[r0 + i][j] = a[r0 + i][j] * rcp;
    }
    return 0;
}

int orc_lu_solve(const double *E, int m, double *y)
{
    double a[16][ORC_LDA];
    int ipiv[16];
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) a[i][j] = E[i * m + j];
    const int blocking = ((m / 2 + 1) / 2) * 2;
    if (blocking <= 4) {
        if (orc_getf2(a, m, 0, 0, m, ipiv)) return 1;
    } else {
        for (int j = 0; j < m; j += blocking) {
            const int jmin = m - j < blocking ? m - j : blocking;
            if (orc_getf2(a, m, j, j, jmin, ipiv)) return 1;
            if (j + jmin >= m) continue;
            for (int c = j + jmin; c < m; ++c)
                for (int i = j; i < j + jmin; ++i)
                    if (ipiv[i] != i) { double t = a[i][c]; a[i][c] = a[ipiv[i]][c]; a[ipiv[i]][c] = t; }
            int bstart[8], bsize[8], nb = 0, r0 = 0, rem = jmin;
            for (int bs = 16; bs >= 1; bs >>= 1)
                while (rem >= bs) { bstart[nb] = r0; bsize[nb++] = bs; r0 += bs; rem -= bs; }
            for (int c = j + jmin; c < m; ++c)
                for (int q = 0; q < nb; ++q) {
                    const int b0 = j + bstart[q], b1 = b0 + bsize[q];
                    if (bstart[q] > 0)
                        for (int i = b0; i < b1; ++i) {
                            double acc = 0.0;
                            for (int k = j; k < b0; ++k) acc = fma(a[i][k], a[k][c], acc);
                            a[i][c] = a[i][c] - acc;
                        }
                    for (int i = b0; i < b1; ++i)
                        for (int k = i + 1; k < b1; ++k) a[k][c] = fma(-a[i][c], a[k][i], a[k][c]);
                }
            for (int i = j + jmin; i < m; ++i)
                for (int c = j + jmin; c < m; ++c) {
                    double acc = 0.0;
                    for (int k = j; k < j + jmin; ++k) acc = fma(a[i][k], a[k][c], acc);
                    a[i][c] = a[i][c] - acc;
                }
        }
        for (int j = 0; j < m; j += blocking) {
            const int jmin = m - j < blocking ? m - j : blocking;
            for (int i = j + jmin; i < m; ++i)
                if (ipiv[i] != i)
                    for (int c = j; c < j + jmin; ++c) { double t = a[i][c]; a[i][c] = a[ipiv[i]][c]; a[ipiv[i]][c] = t; }
        }
    }
    for (int i = 0; i < m; ++i) y[i] = 1.0;
    for (int i = 0; i < m; ++i)
        if (ipiv[i] != i) { double t = y[i]; y[i] = y[ipiv[i]]; y[ipiv[i]] = t; }
    for (int i = 0; i < m; ++i)
        for (int k = i + 1; k < m; ++k) y[k] = fma(-y[i], a[k][i], y[k]);
    for (int i = m - 1; i >= 0; --i) {
        y[i] = y[i] / a[i][i];
        for (int k = 0; k < i; ++k) y[k] = fma(-y[i], a[k][i], y[k]);
    }
    return 0;
}

/* One hv_estimate sample block (hype.py:79-83): given samples S (b x m) and
 * alpha (n1), accumulate contrib[i] += sum_s dom[i,s]*weight[s] in the
 * OpenBLAS dgemv_t order of App. A7.  `counts` receives per-sample dominator
 * counts (size b) and `scratch` must hold n1*b bytes. */
void orc_hv_block(const double *F, int64_t n1, int m, const double *S, int64_t b,
                  const double *alpha, double *contrib, int64_t *counts, uint8_t *scratch)
{
    for (int64_t i = 0; i < n1; ++i) {
        const double *f = F + i * m;
        uint8_t *row = scratch + i * b;
        for (int64_t s = 0; s < b; ++s) {
            const double *x = S + s * m;
            int ok = 1;
            for (int k = 0; k < m; ++k) ok &= (f[k] <= x[k]);
            row[s] = (uint8_t)ok;
        }
    }
    for (int64_t s = 0; s < b; ++s) {
        int64_t c = 0;
        for (int64_t i = 0; i < n1; ++i) c += scratch[i * b + s];
        counts[s] = c;
    }
    int64_t b4 = b - (b % 4);
    int64_t two_lane_lo = -1, two_lane_hi = -1;
    if (n1 % 4 == 2 || n1 % 4 == 3) {
        two_lane_lo = n1 - (n1 % 4);
        two_lane_hi = two_lane_lo + 2;
    }
    for (int64_t i = 0; i < n1; ++i) {
        const uint8_t *row = scratch + i * b;
        int lanes = (i >= two_lane_lo && i < two_lane_hi) ? 2 : 4;
        double y = 0.0;
        for (int64_t lo = 0; lo < b4; lo += 2048) {
            int64_t hi = lo + 2048 < b4 ? lo + 2048 : b4;
            double s[4] = {0.0, 0.0, 0.0, 0.0};
            for (int64_t e = lo; e < hi; ++e) {
                double w = counts[e] > 0 ? alpha[counts[e] - 1] : 0.0;
                double p = (double)row[e] * w;
                int lane = (int)((e - lo) % lanes);
                s[lane] = s[lane] + p;
            }
            double t = lanes == 4 ? (s[0] + s[2]) + (s[1] + s[3]) : s[0] + s[1];
            y = y + t;
        }
        if (b4 < b) {
            double tail = 0.0;
            int first = 1;
            for (int64_t e = b4; e < b; ++e) {
                double w = counts[e] > 0 ? alpha[counts[e] - 1] : 0.0;
                double p = (double)row[e] * w;
                tail = first ? p : tail + p;
                first = 0;
            }
            y = y + tail;
        }
        contrib[i] = contrib[i] + y;
    }
}

/* Elementwise fma for NumPy-side tests: out = a*b + c rounded once. */
void orc_fma(const double *a, const double *b, const double *c, double *out, int64_t n)
{
    for (int64_t i = 0; i < n; ++i) out[i] = fma(a[i], b[i], c[i]);
}
