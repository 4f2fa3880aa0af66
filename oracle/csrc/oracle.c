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

/* 1/np.linalg.solve(E, ones(m)) for m <= 16 via the left-looking LU of App. A4.
 * E is row-major m x m.  Returns 0, or 1 on an exactly singular pivot. */
int orc_lu_solve(const double *E, int m, double *y)
{
    double a[16][16];
    double b[16];
    int ipiv[16];
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) a[i][j] = E[i * m + j];
    for (int j = 0; j < m; ++j) {
        for (int i = 0; i < m; ++i) b[i] = a[i][j];
        for (int i = 0; i < j; ++i)
            if (ipiv[i] != i) { double t = b[i]; b[i] = b[ipiv[i]]; b[ipiv[i]] = t; }
        for (int i = 1; i < j; ++i) {
            double t = a[i][0] * b[0];
            for (int k = 1; k < i; ++k) t = fma(a[i][k], b[k], t);
            b[i] = b[i] - t;
        }
        if (j > 0) {
            for (int i = j; i < m; ++i) {
                double t = a[i][0] * b[0];
                for (int k = 1; k < j; ++k) t = fma(a[i][k], b[k], t);
                b[i] = b[i] - t;
            }
        }
        int jp = j;
        double amax = fabs(b[j]);
        for (int i = j + 1; i < m; ++i)
            if (fabs(b[i]) > amax) { amax = fabs(b[i]); jp = i; }
        ipiv[j] = jp;
        for (int i = 0; i < m; ++i) a[i][j] = b[i];
        if (jp != j)
            for (int k = 0; k <= j; ++k) { double t = a[j][k]; a[j][k] = a[jp][k]; a[jp][k] = t; }
        if (a[j][j] == 0.0) return 1;
        double rcp = 1.0 / a[j][j];
        for (int i = j + 1; i < m; ++i) a[i][j] = a[i][j] * rcp;
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
