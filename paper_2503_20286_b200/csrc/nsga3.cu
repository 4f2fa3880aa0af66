// NSGA-III environmental selection on B200 (replaces temo nsga3.py:61-218).
//
// Everything after the ND sort runs on the device with no host round trip;
// data-dependent sizes (l, promoted count, repair count) live in device
// scalars.  Bit-exactness with the NumPy reference:
//   normalize  nsga3.py:61-93   exact IEEE ops (--fmad=false); LAPACK solve
//                               reproduced by the left-looking LU of SURVEY
//                               App. A4 (explicit fma); the rank/cond gate is
//                               a one-sided Jacobi SVD (same decision).
//   associate  nsga3.py:96-116  cheap FP64 filter s_j = f . w_j/|w_j| with a
//                               running-max margin, then the exact reference
//                               expression (App. A2/A3) on every candidate
//                               within the margin, first index on ties.
//   niche      nsga3.py:119-183 histogram + per-direction (dist, index) argmin
//                               via two atomicMin phases; promotions in
//                               direction order; index-order repair.
#include <cub/cub.cuh>

#include "common.cuh"

namespace temo {

constexpr int NT = 256;
constexpr int STAT_BLOCKS = 296;
constexpr int MAXM = 16;
constexpr double ASF_EPS = 1e-6;
constexpr double COND_LIMIT = 1e8;
constexpr double ICPT_FLOOR = 1e-10;
constexpr double FILTER_MARGIN = 1e-12;  // relative, see k_associate
constexpr double FILTER_MIN_COS = 0.05;  // below this the filter proof does not hold

__device__ __forceinline__ double key_to_double(uint64_t k) {
    uint64_t u = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
    return __longlong_as_double((long long)u);
}

// ---------------------------------------------------------------- gather
__global__ void k_gather_rows(const double *__restrict__ src, const int32_t *__restrict__ idx,
                              const int64_t *__restrict__ idx64, int64_t rows, int64_t cols,
                              double *__restrict__ dst) {
    // one warp per row, vectorised when cols is even
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= rows) return;
    const int64_t s = idx ? (int64_t)idx[warp] : idx64[warp];
    const double *a = src + s * cols;
    double *b = dst + warp * cols;
    if ((cols & 1) == 0 && (((uintptr_t)a | (uintptr_t)b) & 15) == 0) {
        const double2 *a2 = reinterpret_cast<const double2 *>(a);
        double2 *b2 = reinterpret_cast<double2 *>(b);
        for (int64_t c = lane; c < cols / 2; c += 32) b2[c] = __ldg(a2 + c);
    } else {
        for (int64_t c = lane; c < cols; c += 32) b[c] = __ldg(a + c);
    }
}

// composed gather: dst[r] = src[idx_a[idx_b[r]]]
__global__ void k_gather_rows2(const double *__restrict__ src, const int64_t *__restrict__ idx_a,
                               const int32_t *__restrict__ idx_b, int64_t rows, int64_t cols,
                               double *__restrict__ dst) {
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= rows) return;
    const int64_t s = idx_a[idx_b[warp]];
    const double *a = src + s * cols;
    double *b = dst + warp * cols;
    if ((cols & 1) == 0 && (((uintptr_t)a | (uintptr_t)b) & 15) == 0) {
        const double2 *a2 = reinterpret_cast<const double2 *>(a);
        double2 *b2 = reinterpret_cast<double2 *>(b);
        for (int64_t c = lane; c < cols / 2; c += 32) b2[c] = __ldg(a2 + c);
    } else {
        for (int64_t c = lane; c < cols; c += 32) b[c] = __ldg(a + c);
    }
}

// ---------------------------------------------------------------- normalize
// per-block min/max (as order keys) of each column over retained rows r <= l
__global__ void __launch_bounds__(NT) k_colstats(const double *__restrict__ F, int64_t N, int m,
                                                 const int32_t *__restrict__ rank,
                                                 const int32_t *__restrict__ lp,
                                                 uint64_t *__restrict__ part) {
    __shared__ uint64_t smin[NT / 32][MAXM], smax[NT / 32][MAXM];
    const int l = *lp;
    uint64_t mn[MAXM], mx[MAXM];
    for (int k = 0; k < m; ++k) { mn[k] = ~0ull; mx[k] = 0ull; }
    for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < N; i += (int64_t)gridDim.x * NT) {
        if (rank[i] > l) continue;
        for (int k = 0; k < m; ++k) {
            const double x = F[i * m + k];
            if (isnan(x)) continue;  // np.nanmin / np.nanmax
            const uint64_t key = ordered_key(x);
            mn[k] = key < mn[k] ? key : mn[k];
            mx[k] = key > mx[k] ? key : mx[k];
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int k = 0; k < m; ++k) {
        uint64_t a = mn[k], b = mx[k];
        for (int d = 16; d; d >>= 1) {
            uint64_t a2 = __shfl_xor_sync(~0u, a, d), b2 = __shfl_xor_sync(~0u, b, d);
            a = a2 < a ? a2 : a;
            b = b2 > b ? b2 : b;
        }
        if (lane == 0) { smin[warp][k] = a; smax[warp][k] = b; }
    }
    __syncthreads();
    if (threadIdx.x < m) {
        const int k = threadIdx.x;
        uint64_t a = ~0ull, b = 0;
        for (int w = 0; w < NT / 32; ++w) {
            a = smin[w][k] < a ? smin[w][k] : a;
            b = smax[w][k] > b ? smax[w][k] : b;
        }
        part[(int64_t)blockIdx.x * 2 * m + k] = a;
        part[(int64_t)blockIdx.x * 2 * m + m + k] = b;
    }
}

__global__ void k_colstats_final(const uint64_t *__restrict__ part, int nblk, int m,
                                 double *__restrict__ ideal, double *__restrict__ nadir) {
    const int k = threadIdx.x;
    if (k >= m) return;
    uint64_t a = ~0ull, b = 0;
    for (int q = 0; q < nblk; ++q) {
        a = part[q * 2 * m + k] < a ? part[q * 2 * m + k] : a;
        b = part[q * 2 * m + m + k] > b ? part[q * 2 * m + m + k] : b;
    }
    ideal[k] = key_to_double(a);
    nadir[k] = key_to_double(b);
}

// ASF score of row i for axis a: max_k shifted_k / w_a[k], w = max(eye, 1e-6)
__device__ __forceinline__ double asf(const double *f, const double *ideal, int m, int a) {
    // np.max over the row: NaN propagates, otherwise the largest value
    double best = -INFINITY;
    bool nan = false;
    for (int k = 0; k < m; ++k) {
        const double sh = f[k] - ideal[k];
        const double v = k == a ? sh / 1.0 : sh / ASF_EPS;
        if (isnan(v)) nan = true;
        else if (v > best) best = v;
    }
    return nan ? __longlong_as_double(0x7FF8000000000000ll) : best;
}

// per-block first-argmin of the ASF score per axis (excluded rows score BIG)
__global__ void __launch_bounds__(NT) k_asf_argmin(const double *__restrict__ F, int64_t N, int m,
                                                   const int32_t *__restrict__ rank,
                                                   const int32_t *__restrict__ lp,
                                                   const double *__restrict__ ideal,
                                                   uint64_t *__restrict__ pkey,
                                                   int64_t *__restrict__ pidx) {
    __shared__ double s_ideal[MAXM];
    __shared__ uint64_t sk[NT / 32];
    __shared__ int64_t si[NT / 32];
    if (threadIdx.x < m) s_ideal[threadIdx.x] = ideal[threadIdx.x];
    __syncthreads();
    const int l = *lp;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int a = 0; a < m; ++a) {
        uint64_t bk = ~0ull;
        int64_t bi = INT64_MAX;
        for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < N; i += (int64_t)gridDim.x * NT) {
            double sc = TEMO_BIG;
            if (rank[i] <= l) {
                sc = asf(F + i * m, s_ideal, m, a);
                if (isnan(sc)) sc = TEMO_BIG;
            }
            const uint64_t key = ordered_key(sc);
            if (key < bk || (key == bk && i < bi)) { bk = key; bi = i; }
        }
        for (int d = 16; d; d >>= 1) {
            const uint64_t k2 = __shfl_xor_sync(~0u, bk, d);
            const int64_t i2 = __shfl_xor_sync(~0u, bi, d);
            if (k2 < bk || (k2 == bk && i2 < bi)) { bk = k2; bi = i2; }
        }
        if (lane == 0) { sk[warp] = bk; si[warp] = bi; }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < NT / 32; ++w)
                if (sk[w] < bk || (sk[w] == bk && si[w] < bi)) { bk = sk[w]; bi = si[w]; }
            pkey[(int64_t)blockIdx.x * m + a] = bk;
            pidx[(int64_t)blockIdx.x * m + a] = bi;
        }
        __syncthreads();
    }
}

// singular values of an m x m matrix by one-sided Jacobi (only the gate's decision matters)
__device__ void jacobi_singular_values(const double *E, int m, double *sv) {
    double A[MAXM][MAXM];
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) A[i][j] = E[i * m + j];
    for (int sweep = 0; sweep < 60; ++sweep) {
        bool rotated = false;
        for (int p = 0; p < m - 1; ++p)
            for (int q = p + 1; q < m; ++q) {
                double alpha = 0, beta = 0, gamma = 0;
                for (int i = 0; i < m; ++i) {
                    alpha = fma(A[i][p], A[i][p], alpha);
                    beta = fma(A[i][q], A[i][q], beta);
                    gamma = fma(A[i][p], A[i][q], gamma);
                }
                if (gamma == 0.0 || fabs(gamma) <= 1e-17 * sqrt(alpha * beta)) continue;
                rotated = true;
                const double zeta = (beta - alpha) / (2.0 * gamma);
                const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
                for (int i = 0; i < m; ++i) {
                    const double x = A[i][p], y = A[i][q];
                    A[i][p] = c * x - s * y;
                    A[i][q] = s * x + c * y;
                }
            }
        if (!rotated) break;
    }
    for (int j = 0; j < m; ++j) {
        double s = 0;
        for (int i = 0; i < m; ++i) s = fma(A[i][j], A[i][j], s);
        sv[j] = sqrt(s);
    }
}

// np.linalg.solve(E, ones) (nsga3.py:86) bit for bit with NumPy's OpenBLAS 0.3.30 on the
// SkylakeX kernels (LAPACK dgesv = getrf_single + getrs_N_single), for every m <= 16:
//   getf2 column j: earlier pivots applied; rows i < j: b_i -= ddot_k(L[i,:i], b) in the
//     strided ddot order (4-unrolled pairs t1 += fma(y0,x0,y2 x2), t2 += fma(y1,x1,y3 x3),
//     tail fma chain into t1, t1 + t2); rows i >= j: dgemv_n -- rows of the leading
//     (rows & ~3) block subtract 4-column groups (acc = a1 x1, fma a0 x0, fma a2 x2, fma a3 x3),
//     then a 2-column group (fma(a0, x0, a1 x1)), then one column (round(a0 x0)); the last
//     (rows & 3) rows subtract one fma chain over all columns; first max |b| pivot, rows
//     swapped over columns 0..j, L scaled by 1/pivot.
//   getrf_single: blocking = ceil(m/2 / 2) * 2; > 4 (m >= 10) -> panels: getf2 on the panel,
//     its pivots on the trailing columns, unit-lower TRSM in row blocks 16/8/4/2/1 (GEMM
//     update from solved rows as an fma chain from 0, then an in-block fma solve), trailing
//     GEMM (fma chain from 0, one subtraction), later pivots applied to earlier panels.
//   getrs: laswp, unit-lower axpy substitution, upper substitution with true division.
// Derived from the library's own kernels (see oracle/csrc/oracle.c, orc_lu_solve, the
// independent CPU restatement; tests pin both against np.linalg.solve for m = 2..16).
// Returns false on an exactly zero pivot.
__device__ double lu_ddot_strided(const double *x, const double *y, int n) {
    double t1 = 0.0, t2 = 0.0;
    int i = 0;
    for (; i + 4 <= n; i += 4) {
        t1 = t1 + fma(y[i], x[i], y[i + 2] * x[i + 2]);
        t2 = t2 + fma(y[i + 1], x[i + 1], y[i + 3] * x[i + 3]);
    }
    for (; i < n; ++i) t1 = fma(y[i], x[i], t1);
    return t1 + t2;
}

__device__ double lu_gemv_row(const double *a, const double *x, int c, double y, bool block_row) {
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

// getf2 on rows [r0, m) x columns [c0, c0 + nc) (row-major a, leading dimension MAXM)
__device__ bool lu_getf2(double (*a)[MAXM], int m, int r0, int c0, int nc, int *ipiv) {
    const int rows = m - r0;
    double b[MAXM], lrow[MAXM];
    for (int jj = 0; jj < nc; ++jj) {
        const int j = c0 + jj;
        for (int i = 0; i < rows; ++i) b[i] = a[r0 + i][j];
        for (int i = 0; i < jj; ++i) {
            const int jp = ipiv[c0 + i] - r0;
            if (jp != i) { double t = b[i]; b[i] = b[jp]; b[jp] = t; }
        }
        for (int i = 1; i < jj; ++i) {
            for (int k = 0; k < i; ++k) lrow[k] = a[r0 + i][c0 + k];
            b[i] = b[i] - lu_ddot_strided(lrow, b, i);
        }
        const int rr = rows - jj;
        if (jj > 0)
            for (int ii = 0; ii < rr; ++ii) {
                const int i = jj + ii;
                for (int k = 0; k < jj; ++k) lrow[k] = a[r0 + i][c0 + k];
                b[i] = lu_gemv_row(lrow, b, jj, b[i], ii < (rr & ~3));
            }
        int jp = jj;
        double amax = fabs(b[jj]);
        for (int i = jj + 1; i < rows; ++i)
            if (fabs(b[i]) > amax) { amax = fabs(b[i]); jp = i; }
        ipiv[c0 + jj] = r0 + jp;
        for (int i = 0; i < rows; ++i) a[r0 + i][j] = b[i];
        if (b[jp] == 0.0) return false;
        const double rcp = 1.0 / b[jp];
        if (jp != jj)
            for (int k = c0; k <= j; ++k) { double t = a[r0 + jj][k]; a[r0 + jj][k] = a[r0 + jp][k]; a[r0 + jp][k] = t; }
        for (int i = jj + 1; i < rows; ++i) a[r0 + i][j] = a[r0 + i][j] * rcp;
    }
    return true;
}

__device__ bool lu_solve_ones(const double *E, int m, double *y) {
    double a[MAXM][MAXM];
    int ipiv[MAXM];
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) a[i][j] = E[i * m + j];
    const int blocking = ((m / 2 + 1) / 2) * 2;
    if (blocking <= 4) {
        if (!lu_getf2(a, m, 0, 0, m, ipiv)) return false;
    } else {
        for (int j = 0; j < m; j += blocking) {
            const int jmin = m - j < blocking ? m - j : blocking;
            if (!lu_getf2(a, m, j, j, jmin, ipiv)) return false;
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
    return true;
}

// one thread per matrix: the normalize kernel's solve on caller matrices (temo_lu_solve_batch)
__global__ void k_lu_batch(const double *__restrict__ E, const int64_t *__restrict__ E_off,
                           const int32_t *__restrict__ ms, int64_t count, double *__restrict__ y,
                           const int64_t *__restrict__ y_off, int32_t *__restrict__ ok) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= count) return;
    const int m = ms[i];
    if (m < 1 || m > MAXM) {
        ok[i] = 0;
        return;
    }
    double yy[MAXM];
    ok[i] = lu_solve_ones(E + E_off[i], m, yy) ? 1 : 0;
    for (int k = 0; k < m; ++k) y[y_off[i] + k] = yy[k];
}

// single thread: extremes -> E -> gate -> intercepts (nsga3.py:84-93)
__global__ void k_normalize_final(const double *__restrict__ F, int m,
                                  const uint64_t *__restrict__ pkey, const int64_t *__restrict__ pidx,
                                  int nblk, const double *__restrict__ ideal,
                                  const double *__restrict__ nadir, double *__restrict__ icpt,
                                  int64_t *__restrict__ extreme_out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double E[MAXM * MAXM];
    for (int a = 0; a < m; ++a) {
        uint64_t bk = ~0ull;
        int64_t bi = INT64_MAX;
        for (int q = 0; q < nblk; ++q) {
            const uint64_t k = pkey[q * m + a];
            const int64_t i = pidx[q * m + a];
            if (k < bk || (k == bk && i < bi)) { bk = k; bi = i; }
        }
        for (int k = 0; k < m; ++k) E[a * m + k] = F[bi * m + k] - ideal[k];
        if (extreme_out) extreme_out[a] = bi;
    }
    bool ok = false;
    double sv[MAXM], y[MAXM];
    jacobi_singular_values(E, m, sv);
    double smax = 0.0, smin = INFINITY;
    bool finite = true;
    for (int k = 0; k < m; ++k) {
        finite &= isfinite(sv[k]);
        smax = sv[k] > smax ? sv[k] : smax;
        smin = sv[k] < smin ? sv[k] : smin;
    }
    if (finite) {
        const double tol = smax * (double)m * 2.220446049250313e-16;
        int rk = 0;
        for (int k = 0; k < m; ++k) rk += sv[k] > tol;
        const double cond = smin > 0.0 ? smax / smin : INFINITY;
        if (rk == m && cond <= COND_LIMIT && lu_solve_ones(E, m, y)) {
            ok = true;
            for (int k = 0; k < m; ++k) {
                const double c = 1.0 / y[k];
                ok &= c > ICPT_FLOOR;
                icpt[k] = c;
            }
        }
    }
    if (!ok)
        for (int k = 0; k < m; ++k) icpt[k] = nadir[k] > ICPT_FLOOR ? nadir[k] : ICPT_FLOOR;
}

// ---------------------------------------------------------------- associate
// direction norms in NumPy order (App. A1) and unit directions for the filter
__global__ void k_dir_prep(const double *__restrict__ W, int64_t nr, int m, double *__restrict__ nw,
                           double *__restrict__ U) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= nr) return;
    double sq[MAXM];
    for (int k = 0; k < m; ++k) sq[k] = W[j * m + k] * W[j * m + k];
    const double n = sqrt(np_sum<MAXM>(sq, m));
    nw[j] = n;
    for (int k = 0; k < m; ++k) U[j * m + k] = W[j * m + k] / n;
}

__device__ __forceinline__ double exact_D(const double *f, const double *w, int m, double nf,
                                          double nwj) {
    double dot = f[0] * w[0];
    for (int k = 1; k < m; ++k) dot = fma(f[k], w[k], dot);
    const double c = dot / (nf * nwj);
    double t = 1.0 - c * c;
    if (t < 0.0) t = 0.0;
    double d = nf * sqrt(t);
    if (isnan(d)) d = TEMO_BIG;
    return d;
}


template <int M>
__global__ void __launch_bounds__(NT) k_associate(const double *__restrict__ F, int64_t N,
                                                  const int32_t *__restrict__ rank,
                                                  const int32_t *__restrict__ lp,
                                                  const double *__restrict__ ideal,
                                                  const double *__restrict__ icpt,
                                                  const double *__restrict__ W,
                                                  const double *__restrict__ U,
                                                  const double *__restrict__ nw, int64_t nr,
                                                  int32_t *__restrict__ pi_out,
                                                  double *__restrict__ dist_out,
                                                  double *__restrict__ Fp_out) {
    constexpr int DTILE = M <= 4 ? 512 : 256;
    __shared__ double sU[DTILE * M];
    const int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x;
    const int l = *lp;
    const bool live = i < N && rank[i] <= l;
    double f[M];
    double nf = 0.0;
    if (live) {
        double sq[M];
#pragma unroll
        for (int k = 0; k < M; ++k) {
            f[k] = (F[i * M + k] - ideal[k]) / icpt[k];
            sq[k] = f[k] * f[k];
            if (Fp_out) Fp_out[i * M + k] = f[k];
        }
        nf = sqrt(np_sum<M>(sq, M));
    } else {
#pragma unroll
        for (int k = 0; k < M; ++k) f[k] = 0.0;
        if (i < N && Fp_out)
            for (int k = 0; k < M; ++k) Fp_out[i * M + k] = __longlong_as_double(0x7FF8000000000000ll);
    }
    const bool scan = live && nf > 0.0 && isfinite(nf);
    double smax = -INFINITY, thr = -INFINITY, best_d = TEMO_BIG;
    int64_t best = 0;
    for (int64_t j0 = 0; j0 < nr; j0 += DTILE) {
        const int cnt = (int)min((int64_t)DTILE, nr - j0);
        __syncthreads();
        for (int q = threadIdx.x; q < cnt * M; q += NT) sU[q] = U[j0 * M + q];
        __syncthreads();
        if (!scan) continue;
        for (int jj = 0; jj < cnt; ++jj) {
            double s = f[0] * sU[jj * M];
#pragma unroll
            for (int k = 1; k < M; ++k) s = fma(f[k], sU[jj * M + k], s);
            if (s >= thr) {
                const int64_t j = j0 + jj;
                if (s > smax) {
                    smax = s;
                    thr = s - fabs(s) * FILTER_MARGIN;
                }
                const double d = exact_D(f, W + j * M, M, nf, nw[j]);
                if (d < best_d) { best_d = d; best = j; }
            }
        }
    }
    if (scan && !(smax / nf >= FILTER_MIN_COS)) {
        // filter proof needs cos_max well above 0: evaluate every direction exactly
        best_d = TEMO_BIG;
        best = 0;
        for (int64_t j = 0; j < nr; ++j) {
            const double d = exact_D(f, W + j * M, M, nf, nw[j]);
            if (d < best_d || j == 0) { best_d = d; best = j; }
        }
    }
    if (i < N) {
        if (!live) { best = 0; best_d = __longlong_as_double(0x7FF8000000000000ll); }
        else if (!scan) { best = 0; best_d = nf == 0.0 ? 0.0 : __longlong_as_double(0x7FF8000000000000ll); }
        pi_out[i] = (int32_t)best;
        dist_out[i] = best_d;
    }
}

// ---------------------------------------------------------------- lattice association
// W = das_dennis(m, H): row j is the composition a (sum H) whose cut positions
// c_k = a_0 + ... + a_k + k enumerate itertools.combinations(range(H+m-1), m-1)
// in lexicographic order (directions.py:64-82).  For a row f >= 0 the best
// directions lie within a provable angle of f, so only the lattice points in a
// small box around the simplex projection p = f / sum(f) are candidates:
//   - chord <= arc and the projection P(v) = v / sum(v) is (1 + sqrt(m))-Lipschitz
//     on the positive-orthant unit sphere (sum(v) >= 1 there), so any direction
//     within angle theta of f has |P(w) - p|_inf <= (1 + sqrt(m)) theta;
//   - theta* = angle to the nearest-lattice candidate + 1e-6 rad covers the
//     reference's rounding plateau (|dD| <= ~1e-8 |f| near t = 1 - c^2 = 0).
// Every candidate in the box is evaluated with the exact reference expression
// and the (D, index) minimum wins -- identical to the argmin over all rows.
__device__ __forceinline__ int64_t binom64(int64_t n, int k) {
    if (k < 0 || n < k) return 0;
    int64_t r = 1;
    for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
    return r;
}

template <int M>
__device__ __forceinline__ int64_t lattice_index(const int *a, int H) {
    const int np = H + M - 1, r = M - 1;
    int64_t rank = 0;
    int prev = -1;
    for (int k = 0; k < r; ++k) {
        const int c = prev + 1 + a[k];
        const int t = r - 1 - k;
        rank += binom64(np - prev - 1, t + 1) - binom64(np - c, t + 1);
        prev = c;
    }
    return rank;
}

constexpr int LATTICE_MAX_BOX = 20000;  // beyond this a row falls back to the full scan

template <int M>
__global__ void __launch_bounds__(128) k_associate_lattice(
    const double *__restrict__ F, int64_t N, const int32_t *__restrict__ rank,
    const int32_t *__restrict__ lp, const double *__restrict__ ideal, const double *__restrict__ icpt,
    const double *__restrict__ W, const double *__restrict__ U, const double *__restrict__ nw,
    int64_t nr, int H, int32_t *__restrict__ pi_out, double *__restrict__ dist_out,
    double *__restrict__ Fp_out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int l = *lp;
    const double qnan = __longlong_as_double(0x7FF8000000000000ll);
    if (rank[i] > l) {
        if (Fp_out)
            for (int k = 0; k < M; ++k) Fp_out[i * M + k] = qnan;
        pi_out[i] = 0;
        dist_out[i] = qnan;
        return;
    }
    double f[M], sq[M];
#pragma unroll
    for (int k = 0; k < M; ++k) {
        f[k] = (F[i * M + k] - ideal[k]) / icpt[k];
        sq[k] = f[k] * f[k];
        if (Fp_out) Fp_out[i * M + k] = f[k];
    }
    const double nf = sqrt(np_sum<M>(sq, M));
    if (!(nf > 0.0) || !isfinite(nf)) {
        pi_out[i] = 0;
        dist_out[i] = nf == 0.0 ? 0.0 : qnan;
        return;
    }
    bool nonneg = true;
    double S = 0.0;
#pragma unroll
    for (int k = 0; k < M; ++k) {
        nonneg &= f[k] >= 0.0;
        S += f[k];
    }
    double best_d = TEMO_BIG;
    int64_t best = 0;
    bool done = false;
    if (nonneg && S > 0.0) {
        double p[M];
        int a[M];
        // nearest lattice point by largest remainder
        int tot = 0;
#pragma unroll
        for (int k = 0; k < M; ++k) {
            p[k] = f[k] / S;
            a[k] = (int)floor(p[k] * H);
            a[k] = a[k] < 0 ? 0 : (a[k] > H ? H : a[k]);
            tot += a[k];
        }
        for (int rem = H - tot; rem > 0; --rem) {
            int bk = 0;
            double bfrac = -1.0;
            for (int k = 0; k < M; ++k) {
                const double fr = p[k] * H - a[k];
                if (a[k] < H && fr > bfrac) { bfrac = fr; bk = k; }
            }
            a[bk] += 1;
        }
        const int64_t j0 = lattice_index<M>(a, H);
        double s0 = f[0] * U[j0 * M];
#pragma unroll
        for (int k = 1; k < M; ++k) s0 = fma(f[k], U[j0 * M + k], s0);
        double c0 = s0 / nf;
        c0 = c0 > 1.0 ? 1.0 : (c0 < -1.0 ? -1.0 : c0);
        const double theta = acos(c0) + 1e-6;
        const double R = (1.0 + sqrt((double)M)) * theta;
        int lo[M], hi[M];
        double vol = 1.0;
#pragma unroll
        for (int k = 0; k < M; ++k) {
            const double lf = floor((p[k] - R) * H), hf = ceil((p[k] + R) * H);
            lo[k] = lf < 0.0 ? 0 : (lf > H ? H : (int)lf);
            hi[k] = hf > H ? H : (hf < 0.0 ? 0 : (int)hf);
            if (k < M - 1) vol *= (double)(hi[k] - lo[k] + 1);
        }
        if (vol <= LATTICE_MAX_BOX) {
            done = true;
            // odometer over a_0..a_{M-2}; a_{M-1} = H - sum, must lie in [lo, hi]
            int c[M];
            for (int k = 0; k < M - 1; ++k) c[k] = lo[k];
            while (true) {
                int sum = 0;
                for (int k = 0; k < M - 1; ++k) sum += c[k];
                const int last = H - sum;
                if (last >= lo[M - 1] && last <= hi[M - 1]) {
                    c[M - 1] = last;
                    const int64_t j = lattice_index<M>(c, H);
                    const double d = exact_D(f, W + j * M, M, nf, nw[j]);
                    if (d < best_d || (d == best_d && j < best)) { best_d = d; best = j; }
                }
                int k = M - 2;
                while (k >= 0) {
                    if (++c[k] <= hi[k]) break;
                    c[k] = lo[k];
                    --k;
                }
                if (k < 0) break;
            }
        }
    }
    if (!done) {  // general position: exact scan of every direction
        best_d = TEMO_BIG;
        best = 0;
        for (int64_t j = 0; j < nr; ++j) {
            const double d = exact_D(f, W + j * M, M, nf, nw[j]);
            if (d < best_d || j == 0) { best_d = d; best = j; }
        }
    }
    pi_out[i] = (int32_t)best;
    dist_out[i] = best_d;
}

// ---------------------------------------------------------------- niching
__global__ void k_niche_count(const int32_t *__restrict__ rank, const int32_t *__restrict__ pi,
                              const int32_t *__restrict__ lp, int64_t N, int32_t *__restrict__ rho,
                              int32_t *__restrict__ rho_l) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int l = *lp, r = rank[i];
    if (r < l) atomicAdd(rho + pi[i], 1);
    else if (r == l && rho_l) atomicAdd(rho_l + pi[i], 1);
}

__global__ void k_claim_dist(const int32_t *__restrict__ rank, const int32_t *__restrict__ pi,
                             const double *__restrict__ dist, const int32_t *__restrict__ lp,
                             int64_t N, const int32_t *__restrict__ rho,
                             unsigned long long *__restrict__ bkey) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N || rank[i] != *lp) return;
    const int d = pi[i];
    if (rho[d] != 0) return;
    atomicMin(bkey + d, (unsigned long long)ordered_key(dist[i]));
}

__global__ void k_claim_idx(const int32_t *__restrict__ rank, const int32_t *__restrict__ pi,
                            const double *__restrict__ dist, const int32_t *__restrict__ lp,
                            int64_t N, const int32_t *__restrict__ rho,
                            const unsigned long long *__restrict__ bkey, int32_t *__restrict__ bidx) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N || rank[i] != *lp) return;
    const int d = pi[i];
    if (rho[d] != 0 || (unsigned long long)ordered_key(dist[i]) != bkey[d]) return;
    atomicMin(bidx + d, (int32_t)i);
}

__global__ void k_fill_i32(int32_t *p, int64_t n, int32_t v) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

__global__ void k_fill_u64(unsigned long long *p, int64_t n, unsigned long long v) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

__global__ void k_promote_flags(const int32_t *__restrict__ bidx, int64_t nr, int32_t *__restrict__ fl) {
    const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (d < nr) fl[d] = bidx[d] != INT32_MAX;
}

// promoted[pos[d]] = winner of direction d; ranks of winners -> l-1
__global__ void k_promote_apply(const int32_t *__restrict__ bidx, const int32_t *__restrict__ pos,
                                int64_t nr, const int32_t *__restrict__ lp, int32_t *__restrict__ rank,
                                int32_t *__restrict__ promoted) {
    const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (d >= nr) return;
    const int32_t w = bidx[d];
    if (w == INT32_MAX) return;
    promoted[pos[d]] = w;
    rank[w] = *lp - 1;
}

// scalars: [0]=n_promoted [1]=n_s (rows r<l) [2]=n_dif [3]=fill count [4]=kept
__global__ void k_count_below(const int32_t *__restrict__ rank, const int32_t *__restrict__ lp,
                              int64_t N, int32_t *__restrict__ scal) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int c = (i < N && rank[i] < *lp) ? 1 : 0;
    c = __reduce_add_sync(~0u, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(scal + 1, c);
}

__global__ void k_repair_scalars(const int32_t *__restrict__ pos, const int32_t *__restrict__ fl,
                                 int64_t nr, int64_t n, int32_t *__restrict__ scal) {
    const int n_prom = nr ? pos[nr - 1] + fl[nr - 1] : 0;
    scal[0] = n_prom;
    // n_s counted before promotions (scal[1]); n_selected = n_s + n_prom
    scal[2] = (int32_t)(n - (scal[1] + n_prom));
}

__global__ void k_fill_flags(const int32_t *__restrict__ rank, const int32_t *__restrict__ lp,
                             int64_t N, int32_t *__restrict__ fl) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < N) fl[i] = rank[i] == *lp;
}

// n_dif > 0: promote the first n_dif remaining rank-l rows by index;
// n_dif < 0: demote the last |n_dif| promotions (nsga3.py:170-183)
__global__ void k_repair_apply(const int32_t *__restrict__ fl, const int32_t *__restrict__ pos,
                               int64_t N, const int32_t *__restrict__ promoted,
                               const int32_t *__restrict__ lp, int32_t *__restrict__ rank,
                               int32_t *__restrict__ scal, int32_t *status) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int n_dif = scal[2];
    const int l = *lp;
    if (n_dif > 0) {
        const int avail = N ? pos[N - 1] + fl[N - 1] : 0;
        if (avail < n_dif) {
            if (i == 0) flag_status(status, TEMO_ST_FILL);
            return;
        }
        if (i < N && fl[i] && pos[i] < n_dif) rank[i] = l - 1;
    } else if (n_dif < 0) {
        const int np_ = scal[0];
        if (np_ < -n_dif) {
            if (i == 0) flag_status(status, TEMO_ST_DEMOTE);
            return;
        }
        if (i < -n_dif) rank[promoted[np_ + n_dif + i]] = l;
    }
}

__global__ void k_keep_flags(const int32_t *__restrict__ rank, const int32_t *__restrict__ lp,
                             int64_t N, int32_t *__restrict__ fl) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < N) fl[i] = rank[i] < *lp;
}

__global__ void k_keep_write(const int32_t *__restrict__ fl, const int32_t *__restrict__ pos,
                             int64_t N, int64_t n, int32_t *__restrict__ keep,
                             int32_t *__restrict__ scal, int32_t *status) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int kept = N ? pos[N - 1] + fl[N - 1] : 0;
    if (i == 0) {
        scal[4] = kept;
        if (kept != n) flag_status(status, TEMO_ST_COUNT);
    }
    // a failed selection (NaN objectives, peel/fill/count errors; the host raises on the
    // status word) still leaves keep a valid index set, so no consumer reads garbage rows
    if ((status && *status != 0) || kept != n) {
        if (i < n) keep[i] = (int32_t)i;
        return;
    }
    if (i < N && fl[i] && pos[i] < n) keep[pos[i]] = (int32_t)i;
}

// ---------------------------------------------------------------- host
__global__ void k_set_scalar(int32_t *p, int32_t v) { *p = v; }

__global__ void k_apply_norm(const double *__restrict__ F, int64_t N, int m,
                             const double *__restrict__ ideal, const double *__restrict__ icpt,
                             double *__restrict__ Fp) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= N * m) return;
    const int k = (int)(q % m);
    Fp[q] = (F[q] - ideal[k]) / icpt[k];
}

__global__ void k_nan_rows(const double *__restrict__ F, int64_t N, int m, int32_t *__restrict__ rank) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    int bad = 0;
    for (int k = 0; k < m; ++k) bad |= isnan(F[i * m + k]);
    rank[i] = bad;
}

// ---------------------------------------------------------------- host stages
struct SelPlan {
    int64_t N, nr;
    int m;
    uint64_t *part;
    int64_t *pidx;
    double *ideal, *nadir, *nw, *U, *zero, *one;
    int32_t *rho, *bidx, *fl_d, *pos_d, *fl, *pos, *scal, *lbuf, *rankbuf;
    unsigned long long *bkey;
    void *cub_tmp;
    size_t cub_bytes, total;
};

static void plan_sel(SelPlan &p, void *base, int64_t N, int m, int64_t nr) {
    p.N = N;
    p.m = m;
    p.nr = nr;
    size_t a = 0, b = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, a, (int32_t *)nullptr, (int32_t *)nullptr, (int)N);
    cub::DeviceScan::ExclusiveSum(nullptr, b, (int32_t *)nullptr, (int32_t *)nullptr, (int)nr);
    p.cub_bytes = a > b ? a : b;
    Carve c(base);
    p.part = c.take<uint64_t>((size_t)STAT_BLOCKS * 2 * m);
    p.pidx = c.take<int64_t>((size_t)STAT_BLOCKS * m);
    p.ideal = c.take<double>(MAXM);
    p.nadir = c.take<double>(MAXM);
    p.zero = c.take<double>(MAXM);
    p.one = c.take<double>(MAXM);
    p.nw = c.take<double>(nr);
    p.U = c.take<double>((size_t)nr * m);
    p.rho = c.take<int32_t>(nr);
    p.bidx = c.take<int32_t>(nr);
    p.bkey = c.take<unsigned long long>(nr);
    p.fl_d = c.take<int32_t>(nr);
    p.pos_d = c.take<int32_t>(nr);
    p.fl = c.take<int32_t>(N);
    p.pos = c.take<int32_t>(N);
    p.rankbuf = c.take<int32_t>(N);
    p.scal = c.take<int32_t>(8);
    p.lbuf = c.take<int32_t>(1);
    p.cub_tmp = c.take<char>(p.cub_bytes);
    p.total = c.off;
}

static inline dim3 g1(int64_t n, int t = NT) { return dim3((unsigned)((n + t - 1) / t)); }

// nsga3.py:61-93 on rows with rank <= *l
static int stage_normalize(SelPlan &p, const double *F, const int32_t *rank, const int32_t *l,
                           double *ideal, double *icpt, int64_t *extreme, cudaStream_t st) {
    const int64_t N = p.N;
    const int m = p.m;
    const int nblk = (int)std::min<int64_t>(STAT_BLOCKS, (N + NT - 1) / NT);
    k_colstats<<<nblk, NT, 0, st>>>(F, N, m, rank, l, p.part);
    k_colstats_final<<<1, 32, 0, st>>>(p.part, nblk, m, ideal, p.nadir);
    k_asf_argmin<<<nblk, NT, 0, st>>>(F, N, m, rank, l, ideal, p.part, p.pidx);
    k_normalize_final<<<1, 32, 0, st>>>(F, m, p.part, p.pidx, nblk, ideal, p.nadir, icpt, extreme);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

// nsga3.py:96-116 on (F - ideal)/icpt for rows with rank <= *l.  lattice_H > 0
// asserts W == das_dennis(m, H) in its row order: exact lattice search.
static int stage_associate(SelPlan &p, const double *F, const int32_t *rank, const int32_t *l,
                           const double *ideal, const double *icpt, const double *W, int32_t *pi,
                           double *dist, double *Fp, int lattice_H, cudaStream_t st) {
    const int64_t N = p.N, nr = p.nr;
    const int m = p.m;
    k_dir_prep<<<g1(nr), NT, 0, st>>>(W, nr, m, p.nw, p.U);
    if (lattice_H > 0 && m >= 2) {
#define ASSOCL(MM)                                                                                  \
    case MM:                                                                                        \
        k_associate_lattice<MM><<<g1(N, 128), 128, 0, st>>>(F, N, rank, l, ideal, icpt, W, p.U,    \
                                                             p.nw, nr, lattice_H, pi, dist, Fp);  \
        break;
        switch (m) {
            ASSOCL(2) ASSOCL(3) ASSOCL(4) ASSOCL(5) ASSOCL(6) ASSOCL(7) ASSOCL(8) ASSOCL(9)
            ASSOCL(10) ASSOCL(11) ASSOCL(12) ASSOCL(13) ASSOCL(14) ASSOCL(15) ASSOCL(16)
            default: return TEMO_EINVAL;
        }
#undef ASSOCL
        TEMO_LAUNCH_CHECK();
        return TEMO_OK;
    }
#define ASSOC(MM)                                                                                  \
    case MM:                                                                                       \
        k_associate<MM><<<g1(N), NT, 0, st>>>(F, N, rank, l, ideal, icpt, W, p.U, p.nw, nr, pi, \
                                              dist, Fp);                                           \
        break;
    switch (m) {
        ASSOC(1) ASSOC(2) ASSOC(3) ASSOC(4) ASSOC(5) ASSOC(6) ASSOC(7) ASSOC(8) ASSOC(9) ASSOC(10)
        ASSOC(11) ASSOC(12) ASSOC(13) ASSOC(14) ASSOC(15) ASSOC(16)
        default: return TEMO_EINVAL;
    }
#undef ASSOC
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

// nsga3.py:119-123 (+ n_s into scal[1])
static int stage_counts(SelPlan &p, const int32_t *rank, const int32_t *pi, const int32_t *l,
                        int32_t *rho, int32_t *rho_l, cudaStream_t st) {
    TEMO_CUDA(cudaMemsetAsync(rho, 0, sizeof(int32_t) * p.nr, st));
    if (rho_l) TEMO_CUDA(cudaMemsetAsync(rho_l, 0, sizeof(int32_t) * p.nr, st));
    TEMO_CUDA(cudaMemsetAsync(p.scal, 0, sizeof(int32_t) * 8, st));
    k_niche_count<<<g1(p.N), NT, 0, st>>>(rank, pi, l, p.N, rho, rho_l);
    k_count_below<<<g1(p.N), NT, 0, st>>>(rank, l, p.N, p.scal);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

// nsga3.py:126-167: one productive round (claims need rho == 0; a winner's
// direction then holds >= 1, and candidates only shrink, so a second round
// can never claim).  Promotions land in `promoted` in direction order.
static int stage_select(SelPlan &p, int32_t *rank, const int32_t *pi, const double *dist,
                        const int32_t *l, const int32_t *rho, int32_t *promoted, int64_t n,
                        cudaStream_t st) {
    size_t tb = p.cub_bytes;
    const int64_t N = p.N, nr = p.nr;
    k_fill_u64<<<g1(nr), NT, 0, st>>>(p.bkey, nr, ~0ull);
    k_fill_i32<<<g1(nr), NT, 0, st>>>(p.bidx, nr, INT32_MAX);
    k_claim_dist<<<g1(N), NT, 0, st>>>(rank, pi, dist, l, N, rho, p.bkey);
    k_claim_idx<<<g1(N), NT, 0, st>>>(rank, pi, dist, l, N, rho, p.bkey, p.bidx);
    k_promote_flags<<<g1(nr), NT, 0, st>>>(p.bidx, nr, p.fl_d);
    TEMO_CUDA(cub::DeviceScan::ExclusiveSum(p.cub_tmp, tb, p.fl_d, p.pos_d, (int)nr, st));
    k_promote_apply<<<g1(nr), NT, 0, st>>>(p.bidx, p.pos_d, nr, l, rank, promoted);
    k_repair_scalars<<<1, 1, 0, st>>>(p.pos_d, p.fl_d, nr, n, p.scal);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

// nsga3.py:170-183 with n_dif in scal[2] and n_promoted in scal[0]
static int stage_repair(SelPlan &p, int32_t *rank, const int32_t *l, const int32_t *promoted,
                        int32_t *status, cudaStream_t st) {
    size_t tb = p.cub_bytes;
    const int64_t N = p.N, nr = p.nr;
    k_fill_flags<<<g1(N), NT, 0, st>>>(rank, l, N, p.fl);
    TEMO_CUDA(cub::DeviceScan::ExclusiveSum(p.cub_tmp, tb, p.fl, p.pos, (int)N, st));
    k_repair_apply<<<g1(N > nr ? N : nr), NT, 0, st>>>(p.fl, p.pos, N, promoted, l, rank, p.scal, status);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

// nsga3.py:214-217
static int stage_keep(SelPlan &p, const int32_t *rank, const int32_t *l, int64_t n, int32_t *keep,
                      int32_t *status, cudaStream_t st) {
    size_t tb = p.cub_bytes;
    const int64_t N = p.N;
    k_keep_flags<<<g1(N), NT, 0, st>>>(rank, l, N, p.fl);
    TEMO_CUDA(cub::DeviceScan::ExclusiveSum(p.cub_tmp, tb, p.fl, p.pos, (int)N, st));
    k_keep_write<<<g1(N), NT, 0, st>>>(p.fl, p.pos, N, n, keep, p.scal, status);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

#define PLAN_OR_FAIL(p, N, m, nr)                        \
    SelPlan p;                                           \
    plan_sel(p, nullptr, N, m, nr);                      \
    if (!ws || ws_bytes < p.total) return TEMO_EWORKSPACE; \
    plan_sel(p, ws, N, m, nr);

}  // namespace temo

using namespace temo;

extern "C" size_t temo_nsga3_select_ws_bytes(int64_t N, int m, int64_t nr) {
    SelPlan p;
    plan_sel(p, nullptr, N, m, nr > 0 ? nr : 1);
    return p.total;
}

extern "C" int temo_nsga3_select(const double *Fs, int64_t N, int m, const double *W, int64_t nr,
                                 int32_t lattice_H, int64_t n, int32_t *rank, const int32_t *l, int32_t *keep,
                                 int32_t *pi, double *dist, double *Fp, double *ideal_out,
                                 double *icpt, int64_t *extreme, int32_t *rho_out,
                                 int32_t *rho_l_out, int32_t *promoted, int32_t *counts,
                                 int32_t *status, void *ws, size_t ws_bytes, temo_stream_t stream) {
    if (N < 1 || m < 1 || m > MAXM || nr < 1 || n < 1 || n > N) return TEMO_EINVAL;
    if (!Fs || !W || !rank || !l || !keep || !pi || !dist || !icpt || !promoted) return TEMO_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    PLAN_OR_FAIL(p, N, m, nr);
    double *ideal = ideal_out ? ideal_out : p.ideal;
    int32_t *rho = rho_out ? rho_out : p.rho;
    int rc;
    stage_begin(S_NORMALIZE, st);
    if ((rc = stage_normalize(p, Fs, rank, l, ideal, icpt, extreme, st))) return rc;
    stage_end(S_NORMALIZE, st);
    stage_begin(S_ASSOCIATE, st);
    if ((rc = stage_associate(p, Fs, rank, l, ideal, icpt, W, pi, dist, Fp, lattice_H, st))) return rc;
    stage_end(S_ASSOCIATE, st);
    stage_begin(S_NICHE, st);
    if ((rc = stage_counts(p, rank, pi, l, rho, rho_l_out, st))) return rc;
    if ((rc = stage_select(p, rank, pi, dist, l, rho, promoted, n, st))) return rc;
    if ((rc = stage_repair(p, rank, l, promoted, status, st))) return rc;
    if ((rc = stage_keep(p, rank, l, n, keep, status, st))) return rc;
    if (counts) TEMO_CUDA(cudaMemcpyAsync(counts, p.scal, sizeof(int32_t) * 8, cudaMemcpyDeviceToDevice, st));
    stage_end(S_NICHE, st);
    return TEMO_OK;
}

// nsga3.normalize(F) (nsga3.py:61-93): rows containing NaN are excluded rows;
// NaN entries are skipped by the column statistics (np.nanmin / np.nanmax).
extern "C" int temo_nsga3_normalize(const double *F, int64_t N, int m, double *Fp, double *ideal,
                                    double *icpt, int64_t *extreme, void *ws, size_t ws_bytes,
                                    temo_stream_t stream) {
    if (N < 1 || m < 1 || m > MAXM || !F || !Fp || !ideal || !icpt) return TEMO_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    PLAN_OR_FAIL(p, N, m, 1);
    k_set_scalar<<<1, 1, 0, st>>>(p.lbuf, 0);
    k_fill_i32<<<g1(N), NT, 0, st>>>(p.rankbuf, N, 0);  // every row takes part in the stats
    int rc = stage_normalize(p, F, p.rankbuf, p.lbuf, ideal, icpt, extreme, st);
    if (rc) return rc;
    // Fp = shifted / intercepts for all rows (NaN rows stay NaN)
    k_apply_norm<<<g1(N * m), NT, 0, st>>>(F, N, m, ideal, icpt, Fp);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

// nsga3.associate(Fp, R) (nsga3.py:96-116) on a given Fp (rows with NaN -> pi 0, dist NaN)
extern "C" int temo_associate(const double *Fp, int64_t N, int m, const double *W, int64_t nr,
                              int32_t lattice_H, int32_t *pi, double *dist, void *ws, size_t ws_bytes,
                              temo_stream_t stream) {
    if (N < 1 || m < 1 || m > MAXM || nr < 1 || !Fp || !W || !pi || !dist) return TEMO_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    PLAN_OR_FAIL(p, N, m, nr);
    k_nan_rows<<<g1(N), NT, 0, st>>>(Fp, N, m, p.rankbuf);
    k_set_scalar<<<1, 1, 0, st>>>(p.lbuf, 0);
    TEMO_CUDA(cudaMemsetAsync(p.zero, 0, sizeof(double) * MAXM, st));
    k_fill_u64<<<1, MAXM, 0, st>>>((unsigned long long *)p.one, MAXM, 0x3FF0000000000000ull);
    return stage_associate(p, Fp, p.rankbuf, p.lbuf, p.zero, p.one, W, pi, dist, nullptr, lattice_H, st);
}

// nsga3.niche_counts (nsga3.py:119-123); l is a host value
extern "C" int temo_niche_counts(const int32_t *rank, const int32_t *pi, int64_t N, int32_t l,
                                 int64_t nr, int32_t *rho, int32_t *rho_l, void *ws, size_t ws_bytes,
                                 temo_stream_t stream) {
    if (N < 1 || nr < 1 || !rank || !pi || !rho) return TEMO_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    PLAN_OR_FAIL(p, N, 1, nr);
    k_set_scalar<<<1, 1, 0, st>>>(p.lbuf, l);
    return stage_counts(p, rank, pi, p.lbuf, rho, rho_l, st);
}

// nsga3.niche_select (nsga3.py:126-167): rank updated in place; counts[0] =
// number promoted (promoted[0..counts[0]) in direction order)
extern "C" int temo_niche_select(int32_t *rank, const int32_t *pi, const double *dist, int64_t N,
                                 int32_t l, const int32_t *rho, int64_t nr, int32_t *promoted,
                                 int32_t *counts, void *ws, size_t ws_bytes, temo_stream_t stream) {
    if (N < 1 || nr < 1 || !rank || !pi || !dist || !rho || !promoted || !counts) return TEMO_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    PLAN_OR_FAIL(p, N, 1, nr);
    k_set_scalar<<<1, 1, 0, st>>>(p.lbuf, l);
    TEMO_CUDA(cudaMemsetAsync(p.scal, 0, sizeof(int32_t) * 8, st));
    int rc = stage_select(p, rank, pi, dist, p.lbuf, rho, promoted, N, st);
    if (rc) return rc;
    TEMO_CUDA(cudaMemcpyAsync(counts, p.scal, sizeof(int32_t) * 8, cudaMemcpyDeviceToDevice, st));
    return TEMO_OK;
}

// nsga3.update_rank (nsga3.py:170-183): rank updated in place
extern "C" int temo_update_rank(int32_t *rank, int64_t N, const int32_t *promoted, int64_t n_promoted,
                                int64_t n_dif, int32_t l, int32_t *status, void *ws, size_t ws_bytes,
                                temo_stream_t stream) {
    if (N < 1 || !rank) return TEMO_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    PLAN_OR_FAIL(p, N, 1, 1);
    k_set_scalar<<<1, 1, 0, st>>>(p.lbuf, l);
    k_set_scalar<<<1, 1, 0, st>>>(p.scal + 0, (int32_t)n_promoted);
    k_set_scalar<<<1, 1, 0, st>>>(p.scal + 2, (int32_t)n_dif);
    return stage_repair(p, rank, p.lbuf, promoted, status, st);
}

extern "C" int temo_gather_rows(const double *src, const int32_t *idx32, const int64_t *idx64,
                                int64_t rows, int64_t cols, double *dst, temo_stream_t stream) {
    if (rows < 0 || cols < 1 || (!idx32 && !idx64)) return TEMO_EINVAL;
    if (rows == 0) return TEMO_OK;
    cudaStream_t st = (cudaStream_t)stream;
    k_gather_rows<<<g1(rows * 32), NT, 0, st>>>(src, idx32, idx64, rows, cols, dst);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

// ---------------------------------------------------------------- row pool
__global__ void k_pool_survivors(const int64_t *__restrict__ phys, const int64_t *__restrict__ perm,
                                 const int32_t *__restrict__ keep, int64_t n, int64_t *__restrict__ out,
                                 int32_t *__restrict__ kept, const int32_t *__restrict__ status) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    // failed selection (status set): keep the pool as it is (phys' = phys)
    const int64_t r = (status && *status) ? p : perm ? perm[keep[p]] : (int64_t)keep[p];
    out[p] = phys[r];
    kept[r] = 1;
}

__global__ void k_pool_free_flags(const int32_t *__restrict__ kept, int64_t N, int32_t *__restrict__ fr) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r < N) fr[r] = 1 - kept[r];
}

__global__ void k_pool_free(const int64_t *__restrict__ phys, const int32_t *__restrict__ kept,
                            const int32_t *__restrict__ pos, int64_t N, int64_t n, int64_t *__restrict__ out) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r < N && !kept[r]) out[n + pos[r]] = phys[r];
}

extern "C" size_t temo_pool_update_ws_bytes(int64_t N) {
    if (N < 1) return 0;
    size_t c = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, c, (int32_t *)nullptr, (int32_t *)nullptr, (int)N);
    return 3 * ((size_t)N * 4 + 256) + c + 256;
}

extern "C" int temo_pool_update(const int64_t *phys, const int64_t *perm, const int32_t *keep, int64_t N,
                                int64_t n, int64_t *phys_out, const int32_t *status, void *ws,
                                size_t ws_bytes, temo_stream_t stream) {
    if (N < 1 || n < 0 || n > N || !phys || !keep || !phys_out || phys_out == phys) return TEMO_EINVAL;
    if (!ws || ws_bytes < temo_pool_update_ws_bytes(N)) return TEMO_EWORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    Carve c(ws);
    int32_t *kept = c.take<int32_t>(N), *fr = c.take<int32_t>(N), *pos = c.take<int32_t>(N);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, fr, pos, (int)N);
    void *tmp = c.take<char>(tb);
    TEMO_CUDA(cudaMemsetAsync(kept, 0, sizeof(int32_t) * N, st));
    if (n) k_pool_survivors<<<g1(n), NT, 0, st>>>(phys, perm, keep, n, phys_out, kept, status);
    k_pool_free_flags<<<g1(N), NT, 0, st>>>(kept, N, fr);
    TEMO_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, fr, pos, (int)N, st));
    k_pool_free<<<g1(N), NT, 0, st>>>(phys, kept, pos, N, n, phys_out);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

extern "C" int temo_gather_rows2(const double *src, const int64_t *idx_a, const int32_t *idx_b,
                                 int64_t rows, int64_t cols, double *dst, temo_stream_t stream) {
    if (rows < 0 || cols < 1 || !idx_a || !idx_b) return TEMO_EINVAL;
    if (rows == 0) return TEMO_OK;
    cudaStream_t st = (cudaStream_t)stream;
    k_gather_rows2<<<g1(rows * 32), NT, 0, st>>>(src, idx_a, idx_b, rows, cols, dst);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

extern "C" int temo_lu_solve_batch(const double *E, const int64_t *E_off, const int32_t *m, int64_t count,
                                   double *y, const int64_t *y_off, int32_t *ok, temo_stream_t stream) {
    if (count < 0 || (count && (!E || !E_off || !m || !y || !y_off || !ok))) return TEMO_EINVAL;
    if (!count) return TEMO_OK;
    k_lu_batch<<<(unsigned)((count + 127) / 128), 128, 0, (cudaStream_t)stream>>>(E, E_off, m, count, y, y_off, ok);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}
