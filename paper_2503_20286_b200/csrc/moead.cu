// Decoupled MOEA/D generation on B200 (replaces temo moead.py:43-158).
//
//   offspring   moead.py:127-145  k_offspring in single-child mode (variation.cu)
//   compare     moead.py:70-92    one thread per (i, t): g_old / g_new with the
//                                 reference's exact PBI op order (App. A4b) or
//                                 Tchebycheff (new); improves = g_old - g_new >= 0
//   elite       moead.py:95-124   O(n T) instead of the reference's O(n^2):
//                                 per direction j, over the reverse-CSR list
//                                 C_j = {i : j in I_nb[i], improves}, the
//                                 argmin-first-index rule of SURVEY App. A5
//   gather      moead.py:121-123  winners' rows, z <- z_min
#include "common.cuh"

namespace temo {

constexpr int MT = 256;

// PBI (moead.py:43-67): NumPy op order, sums over m sequential (m < 8) / pairwise
__device__ __forceinline__ double pbi_eval(const double *f, const double *w, const double *z, int m,
                                           double theta, bool normalize) {
    double ww[16], vw[16], v[16];
    for (int k = 0; k < m; ++k) {
        v[k] = f[k] - z[k];
        ww[k] = w[k] * w[k];
        vw[k] = v[k] * w[k];
    }
    const double wn = sqrt(np_sum<16>(ww, m));
    const double d1 = fabs(np_sum<16>(vw, m)) / wn;
    double rr[16];
    for (int k = 0; k < m; ++k) {
        const double dir = normalize ? w[k] / wn : w[k];
        const double r = v[k] - d1 * dir;
        rr[k] = r * r;
    }
    const double d2 = sqrt(np_sum<16>(rr, m));
    return d1 + theta * d2;
}

// Tchebycheff g(f|w,z) = max_k w_k |f_k - z_k| (Zhang & Li 2007; no reference, self-oracle)
__device__ __forceinline__ double tch_eval(const double *f, const double *w, const double *z, int m) {
    double best = -INFINITY;
    bool nan = false;
    for (int k = 0; k < m; ++k) {
        const double v = w[k] * fabs(f[k] - z[k]);
        if (isnan(v)) nan = true;
        else if (v > best) best = v;
    }
    return nan ? __longlong_as_double(0x7FF8000000000000ll) : best;
}

__device__ __forceinline__ double agg_eval(int kind, const double *f, const double *w, const double *z,
                                           int m, double theta) {
    return kind == TEMO_AGG_TCH ? tch_eval(f, w, z, m) : pbi_eval(f, w, z, m, theta, true);
}

// z_min = minimum(z, F2.min(0))  (moead.py:81)
__global__ void k_zmin(const double *__restrict__ F2, int64_t n, int m, const double *__restrict__ z,
                       double *__restrict__ zmin) {
    __shared__ double sred[32];
    const int k = blockIdx.x;
    double a = INFINITY;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double v = F2[i * m + k];
        a = v < a ? v : a;
    }
    for (int d = 16; d; d >>= 1) {
        const double b = __shfl_xor_sync(~0u, a, d);
        a = b < a ? b : a;
    }
    if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) a = sred[w] < a ? sred[w] : a;
        // np.minimum(z, mins)
        zmin[k] = (z[k] < a || isnan(z[k])) ? z[k] : a;
    }
}

// per (i, t): g_old(I_nb[i,t]), g_new(i, I_nb[i,t]), improves
__global__ void k_moead_compare(const double *__restrict__ F1, const double *__restrict__ F2,
                                const double *__restrict__ W, const int32_t *__restrict__ I_nb, int64_t n,
                                int T, int m, const double *__restrict__ zmin, double theta, int kind,
                                double *__restrict__ g_new, uint8_t *__restrict__ improves) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= n * T) return;
    const int64_t i = q / T;
    const int64_t j = I_nb[q];
    double z[16];
    for (int k = 0; k < m; ++k) z[k] = zmin[k];
    const double go = agg_eval(kind, F1 + j * m, W + j * m, z, m, theta);
    const double gn = agg_eval(kind, F2 + i * m, W + j * m, z, m, theta);
    g_new[q] = gn;
    improves[q] = (go - gn) >= 0.0;
}

// per direction j: App. A5 rule over the reverse CSR (entries q = i*T + t, ascending i).
// The reference's column argmin (moead.py:118-121) picks the first index among
// {g_new(i,j) : i in C_j} U {g_old(j) : i not in C_j}; with (g*, i*) the
// (value, index) minimum over C_j and i0 the smallest index outside C_j, the
// winner is offspring i* iff g* < g_old(j), or g* == g_old(j) and i* < i0.
__global__ void k_moead_elite(const double *__restrict__ F1, const double *__restrict__ W, int64_t n,
                              int T, int m, const double *__restrict__ zmin, double theta, int kind,
                              const int64_t *__restrict__ rptr, const int32_t *__restrict__ rcol,
                              const double *__restrict__ g_new, const uint8_t *__restrict__ improves,
                              int32_t *__restrict__ winner) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= n) return;
    double z[16];
    for (int k = 0; k < m; ++k) z[k] = zmin[k];
    const double go = agg_eval(kind, F1 + j * m, W + j * m, z, m, theta);
    double gbest = 0.0;
    int64_t ibest = -1, i0 = 0;
    for (int64_t e = rptr[j]; e < rptr[j + 1]; ++e) {
        const int32_t q = rcol[e];
        if (!improves[q]) continue;
        const int64_t i = q / T;
        if (i == i0) ++i0;
        const double gn = g_new[q];
        if (ibest < 0 || gn < gbest) { gbest = gn; ibest = i; }
    }
    int32_t win = -1;
    if (ibest >= 0 && (gbest < go || (gbest == go && ibest < i0))) win = (int32_t)ibest;
    winner[j] = win;
}

__global__ void k_moead_gather(const double *__restrict__ X, const double *__restrict__ F1,
                               const double *__restrict__ O, const double *__restrict__ F2,
                               const int32_t *__restrict__ winner, int64_t n, int64_t d, int m,
                               double *__restrict__ Xn, double *__restrict__ Fn) {
    const int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (j >= n) return;
    const int32_t w = winner[j];
    const double *xs = w >= 0 ? O + (int64_t)w * d : X + j * d;
    const double *fs = w >= 0 ? F2 + (int64_t)w * m : F1 + j * m;
    for (int64_t c = lane; c < d; c += 32) Xn[j * d + c] = xs[c];
    if (lane < m) Fn[j * m + lane] = fs[lane];
}

// pbi / tchebycheff on row-aligned operands (API-level moead.pbi)
__global__ void k_agg_rows(const double *__restrict__ f, const double *__restrict__ w,
                           const double *__restrict__ z, int64_t rows, int m, double theta, int kind,
                           int normalize, double *__restrict__ out) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= rows) return;
    out[r] = kind == TEMO_AGG_TCH ? tch_eval(f + r * m, w + r * m, z + r * m, m)
                                  : pbi_eval(f + r * m, w + r * m, z + r * m, m, theta, normalize != 0);
}

static inline dim3 mg(int64_t n, int t = MT) { return dim3((unsigned)((n + t - 1) / t)); }

}  // namespace temo

using namespace temo;

extern "C" int temo_moead_compare(const double *F1, const double *F2, const double *W,
                                  const int32_t *I_nb, int64_t n, int T, int m, const double *z,
                                  double theta, int kind, double *zmin, double *g_new,
                                  uint8_t *improves, temo_stream_t stream) {
    if (!F1 || !F2 || !W || !I_nb || n < 1 || T < 1 || m < 1 || m > 16 || !z || !zmin || !g_new ||
        !improves)
        return TEMO_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    k_zmin<<<m, 256, 0, st>>>(F2, n, m, z, zmin);
    k_moead_compare<<<mg(n * T), MT, 0, st>>>(F1, F2, W, I_nb, n, T, m, zmin, theta, kind, g_new, improves);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

extern "C" int temo_moead_elite(const double *X, const double *F1, const double *W, const double *O,
                                const double *F2, int64_t n, int64_t d, int T, int m,
                                const double *zmin, double theta, int kind, const int64_t *rptr,
                                const int32_t *rcol, const double *g_new, const uint8_t *improves,
                                int32_t *winner, double *Xn, double *Fn, temo_stream_t stream) {
    if (!X || !F1 || !W || !O || !F2 || n < 1 || d < 1 || T < 1 || m < 1 || m > 16 || !zmin || !rptr ||
        !rcol || !g_new || !improves || !winner || !Xn || !Fn)
        return TEMO_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    k_moead_elite<<<mg(n), MT, 0, st>>>(F1, W, n, T, m, zmin, theta, kind, rptr, rcol, g_new, improves,
                                         winner);
    k_moead_gather<<<mg(n * 32), MT, 0, st>>>(X, F1, O, F2, winner, n, d, m, Xn, Fn);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

extern "C" int temo_aggregate_rows(const double *f, const double *w, const double *z, int64_t rows, int m,
                                   double theta, int kind, int normalize, double *out,
                                   temo_stream_t stream) {
    if (!f || !w || !z || rows < 0 || m < 1 || m > 16 || !out) return TEMO_EINVAL;
    if (rows == 0) return TEMO_OK;
    k_agg_rows<<<mg(rows), MT, 0, (cudaStream_t)stream>>>(f, w, z, rows, m, theta, kind, normalize, out);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}
