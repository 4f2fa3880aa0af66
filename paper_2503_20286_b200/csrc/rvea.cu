// RVEA angle-penalized-distance environmental selection on B200 (replaces temo
// rvea.py:33-68, Alg. S.11 of the paper).
//
//   prep (once per direction set): Vn = W / ||W|| (NumPy's last-axis sum order, App. A1);
//     gamma_j = min over k != j of arccos(clip(Vn_j . Vn_k)) (pi/2 when r = 1).
//   select: Fp = F - min(F, axis 0); norms = ||Fp||; per row i the direction with the
//     smallest angle theta_ij = arccos(clip(Fp_i . Vn_j / norms_i)) (dot as the dgemm FMA
//     chain, App. A2; norms 0 -> cos 0; first index on ties); APD_i = (1 + m p theta / gamma)
//     norms_i with p = (t / t_max)^alpha computed by the host exactly as Python does; per
//     direction the member with the smallest (APD, index) wins (one atomicMin on a packed
//     key); winners are emitted in direction order (np.lexsort((idx, apd, part)) + first).
// Angles use CUDA's acos (NumPy's arccos may differ in the last ulp, like the pow of the
// variation operators); partitions are argmin over those angles.
#include <cub/cub.cuh>

#include "common.cuh"

namespace temo {

constexpr int RV_MAXM = 16;
constexpr int32_t RV_NONE = 0x7F7F7F7F;  // empty partition (memset 0x7F bytes; > any row index)

__global__ void k_rv_unit(const double *__restrict__ W, int64_t r, int m, double *__restrict__ Vn) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= r) return;
    double sq[RV_MAXM];
    for (int k = 0; k < m; ++k) sq[k] = W[j * m + k] * W[j * m + k];
    const double nw = sqrt(np_sum<RV_MAXM>(sq, m));
    for (int k = 0; k < m; ++k) Vn[j * m + k] = W[j * m + k] / nw;
}

// warp per direction j: gamma_j = min_k!=j arccos(clip(Vn_j . Vn_k, -1, 1))
__global__ void k_rv_gamma(const double *__restrict__ Vn, int64_t r, int m, double *__restrict__ gamma) {
    const int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (j >= r) return;
    const double PI = 3.141592653589793;
    double best = INFINITY;
    for (int64_t k = lane; k < r; k += 32) {
        double a;
        if (k == j) {
            a = PI;  // np.fill_diagonal(vv, pi)
        } else {
            double dot = Vn[j * m] * Vn[k * m];
            for (int q = 1; q < m; ++q) dot = fma(Vn[j * m + q], Vn[k * m + q], dot);
            dot = dot < -1.0 ? -1.0 : (dot > 1.0 ? 1.0 : dot);
            a = acos(dot);
        }
        best = a < best ? a : best;
    }
    for (int o = 16; o; o >>= 1) {
        const double y = __shfl_xor_sync(~0u, best, o);
        best = y < best ? y : best;
    }
    if (lane == 0) gamma[j] = r == 1 ? PI / 2.0 : best;
}

// column minima of F (N rows): block partials then a final reduce
__global__ void k_rv_colmin(const double *__restrict__ F, int64_t N, int m, double *__restrict__ part) {
    __shared__ double s[256];
    for (int k = 0; k < m; ++k) {
        double v = INFINITY;
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
            const double x = F[i * m + k];
            v = (x < v || isnan(x)) ? x : v;
        }
        s[threadIdx.x] = v;
        __syncthreads();
        for (int o = blockDim.x / 2; o; o >>= 1) {
            if (threadIdx.x < o) {
                const double y = s[threadIdx.x + o];
                if (y < s[threadIdx.x] || isnan(y)) s[threadIdx.x] = y;
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) part[blockIdx.x * m + k] = s[0];
        __syncthreads();
    }
}

__global__ void k_rv_colmin_final(const double *__restrict__ part, int nb, int m, double *__restrict__ mn) {
    const int k = threadIdx.x;
    if (k >= m) return;
    double v = INFINITY;
    for (int b = 0; b < nb; ++b) {
        const double x = part[b * m + k];
        v = (x < v || isnan(x)) ? x : v;
    }
    mn[k] = v;
}

// APD >= 0 (NaN last), so its bit pattern orders as an unsigned integer; ties are broken by
// the row index in a second pass (k_rv_tie)
__device__ __forceinline__ uint64_t rv_key(double apd, int64_t i) {
    (void)i;
    return (uint64_t)__double_as_longlong(apd == 0.0 ? 0.0 : apd);
}

// warp per row i: partition (first argmin angle), theta, APD; atomicMin of the APD bits per direction
__global__ void k_rv_rows(const double *__restrict__ F, int64_t N, int m, const double *__restrict__ mn,
                          const double *__restrict__ Vn, int64_t r, const double *__restrict__ gamma, double mp,
                          int32_t *__restrict__ part_out, double *__restrict__ apd_out,
                          unsigned long long *__restrict__ best_apd) {
    const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= N) return;
    double fp[RV_MAXM], sq[RV_MAXM];
    for (int k = 0; k < m; ++k) {
        fp[k] = F[i * m + k] - mn[k];
        sq[k] = fp[k] * fp[k];
    }
    const double nrm = sqrt(np_sum<RV_MAXM>(sq, m));
    double best = INFINITY;
    int64_t bj = 0;
    for (int64_t j = lane; j < r; j += 32) {
        double c;
        if (nrm == 0.0) {
            c = 0.0;  // cos[norms == 0] = 0
        } else {
            double dot = fp[0] * Vn[j * m];
            for (int k = 1; k < m; ++k) dot = fma(fp[k], Vn[j * m + k], dot);
            c = dot / nrm;
        }
        c = c < -1.0 ? -1.0 : (c > 1.0 ? 1.0 : c);  // np.clip (NaN passes)
        const double th = acos(c);
        if (th < best || (isnan(th) && !isnan(best))) {  // np.argmin: first minimum, NaN wins
            best = th;
            bj = j;
        }
    }
    for (int o = 16; o; o >>= 1) {  // first index among equal minima
        const double yb = __shfl_xor_sync(~0u, best, o);
        const int64_t yj = __shfl_xor_sync(~0u, bj, o);
        const bool take = (yb < best) || (yb == best && yj < bj) || (isnan(yb) && (!isnan(best) || yj < bj));
        if (take) {
            best = yb;
            bj = yj;
        }
    }
    if (lane != 0) return;
    const double penalty = 1.0 + mp * best / gamma[bj];
    const double apd = penalty * nrm;
    part_out[i] = (int32_t)bj;
    apd_out[i] = apd;
    atomicMin(best_apd + bj, (unsigned long long)rv_key(apd, i));
}

// second pass: smallest index among the partition's members at its minimal APD
__global__ void k_rv_tie(const int32_t *__restrict__ part, const double *__restrict__ apd, int64_t N,
                         const unsigned long long *__restrict__ best_apd, int32_t *__restrict__ win) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int32_t j = part[i];
    if ((unsigned long long)rv_key(apd[i], i) == best_apd[j]) atomicMin(win + j, (int32_t)i);
}

__global__ void k_rv_flags(const int32_t *__restrict__ win, int64_t r, int32_t *__restrict__ flag) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j < r) flag[j] = win[j] != RV_NONE;
}

__global__ void k_rv_keep(const int32_t *__restrict__ win, const int32_t *__restrict__ flag,
                          const int32_t *__restrict__ pos, int64_t r, int32_t *__restrict__ keep,
                          int32_t *__restrict__ count) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= r) return;
    if (flag[j]) keep[pos[j]] = win[j];
    if (j == r - 1) *count = pos[j] + flag[j];
}

static inline unsigned g1(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

}  // namespace temo

using namespace temo;

extern "C" int temo_rvea_prep(const double *W, int64_t r, int m, double *Vn, double *gamma, temo_stream_t stream) {
    if (r < 1 || m < 1 || m > RV_MAXM || !W || !Vn || !gamma) return TEMO_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    k_rv_unit<<<g1(r), 256, 0, st>>>(W, r, m, Vn);
    k_rv_gamma<<<g1(r * 32), 256, 0, st>>>(Vn, r, m, gamma);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

struct RvPlan {
    double *colpart, *mn, *apd;
    int32_t *part, *win, *flag, *pos;
    unsigned long long *best;
    void *cub;
    size_t cub_bytes, total;
};

static void plan_rv(RvPlan &p, void *base, int64_t N, int m, int64_t r) {
    size_t c = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, c, (int32_t *)nullptr, (int32_t *)nullptr, (int)r);
    p.cub_bytes = c;
    Carve cv(base);
    p.colpart = cv.take<double>((size_t)148 * 4 * m);
    p.mn = cv.take<double>(m);
    p.apd = cv.take<double>(N);
    p.part = cv.take<int32_t>(N);
    p.win = cv.take<int32_t>(r);
    p.flag = cv.take<int32_t>(r);
    p.pos = cv.take<int32_t>(r);
    p.best = cv.take<unsigned long long>(r);
    p.cub = cv.take<char>(c);
    p.total = cv.off;
}

extern "C" size_t temo_rvea_select_ws_bytes(int64_t N, int m, int64_t r) {
    if (N < 1 || r < 1 || m < 1) return 0;
    RvPlan p;
    plan_rv(p, nullptr, N, m, r);
    return p.total;
}

// apd_select (rvea.py:33-68) on F (N x m) with prepared directions; keep receives the winners
// (direction order, at most r), count the number of winners (device scalar).  mp = m * (t /
// t_max)^alpha, computed by the caller.
extern "C" int temo_rvea_select(const double *F, int64_t N, int m, const double *Vn, const double *gamma,
                                int64_t r, double mp, int32_t *keep, int32_t *count, int32_t *part_out,
                                double *apd_out, void *ws, size_t ws_bytes, temo_stream_t stream) {
    if (N < 1 || r < 1 || m < 1 || m > RV_MAXM || !F || !Vn || !gamma || !keep || !count) return TEMO_EINVAL;
    RvPlan p;
    plan_rv(p, nullptr, N, m, r);
    if (!ws || ws_bytes < p.total) return TEMO_EWORKSPACE;
    plan_rv(p, ws, N, m, r);
    cudaStream_t st = (cudaStream_t)stream;
    const int nb = (int)((N + 255) / 256 < 148 * 4 ? (N + 255) / 256 : 148 * 4);
    k_rv_colmin<<<nb, 256, 0, st>>>(F, N, m, p.colpart);
    k_rv_colmin_final<<<1, 32, 0, st>>>(p.colpart, nb, m, p.mn);
    TEMO_CUDA(cudaMemsetAsync(p.best, 0xFF, sizeof(unsigned long long) * r, st));
    TEMO_CUDA(cudaMemsetAsync(p.win, 0x7F, sizeof(int32_t) * r, st));  // RV_NONE
    k_rv_rows<<<g1(N * 32), 256, 0, st>>>(F, N, m, p.mn, Vn, r, gamma, mp, p.part, p.apd, p.best);
    k_rv_tie<<<g1(N), 256, 0, st>>>(p.part, p.apd, N, p.best, p.win);
    k_rv_flags<<<g1(r), 256, 0, st>>>(p.win, r, p.flag);
    size_t tb = p.cub_bytes;
    TEMO_CUDA(cub::DeviceScan::ExclusiveSum(p.cub, tb, p.flag, p.pos, (int)r, st));
    k_rv_keep<<<g1(r), 256, 0, st>>>(p.win, p.flag, p.pos, r, keep, count);
    if (part_out) TEMO_CUDA(cudaMemcpyAsync(part_out, p.part, sizeof(int32_t) * N, cudaMemcpyDeviceToDevice, st));
    if (apd_out) TEMO_CUDA(cudaMemcpyAsync(apd_out, p.apd, sizeof(double) * N, cudaMemcpyDeviceToDevice, st));
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}
