// Quality indicators on the device (replaces temo indicators.py:19-100, the per-generation
// metrics of harness.py:250-268).
//
//   temo_igd   igd (indicators.py:19-26): for every reference-front point the nearest
//              solution's distance sqrt(sum(diff^2)) (NumPy's last-axis sum order, App. A1),
//              then np.mean over the reference points (NumPy's pairwise summation).
//   temo_hv    hv_indicator for m = 2, 3 (indicators.py:29-66): rows at or beyond the
//              reference dropped (order kept); m = 2 one x/y sweep, m = 3 one 2-D sweep per
//              z slab (indicators.py:40-47): slabs run in parallel (thread per slab over
//              the kept rows pre-sorted by (x, y)), the slab terms are summed with NumPy's
//              pairwise order and the slab volumes accumulated in slab order -- the
//              reference's bits.  m > 3: the Monte-Carlo estimate over caller samples.
//   temo_eu    eu (indicators.py:69-100): per weight row the best weighted utility (dot
//              products in OpenBLAS's dgemm FMA order, App. A2), mean over the rows.
#include <cub/cub.cuh>

#include "common.cuh"

namespace temo {

constexpr int IND_MAXM = 16;

// NumPy's pairwise summation of a contiguous double array (loops_utils.h pairwise_sum:
// < 8 terms sequential from 0.0, <= 128 terms eight strided accumulators combined pairwise
// then the tail, above that halves split at a multiple of 8) -- the reduction np.sum and
// np.mean apply to a 1-D array (checked against NumPy on 2,000 random lengths).
__device__ double np_pairwise_sum(const double *a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; ++i) res = res + a[i];
        return res;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] = r[j] + a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res = res + a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
}

// ---------------------------------------------------------------- igd
// warp per reference point: min over solutions of the Euclidean distance
__global__ void k_igd_min(const double *__restrict__ F, int64_t n, int m, const double *__restrict__ Fs,
                          int64_t r, double *__restrict__ dmin) {
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= r) return;
    const double *z = Fs + w * m;
    double best = INFINITY;
    for (int64_t j = lane; j < n; j += 32) {
        double sq[IND_MAXM];
        for (int k = 0; k < m; ++k) {
            const double dd = z[k] - F[j * m + k];
            sq[k] = dd * dd;
        }
        const double d = sqrt(np_sum<IND_MAXM>(sq, m));
        best = (d < best || isnan(d)) ? d : best;  // np.min propagates NaN
    }
    for (int o = 16; o; o >>= 1) {
        const double y = __shfl_xor_sync(~0u, best, o);
        best = (y < best || isnan(y)) ? y : best;
    }
    if (lane == 0) dmin[w] = best;
}

__global__ void k_mean(const double *__restrict__ v, int64_t n, double *__restrict__ out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = np_pairwise_sum(v, n) / (double)n;
}

// ---------------------------------------------------------------- hv (m = 2, 3)
__global__ void k_hv_keep(const double *__restrict__ F, int64_t n, int m, const double *__restrict__ ref,
                          int32_t *__restrict__ flag) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int ok = 1;
    for (int k = 0; k < m; ++k) ok &= F[i * m + k] < ref[k];
    flag[i] = ok;
}

__global__ void k_hv_gather(const double *__restrict__ F, int64_t n, int m, const int32_t *__restrict__ flag,
                            const int32_t *__restrict__ pos, double *__restrict__ X, double *__restrict__ Y,
                            double *__restrict__ Z, uint64_t *__restrict__ ky, int32_t *__restrict__ idx) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n || !flag[i]) return;
    const int32_t p = pos[i];
    X[p] = F[i * m];
    Y[p] = F[i * m + 1];
    Z[p] = m == 3 ? F[i * m + 2] : 0.0;
    ky[p] = ordered_key(F[i * m + 1]);
    idx[p] = p;
}

__global__ void k_hv_xkeys(const double *__restrict__ X, const int32_t *__restrict__ idx, int64_t n,
                           uint64_t *__restrict__ kx) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) kx[i] = ordered_key(X[idx[i]]);
}

// one thread per slab s: the 2-D sweep over the rows with z <= zs[s] in (x, y) order
// (indicators.py:29-36), terms to this slab's scratch row, NumPy pairwise sum
__global__ void k_hv_slab(const double *__restrict__ X, const double *__restrict__ Y, const double *__restrict__ Z,
                          const int32_t *__restrict__ ord, int64_t n, const double *__restrict__ zs, int64_t s0,
                          int64_t s1, int m, const double *__restrict__ ref, double *__restrict__ scratch,
                          double *__restrict__ slab_hv) {
    const int64_t s = s0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= s1) return;
    const double z_lo = m == 3 ? zs[s] : INFINITY;
    double *t = scratch + (s - s0) * (n + 1);
    int64_t K = 0;
    double best = INFINITY, px = 0.0;
    bool have = false;
    for (int64_t q = 0; q < n; ++q) {
        const int32_t i = ord[q];
        if (m == 3 && !(Z[i] <= z_lo)) continue;
        const double x = X[i], y = Y[i];
        if (have) t[K++] = (x - px) * (ref[1] - best);  // (xs[k+1] - xs[k]) * (ref1 - best_y[k])
        best = have ? (y < best ? y : best) : y;      // np.minimum.accumulate
        px = x;
        have = true;
    }
    if (!have) {
        slab_hv[s] = 0.0;
        return;
    }
    t[K++] = (ref[0] - px) * (ref[1] - best);
    slab_hv[s] = np_pairwise_sum(t, K);
}

__global__ void k_hv_total(const double *__restrict__ slab_hv, const double *__restrict__ zs, int64_t nslab,
                           int m, double *__restrict__ out) {
    if (threadIdx.x || blockIdx.x) return;
    if (m == 2) {
        out[0] = nslab ? slab_hv[0] : 0.0;
        return;
    }
    double total = 0.0;
    for (int64_t s = 0; s < nslab; ++s) total += slab_hv[s] * (zs[s + 1] - zs[s]);
    out[0] = total;
}

// ---------------------------------------------------------------- hv (m > 3, MC)
__global__ void k_hv_mc(const double *__restrict__ F, int64_t n, int m, const double *__restrict__ S, int64_t ns,
                        int32_t *__restrict__ hits) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= ns) return;
    int h = 0;
    for (int64_t i = 0; i < n && !h; ++i) {
        int dom = 1;
        for (int k = 0; k < m; ++k) dom &= F[i * m + k] <= S[s * m + k];
        h |= dom;
    }
    hits[s] = h;
}

// ---------------------------------------------------------------- eu
// warp per weight row; dot products as the dgemm FMA chain (App. A2)
__global__ void k_eu_rows(const double *__restrict__ U, int64_t n, int m, const double *__restrict__ W, int64_t r,
                          int literal, double *__restrict__ best_out, double *__restrict__ lit_out) {
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= r) return;
    const double *wt = W + w * m;
    if (literal) {  // (weights[:, None, :] * U[None]).max(axis=2): r x n entries
        for (int64_t j = lane; j < n; j += 32) {
            double b = wt[0] * U[j * m];
            for (int k = 1; k < m; ++k) {
                const double v = wt[k] * U[j * m + k];
                b = (v > b || isnan(v)) ? v : b;
            }
            lit_out[w * n + j] = b;
        }
        return;
    }
    double best = -INFINITY;
    for (int64_t j = lane; j < n; j += 32) {
        double dot = wt[0] * U[j * m];
        for (int k = 1; k < m; ++k) dot = fma(wt[k], U[j * m + k], dot);
        best = (dot > best || isnan(dot)) ? dot : best;
    }
    for (int o = 16; o; o >>= 1) {
        const double y = __shfl_xor_sync(~0u, best, o);
        best = (y > best || isnan(y)) ? y : best;
    }
    if (lane == 0) best_out[w] = best;
}

static inline unsigned g1(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

}  // namespace temo

using namespace temo;

extern "C" size_t temo_igd_ws_bytes(int64_t r) { return (size_t)round_up(r * 8, 256) + 256; }

extern "C" int temo_igd(const double *F, int64_t n, int m, const double *Fstar, int64_t r, double *out,
                        void *ws, size_t ws_bytes, temo_stream_t stream) {
    if (n < 1 || r < 1 || m < 1 || m > IND_MAXM || !F || !Fstar || !out) return TEMO_EINVAL;
    if (!ws || ws_bytes < temo_igd_ws_bytes(r)) return TEMO_EWORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    double *dmin = static_cast<double *>(ws);
    k_igd_min<<<g1(r * 32), 256, 0, st>>>(F, n, m, Fstar, r, dmin);
    k_mean<<<1, 32, 0, st>>>(dmin, r, out);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

struct HvPlan {
    int32_t *flag, *pos, *idx_a, *idx_b;
    double *X, *Y, *Z, *zs, *zs2, *slab, *scratch;
    uint64_t *k_a, *k_b;
    int32_t *cnt;
    void *cub;
    size_t cub_bytes, total;
};

// slab scratch: one term row per slab of a wave; waves bound the workspace to 2^25 doubles
static int64_t hv_scratch_doubles(int64_t n) {
    const int64_t full = (n + 1) * (n + 1);
    return full < (int64_t(1) << 25) ? full : (int64_t(1) << 25) > (n + 1) ? (int64_t(1) << 25) : (n + 1);
}

static void plan_hv(HvPlan &p, void *base, int64_t n) {
    size_t a = 0, b = 0, c = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, a, (int32_t *)nullptr, (int32_t *)nullptr, (int)n);
    cub::DeviceRadixSort::SortPairs(nullptr, b, (uint64_t *)nullptr, (uint64_t *)nullptr, (int32_t *)nullptr,
                                    (int32_t *)nullptr, (int)n);
    cub::DeviceRadixSort::SortKeys(nullptr, c, (double *)nullptr, (double *)nullptr, (int)(n + 1));
    p.cub_bytes = a > b ? (a > c ? a : c) : (b > c ? b : c);
    Carve cv(base);
    p.flag = cv.take<int32_t>(n);
    p.pos = cv.take<int32_t>(n);
    p.idx_a = cv.take<int32_t>(n);
    p.idx_b = cv.take<int32_t>(n);
    p.X = cv.take<double>(n);
    p.Y = cv.take<double>(n);
    p.Z = cv.take<double>(n + 1);
    p.zs = cv.take<double>(n + 1);
    p.zs2 = cv.take<double>(n + 1);
    p.slab = cv.take<double>(n + 1);
    p.k_a = cv.take<uint64_t>(n);
    p.k_b = cv.take<uint64_t>(n);
    p.cnt = cv.take<int32_t>(4);
    p.scratch = cv.take<double>(hv_scratch_doubles(n));
    p.cub = cv.take<char>(p.cub_bytes);
    p.total = cv.off;
}

__global__ void k_hv_zs(const double *__restrict__ Z, const int32_t *__restrict__ flag, const int32_t *__restrict__ pos,
                        int64_t n, const double *__restrict__ ref, double *__restrict__ zall, int32_t *__restrict__ cnt) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i == 0) {
        const int32_t kept = n ? pos[n - 1] + flag[n - 1] : 0;
        cnt[0] = kept;
        zall[kept] = ref[2];
    }
    (void)Z;
}

// unique sorted values (np.unique) of the sorted array v[0..len): first of each run
__global__ void k_unique(const double *__restrict__ v, const int32_t *__restrict__ lenp, double *__restrict__ u,
                         int32_t *__restrict__ ulen) {
    if (threadIdx.x || blockIdx.x) return;
    const int32_t len = lenp[0] + 1;
    int32_t k = 0;
    for (int32_t i = 0; i < len; ++i)
        if (i == 0 || v[i] != v[i - 1]) u[k++] = v[i];
    ulen[0] = k;
}

extern "C" size_t temo_hv_ws_bytes(int64_t n, int m) {
    if (n < 1 || m < 2) return 0;
    HvPlan p;
    plan_hv(p, nullptr, n);
    return p.total;
}

// Exact hypervolume for m = 2, 3 (indicators.py:29-66).  The slab count is data dependent:
// one host read of the kept-row and slab counts (the indicator is off the generation path).
extern "C" int temo_hv(const double *F, int64_t n, int m, const double *ref, double *out, void *ws,
                       size_t ws_bytes, temo_stream_t stream) {
    if (n < 1 || (m != 2 && m != 3) || !F || !ref || !out) return TEMO_EINVAL;
    HvPlan p;
    plan_hv(p, nullptr, n);
    if (!ws || ws_bytes < p.total) return TEMO_EWORKSPACE;
    plan_hv(p, ws, n);
    cudaStream_t st = (cudaStream_t)stream;
    size_t tb = p.cub_bytes;
    k_hv_keep<<<g1(n), 256, 0, st>>>(F, n, m, ref, p.flag);
    TEMO_CUDA(cub::DeviceScan::ExclusiveSum(p.cub, tb, p.flag, p.pos, (int)n, st));
    k_hv_gather<<<g1(n), 256, 0, st>>>(F, n, m, p.flag, p.pos, p.X, p.Y, p.Z, p.k_a, p.idx_a);
    k_hv_zs<<<1, 32, 0, st>>>(p.Z, p.flag, p.pos, n, ref, p.Z, p.cnt);
    int32_t kept = 0;
    TEMO_CUDA(cudaMemcpyAsync(&kept, p.cnt, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    TEMO_CUDA(cudaStreamSynchronize(st));
    if (kept == 0) {
        TEMO_CUDA(cudaMemsetAsync(out, 0, sizeof(double), st));
        return TEMO_OK;
    }
    // (x, y) order, stable: by y, then stably by x (np.lexsort((y, x)))
    tb = p.cub_bytes;
    TEMO_CUDA(cub::DeviceRadixSort::SortPairs(p.cub, tb, p.k_a, p.k_b, p.idx_a, p.idx_b, kept, 0, 64, st));
    k_hv_xkeys<<<g1(kept), 256, 0, st>>>(p.X, p.idx_b, kept, p.k_a);
    tb = p.cub_bytes;
    TEMO_CUDA(cub::DeviceRadixSort::SortPairs(p.cub, tb, p.k_a, p.k_b, p.idx_b, p.idx_a, kept, 0, 64, st));
    int64_t nslab = 1;
    if (m == 3) {  // zs = np.unique(r_[z, ref2])
        tb = p.cub_bytes;
        TEMO_CUDA(cub::DeviceRadixSort::SortKeys(p.cub, tb, p.Z, p.zs2, kept + 1, 0, 64, st));
        k_unique<<<1, 32, 0, st>>>(p.zs2, p.cnt, p.zs, p.cnt + 1);
        int32_t nu = 0;
        TEMO_CUDA(cudaMemcpyAsync(&nu, p.cnt + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        TEMO_CUDA(cudaStreamSynchronize(st));
        nslab = nu - 1;
    }
    const int64_t wave = hv_scratch_doubles(n) / (kept + 1);
    for (int64_t s0 = 0; s0 < nslab; s0 += wave) {
        const int64_t s1 = s0 + wave < nslab ? s0 + wave : nslab;
        k_hv_slab<<<g1(s1 - s0, 128), 128, 0, st>>>(p.X, p.Y, p.Z, p.idx_a, kept, p.zs, s0, s1, m, ref, p.scratch,
                                                   p.slab);
    }
    k_hv_total<<<1, 32, 0, st>>>(p.slab, p.zs, nslab, m, out);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

// Monte-Carlo dominated fraction for m > 3 (indicators.py:59-66): hits[s] = any row <= S[s]
extern "C" int temo_hv_mc_hits(const double *F, int64_t n, int m, const double *S, int64_t ns, int32_t *hits,
                               temo_stream_t stream) {
    if (n < 0 || ns < 0 || m < 1 || !S || !hits || (n && !F)) return TEMO_EINVAL;
    if (!ns) return TEMO_OK;
    k_hv_mc<<<g1(ns), 256, 0, (cudaStream_t)stream>>>(F, n, m, S, ns, hits);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

extern "C" size_t temo_eu_ws_bytes(int64_t n, int64_t r, int literal) {
    return (size_t)round_up((literal ? r * n : r) * 8, 256) + 256;
}

extern "C" int temo_eu(const double *U, int64_t n, int m, const double *W, int64_t r, int literal, double *out,
                       void *ws, size_t ws_bytes, temo_stream_t stream) {
    if (n < 1 || r < 1 || m < 1 || m > IND_MAXM || !U || !W || !out) return TEMO_EINVAL;
    if (!ws || ws_bytes < temo_eu_ws_bytes(n, r, literal)) return TEMO_EWORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    double *buf = static_cast<double *>(ws);
    k_eu_rows<<<g1(r * 32), 256, 0, st>>>(U, n, m, W, r, literal, buf, buf);
    k_mean<<<1, 32, 0, st>>>(buf, literal ? r * n : r, out);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}
