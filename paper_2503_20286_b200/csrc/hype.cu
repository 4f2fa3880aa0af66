// HypE Monte-Carlo hypervolume fitness and selection on B200
// (replaces temo hype.py:37-163).
//
//   alpha     hype.py:37-51   one thread: exact elementwise lam, sequential cumprod
//   samples   hype.py:79      S = f_l + U * span, U from the NumPy Philox stream
//                             (blocks of 65536 concatenate into one stream)
//   pass 1    hype.py:80-81   lane = point, samples broadcast from smem; "sample not
//                             dominated" = OR of the sign bits of S_k - F_k, funnel-
//                             shifted into a row word of the point's sample bitmap;
//                             per-sample dominator counts by warp bit-transpose
//   weights   hype.py:82      w = alpha[count - 1] (0 for count 0)
//   pass 2    hype.py:83      per (point, 2048-sample sub-block, lane) the OpenBLAS
//                             dgemv_t lane sums of SURVEY App. A7 over set bits,
//                             combined per point in the same order (bit-exact with
//                             single-threaded OpenBLAS), then * prod(span) / s
//   select    hype.py:153-163 rank -> k -> lexsort(r, -d)[:n] by two stable radix passes
#include <cub/cub.cuh>

#include "common.cuh"
#include "philox.cuh"

namespace temo {

constexpr int HT = 256;            // pass-1 tile (points x samples)
constexpr int SAMPLE_BLOCK = 65536;  // hype.py:58
constexpr int SUB = 2048;          // dgemv_t sub-block (App. A7)

// ---------------------------------------------------------------- alpha
// alpha[c] = cumprod(lam)[c] / (c + 1) with lam[0] = 1, lam[l] = (k - l) / (n1 - l) (hype.py:24-33,
// np.cumprod: a sequential product).  Thread 0 runs the product chain in order and stops once it
// is exactly 0.0 (every later product is 0 too -- bit-exact) or at q = k; the CTA zero-fills the
// rest in parallel.  One CTA of ALPHA_T threads.
constexpr int ALPHA_T = 256;
__device__ __forceinline__ void alpha_body(int64_t n1, int64_t k, double *__restrict__ alpha) {
    __shared__ int64_t s_stop;
    if (threadIdx.x == 0) {
        double c = 1.0;
        int64_t q = 0;
        const int64_t qk = k < n1 ? k : n1;
        for (; q < qk; ++q) {
            if (q > 0) c = c * ((double)(k - q) / (double)(n1 - q));
            if (c == 0.0) break;
            alpha[q] = c / (double)(q + 1);
        }
        s_stop = q;
    }
    __syncthreads();
    for (int64_t q = s_stop + threadIdx.x; q < n1; q += blockDim.x) alpha[q] = 0.0;
}

__global__ void __launch_bounds__(ALPHA_T) k_alpha(int64_t n1, int64_t k, double *__restrict__ alpha) {
    alpha_body(n1, k, alpha);
}

// alpha from the device-side k (scal[1]); only when estimation runs (scal[2])
__global__ void __launch_bounds__(ALPHA_T) k_alpha_dev(int64_t n1, const int32_t *__restrict__ scal,
                                                       double *__restrict__ alpha) {
    if (!scal[2]) return;
    alpha_body(n1, scal[1], alpha);
}

// ---------------------------------------------------------------- column stats
// mn/mx over all rows (hype.py:70, 129-132), one CTA per column
__global__ void k_minmax_cols(const double *__restrict__ F, int64_t n, int m, double *__restrict__ mn,
                              double *__restrict__ mx) {
    __shared__ double smn[32], smx[32];
    const int k = blockIdx.x;
    double a = INFINITY, b = -INFINITY;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double v = F[i * m + k];
        a = v < a ? v : a;
        b = v > b ? v : b;
    }
    for (int d = 16; d; d >>= 1) {
        const double a2 = __shfl_xor_sync(~0u, a, d), b2 = __shfl_xor_sync(~0u, b, d);
        a = a2 < a ? a2 : a;
        b = b2 > b ? b2 : b;
    }
    if ((threadIdx.x & 31) == 0) { smn[threadIdx.x >> 5] = a; smx[threadIdx.x >> 5] = b; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            a = smn[w] < a ? smn[w] : a;
            b = smx[w] > b ? smx[w] : b;
        }
        mn[k] = a;
        mx[k] = b;
    }
}

// v_ref (auto: mx + 0.1 (mx - mn)), span = v_ref - f_l, P = prod(span), ok = all(span > 0)
__global__ void k_hv_box(const double *__restrict__ mn, const double *__restrict__ mx,
                         const double *__restrict__ vref_in, int m, double *__restrict__ vref,
                         double *__restrict__ span, double *__restrict__ prodspan,
                         int32_t *__restrict__ ok) {
    if (threadIdx.x || blockIdx.x) return;
    int good = 1;
    double P = 1.0;
    for (int k = 0; k < m; ++k) {
        const double r = vref_in ? vref_in[k] : mx[k] + 0.1 * (mx[k] - mn[k]);
        vref[k] = r;
        const double sp = r - mn[k];
        span[k] = sp;
        good &= sp > 0.0;
        P = k == 0 ? sp : P * sp;
    }
    *prodspan = P;
    *ok = *ok && good;  // caller's gate (k >= 1) and a non-degenerate box (hype.py:72-73)
}

// S (b x m) = f_l + U * span for stream elements [e0*m, (e0+b)*m)
__global__ void k_hv_samples(Philox ph, uint64_t off, const double *__restrict__ U_in, int64_t e0,
                             int64_t b, int m, const double *__restrict__ fl,
                             const double *__restrict__ span, const int32_t *__restrict__ ok,
                             double *__restrict__ S) {
    if (!*ok) return;
    const int64_t base = 4 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
    PhiloxCursor c;
    for (int64_t t = base; t < base + 4 && t < b * m; ++t) {
        const int k = (int)(t % m);
        const int64_t e = e0 * m + t;
        const double u = U_in ? U_in[e] : c.uniform(ph, off + e);
        S[t] = fl[k] + u * span[k];
    }
}

// ---------------------------------------------------------------- pass 1
struct Transpose32h {
    uint32_t keep[5];
    __device__ __forceinline__ explicit Transpose32h(int lane) {
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            const int s = 16 >> q;
            const uint32_t lowmask = q == 0 ? 0x0000FFFFu : q == 1 ? 0x00FF00FFu : q == 2 ? 0x0F0F0F0Fu
                                   : q == 3 ? 0x33333333u : 0x55555555u;
            keep[q] = (lane & s) == 0 ? lowmask : ~lowmask;
        }
    }
    __device__ __forceinline__ uint32_t operator()(uint32_t x, int lane) const {
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            const int s = 16 >> q;
            const uint32_t y = __shfl_xor_sync(~0u, x, s);
            const uint32_t t = (lane & s) == 0 ? (y << s) : (y >> s);
            x = (x & keep[q]) | (t & ~keep[q]);
        }
        return x;
    }
};

// bitmap row i (Wb words), bit s set iff point i weakly dominates sample s
template <int M>
__global__ void __launch_bounds__(HT) k_hv_dom(const double *__restrict__ F, int64_t n1,
                                               const double *__restrict__ S, int64_t b,
                                               const int32_t *__restrict__ ok, int64_t Wb,
                                               uint32_t *__restrict__ bits, int32_t *__restrict__ cnt) {
    if (!*ok) return;
    __shared__ double sS[HT * M];
    __shared__ int32_t sCnt[HT];
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t i = blockIdx.x * (int64_t)HT + tid;
    const int64_t s0 = blockIdx.y * (int64_t)HT;
    double f[M];
    const bool row_ok = i < n1;
#pragma unroll
    for (int k = 0; k < M; ++k) f[k] = row_ok ? F[i * M + k] : 0.0;
    for (int q = tid; q < HT * M; q += HT) {
        const int64_t e = s0 * M + q;
        sS[q] = e < b * M ? S[e] : -INFINITY;  // padding samples are never dominated
    }
    sCnt[tid] = 0;
    __syncthreads();
    const Transpose32h tr(lane);
#pragma unroll 1
    for (int jw = 0; jw < HT / 32; ++jw) {
        uint32_t acc = 0;
#pragma unroll 8
        for (int bb = 0; bb < 32; ++bb) {
            const double *x = sS + (jw * 32 + bb) * M;
            // sample - point < 0 in any coordinate <=> not dominated (sign of the difference)
            uint32_t hi = 0;
#pragma unroll
            for (int k = 0; k < M; ++k) hi |= (uint32_t)__double2hiint(x[k] - f[k]);
            acc = __funnelshift_l(hi, acc, 1);
        }
        uint32_t word = row_ok ? __brev(~acc) : 0u;
        const int64_t base = s0 + jw * 32;
        word &= base + 32 <= b ? ~0u : (base >= b ? 0u : (1u << (b - base)) - 1u);
        if (row_ok && base < b) bits[i * Wb + base / 32] = word;
        const int c = __popc(tr(word, lane));
        if (c) atomicAdd(&sCnt[jw * 32 + lane], c);
    }
    __syncthreads();
    const int64_t s = s0 + tid;
    if (s < b && sCnt[tid]) atomicAdd(cnt + s, sCnt[tid]);
}

__global__ void k_hv_weights(const int32_t *__restrict__ cnt, int64_t b, const double *__restrict__ alpha,
                             const int32_t *__restrict__ ok, double *__restrict__ w) {
    if (!*ok) return;
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= b) return;
    const int c = cnt[s];
    w[s] = c > 0 ? alpha[c - 1] : 0.0;
}

// ---------------------------------------------------------------- pass 2 (App. A7 order)
// One CTA per (sub-block g, 64 points); 4 threads per point = the 4 dgemv lanes.
// T[g * n1 + i] = (s0 + s2) + (s1 + s3)   (4-lane rows)   or   s0 + s1   (2-lane rows);
// column-major so a rank's contiguous range of sub-block columns is one exchange segment.
__global__ void __launch_bounds__(256) k_hv_partial(const uint32_t *__restrict__ bits, int64_t Wb,
                                                    int64_t n1, int64_t b4, int nsub,
                                                    const double *__restrict__ w,
                                                    const int32_t *__restrict__ ok, int64_t two_lo,
                                                    int64_t two_hi, double *__restrict__ T) {
    if (!*ok) return;
    __shared__ double sw[SUB];
    const int g = blockIdx.y;
    const int64_t e0 = (int64_t)g * SUB;
    const int len = (int)min((int64_t)SUB, b4 - e0);
    for (int q = threadIdx.x; q < len; q += blockDim.x) sw[q] = w[e0 + q];
    __syncthreads();
    const int ln = threadIdx.x & 3;
    const int64_t i = blockIdx.x * 64 + (threadIdx.x >> 2);
    double acc = 0.0;
    const bool two = i >= two_lo && i < two_hi;
    if (i < n1) {
        const uint32_t *row = bits + i * Wb + e0 / 32;
        const int nl = two ? 2 : 4;
        if (!two || ln < 2) {
            // lane ln sums elements e (relative to e0) with e % nl == ln, ascending
            uint32_t lmask = 0;
            for (int p = ln; p < 32; p += nl) lmask |= 1u << p;
            for (int wd = 0; wd * 32 < len; ++wd) {
                uint32_t x = row[wd] & lmask;
                const int rem = len - wd * 32;
                if (rem < 32) x &= (1u << rem) - 1u;
                while (x) {
                    const int p = __ffs(x) - 1;
                    x &= x - 1;
                    acc = acc + sw[wd * 32 + p];
                }
            }
        }
    }
    // combine the lanes of a point (threads 4q .. 4q+3)
    const double a1 = __shfl_down_sync(~0u, acc, 1);
    const double a2 = __shfl_down_sync(~0u, acc, 2);
    const double a3 = __shfl_down_sync(~0u, acc, 3);
    if (ln == 0 && i < n1) T[(int64_t)g * n1 + i] = two ? acc + a1 : (acc + a2) + (a1 + a3);
}

// the b % 4 tail of a sample block (relative samples [t0, t0 + tlen) of the bitmap): the
// grouped sum ((p0 + p1) + p2) of the tail products (App. A7) -> one exchange column
__global__ void k_hv_tail(const uint32_t *__restrict__ bits, int64_t Wb, int64_t n1, int64_t t0, int64_t tlen,
                          const double *__restrict__ w, const int32_t *__restrict__ ok, double *__restrict__ col) {
    if (!*ok) return;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n1) return;
    double tail = 0.0;
    for (int64_t e = t0; e < t0 + tlen; ++e) {
        const double p = ((bits[i * Wb + e / 32] >> (e & 31)) & 1u) ? w[e] : 0.0;
        tail = e == t0 ? p : tail + p;
    }
    col[i] = tail;
}

// per point over every sample block in order: y = sum of its sub-block columns (sequential),
// + the tail column if the block has a b % 4 tail; contrib = contrib + y (hype.py:83)
__global__ void k_hv_combine(const double *__restrict__ Tg, int64_t n1, int64_t s, const int32_t *__restrict__ ok,
                             double *__restrict__ contrib) {
    if (!*ok) return;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n1) return;
    double c = 0.0;
    int64_t col = 0;
    for (int64_t e0 = 0; e0 < s; e0 += SAMPLE_BLOCK) {
        const int64_t b = s - e0 < SAMPLE_BLOCK ? s - e0 : SAMPLE_BLOCK;
        const int64_t b4 = b - b % 4;
        const int64_t nsub = (b4 + SUB - 1) / SUB;
        double y = 0.0;
        for (int64_t g = 0; g < nsub; ++g) y = y + Tg[(col + g) * n1 + i];
        if (b4 < b) y = y + Tg[(col + nsub) * n1 + i];
        c = c + y;
        col += nsub + 1;
    }
    contrib[i] = c;
}

__global__ void k_hv_final(double *__restrict__ contrib, int64_t n1, const double *__restrict__ P,
                           int64_t s, const int32_t *__restrict__ ok) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n1) return;
    contrib[i] = *ok ? contrib[i] * *P / (double)s : 0.0;
}

// ---------------------------------------------------------------- selection
// scalars: [0] = count(r <= l), [1] = k, [2] = estimation ran (k >= 1)
__global__ void k_hype_k(const int32_t *__restrict__ rank, const int32_t *__restrict__ lp, int64_t N,
                         int64_t n, int32_t *__restrict__ scal) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int c = (i < N && rank[i] <= *lp) ? 1 : 0;
    c = __reduce_add_sync(~0u, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(scal, c);
}

__global__ void k_hype_k_final(int32_t *__restrict__ scal, int64_t n, int32_t *__restrict__ ok) {
    const int k = scal[0] - (int)n;
    scal[1] = k;
    scal[2] = k >= 1;
    *ok = k >= 1;  // hype.py:156-160: k < 1 -> no estimation, no draws
}

__global__ void k_hype_keys(const int32_t *__restrict__ rank, const int32_t *__restrict__ lp,
                            const double *__restrict__ vhv, const int32_t *__restrict__ scal,
                            int64_t N, uint64_t *__restrict__ key, int32_t *__restrict__ idx) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    // d = retained ? v_hv : -BIG ; sort key -d (ties: index), -0.0 == +0.0
    const double v = scal[2] ? vhv[i] : 0.0;
    const double d = rank[i] <= *lp ? v : -TEMO_BIG;
    key[i] = ordered_key(-d);
    idx[i] = (int32_t)i;
}

__global__ void k_gather_rank_keys(const int32_t *__restrict__ rank, const int32_t *__restrict__ idx,
                                   int64_t N, uint32_t *__restrict__ key) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p < N) key[p] = (uint32_t)rank[idx[p]];
}

// ---------------------------------------------------------------- host
struct HvPlan {
    int64_t n1, s, Wb, nsub_max;
    int m;
    double *mn, *mx, *vref, *span, *P, *alpha, *S, *w, *T, *contrib;
    int32_t *cnt, *ok;
    uint32_t *bits;
    size_t total;
};

// exchange columns of s samples: per 65,536-sample block its 2048-sample sub-blocks + one tail column
static int64_t hv_columns(int64_t s) {
    int64_t c = 0;
    for (int64_t e0 = 0; e0 < s; e0 += SAMPLE_BLOCK) {
        const int64_t b = s - e0 < SAMPLE_BLOCK ? s - e0 : SAMPLE_BLOCK;
        c += (b - b % 4 + SUB - 1) / SUB + 1;
    }
    return c;
}

static void plan_hv(HvPlan &p, void *base, int64_t n1, int m, int64_t s) {
    p.n1 = n1;
    p.m = m;
    p.s = s;
    const int64_t b = s < SAMPLE_BLOCK ? s : SAMPLE_BLOCK;
    p.Wb = (b + 31) / 32;
    p.nsub_max = (b + SUB - 1) / SUB;
    Carve c(base);
    p.mn = c.take<double>(16);
    p.mx = c.take<double>(16);
    p.vref = c.take<double>(16);
    p.span = c.take<double>(16);
    p.P = c.take<double>(1);
    p.ok = c.take<int32_t>(1);
    p.alpha = c.take<double>(n1);
    p.S = c.take<double>((size_t)b * m);
    p.w = c.take<double>(b);
    p.cnt = c.take<int32_t>(b);
    p.bits = c.take<uint32_t>((size_t)n1 * p.Wb);
    p.T = c.take<double>((size_t)n1 * hv_columns(s));
    p.contrib = c.take<double>(n1);
    p.total = c.off;
}

static inline dim3 gdim(int64_t n, int t = 256) { return dim3((unsigned)((n + t - 1) / t)); }

// hv_estimate, split so a multi-GPU run can shard the samples by exchange column
// (SURVEY 8e): prepare (box, P, ok) -> columns [c_lo, c_hi) of Tg -> (all-gather) -> combine.
// `ok` must already hold whether to estimate (k >= 1); the box check happens here.
static void hv_prepare(HvPlan &p, const double *F, const double *vref_in, cudaStream_t sm) {
    k_minmax_cols<<<p.m, 256, 0, sm>>>(F, p.n1, p.m, p.mn, p.mx);
    k_hv_box<<<1, 1, 0, sm>>>(p.mn, p.mx, vref_in, p.m, p.vref, p.span, p.P, p.ok);
}

static int hv_cols(HvPlan &p, const double *F, const temo_philox_state *st, uint64_t off, const double *U,
                   int64_t c_lo, int64_t c_hi, double *Tg, cudaStream_t sm) {
    const int64_t n1 = p.n1, s = p.s;
    const int m = p.m;
    const Philox ph = st ? philox_from(*st) : Philox{};
    const int64_t two_lo = (n1 % 4 == 2 || n1 % 4 == 3) ? n1 - n1 % 4 : -1;
    const int64_t two_hi = two_lo >= 0 ? two_lo + 2 : -1;
    int64_t cb = 0;  // first exchange column of the block
    for (int64_t e0 = 0; e0 < s; e0 += SAMPLE_BLOCK) {
        const int64_t b = s - e0 < SAMPLE_BLOCK ? s - e0 : SAMPLE_BLOCK;
        const int64_t b4 = b - b % 4;
        const int64_t nsub = (b4 + SUB - 1) / SUB;
        const int64_t lo = c_lo - cb > 0 ? c_lo - cb : 0, hi = c_hi - cb < nsub + 1 ? c_hi - cb : nsub + 1;
        if (lo < hi) {
            // this rank's samples of the block: sub-blocks [lo, min(hi, nsub)) then the tail
            const int64_t e_lo = lo < nsub ? lo * SUB : b4;
            const int64_t e_hi = hi > nsub ? b : (hi * SUB < b4 ? hi * SUB : b4);
            const int64_t len = e_hi - e_lo;
            if (len > 0) {
                const int64_t Wb = (len + 31) / 32;
                k_hv_samples<<<gdim((len * m + 3) / 4), 256, 0, sm>>>(ph, off, U, e0 + e_lo, len, m, p.mn, p.span,
                                                                      p.ok, p.S);
                TEMO_CUDA(cudaMemsetAsync(p.cnt, 0, sizeof(int32_t) * len, sm));
                stage_begin(S_HV_COUNT, sm);
                dim3 g1((unsigned)((n1 + HT - 1) / HT), (unsigned)((len + HT - 1) / HT));
#define HVD(MM) case MM: k_hv_dom<MM><<<g1, HT, 0, sm>>>(F, n1, p.S, len, p.ok, Wb, p.bits, p.cnt); break;
                switch (m) {
                    HVD(1) HVD(2) HVD(3) HVD(4) HVD(5) HVD(6) HVD(7) HVD(8) HVD(9) HVD(10) HVD(11) HVD(12)
                    HVD(13) HVD(14) HVD(15) HVD(16)
                    default: return TEMO_EINVAL;
                }
#undef HVD
                stage_end(S_HV_COUNT, sm);
                k_hv_weights<<<gdim(len), 256, 0, sm>>>(p.cnt, len, p.alpha, p.ok, p.w);
                stage_begin(S_HV_CONTRIB, sm);
                const int64_t sub_hi = hi < nsub ? hi : nsub;
                if (lo < sub_hi) {
                    const int64_t b4r = (b4 < e_hi ? b4 : e_hi) - e_lo;
                    dim3 g2((unsigned)((n1 + 63) / 64), (unsigned)(sub_hi - lo));
                    k_hv_partial<<<g2, 256, 0, sm>>>(p.bits, Wb, n1, b4r, (int)(sub_hi - lo), p.w, p.ok, two_lo, two_hi,
                                                     Tg + (cb + lo - c_lo) * n1);
                }
                if (hi > nsub && b4 < b)  // the tail column
                    k_hv_tail<<<gdim(n1), 256, 0, sm>>>(p.bits, Wb, n1, b4 - e_lo, b - b4, p.w, p.ok,
                                                        Tg + (cb + nsub - c_lo) * n1);
                stage_end(S_HV_CONTRIB, sm);
            }
        }
        cb += nsub + 1;
    }
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

static int hv_combine_final(HvPlan &p, const double *Tg, double *v_hv, cudaStream_t sm) {
    const int64_t n1 = p.n1;
    TEMO_CUDA(cudaMemsetAsync(p.contrib, 0, sizeof(double) * n1, sm));
    k_hv_combine<<<gdim(n1), 256, 0, sm>>>(Tg, n1, p.s, p.ok, p.contrib);
    k_hv_final<<<gdim(n1), 256, 0, sm>>>(p.contrib, n1, p.P, p.s, p.ok);
    TEMO_CUDA(cudaMemcpyAsync(v_hv, p.contrib, sizeof(double) * n1, cudaMemcpyDeviceToDevice, sm));
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

static int hv_run(HvPlan &p, const double *F, const double *vref_in, const temo_philox_state *st,
                  uint64_t off, const double *U, double *v_hv, cudaStream_t sm) {
    hv_prepare(p, F, vref_in, sm);
    const int rc = hv_cols(p, F, st, off, U, 0, hv_columns(p.s), p.T, sm);
    if (rc) return rc;
    return hv_combine_final(p, p.T, v_hv, sm);
}

struct SelHPlan {
    uint64_t *key_a, *key_b;
    uint32_t *rk_a, *rk_b;
    int32_t *idx_a, *idx_b, *scal;
    void *cub;
    size_t cub_bytes, total;
};

static void plan_selh(SelHPlan &p, void *base, int64_t N) {
    size_t a = 0, b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (uint64_t *)nullptr, (uint64_t *)nullptr,
                                    (int32_t *)nullptr, (int32_t *)nullptr, (int)N);
    cub::DeviceRadixSort::SortPairs(nullptr, b, (uint32_t *)nullptr, (uint32_t *)nullptr,
                                    (int32_t *)nullptr, (int32_t *)nullptr, (int)N);
    p.cub_bytes = a > b ? a : b;
    Carve c(base);
    p.key_a = c.take<uint64_t>(N);
    p.key_b = c.take<uint64_t>(N);
    p.rk_a = c.take<uint32_t>(N);
    p.rk_b = c.take<uint32_t>(N);
    p.idx_a = c.take<int32_t>(N);
    p.idx_b = c.take<int32_t>(N);
    p.scal = c.take<int32_t>(8);
    p.cub = c.take<char>(p.cub_bytes);
    p.total = c.off;
}

}  // namespace temo

using namespace temo;

extern "C" int temo_hype_alpha(int64_t n1, int64_t k, double *alpha, temo_stream_t stream) {
    if (n1 < 1 || k < 1 || k > n1 || !alpha) return TEMO_EINVAL;
    k_alpha<<<1, ALPHA_T, 0, (cudaStream_t)stream>>>(n1, k, alpha);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

__global__ void k_auto_ref(const double *__restrict__ mn, const double *__restrict__ mx, int m,
                           double *__restrict__ out) {
    const int k = threadIdx.x;
    if (k < m) out[k] = mx[k] + 0.1 * (mx[k] - mn[k]);
}

// hype.auto_reference (hype.py:129-132): out (m) = max + 0.1 (max - min) over all rows
extern "C" int temo_auto_reference(const double *F, int64_t n, int m, double *out, double *scratch,
                                   temo_stream_t stream) {
    if (!F || n < 1 || m < 1 || m > 16 || !out || !scratch) return TEMO_EINVAL;
    cudaStream_t sm = (cudaStream_t)stream;
    k_minmax_cols<<<m, 256, 0, sm>>>(F, n, m, scratch, scratch + 16);
    k_auto_ref<<<1, 32, 0, sm>>>(scratch, scratch + 16, m, out);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

extern "C" size_t temo_hv_estimate_ws_bytes(int64_t n1, int m, int64_t s) {
    HvPlan p;
    plan_hv(p, nullptr, n1, m, s);
    return p.total;
}

extern "C" int temo_hv_estimate(const double *F, int64_t n1, int m, const double *v_ref, int64_t k,
                                int64_t s, const temo_philox_state *st, uint64_t off, const double *U,
                                double *v_hv, int32_t *drew, void *ws, size_t ws_bytes,
                                temo_stream_t stream) {
    if (!F || n1 < 1 || m < 1 || m > 16 || !v_ref || s < 1 || k < 1 || k > n1 || !v_hv) return TEMO_EINVAL;
    if (!st && !U) return TEMO_EINVAL;
    cudaStream_t sm = (cudaStream_t)stream;
    HvPlan p;
    plan_hv(p, nullptr, n1, m, s);
    if (!ws || ws_bytes < p.total) return TEMO_EWORKSPACE;
    plan_hv(p, ws, n1, m, s);
    k_alpha<<<1, ALPHA_T, 0, sm>>>(n1, k, p.alpha);
    const int32_t one = 1;
    TEMO_CUDA(cudaMemcpyAsync(p.ok, &one, sizeof(int32_t), cudaMemcpyHostToDevice, sm));
    const int rc = hv_run(p, F, v_ref, st, off, U, v_hv, sm);
    if (rc) return rc;
    if (drew) TEMO_CUDA(cudaMemcpyAsync(drew, p.ok, sizeof(int32_t), cudaMemcpyDeviceToDevice, sm));
    return TEMO_OK;
}

extern "C" size_t temo_hype_select_ws_bytes(int64_t N, int m, int64_t s) {
    SelHPlan a;
    plan_selh(a, nullptr, N);
    HvPlan h;
    plan_hv(h, nullptr, N, m, s);
    return round_up(a.total, 256) + h.total;
}

// hype.environmental_selection core (hype.py:153-163) on ranks from temo_rank (SELECT mode),
// in three phases so the Monte-Carlo columns can be sharded over ranks:
//   begin   : k = count(r <= l) - n (device), alpha, box / P / ok
//   columns : exchange columns [c_lo, c_hi) of the contribution partials (column-major n1 x C)
//   end     : combine every column in the reference's order, lexsort (rank, -v_hv, index) -> keep
// `info` (int32[4]) receives {count(r <= l), k, estimated, box_ok}: the host advances its
// Generator by s*m outputs iff estimated && box_ok.
struct HypeWs {
    SelHPlan a;
    HvPlan h;
};

static int hype_ws(HypeWs &w, void *ws, size_t ws_bytes, int64_t N, int m, int64_t s) {
    plan_selh(w.a, nullptr, N);
    plan_hv(w.h, nullptr, N, m, s);
    if (!ws || ws_bytes < round_up(w.a.total, 256) + w.h.total) return TEMO_EWORKSPACE;
    plan_selh(w.a, ws, N);
    plan_hv(w.h, static_cast<char *>(ws) + round_up(w.a.total, 256), N, m, s);
    return TEMO_OK;
}

extern "C" int64_t temo_hype_columns(int64_t s) { return s < 1 ? 0 : hv_columns(s); }

extern "C" int temo_hype_select_begin(const double *F, int64_t N, int m, int64_t n, int64_t s, const double *v_ref,
                                      const int32_t *rank, const int32_t *l, void *ws, size_t ws_bytes,
                                      temo_stream_t stream) {
    if (!F || N < 1 || m < 1 || m > 16 || n < 1 || n > N || s < 1 || !rank || !l) return TEMO_EINVAL;
    HypeWs w;
    if (int rc = hype_ws(w, ws, ws_bytes, N, m, s)) return rc;
    cudaStream_t sm = (cudaStream_t)stream;
    stage_begin(S_HYPE_SELECT, sm);
    TEMO_CUDA(cudaMemsetAsync(w.a.scal, 0, sizeof(int32_t) * 8, sm));
    k_hype_k<<<gdim(N), 256, 0, sm>>>(rank, l, N, n, w.a.scal);
    k_hype_k_final<<<1, 1, 0, sm>>>(w.a.scal, n, w.h.ok);  // estimation only if k >= 1 (hype.py:156)
    stage_end(S_HYPE_SELECT, sm);
    k_alpha_dev<<<1, ALPHA_T, 0, sm>>>(N, w.a.scal, w.h.alpha);
    hv_prepare(w.h, F, v_ref, sm);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

extern "C" int temo_hype_select_columns(const double *F, int64_t N, int m, int64_t s, int64_t c_lo, int64_t c_hi,
                                        const temo_philox_state *st, uint64_t off, const double *U, double *Tseg,
                                        void *ws, size_t ws_bytes, temo_stream_t stream) {
    if (!F || N < 1 || m < 1 || m > 16 || s < 1 || c_lo < 0 || c_hi < c_lo || c_hi > hv_columns(s)) return TEMO_EINVAL;
    if (!st && !U) return TEMO_EINVAL;
    HypeWs w;
    if (int rc = hype_ws(w, ws, ws_bytes, N, m, s)) return rc;
    return hv_cols(w.h, F, st, off, U, c_lo, c_hi, Tseg ? Tseg : w.h.T + c_lo * N, (cudaStream_t)stream);
}

extern "C" int temo_hype_select_end(const double *F, int64_t N, int m, int64_t n, int64_t s, const int32_t *rank,
                                    const int32_t *l, const double *Tg, int32_t *keep, double *v_hv, int32_t *info,
                                    void *ws, size_t ws_bytes, temo_stream_t stream) {
    if (!F || N < 1 || m < 1 || m > 16 || n < 1 || n > N || s < 1 || !rank || !l || !keep || !v_hv) return TEMO_EINVAL;
    HypeWs w;
    if (int rc = hype_ws(w, ws, ws_bytes, N, m, s)) return rc;
    cudaStream_t sm = (cudaStream_t)stream;
    if (int rc = hv_combine_final(w.h, Tg ? Tg : w.h.T, v_hv, sm)) return rc;
    SelHPlan &a = w.a;
    stage_begin(S_HYPE_SELECT, sm);
    k_hype_keys<<<gdim(N), 256, 0, sm>>>(rank, l, v_hv, a.scal, N, a.key_a, a.idx_a);
    size_t tb = a.cub_bytes;
    TEMO_CUDA(cub::DeviceRadixSort::SortPairs(a.cub, tb, a.key_a, a.key_b, a.idx_a, a.idx_b, (int)N, 0, 64, sm));
    k_gather_rank_keys<<<gdim(N), 256, 0, sm>>>(rank, a.idx_b, N, a.rk_a);
    TEMO_CUDA(cub::DeviceRadixSort::SortPairs(a.cub, tb, a.rk_a, a.rk_b, a.idx_b, a.idx_a, (int)N, 0, 32, sm));
    TEMO_CUDA(cudaMemcpyAsync(keep, a.idx_a, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, sm));
    if (info) {
        TEMO_CUDA(cudaMemcpyAsync(info, a.scal, sizeof(int32_t) * 3, cudaMemcpyDeviceToDevice, sm));
        TEMO_CUDA(cudaMemcpyAsync(info + 3, w.h.ok, sizeof(int32_t), cudaMemcpyDeviceToDevice, sm));
    }
    stage_end(S_HYPE_SELECT, sm);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

extern "C" int temo_hype_select(const double *F, int64_t N, int m, int64_t n, int64_t s,
                                const double *v_ref, const int32_t *rank, const int32_t *l,
                                const temo_philox_state *st, uint64_t off, const double *U,
                                int32_t *keep, double *v_hv, int32_t *info, void *ws, size_t ws_bytes,
                                temo_stream_t stream) {
    if (!F || N < 1 || m < 1 || m > 16 || n < 1 || n > N || s < 1 || !rank || !l || !keep || !v_hv)
        return TEMO_EINVAL;
    if (!st && !U) return TEMO_EINVAL;
    if (int rc = temo_hype_select_begin(F, N, m, n, s, v_ref, rank, l, ws, ws_bytes, stream)) return rc;
    if (int rc = temo_hype_select_columns(F, N, m, s, 0, hv_columns(s), st, off, U, nullptr, ws, ws_bytes, stream))
        return rc;
    return temo_hype_select_end(F, N, m, n, s, rank, l, nullptr, keep, v_hv, info, ws, ws_bytes, stream);
}
