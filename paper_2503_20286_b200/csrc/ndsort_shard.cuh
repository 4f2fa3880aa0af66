// Column-sharded ND sort for multi-GPU; included at the end of ndsort.cu.
//
// Every rank holds F (N x m, replicated) and runs K0 identically, so all ranks
// share the lexicographic order.  Rank g owns the sorted columns of tiles
// [jt_lo, jt_hi) (boundaries balance the triangle area, multiples of 4 tiles
// so 1024-column peel blocks never straddle shards).  K1 fills only its column
// range of the bitmap (rows i < 256 jt_hi) and the dominated-by counts of its
// columns -- no exchange.  Each front step is host driven:
//   detect : own columns with count 0 and no rank -> this rank's segment of the
//            front bitmask (sorted index space)
//   (host) : all-gather of the segments (NCCL over NVLink; N/8 bytes per front)
//   apply  : every rank ranks the whole front and subtracts the front rows' bits
//            from the counts of its own columns
// so the only per-front traffic is the N-bit front mask.

namespace temo {

struct ShardPlan {
    RankPlan k0;  // K0 buffers (bits/cnt/... of k0 unused)
    int64_t jt_lo, jt_hi, nblk_lo, nblk_hi;
    int64_t *off, *lo, *stride;
    uint32_t *bits;
    int32_t *cnt, *rank_s, *list, *wpref, *item_pref, *scal;
    uint32_t *wcnt;
    void *cub2;
    size_t cub2_bytes, total;
};

static int64_t shard_words(int64_t jt_lo, int64_t jt_hi) {
    const int64_t S0 = 8 * (jt_hi - jt_lo);
    // rows of tiles [0, jt_lo) store S0 words; tile I in [jt_lo, jt_hi) stores 8 (jt_hi - I)
    return (int64_t)TILE * (jt_lo * S0 + 8 * ((jt_hi - jt_lo) * (jt_hi - jt_lo + 1) / 2));
}

static void plan_shard(ShardPlan &s, void *base, int64_t N, int m, int64_t jt_lo, int64_t jt_hi) {
    RankPlan &p = s.k0;
    p.N = N;
    p.m = m;
    p.Np = round_up(N, 1024);
    p.W = p.Np / 32;
    p.nT = p.Np / TILE;
    p.NB = p.Np / 1024;
    p.NV = (m + 3) / 4;
    int b = 1;
    while ((int64_t(1) << b) < N) ++b;
    p.bitsN = b;
    p.cub_bytes = cub_need(N);
    s.jt_lo = jt_lo;
    s.jt_hi = jt_hi;
    s.nblk_lo = jt_lo / 4;
    s.nblk_hi = jt_hi / 4;
    const int64_t W = p.W;
    size_t c2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, c2, (uint32_t *)nullptr, (int32_t *)nullptr, (int)(W + 1));
    s.cub2_bytes = c2;
    Carve c(base);
    p.keys_a = c.take<uint64_t>(N);
    p.keys_b = c.take<uint64_t>(N);
    p.vals_a = c.take<int32_t>(N);
    p.vals_b = c.take<int32_t>(N);
    p.scan_a = c.take<int32_t>(N);
    p.scan_b = c.take<int32_t>(N);
    p.R = c.take<uint32_t>((size_t)N * 4 * p.NV);
    p.rec = c.take<uint4>((size_t)p.Np * p.NV);
    take_packed(p, c);
    p.cub_tmp = c.take<char>(p.cub_bytes);
    take_k0_lanes(p, c);
    s.off = c.take<int64_t>(p.nT + 1);
    s.lo = c.take<int64_t>(p.nT + 1);
    s.stride = c.take<int64_t>(p.nT + 1);
    s.bits = c.take<uint32_t>((size_t)shard_words(jt_lo, jt_hi));
    s.cnt = c.take<int32_t>((size_t)TILE * (jt_hi - jt_lo));
    s.rank_s = c.take<int32_t>(p.Np);
    s.list = c.take<int32_t>(p.Np);
    s.wcnt = c.take<uint32_t>(W + 1);
    s.wpref = c.take<int32_t>(W + 1);
    s.item_pref = c.take<int32_t>(p.NB + 1);
    s.scal = c.take<int32_t>(8);
    s.cub2 = c.take<char>(s.cub2_bytes);
    s.total = c.off;
}

__global__ void k_shard_offsets(int64_t nT, int64_t jt_lo, int64_t jt_hi, int64_t *off, int64_t *lo,
                                int64_t *stride) {
    const int64_t I = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (I >= nT) return;
    const int64_t S0 = 8 * (jt_hi - jt_lo);
    if (I < jt_lo) {
        off[I] = (int64_t)TILE * I * S0;
        lo[I] = 8 * jt_lo;
        stride[I] = S0;
    } else if (I < jt_hi) {
        const int64_t q = I - jt_lo;
        // sum_{t=0}^{q-1} 8 (jt_hi - jt_lo - t)
        off[I] = (int64_t)TILE * (jt_lo * S0 + 8 * (q * (jt_hi - jt_lo) - q * (q - 1) / 2));
        lo[I] = 8 * I;
        stride[I] = 8 * (jt_hi - I);
    } else {
        off[I] = 0;
        lo[I] = 8 * jt_hi;
        stride[I] = 0;
    }
}

__global__ void k_shard_init(int32_t *rank_s, int64_t N, int64_t Np, int32_t *scal) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p < Np) rank_s[p] = p < N ? -1 : 0x7FFFFFFF;
    if (p < 8) scal[p] = 0;
}

// own columns with count 0 and no rank -> segment bits (segment word 0 = column 256 jt_lo)
__global__ void k_shard_detect(const int32_t *__restrict__ cnt, const int32_t *__restrict__ rank_s,
                               int64_t N, int64_t jt_lo, int64_t jt_hi, uint32_t *__restrict__ seg,
                               int32_t *__restrict__ count) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // local column
    const int64_t ncol = (int64_t)TILE * (jt_hi - jt_lo);
    const int64_t c = (int64_t)TILE * jt_lo + q;
    const bool f = q < ncol && c < N && rank_s[c] < 0 && cnt[q] == 0;
    const uint32_t bal = __ballot_sync(~0u, f);
    if ((threadIdx.x & 31) == 0 && q < ncol) {
        seg[q >> 5] = bal;
        if (bal) atomicAdd(count, __popc(bal));
    }
}

// ranks of the front, per-word popcounts for the ordered front list
__global__ void k_shard_rank_front(const uint32_t *__restrict__ full, int64_t W, int32_t k,
                                   int32_t *__restrict__ rank_s, uint32_t *__restrict__ wcnt,
                                   int32_t *__restrict__ scal) {
    const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (w > W) return;
    if (w == W) { wcnt[w] = 0; return; }
    uint32_t x = full[w];
    wcnt[w] = __popc(x);
    if (x) atomicAdd(scal + 0, __popc(x));
    while (x) {
        const int b = __ffs(x) - 1;
        x &= x - 1;
        rank_s[w * 32 + b] = k;
    }
}

__global__ void k_shard_list(const uint32_t *__restrict__ full, const int32_t *__restrict__ wpref,
                             int64_t W, int32_t *__restrict__ list) {
    const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (w >= W) return;
    uint32_t x = full[w];
    int pos = wpref[w];
    while (x) {
        const int b = __ffs(x) - 1;
        x &= x - 1;
        list[pos++] = (int32_t)(w * 32 + b);
    }
}

// item prefix over own 1024-column blocks: rows_below(b) = wpref[32 (b+1)]
__global__ void k_shard_items(const int32_t *__restrict__ wpref, int64_t nb_lo, int64_t nb_hi,
                              int32_t *__restrict__ item_pref) {
    if (threadIdx.x || blockIdx.x) return;
    int acc = 0;
    for (int64_t b = nb_lo; b < nb_hi; ++b) {
        item_pref[b - nb_lo] = acc;
        acc += (wpref[32 * (b + 1)] + LC - 1) / LC;
    }
    item_pref[nb_hi - nb_lo] = acc;
}

// subtract the listed front rows' bits from the own columns' counts
__global__ void __launch_bounds__(PEEL_T) k_shard_subtract(
    const uint32_t *__restrict__ bits, const int64_t *__restrict__ off, const int64_t *__restrict__ lo,
    const int64_t *__restrict__ stride, const int32_t *__restrict__ list, const int32_t *__restrict__ wpref,
    const int32_t *__restrict__ item_pref, int64_t nb_lo, int64_t nb_hi, int64_t jt_lo,
    int32_t *__restrict__ cnt) {
    __shared__ uint32_t sred[8 * 8 * 32];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nb = (int)(nb_hi - nb_lo);
    const int total = item_pref[nb];
    for (int item = blockIdx.x; item < total; item += gridDim.x) {
        int l0 = 0, h0 = nb - 1;
        while (l0 < h0) {
            const int mid = (l0 + h0 + 1) >> 1;
            if (item_pref[mid] <= item) l0 = mid; else h0 = mid - 1;
        }
        const int64_t wb = nb_lo + l0;
        const int chunk = item - item_pref[l0];
        const int rows_below = wpref[32 * (wb + 1)];
        const int r0 = chunk * LC + warp * ROWS_PER_WARP;
        const int r1 = min(r0 + ROWS_PER_WARP, rows_below);
        const int64_t w = wb * 32 + lane;  // global word column
        const int rr = max(r1 - r0, 0);
        int64_t my_base = 0;
        int64_t my_w0 = INT64_MAX, my_w1 = 0;
        if (lane < rr) {
            const int i = list[r0 + lane];
            const int64_t it = i >> 8;
            my_base = off[it] + (int64_t)(i & 255) * stride[it] - lo[it];
            my_w0 = lo[it];
            my_w1 = lo[it] + stride[it];
        }
        uint32_t e0 = 0, e1 = 0, e2 = 0, e3 = 0, o0 = 0, o1 = 0, o2 = 0, o3 = 0;
        for (int g = 0; g < rr; g += 15) {
            uint32_t xs[15];
#pragma unroll
            for (int q = 0; q < 15; ++q) {
                const int64_t bb = __shfl_sync(~0u, my_base, (g + q) & 31);
                const int64_t w0 = __shfl_sync(~0u, my_w0, (g + q) & 31);
                const int64_t w1 = __shfl_sync(~0u, my_w1, (g + q) & 31);
                xs[q] = (g + q < rr && w >= w0 && w < w1) ? __ldg(bits + bb + w) : 0u;
            }
            uint32_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
            for (int q = 0; q < 15; ++q) {
                const uint32_t x = xs[q];
                a0 += x & 0x11111111u;
                a1 += (x >> 1) & 0x11111111u;
                a2 += (x >> 2) & 0x11111111u;
                a3 += (x >> 3) & 0x11111111u;
            }
            e0 += a0 & 0x0F0F0F0Fu; o0 += (a0 >> 4) & 0x0F0F0F0Fu;
            e1 += a1 & 0x0F0F0F0Fu; o1 += (a1 >> 4) & 0x0F0F0F0Fu;
            e2 += a2 & 0x0F0F0F0Fu; o2 += (a2 >> 4) & 0x0F0F0F0Fu;
            e3 += a3 & 0x0F0F0F0Fu; o3 += (a3 >> 4) & 0x0F0F0F0Fu;
        }
        uint32_t *mine = sred + warp * 8 * 32 + lane;
        mine[0 * 32] = e0; mine[1 * 32] = e1; mine[2 * 32] = e2; mine[3 * 32] = e3;
        mine[4 * 32] = o0; mine[5 * 32] = o1; mine[6 * 32] = o2; mine[7 * 32] = o3;
        __syncthreads();
        {
            const int q = tid >> 5, l = tid & 31;
            int sb[4] = {0, 0, 0, 0};  // per-byte sums over the 8 warps (each byte <= ROWS_PER_WARP)
#pragma unroll
            for (int ww = 0; ww < 8; ++ww) {
                const uint32_t v = sred[(ww * 8 + q) * 32 + l];
#pragma unroll
                for (int nbyte = 0; nbyte < 4; ++nbyte) sb[nbyte] += (v >> (8 * nbyte)) & 255;
            }
            const int64_t col = (wb * 32 + l) * 32 - (int64_t)TILE * jt_lo;  // local column
            const int kk = q & 3, half = q >> 2;
#pragma unroll
            for (int nbyte = 0; nbyte < 4; ++nbyte) {
                const int c = sb[nbyte];
                if (c) atomicSub(cnt + col + 8 * nbyte + 4 * half + kk, c);
            }
        }
        __syncthreads();
    }
}

__global__ void k_shard_finish(const int32_t *__restrict__ rank_s, const int32_t *__restrict__ order,
                               const int32_t *__restrict__ fill, int64_t N, int32_t *__restrict__ rank) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= N) return;
    const int32_t r = rank_s[p];
    // unranked rows, and (SELECT with batched fronts) rows ranked after the stop front, get fill
    rank[order[p]] = (r < 0 || r > *fill) ? *fill : r;
}

static bool shard_ok(int64_t N, int m, int64_t jt_lo, int64_t jt_hi) {
    const int64_t nT = round_up(N, 1024) / TILE;
    return N >= 1 && N <= (1 << 20) && m >= 1 && m <= MAX_M && jt_lo >= 0 && jt_lo < jt_hi &&
           jt_hi <= nT && jt_lo % 4 == 0 && jt_hi % 4 == 0;
}

}  // namespace temo

// Column-tile ranges [lo, hi) for G shards: contiguous 4-tile (1024-column) blocks,
// balancing the triangle area (block q holds 16 q + 10 tile pairs).  When there
// are fewer blocks than shards the trailing shards are empty (lo == hi).
extern "C" void temo_rank_shard_bounds(int64_t N, int G, int64_t *lo_hi) {
    const int64_t nT = round_up(N, 1024) / TILE, nq = nT / 4;
    double total = 0;
    for (int64_t q = 0; q < nq; ++q) total += 16.0 * q + 10.0;
    int64_t q = 0;
    double acc = 0;
    for (int g = 0; g < G; ++g) {
        lo_hi[2 * g] = 4 * q;
        const double target = total * (g + 1) / G;
        const int64_t keep_for_rest = (int64_t)(G - 1 - g) < nq - q ? (G - 1 - g) : 0;
        bool took = false;
        while (q < nq - keep_for_rest && (!took || acc + 16.0 * q + 10.0 <= target || g == G - 1)) {
            acc += 16.0 * q + 10.0;
            ++q;
            took = true;
        }
        lo_hi[2 * g + 1] = 4 * q;
    }
}

extern "C" size_t temo_rank_shard_ws_bytes(int64_t N, int m, int64_t jt_lo, int64_t jt_hi) {
    if (!shard_ok(N, m, jt_lo, jt_hi)) return 0;
    ShardPlan s;
    plan_shard(s, nullptr, N, m, jt_lo, jt_hi);
    return s.total;
}

#define SHARD_PLAN()                                         \
    if (!shard_ok(N, m, jt_lo, jt_hi)) return TEMO_EINVAL;   \
    ShardPlan s;                                             \
    plan_shard(s, nullptr, N, m, jt_lo, jt_hi);              \
    if (!ws || ws_bytes < s.total) return TEMO_EWORKSPACE;   \
    plan_shard(s, ws, N, m, jt_lo, jt_hi);                   \
    cudaStream_t st = (cudaStream_t)stream;

extern "C" int temo_rank_shard_build(const double *F, int64_t N, int m, int64_t jt_lo, int64_t jt_hi,
                                     int32_t *status, void *ws, size_t ws_bytes, temo_stream_t stream) {
    SHARD_PLAN();
    int rc = build_records(s.k0, F, status, st);
    if (rc) return rc;
    const int64_t nT = s.k0.nT;
    k_shard_offsets<<<grid1(nT), 256, 0, st>>>(nT, jt_lo, jt_hi, s.off, s.lo, s.stride);
    BitLayout L{jt_lo, jt_hi, s.off, s.lo, s.stride, 1};
    rc = launch_dom(s.k0, L, s.bits, s.cnt, st);
    if (rc) return rc;
    k_shard_init<<<grid1(s.k0.Np), 256, 0, st>>>(s.rank_s, N, s.k0.Np, s.scal);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

extern "C" int temo_rank_shard_detect(int64_t N, int m, int64_t jt_lo, int64_t jt_hi, uint32_t *seg,
                                      int32_t *count, void *ws, size_t ws_bytes, temo_stream_t stream) {
    SHARD_PLAN();
    TEMO_CUDA(cudaMemsetAsync(count, 0, sizeof(int32_t), st));
    const int64_t ncol = (int64_t)TILE * (jt_hi - jt_lo);
    k_shard_detect<<<grid1(ncol), 256, 0, st>>>(s.cnt, s.rank_s, N, jt_lo, jt_hi, seg, count);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

extern "C" int temo_rank_shard_apply(int64_t N, int m, int64_t jt_lo, int64_t jt_hi, const uint32_t *full,
                                     int32_t k, int32_t *front_total, void *ws, size_t ws_bytes,
                                     temo_stream_t stream) {
    SHARD_PLAN();
    const int64_t W = s.k0.W;
    TEMO_CUDA(cudaMemsetAsync(s.scal, 0, sizeof(int32_t), st));
    k_shard_rank_front<<<grid1(W + 1), 256, 0, st>>>(full, W, k, s.rank_s, s.wcnt, s.scal);
    size_t tb = s.cub2_bytes;
    TEMO_CUDA(cub::DeviceScan::ExclusiveSum(s.cub2, tb, s.wcnt, s.wpref, (int)(W + 1), st));
    k_shard_list<<<grid1(W), 256, 0, st>>>(full, s.wpref, W, s.list);
    k_shard_items<<<1, 1, 0, st>>>(s.wpref, s.nblk_lo, s.nblk_hi, s.item_pref);
    k_shard_subtract<<<num_sms() * 4, PEEL_T, 0, st>>>(s.bits, s.off, s.lo, s.stride, s.list, s.wpref,
                                                      s.item_pref, s.nblk_lo, s.nblk_hi, jt_lo, s.cnt);
    if (front_total) TEMO_CUDA(cudaMemcpyAsync(front_total, s.scal, sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

extern "C" int temo_rank_shard_finish(int64_t N, int m, int64_t jt_lo, int64_t jt_hi, const int32_t *fill,
                                      int32_t *rank, void *ws, size_t ws_bytes, temo_stream_t stream) {
    SHARD_PLAN();
    k_shard_finish<<<grid1(N), 256, 0, st>>>(s.rank_s, s.k0.vals_a, fill, N, rank);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}
