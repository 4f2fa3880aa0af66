// Staircase ND sort for m <= 3 (replaces the O(N^2) bitmap K1 + peel K2 of
// ndsort.cu for two and three objectives; same ranks bit for bit -- the
// fronts of a finite set are unique).  Included by ndsort.cu (base unit).
//
// After K0 the rows are in lexicographic order of their dense rank tuples and
// identical tuples form runs.  Collapse every run to one unique point k
// (k = 0..u-1 in lex order, multiplicity = run length; identical rows never
// dominate each other and share a rank).  With a = r_1, b = r_2 for m = 3
// (a = 0, b = r_1 for m = 2):
//
//     q dominates p  <=>  k_q < k_p  &&  a_q <= a_p  &&  b_q <= b_p
//
// (lex order gives column 0; distinct tuples make the <= strict somewhere).
// So p is dominated by a live point iff, over the prefix [0, k_p), the minimum
// live b among points with a <= a_p is <= b_p.  The prefix [0, k) is the union
// of the "left sibling" segments of k's binary decomposition: for every level
// j with bit j of k set, the aligned segment S = [(k >> j) - 1) << j, k >> j << j).
// Keep every aligned segment sorted by (a, k) (a merge-sort tree, built once
// per sort top down); then the live points of S with a <= a_p are a prefix of
// S's sorted order whose length kL_j(p) is static, and
//
//     dominated(p)  <=>  OR_j  prefmin_j(S)[kL_j(p) - 1] <= b_p
//
// where prefmin_j(S) is the prefix minimum of live b over S's sorted order.
// A front is then: live and not dominated.  Per front (one cooperative
// persistent kernel, two grid barriers per front, no host round trip):
//   phase A  levels j >= 11 (segments of >= 2048 points): prefix minima of the
//            live b of every left segment, per 2048-slot block (+ block minima)
//   phase B  per tile of 2048 unique points: the high-level queries (block
//            prefix + carried block minima), then levels j < 11 entirely in
//            shared memory (segmented min-scans + queries), then the front:
//            ranks, live bits, the removed points' b -> INF in the high-level
//            arrays, and the front's row count (multiplicities).
// Work per front is O(u log u) integer min/compare operations over arrays that
// stay in L2 (u = 400k: ~9 high-level arrays of 1.6 MB) instead of reading the
// front rows of an N^2/2-bit bitmap.

namespace temo {

constexpr int ST_T = 256;        // threads per CTA (8 slots / points per thread)
constexpr int ST_TILE = 2048;    // unique points per tile
constexpr int ST_LT = 11;        // log2(ST_TILE): levels below are tile-local
constexpr int ST_MAXH = 10;      // high levels (N <= 2^20 -> Lv <= 20)
constexpr uint32_t ST_INF = 0xFFFFFFFFu;

struct StairPlan {
    RankPlan k0;                 // K0 buffers (lex order, run ids, records)
    int64_t N, Np, NT;           // Np = N rounded up to ST_TILE, NT tiles
    int m, Lv, Lh;               // 2^Lv >= N levels; Lh = max(Lv - 11, 0) high levels
    int32_t *uflag, *uex, *uk, *ustart, *mult, *scal;
    uint32_t *A, *B, *E0, *E1, *iota;
    uint32_t *V, *Pl, *kLh, *posh, *agg;   // Lh x Np (agg: Lh x NT)
    int32_t *bcnt;
    uint16_t *VLg, *posl, *kLl;  // 11 x Np: live local b in slot order, slot of k, kL (tile levels)
    uint16_t *lb;                // Np: tile-local rank of b (count of smaller b in the tile)
    uint32_t *alive;             // Np / 32 words
    int32_t *rank_u, *rank_s, *fcount;
    void *cub2;
    size_t cub2_bytes, total;
};

// K0 buffers shared by every ND-sort plan
static void plan_k0(RankPlan &p, Carve &c, int64_t N, int m) {
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
    p.keys_a = c.take<uint64_t>(N);
    p.keys_b = c.take<uint64_t>(N);
    p.vals_a = c.take<int32_t>(N);
    p.vals_b = c.take<int32_t>(N);
    p.scan_a = c.take<int32_t>(N);
    p.scan_b = c.take<int32_t>(N);
    p.R = c.take<uint32_t>((size_t)N * 4 * p.NV);
    p.rec = c.take<uint4>((size_t)p.Np * p.NV);
    p.cub_tmp = c.take<char>(p.cub_bytes);
    take_k0_lanes(p, c);
}

static void plan_stair(StairPlan &s, void *base, int64_t N, int m) {
    Carve c(base);
    plan_k0(s.k0, c, N, m);
    s.N = N;
    s.m = m;
    s.Np = round_up(N, ST_TILE);
    s.NT = s.Np / ST_TILE;
    s.Lv = s.k0.bitsN;
    s.Lh = s.Lv > ST_LT ? s.Lv - ST_LT : 0;
    const int64_t Np = s.Np;
    size_t a = 0, b = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, a, (int32_t *)nullptr, (int32_t *)nullptr, (int)N);
    cub::DeviceRadixSort::SortPairs(nullptr, b, (uint32_t *)nullptr, (uint32_t *)nullptr,
                                    (uint32_t *)nullptr, (uint32_t *)nullptr, (int)Np);
    s.cub2_bytes = a > b ? a : b;
    s.uflag = c.take<int32_t>(N);
    s.uex = c.take<int32_t>(N);
    s.uk = c.take<int32_t>(N);
    s.ustart = c.take<int32_t>(Np + 1);
    s.mult = c.take<int32_t>(Np);
    s.scal = c.take<int32_t>(8);
    s.A = c.take<uint32_t>(Np);
    s.B = c.take<uint32_t>(Np);
    s.E0 = c.take<uint32_t>(Np);
    s.E1 = c.take<uint32_t>(Np);
    s.iota = c.take<uint32_t>(Np);
    const size_t H = (size_t)(s.Lh > 0 ? s.Lh : 1);
    s.V = c.take<uint32_t>(H * Np);
    s.Pl = c.take<uint32_t>(H * Np);
    s.kLh = c.take<uint32_t>(H * Np);
    s.posh = c.take<uint32_t>(H * Np);
    s.agg = c.take<uint32_t>(H * s.NT);
    s.bcnt = c.take<int32_t>(s.NT);
    s.VLg = c.take<uint16_t>((size_t)ST_LT * Np);
    s.posl = c.take<uint16_t>((size_t)ST_LT * Np);
    s.kLl = c.take<uint16_t>((size_t)ST_LT * Np);
    s.lb = c.take<uint16_t>(Np);
    s.alive = c.take<uint32_t>(Np / 32);
    s.rank_u = c.take<int32_t>(Np);
    s.rank_s = c.take<int32_t>(N);
    s.fcount = c.take<int32_t>(Np + 1);
    s.cub2 = c.take<char>(s.cub2_bytes);
    s.total = c.off;
}

// ------------------------------------------------------------ setup kernels
__global__ void k_st_uflag(const int32_t *__restrict__ runid, int64_t N, int32_t *__restrict__ flag) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p < N) flag[p] = runid[p] == (int32_t)p;
}

// unique points in lex order: a, b, first lex position; uk[p] = unique index of row p
__global__ void k_st_ufill(const uint4 *__restrict__ rec, const int32_t *__restrict__ runid,
                           const int32_t *__restrict__ flag, const int32_t *__restrict__ ex, int64_t N,
                           int m, int32_t *__restrict__ uk, uint32_t *__restrict__ A,
                           uint32_t *__restrict__ B, int32_t *__restrict__ ustart, int32_t *__restrict__ scal) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= N) return;
    const int32_t k = ex[runid[p]];
    uk[p] = k;
    if (flag[p]) {
        const uint4 r = rec[p];  // m = 3: {r1, r2, id, 0}; m = 2: {r1, id, .., ..}
        A[k] = m == 3 ? r.x : 0u;
        B[k] = m == 3 ? r.y : r.x;
        ustart[k] = (int32_t)p;
    }
    if (p == N - 1) scal[0] = ex[p] + flag[p];
}

// multiplicities, padding points k >= u (sort last, never live), iota, live bits, ranks
__global__ void k_st_upad(int64_t N, int64_t Np, int bitsN, const int32_t *__restrict__ scal,
                          uint32_t *__restrict__ A, uint32_t *__restrict__ B,
                          const int32_t *__restrict__ ustart, int32_t *__restrict__ mult,
                          uint32_t *__restrict__ iota, int32_t *__restrict__ rank_u,
                          uint32_t *__restrict__ alive) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= Np) return;
    const int64_t u = scal[0];
    if (k < u) {
        mult[k] = (int32_t)((k + 1 < u ? ustart[k + 1] : N) - ustart[k]);
    } else {
        A[k] = 1u << bitsN;
        B[k] = ST_INF;
        mult[k] = 0;
    }
    iota[k] = (uint32_t)k;
    rank_u[k] = -1;
    if ((k & 31) == 0) {
        uint32_t w = 0;
        for (int i = 0; i < 32; ++i) w |= (uint32_t)(k + i < u) << i;
        alive[k >> 5] = w;
    }
}

// CTA-wide exclusive scan (sum) of 8 values per thread (256 threads); returns the block total
__device__ __forceinline__ int st_block_scan8(int v[8], int *s_w) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int run = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int x = v[i];
        v[i] = run;
        run += x;
    }
    int inc = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(~0u, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    int wpre = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < ST_T / 32; ++w) {
        const int x = s_w[w];
        wpre += w < warp ? x : 0;
        tot += x;
    }
    const int ex = wpre + inc - run;
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] += ex;
    __syncthreads();
    return tot;
}

// high level split, pass 1: zeros (bit j of k == 0) per 2048-slot block of E_{j+1}
__global__ void __launch_bounds__(ST_T) k_st_split_count(const uint32_t *__restrict__ E, int j,
                                                        int32_t *__restrict__ bcnt) {
    const int64_t s0 = (int64_t)blockIdx.x * ST_TILE + 8 * threadIdx.x;
    const uint4 *e4 = reinterpret_cast<const uint4 *>(E + s0);
    const uint4 x = e4[0], y = e4[1];
    const uint32_t e[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
    int z = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) z += !((e[i] >> j) & 1u);
    z = __reduce_add_sync(~0u, z);
    __shared__ int s_w[ST_T / 32];
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = z;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < ST_T / 32; ++w) t += s_w[w];
        bcnt[blockIdx.x] = t;
    }
}

// high level split, pass 2: stable partition of every parent segment (2^(j+1) slots) by bit j
// of k -> E_j; kLh (left points before a right point), posh (slot of k), V (b at the slot)
__global__ void __launch_bounds__(ST_T) k_st_split_scatter(const uint32_t *__restrict__ E, int j,
                                                          const int32_t *__restrict__ bcnt,
                                                          const uint32_t *__restrict__ B,
                                                          uint32_t *__restrict__ Eo, uint32_t *__restrict__ V,
                                                          uint32_t *__restrict__ kLh, uint32_t *__restrict__ posh) {
    __shared__ int s_w[ST_T / 32];
    __shared__ int s_base;
    const int64_t blk = blockIdx.x;
    const int64_t s0 = blk * ST_TILE + 8 * threadIdx.x;
    const int64_t pstart = (blk * ST_TILE) >> (j + 1) << (j + 1);
    const int64_t pb0 = pstart / ST_TILE;
    // zeros in the parent segment's earlier blocks
    int zb = 0;
    for (int64_t b = pb0 + threadIdx.x; b < blk; b += ST_T) zb += bcnt[b];
    zb = __reduce_add_sync(~0u, zb);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = zb;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < ST_T / 32; ++w) t += s_w[w];
        s_base = t;
    }
    __syncthreads();
    const int base = s_base;
    const uint4 *e4 = reinterpret_cast<const uint4 *>(E + s0);
    const uint4 x = e4[0], y = e4[1];
    const uint32_t e[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
    int z[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) z[i] = !((e[i] >> j) & 1u);
    st_block_scan8(z, s_w);
    const int64_t half = int64_t(1) << j;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t s = s0 + i;
        const uint32_t k = e[i];
        const int64_t Z = base + z[i];  // zeros before s in the parent segment
        int64_t ns;
        if (!((k >> j) & 1u)) {
            ns = pstart + Z;
        } else {
            ns = pstart + half + (s - pstart - Z);
            kLh[k] = (uint32_t)Z;
        }
        Eo[ns] = k;
        V[ns] = B[k];
        posh[k] = (uint32_t)ns;
    }
}

// levels j < L0 (<= 11) of one tile in shared memory.  b is replaced by its tile-local
// rank lb = #{q in tile: b_q < b_k} (b_q <= b_p <=> lb_q <= lb_p inside the tile), so the
// tile levels work on u16.  Outputs per level j: kLl[j][k]; for j >= 1 also VLg[j][slot]
// (lb of the point at that slot, 0xFFFF for padding points) and posl[j][k] (its slot).
__global__ void __launch_bounds__(ST_T) k_st_local(const uint32_t *__restrict__ E, const uint32_t *__restrict__ B,
                                                  const int32_t *__restrict__ scal, int L0, int64_t Np,
                                                  uint16_t *__restrict__ VLg, uint16_t *__restrict__ posl,
                                                  uint16_t *__restrict__ kLl, uint16_t *__restrict__ lbo) {
    using Sort = cub::BlockRadixSort<uint32_t, ST_T, 8>;
    __shared__ union {
        typename Sort::TempStorage sort;
        int z[ST_TILE];
    } s_u;
    __shared__ uint16_t s_o[2][ST_TILE];
    __shared__ uint32_t s_sb[ST_TILE];
    __shared__ uint16_t s_lb[ST_TILE];
    __shared__ int s_w[ST_T / 32];
    const int64_t t0 = (int64_t)blockIdx.x * ST_TILE;
    const int64_t u = scal[0];
    const int tid = threadIdx.x;
    {  // tile-local ranks of b
        uint32_t kb[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) kb[i] = B[t0 + 8 * tid + i];
        Sort(s_u.sort).Sort(kb);  // blocked arrangement: thread tid holds ranks 8 tid .. 8 tid + 7
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 8; ++i) s_sb[8 * tid + i] = kb[i];
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int k = 8 * tid + i;
            const uint32_t v = B[t0 + k];
            int lo = 0, hi = ST_TILE;  // lower bound of v
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (s_sb[mid] < v) lo = mid + 1;
                else hi = mid;
            }
            const uint16_t r = (t0 + k < u) ? (uint16_t)lo : (uint16_t)0xFFFF;
            s_lb[k] = r;
            lbo[t0 + k] = r;
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int s = 8 * tid + i;
        s_o[0][s] = (uint16_t)(E[t0 + s] - (uint32_t)t0);
    }
    __syncthreads();
    int cur = 0;
    for (int j = L0 - 1; j >= 0; --j) {
        int z[8];
        uint16_t kk[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            kk[i] = s_o[cur][8 * tid + i];
            z[i] = !((kk[i] >> j) & 1);
        }
        // positions within the 2^(j+1) parent segments: block scan minus the value at the
        // segment start (read back through shared memory)
        st_block_scan8(z, s_w);
#pragma unroll
        for (int i = 0; i < 8; ++i) s_u.z[8 * tid + i] = z[i];
        __syncthreads();
        const int half = 1 << j;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int s = 8 * tid + i;
            const int ps = s >> (j + 1) << (j + 1);
            const int Z = z[i] - s_u.z[ps];
            int ns;
            if (!((kk[i] >> j) & 1)) {
                ns = ps + Z;
            } else {
                ns = ps + half + (s - ps - Z);
                kLl[(size_t)j * Np + t0 + kk[i]] = (uint16_t)Z;
            }
            s_o[cur ^ 1][ns] = kk[i];
            if (j >= 1) posl[(size_t)j * Np + t0 + kk[i]] = (uint16_t)ns;
        }
        __syncthreads();
        cur ^= 1;
        if (j >= 1) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int s = 8 * tid + i;
                VLg[(size_t)j * Np + t0 + s] = s_lb[s_o[cur][s]];
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------ the peel
struct StairArgs {
    const uint32_t *B;
    const int32_t *mult;
    uint32_t *V, *Pl, *agg;
    const uint32_t *kLh, *posh;
    uint16_t *VLg;
    const uint16_t *posl, *kLl, *lb;
    uint32_t *alive;
    int32_t *rank_u, *fcount;
    const int32_t *scal;
    int64_t N, Np, NT;
    int Lv, Lh, n, mode;
    int32_t *out_l, *out_nfronts, *status;
    int prof;  // diagnostics: block 0 records %globaltimer at the phase boundaries of each front
};

// per-front phase timestamps of block 0 (temo_stair_prof_*; diagnostics only)
constexpr int ST_PROF_FRONTS = 2048, ST_PROF_PTS = 8;
__device__ uint64_t g_st_prof[ST_PROF_FRONTS * ST_PROF_PTS];
static int g_st_prof_on = 0;

__device__ __forceinline__ void st_mark(const StairArgs &a, int f, int pt) {
    if (a.prof && (int)blockIdx.x == a.prof - 1 && threadIdx.x == 0 && f < ST_PROF_FRONTS) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_st_prof[f * ST_PROF_PTS + pt] = t;
    }
}

__device__ __forceinline__ uint32_t umin(uint32_t a, uint32_t b) { return a < b ? a : b; }

// inclusive min-scan of 8 consecutive values per thread over the whole CTA (2048 slots);
// returns the block minimum
__device__ __forceinline__ uint32_t st_block_minscan8(uint32_t v[8], uint32_t *s_w) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 1; i < 8; ++i) v[i] = umin(v[i], v[i - 1]);
    uint32_t inc = v[7];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(~0u, inc, o);
        if (lane >= o) inc = umin(inc, y);
    }
    uint32_t ex = __shfl_up_sync(~0u, inc, 1);
    if (lane == 0) ex = ST_INF;
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    uint32_t wpre = ST_INF, tot = ST_INF;
#pragma unroll
    for (int w = 0; w < ST_T / 32; ++w) {
        const uint32_t x = s_w[w];
        if (w < warp) wpre = umin(wpre, x);
        tot = umin(tot, x);
    }
    ex = umin(ex, wpre);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = umin(v[i], ex);
    __syncthreads();
    return tot;
}

// segmented inclusive min-scan, segments of 2^j slots (8 consecutive slots per thread)
__device__ __forceinline__ void st_seg_minscan8(uint32_t v[8], int j, uint32_t *s_w) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (j < 3) {
        const int g = 1 << j;
#pragma unroll
        for (int i = 1; i < 8; ++i)
            if (i & (g - 1)) v[i] = umin(v[i], v[i - 1]);
        return;
    }
#pragma unroll
    for (int i = 1; i < 8; ++i) v[i] = umin(v[i], v[i - 1]);
    if (j == 3) return;
    const int tps = 1 << (j - 3);  // threads per segment (2 .. 128)
    uint32_t inc = v[7];
    const int gl = tps < 32 ? tps : 32;  // lanes per warp-level group
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(~0u, inc, o);
        if (o < gl && (lane & (gl - 1)) >= o) inc = umin(inc, y);
    }
    uint32_t ex = __shfl_up_sync(~0u, inc, 1);
    if ((lane & (gl - 1)) == 0) ex = ST_INF;
    if (tps > 32) {  // segments of 2 or 4 warps
        if (lane == 31) s_w[warp] = inc;
        __syncthreads();
        const int wps = tps >> 5;
        const int w0 = warp & ~(wps - 1);
        for (int w = w0; w < warp; ++w) ex = umin(ex, s_w[w]);
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = umin(v[i], ex);
}

__device__ __forceinline__ void ld8u32(const uint32_t *p, uint32_t v[8]) {
    const uint4 x = __ldcg(reinterpret_cast<const uint4 *>(p)), y = __ldcg(reinterpret_cast<const uint4 *>(p) + 1);
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w; v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
}

__device__ __forceinline__ void ld8u16(const uint16_t *p, uint32_t v[8]) {
    const uint4 x = __ldg(reinterpret_cast<const uint4 *>(p));
    v[0] = x.x & 0xFFFF; v[1] = x.x >> 16; v[2] = x.y & 0xFFFF; v[3] = x.y >> 16;
    v[4] = x.z & 0xFFFF; v[5] = x.z >> 16; v[6] = x.w & 0xFFFF; v[7] = x.w >> 16;
}

// dynamic shared memory of k_st_peel: the tile's level data stays resident (each CTA owns
// at most one tile when the grid covers all tiles); tile levels use 16-bit local b ranks
constexpr int ST_LOWS = ST_LT - 1;  // levels 1..10 staged (level 0 is one bit per point)
constexpr int ST_MAXA = 9;          // high levels (Lv <= 20)
constexpr size_t ST_SMEM = (size_t)ST_LOWS * ST_TILE * 2 * 2   // s_VL, s_kLl (u16)
                           + 2 * ST_TILE * 2                      // s_P (u16, double buffer)
                           + 512 * 4                              // s_carry
                           + 2 * (ST_TILE / 32) * 4               // s_alive, s_k0
                           + 3 * (ST_T / 32) * 4;                 // s_w, s_red, flags

__device__ __forceinline__ void unpack8u16(const uint4 x, uint32_t v[8]) {
    v[0] = x.x & 0xFFFF; v[1] = x.x >> 16; v[2] = x.y & 0xFFFF; v[3] = x.y >> 16;
    v[4] = x.z & 0xFFFF; v[5] = x.z >> 16; v[6] = x.w & 0xFFFF; v[7] = x.w >> 16;
}

__global__ void __launch_bounds__(ST_T, 2) k_st_peel(StairArgs a) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) uint32_t st_sm[];
    uint16_t *s_VL = reinterpret_cast<uint16_t *>(st_sm);             // [10][2048] live lb by slot
    uint16_t *s_kLl = s_VL + ST_LOWS * ST_TILE;                       // [10][2048]
    uint16_t *s_P = s_kLl + ST_LOWS * ST_TILE;                        // [2][2048]
    uint32_t *s_carry = reinterpret_cast<uint32_t *>(s_P + 2 * ST_TILE);  // 512
    uint32_t *s_alive = s_carry + 512;                                // 64
    uint32_t *s_k0 = s_alive + ST_TILE / 32;                          // 64: bit k = a_{k-1} <= a_k
    uint32_t *s_w = s_k0 + ST_TILE / 32;                              // 8
    int *s_red = reinterpret_cast<int *>(s_w + ST_T / 32);            // 8
    int *s_flag = s_red + ST_T / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t u = a.scal[0];
    const int64_t NTu = (u + ST_TILE - 1) / ST_TILE;
    const int L0 = a.Lv < ST_LT ? a.Lv : ST_LT;
    int64_t ranked = 0, loaded_t = -1;
    int l = -1, f = 0;
    while (true) {
        st_mark(a, f, 0);
        // ---- phase A: block prefix minima of live b in the left segments of the high levels
        const int64_t items = (int64_t)a.Lh * NTu;
        for (int64_t it0 = blockIdx.x; it0 < items; it0 += 4 * (int64_t)gridDim.x) {
            uint32_t v[4][8];
            bool ok[4];
            int hh[4];
            int64_t bb[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int64_t it = it0 + r * (int64_t)gridDim.x;
                hh[r] = (int)(it / NTu);
                bb[r] = it - hh[r] * NTu;
                const int j = ST_LT + hh[r];
                const int64_t s0 = bb[r] * ST_TILE;
                // left segments only, and only when the right sibling holds points
                ok[r] = it < items && !((s0 >> j) & 1) && (((s0 >> j) + 1) << j) < u;
                if (ok[r]) ld8u32(a.V + (size_t)hh[r] * a.Np + s0 + 8 * tid, v[r]);
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                if (!ok[r]) continue;
                const uint32_t tot = st_block_minscan8(v[r], s_w);
                uint4 *o = reinterpret_cast<uint4 *>(a.Pl + (size_t)hh[r] * a.Np + bb[r] * ST_TILE + 8 * tid);
                __stcg(o, make_uint4(v[r][0], v[r][1], v[r][2], v[r][3]));
                __stcg(o + 1, make_uint4(v[r][4], v[r][5], v[r][6], v[r][7]));
                if (tid == 0) __stcg(a.agg + (size_t)hh[r] * a.NT + bb[r], tot);
            }
        }
        st_mark(a, f, 1);
        grid.sync();
        st_mark(a, f, 2);
        // ---- phase B: fronts of the tiles
        for (int64_t t = blockIdx.x; t < NTu; t += gridDim.x) {
            const int64_t t0 = t * ST_TILE;
            if (t != loaded_t) {  // tile level data (once per kernel when resident)
                const uint4 *gv = reinterpret_cast<const uint4 *>(a.VLg);
                const uint4 *gk = reinterpret_cast<const uint4 *>(a.kLl);
                uint4 *sv = reinterpret_cast<uint4 *>(s_VL), *sk = reinterpret_cast<uint4 *>(s_kLl);
                for (int j = 1; j < L0; ++j) {
                    const size_t g = ((size_t)j * a.Np + t0) / 8 + tid;
                    sv[(j - 1) * (ST_TILE / 8) + tid] = __ldcg(gv + g);
                    sk[(j - 1) * (ST_TILE / 8) + tid] = __ldg(gk + g);
                }
                uint32_t k0[8];
                unpack8u16(__ldg(reinterpret_cast<const uint4 *>(a.kLl + t0) + tid), k0);  // level 0 kL
                uint32_t w = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) w |= (k0[i] ? 1u : 0u) << i;
                w <<= 8 * (tid & 3);
                w |= __shfl_xor_sync(~0u, w, 1);
                w |= __shfl_xor_sync(~0u, w, 2);
                if ((tid & 3) == 0) s_k0[tid >> 2] = w;
                loaded_t = t;
            }
            if (tid < ST_TILE / 32) s_alive[tid] = __ldcg(a.alive + t0 / 32 + tid);
            if (tid == 0) *s_flag = 0;
            __syncthreads();
            if (tid < ST_TILE / 32 && s_alive[tid]) *s_flag = 1;
            __syncthreads();
            if (!*s_flag) continue;  // uniform across the CTA
            if (t == blockIdx.x) st_mark(a, f, 3);
            const uint32_t mybits = (s_alive[tid >> 2] >> (8 * (tid & 3))) & 0xFFu;  // points 8 tid + i
            uint32_t myb[8], mylb[8];
            ld8u32(a.B + t0 + 8 * tid, myb);
            unpack8u16(__ldg(reinterpret_cast<const uint4 *>(a.lb + t0) + tid), mylb);
            uint32_t dom = 0;
            // ---- high levels: the tile lies in the right segment of level 11 + h iff bit h of t is set
            const uint32_t act = (uint32_t)t & ((1u << a.Lh) - 1u);
            const int na = __popc(act);
            if (na) {
                // carried block minima of each active level's left sibling: warp w <-> w-th active level
                if (warp < na) {
                    uint32_t rest = act;
                    int off = 0;
                    for (int q = 0; q < warp; ++q) {
                        off += 1 << (__ffs(rest) - 1);
                        rest &= rest - 1;
                    }
                    const int h = __ffs(rest) - 1;
                    const int j = ST_LT + h;
                    const int nb = 1 << h;  // <= 256 blocks
                    const int64_t blk0 = ((t0 >> (j + 1)) << (j + 1)) / ST_TILE;
                    uint32_t x[8];
#pragma unroll
                    for (int r = 0; r < 8; ++r) {
                        const int c = 8 * lane + r;
                        x[r] = c < nb ? __ldcg(a.agg + (size_t)h * a.NT + blk0 + c) : ST_INF;
                    }
                    uint32_t run = ST_INF;
#pragma unroll
                    for (int r = 0; r < 8; ++r) {
                        const uint32_t y = x[r];
                        x[r] = run;
                        run = umin(run, y);
                    }
                    uint32_t inc = run;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t y = __shfl_up_sync(~0u, inc, o);
                        if (lane >= o) inc = umin(inc, y);
                    }
                    uint32_t ex = __shfl_up_sync(~0u, inc, 1);
                    if (lane == 0) ex = ST_INF;
#pragma unroll
                    for (int r = 0; r < 8; ++r)
                        if (8 * lane + r < nb) s_carry[off + 8 * lane + r] = umin(ex, x[r]);
                }
                __syncthreads();
                if (mybits) {
#pragma unroll
                    for (int half = 0; half < 2; ++half) {
                        uint32_t q[ST_MAXA][4];
                        {
                            uint32_t rest = act;
#pragma unroll
                            for (int w = 0; w < ST_MAXA; ++w) {
                                if (w < na) {
                                    const int h = __ffs(rest) - 1;
                                    rest &= rest - 1;
                                    const uint4 x = __ldg(reinterpret_cast<const uint4 *>(
                                        a.kLh + (size_t)h * a.Np + t0 + 8 * tid + 4 * half));
                                    q[w][0] = x.x; q[w][1] = x.y; q[w][2] = x.z; q[w][3] = x.w;
                                }
                            }
                        }
                        uint64_t pend = 0;
                        {
                            uint32_t rest = act;
                            int off = 0;
#pragma unroll
                            for (int w = 0; w < ST_MAXA; ++w) {
                                if (w < na) {
                                    const int h = __ffs(rest) - 1;
                                    rest &= rest - 1;
                                    const int j = ST_LT + h;
                                    const int64_t Ls = (t0 >> (j + 1)) << (j + 1);
#pragma unroll
                                    for (int i = 0; i < 4; ++i) {
                                        const int pi = 4 * half + i;
                                        const uint32_t c = q[w][i];
                                        if (!((mybits >> pi) & 1) || ((dom >> pi) & 1) || c == 0) continue;
                                        const uint32_t cv = s_carry[off + ((c - 1) >> 11)];
                                        if (cv <= myb[pi]) {
                                            dom |= 1u << pi;
                                        } else {
                                            q[w][i] = __ldcg(a.Pl + (size_t)h * a.Np + Ls + c - 1);
                                            pend |= 1ull << (4 * w + i);
                                        }
                                    }
                                    off += 1 << h;
                                }
                            }
                        }
#pragma unroll
                        for (int w = 0; w < ST_MAXA; ++w)
#pragma unroll
                            for (int i = 0; i < 4; ++i)
                                if ((pend >> (4 * w + i)) & 1) dom |= (uint32_t)(q[w][i] <= myb[4 * half + i]) << (4 * half + i);
                    }
                }
            }
            if (t == blockIdx.x) st_mark(a, f, 4);
            // ---- tile levels in shared memory (16-bit local ranks)
            if (L0 > 0 && mybits) {  // level 0: the left sibling of odd k is k - 1
#pragma unroll
                for (int i = 1; i < 8; i += 2) {
                    const int k = 8 * tid + i;
                    if (((mybits >> i) & 1) && ((mybits >> (i - 1)) & 1) && ((s_k0[k >> 5] >> (k & 31)) & 1) &&
                        mylb[i - 1] <= mylb[i])
                        dom |= 1u << i;
                }
            }
            for (int j = 1; j < L0; ++j) {
                uint16_t *P = s_P + (j & 1) * ST_TILE;
                uint32_t v[8];
                unpack8u16(reinterpret_cast<const uint4 *>(s_VL + (j - 1) * ST_TILE)[tid], v);
                st_seg_minscan8(v, j, s_w);
                reinterpret_cast<uint4 *>(P)[tid] =
                    make_uint4(v[0] | v[1] << 16, v[2] | v[3] << 16, v[4] | v[5] << 16, v[6] | v[7] << 16);
                __syncthreads();
                const bool right = j < 3 ? true : (((8 * tid) >> j) & 1);
                if (mybits && right) {
                    uint32_t kl[8];
                    unpack8u16(reinterpret_cast<const uint4 *>(s_kLl + (j - 1) * ST_TILE)[tid], kl);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int k = 8 * tid + i;
                        if (!((k >> j) & 1) || !((mybits >> i) & 1) || ((dom >> i) & 1) || kl[i] == 0) continue;
                        const int s = ((k >> (j + 1)) << (j + 1)) + (int)kl[i] - 1;
                        dom |= (uint32_t)(P[s] <= mylb[i]) << i;
                    }
                }
            }
            if (t == blockIdx.x) st_mark(a, f, 5);
            // ---- the front: live and not dominated
            const uint32_t front = mybits & ~dom;
            int cnt = 0;
            __syncthreads();  // every thread is done reading s_VL for this front
            if (front) {
#pragma unroll 1
                for (int i = 0; i < 8; ++i) {
                    if (!((front >> i) & 1)) continue;
                    const int kl = 8 * tid + i;
                    const int64_t k = t0 + kl;
                    a.rank_u[k] = f;
                    cnt += __ldg(a.mult + k);
                    // removed from every level's slot arrays: loads first, then the stores
                    uint32_t ph[ST_MAXA], pl[ST_LOWS];
#pragma unroll
                    for (int h = 0; h < ST_MAXA; ++h)
                        if (h < a.Lh && !((k >> (ST_LT + h)) & 1)) ph[h] = __ldg(a.posh + (size_t)h * a.Np + k);
#pragma unroll
                    for (int j = 1; j <= ST_LOWS; ++j)
                        if (j < L0) pl[j - 1] = __ldg(a.posl + (size_t)j * a.Np + k);
#pragma unroll
                    for (int h = 0; h < ST_MAXA; ++h)
                        if (h < a.Lh && !((k >> (ST_LT + h)) & 1)) __stcg(a.V + (size_t)h * a.Np + ph[h], ST_INF);
#pragma unroll
                    for (int j = 1; j <= ST_LOWS; ++j)
                        if (j < L0) {
                            s_VL[(j - 1) * ST_TILE + pl[j - 1]] = 0xFFFF;
                            __stcg(a.VLg + (size_t)j * a.Np + t0 + pl[j - 1], (uint16_t)0xFFFF);
                        }
                }
            }
            uint32_t w = (mybits & ~front) << (8 * (tid & 3));  // live bits: 4 threads per word
            w |= __shfl_xor_sync(~0u, w, 1);
            w |= __shfl_xor_sync(~0u, w, 2);
            if ((tid & 3) == 0) __stcg(a.alive + t0 / 32 + (tid >> 2), w);
            cnt = __reduce_add_sync(~0u, cnt);
            if (lane == 0) s_red[warp] = cnt;
            __syncthreads();
            if (tid == 0) {
                int c = 0;
                for (int q = 0; q < ST_T / 32; ++q) c += s_red[q];
                if (c) atomicAdd(a.fcount + f, c);
            }
            __syncthreads();
        }
        st_mark(a, f, 6);
        grid.sync();
        st_mark(a, f, 7);
        const int total = __ldcg(a.fcount + f);
        if (total == 0) {
            if (ranked < a.N && blockIdx.x == 0 && tid == 0) flag_status(a.status, TEMO_ST_PEEL);
            break;
        }
        ranked += total;
        if (l < 0 && ranked >= a.n) l = f;
        ++f;
        if ((a.mode == TEMO_RANK_SELECT && ranked >= a.n) || ranked >= a.N || f > a.N) break;
    }
    if (blockIdx.x == 0 && tid == 0) {
        *a.out_l = l;
        if (a.out_nfronts) *a.out_nfronts = f;
    }
}

__global__ void k_st_rank_lex(const int32_t *__restrict__ uk, const int32_t *__restrict__ rank_u, int64_t N,
                              int32_t *__restrict__ rank_s) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p < N) rank_s[p] = rank_u[uk[p]];
}

static int stair_grid(int64_t NT, int Lh) {
    static int occ = 0;
    if (!occ) {
        cudaFuncSetAttribute(k_st_peel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ST_SMEM);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_st_peel, ST_T, ST_SMEM);
        if (occ <= 0) occ = 1;
    }
    const int64_t P = (int64_t)num_sms() * occ;
    int64_t want = NT;
    if ((int64_t)Lh * NT / 2 > want) want = (int64_t)Lh * NT / 2;
    return (int)(want < P ? (want > 0 ? want : 1) : P);
}

// K0 + staircase structures + peel; ranks in original order like temo_rank's bitmap path
static int stair_rank(StairPlan &s, const double *F, int64_t n, int mode, int32_t *rank, int32_t *l_out,
                      int32_t *nfronts, int32_t *status, cudaStream_t st) {
    RankPlan &p = s.k0;
    const int64_t N = s.N, Np = s.Np;
    int rc = build_records(p, F, status, st);
    if (rc) return rc;
    stage_begin(S_DOM_BITS, st);  // the staircase structures take the place of the bitmap
    k_st_uflag<<<grid1(N), 256, 0, st>>>(p.scan_b, N, s.uflag);
    size_t tb = s.cub2_bytes;
    TEMO_CUDA(cub::DeviceScan::ExclusiveSum(s.cub2, tb, s.uflag, s.uex, (int)N, st));
    k_st_ufill<<<grid1(N), 256, 0, st>>>(p.rec, p.scan_b, s.uflag, s.uex, N, s.m, s.uk, s.A, s.B, s.ustart, s.scal);
    k_st_upad<<<grid1(Np), 256, 0, st>>>(N, Np, p.bitsN, s.scal, s.A, s.B, s.ustart, s.mult, s.iota,
                                         s.rank_u, s.alive);
    TEMO_CUDA(cudaMemsetAsync(s.fcount, 0, sizeof(int32_t) * (Np + 1), st));
    // top level: all points sorted by (a, k)
    tb = s.cub2_bytes;
    TEMO_CUDA(cub::DeviceRadixSort::SortPairs(s.cub2, tb, s.A, s.E1, s.iota, s.E0, (int)Np, 0, p.bitsN + 1,
                                              st));  // (sorted keys land in E1, overwritten below)
    uint32_t *cur = s.E0, *nxt = s.E1;
    for (int j = s.Lv - 1; j >= ST_LT; --j) {
        const int h = j - ST_LT;
        k_st_split_count<<<(unsigned)s.NT, ST_T, 0, st>>>(cur, j, s.bcnt);
        k_st_split_scatter<<<(unsigned)s.NT, ST_T, 0, st>>>(cur, j, s.bcnt, s.B, nxt, s.V + (size_t)h * Np,
                                                          s.kLh + (size_t)h * Np, s.posh + (size_t)h * Np);
        std::swap(cur, nxt);
    }
    const int L0 = s.Lv < ST_LT ? s.Lv : ST_LT;
    k_st_local<<<(unsigned)s.NT, ST_T, 0, st>>>(cur, s.B, s.scal, L0, Np, s.VLg, s.posl, s.kLl, s.lb);
    TEMO_LAUNCH_CHECK();
    stage_end(S_DOM_BITS, st);
    StairArgs a;
    a.B = s.B;
    a.mult = s.mult;
    a.V = s.V;
    a.Pl = s.Pl;
    a.agg = s.agg;
    a.kLh = s.kLh;
    a.posh = s.posh;
    a.VLg = s.VLg;
    a.posl = s.posl;
    a.kLl = s.kLl;
    a.lb = s.lb;
    a.alive = s.alive;
    a.rank_u = s.rank_u;
    a.fcount = s.fcount;
    a.scal = s.scal;
    a.N = N;
    a.Np = Np;
    a.NT = s.NT;
    a.Lv = s.Lv;
    a.Lh = s.Lh;
    a.n = (int)n;
    a.mode = mode;
    a.out_l = l_out;
    a.out_nfronts = nfronts;
    a.status = status;
    a.prof = g_st_prof_on;
    void *args[] = {&a};
    const int P = stair_grid(s.NT, s.Lh);
    stage_begin(S_PEEL, st);
    TEMO_CUDA(cudaLaunchCooperativeKernel((void *)k_st_peel, dim3(P), dim3(ST_T), args, ST_SMEM, st));
    stage_end(S_PEEL, st);
    k_st_rank_lex<<<grid1(N), 256, 0, st>>>(s.uk, s.rank_u, N, s.rank_s);
    k_unsort_ranks<<<grid1(N), 256, 0, st>>>(s.rank_s, p.vals_a, l_out, N, rank);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

// TEMO_RANK_BITMAP=1 (or temo_rank_force_bitmap(1)) keeps m <= 3 on the bitmap path (A/B comparisons)
static int g_force_bitmap = -1;
static bool stair_disabled() {
    if (g_force_bitmap < 0) {
        const char *e = getenv("TEMO_RANK_BITMAP");
        g_force_bitmap = (e && e[0] == '1') ? 1 : 0;
    }
    return g_force_bitmap == 1;
}

static bool use_stair(int m) { return (m == 2 || m == 3) && !stair_disabled(); }

}  // namespace temo

extern "C" void temo_rank_force_bitmap(int on) { temo::g_force_bitmap = on ? 1 : 0; }

extern "C" void temo_stair_prof_enable(int on) { temo::g_st_prof_on = on; }  // 1 + profiled block, 0 = off

extern "C" int temo_stair_prof_read(uint64_t *host, int64_t count) {
    if (!host || count < 0 || count > temo::ST_PROF_FRONTS * temo::ST_PROF_PTS) return TEMO_EINVAL;
    TEMO_CUDA(cudaMemcpyFromSymbol(host, temo::g_st_prof, (size_t)count * sizeof(uint64_t)));
    return TEMO_OK;
}
