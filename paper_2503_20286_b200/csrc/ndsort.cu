// Non-dominated sorting on B200 (replaces temo ndsort.py:25-71).
//
// Pipeline (all on one stream, no host round trip):
//   K0  per-column dense ranks of the objectives (u32; -0.0 == +0.0), so every
//       dominance compare becomes an integer ISETP;
//       lexicographic sort of the rank tuples; run-start id for duplicate tuples.
//       In lex order row i can only dominate rows j > i, and for i < j
//           i dom j  <=>  id_i < id_j  &&  r_k(i) <= r_k(j)  for k = 1..m-1
//       (column 0 is implied by the order), so D is strictly upper triangular.
//   K1  k_dom_bits: 256x256 tiles of the upper triangle; lane = column j,
//       loop over rows i staged in shared memory, warp ballot -> one 32-bit
//       word of row i; rows written as a packed triangular bitmap (N^2/16 B).
//   K2  k_peel: one cooperative persistent kernel.  Dominated-by counts are a
//       vertical popcount of the bitmap (nibble-SWAR counters, coalesced 128 B
//       row segments); each front is detected (count == 0, unranked),
//       compacted in index order, and its rows' bits are subtracted from the
//       counts, front after front, with grid-wide barriers instead of host
//       round trips (ndsort.py:60-69).
#include <cooperative_groups.h>
#include <cub/cub.cuh>
#include <cstdlib>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace temo {

constexpr int TILE = 256;        // K1 tile edge (rows i and columns j)
constexpr int CHUNK = 8;         // K1: row tiles per work item
constexpr int PEEL_T = 256;      // K2 threads per CTA
constexpr int ROWS_PER_WARP = 30;       // K2 (shard path): list rows per warp per work item
constexpr int LC = 8 * ROWS_PER_WARP;    // K2 (shard path): list rows per work item (<= 255 per byte)
#ifndef PEEL_HALVES
#define PEEL_HALVES 2
#endif
constexpr int PEEL_RPW = 30 * PEEL_HALVES;  // K2: rows per warp per item, resolved 30 at a time (<= 255)
constexpr int PEEL_LC = 8 * PEEL_RPW;       // K2: rows per item (cross-warp sums unpacked to int)
constexpr int MAX_M = 16;
constexpr int K0_LANES = 3;  // K0: column rank sorts in flight at once (latency-bound at N <= 500k)

#ifndef TEMO_M_ONLY
int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}
#endif

// ------------------------------------------------------------------ plan
struct RankPlan {
    int64_t N, Np, W, nT, NB;
    int m, NV, bitsN;
    size_t cub_bytes;
    // buffers
    uint64_t *keys_a, *keys_b;
    int32_t *vals_a, *vals_b, *scan_a, *scan_b;
    uint32_t *R;       // N x MP column ranks
    uint4 *rec;        // Np x NV records in lex order
    uint32_t *lsorted; // K1 packed: sorted local rank fields per column super-tile
    uint32_t *qpk;     // K1 packed: column-pair local ranks, 16-bit halves
    int64_t *rt_off;   // nT row-tile offsets into bits
    int64_t *rt_lo;    // nT first stored word of each row tile
    int64_t *rt_stride;  // nT words per row of each row tile
    uint32_t *bits;    // packed triangular bitmap
    int32_t *cnt, *rank_s, *list, *blkcnt;
    void *cub_tmp;
    // K0 column lanes 1..K0_LANES-1 (lane 0 is keys_a .. cub_tmp above): own sort scratch,
    // so the per-column rank sorts run concurrently on side streams
    uint64_t *lk_a[K0_LANES], *lk_b[K0_LANES];
    int32_t *lv_a[K0_LANES], *lv_b[K0_LANES], *ls_a[K0_LANES], *ls_b[K0_LANES];
    void *ltmp[K0_LANES];
    size_t total;
};

// K0 lane scratch (after keys_a .. cub_tmp are carved): lane 0 aliases the main buffers
static void take_k0_lanes(RankPlan &p, Carve &c) {
    p.lk_a[0] = p.keys_a; p.lk_b[0] = p.keys_b; p.lv_a[0] = p.vals_a; p.lv_b[0] = p.vals_b;
    p.ls_a[0] = p.scan_a; p.ls_b[0] = p.scan_b; p.ltmp[0] = p.cub_tmp;
    for (int l = 1; l < K0_LANES; ++l) {
        const bool use = l < p.m;
        const int64_t n = use ? p.N : 0;
        p.lk_a[l] = c.take<uint64_t>(n);
        p.lk_b[l] = c.take<uint64_t>(n);
        p.lv_a[l] = c.take<int32_t>(n);
        p.lv_b[l] = c.take<int32_t>(n);
        p.ls_a[l] = c.take<int32_t>(n);
        p.ls_b[l] = c.take<int32_t>(n);
        p.ltmp[l] = c.take<char>(use ? p.cub_bytes : 0);
    }
}

static int64_t bitmap_words(int64_t nT, int64_t W) {
    // row tile I stores words [8I, W) for its 256 rows
    return (int64_t)TILE * (nT * W - 8 * nT * (nT - 1) / 2);
}

static size_t cub_need(int64_t N) {
    size_t a = 0, b = 0, c = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (uint64_t *)nullptr, (uint64_t *)nullptr,
                                    (int32_t *)nullptr, (int32_t *)nullptr, (int)N);
    cub::DeviceScan::InclusiveSum(nullptr, b, (int32_t *)nullptr, (int32_t *)nullptr, (int)N);
    cub::DeviceScan::InclusiveScan(nullptr, c, (int32_t *)nullptr, (int32_t *)nullptr,
                                   cub::Max(), (int)N);
    return a > b ? (a > c ? a : c) : (b > c ? b : c);
}

// K1 packed-path buffers (sizes in k_local_ranks / k_dom_packed)
static void take_packed(RankPlan &p, Carve &c) {
    const int64_t K = (p.nT + 7) / 8;  // 2048-column super-tiles
    const int FD = p.m > 1 ? p.m - 1 : 1;
    p.lsorted = c.take<uint32_t>((size_t)K * FD * 2048);
    p.qpk = c.take<uint32_t>((size_t)p.nT * 128 * FD);
}

static void plan_rank(RankPlan &p, void *base, int64_t N, int m) {
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
    p.rt_off = c.take<int64_t>(p.nT);
    p.rt_lo = c.take<int64_t>(p.nT);
    p.rt_stride = c.take<int64_t>(p.nT);
    p.bits = c.take<uint32_t>((size_t)bitmap_words(p.nT, p.W));
    p.cnt = c.take<int32_t>(p.Np);
    p.rank_s = c.take<int32_t>(p.Np);
    p.list = c.take<int32_t>(p.Np);
    p.blkcnt = c.take<int32_t>(p.NB + 1);
    p.cub_tmp = c.take<char>(p.cub_bytes);
    take_k0_lanes(p, c);
    p.total = c.off;
}

// Side streams + fork/join events of the concurrent K0 column sorts: created once per host
// thread and device (stream/event handles, no device memory); the fork/join pattern is
// legal inside CUDA-graph stream capture.  TEMO_K0_LANES=1 keeps everything on one stream.
struct K0Side {
    cudaStream_t s[K0_LANES];
    cudaEvent_t fork, join[K0_LANES];
    bool ready = false;
};

static int k0_lanes_env() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("TEMO_K0_LANES");
        v = e ? atoi(e) : K0_LANES;
        if (v < 1) v = 1;
        if (v > K0_LANES) v = K0_LANES;
    }
    return v;
}

static K0Side *k0_side() {
    thread_local K0Side side[16];
    int dev = 0;
    cudaGetDevice(&dev);
    K0Side &k = side[dev & 15];
    if (!k.ready) {
        int lo = 0, hi = 0;  // the sorts are on the critical path: highest priority
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        for (int l = 1; l < K0_LANES; ++l) {
            if (cudaStreamCreateWithPriority(&k.s[l], cudaStreamNonBlocking, hi) != cudaSuccess) return nullptr;
            if (cudaEventCreateWithFlags(&k.join[l], cudaEventDisableTiming) != cudaSuccess) return nullptr;
        }
        if (cudaEventCreateWithFlags(&k.fork, cudaEventDisableTiming) != cudaSuccess) return nullptr;
        k.ready = true;
    }
    return &k;
}

#ifndef TEMO_M_ONLY  // non-template kernels: base translation unit only
// ------------------------------------------------------------------ K0
__global__ void k_col_keys(const double *__restrict__ F, int64_t N, int m, int col,
                           uint64_t *__restrict__ keys, int32_t *__restrict__ vals,
                           int32_t *status) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    double x = F[i * m + col];
    if (isnan(x)) flag_status(status, TEMO_ST_NAN);
    keys[i] = ordered_key(x);
    vals[i] = (int32_t)i;
}

// Small-N K0 (N <= K0_SMALL_MAX, m <= 4): ranks and lexicographic order by direct counting in
// one kernel instead of m + 1 radix sorts (~40 launches, the whole cost at config A).  Ranks
// are competition ranks (#keys smaller) -- the same order and ties as dense ranks, which is
// all every consumer uses (comparisons, < 2^bitsN); the lex position of row i is the number
// of rows with a smaller key tuple, plus equal tuples with a smaller row index (stable).
constexpr int64_t K0_SMALL_MAX = 8192;

struct KeyCols {
    uint64_t *c[4];
};

__global__ void k_keys_all(const double *__restrict__ F, int64_t N, int m, KeyCols kc, int32_t *__restrict__ status) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    for (int c = 0; c < m; ++c) {
        const double x = F[i * m + c];
        if (isnan(x)) flag_status(status, TEMO_ST_NAN);
        kc.c[c][i] = ordered_key(x);
    }
}

template <int M>
__global__ void __launch_bounds__(256) k_small_k0(const KeyCols kc, int64_t N, int MP,
                                                  uint32_t *__restrict__ R, int32_t *__restrict__ order) {
    __shared__ uint64_t sk[M][256];
    const int64_t i = blockIdx.x * 256LL + threadIdx.x;
    uint64_t ki[M];
    uint32_t rk[M];
#pragma unroll
    for (int c = 0; c < M; ++c) {
        ki[c] = i < N ? kc.c[c][i] : 0ull;
        rk[c] = 0;
    }
    int64_t pos = 0;
    for (int64_t j0 = 0; j0 < N; j0 += 256) {
        __syncthreads();
#pragma unroll
        for (int c = 0; c < M; ++c) sk[c][threadIdx.x] = j0 + threadIdx.x < N ? kc.c[c][j0 + threadIdx.x] : 0ull;
        __syncthreads();
        const int jn = (int)(N - j0 < 256 ? N - j0 : 256);
        for (int jj = 0; jj < jn; ++jj) {
            bool lt_lex = false, eq_lex = true;
#pragma unroll
            for (int c = 0; c < M; ++c) {
                const uint64_t kj = sk[c][jj];
                const bool lt = kj < ki[c];
                rk[c] += lt;
                lt_lex = lt_lex || (eq_lex && lt);
                eq_lex = eq_lex && kj == ki[c];
            }
            pos += (lt_lex || (eq_lex && j0 + jj < i)) ? 1 : 0;
        }
    }
    if (i >= N) return;
#pragma unroll
    for (int c = 0; c < M; ++c) R[i * MP + c] = rk[c];
    order[pos] = (int32_t)i;
}

__global__ void k_key_change(const uint64_t *__restrict__ k, int64_t N, int32_t *__restrict__ f) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= N) return;
    f[p] = (p > 0 && k[p] != k[p - 1]) ? 1 : 0;
}

__global__ void k_scatter_rank(const int32_t *__restrict__ who, const int32_t *__restrict__ dense,
                               int64_t N, int MP, int col, uint32_t *__restrict__ R) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= N) return;
    R[(int64_t)who[p] * MP + col] = (uint32_t)dense[p];
}

__global__ void k_iota(int32_t *v, int64_t N) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p < N) v[p] = (int32_t)p;
}

// pack columns [c0, c0+g) of the rank tuple of row perm[p] into one u64 key
__global__ void k_pack_keys(const uint32_t *__restrict__ R, const int32_t *__restrict__ perm,
                            int64_t N, int MP, int c0, int g, int bits, uint64_t *__restrict__ keys) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= N) return;
    const uint32_t *r = R + (int64_t)perm[p] * MP;
    uint64_t k = 0;
    for (int c = c0; c < c0 + g; ++c) k = (k << bits) | r[c];
    keys[p] = k;
}

// v[p] = p at the start of each run of equal tuples (0 otherwise); max-scan -> run id
__global__ void k_tuple_start(const uint32_t *__restrict__ R, const int32_t *__restrict__ order,
                              int64_t N, int m, int MP, int32_t *__restrict__ v) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= N) return;
    int start = 1;
    if (p > 0) {
        const uint32_t *a = R + (int64_t)order[p] * MP;
        const uint32_t *b = R + (int64_t)order[p - 1] * MP;
        start = 0;
        for (int c = 0; c < m; ++c) start |= (a[c] != b[c]);
    }
    v[p] = start ? (int32_t)p : 0;
}

// record p (lex order): {r1, ..., r_{m-1}, id, 0 ...}; padding rows all-ones
__global__ void k_records(const uint32_t *__restrict__ R, const int32_t *__restrict__ order,
                          const int32_t *__restrict__ id, int64_t N, int64_t Np, int m, int MP,
                          int NV, uint4 *__restrict__ rec) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= Np) return;
    uint32_t f[16];
    if (p < N) {
        const uint32_t *r = R + (int64_t)order[p] * MP;
        for (int c = 0; c < 4 * NV; ++c) f[c] = c + 1 < m ? r[c + 1] : 0u;
        f[m - 1] = (uint32_t)id[p];
    } else {
        for (int c = 0; c < 4 * NV; ++c) f[c] = 0xFFFFFFFFu;
    }
    for (int v = 0; v < NV; ++v)
        rec[p * NV + v] = make_uint4(f[4 * v], f[4 * v + 1], f[4 * v + 2], f[4 * v + 3]);
}

__global__ void k_rowtile_offsets(int64_t nT, int64_t W, int64_t *off, int64_t *lo, int64_t *stride) {
    int64_t I = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (I >= nT) return;
    off[I] = (int64_t)TILE * (I * W - 8 * I * (I - 1) / 2);
    lo[I] = 8 * I;
    stride[I] = W - 8 * I;
}

#endif  // TEMO_M_ONLY

// ------------------------------------------------------------------ K1
__device__ __forceinline__ uint32_t fld(const uint4 *r, int k) {
    const uint4 v = r[k >> 2];
    switch (k & 3) {
        case 0: return v.x;
        case 1: return v.y;
        case 2: return v.z;
        default: return v.w;
    }
}

// items before strip T when strip t owns floor(t/CHUNK)+1 items
__device__ __forceinline__ int64_t items_before(int64_t T) {
    int64_t a = T / CHUNK, r = T % CHUNK;
    return T + CHUNK * a * (a - 1) / 2 + r * a;
}

// 32x32 bit transpose across a warp: lane r holds row r (bit c = element (r, c));
// returns, in lane c, the column c (bit r = element (r, c)).  Each butterfly
// stage is SHFL + one per-lane rotate + one LOP3: the rotate amount (s or 32-s)
// and the keep mask are lane constants, and wrapped-around bits always land in
// the masked-off half.
struct Transpose32 {
    uint32_t keep[5];
    uint32_t rot[5];
    __device__ __forceinline__ explicit Transpose32(int lane) {
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            const int s = 16 >> q;
            const uint32_t lowmask = q == 0 ? 0x0000FFFFu : q == 1 ? 0x00FF00FFu : q == 2 ? 0x0F0F0F0Fu
                                   : q == 3 ? 0x33333333u : 0x55555555u;
            const bool top = (lane & s) == 0;
            // opaque to the optimiser: keeps keep[] in registers (one LOP3 per stage)
            asm("mov.b32 %0, %1;" : "=r"(keep[q]) : "r"(top ? lowmask : ~lowmask));
            rot[q] = top ? s : 32 - s;
        }
    }
    __device__ __forceinline__ uint32_t operator()(uint32_t x) const {
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            const uint32_t y = __shfl_xor_sync(~0u, x, 16 >> q);
            const uint32_t t = __funnelshift_l(y, y, rot[q]);  // rotate left
            uint32_t r;  // (x & keep) | (t & ~keep)
            asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(r) : "r"(x), "r"(t), "r"(keep[q]));
            x = r;
        }
        return x;
    }
};

// K1: lane owns row i (sorted order) and walks the columns j of a 256-wide
// tile broadcast from shared memory.  With d_k = r_k(j) - r_k(i) (two's
// complement, ranks < 2^20) row i dominates j iff no d_k is negative, so one
// OR of the differences puts "not dominated" in the sign bit and a funnel
// shift collects 32 of them into a register word: per (lane, column) the
// integer subtractions issue on the FMA pipe (IMAD.IADD) and one LOP3 + one
// SHF on the ALU pipe -- no ballot, no per-pair shared-memory store.  For
// m <= 3 the columns' rank fields are packed densely in shared memory so one
// LDS.128 serves 2 (m = 3) or 4 (m = 2) columns.  Each finished word is also
// transposed across the warp and popcounted, which yields the dominated-by
// counts of the 32 columns among the warp's 32 rows (the peel's initial
// counts; no full-triangle counting pass).
// Bitmap layout: columns tiles [jt_lo, jt_hi) are stored; row tile I keeps
// words [lo_w[I], lo_w[I] + stride[I]) at bits + off[I] + r * stride[I].
// The single-GPU triangle is jt_lo = 0, jt_hi = nT, lo_w = 8 I, stride = W - 8 I;
// a column shard (multi-GPU) owns a contiguous [jt_lo, jt_hi).
struct BitLayout {
    int64_t jt_lo, jt_hi;
    const int64_t *off;
    const int64_t *lo_w;
    const int64_t *stride;
    int grid2d;  // 0: closed-form triangle items; 1: (chunk, strip) grid with early exit
};

template <int M>
__global__ void __launch_bounds__(TILE) k_dom_rows(const uint4 *__restrict__ rec, int64_t N,
                                                   int64_t nT, BitLayout L,
                                                   uint32_t *__restrict__ bits,
                                                   int32_t *__restrict__ cnt) {
    constexpr int NV = (M + 3) / 4;
    constexpr int FD = M - 1;                    // rank fields compared in disjoint tiles
    constexpr bool PACK = FD == 1 || FD == 2;    // dense packing for m = 2, 3
    __shared__ uint4 sJ[TILE * NV];
    __shared__ __align__(16) uint32_t sP[PACK ? TILE * FD : 4];
    __shared__ uint32_t sB[TILE * 9];  // row-major [i][jw], stride 9: conflict-free
    __shared__ int32_t sCnt[TILE];
    __shared__ int64_t s_it, s_chunk;
    const int tid = threadIdx.x, lane = tid & 31;
    if (!L.grid2d) {
        if (tid == 0) {
            // strip t = nT-1-I owns t+1 column tiles -> floor(t/CHUNK)+1 items
            int64_t item = blockIdx.x, lo = 0, hi = nT - 1;
            while (lo < hi) {
                int64_t mid = (lo + hi + 1) >> 1;
                if (items_before(mid) <= item) lo = mid; else hi = mid - 1;
            }
            s_it = nT - 1 - lo;
            s_chunk = item - items_before(lo);
        }
        __syncthreads();
    }
    const int64_t it = L.grid2d ? (int64_t)blockIdx.y : s_it;
    const int64_t chunk = L.grid2d ? (int64_t)blockIdx.x : s_chunk;
    const int64_t jstart = it > L.jt_lo ? it : L.jt_lo;  // first column tile of this strip
    if (jstart + chunk * CHUNK >= L.jt_hi) return;      // (grid2d) empty item
    const int64_t i = it * TILE + tid;
    // own row: negated fields so that v + n = r(j) - r(i); id field: id(j) - id(i) - 1
    uint32_t nf[4 * NV];
    {
        uint4 ri[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) ri[v] = rec[i * NV + v];
#pragma unroll
        for (int k = 0; k < 4 * NV; ++k) nf[k] = 0u - fld(ri, k);
        nf[M - 1] -= 1u;
    }
    const bool row_ok = i < N;
    const uint32_t last_i_id = fld(&rec[(it * TILE + TILE - 1) * NV], M - 1);
    const Transpose32 transpose(lane);
    const int64_t jt0 = jstart + chunk * CHUNK;
    const int64_t jt1 = min(jt0 + CHUNK, L.jt_hi);
    const int64_t row_off = L.off[it], row_lo = L.lo_w[it], row_stride = L.stride[it];
    for (int64_t jt = jt0; jt < jt1; ++jt) {
        __syncthreads();
        uint4 rv[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            rv[v] = rec[(jt * TILE + tid) * NV + v];
            sJ[tid * NV + v] = rv[v];
        }
        if (PACK) {
#pragma unroll
            for (int k = 0; k < FD; ++k) sP[tid * FD + k] = fld(rv, k);
        }
        sCnt[tid] = 0;
        __syncthreads();
        // ids of the two tiles do not overlap -> the id test is implied (and M == 1 needs it)
        const bool disjoint = M > 1 && last_i_id < fld(&sJ[0], M - 1);
        const bool last_tile = jt == nT - 1;
#pragma unroll 1
        for (int jw = 0; jw < 8; ++jw) {
            uint32_t acc = 0;
            if (disjoint && PACK) {
                const uint4 *q4 = reinterpret_cast<const uint4 *>(sP) + jw * 32 * FD / 4;
#pragma unroll
                for (int c = 0; c < 8 * FD; ++c) {
                    const uint4 v = q4[c];
                    if (FD == 2) {
                        acc = __funnelshift_l((v.x + nf[0]) | (v.y + nf[1]), acc, 1);
                        acc = __funnelshift_l((v.z + nf[0]) | (v.w + nf[1]), acc, 1);
                    } else {
                        acc = __funnelshift_l(v.x + nf[0], acc, 1);
                        acc = __funnelshift_l(v.y + nf[0], acc, 1);
                        acc = __funnelshift_l(v.z + nf[0], acc, 1);
                        acc = __funnelshift_l(v.w + nf[0], acc, 1);
                    }
                }
            } else if (disjoint) {
#pragma unroll 8
                for (int b = 0; b < 32; ++b) {
                    const uint4 *v = &sJ[(jw * 32 + b) * NV];
                    uint32_t x = 0;
#pragma unroll
                    for (int k = 0; k < M - 1; ++k) x |= fld(v, k) + nf[k];
                    acc = __funnelshift_l(x, acc, 1);
                }
            } else {
#pragma unroll 8
                for (int b = 0; b < 32; ++b) {
                    const uint4 *v = &sJ[(jw * 32 + b) * NV];
                    uint32_t x = fld(v, M - 1) + nf[M - 1];
#pragma unroll
                    for (int k = 0; k < M - 1; ++k) x |= fld(v, k) + nf[k];
                    acc = __funnelshift_l(x, acc, 1);
                }
            }
            // bit 31-b of acc = "j = 32 jw + b not dominated by i"
            uint32_t word = row_ok ? __brev(~acc) : 0u;
            if (last_tile) {  // padding columns past N
                const int64_t base = jt * TILE + 32 * jw;
                word &= base + 32 <= N ? ~0u : (base >= N ? 0u : (1u << (N - base)) - 1u);
            }
            sB[tid * 9 + jw] = word;
            const int c = __popc(transpose(word));
            if (c) atomicAdd(&sCnt[jw * 32 + lane], c);
        }
        __syncthreads();
        if (row_ok) {
            uint32_t *dst = bits + row_off + (int64_t)tid * row_stride + (8 * jt - row_lo);
            const uint32_t *s = sB + tid * 9;
            reinterpret_cast<uint4 *>(dst)[0] = make_uint4(s[0], s[1], s[2], s[3]);
            reinterpret_cast<uint4 *>(dst)[1] = make_uint4(s[4], s[5], s[6], s[7]);
        }
        const int c = sCnt[tid];
        if (c) atomicAdd(cnt + (jt - L.jt_lo) * TILE + tid, c);
    }
}

// ---------------------------------------------------------- K1 (packed)
// Two columns per integer subtraction.  Column super-tiles of SUPER = 2048
// sorted columns (8 tiles) get LOCAL ranks per rank field k:
//     q_k(j) = #{j' in super-tile : r_k(j') < r_k(j)}      (column side)
//     p_k(i) = #{j' in super-tile : r_k(j') < r_k(i)}      (row side, any i)
// and r_k(i) <= r_k(j)  <=>  p_k(i) <= q_k(j)  (if r_k(i) > r_k(j), j itself
// is counted by p but not by q).  Local ranks are < 2^12, so two columns fit
// one 32-bit word as 16-bit fields with a guard bit: (q | 0x8000) - p keeps
// bit 15 iff q >= p, and the halves never borrow from each other.  For a pair
// of columns (s, 16 + s) of a 32-column word:
//     g = AND_k ((Qpair_k | guards) - p_k * 0x10001) & 0x80008000
//     acc = (acc >> 1) + g          (16 steps; no bit ever crosses a half)
// leaves bit c of acc = "row i dominates column c" in natural order: per
// column pair (m-1) IMAD-pipe subtractions, ceil((m-1)/2) LOP3 and one LEA --
// about half the instructions of the per-column sign-bit funnel above.
constexpr int SUPER = 2048;
constexpr int SUPER_TILES = SUPER / TILE;

// lsorted[(T*FD + k)*SUPER ..] = sorted r_{k+1} of super-tile T's columns (padding: ~0u);
// qpk: per tile jt, words ((jw*16 + s)*FD + k): low half column 32jw+s, high half 32jw+16+s.
template <int FD>
__global__ void __launch_bounds__(256) k_local_ranks(const uint4 *__restrict__ rec, int64_t Np,
                                                     uint32_t *__restrict__ lsorted,
                                                     uint32_t *__restrict__ qpk) {
    constexpr int NV = (FD + 1 + 3) / 4;
    constexpr int IPT = SUPER / 256;
    using Sort = cub::BlockRadixSort<uint32_t, 256, IPT>;
    __shared__ typename Sort::TempStorage tmp;
    __shared__ uint32_t srt[SUPER];
    const int64_t T = blockIdx.x;
    const int k = blockIdx.y;
    const int tid = threadIdx.x;
    uint32_t key[IPT], mine[IPT];
#pragma unroll
    for (int t = 0; t < IPT; ++t) {
        const int64_t j = T * SUPER + tid * IPT + t;
        key[t] = j < Np ? fld(rec + j * NV, k) : 0xFFFFFFFFu;
        mine[t] = key[t];
    }
    Sort(tmp).Sort(key);
    __syncthreads();
#pragma unroll
    for (int t = 0; t < IPT; ++t) {
        srt[tid * IPT + t] = key[t];
        lsorted[((int64_t)T * FD + k) * SUPER + tid * IPT + t] = key[t];
    }
    __syncthreads();
    uint16_t *q16 = reinterpret_cast<uint16_t *>(qpk);
#pragma unroll
    for (int t = 0; t < IPT; ++t) {
        const int64_t j = T * SUPER + tid * IPT + t;
        if (j >= Np) break;
        const uint32_t v = mine[t];
        int lo = 0;  // first position with srt[pos] >= v
#pragma unroll
        for (int step = SUPER / 2; step; step >>= 1)
            if (srt[lo + step - 1] < v) lo += step;
        const int64_t jt = j / TILE;
        const int c = (int)(j % TILE), jw = c >> 5, cc = c & 31;
        const int64_t word = jt * (TILE / 2) * FD + ((jw * 16 + (cc & 15)) * FD + k);
        q16[2 * word + (cc >> 4)] = (uint16_t)(lo | 0x8000);
    }
}

// acc >> 1 plus g: LEA.HI on the ALU pipe, or mad.hi (hi32(acc * 2^31) + g) on the FMA pipe;
// alternating the two balances the ALU and FMA pipes of the packed K1 inner loop
#ifndef K1_ACC_MODE
#define K1_ACC_MODE 1
#endif
template <bool FMA>
__device__ __forceinline__ uint32_t acc_step(uint32_t acc, uint32_t g) {
    if (FMA) {
        uint32_t d;
        asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(acc), "r"(0x80000000u), "r"(g));
        return d;
    }
    return (acc >> 1) + g;
}

// lower bound count of v in a sorted SUPER-long array
__device__ __forceinline__ uint32_t count_below(const uint32_t *__restrict__ srt, uint32_t v) {
    int lo = 0;
#pragma unroll
    for (int step = SUPER / 2; step; step >>= 1)
        if (__ldg(srt + lo + step - 1) < v) lo += step;
    if (__ldg(srt + lo) < v) ++lo;  // only possible at lo == SUPER - 1
    return (uint32_t)lo;
}

// super-row a (row tiles [8a, 8a+8)) x super-tiles [a, K): items before super-row a
__device__ __forceinline__ int64_t packed_items_before(int64_t a, int64_t K) {
    return SUPER_TILES * (a * K - a * (a - 1) / 2);
}

// 8 independent 32x32 transposes interleaved stage by stage (SHFL latency hidden)
__device__ __forceinline__ void transpose8(const Transpose32 &t, uint32_t x[8]) {
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        uint32_t y[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) y[k] = __shfl_xor_sync(~0u, x[k], 16 >> q);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t r = __funnelshift_l(y[k], y[k], t.rot[q]);
            uint32_t o;
            asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(o) : "r"(x[k]), "r"(r), "r"(t.keep[q]));
            x[k] = o;
        }
    }
}

// Dynamic shared memory of k_dom_packed: sQ (all tiles of the item), sCnt, sJ (one tile)
__host__ __device__ constexpr size_t packed_smem(int M) {
    return (size_t)SUPER_TILES * (TILE / 2) * (M - 1) * 4 + SUPER_TILES * TILE * 4 +
           (size_t)TILE * ((M + 3) / 4) * 16;
}

template <int M>
__global__ void __launch_bounds__(TILE) k_dom_packed(const uint4 *__restrict__ rec,
                                                     const uint32_t *__restrict__ qpk,
                                                     const uint32_t *__restrict__ lsorted, int64_t N,
                                                     int64_t nT, BitLayout L,
                                                     uint32_t *__restrict__ bits,
                                                     int32_t *__restrict__ cnt) {
    constexpr int NV = (M + 3) / 4;
    constexpr int FD = M - 1;
    static_assert(FD >= 1, "packed K1 needs m >= 2");
    extern __shared__ __align__(16) uint32_t dsm[];
    uint32_t *sQ = dsm;                                                  // SUPER_TILES x 128 x FD
    int32_t *sCnt = reinterpret_cast<int32_t *>(dsm + SUPER_TILES * (TILE / 2) * FD);  // SUPER_TILES x 256
    uint4 *sJ = reinterpret_cast<uint4 *>(sCnt + SUPER_TILES * TILE);    // TILE x NV (general path)
    __shared__ int64_t s_it, s_T;
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t K = (nT + SUPER_TILES - 1) / SUPER_TILES;
    int64_t it, T;
    if (!L.grid2d) {
        if (tid == 0) {
            const int64_t item = blockIdx.x;
            int64_t lo = 0, hi = K - 1;
            while (lo < hi) {
                const int64_t mid = (lo + hi + 1) >> 1;
                if (packed_items_before(mid, K) <= item) lo = mid; else hi = mid - 1;
            }
            const int64_t local = item - packed_items_before(lo, K);
            s_it = SUPER_TILES * lo + local / (K - lo);
            s_T = lo + local % (K - lo);
        }
        __syncthreads();
        it = s_it;
        T = s_T;
    } else {
        it = blockIdx.y;
        T = L.jt_lo / SUPER_TILES + blockIdx.x;
    }
    if (it >= nT) return;
    int64_t jt0 = T * SUPER_TILES;
    jt0 = max(jt0, max(it, L.jt_lo));
    const int64_t jt1 = min((T + 1) * SUPER_TILES, L.jt_hi);
    if (jt0 >= jt1) return;
    const int64_t i = it * TILE + tid;
    const bool row_ok = i < N;
    uint32_t nf[4 * NV];  // general path: v + nf = r(j) - r(i) (id field: id(j) - id(i) - 1)
    uint32_t P[FD];       // packed path: local rank of r_k(i), replicated in both halves
    {
        uint4 ri[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) ri[v] = rec[i * NV + v];
#pragma unroll
        for (int k = 0; k < 4 * NV; ++k) nf[k] = 0u - fld(ri, k);
        nf[M - 1] -= 1u;
#pragma unroll
        for (int k = 0; k < FD; ++k)
            P[k] = count_below(lsorted + (T * FD + k) * SUPER, fld(ri, k)) * 0x10001u;
    }
    // stage the column-pair words of every tile of the item once; zero the counts
    const int64_t t0 = jt0 - T * SUPER_TILES, nt = jt1 - jt0;  // tile slots [t0, t0 + nt)
    {
        const uint4 *src = reinterpret_cast<const uint4 *>(qpk + jt0 * (TILE / 2) * FD);
        uint4 *dst = reinterpret_cast<uint4 *>(sQ + t0 * (TILE / 2) * FD);
        const int n4 = (int)(nt * (TILE / 2) * FD / 4);
        for (int w = tid; w < n4; w += TILE) dst[w] = src[w];
        for (int w = tid; w < SUPER_TILES * TILE; w += TILE) sCnt[w] = 0;
    }
    const uint32_t last_i_id = fld(&rec[(it * TILE + TILE - 1) * NV], M - 1);
    const Transpose32 transpose(lane);
    const int64_t row_off = L.off[it], row_lo = L.lo_w[it], row_stride = L.stride[it];
    __syncthreads();
    for (int64_t jt = jt0; jt < jt1; ++jt) {
        const int slot = (int)(jt - T * SUPER_TILES);
        // run ids of the two tiles do not overlap -> no duplicate tuples across them
        const bool disjoint = last_i_id < fld(&rec[(jt * TILE) * NV], M - 1);
        uint32_t w[8];
        if (disjoint) {
            const uint32_t *qt = sQ + slot * (TILE / 2) * FD;
#pragma unroll
            for (int jw = 0; jw < 8; ++jw) {
                uint32_t acc = 0;
                if constexpr (FD == 2) {
                    const uint4 *q4 = reinterpret_cast<const uint4 *>(qt) + jw * 8;
#pragma unroll
                    for (int s2 = 0; s2 < 8; ++s2) {
                        const uint4 v = q4[s2];
                        acc = acc_step<K1_ACC_MODE != 0>(acc, (v.x - P[0]) & (v.y - P[FD - 1]) & 0x80008000u);
                        acc = acc_step<K1_ACC_MODE == 2>(acc, (v.z - P[0]) & (v.w - P[FD - 1]) & 0x80008000u);
                    }
                } else {
                    const uint32_t *q = qt + jw * 16 * FD;
#pragma unroll
                    for (int s = 0; s < 16; ++s) {
                        uint32_t g = 0x80008000u;
#pragma unroll
                        for (int k = 0; k < FD; ++k) g &= q[s * FD + k] - P[k];
                        acc = (acc >> 1) + g;
                    }
                }
                w[jw] = acc;
            }
        } else {  // (rare) duplicate tuples may straddle the tiles: per-column test with run ids
            __syncthreads();
#pragma unroll
            for (int v = 0; v < NV; ++v) sJ[tid * NV + v] = rec[(jt * TILE + tid) * NV + v];
            __syncthreads();
#pragma unroll
            for (int jw = 0; jw < 8; ++jw) {
                uint32_t acc = 0;
#pragma unroll 4
                for (int b = 0; b < 32; ++b) {
                    const uint4 *v = &sJ[(jw * 32 + b) * NV];
                    uint32_t x = fld(v, M - 1) + nf[M - 1];
#pragma unroll
                    for (int k = 0; k < M - 1; ++k) x |= fld(v, k) + nf[k];
                    acc = __funnelshift_l(x, acc, 1);
                }
                w[jw] = __brev(~acc);
            }
        }
        const int64_t tail = N - jt * TILE;  // columns past N are masked
#pragma unroll
        for (int jw = 0; jw < 8; ++jw) {
            if (!row_ok) w[jw] = 0u;
            if (tail < TILE) {
                const int64_t base = 32 * jw;
                if (tail < base + 32) w[jw] &= tail <= base ? 0u : (1u << (tail - base)) - 1u;
            }
        }
        if (row_ok) {
            uint4 *dst = reinterpret_cast<uint4 *>(bits + row_off + (int64_t)tid * row_stride + (8 * jt - row_lo));
            dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
            dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
        }
        transpose8(transpose, w);
#pragma unroll
        for (int jw = 0; jw < 8; ++jw) atomicAdd(&sCnt[slot * TILE + jw * 32 + lane], __popc(w[jw]));
    }
    __syncthreads();
    for (int w = tid; w < nt * TILE; w += TILE) {
        const int c = sCnt[t0 * TILE + w];
        if (c) atomicAdd(cnt + (jt0 - L.jt_lo) * TILE + w, c);
    }
}

// ------------------------------------------------- K1 (packed, 8 rows/lane)
// k_dom_rows8: same packed test as k_dom_packed, but a warp owns a whole row
// tile (lane l holds rows 32 r + l, r = 0..7) and a CTA owns 4 row tiles of
// one column super-tile.  Every broadcast LDS.128 of column-pair words now
// feeds 8 rows (1 LDS per 32x32 word instead of 8), the super-tile's sorted
// rank fields are staged once per CTA for the rows' local-rank searches, and
// the column counts of the 8 row words are first summed bit-sliced per lane
// (carry-save adders -> 4 slice words) so only 4 warp transposes are needed
// per 8 row words (instead of 8).
constexpr int K1W = 4;   // warps = row tiles per CTA
#ifndef K1_JW_UNROLL
#define K1_JW_UNROLL 2
#endif
constexpr int K1_JWU = K1_JW_UNROLL;
#ifndef K1_R8_MINB
#define K1_R8_MINB 4
#endif
#ifndef K1_R8_FMA
#define K1_R8_FMA 0
#endif

constexpr int RPL = 8;   // rows per lane (TILE / 32)

// sQ | sCnt | union{ sS (sorted fields, only while the rows' local ranks are searched),
//                     sW (per warp 256 rows x 9 words: row words staged for 32-byte stores) }
__host__ __device__ constexpr size_t rows8_union(int M) {
    return (size_t)(M - 1) * SUPER * 4 > (size_t)K1W * TILE * 9 * 4 ? (size_t)(M - 1) * SUPER * 4
                                                                    : (size_t)K1W * TILE * 9 * 4;
}
__host__ __device__ constexpr size_t rows8_smem(int M) {
    return (size_t)SUPER_TILES * (TILE / 2) * (M - 1) * 4 + (size_t)SUPER_TILES * TILE * 4 + rows8_union(M);
}

__device__ __forceinline__ uint32_t count_below_s(const uint32_t *srt, uint32_t v) {
    int lo = 0;
#pragma unroll
    for (int step = SUPER / 2; step; step >>= 1)
        if (srt[lo + step - 1] < v) lo += step;
    if (srt[lo] < v) ++lo;
    return (uint32_t)lo;
}

// bit-sliced sum of 8 words: bit j of out[b] = bit b of (number of inputs with bit j set)
__device__ __forceinline__ void csa8(const uint32_t x[8], uint32_t out[4]) {
    auto fa = [](uint32_t a, uint32_t b, uint32_t c, uint32_t &sum, uint32_t &car) {
        sum = a ^ b ^ c;
        car = (a & b) | (c & (a ^ b));
    };
    uint32_t s1, c1, s2, c2, s3, c3, s5, c5;
    fa(x[0], x[1], x[2], s1, c1);
    fa(x[3], x[4], x[5], s2, c2);
    fa(s1, s2, x[6], s3, c3);
    out[0] = s3 ^ x[7];
    const uint32_t c4 = s3 & x[7];
    fa(c1, c2, c3, s5, c5);
    out[1] = s5 ^ c4;
    const uint32_t c6 = s5 & c4;
    out[2] = c5 ^ c6;
    out[3] = c5 & c6;
}

__device__ __forceinline__ void transpose4(const Transpose32 &t, uint32_t x[4]) {
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        uint32_t y[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) y[k] = __shfl_xor_sync(~0u, x[k], 16 >> q);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t r = __funnelshift_l(y[k], y[k], t.rot[q]);
            uint32_t o;
            asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(o) : "r"(x[k]), "r"(r), "r"(t.keep[q]));
            x[k] = o;
        }
    }
}

template <int M>
__global__ void __launch_bounds__(K1W * 32, K1_R8_MINB) k_dom_rows8(const uint4 *__restrict__ rec,
                                                           const uint32_t *__restrict__ qpk,
                                                           const uint32_t *__restrict__ lsorted,
                                                           int64_t N, int64_t nT, BitLayout L,
                                                           uint32_t *__restrict__ bits,
                                                           int32_t *__restrict__ cnt) {
    constexpr int NV = (M + 3) / 4;
    constexpr int FD = M - 1;
    static_assert(FD >= 1, "packed K1 needs m >= 2");
    extern __shared__ __align__(16) uint32_t dsm[];
    uint32_t *sQ = dsm;                                                         // SUPER_TILES x 128 x FD
    int32_t *sCnt = reinterpret_cast<int32_t *>(sQ + SUPER_TILES * (TILE / 2) * FD);  // SUPER_TILES x TILE
    uint32_t *sS = reinterpret_cast<uint32_t *>(sCnt + SUPER_TILES * TILE);    // FD x SUPER (phase 1)
    uint32_t *sW = sS;                                                          // K1W x TILE x 9 (phase 2)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int64_t T, g;
    if (!L.grid2d) {
        // super-tile T has 2T + 2 items (row-tile groups) -> items before T = T (T + 1)
        const int64_t item = blockIdx.x;
        int64_t t = (int64_t)((sqrt(4.0 * (double)item + 1.0) - 1.0) * 0.5);
        while (t * (t + 1) > item) --t;
        while ((t + 1) * (t + 2) <= item) ++t;
        T = t;
        g = item - t * (t + 1);
    } else {
        T = L.jt_lo / SUPER_TILES + blockIdx.x;
        g = blockIdx.y;
    }
    const int64_t ct0 = max(T * SUPER_TILES, L.jt_lo);                // column tiles of the CTA
    const int64_t ct1 = min(min((T + 1) * SUPER_TILES, L.jt_hi), nT);
    const int64_t it0 = g * K1W;
    if (ct0 >= ct1 || it0 >= ct1) return;
    {
        const int64_t s0 = ct0 - T * SUPER_TILES;
        const uint4 *src = reinterpret_cast<const uint4 *>(qpk + ct0 * (TILE / 2) * FD);
        uint4 *dst = reinterpret_cast<uint4 *>(sQ + s0 * (TILE / 2) * FD);
        const int n4 = (int)((ct1 - ct0) * (TILE / 2) * FD / 4);
        for (int w = tid; w < n4; w += K1W * 32) dst[w] = src[w];
        const uint4 *ss = reinterpret_cast<const uint4 *>(lsorted + T * FD * SUPER);
        uint4 *sd = reinterpret_cast<uint4 *>(sS);
        for (int w = tid; w < FD * SUPER / 4; w += K1W * 32) sd[w] = ss[w];
        for (int w = tid; w < SUPER_TILES * TILE; w += K1W * 32) sCnt[w] = 0;
    }
    __syncthreads();
    const int64_t it = it0 + warp;
    const int64_t jt0 = max(ct0, it), jt1 = ct1;
    const bool active = it < nT && jt0 < jt1;
    // this lane's rows it*256 + 32 r + lane: local ranks (both halves) and validity
    uint32_t P[RPL][FD];
    uint32_t row_ok = 0;
    if (active) {
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
            const int64_t i = it * TILE + 32 * r + lane;
            row_ok |= (uint32_t)(i < N) << r;
            uint4 ri[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) ri[v] = rec[i * NV + v];
#pragma unroll
            for (int k = 0; k < FD; ++k) P[r][k] = count_below_s(sS + k * SUPER, fld(ri, k)) * 0x10001u;
        }
    }
    __syncthreads();  // sS is dead from here on; its space becomes sW
    if (active) {
        const uint32_t last_i_id = fld(&rec[(it * TILE + TILE - 1) * NV], M - 1);
        const Transpose32 transpose(lane);
        const int64_t row_off = L.off[it], row_lo = L.lo_w[it], row_stride = L.stride[it];
        for (int64_t jt = jt0; jt < jt1; ++jt) {
            const int slot = (int)(jt - T * SUPER_TILES);
            const bool disjoint = last_i_id < fld(&rec[(jt * TILE) * NV], M - 1);
            const int64_t tail = N - jt * TILE;  // columns past N are masked
            const uint32_t *qt = sQ + slot * (TILE / 2) * FD;
            const uint4 *sj = rec + jt * TILE * NV;  // (rare path) column records straight from L1/L2
            uint32_t *sw = sW + warp * TILE * 9 + lane * 9;  // row 32 r + lane at sw + 32 * 9 r
#pragma unroll K1_JWU
            for (int jw = 0; jw < 8; ++jw) {
                uint32_t acc[RPL];
#pragma unroll
                for (int r = 0; r < RPL; ++r) acc[r] = 0;
                if (disjoint) {
                    if constexpr (FD == 2) {
                        const uint4 *q4 = reinterpret_cast<const uint4 *>(qt) + jw * 8;
#pragma unroll
                        for (int s2 = 0; s2 < 8; ++s2) {
                            const uint4 v = q4[s2];
#pragma unroll
                            for (int r = 0; r < RPL; ++r) {
                                acc[r] = acc_step<K1_R8_FMA >= 2>(acc[r], (v.x - P[r][0]) & (v.y - P[r][FD - 1]) & 0x80008000u);
                                acc[r] = acc_step<K1_R8_FMA >= 1>(acc[r], (v.z - P[r][0]) & (v.w - P[r][FD - 1]) & 0x80008000u);
                            }
                        }
                    } else {
                        const uint32_t *q = qt + jw * 16 * FD;
#pragma unroll
                        for (int st = 0; st < 16; ++st) {
                            uint32_t qv[FD];
#pragma unroll
                            for (int k = 0; k < FD; ++k) qv[k] = q[st * FD + k];
#pragma unroll
                            for (int r = 0; r < RPL; ++r) {
                                uint32_t gg = 0x80008000u;
#pragma unroll
                                for (int k = 0; k < FD; ++k) gg &= qv[k] - P[r][k];
                                acc[r] = acc_step<false>(acc[r], gg);
                            }
                        }
                    }
                } else {
#pragma unroll 1
                    for (int r = 0; r < RPL; ++r) {
                        const int64_t i = it * TILE + 32 * r + lane;
                        uint32_t nf[4 * NV];
                        uint4 ri[NV];
#pragma unroll
                        for (int v = 0; v < NV; ++v) ri[v] = rec[i * NV + v];
#pragma unroll
                        for (int k = 0; k < 4 * NV; ++k) nf[k] = 0u - fld(ri, k);
                        nf[M - 1] -= 1u;
                        uint32_t a = 0;
#pragma unroll 4
                        for (int b = 0; b < 32; ++b) {
                            const uint4 *v = &sj[(jw * 32 + b) * NV];
                            uint32_t x = fld(v, M - 1) + nf[M - 1];
#pragma unroll
                            for (int k = 0; k < M - 1; ++k) x |= fld(v, k) + nf[k];
                            a = __funnelshift_l(x, a, 1);
                        }
#pragma unroll
                        for (int r2 = 0; r2 < RPL; ++r2)
                            if (r2 == r) acc[r2] = __brev(~a);
                    }
                }
                // masks: rows past N, columns past N (only the last row/column tiles need them)
                if (tail < TILE || row_ok != 0xFFu) {
                    uint32_t cm = ~0u;
                    if (tail < TILE) {
                        const int64_t base = 32 * jw;
                        if (tail < base + 32) cm = tail <= base ? 0u : (1u << (tail - base)) - 1u;
                    }
#pragma unroll
                    for (int r = 0; r < RPL; ++r) acc[r] &= ((row_ok >> r) & 1) ? cm : 0u;
                }
#pragma unroll
                for (int r = 0; r < RPL; ++r) sw[32 * 9 * r + jw] = acc[r];
                // column counts over the warp's 256 rows: bit-sliced sum of 8 rows, 4 transposes
                uint32_t sl[4];
                csa8(acc, sl);
                transpose4(transpose, sl);
                const int c = __popc(sl[0]) + 2 * __popc(sl[1]) + 4 * __popc(sl[2]) + 8 * __popc(sl[3]);
                atomicAdd(&sCnt[slot * TILE + jw * 32 + lane], c);
            }
            __syncwarp();
            // each lane writes its 8 rows' 8 words for this tile as two 16-byte stores per row
            uint32_t *rowp = bits + row_off + (int64_t)lane * row_stride + (8 * jt - row_lo);
#pragma unroll
            for (int r = 0; r < RPL; ++r) {
                const uint32_t *x = sw + 32 * 9 * r;
                if ((row_ok >> r) & 1) {
                    uint4 *dst = reinterpret_cast<uint4 *>(rowp + (int64_t)(32 * r) * row_stride);
                    dst[0] = make_uint4(x[0], x[1], x[2], x[3]);
                    dst[1] = make_uint4(x[4], x[5], x[6], x[7]);
                }
            }
            __syncwarp();
        }
    }
    __syncthreads();
    const int64_t s0 = ct0 - T * SUPER_TILES;
    for (int w = tid; w < (ct1 - ct0) * TILE; w += K1W * 32) {
        const int c = sCnt[s0 * TILE + w];
        if (c) atomicAdd(cnt + (ct0 - L.jt_lo) * TILE + w, c);
    }
}

// ------------------------------------------------------ per-M K1 launchers
// build.py compiles this file as a base unit plus one unit per objective count
// (-DTEMO_M_ONLY=M), each instantiating only its dom_m<M>.
// TEMO_K1_UNPACKED=1 selects the per-column sign-bit kernel (A/B comparisons)
static bool packed_disabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("TEMO_K1_UNPACKED");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

// TEMO_K1_ROWS8=0 selects the 1-row-per-lane packed kernel (A/B comparisons)
static bool rows8_disabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("TEMO_K1_ROWS8");
        v = (e && e[0] == '0') ? 1 : 0;
    }
    return v == 1;
}

template <int M>
int dom_m(const RankPlan &p, const BitLayout &L, uint32_t *bits, int32_t *cnt, cudaStream_t st) {
    const uint4 *rec = p.rec;
    const int64_t N = p.N, nT = p.nT;
    if constexpr (M >= 2) {
        if (!packed_disabled()) {
            const int64_t K = (nT + SUPER_TILES - 1) / SUPER_TILES;
            dim3 g;
            if (L.grid2d) {
                const int64_t T0 = L.jt_lo / SUPER_TILES, T1 = (L.jt_hi + SUPER_TILES - 1) / SUPER_TILES;
                g = dim3((unsigned)(T1 - T0), (unsigned)L.jt_hi);
            } else {
                g = dim3((unsigned)(SUPER_TILES * (K * (K + 1) / 2)));
            }
            TEMO_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * TILE * (L.jt_hi - L.jt_lo), st));
            k_local_ranks<M - 1><<<dim3((unsigned)K, M - 1), 256, 0, st>>>(rec, p.Np, p.lsorted, p.qpk);
            if (M <= 5 && !rows8_disabled()) {
                dim3 g8;
                if (L.grid2d) {
                    const int64_t T0 = L.jt_lo / SUPER_TILES, T1 = (L.jt_hi + SUPER_TILES - 1) / SUPER_TILES;
                    g8 = dim3((unsigned)(T1 - T0), (unsigned)((L.jt_hi + K1W - 1) / K1W));
                } else {
                    g8 = dim3((unsigned)(K * (K + 1)));
                }
                if (rows8_smem(M) > 48 * 1024)
                    TEMO_CUDA(cudaFuncSetAttribute(k_dom_rows8<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)rows8_smem(M)));
                k_dom_rows8<M><<<g8, K1W * 32, rows8_smem(M), st>>>(rec, p.qpk, p.lsorted, N, nT, L, bits, cnt);
                return TEMO_OK;
            }
            if (packed_smem(M) > 48 * 1024)
                TEMO_CUDA(cudaFuncSetAttribute(k_dom_packed<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)packed_smem(M)));
            k_dom_packed<M><<<g, TILE, packed_smem(M), st>>>(rec, p.qpk, p.lsorted, N, nT, L, bits, cnt);
            return TEMO_OK;
        }
    }
    dim3 g;
    if (L.grid2d) {
        g = dim3((unsigned)((L.jt_hi - L.jt_lo + CHUNK - 1) / CHUNK), (unsigned)L.jt_hi);
    } else {
        g = dim3((unsigned)(nT + CHUNK * ((nT / CHUNK) * ((nT / CHUNK) - 1) / 2) + (nT % CHUNK) * (nT / CHUNK)));
    }
    TEMO_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * TILE * (L.jt_hi - L.jt_lo), st));
    k_dom_rows<M><<<g, TILE, 0, st>>>(rec, N, nT, L, bits, cnt);
    return TEMO_OK;
}

#define TEMO_ND_M_LIST(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16)
#define TEMO_ND_DECL(MM, EXT) \
    EXT template int dom_m<MM>(const RankPlan &, const BitLayout &, uint32_t *, int32_t *, cudaStream_t);
#ifdef TEMO_M_ONLY
TEMO_ND_DECL(TEMO_M_ONLY, )
}  // namespace temo
#else
#define TEMO_ND_EXTERN(MM) TEMO_ND_DECL(MM, extern)
TEMO_ND_EXTERN(2) TEMO_ND_EXTERN(3) TEMO_ND_EXTERN(4) TEMO_ND_EXTERN(5) TEMO_ND_EXTERN(6) TEMO_ND_EXTERN(7)
TEMO_ND_EXTERN(8) TEMO_ND_EXTERN(9) TEMO_ND_EXTERN(10) TEMO_ND_EXTERN(11) TEMO_ND_EXTERN(12)
TEMO_ND_EXTERN(13) TEMO_ND_EXTERN(14) TEMO_ND_EXTERN(15) TEMO_ND_EXTERN(16)
TEMO_ND_DECL(1, )  // m = 1 (per-column path only) lives in the base unit

// ------------------------------------------------------------------ K2
struct PeelArgs {
    const uint32_t *bits;
    const int64_t *rt_off;
    int64_t W;
    int N, NB, n, mode;
    int32_t *cnt, *rank_s, *list, *blkcnt;
    int32_t *out_l, *out_nfronts, *status;
};

// in-place exclusive scan of s[0..len) (len <= 4096) by one CTA of PEEL_T threads;
// returns the total.  Uses `tmp` (PEEL_T/32 ints).
__device__ int block_exclusive_scan(int *s, int len, int *tmp) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per = (len + PEEL_T - 1) / PEEL_T;
    const int lo = tid * per, hi = min(lo + per, len);
    int sum = 0;
    for (int q = lo; q < hi; ++q) sum += s[q];
    int incl = sum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        int y = __shfl_up_sync(~0u, incl, d);
        if (lane >= d) incl += y;
    }
    if (lane == 31) tmp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int v = lane < PEEL_T / 32 ? tmp[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            int y = __shfl_up_sync(~0u, v, d);
            if (lane >= d) v += y;
        }
        if (lane < PEEL_T / 32) tmp[lane] = v;
    }
    __syncthreads();
    int run = incl - sum + (warp ? tmp[warp - 1] : 0);
    const int total = tmp[PEEL_T / 32 - 1];
    for (int q = lo; q < hi; ++q) {
        int v = s[q];
        s[q] = run;
        run += v;
    }
    __syncthreads();
    return total;
}

// Subtract (sign=-1) or add (sign=+1) the bits of listed rows into cnt.
// rows_below[wb] (wb < NB) = number of list rows with index < 1024*(wb+1);
// item_pref = exclusive prefix of ceil(rows_below/LC).
__device__ void vertical_pass(const PeelArgs &a, const int *rows_below, const int *item_pref,
                              bool identity, int sign, uint32_t *sred) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int total = item_pref[a.NB];
    for (int item = blockIdx.x; item < total; item += gridDim.x) {
        int lo = 0, hi = a.NB - 1;
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (item_pref[mid] <= item) lo = mid; else hi = mid - 1;
        }
        const int wb = lo;
        const int chunk = item - item_pref[wb];
        const int rw0 = chunk * PEEL_LC + warp * PEEL_RPW;
        const int rw1 = min(rw0 + PEEL_RPW, rows_below[wb]);
        const int64_t w = (int64_t)wb * 32 + lane;
        uint32_t e0 = 0, e1 = 0, e2 = 0, e3 = 0, o0 = 0, o1 = 0, o2 = 0, o3 = 0;
        for (int r0 = rw0; r0 < rw1; r0 += 30) {  // 30 rows per round: one row per lane
            const int rr = min(30, rw1 - r0);
            // lane k resolves row r0+k once (list entry, row base address, first stored
            // word); the row loop then only shuffles and issues independent loads
            int64_t my_base = 0;
            int my_w0 = 0x7FFFFFFF;
            if (lane < rr) {
                const int i = identity ? r0 + lane : a.list[r0 + lane];
                const int64_t it = i >> 8;
                my_base = a.rt_off[it] + (int64_t)(i & 255) * (a.W - 8 * it) - 8 * it;
                my_w0 = (int)(8 * it);
            }
            for (int g = 0; g < rr; g += 15) {
                uint32_t xs[15];
#pragma unroll
                for (int q = 0; q < 15; ++q) {
                    const int64_t b = __shfl_sync(~0u, my_base, (g + q) & 31);
                    const int w0 = __shfl_sync(~0u, my_w0, (g + q) & 31);
                    xs[q] = (g + q < rr && w >= w0) ? __ldg(a.bits + b + w) : 0u;
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
        }
        uint32_t *mine = sred + warp * 8 * 32 + lane;
        mine[0 * 32] = e0; mine[1 * 32] = e1; mine[2 * 32] = e2; mine[3 * 32] = e3;
        mine[4 * 32] = o0; mine[5 * 32] = o1; mine[6 * 32] = o2; mine[7 * 32] = o3;
        __syncthreads();
        {
            const int q = tid >> 5, l = tid & 31;  // q: which byte register, l: word column
            int sb[4] = {0, 0, 0, 0};  // per-byte sums over the 8 warps (each byte <= ROWS_PER_WARP)
#pragma unroll
            for (int ww = 0; ww < 8; ++ww) {
                const uint32_t v = sred[(ww * 8 + q) * 32 + l];
#pragma unroll
                for (int nb = 0; nb < 4; ++nb) sb[nb] += (v >> (8 * nb)) & 255;
            }
            const int64_t col = ((int64_t)wb * 32 + l) * 32;
            const int kk = q & 3, half = q >> 2;
#pragma unroll
            for (int nb = 0; nb < 4; ++nb) {
                const int c = sb[nb];
                if (c) atomicAdd(a.cnt + col + 8 * nb + 4 * half + kk, sign * c);
            }
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(PEEL_T) k_peel(PeelArgs a) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ int psm[];
    int *s_rows = psm;                 // NB + 1
    int *s_items = psm + (a.NB + 1);   // NB + 1
    int *s_tmp = s_items + (a.NB + 1); // 32
    uint32_t *sred = reinterpret_cast<uint32_t *>(s_tmp + 32);  // 8*8*32
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    // initial dominated-by counts come from K1 (column popcounts of each tile)

    int ranked = 0, l = -1, k = 0;
    while (true) {
        // A1: front rows per 1024-row block
        for (int wb = blockIdx.x; wb < a.NB; wb += gridDim.x) {
            int c = 0;
            for (int t = tid; t < 1024; t += PEEL_T) {
                const int i = wb * 1024 + t;
                c += (i < a.N && a.rank_s[i] < 0 && a.cnt[i] == 0);
            }
            c = __reduce_add_sync(~0u, c);
            if (lane == 0) s_tmp[warp] = c;
            __syncthreads();
            if (tid == 0) {
                int s = 0;
                for (int q = 0; q < PEEL_T / 32; ++q) s += s_tmp[q];
                a.blkcnt[wb] = s;
            }
            __syncthreads();
        }
        grid.sync();
        // A2: ordered compaction of the front, ranks := k
        for (int wb = tid; wb <= a.NB; wb += PEEL_T) s_rows[wb] = wb < a.NB ? a.blkcnt[wb] : 0;
        __syncthreads();
        const int total = block_exclusive_scan(s_rows, a.NB + 1, s_tmp);  // s_rows[wb] = start
        if (total == 0) {
            if (ranked < a.N && blockIdx.x == 0 && tid == 0) flag_status(a.status, TEMO_ST_PEEL);
            break;
        }
        for (int wb = blockIdx.x; wb < a.NB; wb += gridDim.x) {
            int base = s_rows[wb];
            for (int t0 = 0; t0 < 1024; t0 += PEEL_T) {
                const int i = wb * 1024 + t0 + tid;
                const bool f = i < a.N && a.rank_s[i] < 0 && a.cnt[i] == 0;
                const uint32_t bal = __ballot_sync(~0u, f);
                if (lane == 0) s_tmp[warp] = __popc(bal);
                __syncthreads();
                int before = 0, chunk_total = 0;
                for (int q = 0; q < PEEL_T / 32; ++q) {
                    before += q < warp ? s_tmp[q] : 0;
                    chunk_total += s_tmp[q];
                }
                if (f) {
                    a.list[base + before + __popc(bal & ((1u << lane) - 1))] = i;
                    a.rank_s[i] = k;
                }
                base += chunk_total;
                __syncthreads();
            }
        }
        ranked += total;
        if (l < 0 && ranked >= a.n) l = k;
        ++k;
        if ((a.mode == TEMO_RANK_SELECT && ranked >= a.n) || ranked >= a.N || k > a.N) break;
        grid.sync();
        // B: subtract the front's bits.  s_rows holds exclusive starts with
        // s_rows[NB] = total, so rows_below(wb) = s_rows[wb + 1].
        for (int wb = tid; wb <= a.NB; wb += PEEL_T)
            s_items[wb] = wb < a.NB ? (s_rows[wb + 1] + PEEL_LC - 1) / PEEL_LC : 0;
        __syncthreads();
        block_exclusive_scan(s_items, a.NB + 1, s_tmp);
        vertical_pass(a, s_rows + 1, s_items, false, -1, sred);
        grid.sync();
    }
    if (blockIdx.x == 0 && tid == 0) {
        *a.out_l = l;
        if (a.out_nfronts) *a.out_nfronts = k;
    }
}

__global__ void k_peel_init(int32_t *rank_s, int32_t *cnt, int64_t N, int64_t Np) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= Np) return;
    rank_s[p] = p < N ? -1 : 0x7FFFFFFF;
    (void)cnt;  // counts were produced by K1
}

__global__ void k_unsort_ranks(const int32_t *__restrict__ rank_s, const int32_t *__restrict__ order,
                               const int32_t *__restrict__ l, int64_t N, int32_t *__restrict__ rank) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= N) return;
    const int32_t r = rank_s[p];
    rank[order[p]] = r < 0 ? *l + 1 : r;
}

// expand the packed bitmap to the dense N x ceil(N/32) layout of original indices
__global__ void k_expand_dense(const uint32_t *__restrict__ bits, const int64_t *__restrict__ rt_off,
                               int64_t W, const int32_t *__restrict__ pos, int64_t N, int64_t Wd,
                               uint32_t *__restrict__ D) {
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= N * Wd) return;
    const int64_t i = q / Wd, jw = q % Wd;
    const int64_t pi = pos[i], it = pi >> 8;
    uint32_t word = 0;
    for (int b = 0; b < 32; ++b) {
        const int64_t j = jw * 32 + b;
        if (j >= N) break;
        const int64_t pj = pos[j];
        if (pj <= pi) continue;
        const int64_t w = pj >> 5;
        const uint32_t x = bits[rt_off[it] + (pi & 255) * (W - 8 * it) + (w - 8 * it)];
        word |= ((x >> (pj & 31)) & 1u) << b;
    }
    D[q] = word;
}

__global__ void k_inverse(const int32_t *__restrict__ order, int64_t N, int32_t *__restrict__ pos) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p < N) pos[order[p]] = (int32_t)p;
}

// ------------------------------------------------------------------ host
static inline dim3 grid1(int64_t n, int t = 256) { return dim3((unsigned)((n + t - 1) / t)); }

// K0: column ranks, lex order (p.vals_a), run ids and records (p.rec)
static int build_records(RankPlan &p, const double *F, int32_t *status, cudaStream_t st) {
    const int64_t N = p.N;
    const int m = p.m, MP = 4 * p.NV;
    size_t tb = p.cub_bytes;
    stage_begin(S_RANK_PREP, st);
    // key columns 2, 3 of the small path live in the (unused here) radix-sort scratch
    const bool small = N <= K0_SMALL_MAX && m >= 2 && m <= 4 && p.cub_bytes >= (size_t)(2 * N) * sizeof(uint64_t);
    if (small) {  // one counting kernel instead of m + 1 radix sorts
        KeyCols kc;
        kc.c[0] = p.keys_a;
        kc.c[1] = p.keys_b;
        kc.c[2] = static_cast<uint64_t *>(p.cub_tmp);
        kc.c[3] = static_cast<uint64_t *>(p.cub_tmp) + N;
        k_keys_all<<<grid1(N), 256, 0, st>>>(F, N, m, kc, status);
        const unsigned gb = (unsigned)((N + 255) / 256);
        if (m == 2) k_small_k0<2><<<gb, 256, 0, st>>>(kc, N, MP, p.R, p.vals_a);
        else if (m == 3) k_small_k0<3><<<gb, 256, 0, st>>>(kc, N, MP, p.R, p.vals_a);
        else k_small_k0<4><<<gb, 256, 0, st>>>(kc, N, MP, p.R, p.vals_a);
    } else {
    // K0: per-column dense ranks, up to K0_LANES columns in flight (fork/join on side streams)
    int lanes = m < k0_lanes_env() ? m : k0_lanes_env();
    K0Side *side = lanes > 1 ? k0_side() : nullptr;
    if (!side) lanes = 1;
    if (lanes > 1) {
        TEMO_CUDA(cudaEventRecord(side->fork, st));
        for (int l = 1; l < lanes; ++l) TEMO_CUDA(cudaStreamWaitEvent(side->s[l], side->fork, 0));
    }
    for (int col = 0; col < m; ++col) {
        const int l = col % lanes;
        cudaStream_t cs = l ? side->s[l] : st;
        k_col_keys<<<grid1(N), 256, 0, cs>>>(F, N, m, col, p.lk_a[l], p.lv_a[l], status);
        TEMO_CUDA(cub::DeviceRadixSort::SortPairs(p.ltmp[l], tb, p.lk_a[l], p.lk_b[l], p.lv_a[l],
                                                  p.lv_b[l], (int)N, 0, 64, cs));
        k_key_change<<<grid1(N), 256, 0, cs>>>(p.lk_b[l], N, p.ls_a[l]);
        TEMO_CUDA(cub::DeviceScan::InclusiveSum(p.ltmp[l], tb, p.ls_a[l], p.ls_b[l], (int)N, cs));
        k_scatter_rank<<<grid1(N), 256, 0, cs>>>(p.lv_b[l], p.ls_b[l], N, MP, col, p.R);
    }
    for (int l = 1; l < lanes; ++l) {
        TEMO_CUDA(cudaEventRecord(side->join[l], side->s[l]));
        TEMO_CUDA(cudaStreamWaitEvent(st, side->join[l], 0));
    }
    // lexicographic order of rank tuples: LSD passes, several columns per u64 key
    k_iota<<<grid1(N), 256, 0, st>>>(p.vals_a, N);
    int32_t *const va0 = p.vals_a, *const vb0 = p.vals_b;
    const int per = 64 / p.bitsN;
    for (int hi = m; hi > 0;) {
        const int g = hi < per ? hi : per;
        const int c0 = hi - g;
        k_pack_keys<<<grid1(N), 256, 0, st>>>(p.R, p.vals_a, N, MP, c0, g, p.bitsN, p.keys_a);
        TEMO_CUDA(cub::DeviceRadixSort::SortPairs(p.cub_tmp, tb, p.keys_a, p.keys_b, p.vals_a,
                                                  p.vals_b, (int)N, 0, g * p.bitsN, st));
        std::swap(p.vals_a, p.vals_b);
        hi = c0;
    }
    if (p.vals_a != va0) {  // keep the order in the plan's canonical buffer (re-planned calls read it)
        TEMO_CUDA(cudaMemcpyAsync(va0, p.vals_a, sizeof(int32_t) * N, cudaMemcpyDeviceToDevice, st));
        p.vals_a = va0;
        p.vals_b = vb0;
    }
    }
    // run ids of equal tuples
    k_tuple_start<<<grid1(N), 256, 0, st>>>(p.R, p.vals_a, N, m, MP, p.scan_a);
    TEMO_CUDA(cub::DeviceScan::InclusiveScan(p.cub_tmp, tb, p.scan_a, p.scan_b, cub::Max(), (int)N, st));
    k_records<<<grid1(p.Np), 256, 0, st>>>(p.R, p.vals_a, p.scan_b, N, p.Np, m, MP, p.NV, p.rec);
    TEMO_LAUNCH_CHECK();
    stage_end(S_RANK_PREP, st);
    return TEMO_OK;
}

// K1 over the column tiles of `L`; cnt (zeroed in dom_m) is indexed from column tile L.jt_lo
static int launch_dom(const RankPlan &p, const BitLayout &L, uint32_t *bits, int32_t *cnt,
                      cudaStream_t st) {
    stage_begin(S_DOM_BITS, st);
    int rc = TEMO_EINVAL;
#define DOM_CASE(MM) case MM: rc = dom_m<MM>(p, L, bits, cnt, st); break;
    switch (p.m) {
        TEMO_ND_M_LIST(DOM_CASE)
        default: return TEMO_EINVAL;
    }
#undef DOM_CASE
    if (rc) return rc;
    TEMO_LAUNCH_CHECK();
    stage_end(S_DOM_BITS, st);
    return TEMO_OK;
}

// K0 + K1 on the full triangle.  Leaves order in p.vals_a, records in p.rec, bitmap in p.bits.
static int build_bitmap(RankPlan &p, const double *F, int32_t *status, cudaStream_t st) {
    int rc = build_records(p, F, status, st);
    if (rc) return rc;
    k_rowtile_offsets<<<grid1(p.nT), 256, 0, st>>>(p.nT, p.W, p.rt_off, p.rt_lo, p.rt_stride);
    BitLayout L{0, p.nT, p.rt_off, p.rt_lo, p.rt_stride, 0};
    return launch_dom(p, L, p.bits, p.cnt, st);
}

static int peel_grid(int NB, size_t smem) {
    static int occ = 0;
    if (!occ) {
        cudaFuncSetAttribute(k_peel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_peel, PEEL_T, 24 * 1024);
        if (occ <= 0) occ = 1;
    }
    (void)smem;
    int P = num_sms() * occ;
    const int want = NB * 16;
    return want < P ? (want > 0 ? want : 1) : P;
}

}  // namespace temo

#include "ndsort_stair.cuh"

using namespace temo;

static size_t bitmap_ws_bytes(int64_t N, int m) {
    RankPlan p;
    plan_rank(p, nullptr, N, m);
    return p.total;
}

extern "C" size_t temo_rank_ws_bytes(int64_t N, int m) {
    if (N < 1 || m < 1 || m > MAX_M) return 0;
    if (use_stair(m)) {
        StairPlan s;
        plan_stair(s, nullptr, N, m);
        return s.total;
    }
    return bitmap_ws_bytes(N, m);
}

extern "C" int temo_rank(const double *F, int64_t N, int m, int64_t n, int mode, int32_t *rank,
                         int32_t *l_out, int32_t *nfronts, int32_t *status, void *ws,
                         size_t ws_bytes, temo_stream_t stream) {
    if (N < 1 || N > (1 << 20) || m < 1 || m > MAX_M) return TEMO_EINVAL;
    if (n < 1 || n > N) return TEMO_EINVAL;
    if (mode != TEMO_RANK_SORT && mode != TEMO_RANK_SELECT) return TEMO_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    if (use_stair(m)) {
        StairPlan s;
        plan_stair(s, nullptr, N, m);
        if (ws_bytes < s.total || !ws) return TEMO_EWORKSPACE;
        plan_stair(s, ws, N, m);
        return stair_rank(s, F, n, mode, rank, l_out, nfronts, status, st);
    }
    RankPlan p;
    plan_rank(p, nullptr, N, m);
    if (ws_bytes < p.total || !ws) return TEMO_EWORKSPACE;
    plan_rank(p, ws, N, m);
    int rc = build_bitmap(p, F, status, st);
    if (rc) return rc;
    k_peel_init<<<grid1(p.Np), 256, 0, st>>>(p.rank_s, p.cnt, N, p.Np);
    PeelArgs a;
    a.bits = p.bits;
    a.rt_off = p.rt_off;
    a.W = p.W;
    a.N = (int)N;
    a.NB = (int)p.NB;
    a.n = (int)n;
    a.mode = mode;
    a.cnt = p.cnt;
    a.rank_s = p.rank_s;
    a.list = p.list;
    a.blkcnt = p.blkcnt;
    a.out_l = l_out;
    a.out_nfronts = nfronts;
    a.status = status;
    const size_t smem = (size_t)(2 * (p.NB + 1) + 32) * sizeof(int) + 8 * 8 * 32 * sizeof(uint32_t);
    const int P = peel_grid((int)p.NB, smem);
    void *args[] = {&a};
    stage_begin(S_PEEL, st);
    TEMO_CUDA(cudaLaunchCooperativeKernel((void *)k_peel, dim3(P), dim3(PEEL_T), args, smem, st));
    stage_end(S_PEEL, st);
    k_unsort_ranks<<<grid1(N), 256, 0, st>>>(p.rank_s, p.vals_a, l_out, N, rank);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

extern "C" size_t temo_dominance_ws_bytes(int64_t N, int m) {
    if (N < 1 || m < 1 || m > MAX_M) return 0;
    return bitmap_ws_bytes(N, m) + (size_t)N * 4 + 256;
}

extern "C" int temo_dominance(const double *F, int64_t N, int m, uint32_t *D_out, int32_t *status,
                              void *ws, size_t ws_bytes, temo_stream_t stream) {
    if (N < 1 || N > (1 << 20) || m < 1 || m > MAX_M) return TEMO_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    RankPlan p;
    plan_rank(p, nullptr, N, m);
    if (ws_bytes < p.total + (size_t)N * 4 + 256 || !ws) return TEMO_EWORKSPACE;
    plan_rank(p, ws, N, m);
    int32_t *pos = reinterpret_cast<int32_t *>(static_cast<char *>(ws) + round_up(p.total, 256));
    int rc = build_bitmap(p, F, status, st);
    if (rc) return rc;
    k_inverse<<<grid1(N), 256, 0, st>>>(p.vals_a, N, pos);
    const int64_t Wd = (N + 31) / 32;
    k_expand_dense<<<grid1(N * Wd), 256, 0, st>>>(p.bits, p.rt_off, p.W, pos, N, Wd, D_out);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

#include "ndsort_shard.cuh"

#endif  // TEMO_M_ONLY
