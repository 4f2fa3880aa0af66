// Measured ceilings for the roofline denominators of the two compute-bound kernels
// (bench.py `roofline_compute`).  Neither is on the data path; each runs the
// kernel's inner-loop instruction mix on register operands only, so its rate is
// the issue/pipe ceiling of that mix on this GPU and clock.
//
//   k_probe_philox : Philox4x64-10 blocks (NumPy's stream, philox.cuh), 4 blocks in
//                    lockstep per thread -- the core of k_offspring_rand (5 blocks per
//                    gene quad).  Rate = blocks/s.
//   k_probe_packed : the packed dominance step of K1 (ndsort.cu k_dom_rows8, m = 3):
//                    per column pair 2 IMAD subtractions, one LOP3, one LEA/shift-add.
//                    Rate = pair tests/s (2 per step).
//   k_probe_dsub   : FP64 subtract + add chains (HypE's sample-dominance test).  Rate =
//                    FP64 add/sub operations/s.
// The caller passes an 8-byte device scratch word (the library allocates nothing).
#include "common.cuh"
#include "philox.cuh"

namespace temo {

__global__ void __launch_bounds__(256) k_probe_philox(Philox ph, int iters, uint64_t *out) {
    uint64_t c[4][4];
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
#pragma unroll
    for (int b = 0; b < 4; ++b) ctr_add(ph.ctr, 4 * t + b, c[b]);
    uint64_t acc = 0;
    for (int it = 0; it < iters; ++it) {
        uint64_t o[4][4];
        philox_blocks_rk<4>(c, ph.rk, o);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            acc ^= o[b][0] ^ o[b][1] ^ o[b][2] ^ o[b][3];
            c[b][0] += 0x100000000ull;  // next counters (stays in the low word's upper half)
        }
    }
    if (acc == 0x123456789ull) out[0] = acc;  // keep the work live
}

__global__ void __launch_bounds__(128) k_probe_packed(int iters, uint32_t seed, uint64_t *out) {
    // 8 rows per lane (k_dom_rows8), column-pair words broadcast: per step and row
    // g = ((Q1 | G) - p1 * 0x10001) & ((Q2 | G) - p2 * 0x10001) & 0x80008000; acc = (acc >> 1) + g
    uint32_t p1[8], p2[8], acc[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        p1[r] = (seed + threadIdx.x * 31u + r * 7u) & 0x7FF;
        p2[r] = (seed * 3u + threadIdx.x * 17u + r * 5u) & 0x7FF;
        acc[r] = 0;
    }
    uint32_t q1 = seed * 2654435761u, q2 = seed * 40503u;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int s = 0; s < 16; ++s) {
            const uint32_t a = (q1 + s * 0x00010001u) | 0x80008000u, b = (q2 + s * 0x00030003u) | 0x80008000u;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const uint32_t g = (a - p1[r] * 0x10001u) & (b - p2[r] * 0x10001u) & 0x80008000u;
                acc[r] = (acc[r] >> 1) + g;
            }
        }
        q1 += acc[0];
        q2 ^= acc[7];
    }
    uint32_t x = 0;
#pragma unroll
    for (int r = 0; r < 8; ++r) x ^= acc[r];
    if (x == 0x12345678u) out[0] = x;
}

// HypE's dominance test (hype.cu k_hv_dom): per (point, sample, objective) one FP64
// subtraction whose sign bits are OR-ed; 8 independent chains per thread.
__global__ void __launch_bounds__(256) k_probe_dsub(int iters, double seed, uint64_t *out) {
    double f[8], acc[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        f[r] = seed + 0.125 * r + 1e-3 * threadIdx.x;
        acc[r] = 0.0;
    }
    double smp = seed * 0.5;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int s = 0; s < 16; ++s) {
            const double x = smp + 0.0625 * s;
#pragma unroll
            for (int r = 0; r < 8; ++r) acc[r] = acc[r] + (x - f[r]);
        }
        smp = smp + acc[0] * 1e-300;
    }
    double x = 0.0;
#pragma unroll
    for (int r = 0; r < 8; ++r) x += acc[r];
    if (x == 1234.5) out[0] = 1;
}

// The apply phase's data movement alone: per pair q two gathered parent rows and one
// streamed row in, two scattered child rows out (rows of d doubles, 16-byte vector accesses,
// warp per pair) -- the achievable rate of k_offspring_apply's access pattern.
__global__ void __launch_bounds__(256) k_probe_rows(const double2 *__restrict__ X, const int64_t *__restrict__ pa,
                                                    const int64_t *__restrict__ pb, const double2 *__restrict__ B,
                                                    const int64_t *__restrict__ dst, int64_t h, int64_t d2,
                                                    double2 *__restrict__ O) {
    const int lane = threadIdx.x & 31;
    for (int64_t q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; q < h;
         q += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const double2 *x1 = X + pa[q] * d2, *x2 = X + pb[q] * d2, *bq = B + q * d2;
        double2 *o1 = O + dst[q] * d2, *o2 = O + dst[h + q] * d2;
        for (int64_t j = lane; j < d2; j += 32) {
            const double2 a = x1[j], b = x2[j], c = bq[j];
            o1[j] = make_double2(a.x + c.x * (b.x - a.x), a.y + c.y * (b.y - a.y));
            o2[j] = make_double2(b.x + c.x * (a.x - b.x), b.y + c.y * (a.y - b.y));
        }
    }
}

}  // namespace temo

namespace {
double time_launches(void (*launch)(cudaStream_t, int), int iters, cudaStream_t st) {
    cudaEvent_t a, b;
    if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) return -1.0;
    launch(st, iters / 4 > 0 ? iters / 4 : 1);  // warm-up
    cudaEventRecord(a, st);
    launch(st, iters);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return cudaGetLastError() == cudaSuccess ? ms * 1e-3 : -1.0;
}

int g_blocks;
uint64_t *g_scratch;
void launch_philox(cudaStream_t st, int iters) {
    temo_philox_state z = {};
    z.buffer_pos = 4;
    temo::k_probe_philox<<<g_blocks, 256, 0, st>>>(temo::philox_from(z), iters, g_scratch);
}
void launch_packed(cudaStream_t st, int iters) {
    temo::k_probe_packed<<<g_blocks, 128, 0, st>>>(iters, 1u, g_scratch);
}
void launch_dsub(cudaStream_t st, int iters) {
    temo::k_probe_dsub<<<g_blocks, 256, 0, st>>>(iters, 1.0, g_scratch);
}
}  // namespace

// Philox4x64-10 blocks per second (4 blocks per thread per iteration), CUDA events.
extern "C" double temo_probe_philox_rate(int blocks, int iters, uint64_t *scratch, temo_stream_t stream) {
    if (blocks < 1 || iters < 1 || !scratch) return -1.0;
    g_blocks = blocks;
    g_scratch = scratch;
    const double s = time_launches(launch_philox, iters, (cudaStream_t)stream);
    return s > 0 ? (double)blocks * 256.0 * 4.0 * iters / s : -1.0;
}

// Packed dominance pair tests per second (k_dom_rows8 inner step, m = 3), CUDA events.
extern "C" double temo_probe_packed_rate(int blocks, int iters, uint64_t *scratch, temo_stream_t stream) {
    if (blocks < 1 || iters < 1 || !scratch) return -1.0;
    g_blocks = blocks;
    g_scratch = scratch;
    const double s = time_launches(launch_packed, iters, (cudaStream_t)stream);
    return s > 0 ? (double)blocks * 128.0 * 8.0 * 16.0 * 2.0 * iters / s : -1.0;
}

// FP64 add/subtract operations per second (2 per step and chain: x - f, acc + .), CUDA events.
extern "C" double temo_probe_dsub_rate(int blocks, int iters, uint64_t *scratch, temo_stream_t stream) {
    if (blocks < 1 || iters < 1 || !scratch) return -1.0;
    g_blocks = blocks;
    g_scratch = scratch;
    const double s = time_launches(launch_dsub, iters, (cudaStream_t)stream);
    return s > 0 ? (double)blocks * 256.0 * 8.0 * 16.0 * 2.0 * iters / s : -1.0;
}

// Bytes per second of k_probe_rows over h pairs of d-double rows (5 d doubles moved per pair);
// X holds the parents (>= max(pa, pb) + 1 rows), O the children (>= max(dst) + 1 rows), B h rows.
extern "C" double temo_probe_rows_rate(const double *X, const int64_t *pa, const int64_t *pb, const double *B,
                                       const int64_t *dst, int64_t h, int64_t d, double *O, int iters,
                                       temo_stream_t stream) {
    if (!X || !pa || !pb || !B || !dst || !O || h < 1 || d < 2 || d % 2 || iters < 1) return -1.0;
    cudaStream_t st = (cudaStream_t)stream;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = (unsigned)(sms * 8);
    auto launch = [&]() {
        temo::k_probe_rows<<<grid, 256, 0, st>>>(reinterpret_cast<const double2 *>(X), pa, pb,
                                                 reinterpret_cast<const double2 *>(B), dst, h, d / 2,
                                                 reinterpret_cast<double2 *>(O));
    };
    launch();
    cudaEvent_t a, b;
    if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) return -1.0;
    cudaEventRecord(a, st);
    for (int i = 0; i < iters; ++i) launch();
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (cudaGetLastError() != cudaSuccess || ms <= 0.f) return -1.0;
    return 5.0 * 8.0 * (double)h * (double)d * iters / (ms * 1e-3);
}
