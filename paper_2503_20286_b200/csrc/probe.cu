// Diagnostic microbenchmark: the first K1 design's inner-loop instruction mix
// (two chained unsigned ISETP + one warp VOTE per (warp, row)) on register
// operands only.  Kept as a probe of the compare/vote issue rate; the packed K1
// beats it, so it is not used as a roofline denominator (bench.py uses the SM
// issue rate).
#include "common.cuh"

namespace temo {

__global__ void __launch_bounds__(256) k_probe_compare(int iters, uint32_t seed, uint32_t *out) {
    uint32_t a = seed ^ (threadIdx.x * 2654435761u), b = a * 7u + 3u;
    uint32_t r1 = a & 0xFFFFF, r2 = b & 0xFFFFF;
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll 16
        for (int k = 0; k < 16; ++k) {
            // operands vary per step but stay in registers (like LDS broadcasts of i)
            const uint32_t x = (r1 + k * 977u) & 0xFFFFF, y = (r2 + k * 1931u) & 0xFFFFF;
            const bool P = (x <= r1) & (y <= r2);
            acc ^= __ballot_sync(~0u, P);
        }
        r1 += acc & 1;
        r2 ^= acc >> 31;
    }
    if (acc == 0x12345678u) out[0] = acc;  // keep the work live
}

}  // namespace temo

// Returns compares per second (2 compares per lane per step) measured with CUDA events.
extern "C" double temo_probe_compare_rate(int blocks, int iters, temo_stream_t stream) {
    cudaStream_t st = (cudaStream_t)stream;
    uint32_t *dummy = nullptr;
    if (cudaMalloc(&dummy, 4) != cudaSuccess) return -1.0;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    temo::k_probe_compare<<<blocks, 256, 0, st>>>(iters / 4, 1u, dummy);  // warm-up
    cudaEventRecord(a, st);
    temo::k_probe_compare<<<blocks, 256, 0, st>>>(iters, 1u, dummy);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(dummy);
    const double lanes = (double)blocks * 256.0;
    return lanes * (double)iters * 16.0 * 2.0 / (ms * 1e-3);
}
