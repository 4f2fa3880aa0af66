/* Standalone C driver for temo_offspring (fused SBX + PM + LSMOP1 evaluation), for ncu.
 *   offspring_driver pop d reps
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "temo_b200.h"

int main(int argc, char **argv) {
    long long n = argc > 1 ? atoll(argv[1]) : 200000;
    long long d = argc > 2 ? atoll(argv[2]) : 1000;
    int reps = argc > 3 ? atoi(argv[3]) : 2;
    int use_ws = argc > 4 && argv[4][0] == 'w';  /* "ws": two-phase temo_offspring_ws */
    const int m = 3;
    long long h = n / 2;
    double *hX = (double *)malloc(sizeof(double) * n * d);
    double *lo = (double *)malloc(sizeof(double) * d), *hi = (double *)malloc(sizeof(double) * d);
    for (long long g = 0; g < d; ++g) { lo[g] = 0.0; hi[g] = g < m - 1 ? 1.0 : 10.0; }
    unsigned long long s = 88172645463325252ull;
    for (long long i = 0; i < n * d; ++i) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        hX[i] = hi[i % d] * (double)(s >> 11) * (1.0 / 9007199254740992.0);
    }
    long long *hidx = (long long *)malloc(sizeof(long long) * n);
    for (long long i = 0; i < n; ++i) hidx[i] = (i * 7919) % n;
    double *X, *O, *FO, *dlo, *dhi;
    long long *idx;
    cudaMalloc((void **)&X, sizeof(double) * n * d);
    cudaMalloc((void **)&O, sizeof(double) * 2 * h * d);
    cudaMalloc((void **)&FO, sizeof(double) * 2 * h * m);
    cudaMalloc((void **)&dlo, sizeof(double) * d);
    cudaMalloc((void **)&dhi, sizeof(double) * d);
    cudaMalloc((void **)&idx, sizeof(long long) * n);
    cudaMemcpy(X, hX, sizeof(double) * n * d, cudaMemcpyHostToDevice);
    cudaMemcpy(dlo, lo, sizeof(double) * d, cudaMemcpyHostToDevice);
    cudaMemcpy(dhi, hi, sizeof(double) * d, cudaMemcpyHostToDevice);
    cudaMemcpy(idx, hidx, sizeof(long long) * n, cudaMemcpyHostToDevice);
    temo_problem P;
    memset(&P, 0, sizeof(P));
    P.id = TEMO_PROB_LSMOP1; P.m = m; P.d = d; P.nk = 5;
    /* chaotic sizes (problems.py lsmop_groups) */
    double c[3] = {3.8 * 0.1 * 0.9, 0, 0}, cs = 0;
    for (int i = 1; i < m; ++i) c[i] = 3.8 * c[i - 1] * (1 - c[i - 1]);
    for (int i = 0; i < m; ++i) cs += c[i];
    int off = 0;
    P.offset[0] = 0;
    for (int i = 0; i < m; ++i) {
        P.sublen[i] = (int)floor(c[i] / cs * (double)(d - m + 1) / 5);
        off += P.sublen[i] * 5;
        P.offset[i + 1] = off;
    }
    temo_variation V = {20.0, 20.0, 1.0 / (double)d, 1, 0, dlo, dhi};
    temo_philox_state st;
    memset(&st, 0, sizeof(st));
    st.key[0] = 0x1234; st.key[1] = 0x5678; st.buffer_pos = 4;
    size_t ws_bytes = temo_offspring_ws_bytes(h, d);
    void *ws = NULL;
    cudaMalloc(&ws, ws_bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(a, 0);
        int rc = use_ws ? temo_offspring_ws(&P, &V, X, (const int64_t *)idx, (const int64_t *)(idx + h), h, &st, 0,
                                            O, FO, NULL, NULL, ws, ws_bytes, 0)
                        : temo_offspring(&P, &V, X, (const int64_t *)idx, (const int64_t *)(idx + h), h, &st, 0, O, FO, 0);
        cudaEventRecord(b, 0);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("rc=%d pop=%lld d=%lld ms=%.3f err=%s\n", rc, n, d, ms, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
