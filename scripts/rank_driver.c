/* Standalone C driver for the temo_b200 C ABI (no Python, no torch).
 * Used for ncu captures and as a C-level usage example of include/temo_b200.h.
 *   rank_driver N m mode reps
 * Build: nvcc -O2 -I include scripts/rank_driver.c -L paper_2503_20286_b200/_lib -ltemo_b200 -o rank_driver
 */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "temo_b200.h"

int main(int argc, char **argv) {
    long long N = argc > 1 ? atoll(argv[1]) : 100000;
    int m = argc > 2 ? atoi(argv[2]) : 3;
    int mode = argc > 3 ? atoi(argv[3]) : TEMO_RANK_SELECT;
    int reps = argc > 4 ? atoi(argv[4]) : 2;
    double *hF = (double *)malloc(sizeof(double) * N * m);
    unsigned long long s = 88172645463325252ull;
    for (long long i = 0; i < N * m; ++i) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        hF[i] = (double)(s >> 11) * (1.0 / 9007199254740992.0);
    }
    double *dF; int *rank, *l, *nf, *status; void *ws;
    size_t wsb = temo_rank_ws_bytes(N, m);
    cudaMalloc((void **)&dF, sizeof(double) * N * m);
    cudaMalloc((void **)&rank, sizeof(int) * N);
    cudaMalloc((void **)&l, 4); cudaMalloc((void **)&nf, 4); cudaMalloc((void **)&status, 4);
    cudaMalloc(&ws, wsb);
    cudaMemcpy(dF, hF, sizeof(double) * N * m, cudaMemcpyHostToDevice);
    cudaMemset(status, 0, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(a, 0);
        int rc = temo_rank(dF, N, m, N / 2, mode, rank, l, nf, status, ws, wsb, 0);
        cudaEventRecord(b, 0);
        cudaEventSynchronize(b);
        float ms = 0; cudaEventElapsedTime(&ms, a, b);
        int hl, hn, hs;
        cudaMemcpy(&hl, l, 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(&hn, nf, 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(&hs, status, 4, cudaMemcpyDeviceToHost);
        printf("rc=%d N=%lld m=%d mode=%d l=%d fronts=%d status=%d ms=%.3f err=%s\n", rc, N, m, mode, hl,
               hn, hs, ms, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
