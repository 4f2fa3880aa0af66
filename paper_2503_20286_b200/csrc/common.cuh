// Shared helpers for the temo_b200 CUDA library (sm_100a).
//
// Build flags (see paper_2503_20286_b200/build.py): -gencode arch=compute_100a,code=sm_100a
// --fmad=false.  FMA contraction is OFF for the whole library so every double
// expression rounds exactly like the NumPy reference op-by-op; the few places
// where the reference itself fuses (OpenBLAS dgemm / LAPACK getrf, SURVEY App.
// A2/A4) call fma() explicitly.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>
#include <float.h>

#include "../../include/temo_b200.h"

#define TEMO_BIG DBL_MAX  // tensorops.py:18 sentinel

namespace temo {

// ---------------------------------------------------------------- workspace
// Caller-provided workspace is carved in a fixed order; a dry run with
// base == nullptr computes the byte count (no allocation inside the library).
struct Carve {
    char *base;
    size_t off = 0;
    explicit Carve(void *b) : base(static_cast<char *>(b)) {}
    template <class T>
    T *take(size_t count, size_t align = 256) {
        off = (off + align - 1) / align * align;
        T *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
        off += count * sizeof(T);
        return p;
    }
};

#define TEMO_CUDA(expr)                                  \
    do {                                                 \
        cudaError_t _e = (expr);                         \
        if (_e != cudaSuccess) return TEMO_ECUDA;        \
    } while (0)

#define TEMO_LAUNCH_CHECK()                              \
    do {                                                 \
        if (cudaPeekAtLastError() != cudaSuccess) {      \
            (void)cudaGetLastError();                    \
            return TEMO_ECUDA;                           \
        }                                                \
    } while (0)

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }
inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

int num_sms();

// stage ids for temo_timing_* (names in capi.cu)
enum Stage {
    S_RANK_PREP = 0, S_DOM_BITS, S_PEEL, S_NORMALIZE, S_ASSOCIATE, S_NICHE, S_OFFSPRING,
    S_EVALUATE, S_HV_COUNT, S_HV_CONTRIB, S_HYPE_SELECT, S_MOEAD, S_GATHER, S_MISC,
    S_OFFSPRING_APPLY,  // the apply stage of the two-phase offspring step (S_OFFSPRING: its randomness kernel)
    S_APPLY_VEC         // the streaming kernel inside S_OFFSPRING_APPLY (k_offspring_apply_v)
};
void stage_begin(int stage, cudaStream_t st);
void stage_end(int stage, cudaStream_t st);

// ------------------------------------------------------------ order keys
// Order-preserving u64 image of a double; -0.0 is folded onto +0.0 so that
// equal doubles map to equal keys (np comparisons treat them as equal).
__device__ __forceinline__ uint64_t ordered_key(double x) {
    if (x == 0.0) x = 0.0;
    uint64_t u = (uint64_t)__double_as_longlong(x);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

__device__ __forceinline__ void flag_status(int32_t *status, int bit) {
    if (status) atomicOr(status, bit);
}

// NumPy add.reduce over a short contiguous last axis:
// sequential below 8 terms, 8 strided accumulators + pairwise combine above.
template <int MAXM>
__device__ __forceinline__ double np_sum(const double *v, int m) {
    if (m < 8) {
        double s = v[0];
        for (int k = 1; k < m; ++k) s = s + v[k];
        return s;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = v[j];
    int i = 8;
    for (; i + 8 <= m; i += 8)
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = r[j] + v[i + j];
    double s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < m; ++i) s = s + v[i];
    return s;
}

}  // namespace temo
