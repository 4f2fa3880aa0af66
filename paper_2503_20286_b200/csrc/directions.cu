// Neighbour tables of direction sets (replaces temo directions.py:104-114).
// Setup-time kernel: one thread per row, directions staged in shared memory,
// Euclidean distance in NumPy's op order (App. A1), and an insertion list that
// keeps the T smallest (distance, index) pairs -- the stable-argsort tie rule.
#include "common.cuh"

namespace temo {

constexpr int NB_T = 128;
constexpr int NB_TILE = 256;
constexpr int NB_MAXT = 64;

__global__ void __launch_bounds__(NB_T) k_neighbors(const double *__restrict__ W, int64_t r, int m,
                                                    int T, int32_t *__restrict__ out) {
    __shared__ double sW[NB_TILE * 16];
    const int64_t i = blockIdx.x * (int64_t)NB_T + threadIdx.x;
    double wi[16];
    if (i < r)
        for (int k = 0; k < m; ++k) wi[k] = W[i * m + k];
    double bd[NB_MAXT];
    int32_t bj[NB_MAXT];
    int cnt = 0;
    for (int64_t j0 = 0; j0 < r; j0 += NB_TILE) {
        const int c = (int)min((int64_t)NB_TILE, r - j0);
        __syncthreads();
        for (int q = threadIdx.x; q < c * m; q += NB_T) sW[q] = W[j0 * m + q];
        __syncthreads();
        if (i >= r) continue;
        for (int jj = 0; jj < c; ++jj) {
            double sq[16];
            for (int k = 0; k < m; ++k) {
                const double d = wi[k] - sW[jj * m + k];
                sq[k] = d * d;
            }
            const double dist = sqrt(np_sum<16>(sq, m));
            if (cnt == T && !(dist < bd[T - 1])) continue;
            int p = cnt < T ? cnt : T - 1;
            while (p > 0 && bd[p - 1] > dist) {
                bd[p] = bd[p - 1];
                bj[p] = bj[p - 1];
                --p;
            }
            bd[p] = dist;
            bj[p] = (int32_t)(j0 + jj);
            if (cnt < T) ++cnt;
        }
    }
    if (i < r)
        for (int t = 0; t < T; ++t) out[i * T + t] = bj[t];
}

}  // namespace temo

extern "C" int temo_neighbors(const double *W, int64_t r, int m, int T, int32_t *out,
                              temo_stream_t stream) {
    if (r < 1 || m < 1 || m > 16 || T < 1 || T > r || T > temo::NB_MAXT || !W || !out)
        return TEMO_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    temo::k_neighbors<<<(unsigned)((r + temo::NB_T - 1) / temo::NB_T), temo::NB_T, 0, st>>>(W, r, m, T, out);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}
