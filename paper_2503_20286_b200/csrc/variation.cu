// Offspring generation and problem evaluation on B200
// (replaces temo variation.py:48-120, problems.py:69-136, harness.py:201-204).
//
// The generation front end is ONE kernel: a CTA owns a parent pair, draws its
// uniforms straight from the NumPy-compatible Philox stream (philox.cuh),
// applies SBX and polynomial mutation with the reference's op sequence
// (only the taken np.where branch is evaluated, which is
// bit-identical), stages both children in shared memory and evaluates them
// (DTLZ1-7 or LSMOP1) with block reductions -- no uniform matrices, children
// or objectives round-trip through HBM except the final O and FO rows.
//
// Each thread owns quads of 4 consecutive genes: parents and children move
// as 32-byte vectors, and every stream's 4 uniforms come from at most two
// Philox blocks generated on the spot (no long-lived per-stream cursor
// state), which keeps the kernel at <= 80 registers.  Evaluation is
// templated on m so per-objective accumulators live in registers.
#include "common.cuh"
#include "philox.cuh"
#include "sbx_pow.cuh"

namespace temo {

// integer knob from the environment (A/B experiments; the default otherwise)
static int env_int(const char *name, int dflt) {
    const char *e = getenv(name);
    return (e && *e) ? atoi(e) : dflt;
}

constexpr int VT = 128;
constexpr double PI = 3.141592653589793;

__device__ __forceinline__ double clipv(double x, double lo, double hi) {
    // np.clip(a, lo, hi) == minimum(maximum(a, lo), hi)
    double y = x < lo ? lo : x;
    return y > hi ? hi : y;
}

// SBX spread factor (variation.py:77-78) shared by every offspring kernel, so all paths agree bitwise
__device__ __forceinline__ double sbx_beta_any(double mu, double e) {
#if !defined(OFF_CUDA_POW) || OFF_CUDA_POW
    return pow((0.5 - mu >= 0.0) ? 2.0 * mu : 1.0 / (2.0 - 2.0 * mu), e);
#else
    return sbx_beta_fast(mu, e);
#endif
}

__device__ __forceinline__ void sbx_gene(double x1, double x2, double mu, double swp, double crs,
                                         double e, bool gene_swap, double &c1, double &c2) {
    double beta;
    if (gene_swap && !(crs < 0.5)) {
        beta = 1.0;  // not crossed: masked_blend(crossed, beta, 1)
    } else {
        beta = sbx_beta_any(mu, e);
        if (gene_swap) beta = beta * (1.0 - 2.0 * (swp < 0.5 ? 1.0 : 0.0));
    }
    const double shift = 0.5 * (1.0 - beta);
    c1 = x1 + shift * (x2 - x1);
    c2 = x2 + shift * (x1 - x2);
}

static __device__ __noinline__ double pm_step(double x, double lo, double hi, double mu, double eta) {
    const double span = hi - lo;
    double step;
    if (0.5 - mu >= 0.0) {
        const double gap = (x - lo) / span;
        step = pow(2.0 * mu + (1.0 - 2.0 * mu) * pow(1.0 - gap, eta), 1.0 / eta) - 1.0;
    } else {
        const double gap = (hi - x) / span;
        step = 1.0 - pow(2.0 - 2.0 * mu + (2.0 * mu - 1.0) * pow(1.0 - gap, eta), 1.0 / eta);
    }
    return x + step * span;
}

// `cnt` consecutive uniforms of the stream starting at element e0 (<= 2 Philox blocks)
__device__ __forceinline__ void uniforms4(const Philox &ph, uint64_t e0, int cnt, double u[4]) {
    PhiloxCursor c;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (k < cnt) u[k] = c.uniform(ph, e0 + k);
}

__device__ __forceinline__ double uniform1(const Philox &ph, uint64_t e) {
    PhiloxCursor c;
    return c.uniform(ph, e);
}

// ------------------------------------------------------------------ evaluation
static __device__ double block_sum(double v, double *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(~0u, v, d);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    return s;
}

// objectives of one row x (length d) -> f[0..M); called by every thread of the CTA
template <int M>
__device__ void eval_row(const temo_problem &P, const double *x, double *f, double *red) {
    const int64_t d = P.d;
    const int id = P.id;
    if (id == TEMO_PROB_LSMOP1) {
        double part[M];
#pragma unroll
        for (int i = 0; i < M; ++i) part[i] = 0.0;
        const double x0 = x[0];
        const int64_t span_s = P.offset[M];
        for (int64_t g = (M - 1) + threadIdx.x; g < d; g += blockDim.x) {
            const int64_t rel = g - (M - 1);
            if (rel >= span_s) continue;
            const double a = (double)(g + 1);
            const double xs = (1.0 + a / (double)d) * x[g] - 10.0 * x0;
            const double sq = xs * xs;
#pragma unroll
            for (int i = 0; i < M; ++i)
                if (rel >= P.offset[i] && rel < P.offset[i + 1]) part[i] += sq;
        }
        double G[M];
#pragma unroll
        for (int i = 0; i < M; ++i) G[i] = block_sum(part[i], red);
        if (threadIdx.x == 0) {
#pragma unroll
            for (int i = 0; i < M; ++i) {
                const double gi = G[i] / (double)P.sublen[i] / (double)P.nk;
                double head = 1.0;
                for (int k = 0; k < M - 1 - i; ++k) head = head * x[k];
                const double tail = i == 0 ? 1.0 : 1.0 - x[M - 1 - i];
                f[i] = (1.0 + gi) * head * tail;
            }
        }
        return;
    }
    // DTLZ family: g over the distance variables xm = x[m-1:]
    const int64_t k = d - M + 1;
    double acc = 0.0;
    for (int64_t g = (M - 1) + threadIdx.x; g < d; g += blockDim.x) {
        const double v = x[g];
        switch (id) {
            case 1:
            case 3: {
                const double z = v - 0.5;
                acc += z * z - cos(20.0 * PI * z);
                break;
            }
            case 2:
            case 4:
            case 5: {
                const double z = v - 0.5;
                acc += z * z;
                break;
            }
            case 6: acc += pow(v, 0.1); break;
            default: acc += v; break;  // dtlz7
        }
    }
    const double s = block_sum(acc, red);
    if (threadIdx.x != 0) return;
    double g;
    if (id == 1 || id == 3) g = 100.0 * ((double)k + s);
    else if (id == 7) g = 1.0 + 9.0 / (double)k * s;
    else g = s;
    if (id == 1) {
#pragma unroll
        for (int i = 0; i < M; ++i) {
            double p = 1.0;
            for (int q = 0; q < M - 1 - i; ++q) p = p * x[q];
            if (i) p = p * (1.0 - x[M - 1 - i]);
            f[i] = 0.5 * (1.0 + g) * p;
        }
        return;
    }
    if (id == 7) {
        double h = 0.0;
        for (int q = 0; q < M - 1; ++q) {
            f[q] = x[q];
            h += x[q] / (1.0 + g) * (1.0 + sin(3.0 * PI * x[q]));
        }
        f[M - 1] = (1.0 + g) * ((double)M - h);
        return;
    }
    double th[M];
#pragma unroll
    for (int q = 0; q < M - 1; ++q) {
        if (id == 4) th[q] = pow(x[q], 100.0) * (PI / 2.0);
        else if (id == 5 || id == 6) {
            if (q == 0) th[q] = x[0] * (PI / 2.0);
            else th[q] = PI / (4.0 * (1.0 + g)) * (1.0 + 2.0 * g * x[q]);
        } else th[q] = x[q] * (PI / 2.0);
    }
#pragma unroll
    for (int i = 0; i < M; ++i) {
        double p = 1.0;
        for (int q = 0; q < M - 1 - i; ++q) p = p * cos(th[q]);
        if (i) p = p * sin(th[M - 1 - i]);
        f[i] = (1.0 + g) * p;
    }
}

template <int M>
__global__ void __launch_bounds__(VT) k_evaluate(temo_problem P, const double *__restrict__ X,
                                                 const int64_t *__restrict__ map, int64_t lo1, int64_t c1,
                                                 int64_t lo2, int64_t c2, double *__restrict__ F) {
    __shared__ double red[VT / 32];
    __shared__ double f[16];
    const int64_t w = blockIdx.x;
    if (w >= c1 + c2) return;
    const int64_t r = w < c1 ? lo1 + w : lo2 + (w - c1);
    eval_row<M>(P, X + (map ? map[r] : r) * P.d, f, red);
    __syncthreads();
    if (threadIdx.x < M) F[r * M + threadIdx.x] = f[threadIdx.x];
}

// ------------------------------------------------------------------ LSMOP2..9
// Cheng et al. 2017 in the PlatEMO formulation (no reference implementation; self-oracle
// oracle/problems.py evaluate_lsmop).  Objective i (0-based) sums its nk subcomponents of
// x^s through eta1 (even i, PlatEMO's odd objectives) or eta2 (odd i); linkage
// z = (1 + c(j)) x_j - 10 x_1 with c = j/D (LSMOP1-4) or cos(j/D pi/2) (LSMOP5-9).
enum LsFn { LS_SPHERE, LS_GRIEWANK, LS_SCHWEFEL, LS_RASTRIGIN, LS_ROSENBROCK, LS_ACKLEY };

__device__ __forceinline__ int lsmop_fn(int k, int i) {
    const bool odd = i & 1;  // PlatEMO's even-numbered objective: eta2
    switch (k) {
        case 2: return odd ? LS_SCHWEFEL : LS_GRIEWANK;
        case 3: return odd ? LS_ROSENBROCK : LS_RASTRIGIN;
        case 4: return odd ? LS_GRIEWANK : LS_ACKLEY;
        case 6: return odd ? LS_SCHWEFEL : LS_ROSENBROCK;
        case 7: return odd ? LS_ROSENBROCK : LS_ACKLEY;
        case 8: return odd ? LS_SPHERE : LS_GRIEWANK;
        case 9: return odd ? LS_ACKLEY : LS_SPHERE;
        default: return LS_SPHERE;  // LSMOP1, LSMOP5
    }
}

__device__ __forceinline__ double lsmop_link(int k, int64_t g, int64_t d, double x, double x0) {
    const double j = (double)(g + 1) / (double)d;  // PlatEMO's (M:D)./D
    const double c = k >= 5 ? cos(j * PI / 2.0) : j;
    return (1.0 + c) * x - 10.0 * x0;
}

// One warp per row; logical rows [lo1, lo1 + c1) then [lo2, lo2 + c2); row l is read from
// X + (map ? map[l] : l) * d and written to F + l * M.
template <int M>
__global__ void __launch_bounds__(256) k_eval_lsmop(temo_problem P, const double *__restrict__ X,
                                                    const int64_t *__restrict__ map, int64_t lo1, int64_t c1,
                                                    int64_t lo2, int64_t c2, double *__restrict__ F) {
    const int lane = threadIdx.x & 31;
    const int64_t d = P.d, nrow = c1 + c2;
    const int k = P.id - TEMO_PROB_LSMOP1 + 1;
    for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < nrow;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t l = w < c1 ? lo1 + w : lo2 + (w - c1);
        const double *x = X + (map ? map[l] : l) * d;
        const double x0 = x[0];
        double G[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const int fn = lsmop_fn(k, i);
            const int64_t L = P.sublen[i];
            double gi = 0.0;
            for (int j = 0; j < P.nk; ++j) {
                const int64_t start = (M - 1) + P.offset[i] + j * L;
                double s2 = 0.0, sc = 0.0, pr = 1.0, mx = 0.0;
                for (int64_t t = lane; t < L; t += 32) {
                    const int64_t g = start + t;
                    const double z = lsmop_link(k, g, d, x[g], x0);
                    switch (fn) {
                        case LS_SPHERE: s2 += z * z; break;
                        case LS_GRIEWANK:
                            s2 += z * z;
                            pr *= cos(z / sqrt((double)(t + 1)));
                            break;
                        case LS_SCHWEFEL: mx = fmax(mx, fabs(z)); break;
                        case LS_RASTRIGIN: s2 += z * z - 10.0 * cos(2.0 * PI * z) + 10.0; break;
                        case LS_ROSENBROCK:
                            if (t + 1 < L) {
                                const double z2 = lsmop_link(k, g + 1, d, x[g + 1], x0);
                                const double a = z * z - z2, b = z - 1.0;
                                s2 += 100.0 * (a * a) + b * b;
                            }
                            break;
                        default:  // LS_ACKLEY
                            s2 += z * z;
                            sc += cos(2.0 * PI * z);
                            break;
                    }
                }
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    s2 += __shfl_xor_sync(~0u, s2, o);
                    sc += __shfl_xor_sync(~0u, sc, o);
                    pr *= __shfl_xor_sync(~0u, pr, o);
                    mx = fmax(mx, __shfl_xor_sync(~0u, mx, o));
                }
                double v;
                if (fn == LS_GRIEWANK) v = s2 / 4000.0 - pr + 1.0;
                else if (fn == LS_SCHWEFEL) v = mx;
                else if (fn == LS_ACKLEY)
                    v = 20.0 - 20.0 * exp(-0.2 * sqrt(s2 / (double)L)) - exp(sc / (double)L) + exp(1.0);
                else v = s2;
                gi += v;
            }
            G[i] = gi / (double)L / (double)P.nk;
        }
        if (lane != 0) continue;
        double *f = F + l * M;
        if (k <= 4) {  // linear front (LSMOP1-4)
#pragma unroll
            for (int i = 0; i < M; ++i) {
                double head = 1.0;
                for (int q = 0; q < M - 1 - i; ++q) head = head * x[q];
                const double tail = i == 0 ? 1.0 : 1.0 - x[M - 1 - i];
                f[i] = (1.0 + G[i]) * head * tail;
            }
        } else if (k <= 8) {  // concave front (LSMOP5-8): (1 + G_i + G_{i+1})
#pragma unroll
            for (int i = 0; i < M; ++i) {
                double head = 1.0;
                for (int q = 0; q < M - 1 - i; ++q) head = head * cos(x[q] * PI / 2.0);
                const double tail = i == 0 ? 1.0 : sin(x[M - 1 - i] * PI / 2.0);
                const double gn = i + 1 < M ? G[i + 1] : 0.0;
                f[i] = (1.0 + G[i] + gn) * head * tail;
            }
        } else {  // LSMOP9: disconnected front
            double gs = 0.0;
#pragma unroll
            for (int i = 0; i < M; ++i) gs += G[i];
            gs = 1.0 + gs;
            double hsum = 0.0;
            for (int q = 0; q < M - 1; ++q) {
                f[q] = x[q];
                hsum += x[q] / (1.0 + gs) * (1.0 + sin(3.0 * PI * x[q]));
            }
            f[M - 1] = (1.0 + gs) * ((double)M - hsum);
        }
    }
}

// ------------------------------------------------------------------ fused offspring
struct VarArgs {
    double eta_c, eta_m, p_m;
    int gene_swap;
    const double *lower, *upper;
};

template <int M>
__global__ void __launch_bounds__(VT, 6) k_offspring(temo_problem P, VarArgs V, const double *__restrict__ X,
                                                     const int64_t *__restrict__ i1,
                                                     const int64_t *__restrict__ i2, int64_t h,
                                                     Philox ph, uint64_t off, double *__restrict__ O,
                                                     double *__restrict__ FO, int smem_rows, int single) {
    // single != 0: MOEA/D mode (moead.py:136-144) -- keep child c1 only and mutate
    // h rows, so the PM draws are (h, d) blocks instead of (2h, d)
    extern __shared__ double srow[];  // 2 x d children when smem_rows
    __shared__ double red[VT / 32];
    __shared__ double f[16];
    const int64_t q = blockIdx.x;
    const int64_t d = P.d;
    const double *x1 = X + i1[q] * d;
    const double *x2 = X + i2[q] * d;
    double *o1 = O + q * d;
    double *o2 = O + (h + q) * d;
    const uint64_t hd = (uint64_t)h * d;
    const uint64_t o_mu = off, o_swap = off + hd, o_cross = off + (V.gene_swap ? 2 * hd : 0);
    const uint64_t o_pmu = off + (V.gene_swap ? 3 * hd : hd);
    const uint64_t o_hit = o_pmu + (single ? hd : 2 * hd);
    const double e = 1.0 / (V.eta_c + 1.0);
    const double eta = V.eta_m + 1.0;
    // Quads are shifted by `sh` so that 4 consecutive genes are exactly one
    // Philox block of the crossed stream (and of every stream whose offset is
    // congruent mod 4): one block per stream per quad instead of up to two.
    const uint64_t avail = (uint64_t)(4 - ph.pos);
    const int sh = (int)((o_cross + (uint64_t)q * d + 4 * 1024 - avail) & 3);  // genes before 1st boundary
    const int64_t first = -sh;  // quad t covers genes [first + 4t, first + 4t + 4)
    for (int64_t g0 = first + 4 * (int64_t)threadIdx.x; g0 < d; g0 += 4 * VT) {
        const int64_t ga = g0 < 0 ? 0 : g0;
        const int cnt = (int)((g0 + 4 < d ? g0 + 4 : d) - ga);
        double c1[4], c2[4];
        const uint64_t es = (uint64_t)q * d + ga;
        // SBX (variation.py:72-91): crossed first, mu/swap only where crossed
        double crs[4] = {0.0, 0.0, 0.0, 0.0};
        bool any = !V.gene_swap;
        if (V.gene_swap) {
            uniforms4(ph, o_cross + es, cnt, crs);
#pragma unroll
            for (int k = 0; k < 4; ++k) any |= (k < cnt) && crs[k] < 0.5;
        }
        double mu[4] = {0.0, 0.0, 0.0, 0.0}, sw[4] = {1.0, 1.0, 1.0, 1.0};
        if (any) {
            uniforms4(ph, o_mu + es, cnt, mu);
            if (V.gene_swap) uniforms4(ph, o_swap + es, cnt, sw);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (k < cnt) {
                const int64_t g = ga + k;
                const double lo = V.lower[g], hi = V.upper[g];
                sbx_gene(x1[g], x2[g], mu[k], sw[k], crs[k], e, V.gene_swap != 0, c1[k], c2[k]);
                c1[k] = clipv(c1[k], lo, hi);
                c2[k] = clipv(c2[k], lo, hi);
            }
        }
        // polynomial mutation (variation.py:104-120) on rows q (c1) and h+q (c2)
        double hit[4];
        uniforms4(ph, o_hit + es, cnt, hit);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (k < cnt && V.p_m - hit[k] >= 0.0) {  // PM only where hit (rate p_m)
                const int64_t g = ga + k;
                c1[k] = clipv(pm_step(c1[k], V.lower[g], V.upper[g], uniform1(ph, o_pmu + es + k), eta),
                              V.lower[g], V.upper[g]);
            }
        }
        if (!single) {
            const uint64_t e2 = (uint64_t)(h + q) * d + ga;
            uniforms4(ph, o_hit + e2, cnt, hit);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (k < cnt && V.p_m - hit[k] >= 0.0) {
                    const int64_t g = ga + k;
                    c2[k] = clipv(pm_step(c2[k], V.lower[g], V.upper[g], uniform1(ph, o_pmu + e2 + k), eta),
                                  V.lower[g], V.upper[g]);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (k < cnt) {
                o1[ga + k] = c1[k];
                if (!single) o2[ga + k] = c2[k];
                if (smem_rows) {
                    srow[ga + k] = c1[k];
                    if (!single) srow[d + ga + k] = c2[k];
                }
            }
    }
    if (!FO) return;
    __syncthreads();
    const double *r1 = smem_rows ? srow : o1;
    const double *r2 = smem_rows ? srow + d : o2;
    eval_row<M>(P, r1, f, red);
    __syncthreads();
    if (threadIdx.x < M) FO[q * M + threadIdx.x] = f[threadIdx.x];
    if (single) return;
    __syncthreads();
    eval_row<M>(P, r2, f, red);
    __syncthreads();
    if (threadIdx.x < M) FO[(h + q) * M + threadIdx.x] = f[threadIdx.x];
}

// ------------------------------------------------- fused offspring, warp per pair
// One warp owns a parent pair; lane t owns the Philox-aligned gene quad
// [4t - sh, 4t - sh + 4) (+128 per round), so every stream's 4 uniforms are
// exactly one Philox block (valid when h*d % 4 == 0, i.e. all streams are
// congruent mod 4).  Straight-line per quad: 3 (SBX) + 2 (PM hit) blocks;
// crossed/swap draws reduce to the raw word's top bit (U < 0.5 <=> raw < 2^63);
// pow only on crossed genes (one call site per gene); PM only where hit.
// Children go to O as they are made; the objective accumulation (LSMOP1 group
// sums with x_1 broadcast from lane 0, or the DTLZ g sum) is a per-lane
// partial reduced with warp shuffles -- no CTA barriers.
#ifndef OFF_LOCKSTEP
#define OFF_LOCKSTEP 1
#endif
#ifndef OFF_EXPLOG
#define OFF_EXPLOG 0
#endif
#ifndef OFF_ACC_QUAD
#define OFF_ACC_QUAD 0
#endif
#ifndef OFF_OW
#define OFF_OW 8
#endif
#ifndef OFF_MINB
#define OFF_MINB 2
#endif
constexpr int OW = OFF_OW;  // pairs (warps) per CTA

// the 4 raw words of stream elements [e, e + 4) where (e - avail) % 4 == 0 (or e < avail)
__device__ __forceinline__ void raw_quad(const Philox &ph, int64_t e, int64_t avail, uint64_t r[4]) {
    if (e >= avail) {
        uint64_t c[1][4], o[1][4];
        ctr_add(ph.ctr, (uint64_t)((e - avail) >> 2) + 1, c[0]);
        philox_blocks_rk<1>(c, ph.rk, o);
#pragma unroll
        for (int k = 0; k < 4; ++k) r[k] = o[0][k];
    } else {  // head of the stream: buffered words of the host generator (negative e: masked genes)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t x = e + k;
            r[k] = (x >= 0 && x < avail) ? ph.buf[ph.pos + x] : 0ull;
        }
    }
}

// raw words of NS streams at elements E[s] (each aligned as in raw_quad), blocks in lockstep
template <int NS>
__device__ __forceinline__ void raw_quads(const Philox &ph, const int64_t E[NS], int64_t avail,
                                          uint64_t r[NS][4]) {
    bool head = false;
#pragma unroll
    for (int s = 0; s < NS; ++s) head |= E[s] < avail;
    if (!head) {
        uint64_t c[NS][4];
#pragma unroll
        for (int s = 0; s < NS; ++s) ctr_add(ph.ctr, (uint64_t)((E[s] - avail) >> 2) + 1, c[s]);
        philox_blocks_rk<NS>(c, ph.rk, r);
    } else {
#pragma unroll
        for (int s = 0; s < NS; ++s) raw_quad(ph, E[s], avail, r[s]);
    }
}

__device__ __forceinline__ double u01(uint64_t raw) {
    return (double)(raw >> 11) * (1.0 / 9007199254740992.0);
}

template <int M>
__device__ __forceinline__ void acc_gene(const temo_problem &P, int64_t g, double x, double x0,
                                         double part[M]) {
    if (P.id == TEMO_PROB_LSMOP1) {
        const int64_t rel = g - (M - 1);
        if (rel < 0 || rel >= P.offset[M]) return;
        const double xs = (1.0 + (double)(g + 1) / (double)P.d) * x - 10.0 * x0;
        const double sq = xs * xs;
#pragma unroll
        for (int i = 0; i < M; ++i)
            if (rel >= P.offset[i] && rel < P.offset[i + 1]) part[i] += sq;
        return;
    }
    if (g < M - 1) return;
    switch (P.id) {
        case 1:
        case 3: {
            const double z = x - 0.5;
            part[0] += z * z - cos(20.0 * PI * z);
            break;
        }
        case 2:
        case 4:
        case 5: {
            const double z = x - 0.5;
            part[0] += z * z;
            break;
        }
        case 6: part[0] += pow(x, 0.1); break;
        default: part[0] += x; break;
    }
}

// four consecutive genes [g, g+4) of one child; one group lookup when the quad lies in one group
template <int M>
__device__ __forceinline__ void acc_quad(const temo_problem &P, int64_t g, const double x[4],
                                         const bool ok[4], bool full, double x0, double part[M]) {
    if (P.id == TEMO_PROB_LSMOP1 && full) {
        const int64_t rel = g - (M - 1);
        int grp = -1;
#pragma unroll
        for (int i = 0; i < M; ++i)
            if (rel >= P.offset[i] && rel + 3 < P.offset[i + 1]) grp = i;
        if (grp >= 0) {
            const double inv_d = 1.0 / (double)P.d;
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const double xs = (1.0 + (double)(g + k + 1) * inv_d) * x[k] - 10.0 * x0;
                s += xs * xs;
            }
#pragma unroll
            for (int i = 0; i < M; ++i)
                if (i == grp) part[i] += s;
            return;
        }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (ok[k]) acc_gene<M>(P, g + k, x[k], x0, part);
}

// objectives from the reduced sums (same formulas as eval_row); x = the child row
template <int M>
__device__ void finish_objs(const temo_problem &P, const double *x, const double part[M], double *f) {
    if (P.id == TEMO_PROB_LSMOP1) {
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const double gi = part[i] / (double)P.sublen[i] / (double)P.nk;
            double head = 1.0;
            for (int k = 0; k < M - 1 - i; ++k) head = head * x[k];
            const double tail = i == 0 ? 1.0 : 1.0 - x[M - 1 - i];
            f[i] = (1.0 + gi) * head * tail;
        }
        return;
    }
    const int id = P.id;
    const int64_t k = P.d - M + 1;
    const double s = part[0];
    double g;
    if (id == 1 || id == 3) g = 100.0 * ((double)k + s);
    else if (id == 7) g = 1.0 + 9.0 / (double)k * s;
    else g = s;
    if (id == 1) {
#pragma unroll
        for (int i = 0; i < M; ++i) {
            double p = 1.0;
            for (int q = 0; q < M - 1 - i; ++q) p = p * x[q];
            if (i) p = p * (1.0 - x[M - 1 - i]);
            f[i] = 0.5 * (1.0 + g) * p;
        }
        return;
    }
    if (id == 7) {
        double hsum = 0.0;
        for (int q = 0; q < M - 1; ++q) {
            f[q] = x[q];
            hsum += x[q] / (1.0 + g) * (1.0 + sin(3.0 * PI * x[q]));
        }
        f[M - 1] = (1.0 + g) * ((double)M - hsum);
        return;
    }
    double th[M];
#pragma unroll
    for (int q = 0; q < M - 1; ++q) {
        if (id == 4) th[q] = pow(x[q], 100.0) * (PI / 2.0);
        else if (id == 5 || id == 6) {
            if (q == 0) th[q] = x[0] * (PI / 2.0);
            else th[q] = PI / (4.0 * (1.0 + g)) * (1.0 + 2.0 * g * x[q]);
        } else th[q] = x[q] * (PI / 2.0);
    }
#pragma unroll
    for (int i = 0; i < M; ++i) {
        double p = 1.0;
        for (int q = 0; q < M - 1 - i; ++q) p = p * cos(th[q]);
        if (i) p = p * sin(th[M - 1 - i]);
        f[i] = (1.0 + g) * p;
    }
}

__device__ __forceinline__ uint64_t pick4u(const uint64_t v[4], int k) {
    return k == 0 ? v[0] : k == 1 ? v[1] : k == 2 ? v[2] : v[3];
}

__device__ __forceinline__ double pick4(const double v[4], int k) {
    return k == 0 ? v[0] : k == 1 ? v[1] : k == 2 ? v[2] : v[3];
}

template <int M, bool SWAP>
__global__ void __launch_bounds__(OW * 32, OFF_MINB) k_offspring_w(temo_problem P, VarArgs V,
                                                         const double *__restrict__ X,
                                                         const int64_t *__restrict__ i1,
                                                         const int64_t *__restrict__ i2, int64_t h,
                                                         Philox ph, uint64_t off,
                                                         double *__restrict__ O,
                                                         double *__restrict__ FO, int single) {
    const int lane = threadIdx.x & 31;
    const int64_t q = (int64_t)blockIdx.x * OW + (threadIdx.x >> 5);
    if (q >= h) return;
    const int64_t d = P.d;
    const double *x1 = X + i1[q] * d;
    const double *x2 = X + i2[q] * d;
    double *o1 = O + q * d;
    double *o2 = O + (h + q) * d;
    const int64_t hd = h * d;
    const int64_t o_mu = (int64_t)off, o_swap = o_mu + hd, o_cross = o_mu + (SWAP ? 2 * hd : 0);
    const int64_t o_pmu = o_mu + (SWAP ? 3 * hd : hd);
    const int64_t o_hit = o_pmu + (single ? hd : 2 * hd);
    const int64_t avail = 4 - ph.pos;
    const double e = 1.0 / (V.eta_c + 1.0);
    const double eta = V.eta_m + 1.0;
    // gene 0 sits at lane position sh of its Philox block (same for every stream)
    const int sh = (int)((o_mu + q * d - avail) & 3);
    double part1[M], part2[M];
#pragma unroll
    for (int i = 0; i < M; ++i) part1[i] = part2[i] = 0.0;
    double x0a = 0.0, x0b = 0.0;
    for (int64_t base = -sh; base < d; base += 128) {
        const int64_t gs = base + 4 * lane;
        const int64_t es = q * d + gs;  // stream element of gene gs (child 1 / pair index)
        // --- the quad's uniform streams, Philox blocks in lockstep groups:
        //     [cross, swap,] mu  then  hit c1, hit c2
        constexpr int NS = SWAP ? 5 : 3;
        uint64_t R[NS][4];
        {
            constexpr int NA = NS - 2;
            int64_t E[NA];
            if (SWAP) {
                E[0] = o_cross + es;
                E[1] = o_swap + es;
            }
            E[NA - 1] = o_mu + es;
            const int64_t EH[2] = {o_hit + es, o_hit + hd + es};  // (second unused in single mode)
#if OFF_LOCKSTEP == 2
            {
                int64_t EA[NS];
#pragma unroll
                for (int t = 0; t < NA; ++t) EA[t] = E[t];
                EA[NA] = EH[0];
                EA[NA + 1] = EH[1];
                raw_quads<NS>(ph, EA, avail, R);
            }
#elif OFF_LOCKSTEP
            raw_quads<NA>(ph, E, avail, R);
            raw_quads<2>(ph, EH, avail, R + NA);
#else
#pragma unroll
            for (int t = 0; t < NA; ++t) raw_quad(ph, E[t], avail, R[t]);
            raw_quad(ph, EH[0], avail, R[NA]);
            raw_quad(ph, EH[1], avail, R[NA + 1]);
#endif
        }
        double a[4], b[4], c1[4], c2[4];
        bool ok[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t g = gs + k;
            ok[k] = g >= 0 && g < d;
            a[k] = ok[k] ? __ldg(x1 + g) : 0.0;
            b[k] = ok[k] ? __ldg(x2 + g) : 0.0;
        }
        // --- SBX (variation.py:72-91)
        uint32_t crossed = 0xF, negate = 0;
        if (SWAP) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                crossed &= ~((uint32_t)(R[0][k] >> 63) << k);  // U < 0.5 <=> top bit 0
                negate |= (uint32_t)(1u - (uint32_t)(R[1][k] >> 63)) << k;
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t g = gs + k;
            double y1 = a[k], y2 = b[k];
            if ((crossed >> k) & 1) {
                // pow(2 mu, e) or pow(1 / (2 - 2 mu), e) as exp(+-e log(.)): e = 1/(eta_c+1) is
                // small, so plain double log/exp keep ~1 ulp (children agree to rtol 1e-13)
                const double mu = u01(R[NS - 3][k]);
#if OFF_EXPLOG
                const double beta0 = (0.5 - mu >= 0.0) ? exp(e * log(2.0 * mu)) : exp(-e * log(2.0 - 2.0 * mu));
#elif OFF_ABL_POW
                const double beta0 = (0.5 - mu >= 0.0) ? 2.0 * mu : 1.0 / (2.0 - 2.0 * mu);
#else
                const double beta0 = sbx_beta_any(mu, e);
#endif
                const double beta = SWAP ? beta0 * (1.0 - 2.0 * (double)((negate >> k) & 1)) : beta0;
                const double shift = 0.5 * (1.0 - beta);
                y1 = a[k] + shift * (b[k] - a[k]);
                y2 = b[k] + shift * (a[k] - b[k]);
            }
            if (ok[k]) {
                const double lo = __ldg(V.lower + g), hi = __ldg(V.upper + g);
                y1 = clipv(y1, lo, hi);
                y2 = clipv(y2, lo, hi);
            }
            c1[k] = y1;
            c2[k] = y2;
        }
        // --- polynomial mutation (variation.py:104-120), only where hit
        {
            uint32_t hit = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                hit |= (uint32_t)(ok[k] && V.p_m - u01(R[NS - 2][k]) >= 0.0) << k;
                if (!single) hit |= (uint32_t)(ok[k] && V.p_m - u01(R[NS - 1][k]) >= 0.0) << (4 + k);
            }
            if (hit) {
                uint64_t m1[4], m2[4];
                if (hit & 0xF) raw_quad(ph, o_pmu + es, avail, m1);
                if (hit & 0xF0) raw_quad(ph, o_pmu + hd + es, avail, m2);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int64_t g = gs + k;
                    if ((hit >> k) & 1) {
                        const double lo = V.lower[g], hi = V.upper[g];
                        c1[k] = clipv(pm_step(c1[k], lo, hi, u01(m1[k]), eta), lo, hi);
                    }
                    if ((hit >> (4 + k)) & 1) {
                        const double lo = V.lower[g], hi = V.upper[g];
                        c2[k] = clipv(pm_step(c2[k], lo, hi, u01(m2[k]), eta), lo, hi);
                    }
                }
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (ok[k]) {
                o1[gs + k] = c1[k];
                if (!single) o2[gs + k] = c2[k];
            }
        if (!FO) continue;
        if (base == -sh) {  // first round: lane 0 holds gene 0 at quad position sh
            x0a = __shfl_sync(~0u, pick4(c1, sh), 0);
            x0b = __shfl_sync(~0u, pick4(c2, sh), 0);
        }
        const bool full = gs >= 0 && gs + 4 <= d;
#if OFF_ABL_EVAL
        (void)full;
#elif OFF_ACC_QUAD
        acc_quad<M>(P, gs, c1, ok, full, x0a, part1);
        if (!single) acc_quad<M>(P, gs, c2, ok, full, x0b, part2);
#else
        (void)full;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (ok[k]) {
                acc_gene<M>(P, gs + k, c1[k], x0a, part1);
                if (!single) acc_gene<M>(P, gs + k, c2[k], x0b, part2);
            }
#endif
    }
    if (!FO) return;
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
        for (int s = 16; s; s >>= 1) {
            part1[i] += __shfl_xor_sync(~0u, part1[i], s);
            part2[i] += __shfl_xor_sync(~0u, part2[i], s);
        }
    __syncwarp();
    if (lane == 0) {
        double f[M];
        finish_objs<M>(P, o1, part1, f);
#pragma unroll
        for (int i = 0; i < M; ++i) FO[q * M + i] = f[i];
    } else if (lane == 1 && !single) {
        double f[M];
        finish_objs<M>(P, o2, part2, f);
#pragma unroll
        for (int i = 0; i < M; ++i) FO[(h + q) * M + i] = f[i];
    }
}

// -------------------------------------- fused offspring, persistent warps
// k_offspring_s: the warp-per-pair scheme above, with
//   - per-gene constants (bounds, LSMOP linkage coefficient 1 + g/d and
//     group id) staged once per CTA in shared memory -- no per-gene DDIV;
//   - persistent warps looping over pairs (the staging is amortised);
//   - Philox blocks in two lockstep groups ([cross, swap,] mu | hit1, hit2);
//   - SBX pows compacted across the warp: only crossed genes (about half)
//     are queued in shared memory and every lane takes queue slots, so a
//     warp round issues ceil(#crossed/32) pows instead of 4.
#ifndef OFF_FAST_POW
#define OFF_FAST_POW 0
#endif
#ifndef OFF_CUDA_POW
#define OFF_CUDA_POW 1  // 0: the exp/log form of sbx_pow.cuh (measured no faster on B200)
#endif
#ifndef OFF_PREFETCH
#define OFF_PREFETCH 1
#endif
#ifndef OFF_S_MINB
#define OFF_S_MINB 2
#endif
constexpr int SW = 8;            // warps per CTA

// SBX spread factor of one crossed gene (variation.py:77-78); out of line so pow's
// internal registers do not inflate the register budget of the offspring kernel
static __device__ __noinline__ double sbx_beta(double mu, double e) {
#if OFF_CUDA_POW
    return pow((0.5 - mu >= 0.0) ? 2.0 * mu : 1.0 / (2.0 - 2.0 * mu), e);
#else
    return sbx_beta_fast(mu, e);  // exp/log form (sbx_pow.cuh)
#endif
}
constexpr int SMAX_D = 3000;     // genes staged in shared memory (else k_offspring_w)

// DEVST: the Philox state is read from device memory (st_dev) instead of the launch
// parameters, so a captured CUDA graph can replay the kernel with each generation's state
template <int M, bool SWAP, bool DEVST = false>
__global__ void __launch_bounds__(SW * 32, OFF_S_MINB) k_offspring_s(temo_problem P, VarArgs V,
                                                            const double *__restrict__ X,
                                                            const int64_t *__restrict__ i1,
                                                            const int64_t *__restrict__ i2, int64_t h,
                                                            const __grid_constant__ Philox ph_arg,
                                                            const temo_philox_state *__restrict__ st_dev,
                                                            uint64_t off,
                                                            double *__restrict__ O,
                                                            double *__restrict__ FO, int single) {
    extern __shared__ double ssm[];
    __shared__ Philox s_ph;
    if (DEVST && threadIdx.x == 0) s_ph = philox_from(*st_dev);  // published by the barrier below
    const Philox &ph = DEVST ? s_ph : ph_arg;
    const int64_t d = P.d;
    double *s_lo = ssm, *s_hi = ssm + d, *s_cf = ssm + 2 * d;
    double *s_q = ssm + 3 * d + (threadIdx.x >> 5) * 128;  // per-warp pow queue
    signed char *s_grp = reinterpret_cast<signed char *>(ssm + 3 * d + SW * 128);
    const bool lsmop = P.id == TEMO_PROB_LSMOP1;
    for (int64_t g = threadIdx.x; g < d; g += blockDim.x) {
        s_lo[g] = V.lower[g];
        s_hi[g] = V.upper[g];
        s_cf[g] = 1.0 + (double)(g + 1) / (double)d;
        int grp = -1;
        const int64_t rel = g - (M - 1);
        if (lsmop) {
            for (int i = 0; i < M; ++i)
                if (rel >= P.offset[i] && rel < P.offset[i + 1]) grp = i;
        } else if (rel >= 0) {
            grp = 0;
        }
        s_grp[g] = (signed char)grp;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t hd = h * d;
    const int64_t o_mu = (int64_t)off, o_swap = o_mu + hd, o_cross = o_mu + (SWAP ? 2 * hd : 0);
    const int64_t o_pmu = o_mu + (SWAP ? 3 * hd : hd);
    const int64_t o_hit = o_pmu + (single ? hd : 2 * hd);
    const int64_t avail = 4 - ph.pos;
    const double e = 1.0 / (V.eta_c + 1.0);
    const double eta = V.eta_m + 1.0;
    const uint32_t lt_mask = (1u << lane) - 1u;
    // U = k 2^-53 <= p_m  <=>  k <= floor(p_m 2^53)  (p_m - U >= 0 is exact for doubles)
    int64_t pm_thr = -1;
    if (V.p_m >= 1.0) pm_thr = INT64_MAX;
    else if (V.p_m >= 0.0) pm_thr = (int64_t)floor(V.p_m * 9007199254740992.0);
    for (int64_t q = (int64_t)blockIdx.x * SW + (threadIdx.x >> 5); q < h; q += (int64_t)gridDim.x * SW) {
        const double *x1 = X + i1[q] * d;
        const double *x2 = X + i2[q] * d;
        double *o1 = O + q * d;
        double *o2 = O + (h + q) * d;
        const int sh = (int)((o_mu + q * d - avail) & 3);
        double part1[M], part2[M];
#pragma unroll
        for (int i = 0; i < M; ++i) part1[i] = part2[i] = 0.0;
        double x0a = 0.0, x0b = 0.0;
        for (int64_t base = -sh; base < d; base += 128) {
            const int64_t gs = base + 4 * lane;
            const int64_t es = q * d + gs;
            // parents' quads: prefetched into L1 now (no registers held), loaded after the randomness
#if OFF_PREFETCH
            if (gs >= 0 && gs < d) {
                asm volatile("prefetch.global.L1 [%0];" ::"l"(x1 + gs));
                asm volatile("prefetch.global.L1 [%0];" ::"l"(x2 + gs));
            }
#endif
            // randomness first, in phases that keep few raw words live:
            //   cross/swap (top bits) -> mu of crossed genes into the warp's pow queue -> hit bits
            bool ok[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) ok[k] = gs + k >= 0 && gs + k < d;
            uint32_t crossed = 0xF, negate = 0;
            if (SWAP) {
                uint64_t R[2][4];
                const int64_t E[2] = {o_cross + es, o_swap + es};
                raw_quads<2>(ph, E, avail, R);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    crossed &= ~((uint32_t)(R[0][k] >> 63) << k);  // U < 0.5 <=> top bit 0
                    negate |= (uint32_t)(1u - (uint32_t)(R[1][k] >> 63)) << k;
                }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) crossed &= (uint32_t)ok[k] << k | ~(1u << k);
            const int nq = __popc(crossed);
            int incl = nq;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(~0u, incl, o);
                if (lane >= o) incl += y;
            }
            const int total = __shfl_sync(~0u, incl, 31);
            int slot = incl - nq;
            {
                uint64_t R[1][4];
                const int64_t E[1] = {o_mu + es};
                raw_quads<1>(ph, E, avail, R);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if ((crossed >> k) & 1) s_q[slot++] = u01(R[0][k]);
            }
            uint32_t hit = 0;  // PM hit (p_m - U >= 0) as an integer test on the raw word
            {
                uint64_t R[2][4];
                const int64_t E[2] = {o_hit + es, o_hit + hd + es};  // (second unused in single mode)
                raw_quads<2>(ph, E, avail, R);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    hit |= (uint32_t)(ok[k] && (int64_t)(R[0][k] >> 11) <= pm_thr) << k;
                    if (!single) hit |= (uint32_t)(ok[k] && (int64_t)(R[1][k] >> 11) <= pm_thr) << (4 + k);
                }
            }
            __syncwarp();
#if OFF_FAST_POW
            for (int t = lane; t < total; t += 32) s_q[t] = sbx_beta_fast(s_q[t], e);
#else
            for (int t = lane; t < total; t += 32) s_q[t] = sbx_beta(s_q[t], e);
#endif
            __syncwarp();
            double a[4], b[4], c1[4], c2[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                a[k] = ok[k] ? __ldg(x1 + gs + k) : 0.0;
                b[k] = ok[k] ? __ldg(x2 + gs + k) : 0.0;
            }
            slot = incl - nq;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int64_t g = gs + k;
                double y1 = a[k], y2 = b[k];
                if ((crossed >> k) & 1) {
                    const double beta0 = s_q[slot++];
                    const double beta = SWAP ? beta0 * (1.0 - 2.0 * (double)((negate >> k) & 1)) : beta0;
                    const double shift = 0.5 * (1.0 - beta);
                    y1 = a[k] + shift * (b[k] - a[k]);
                    y2 = b[k] + shift * (a[k] - b[k]);
                }
                if (ok[k]) {
                    const double lo = s_lo[g], hi = s_hi[g];
                    y1 = clipv(y1, lo, hi);
                    y2 = clipv(y2, lo, hi);
                }
                c1[k] = y1;
                c2[k] = y2;
            }
            __syncwarp();  // s_q reused next round
            (void)lt_mask;
            // --- polynomial mutation (variation.py:104-120), only where hit
            if (hit) {
                uint64_t m1[4], m2[4];
                if (hit & 0xF) raw_quad(ph, o_pmu + es, avail, m1);
                if (hit & 0xF0) raw_quad(ph, o_pmu + hd + es, avail, m2);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int64_t g = gs + k;
                    if ((hit >> k) & 1)
                        c1[k] = clipv(pm_step(c1[k], s_lo[g], s_hi[g], u01(m1[k]), eta), s_lo[g], s_hi[g]);
                    if ((hit >> (4 + k)) & 1)
                        c2[k] = clipv(pm_step(c2[k], s_lo[g], s_hi[g], u01(m2[k]), eta), s_lo[g], s_hi[g]);
                }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (ok[k]) {
                    o1[gs + k] = c1[k];
                    if (!single) o2[gs + k] = c2[k];
                }
            if (!FO) continue;
            if (base == -sh) {  // lane 0 holds gene 0 at quad position sh
                x0a = __shfl_sync(~0u, pick4(c1, sh), 0);
                x0b = __shfl_sync(~0u, pick4(c2, sh), 0);
            }
            if (lsmop) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int grp = ok[k] ? (int)s_grp[gs + k] : -1;
                    if (grp < 0) continue;
                    const double cf = s_cf[gs + k];
                    const double xa = cf * c1[k] - 10.0 * x0a;
                    const double sa = xa * xa;
                    const double xb = cf * c2[k] - 10.0 * x0b;
                    const double sb = xb * xb;
#pragma unroll
                    for (int i = 0; i < M; ++i) {
                        if (grp == i) {
                            part1[i] += sa;
                            if (!single) part2[i] += sb;
                        }
                    }
                }
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (ok[k]) {
                        acc_gene<M>(P, gs + k, c1[k], x0a, part1);
                        if (!single) acc_gene<M>(P, gs + k, c2[k], x0b, part2);
                    }
            }
        }
        if (!FO) continue;
#pragma unroll
        for (int i = 0; i < M; ++i)
#pragma unroll
            for (int s = 16; s; s >>= 1) {
                part1[i] += __shfl_xor_sync(~0u, part1[i], s);
                part2[i] += __shfl_xor_sync(~0u, part2[i], s);
            }
        __syncwarp();
        if (lane == 0) {
            double f[M];
            finish_objs<M>(P, o1, part1, f);
#pragma unroll
            for (int i = 0; i < M; ++i) FO[q * M + i] = f[i];
        } else if (lane == 1 && !single) {
            double f[M];
            finish_objs<M>(P, o2, part2, f);
#pragma unroll
            for (int i = 0; i < M; ++i) FO[(h + q) * M + i] = f[i];
        }
    }
}

// ---------------------------------------------- two-phase offspring (ws)
// Phase 1 `k_offspring_rand`: pure randomness, no population traffic.  Warp per
// pair, lane per Philox-aligned quad as above; per quad it emits one flag word
// (crossed | hit c1 << 4 | hit c2 << 8) and, for crossed genes, beta (sign of
// the swap folded in) into a pair-major array.  The SBX pows of a warp round
// are queued (gene, mu) in shared memory and spread over all lanes, each lane
// writing its results straight to global memory.  Small register footprint ->
// high occupancy for the serial Philox and pow chains.
// Phase 2 `k_offspring_apply`: parents, flags and betas in, children and
// objectives out (PM's rare mu draws on the spot) -- a streaming kernel.
#ifndef OFF_APPLY_PREFETCH
#define OFF_APPLY_PREFETCH 0
#endif
#ifndef OFF_RAND_MINB
#define OFF_RAND_MINB 4
#endif
#ifndef OFF_RAND_ONEGROUP
#define OFF_RAND_ONEGROUP 1  // measured: rand 2.36 vs 2.39 ms at pop 200k (MINB 3: 2.43)
#endif
#ifndef OFF_APPLY_MINB
#define OFF_APPLY_MINB 2
#endif
#ifndef OFF_APPLY_IDXPF
#define OFF_APPLY_IDXPF 1
#endif
#ifndef OFF_APPLY_BQALL
#define OFF_APPLY_BQALL 1
#endif
#ifndef OFF_APPLY_CSTORE
#define OFF_APPLY_CSTORE 0
#endif
constexpr int RW = 8;  // warps per CTA of both phases

__host__ __device__ inline int64_t quads_per_pair(int64_t d) { return (d + 3) / 4 + 1; }
// per-pair stride of the flag rows: a multiple of 8 flags (16 bytes) so one pair's flags are one bulk copy
__host__ __device__ inline int64_t flag_stride(int64_t d) { return (quads_per_pair(d) + 7) & ~(int64_t)7; }

template <bool SWAP>
__global__ void __launch_bounds__(RW * 32, OFF_RAND_MINB) k_offspring_rand(int64_t d, VarArgs V, int64_t h,
                                                               int64_t q0, int64_t q1, Philox ph,
                                                               uint64_t off, int single,
                                                               double *__restrict__ beta,
                                                               uint16_t *__restrict__ flags) {
    __shared__ double s_mu[RW][128];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t hd = h * d;
    const int64_t o_mu = (int64_t)off, o_swap = o_mu + hd, o_cross = o_mu + (SWAP ? 2 * hd : 0);
    const int64_t o_pmu = o_mu + (SWAP ? 3 * hd : hd);
    const int64_t o_hit = o_pmu + (single ? hd : 2 * hd);
    const int64_t avail = 4 - ph.pos;
    const double e = 1.0 / (V.eta_c + 1.0);
    int64_t pm_thr = -1;
    if (V.p_m >= 1.0) pm_thr = INT64_MAX;
    else if (V.p_m >= 0.0) pm_thr = (int64_t)floor(V.p_m * 9007199254740992.0);
    const int64_t QP = quads_per_pair(d);
    // work unit = (pair, 128-gene chunk): short units let a high-priority stream's kernels take
    // SMs back quickly when this kernel overlaps the previous generation's selection
    const int64_t NC = (d + 3 + 127) / 128;
    const int64_t units = (q1 - q0) * NC;
    for (int64_t u = (int64_t)blockIdx.x * RW + warp; u < units; u += (int64_t)gridDim.x * RW) {
        const int64_t q = q0 + u / NC, c = u % NC;
        const int sh = (int)((o_mu + q * d - avail) & 3);
        double *bq = beta + q * d;
        {
            const int64_t base = -sh + 128 * c, j0 = 32 * c;
            if (base >= d) continue;
            const int64_t gs = base + 4 * lane;
            const int64_t es = q * d + gs;
            uint32_t okm = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) okm |= (uint32_t)(gs + k >= 0 && gs + k < d) << k;
            uint32_t crossed = okm, negate = 0;
#if OFF_RAND_ONEGROUP
            // all streams of the quad in one lockstep group (more ILP, more registers)
            constexpr int NS = SWAP ? 5 : 3;
            uint64_t RA[NS][4];
            {
                int64_t E[NS];
                if (SWAP) { E[0] = o_cross + es; E[1] = o_swap + es; }
                E[NS - 3] = o_mu + es;
                E[NS - 2] = o_hit + es;
                E[NS - 1] = o_hit + hd + es;  // (unused in single mode)
                raw_quads<NS>(ph, E, avail, RA);
            }
            if (SWAP) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    crossed &= ~((uint32_t)(RA[0][k] >> 63) << k);
                    negate |= (uint32_t)(1u - (uint32_t)(RA[SWAP ? 1 : 0][k] >> 63)) << k;
                }
            }
#else
            if (SWAP) {
                uint64_t R[2][4];
                const int64_t E[2] = {o_cross + es, o_swap + es};
                raw_quads<2>(ph, E, avail, R);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    crossed &= ~((uint32_t)(R[0][k] >> 63) << k);
                    negate |= (uint32_t)(1u - (uint32_t)(R[1][k] >> 63)) << k;
                }
            }
#endif
            const int nq = __popc(crossed);
            int incl = nq;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(~0u, incl, o);
                if (lane >= o) incl += y;
            }
            const int total = __shfl_sync(~0u, incl, 31);
#if OFF_RAND_ONEGROUP
            {
                int slot = incl - nq;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if ((crossed >> k) & 1) s_mu[warp][slot++] = u01(RA[NS - 3][k]);
            }
            uint32_t hit = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                hit |= (uint32_t)(((okm >> k) & 1) && (int64_t)(RA[NS - 2][k] >> 11) <= pm_thr) << k;
                if (!single) hit |= (uint32_t)(((okm >> k) & 1) && (int64_t)(RA[NS - 1][k] >> 11) <= pm_thr) << (4 + k);
            }
#else
            {
                uint64_t R[1][4];
                const int64_t E[1] = {o_mu + es};
                raw_quads<1>(ph, E, avail, R);
                int slot = incl - nq;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if ((crossed >> k) & 1) s_mu[warp][slot++] = u01(R[0][k]);
            }
            uint32_t hit = 0;
            {
                uint64_t R[2][4];
                const int64_t E[2] = {o_hit + es, o_hit + hd + es};  // (second unused in single mode)
                raw_quads<2>(ph, E, avail, R);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    hit |= (uint32_t)(((okm >> k) & 1) && (int64_t)(R[0][k] >> 11) <= pm_thr) << k;
                    if (!single) hit |= (uint32_t)(((okm >> k) & 1) && (int64_t)(R[1][k] >> 11) <= pm_thr) << (4 + k);
                }
            }
#endif
            if (j0 + lane < QP) flags[q * flag_stride(d) + j0 + lane] = (uint16_t)(crossed | hit << 4);
            __syncwarp();
            for (int t = lane; t < total; t += 32) s_mu[warp][t] = sbx_beta(s_mu[warp][t], e);
            __syncwarp();
            // the owner lane writes its quad's 4 betas (uncrossed: 1), so every 32-byte sector
            // of the beta array is written whole (scattered 8-byte writes cost a DRAM read-modify-write)
            {
                int slot = incl - nq;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    double b = 1.0;
                    if ((crossed >> k) & 1) {
                        b = s_mu[warp][slot++];
                        if (SWAP && ((negate >> k) & 1)) b = -b;  // beta * (1 - 2 [swap])
                    }
                    if ((okm >> k) & 1) bq[gs + k] = b;
                }
            }
            __syncwarp();
        }
    }
}

template <int M, bool LSMOP>
__global__ void __launch_bounds__(RW * 32, OFF_APPLY_MINB) k_offspring_apply(temo_problem P, VarArgs V,
                                                                const double *__restrict__ X,
                                                                const int64_t *__restrict__ i1,
                                                                const int64_t *__restrict__ i2, int64_t h,
                                                                int64_t q0, int64_t q1,
                                                                Philox ph, uint64_t off, int swap,
                                                                const double *__restrict__ beta,
                                                                const uint16_t *__restrict__ flags,
                                                                double *__restrict__ O,
                                                                double *__restrict__ FO, int single,
                                                                const int64_t *__restrict__ src_map,
                                                                const int64_t *__restrict__ dst_rows) {
    extern __shared__ double ssm[];
    const int64_t d = P.d;
    double *s_lo = ssm, *s_hi = ssm + d, *s_cf = ssm + 2 * d;
    double *s_wb = ssm + 3 * d;  // OFF_APPLY_CSTORE: RW x 2 x 128 doubles
    signed char *s_grp = reinterpret_cast<signed char *>(ssm + 3 * d + (OFF_APPLY_CSTORE ? RW * 256 : 0));
    constexpr bool lsmop = LSMOP;
    for (int64_t g = threadIdx.x; g < d; g += blockDim.x) {
        s_lo[g] = V.lower[g];
        s_hi[g] = V.upper[g];
        s_cf[g] = 1.0 + (double)(g + 1) / (double)d;
        int grp = -1;
        const int64_t rel = g - (M - 1);
        if (lsmop) {
            for (int i = 0; i < M; ++i)
                if (rel >= P.offset[i] && rel < P.offset[i + 1]) grp = i;
        } else if (rel >= 0) {
            grp = 0;
        }
        s_grp[g] = (signed char)grp;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t hd = h * d;
    const int64_t o_mu = (int64_t)off;
    const int64_t o_pmu = o_mu + (swap ? 3 * hd : hd);
    const int64_t avail = 4 - ph.pos;
    const double eta = V.eta_m + 1.0;
    const int64_t QP = quads_per_pair(d);
    const int64_t qstride = (int64_t)gridDim.x * RW;
#if OFF_APPLY_IDXPF
    // index pipeline: pool rows of the next pair and raw parent indices of the one after are
    // loaded while this pair streams (no dependent-load chain at the start of a pair)
    int64_t qa = q0 + (int64_t)blockIdx.x * RW + (threadIdx.x >> 5);
    auto prow = [&](const int64_t *ix, int64_t qq) { return src_map ? src_map[ix[qq]] : ix[qq]; };
    auto drow = [&](int64_t r) { return dst_rows ? dst_rows[r] : r; };
    int64_t np1 = 0, np2 = 0, nd1 = 0, nd2 = 0, nr1 = 0, nr2 = 0;
    if (qa < q1) {
        np1 = prow(i1, qa);
        np2 = prow(i2, qa);
        nd1 = drow(qa);
        nd2 = drow(h + qa);
    }
    if (qa + qstride < q1) {
        nr1 = i1[qa + qstride];
        nr2 = i2[qa + qstride];
    }
#endif
    for (int64_t q = q0 + (int64_t)blockIdx.x * RW + (threadIdx.x >> 5); q < q1; q += qstride) {
        // row pool (harness): parents at physical rows src_map[i], children into rows dst_rows[r]
#if OFF_APPLY_IDXPF
        const int64_t p1 = np1, p2 = np2;
        double *o1 = O + nd1 * d;
        double *o2 = O + nd2 * d;
        if (q + qstride < q1) {
            np1 = src_map ? src_map[nr1] : nr1;
            np2 = src_map ? src_map[nr2] : nr2;
            nd1 = drow(q + qstride);
            nd2 = drow(h + q + qstride);
        }
        if (q + 2 * qstride < q1) {
            nr1 = i1[q + 2 * qstride];
            nr2 = i2[q + 2 * qstride];
        }
#else
        const int64_t p1 = src_map ? src_map[i1[q]] : i1[q];
        const int64_t p2 = src_map ? src_map[i2[q]] : i2[q];
        double *o1 = O + (dst_rows ? dst_rows[q] : q) * d;
        double *o2 = O + (dst_rows ? dst_rows[h + q] : h + q) * d;
#endif
        const double *x1 = X + p1 * d;
        const double *x2 = X + p2 * d;
        const double *bq = beta + q * d;
        const int sh = (int)((o_mu + q * d - avail) & 3);
        double part1[M], part2[M];
#pragma unroll
        for (int i = 0; i < M; ++i) part1[i] = part2[i] = 0.0;
        double x0a = 0.0, x0b = 0.0;
        for (int64_t base = -sh, j0 = 0; base < d; base += 128, j0 += 32) {
            const int64_t gs = base + 4 * lane;
            const int64_t es = q * d + gs;
#if OFF_APPLY_PREFETCH
            {  // next round's parent and beta quads into L1 (no registers held)
                const int64_t gn = gs + 128;
                if (gn < d) {
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(x1 + gn));
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(x2 + gn));
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(bq + gn));
                }
            }
#endif
            const uint32_t fl = (j0 + lane < QP) ? flags[q * flag_stride(d) + j0 + lane] : 0u;
            const uint32_t crossed = fl & 0xF, hit = (fl >> 4) & 0xFF;
            double c1[4], c2[4];
            bool ok[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int64_t g = gs + k;
                ok[k] = g >= 0 && g < d;
                const double a = ok[k] ? __ldg(x1 + g) : 0.0;
                const double b = ok[k] ? __ldg(x2 + g) : 0.0;
#if OFF_APPLY_BQALL
                const double bb = ok[k] ? __ldg(bq + g) : 0.0;  // same sectors either way: issue with a, b
#endif
                double y1 = a, y2 = b;
                if ((crossed >> k) & 1) {
#if OFF_APPLY_BQALL
                    const double shift = 0.5 * (1.0 - bb);
#else
                    const double shift = 0.5 * (1.0 - __ldg(bq + g));
#endif
                    y1 = a + shift * (b - a);
                    y2 = b + shift * (a - b);
                }
                if (ok[k]) {
                    y1 = clipv(y1, s_lo[g], s_hi[g]);
                    y2 = clipv(y2, s_lo[g], s_hi[g]);
                }
                c1[k] = y1;
                c2[k] = y2;
            }
            if (hit) {  // polynomial mutation (variation.py:104-120), only where hit
                uint64_t m1[4], m2[4];
                if (hit & 0xF) raw_quad(ph, o_pmu + es, avail, m1);
                if (hit & 0xF0) raw_quad(ph, o_pmu + hd + es, avail, m2);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int64_t g = gs + k;
                    if ((hit >> k) & 1)
                        c1[k] = clipv(pm_step(c1[k], s_lo[g], s_hi[g], u01(m1[k]), eta), s_lo[g], s_hi[g]);
                    if ((hit >> (4 + k)) & 1)
                        c2[k] = clipv(pm_step(c2[k], s_lo[g], s_hi[g], u01(m2[k]), eta), s_lo[g], s_hi[g]);
                }
            }
#if OFF_APPLY_CSTORE
            {  // children through a per-warp staging row: 256-byte coalesced stores (8 full sectors)
                // instead of lane-strided quads (32 partial sectors per store instruction)
                double *w1 = s_wb + (int64_t)(threadIdx.x >> 5) * 256, *w2 = w1 + 128;
                __syncwarp();
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    w1[4 * lane + k] = c1[k];
                    w2[4 * lane + k] = c2[k];
                }
                __syncwarp();
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int64_t g = base + lane + 32 * i;
                    if (g >= 0 && g < d) {
                        o1[g] = w1[lane + 32 * i];
                        if (!single) o2[g] = w2[lane + 32 * i];
                    }
                }
            }
#else
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (ok[k]) {
                    o1[gs + k] = c1[k];
                    if (!single) o2[gs + k] = c2[k];
                }
#endif
            if (!FO) continue;
            if (base == -sh) {
                x0a = __shfl_sync(~0u, pick4(c1, sh), 0);
                x0b = __shfl_sync(~0u, pick4(c2, sh), 0);
            }
            if constexpr (LSMOP) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int grp = ok[k] ? (int)s_grp[gs + k] : -1;
                    if (grp < 0) continue;
                    const double cf = s_cf[gs + k];
                    const double xa = cf * c1[k] - 10.0 * x0a;
                    const double sa = xa * xa;
                    const double xb = cf * c2[k] - 10.0 * x0b;
                    const double sb = xb * xb;
#pragma unroll
                    for (int i = 0; i < M; ++i)
                        if (grp == i) {
                            part1[i] += sa;
                            if (!single) part2[i] += sb;
                        }
                }
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (ok[k]) {
                        acc_gene<M>(P, gs + k, c1[k], x0a, part1);
                        if (!single) acc_gene<M>(P, gs + k, c2[k], x0b, part2);
                    }
            }
        }
        if (!FO) continue;
#pragma unroll
        for (int i = 0; i < M; ++i)
#pragma unroll
            for (int s = 16; s; s >>= 1) {
                part1[i] += __shfl_xor_sync(~0u, part1[i], s);
                part2[i] += __shfl_xor_sync(~0u, part2[i], s);
            }
        __syncwarp();
        if (lane == 0) {
            double f[M];
            finish_objs<M>(P, o1, part1, f);
#pragma unroll
            for (int i = 0; i < M; ++i) FO[q * M + i] = f[i];
        } else if (lane == 1 && !single) {
            double f[M];
            finish_objs<M>(P, o2, part2, f);
#pragma unroll
            for (int i = 0; i < M; ++i) FO[(h + q) * M + i] = f[i];
        }
    }
}

// ------------------------------------------------- apply phase, gene-major lanes (d >= 128)
// k_offspring_apply with lane t owning genes 128 r + 32 k + t (k = 0..3) instead of the
// Philox-aligned quad 4 t - sh: every global and shared access of the warp is a contiguous
// 256-byte run (2 L1 wavefronts) instead of a 32-byte-strided one (8 wavefronts) -- the
// quad kernel is L1-throughput bound (profiles/r02_ncu_D_offspring_apply_quad.txt: l1tex
// 62-73 % of peak, DRAM 36 %).  A gene's flag bits come from its stream quad
// (g + sh) >> 2 by warp shuffle; PM's rare draws use the same aligned Philox block.
// Children are bit-identical to the quad kernels; the objective sums run in another order.
template <int M, bool LSMOP>
__global__ void __launch_bounds__(RW * 32, OFF_APPLY_MINB) k_offspring_apply_t(temo_problem P, VarArgs V,
                                                                  const double *__restrict__ X,
                                                                  const int64_t *__restrict__ i1,
                                                                  const int64_t *__restrict__ i2, int64_t h,
                                                                  int64_t q0, int64_t q1,
                                                                  Philox ph, uint64_t off, int swap,
                                                                  const double *__restrict__ beta,
                                                                  const uint16_t *__restrict__ flags,
                                                                  double *__restrict__ O,
                                                                  double *__restrict__ FO,
                                                                  const int64_t *__restrict__ src_map,
                                                                  const int64_t *__restrict__ dst_rows) {
    extern __shared__ double tsm[];
    const int64_t d = P.d;
    double *s_lo = tsm, *s_hi = tsm + d, *s_cf = tsm + 2 * d;
    signed char *s_grp = reinterpret_cast<signed char *>(tsm + 3 * d);
    for (int64_t g = threadIdx.x; g < d; g += blockDim.x) {
        s_lo[g] = V.lower[g];
        s_hi[g] = V.upper[g];
        s_cf[g] = 1.0 + (double)(g + 1) / (double)d;
        int grp = -1;
        const int64_t rel = g - (M - 1);
        if (LSMOP) {
            for (int i = 0; i < M; ++i)
                if (rel >= P.offset[i] && rel < P.offset[i + 1]) grp = i;
        } else if (rel >= 0) {
            grp = 0;
        }
        s_grp[g] = (signed char)grp;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t hd = h * d;
    const int64_t o_mu = (int64_t)off;
    const int64_t o_pmu = o_mu + (swap ? 3 * hd : hd);
    const int64_t avail = 4 - ph.pos;
    const double eta = V.eta_m + 1.0;
    const int64_t QP = quads_per_pair(d), QS = flag_stride(d);
    const int64_t qstride = (int64_t)gridDim.x * RW;
    const int64_t qa = q0 + (int64_t)blockIdx.x * RW + (threadIdx.x >> 5);
    auto prow = [&](const int64_t *ix, int64_t qq) { return src_map ? src_map[ix[qq]] : ix[qq]; };
    auto drow = [&](int64_t r) { return dst_rows ? dst_rows[r] : r; };
    int64_t np1 = 0, np2 = 0, nd1 = 0, nd2 = 0, nr1 = 0, nr2 = 0;  // index pipeline (next pairs)
    if (qa < q1) {
        np1 = prow(i1, qa);
        np2 = prow(i2, qa);
        nd1 = drow(qa);
        nd2 = drow(h + qa);
    }
    if (qa + qstride < q1) {
        nr1 = i1[qa + qstride];
        nr2 = i2[qa + qstride];
    }
    for (int64_t q = qa; q < q1; q += qstride) {
        const double *x1 = X + np1 * d;
        const double *x2 = X + np2 * d;
        double *o1 = O + nd1 * d;
        double *o2 = O + nd2 * d;
        if (q + qstride < q1) {
            np1 = src_map ? src_map[nr1] : nr1;
            np2 = src_map ? src_map[nr2] : nr2;
            nd1 = drow(q + qstride);
            nd2 = drow(h + q + qstride);
        }
        if (q + 2 * qstride < q1) {
            nr1 = i1[q + 2 * qstride];
            nr2 = i2[q + 2 * qstride];
        }
        const double *bq = beta + q * d;
        const uint16_t *fq = flags + q * QS;
        const int sh = (int)((o_mu + q * d - avail) & 3);
        const int bit = (lane + sh) & 3;        // position of this lane's genes in their stream quads
        const int jl = (lane + sh) >> 2;        // quad of gene (32 k + lane) is 8 k + jl within the round
        double part1[M], part2[M];
#pragma unroll
        for (int i = 0; i < M; ++i) part1[i] = part2[i] = 0.0;
        double x0a = 0.0, x0b = 0.0;
        for (int64_t base = 0, j0 = 0; base < d; base += 128, j0 += 32) {
            const uint32_t fa = (j0 + lane < QP) ? fq[j0 + lane] : 0u;
            const uint32_t fb = (j0 + 32 < QP) ? fq[j0 + 32] : 0u;
            double a[4], b[4], bb[4];
            bool ok[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int64_t g = base + 32 * k + lane;
                ok[k] = g < d;
                a[k] = ok[k] ? __ldg(x1 + g) : 0.0;
                b[k] = ok[k] ? __ldg(x2 + g) : 0.0;
                bb[k] = ok[k] ? __ldg(bq + g) : 0.0;
            }
            double c1[4], c2[4];
            uint32_t hit = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int src = 8 * k + jl;  // <= 32
                const uint32_t w0 = __shfl_sync(~0u, fa, src & 31);
                const uint32_t w = src < 32 ? w0 : fb;
                const int64_t g = base + 32 * k + lane;
                double y1 = a[k], y2 = b[k];
                if ((w >> bit) & 1) {
                    const double shift = 0.5 * (1.0 - bb[k]);
                    y1 = a[k] + shift * (b[k] - a[k]);
                    y2 = b[k] + shift * (a[k] - b[k]);
                }
                if (ok[k]) {
                    y1 = clipv(y1, s_lo[g], s_hi[g]);
                    y2 = clipv(y2, s_lo[g], s_hi[g]);
                    hit |= ((w >> (4 + bit)) & 1u) << k;
                    hit |= ((w >> (8 + bit)) & 1u) << (4 + k);
                }
                c1[k] = y1;
                c2[k] = y2;
            }
            if (hit) {  // polynomial mutation (variation.py:104-120), only where hit
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (!((hit >> k) & 0x11)) continue;
                    const int64_t g = base + 32 * k + lane;
                    const int64_t es = q * d + g - bit;  // start of the gene's stream quad
                    if ((hit >> k) & 1) {
                        uint64_t m[4];
                        raw_quad(ph, o_pmu + es, avail, m);
                        c1[k] = clipv(pm_step(c1[k], s_lo[g], s_hi[g], u01(pick4u(m, bit)), eta), s_lo[g], s_hi[g]);
                    }
                    if ((hit >> (4 + k)) & 1) {
                        uint64_t m[4];
                        raw_quad(ph, o_pmu + hd + es, avail, m);
                        c2[k] = clipv(pm_step(c2[k], s_lo[g], s_hi[g], u01(pick4u(m, bit)), eta), s_lo[g], s_hi[g]);
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (ok[k]) {
                    o1[base + 32 * k + lane] = c1[k];
                    o2[base + 32 * k + lane] = c2[k];
                }
            if (!FO) continue;
            if (base == 0) {
                x0a = __shfl_sync(~0u, c1[0], 0);
                x0b = __shfl_sync(~0u, c2[0], 0);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (!ok[k]) continue;
                const int64_t g = base + 32 * k + lane;
                if constexpr (LSMOP) {
                    const int grp = (int)s_grp[g];
                    if (grp < 0) continue;
                    const double cf = s_cf[g];
                    const double xa = cf * c1[k] - 10.0 * x0a;
                    const double xb = cf * c2[k] - 10.0 * x0b;
#pragma unroll
                    for (int i = 0; i < M; ++i)
                        if (grp == i) {
                            part1[i] += xa * xa;
                            part2[i] += xb * xb;
                        }
                } else {
                    acc_gene<M>(P, g, c1[k], x0a, part1);
                    acc_gene<M>(P, g, c2[k], x0b, part2);
                }
            }
        }
        if (!FO) continue;
#pragma unroll
        for (int i = 0; i < M; ++i)
#pragma unroll
            for (int s = 16; s; s >>= 1) {
                part1[i] += __shfl_xor_sync(~0u, part1[i], s);
                part2[i] += __shfl_xor_sync(~0u, part2[i], s);
            }
        __syncwarp();
        if (lane == 0) {
            double f[M];
            finish_objs<M>(P, o1, part1, f);
#pragma unroll
            for (int i = 0; i < M; ++i) FO[q * M + i] = f[i];
        } else if (lane == 1) {
            double f[M];
            finish_objs<M>(P, o2, part2, f);
#pragma unroll
            for (int i = 0; i < M; ++i) FO[(h + q) * M + i] = f[i];
        }
    }
}

// ------------------------------------------------- apply phase, vector gene-major (d even)
// The apply phase's data movement runs at 6.2 TB/s as a plain warp-per-pair double2 stream
// (temo_probe_rows_rate: two gathered rows + one streamed row in, two scattered rows out) --
// at 64 warps/SM.  This kernel keeps that shape: lane t owns genes 64 s + 2 t + {0, 1}
// (16-byte loads and stores, every warp access one contiguous 512-byte run), registers are
// capped for 4 CTAs/SM, a gene's flag bits come from its stream quad (g + sh) >> 2 by warp
// shuffle and PM's rare draws from the same aligned Philox block (out of line).  Children are
// bit-identical to the quad kernels; the objective sums run in another order.  Measured at
// pop 200k (ms): quad kernel 1.41; this kernel 1.22 (3 CTAs/SM, PM out of line), 1.26 (4 CTAs/SM,
// spills), 1.36 / 1.28 with PM inlined (3 / 4 CTAs/SM); scalar gene-major 1.68; per-warp bulk
// ring 1.66; CTA-per-pair bulk stages 1.86; coalesced-store staging 1.48.
#ifndef OFF_APPLYV_MINB
#define OFF_APPLYV_MINB 3
#endif
#ifndef OFF_PMFIX_MINB
#define OFF_PMFIX_MINB 4
#endif

template <int M, bool LSMOP>
__global__ void __launch_bounds__(RW * 32, OFF_APPLYV_MINB) k_offspring_apply_v(temo_problem P, VarArgs V,
                                                                   const double *__restrict__ X,
                                                                   const int64_t *__restrict__ i1,
                                                                   const int64_t *__restrict__ i2, int64_t h,
                                                                   int64_t q0, int64_t q1,
                                                                   const __grid_constant__ Philox ph, uint64_t off, int swap,
                                                                   const double *__restrict__ beta,
                                                                   const uint16_t *__restrict__ flags,
                                                                   double *__restrict__ O,
                                                                   double *__restrict__ FO,
                                                                   const int64_t *__restrict__ src_map,
                                                                   const int64_t *__restrict__ dst_rows) {
    extern __shared__ __align__(16) double vsm[];
    const int64_t d = P.d;
    double *s_lo = vsm, *s_hi = vsm + d, *s_cf = vsm + 2 * d;
    signed char *s_grp = reinterpret_cast<signed char *>(vsm + 3 * d);
    for (int64_t g = threadIdx.x; g < d; g += blockDim.x) {
        s_lo[g] = V.lower[g];
        s_hi[g] = V.upper[g];
        s_cf[g] = 1.0 + (double)(g + 1) / (double)d;
        int grp = -1;
        const int64_t rel = g - (M - 1);
        if (LSMOP) {
            for (int i = 0; i < M; ++i)
                if (rel >= P.offset[i] && rel < P.offset[i + 1]) grp = i;
        } else if (rel >= 0) {
            grp = 0;
        }
        s_grp[g] = (signed char)grp;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t hd = h * d;
    const int64_t o_mu = (int64_t)off;
    const int64_t o_pmu = o_mu + (swap ? 3 * hd : hd);
    const int64_t avail = 4 - ph.pos;
    const double eta = V.eta_m + 1.0;
    const int64_t QP = quads_per_pair(d), QS = flag_stride(d);
    const int64_t d2 = d >> 1;
    for (int64_t q = q0 + (int64_t)blockIdx.x * RW + (threadIdx.x >> 5); q < q1; q += (int64_t)gridDim.x * RW) {
        const int64_t p1 = src_map ? src_map[i1[q]] : i1[q];
        const int64_t p2 = src_map ? src_map[i2[q]] : i2[q];
        const double2 *x1 = reinterpret_cast<const double2 *>(X + p1 * d);
        const double2 *x2 = reinterpret_cast<const double2 *>(X + p2 * d);
        const double2 *bq = reinterpret_cast<const double2 *>(beta + q * d);
        double2 *o1 = reinterpret_cast<double2 *>(O + (dst_rows ? dst_rows[q] : q) * d);
        double2 *o2 = reinterpret_cast<double2 *>(O + (dst_rows ? dst_rows[h + q] : h + q) * d);
        const uint16_t *fq = flags + q * QS;
        const int sh = (int)((o_mu + q * d - avail) & 3);
        double part1[M], part2[M];
#pragma unroll
        for (int i = 0; i < M; ++i) part1[i] = part2[i] = 0.0;
        double x0a = 0.0, x0b = 0.0;
        for (int64_t v0 = 0; v0 < d2; v0 += 32) {  // 64 genes per round: lane owns pair v = v0 + lane
            const int64_t v = v0 + lane;
            const bool ok = v < d2;
            const int64_t jq = (2 * v0) >> 2;           // first stream quad of the round (v0 % 32 == 0)
            const uint32_t fw = (lane <= 16 && jq + lane < QP) ? fq[jq + lane] : 0u;
            const double2 a = ok ? __ldg(x1 + v) : make_double2(0.0, 0.0);
            const double2 b = ok ? __ldg(x2 + v) : make_double2(0.0, 0.0);
            const double2 bb = ok ? __ldg(bq + v) : make_double2(0.0, 0.0);
            const int g0 = 2 * lane + sh;                 // round-relative stream position of gene 2v
            const uint32_t w0 = __shfl_sync(~0u, fw, g0 >> 2), w1 = __shfl_sync(~0u, fw, (g0 + 1) >> 2);
            const int b0 = g0 & 3, b1 = (g0 + 1) & 3;
            double y[2][2];
            const double av[2] = {a.x, a.y}, bv[2] = {b.x, b.y}, sv[2] = {bb.x, bb.y};
            uint32_t hitm = 0;  // bit 2 e + c: gene 2 v + e of child c is a PM hit
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const uint32_t w = e ? w1 : w0;
                const int bit = e ? b1 : b0;
                double y1 = av[e], y2 = bv[e];
                if ((w >> bit) & 1) {
                    const double shift = 0.5 * (1.0 - sv[e]);
                    y1 = av[e] + shift * (bv[e] - av[e]);
                    y2 = bv[e] + shift * (av[e] - bv[e]);
                }
                const int64_t g = 2 * v + e;
                if (ok) {
                    const double lo = s_lo[g], hi = s_hi[g];
                    y1 = clipv(y1, lo, hi);
                    y2 = clipv(y2, lo, hi);
                    // PM hits are applied by k_offspring_pm_fix (their terms are added there)
                    hitm |= ((w >> (4 + bit)) & 1u) << (2 * e);
                    hitm |= ((w >> (8 + bit)) & 1u) << (2 * e + 1);
                }
                y[0][e] = y1;
                y[1][e] = y2;
            }
            if (ok) {
                o1[v] = make_double2(y[0][0], y[0][1]);
                o2[v] = make_double2(y[1][0], y[1][1]);
            }
            if (!FO) continue;
            if (v0 == 0) {
                x0a = __shfl_sync(~0u, y[0][0], 0);
                x0b = __shfl_sync(~0u, y[1][0], 0);
            }
            if (!ok) continue;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int64_t g = 2 * v + e;
                const bool h1 = (hitm >> (2 * e)) & 1, h2 = (hitm >> (2 * e + 1)) & 1;
                if constexpr (LSMOP) {
                    const int grp = (int)s_grp[g];
                    if (grp < 0) continue;
                    const double cf = s_cf[g];
                    const double xa = cf * y[0][e] - 10.0 * x0a;
                    const double xb = cf * y[1][e] - 10.0 * x0b;
#pragma unroll
                    for (int i = 0; i < M; ++i)
                        if (grp == i) {
                            if (!h1) part1[i] += xa * xa;
                            if (!h2) part2[i] += xb * xb;
                        }
                } else {
                    if (!h1) acc_gene<M>(P, g, y[0][e], x0a, part1);
                    if (!h2) acc_gene<M>(P, g, y[1][e], x0b, part2);
                }
            }
        }
        if (!FO) continue;
#pragma unroll
        for (int i = 0; i < M; ++i)
#pragma unroll
            for (int s = 16; s; s >>= 1) {
                part1[i] += __shfl_xor_sync(~0u, part1[i], s);
                part2[i] += __shfl_xor_sync(~0u, part2[i], s);
            }
        if (lane == 0) {  // the group sums of the non-hit genes; k_offspring_pm_fix finishes them
#pragma unroll
            for (int i = 0; i < M; ++i) FO[q * M + i] = part1[i];
        } else if (lane == 1) {
#pragma unroll
            for (int i = 0; i < M; ++i) FO[(h + q) * M + i] = part2[i];
        }
    }
}

// Hit list of the PM pass: thread per (pair, stream quad); warp-aggregated append of
// (q << 13 | child << 12 | gene).  The counter keeps counting past the capacity (overflow ->
// the per-pair pass applies the PM itself).
static __global__ void __launch_bounds__(256) k_pm_list(int64_t d, int64_t h, int64_t q0, int64_t q1, uint64_t off,
                                                 int ph_pos, const uint16_t *__restrict__ flags,
                                                 int64_t *__restrict__ list, int64_t cap) {
    const int lane = threadIdx.x & 31;
    const int64_t QP = quads_per_pair(d), QS = flag_stride(d);
    const int64_t items = (q1 - q0) * QP;
    const int64_t avail = 4 - ph_pos;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < items; base += stride) {
        const int64_t it = base + threadIdx.x;
        int64_t q = 0, j = 0;
        uint32_t hit = 0;
        if (it < items) {
            q = q0 + it / QP;
            j = it % QP;
            hit = (flags[q * QS + j] >> 4) & 0xFF;
        }
        const int sh = (int)(((int64_t)off + q * d - avail) & 3);
        const int n = __popc(hit);
        int incl = n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(~0u, incl, o);
            if (lane >= o) incl += y;
        }
        const int total = __shfl_sync(~0u, incl, 31);
        if (total == 0) continue;
        unsigned long long b0 = 0;
        if (lane == 31) b0 = atomicAdd(reinterpret_cast<unsigned long long *>(list), (unsigned long long)total);
        b0 = __shfl_sync(~0u, b0, 31);
        int64_t w = (int64_t)b0 + incl - n;
        for (int k = 0; k < 8; ++k) {
            if (!((hit >> k) & 1)) continue;
            const int c = k >> 2;
            const int64_t g = 4 * j - sh + (k & 3);
            if (w < cap) list[1 + w] = (q << 13) | ((int64_t)c << 12) | g;
            ++w;
        }
    }
}

// PM of every listed hit (variation.py:104-120): its aligned Philox block, pm_step on the stored
// SBX child value, the write-back.  Each entry's result is independent of the list order.
static __global__ void __launch_bounds__(256) k_pm_apply(VarArgs V, int64_t d, int64_t h, const __grid_constant__ Philox ph,
                                                  uint64_t off, int swap, const int64_t *__restrict__ list, int64_t cap,
                                                  double *__restrict__ O, const int64_t *__restrict__ dst_rows) {
    const int64_t n = list[0];
    if (n > cap) return;  // overflow: the per-pair pass does it
    const int64_t hd = h * d;
    const int64_t o_mu = (int64_t)off;
    const int64_t o_pmu = o_mu + (swap ? 3 * hd : hd);
    const int64_t avail = 4 - ph.pos;
    const double eta = V.eta_m + 1.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = list[1 + i];
        const int64_t q = e >> 13, g = e & 0xFFF;
        const int c = (int)((e >> 12) & 1);
        const int sh = (int)((o_mu + q * d - avail) & 3);
        const int bit = (int)((g + sh) & 3);
        uint64_t mm[4];
        raw_quad(ph, o_pmu + (c ? hd : 0) + q * d + g - bit, avail, mm);
        const int64_t r = c ? h + q : q;
        double *y = O + (dst_rows ? dst_rows[r] : r) * d + g;
        const double lo = V.lower[g], hi = V.upper[g];
        *y = clipv(pm_step(*y, lo, hi, u01(pick4u(mm, bit)), eta), lo, hi);
    }
}

// PM pass after k_offspring_apply_v (warp per pair): for every hit gene of both children the
// PM draw (its aligned Philox block), pm_step on the stored SBX child value and the write-back,
// then the objectives from the apply kernel's sums plus the hit genes' terms.  A child whose
// gene 0 was hit (the LSMOP linkage uses it for every gene) has its sums recomputed from its
// row.  Children are bit-identical to the inline-PM kernels.
constexpr int PMFIX_QS = 768;  // flag_stride(d) for d <= 3000
template <int M, bool LSMOP>
__global__ void __launch_bounds__(RW * 32, OFF_PMFIX_MINB) k_offspring_pm_fix(temo_problem P, VarArgs V, int64_t h, int64_t q0,
                                                              int64_t q1, const __grid_constant__ Philox ph,
                                                              uint64_t off, int swap,
                                                              const uint16_t *__restrict__ flags,
                                                              double *__restrict__ O, double *__restrict__ FO,
                                                              const int64_t *__restrict__ dst_rows,
                                                              const int64_t *__restrict__ pm_list, int64_t pm_cap) {
    const bool applied = pm_list[0] <= pm_cap;  // k_pm_apply already wrote every hit's PM value
    if (applied && !FO) return;
    const int lane = threadIdx.x & 31;
    const int64_t d = P.d;
    const int64_t hd = h * d;
    const int64_t o_mu = (int64_t)off;
    const int64_t o_pmu = o_mu + (swap ? 3 * hd : hd);
    const int64_t avail = 4 - ph.pos;
    const double eta = V.eta_m + 1.0;
    const int64_t QP = quads_per_pair(d), QS = flag_stride(d);
    // the pair's flag row is staged in shared memory with 16-byte loads (one per lane for
    // d <= 1020) instead of 32 lane-strided 2-byte loads per round; same gene order after
    __shared__ __align__(16) uint16_t s_fl[RW][PMFIX_QS];
    const bool staged = QS <= PMFIX_QS;
    const int warp = threadIdx.x >> 5;
    for (int64_t q = q0 + (int64_t)blockIdx.x * RW + warp; q < q1; q += (int64_t)gridDim.x * RW) {
        const uint16_t *fq = flags + q * QS;
        if (staged) {
            const uint4 *src = reinterpret_cast<const uint4 *>(fq);
            uint4 *dst = reinterpret_cast<uint4 *>(s_fl[warp]);
            __syncwarp();  // every lane is done with the previous pair's row
            for (int64_t v = lane; v < QS / 8; v += 32) dst[v] = __ldg(src + v);
            __syncwarp();
            fq = s_fl[warp];
        }
        const int sh = (int)((o_mu + q * d - avail) & 3);
        double *orow[2] = {O + (dst_rows ? dst_rows[q] : q) * d, O + (dst_rows ? dst_rows[h + q] : h + q) * d};
        // gene 0 first (its final value enters every LSMOP term)
        const uint32_t f0 = fq[0];
        bool dirty[2];
        double x0[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            dirty[c] = (f0 >> (4 + 4 * c + sh)) & 1;
            if (dirty[c] && lane == 0 && !applied) {
                uint64_t mm[4];
                raw_quad(ph, o_pmu + (c ? hd : 0) + q * d - sh, avail, mm);
                const double lo = V.lower[0], hi = V.upper[0];
                orow[c][0] = clipv(pm_step(orow[c][0], lo, hi, u01(pick4u(mm, sh)), eta), lo, hi);
            }
        }
        __syncwarp();
#pragma unroll
        for (int c = 0; c < 2; ++c) x0[c] = orow[c][0];
        double t[2][M];
#pragma unroll
        for (int i = 0; i < M; ++i) t[0][i] = t[1][i] = 0.0;
        for (int64_t j = lane; j < QP; j += 32) {
            const uint32_t fl = fq[j];
            const uint32_t hit = (fl >> 4) & 0xFF;
            if (!hit) continue;
            const int64_t gs = 4 * j - sh;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                if (!((hit >> (4 * c)) & 0xF)) continue;
                uint64_t mm[4];
                if (!applied) raw_quad(ph, o_pmu + (c ? hd : 0) + q * d + gs, avail, mm);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int64_t g = gs + k;
                    if (!((hit >> (4 * c + k)) & 1) || g <= 0 || g >= d) continue;  // gene 0 done above
                    double y = orow[c][g];
                    if (!applied) {
                        const double lo = V.lower[g], hi = V.upper[g];
                        y = clipv(pm_step(y, lo, hi, u01(mm[k]), eta), lo, hi);
                        orow[c][g] = y;
                    }
                    if (!FO || dirty[c]) continue;
                    if constexpr (LSMOP) {
                        const int64_t rel = g - (M - 1);
                        const double xs = (1.0 + (double)(g + 1) / (double)d) * y - 10.0 * x0[c];
#pragma unroll
                        for (int i = 0; i < M; ++i)
                            if (rel >= P.offset[i] && rel < P.offset[i + 1]) t[c][i] += xs * xs;
                    } else {
                        acc_gene<M>(P, g, y, x0[c], t[c]);
                    }
                }
            }
        }
        if (!FO) continue;
        __syncwarp();
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            if (dirty[c]) {  // recompute this child's sums from its final row
#pragma unroll
                for (int i = 0; i < M; ++i) t[c][i] = 0.0;
                for (int64_t g = lane; g < d; g += 32) {
                    const double y = orow[c][g];
                    if constexpr (LSMOP) {
                        const int64_t rel = g - (M - 1);
                        if (rel < 0) continue;
                        const double xs = (1.0 + (double)(g + 1) / (double)d) * y - 10.0 * x0[c];
#pragma unroll
                        for (int i = 0; i < M; ++i)
                            if (rel >= P.offset[i] && rel < P.offset[i + 1]) t[c][i] += xs * xs;
                    } else {
                        acc_gene<M>(P, g, y, x0[c], t[c]);
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < M; ++i)
#pragma unroll
                for (int s = 16; s; s >>= 1) t[c][i] += __shfl_xor_sync(~0u, t[c][i], s);
        }
        if (lane < 2) {
            const int c = lane;
            double part[M], f[M];
            double *fo = FO + ((c ? h : 0) + q) * M;
#pragma unroll
            for (int i = 0; i < M; ++i) part[i] = (dirty[c] ? 0.0 : fo[i]) + t[c][i];
            finish_objs<M>(P, orow[c], part, f);
#pragma unroll
            for (int i = 0; i < M; ++i) fo[i] = f[i];
        }
    }
}

// ------------------------------------------------- apply phase, per-warp bulk ring (d even)
// k_offspring_apply with its loads moved off the critical path: each warp keeps a ring of
// OFF_RING_S stages in shared memory, and its lane 0 streams the next rounds' parent-row,
// spread-factor and flag chunks (<= 130 + 130 + 130 doubles + 32 flags per round) into it
// with cp.async.bulk on a per-stage mbarrier, crossing pair boundaries (the pool rows of the
// next pair are looked up one pair ahead).  Up to OFF_RING_S rounds per warp are in flight
// while it computes, instead of one.  Gene quads, lanes, rounds and the summation order are
// those of k_offspring_apply, so children and objectives are bit-identical to it.
// (A CTA-per-pair variant with whole-row bulk stages measured 1.86 ms vs 1.44 ms at pop 200k,
// barrier-bound: profiles/r02_ncu_D_offspring_apply_bulk.txt.)
#ifndef OFF_RING_S
#define OFF_RING_S 3
#endif
constexpr int RING_CH = 130;                        // doubles per row chunk (128 genes + alignment)
constexpr int RING_STAGE = 3 * RING_CH + 8;         // doubles per stage: x1, x2, beta chunks + 32 flags

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}


template <int M, bool LSMOP>
__global__ void __launch_bounds__(RW * 32, OFF_APPLY_MINB) k_offspring_apply_ring(temo_problem P, VarArgs V,
                                                                     const double *__restrict__ X,
                                                                     const int64_t *__restrict__ i1,
                                                                     const int64_t *__restrict__ i2, int64_t h,
                                                                     int64_t q0, int64_t q1,
                                                                     Philox ph, uint64_t off, int swap,
                                                                     const double *__restrict__ beta,
                                                                     const uint16_t *__restrict__ flags,
                                                                     double *__restrict__ O,
                                                                     double *__restrict__ FO,
                                                                     const int64_t *__restrict__ src_map,
                                                                     const int64_t *__restrict__ dst_rows) {
    constexpr int RS = OFF_RING_S;
    extern __shared__ __align__(16) double rsm[];
    const int64_t d = P.d;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *ring = rsm + (int64_t)warp * RS * RING_STAGE;                     // this warp's stages
    uint64_t *bar = reinterpret_cast<uint64_t *>(rsm + (int64_t)RW * RS * RING_STAGE) + warp * RS;
    double *s_lo = rsm + (int64_t)RW * RS * RING_STAGE + RW * RS, *s_hi = s_lo + d, *s_cf = s_hi + d;
    double *s_wb = s_cf + d;  // OFF_APPLY_CSTORE staging rows
    signed char *s_grp = reinterpret_cast<signed char *>(s_cf + d + (OFF_APPLY_CSTORE ? RW * 256 : 0));
    for (int64_t g = threadIdx.x; g < d; g += blockDim.x) {
        s_lo[g] = V.lower[g];
        s_hi[g] = V.upper[g];
        s_cf[g] = 1.0 + (double)(g + 1) / (double)d;
        int grp = -1;
        const int64_t rel = g - (M - 1);
        if (LSMOP) {
            for (int i = 0; i < M; ++i)
                if (rel >= P.offset[i] && rel < P.offset[i + 1]) grp = i;
        } else if (rel >= 0) {
            grp = 0;
        }
        s_grp[g] = (signed char)grp;
    }
    if (lane == 0) {
        for (int st = 0; st < RS; ++st) mbar_init(&bar[st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int64_t hd = h * d;
    const int64_t o_mu = (int64_t)off;
    const int64_t o_pmu = o_mu + (swap ? 3 * hd : hd);
    const int64_t avail = 4 - ph.pos;
    const double eta = V.eta_m + 1.0;
    const int64_t QP = quads_per_pair(d), QS = flag_stride(d);
    const int64_t qstride = (int64_t)gridDim.x * RW;
    const int64_t qa = q0 + (int64_t)blockIdx.x * RW + warp;
    auto shift_of = [&](int64_t q) { return (int)((o_mu + q * d - avail) & 3); };
    auto rounds_of = [&](int sh) { return (d + sh + 127) / 128; };
    auto mapped = [&](int64_t r) { return src_map ? src_map[r] : r; };
    auto drow = [&](int64_t r) { return dst_rows ? dst_rows[r] : r; };
    // producer cursor (uniform over the warp; lane 0 issues): pair pq, round pr of pR, rows pp1/pp2
    int64_t pq = qa, pr = 0, pR = 0, pp1 = 0, pp2 = 0, np1 = 0, np2 = 0, nr1 = 0, nr2 = 0;
    int psh = 0;
    if (pq < q1) {
        pp1 = mapped(i1[pq]);
        pp2 = mapped(i2[pq]);
        psh = shift_of(pq);
        pR = rounds_of(psh);
        if (pq + qstride < q1) {
            np1 = mapped(i1[pq + qstride]);
            np2 = mapped(i2[pq + qstride]);
        }
        if (pq + 2 * qstride < q1) {
            nr1 = i1[pq + 2 * qstride];
            nr2 = i2[pq + 2 * qstride];
        }
    }
    int64_t issued = 0;
    auto issue_next = [&]() {
        if (pq >= q1) return;
        const int st = (int)(issued % RS);
        if (lane == 0) {
            const int64_t b = -psh + 128 * pr;
            const int64_t lo = (b < 0 ? 0 : b) & ~(int64_t)1;
            const int64_t hi = ((b + 128 < d ? b + 128 : d) + 1) & ~(int64_t)1;
            const uint32_t nb = (uint32_t)((hi - lo) * sizeof(double));
            const int64_t f0 = 32 * pr, fn = (QS - f0 < 32 ? QS - f0 : 32);
            const uint32_t fb = (uint32_t)(fn * sizeof(uint16_t));
            double *dst = ring + (int64_t)st * RING_STAGE;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&bar[st], 3 * nb + fb);
            bulk_g2s(dst, X + pp1 * d + lo, nb, &bar[st]);
            bulk_g2s(dst + RING_CH, X + pp2 * d + lo, nb, &bar[st]);
            bulk_g2s(dst + 2 * RING_CH, beta + pq * d + lo, nb, &bar[st]);
            bulk_g2s(dst + 3 * RING_CH, flags + pq * QS + f0, fb, &bar[st]);
        }
        ++issued;
        if (++pr == pR) {  // next pair of this warp
            pq += qstride;
            pr = 0;
            if (pq < q1) {
                pp1 = np1;
                pp2 = np2;
                psh = shift_of(pq);
                pR = rounds_of(psh);
                if (pq + qstride < q1) {
                    np1 = mapped(nr1);
                    np2 = mapped(nr2);
                }
                if (pq + 2 * qstride < q1) {
                    nr1 = i1[pq + 2 * qstride];
                    nr2 = i2[pq + 2 * qstride];
                }
            }
        }
    };
    for (int k = 0; k < RS; ++k) issue_next();
    int64_t used = 0;
    int64_t nd1 = 0, nd2 = 0;
    if (qa < q1) {
        nd1 = drow(qa);
        nd2 = drow(h + qa);
    }
    for (int64_t q = qa; q < q1; q += qstride) {
        double *o1 = O + nd1 * d;
        double *o2 = O + nd2 * d;
        if (q + qstride < q1) {
            nd1 = drow(q + qstride);
            nd2 = drow(h + q + qstride);
        }
        const int sh = shift_of(q);
        double part1[M], part2[M];
#pragma unroll
        for (int i = 0; i < M; ++i) part1[i] = part2[i] = 0.0;
        double x0a = 0.0, x0b = 0.0;
        for (int64_t base = -sh, j0 = 0; base < d; base += 128, j0 += 32) {
            const int st = (int)(used % RS);
            mbar_wait(&bar[st], (uint32_t)((used / RS) & 1));
            const double *cx1 = ring + (int64_t)st * RING_STAGE;
            const double *cx2 = cx1 + RING_CH, *cbq = cx2 + RING_CH;
            const uint16_t *cfl = reinterpret_cast<const uint16_t *>(cbq + RING_CH);
            const int64_t lo = (base < 0 ? 0 : base) & ~(int64_t)1;
            const int64_t gs = base + 4 * lane;
            const int64_t es = q * d + gs;
            const uint32_t fl = (j0 + lane < QP) ? cfl[lane] : 0u;
            const uint32_t crossed = fl & 0xF, hit = (fl >> 4) & 0xFF;
            double c1[4], c2[4];
            bool ok[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int64_t g = gs + k;
                ok[k] = g >= 0 && g < d;
                const double a = ok[k] ? cx1[g - lo] : 0.0;
                const double b = ok[k] ? cx2[g - lo] : 0.0;
                const double bb = ok[k] ? cbq[g - lo] : 0.0;
                double y1 = a, y2 = b;
                if ((crossed >> k) & 1) {
                    const double shift = 0.5 * (1.0 - bb);
                    y1 = a + shift * (b - a);
                    y2 = b + shift * (a - b);
                }
                if (ok[k]) {
                    y1 = clipv(y1, s_lo[g], s_hi[g]);
                    y2 = clipv(y2, s_lo[g], s_hi[g]);
                }
                c1[k] = y1;
                c2[k] = y2;
            }
            __syncwarp();  // stage consumed by every lane: refill it with the round RS ahead
            ++used;
            issue_next();
            if (hit) {  // polynomial mutation (variation.py:104-120), only where hit
                uint64_t m1[4], m2[4];
                if (hit & 0xF) raw_quad(ph, o_pmu + es, avail, m1);
                if (hit & 0xF0) raw_quad(ph, o_pmu + hd + es, avail, m2);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int64_t g = gs + k;
                    if ((hit >> k) & 1)
                        c1[k] = clipv(pm_step(c1[k], s_lo[g], s_hi[g], u01(m1[k]), eta), s_lo[g], s_hi[g]);
                    if ((hit >> (4 + k)) & 1)
                        c2[k] = clipv(pm_step(c2[k], s_lo[g], s_hi[g], u01(m2[k]), eta), s_lo[g], s_hi[g]);
                }
            }
#if OFF_APPLY_CSTORE
            {
                double *w1 = s_wb + (int64_t)warp * 256, *w2 = w1 + 128;
                __syncwarp();
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    w1[4 * lane + k] = c1[k];
                    w2[4 * lane + k] = c2[k];
                }
                __syncwarp();
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int64_t g = base + lane + 32 * i;
                    if (g >= 0 && g < d) {
                        o1[g] = w1[lane + 32 * i];
                        o2[g] = w2[lane + 32 * i];
                    }
                }
            }
#else
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (ok[k]) {
                    o1[gs + k] = c1[k];
                    o2[gs + k] = c2[k];
                }
#endif
            if (!FO) continue;
            if (base == -sh) {
                x0a = __shfl_sync(~0u, pick4(c1, sh), 0);
                x0b = __shfl_sync(~0u, pick4(c2, sh), 0);
            }
            if constexpr (LSMOP) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int grp = ok[k] ? (int)s_grp[gs + k] : -1;
                    if (grp < 0) continue;
                    const double cf = s_cf[gs + k];
                    const double xa = cf * c1[k] - 10.0 * x0a;
                    const double sa = xa * xa;
                    const double xb = cf * c2[k] - 10.0 * x0b;
                    const double sb = xb * xb;
#pragma unroll
                    for (int i = 0; i < M; ++i)
                        if (grp == i) {
                            part1[i] += sa;
                            part2[i] += sb;
                        }
                }
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (ok[k]) {
                        acc_gene<M>(P, gs + k, c1[k], x0a, part1);
                        acc_gene<M>(P, gs + k, c2[k], x0b, part2);
                    }
            }
        }
        if (!FO) continue;
#pragma unroll
        for (int i = 0; i < M; ++i)
#pragma unroll
            for (int s = 16; s; s >>= 1) {
                part1[i] += __shfl_xor_sync(~0u, part1[i], s);
                part2[i] += __shfl_xor_sync(~0u, part2[i], s);
            }
        __syncwarp();
        if (lane == 0) {
            double f[M];
            finish_objs<M>(P, o1, part1, f);
#pragma unroll
            for (int i = 0; i < M; ++i) FO[q * M + i] = f[i];
        } else if (lane == 1) {
            double f[M];
            finish_objs<M>(P, o2, part2, f);
#pragma unroll
            for (int i = 0; i < M; ++i) FO[(h + q) * M + i] = f[i];
        }
    }
}

#ifndef TEMO_M_ONLY  // non-template kernels live in the base translation unit only
// ------------------------------------------------------------------ standalone operators
__global__ void k_sbx(VarArgs V, const double *__restrict__ X1, const double *__restrict__ X2,
                      int64_t q, int64_t d, Philox ph, USrc umu, USrc usw, USrc ucr,
                      double *__restrict__ C) {
    const int64_t base = 4 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
    const double e = 1.0 / (V.eta_c + 1.0);
    PhiloxCursor a, b, c;
    for (int64_t t = base; t < base + 4 && t < q * d; ++t) {
        const int64_t g = t % d;
        const double mu = umu.get(ph, a, t);
        const double sw = V.gene_swap ? usw.get(ph, b, t) : 1.0;
        const double cr = V.gene_swap ? ucr.get(ph, c, t) : 0.0;
        double c1, c2;
        sbx_gene(X1[t], X2[t], mu, sw, cr, e, V.gene_swap, c1, c2);
        C[t] = clipv(c1, V.lower[g], V.upper[g]);
        C[q * d + t] = clipv(c2, V.lower[g], V.upper[g]);
    }
}

__global__ void k_pm(VarArgs V, const double *__restrict__ X, int64_t rows, int64_t d, Philox ph,
                     USrc umu, USrc uhit, double *__restrict__ Y) {
    const int64_t base = 4 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
    const double eta = V.eta_m + 1.0;
    PhiloxCursor a, b;
    for (int64_t t = base; t < base + 4 && t < rows * d; ++t) {
        const int64_t g = t % d;
        const double lo = V.lower[g], hi = V.upper[g];
        const double mu = umu.get(ph, a, t);
        const double hu = uhit.get(ph, b, t);
        double y = X[t];
        if (V.p_m - hu >= 0.0) y = pm_step(y, lo, hi, mu, eta);
        Y[t] = clipv(y, lo, hi);
    }
}

__global__ void k_uniform(Philox ph, uint64_t off, int64_t count, double *__restrict__ out) {
    const int64_t base = 4 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
    PhiloxCursor c;
    for (int64_t t = base; t < base + 4 && t < count; ++t) out[t] = c.uniform(ph, off + t);
}

// harness.py:188-190: X = lower + U * (upper - lower)
__global__ void k_init_population(Philox ph, uint64_t off, int64_t rows, int64_t d,
                                  const double *__restrict__ lo, const double *__restrict__ hi,
                                  double *__restrict__ X) {
    const int64_t base = 4 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
    PhiloxCursor c;
    for (int64_t t = base; t < base + 4 && t < rows * d; ++t) {
        const int64_t g = t % d;
        X[t] = lo[g] + c.uniform(ph, off + t) * (hi[g] - lo[g]);
    }
}

#endif  // TEMO_M_ONLY

// TEMO_OFFSPRING_S=0 disables the persistent staged kernel (A/B comparisons)
static bool offspring_s_disabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("TEMO_OFFSPRING_S");
        v = (e && e[0] == '0') ? 1 : 0;
    }
    return v == 1;
}

// TEMO_APPLY_VEC=0 disables the vector gene-major apply kernel (d even, >= 128) (A/B)
static bool apply_vec();
// The PM hit list (k_pm_list) needs only the randomness phase's flags: it is built at the end of
// temo_offspring_rand_ws (on the randomness stream, overlapped with the previous generation
// when the harness runs the randomness ahead) instead of inside the apply stage.
static bool pm_list_early(int64_t d) {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("TEMO_PMLIST_EARLY");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v && d >= 128 && d % 2 == 0 && apply_vec();
}

static bool apply_vec() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("TEMO_APPLY_VEC");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

// TEMO_APPLY_GENE=1 selects the scalar gene-major apply kernel for d >= 128 (A/B; slower)
static bool apply_gene_major() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("TEMO_APPLY_GENE");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

// TEMO_APPLY_RING=1 selects the bulk-ring apply kernel instead of the plain warp-per-pair one (A/B)
static bool apply_ring_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("TEMO_APPLY_RING");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

// TEMO_OFFSPRING_CTA=1 selects the CTA-per-pair kernel (A/B comparisons)
static bool offspring_cta_forced() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("TEMO_OFFSPRING_CTA");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

static VarArgs var_args(const temo_variation *v) {
    VarArgs a;
    a.eta_c = v->eta_c;
    a.eta_m = v->eta_m;
    a.p_m = v->p_m;
    a.gene_swap = v->gene_swap;
    a.lower = v->lower;
    a.upper = v->upper;
    return a;
}

static bool prob_ok(const temo_problem *p) {
    if (!p || p->m < 2 || p->m > 16 || p->d < p->m) return false;
    if (p->id >= TEMO_PROB_LSMOP1 && p->id <= TEMO_PROB_LSMOP9) return p->nk >= 1;
    return p->id >= 1 && p->id <= 7;
}

static Philox philox_or_zero(const temo_philox_state *st) {
    if (st) return philox_from(*st);
    temo_philox_state z = {};
    z.buffer_pos = 4;
    return philox_from(z);
}

#define TEMO_M_SWITCH(m, CASE)                                                                     \
    switch (m) {                                                                                   \
        CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) \
        CASE(13) CASE(14) CASE(15) CASE(16)                                                        \
        default: return TEMO_EINVAL;                                                               \
    }


// ------------------------------------------------------------ per-M launchers
// build.py compiles this file once as the base unit and once per objective
// count with -DTEMO_M_ONLY=M; each per-M unit instantiates only its M (the
// base unit declares them extern), so the M-templated kernels build in parallel.
template <int M>
int eval_m(const temo_problem *prob, const double *X, const int64_t *map, int64_t lo1, int64_t c1, int64_t lo2,
           int64_t c2, double *F, cudaStream_t s) {
    const int64_t n = c1 + c2;
    if (n <= 0) return TEMO_OK;
    if (prob->id > TEMO_PROB_LSMOP1 || (prob->id == TEMO_PROB_LSMOP1 && env_int("TEMO_LSMOP1_WARP_EVAL", 0))) {
        // LSMOP: warp per row
        const int64_t want = (n + 7) / 8;
        const unsigned grid = (unsigned)(want < num_sms() * 8 * 4 ? want : num_sms() * 8 * 4);
        k_eval_lsmop<M><<<grid, 256, 0, s>>>(*prob, X, map, lo1, c1, lo2, c2, F);
    } else {
        k_evaluate<M><<<(unsigned)n, VT, 0, s>>>(*prob, X, map, lo1, c1, lo2, c2, F);
    }
    return TEMO_OK;
}

template <int M>
int offspring_m(const temo_problem *prob, const temo_variation *var, const double *X,
                const int64_t *i1, const int64_t *i2, int64_t h, const temo_philox_state *st,
                uint64_t off, double *O, double *FO, int single, bool warp_path, size_t smem,
                int smem_rows, cudaStream_t s, const temo_philox_state *st_dev) {
    const int64_t d = prob->d;
    if (warp_path && d <= SMAX_D && !offspring_s_disabled()) {
        const size_t sm_s = (3 * d + SW * 128) * sizeof(double) + d + 16;
        if (sm_s > 48 * 1024) {
            TEMO_CUDA(cudaFuncSetAttribute(k_offspring_s<M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_s));
            TEMO_CUDA(cudaFuncSetAttribute(k_offspring_s<M, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_s));
            TEMO_CUDA(cudaFuncSetAttribute(k_offspring_s<M, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_s));
            TEMO_CUDA(cudaFuncSetAttribute(k_offspring_s<M, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_s));
        }
        const int64_t want = (h + SW - 1) / SW;
        const unsigned grid = (unsigned)(want < num_sms() * 2 * 4 ? want : num_sms() * 2 * 4);
        const Philox ph = st_dev ? Philox{} : philox_from(*st);
        if (st_dev && var->gene_swap)
            k_offspring_s<M, true, true><<<grid, SW * 32, sm_s, s>>>(*prob, var_args(var), X, i1, i2, h, ph, st_dev,
                                                                     off, O, FO, single);
        else if (st_dev)
            k_offspring_s<M, false, true><<<grid, SW * 32, sm_s, s>>>(*prob, var_args(var), X, i1, i2, h, ph, st_dev,
                                                                      off, O, FO, single);
        else if (var->gene_swap)
            k_offspring_s<M, true><<<grid, SW * 32, sm_s, s>>>(*prob, var_args(var), X, i1, i2, h, ph, nullptr,
                                                               off, O, FO, single);
        else
            k_offspring_s<M, false><<<grid, SW * 32, sm_s, s>>>(*prob, var_args(var), X, i1, i2, h, ph, nullptr,
                                                                off, O, FO, single);
        return TEMO_OK;
    }
    if (st_dev) return TEMO_EINVAL;  // device-resident state: the staged kernel only
    if (warp_path && var->gene_swap) {
        k_offspring_w<M, true><<<(unsigned)((h + OW - 1) / OW), OW * 32, 0, s>>>(
            *prob, var_args(var), X, i1, i2, h, philox_from(*st), off, O, FO, single);
    } else if (warp_path) {
        k_offspring_w<M, false><<<(unsigned)((h + OW - 1) / OW), OW * 32, 0, s>>>(
            *prob, var_args(var), X, i1, i2, h, philox_from(*st), off, O, FO, single);
    } else {
        if (smem > 48 * 1024)
            TEMO_CUDA(cudaFuncSetAttribute(k_offspring<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
        k_offspring<M><<<(unsigned)h, VT, smem, s>>>(*prob, var_args(var), X, i1, i2, h,
                                                     philox_from(*st), off, O, FO, smem_rows, single);
    }
    return TEMO_OK;
}

template <int M>
int apply_m(const temo_problem *prob, const VarArgs &V, const double *X, const int64_t *i1,
            const int64_t *i2, int64_t h, int64_t q0, int64_t q1, const Philox &ph, uint64_t off, int gene_swap,
            const double *beta, const uint16_t *flags, double *O, double *FO,
            const int64_t *src_map, const int64_t *dst_rows, size_t sm_a, unsigned grid,
            cudaStream_t s, int64_t *pm_list, int64_t pm_cap) {
    const int64_t d = prob->d;
    if (d >= 128 && d % 2 == 0 && apply_vec()) {
        const size_t sm_v = 3 * d * sizeof(double) + d + 16;
        if (sm_v > 48 * 1024) {
            TEMO_CUDA(cudaFuncSetAttribute(k_offspring_apply_v<M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_v));
            TEMO_CUDA(cudaFuncSetAttribute(k_offspring_apply_v<M, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_v));
        }
        const int64_t want = (q1 - q0 + RW - 1) / RW;
        const int64_t capv = (int64_t)num_sms() * (env_int("TEMO_APPLY_GRID_PER_SM", OFF_APPLYV_MINB * 8));
        const unsigned gv = (unsigned)(want < capv ? want : capv);
        const int64_t wantf = (q1 - q0 + RW - 1) / RW;
        const unsigned gf = (unsigned)wantf;
        // PM hits: compacted list (order irrelevant: each entry's result is fixed), one thread per
        // hit, then per pair the objectives from the apply sums + the hit genes' terms in gene order
        const bool early = pm_list_early(d);
        if (!early) TEMO_CUDA(cudaMemsetAsync(pm_list, 0, sizeof(int64_t), s));
        const int64_t items = (q1 - q0) * quads_per_pair(d);
        const unsigned gl = (unsigned)((items + 255) / 256 < num_sms() * 32 ? (items + 255) / 256 : num_sms() * 32);
        const unsigned gp = (unsigned)((pm_cap + 255) / 256 < num_sms() * 16 ? (pm_cap + 255) / 256 : num_sms() * 16);
        stage_begin(S_APPLY_VEC, s);
        if (prob->id == TEMO_PROB_LSMOP1)
            k_offspring_apply_v<M, true><<<gv, RW * 32, sm_v, s>>>(*prob, V, X, i1, i2, h, q0, q1, ph, off,
                                                                gene_swap, beta, flags, O, FO, src_map, dst_rows);
        else
            k_offspring_apply_v<M, false><<<gv, RW * 32, sm_v, s>>>(*prob, V, X, i1, i2, h, q0, q1, ph, off,
                                                                 gene_swap, beta, flags, O, FO, src_map, dst_rows);
        stage_end(S_APPLY_VEC, s);
        if (!early) k_pm_list<<<gl, 256, 0, s>>>(d, h, q0, q1, off, ph.pos, flags, pm_list, pm_cap);
        k_pm_apply<<<gp, 256, 0, s>>>(V, d, h, ph, off, gene_swap, pm_list, pm_cap, O, dst_rows);
        if (prob->id == TEMO_PROB_LSMOP1)
            k_offspring_pm_fix<M, true><<<gf, RW * 32, 0, s>>>(*prob, V, h, q0, q1, ph, off, gene_swap, flags, O, FO,
                                                               dst_rows, pm_list, pm_cap);
        else
            k_offspring_pm_fix<M, false><<<gf, RW * 32, 0, s>>>(*prob, V, h, q0, q1, ph, off, gene_swap, flags, O,
                                                                FO, dst_rows, pm_list, pm_cap);
        return TEMO_OK;
    }
    if (d >= 128 && apply_gene_major()) {
        const size_t sm_t = 3 * d * sizeof(double) + d + 16;
        if (sm_t > 48 * 1024) {
            TEMO_CUDA(cudaFuncSetAttribute(k_offspring_apply_t<M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_t));
            TEMO_CUDA(cudaFuncSetAttribute(k_offspring_apply_t<M, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_t));
        }
        if (prob->id == TEMO_PROB_LSMOP1)
            k_offspring_apply_t<M, true><<<grid, RW * 32, sm_t, s>>>(*prob, V, X, i1, i2, h, q0, q1, ph, off,
                                                                  gene_swap, beta, flags, O, FO, src_map, dst_rows);
        else
            k_offspring_apply_t<M, false><<<grid, RW * 32, sm_t, s>>>(*prob, V, X, i1, i2, h, q0, q1, ph, off,
                                                                   gene_swap, beta, flags, O, FO, src_map, dst_rows);
        return TEMO_OK;
    }
    if (d % 2 == 0 && d >= 128 && apply_ring_enabled()) {  // per-warp bulk ring (rows 16-byte aligned)
        const size_t sm_r = (size_t)RW * OFF_RING_S * (RING_STAGE * sizeof(double) + sizeof(uint64_t)) + sm_a;
        if (sm_r <= 227 * 1024) {
            TEMO_CUDA(cudaFuncSetAttribute(k_offspring_apply_ring<M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_r));
            TEMO_CUDA(cudaFuncSetAttribute(k_offspring_apply_ring<M, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_r));
            if (prob->id == TEMO_PROB_LSMOP1)
                k_offspring_apply_ring<M, true><<<grid, RW * 32, sm_r, s>>>(*prob, V, X, i1, i2, h, q0, q1, ph, off,
                                                                         gene_swap, beta, flags, O, FO, src_map,
                                                                         dst_rows);
            else
                k_offspring_apply_ring<M, false><<<grid, RW * 32, sm_r, s>>>(*prob, V, X, i1, i2, h, q0, q1, ph,
                                                                          off, gene_swap, beta, flags, O, FO,
                                                                          src_map, dst_rows);
            return TEMO_OK;
        }
    }
    if (sm_a > 48 * 1024) {
        TEMO_CUDA(cudaFuncSetAttribute(k_offspring_apply<M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_a));
        TEMO_CUDA(cudaFuncSetAttribute(k_offspring_apply<M, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_a));
    }
    if (prob->id == TEMO_PROB_LSMOP1)
        k_offspring_apply<M, true><<<grid, RW * 32, sm_a, s>>>(*prob, V, X, i1, i2, h, q0, q1, ph, off, gene_swap,
                                                              beta, flags, O, FO, 0, src_map, dst_rows);
    else
        k_offspring_apply<M, false><<<grid, RW * 32, sm_a, s>>>(*prob, V, X, i1, i2, h, q0, q1, ph, off, gene_swap,
                                                               beta, flags, O, FO, 0, src_map, dst_rows);
    return TEMO_OK;
}

#define TEMO_M_LIST(X) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16)
#define TEMO_VAR_DECL(MM, EXT)                                                                      \
    EXT template int eval_m<MM>(const temo_problem *, const double *, const int64_t *, int64_t, int64_t,     \
                                int64_t, int64_t, double *, cudaStream_t);                                  \
    EXT template int offspring_m<MM>(const temo_problem *, const temo_variation *, const double *,   \
                                     const int64_t *, const int64_t *, int64_t,                      \
                                     const temo_philox_state *, uint64_t, double *, double *, int,    \
                                     bool, size_t, int, cudaStream_t, const temo_philox_state *);     \
    EXT template int apply_m<MM>(const temo_problem *, const VarArgs &, const double *,              \
                                 const int64_t *, const int64_t *, int64_t, int64_t, int64_t,         \
                                 const Philox &, uint64_t,                                             \
                                 int, const double *, const uint16_t *, double *, double *,           \
                                 const int64_t *, const int64_t *, size_t, unsigned, cudaStream_t, int64_t *,  \
                                 int64_t);
#ifdef TEMO_M_ONLY
TEMO_VAR_DECL(TEMO_M_ONLY, )
#else
#define TEMO_VAR_EXTERN(MM) TEMO_VAR_DECL(MM, extern)
TEMO_M_LIST(TEMO_VAR_EXTERN)
#endif

}  // namespace temo

using namespace temo;

#ifndef TEMO_M_ONLY

// objectives of logical rows [lo1, lo1 + c1) u [lo2, lo2 + c2) (row l read at map[l], written to F + l m)
static int eval_rows(const temo_problem *prob, const double *X, const int64_t *map, int64_t lo1, int64_t c1,
                     int64_t lo2, int64_t c2, double *F, cudaStream_t s) {
#define EVAL_CASE(MM) case MM: { int rc = eval_m<MM>(prob, X, map, lo1, c1, lo2, c2, F, s); if (rc) return rc; } break;
    TEMO_M_SWITCH(prob->m, EVAL_CASE)
#undef EVAL_CASE
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

extern "C" int temo_evaluate(const temo_problem *prob, const double *X, int64_t n, double *F,
                             temo_stream_t stream) {
    if (!prob_ok(prob) || n < 0 || !X || !F) return TEMO_EINVAL;
    if (n == 0) return TEMO_OK;
    cudaStream_t s = (cudaStream_t)stream;
    stage_begin(S_EVALUATE, s);
    const int rc = eval_rows(prob, X, nullptr, 0, n, 0, 0, F, s);
    if (rc) return rc;
    stage_end(S_EVALUATE, s);
    return TEMO_OK;
}

extern "C" int temo_evaluate_rows(const temo_problem *prob, const double *X, const int64_t *rows, int64_t n,
                                  double *F, temo_stream_t stream) {
    if (!prob_ok(prob) || n < 0 || !X || !F) return TEMO_EINVAL;
    if (n == 0) return TEMO_OK;
    cudaStream_t s = (cudaStream_t)stream;
    stage_begin(S_EVALUATE, s);
    const int rc = eval_rows(prob, X, rows, 0, n, 0, 0, F, s);
    if (rc) return rc;
    stage_end(S_EVALUATE, s);
    return TEMO_OK;
}

__global__ void k_sbx_beta(const double *__restrict__ mu, int64_t n, double e, int fast,
                           double *__restrict__ beta) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < n) beta[t] = fast ? temo::sbx_beta_fast(mu[t], e) : temo::sbx_beta(mu[t], e);
}

extern "C" int temo_sbx_beta(const double *mu, int64_t n, double eta_c, int fast, double *beta,
                             temo_stream_t stream) {
    if (n < 0 || !mu || !beta || !(eta_c > -1.0)) return TEMO_EINVAL;
    if (n == 0) return TEMO_OK;
    k_sbx_beta<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(mu, n, 1.0 / (eta_c + 1.0),
                                                                             fast, beta);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

extern "C" int temo_uniform(const temo_philox_state *st, uint64_t off, int64_t count, double *out,
                            temo_stream_t stream) {
    if (!st || count < 0 || !out) return TEMO_EINVAL;
    if (count == 0) return TEMO_OK;
    const int64_t th = (count + 3) / 4;
    k_uniform<<<(unsigned)((th + 255) / 256), 256, 0, (cudaStream_t)stream>>>(philox_from(*st), off,
                                                                             count, out);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

extern "C" int temo_sbx(const temo_variation *var, const double *X1, const double *X2, int64_t q,
                        int64_t d, const temo_philox_state *st, uint64_t off, const double *u_mu,
                        const double *u_swap, const double *u_cross, double *C,
                        temo_stream_t stream) {
    if (!var || q < 0 || d < 1 || !X1 || !X2 || !C) return TEMO_EINVAL;
    if (!st && (!u_mu || (var->gene_swap && (!u_swap || !u_cross)))) return TEMO_EINVAL;
    if (q == 0) return TEMO_OK;
    const uint64_t qd = (uint64_t)q * d;
    USrc a{u_mu, off}, b{u_swap, off + qd}, c{u_cross, off + 2 * qd};
    const int64_t th = (q * d + 3) / 4;
    k_sbx<<<(unsigned)((th + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        var_args(var), X1, X2, q, d, philox_or_zero(st), a, b, c, C);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

extern "C" int temo_pm(const temo_variation *var, const double *X, int64_t rows, int64_t d,
                       const temo_philox_state *st, uint64_t off, const double *u_mu,
                       const double *u_hit, double *Y, temo_stream_t stream) {
    if (!var || rows < 0 || d < 1 || !X || !Y) return TEMO_EINVAL;
    if (!st && (!u_mu || !u_hit)) return TEMO_EINVAL;
    if (rows == 0) return TEMO_OK;
    const uint64_t rd = (uint64_t)rows * d;
    USrc a{u_mu, off}, b{u_hit, off + rd};
    const int64_t th = (rows * d + 3) / 4;
    k_pm<<<(unsigned)((th + 255) / 256), 256, 0, (cudaStream_t)stream>>>(var_args(var), X, rows, d,
                                                                         philox_or_zero(st), a, b, Y);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

// LSMOP2..9 are evaluated by a separate warp-per-row pass over the children (no fused sums);
// TEMO_SPLIT_EVAL=1 does the same for LSMOP1 (A/B of the apply kernel without its sums)
static bool fused_eval(const temo_problem *prob) {
    return prob->id < TEMO_PROB_LSMOP1 || (prob->id == TEMO_PROB_LSMOP1 && !env_int("TEMO_SPLIT_EVAL", 0));
}

static int launch_offspring(const temo_problem *prob, const temo_variation *var, const double *X,
                            const int64_t *i1, const int64_t *i2, int64_t h,
                            const temo_philox_state *st, uint64_t off, double *O, double *FO,
                            int single, cudaStream_t s, const temo_philox_state *st_dev = nullptr) {
    if (!prob_ok(prob) || !var || !X || !i1 || !i2 || h < 0 || !(st || st_dev) || !O) return TEMO_EINVAL;
    if (h == 0) return TEMO_OK;
    const int64_t d = prob->d;
    const int smem_rows = 2 * d * (int64_t)sizeof(double) <= 96 * 1024;
    const size_t smem = smem_rows ? 2 * d * sizeof(double) : 0;
    // warp-per-pair kernel whenever every stream is congruent mod 4 (one Philox block per quad)
    const bool warp_path = (h * d) % 4 == 0 && !offspring_cta_forced();
    double *FOk = fused_eval(prob) ? FO : nullptr;
    stage_begin(S_OFFSPRING, s);
#define OFF_CASE(MM)                                                                               \
    case MM: {                                                                                     \
        int rc = offspring_m<MM>(prob, var, X, i1, i2, h, st, off, O, FOk, single, warp_path, smem, \
                                 smem_rows, s, st_dev);                                            \
        if (rc) return rc;                                                                         \
    } break;
    TEMO_M_SWITCH(prob->m, OFF_CASE)
#undef OFF_CASE
    TEMO_LAUNCH_CHECK();
    if (FO && !FOk) {
        const int rc = eval_rows(prob, O, nullptr, 0, single ? h : 2 * h, 0, 0, FO, s);
        if (rc) return rc;
    }
    stage_end(S_OFFSPRING, s);
    return TEMO_OK;
}

// PM hit list of the vector apply path: a counter and up to pm_list_cap entries (expected
// hits per generation 2 h d p_m = 2 h at the default p_m = 1/d; beyond the cap the per-pair
// fallback applies the PM)
static int64_t pm_list_cap(int64_t h, int64_t d) {
    const int64_t c = 16 * h + 65536;
    return c < 2 * h * d ? c : 2 * h * d;
}

extern "C" size_t temo_offspring_ws_bytes(int64_t h, int64_t d) {
    if (h < 0 || d < 1) return 0;
    return (size_t)round_up((int64_t)(h * d * sizeof(double)), 256) +
           (size_t)round_up((int64_t)(h * flag_stride(d) * sizeof(uint16_t)), 256) +
           (size_t)((1 + pm_list_cap(h, d)) * sizeof(int64_t)) + 256;
}

// two-phase path: congruent streams (one Philox block per quad) and staged constants
extern "C" int temo_offspring_two_phase(int64_t h, int64_t d) {
    return h >= 0 && d >= 1 && (h * d) % 4 == 0 && d <= SMAX_D;
}

static void offspring_ws_split(void *ws, int64_t h, int64_t d, double **beta, uint16_t **flags,
                               int64_t **pm_list = nullptr) {
    char *b = static_cast<char *>(ws);
    *beta = reinterpret_cast<double *>(b);
    b += round_up((int64_t)(h * d * sizeof(double)), 256);
    *flags = reinterpret_cast<uint16_t *>(b);
    b += round_up((int64_t)(h * flag_stride(d) * sizeof(uint16_t)), 256);
    if (pm_list) *pm_list = reinterpret_cast<int64_t *>(b);
}

// phase 1 of temo_offspring_ws_range: randomness of pairs [q0, q1) into the workspace
extern "C" int temo_offspring_rand_ws(const temo_variation *var, int64_t d, int64_t h, int64_t q0, int64_t q1,
                                      const temo_philox_state *st, uint64_t off, void *ws, size_t ws_bytes,
                                      temo_stream_t stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!var || !st || h < 0 || d < 1 || q0 < 0 || q1 > h || q0 > q1) return TEMO_EINVAL;
    if (!temo_offspring_two_phase(h, d)) return TEMO_EINVAL;
    if (q1 == q0) return TEMO_OK;
    if (!ws || ws_bytes < temo_offspring_ws_bytes(h, d)) return TEMO_EWORKSPACE;
    double *beta;
    uint16_t *flags;
    offspring_ws_split(ws, h, d, &beta, &flags);
    const Philox ph = philox_from(*st);
    const VarArgs V = var_args(var);
    const int64_t want = ((q1 - q0) * ((d + 3 + 127) / 128) + RW - 1) / RW;
    stage_begin(S_OFFSPRING, s);
    const int64_t capr = (int64_t)num_sms() * env_int("TEMO_RAND_GRID_PER_SM", 1024);
    const unsigned grid = (unsigned)(want < capr ? want : capr);
    // TEMO_RAND_SMEM: dynamic shared memory per CTA (unused) to cap the resident randomness
    // CTAs per SM, leaving room for overlapped selection kernels (A/B knob)
    static const int pad = env_int("TEMO_RAND_SMEM", 0);
    static bool attr = false;
    if (pad > 48 * 1024 && !attr) {
        cudaFuncSetAttribute(k_offspring_rand<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, pad);
        cudaFuncSetAttribute(k_offspring_rand<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, pad);
        attr = true;
    }
    if (var->gene_swap)
        k_offspring_rand<true><<<grid, RW * 32, pad, s>>>(d, V, h, q0, q1, ph, off, 0, beta, flags);
    else
        k_offspring_rand<false><<<grid, RW * 32, pad, s>>>(d, V, h, q0, q1, ph, off, 0, beta, flags);
    if (pm_list_early(d)) {
        int64_t *pm_list = nullptr;
        double *b2;
        uint16_t *f2;
        offspring_ws_split(ws, h, d, &b2, &f2, &pm_list);
        const int64_t items = (q1 - q0) * quads_per_pair(d);
        const unsigned gl = (unsigned)((items + 255) / 256 < num_sms() * 32 ? (items + 255) / 256 : num_sms() * 32);
        TEMO_CUDA(cudaMemsetAsync(pm_list, 0, sizeof(int64_t), s));
        k_pm_list<<<gl, 256, 0, s>>>(d, h, q0, q1, off, ph.pos, flags, pm_list, pm_list_cap(h, d));
    }
    TEMO_LAUNCH_CHECK();
    stage_end(S_OFFSPRING, s);
    return TEMO_OK;
}

// phase 2: children (and objectives) of pairs [q0, q1) from the parents and the workspace
extern "C" int temo_offspring_apply_ws(const temo_problem *prob, const temo_variation *var, const double *X,
                                       const int64_t *i1, const int64_t *i2, int64_t h, int64_t q0, int64_t q1,
                                       const temo_philox_state *st, uint64_t off, double *O, double *FO,
                                       const int64_t *src_map, const int64_t *dst_rows,
                                       void *ws, size_t ws_bytes, temo_stream_t stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!prob_ok(prob) || !var || !X || !i1 || !i2 || h < 0 || !st || !O) return TEMO_EINVAL;
    if (q0 < 0 || q1 > h || q0 > q1) return TEMO_EINVAL;
    const int64_t d = prob->d;
    if (!temo_offspring_two_phase(h, d)) return TEMO_EINVAL;
    if (q1 == q0) return TEMO_OK;
    if (!ws || ws_bytes < temo_offspring_ws_bytes(h, d)) return TEMO_EWORKSPACE;
    double *beta;
    uint16_t *flags;
    int64_t *pm_list;
    offspring_ws_split(ws, h, d, &beta, &flags, &pm_list);
    const Philox ph = philox_from(*st);
    const VarArgs V = var_args(var);
    const int64_t want = (q1 - q0 + RW - 1) / RW;
    const int64_t pm_cap = pm_list_cap(h, d);
    stage_begin(S_OFFSPRING_APPLY, s);
    const size_t sm_a = 3 * d * sizeof(double) + (OFF_APPLY_CSTORE ? RW * 256 * sizeof(double) : 0) + d + 16;
    const unsigned grid = (unsigned)(want < num_sms() * 3 * 8 ? want : num_sms() * 3 * 8);
    double *FOk = fused_eval(prob) ? FO : nullptr;
#define APPLY_CASE(MM)                                                                              \
    case MM: {                                                                                      \
        int rc = apply_m<MM>(prob, V, X, i1, i2, h, q0, q1, ph, off, var->gene_swap, beta, flags, O, FOk, \
                             src_map, dst_rows, sm_a, grid, s, pm_list, pm_cap);                    \
        if (rc) return rc;                                                                          \
    } break;
    TEMO_M_SWITCH(prob->m, APPLY_CASE)
#undef APPLY_CASE
    TEMO_LAUNCH_CHECK();
    if (FO && !FOk) {  // children of pairs [q0, q1): logical rows q and h + q
        const int rc = eval_rows(prob, O, dst_rows, q0, q1 - q0, h + q0, q1 - q0, FO, s);
        if (rc) return rc;
    }
    stage_end(S_OFFSPRING_APPLY, s);
    return TEMO_OK;
}

extern "C" int temo_offspring_ws_range(const temo_problem *prob, const temo_variation *var, const double *X,
                                       const int64_t *i1, const int64_t *i2, int64_t h, int64_t q0, int64_t q1,
                                       const temo_philox_state *st, uint64_t off, double *O, double *FO,
                                       const int64_t *src_map, const int64_t *dst_rows,
                                       void *ws, size_t ws_bytes, temo_stream_t stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!prob_ok(prob) || !var || !X || !i1 || !i2 || h < 0 || !st || !O) return TEMO_EINVAL;
    if (q0 < 0 || q1 > h || q0 > q1) return TEMO_EINVAL;
    if (q1 == q0) return TEMO_OK;
    const int64_t d = prob->d;
    if (!temo_offspring_two_phase(h, d)) {
        if (src_map || dst_rows || q0 != 0 || q1 != h) return TEMO_EINVAL;  // row maps / ranges: two-phase only
        return launch_offspring(prob, var, X, i1, i2, h, st, off, O, FO, 0, s);
    }
    const int rc = temo_offspring_rand_ws(var, d, h, q0, q1, st, off, ws, ws_bytes, stream);
    if (rc) return rc;
    return temo_offspring_apply_ws(prob, var, X, i1, i2, h, q0, q1, st, off, O, FO, src_map, dst_rows, ws,
                                   ws_bytes, stream);
}

extern "C" int temo_offspring_ws(const temo_problem *prob, const temo_variation *var, const double *X,
                                 const int64_t *i1, const int64_t *i2, int64_t h,
                                 const temo_philox_state *st, uint64_t off, double *O, double *FO,
                                 const int64_t *src_map, const int64_t *dst_rows,
                                 void *ws, size_t ws_bytes, temo_stream_t stream) {
    return temo_offspring_ws_range(prob, var, X, i1, i2, h, 0, h, st, off, O, FO, src_map, dst_rows, ws, ws_bytes,
                                   stream);
}

extern "C" int temo_offspring(const temo_problem *prob, const temo_variation *var, const double *X,
                              const int64_t *i1, const int64_t *i2, int64_t h,
                              const temo_philox_state *st, uint64_t off, double *O, double *FO,
                              temo_stream_t stream) {
    return launch_offspring(prob, var, X, i1, i2, h, st, off, O, FO, 0, (cudaStream_t)stream);
}

// temo_moead_offspring with the Philox state in device memory (CUDA-graph capturable)
extern "C" int temo_moead_offspring_dev(const temo_problem *prob, const temo_variation *var,
                                        const double *X, const int64_t *p1, const int64_t *p2, int64_t n,
                                        const temo_philox_state *st_dev, uint64_t off, double *O, double *FO,
                                        temo_stream_t stream) {
    if (!st_dev) return TEMO_EINVAL;
    return launch_offspring(prob, var, X, p1, p2, n, nullptr, off, O, FO, 1, (cudaStream_t)stream, st_dev);
}

extern "C" int temo_moead_offspring(const temo_problem *prob, const temo_variation *var,
                                    const double *X, const int64_t *p1, const int64_t *p2, int64_t n,
                                    const temo_philox_state *st, uint64_t off, double *O, double *FO,
                                    temo_stream_t stream) {
    return launch_offspring(prob, var, X, p1, p2, n, st, off, O, FO, 1, (cudaStream_t)stream);
}

extern "C" int temo_init_population(const temo_philox_state *st, uint64_t off, int64_t rows,
                                    int64_t d, const double *lower, const double *upper, double *X,
                                    temo_stream_t stream) {
    if (!st || rows < 0 || d < 1 || !lower || !upper || !X) return TEMO_EINVAL;
    if (rows == 0) return TEMO_OK;
    const int64_t th = (rows * d + 3) / 4;
    k_init_population<<<(unsigned)((th + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        philox_from(*st), off, rows, d, lower, upper, X);
    TEMO_LAUNCH_CHECK();
    return TEMO_OK;
}

#endif  // TEMO_M_ONLY
