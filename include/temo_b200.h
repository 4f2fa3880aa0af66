/*
 * temo_b200 -- C ABI of the B200-native tensorized EMO selection hot path.
 *
 * Drop-in boundary for the reference package `temo` 0.1.0
 * (/root/reference/pkg/src/temo).  The reference is pure Python/NumPy and has
 * no FFI of its own; every entry point below replaces one NumPy stage and is
 * bound from Python with ctypes (paper_2503_20286_b200/_lib.py; the stub a
 * maintainer adds on the reference side is in INTEGRATION.md).
 *
 * Conventions (all entry points):
 *   - device pointers, int64 sizes, row-major C-contiguous float64 matrices;
 *   - `stream` is a cudaStream_t; work is enqueued, never synchronised;
 *   - `ws`/`ws_bytes` is caller-provided device workspace (size from the
 *     matching *_ws_bytes query); the library allocates nothing;
 *   - return value: TEMO_OK or a host-side error (bad arguments, short
 *     workspace, launch failure);
 *   - `status` (device int32, may be NULL) receives TEMO_ST_* bits for
 *     data-dependent errors detected on the device (NaN input, peel failure,
 *     count repair failure) -- read it after the stream completes.  The Python
 *     layer maps them to the reference's ValueError / RuntimeError.
 */
#ifndef TEMO_B200_H
#define TEMO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *temo_stream_t; /* == cudaStream_t */

/* host-side return codes */
#define TEMO_OK 0
#define TEMO_EINVAL 1     /* ValueError in the reference */
#define TEMO_ENAN 2       /* ValueError (NaN objectives) */
#define TEMO_ERUNTIME 3   /* RuntimeError */
#define TEMO_EWORKSPACE 4 /* workspace too small */
#define TEMO_ECUDA 5      /* CUDA launch/runtime failure */

/* device-side status bits */
#define TEMO_ST_NAN 1     /* ndsort.py:35-36  NaN objective -> ValueError */
#define TEMO_ST_PEEL 2    /* ndsort.py:64-65  peeling did not terminate -> RuntimeError */
#define TEMO_ST_FILL 4    /* nsga3.py:176-177 not enough last-front rows -> RuntimeError */
#define TEMO_ST_DEMOTE 8  /* nsga3.py:180-181 demotion exceeds promotions -> RuntimeError */
#define TEMO_ST_COUNT 16  /* nsga3.py:216-217 selection size mismatch -> RuntimeError */
#define TEMO_ST_KRANGE 32 /* hype.py:43-44 / 68-69 k out of range -> ValueError */

int temo_abi_version(void);
const char *temo_strerror(int code);

/* ---------------------------------------------------------------- ND sort
 * Replaces ndsort.rank_assign (ndsort.py:47-71) and the dominance-matrix
 * construction it relies on (ndsort.py:25-44).
 *   F      : N x m float64 objectives (no NaN), 1 <= m <= 16, 1 <= N <= 2^20
 *   n      : 1 <= n <= N; l_out receives sort(r)[n-1]
 *   mode   : TEMO_RANK_SORT ranks every row (rank_assign semantics);
 *            TEMO_RANK_SELECT stops once >= n rows are ranked and gives every
 *            remaining row rank l+1 (exact for NSGA-III/HypE)
 *   rank   : N int32 outputs
 *   nfronts: (may be NULL) device int32, number of fronts peeled
 */
#define TEMO_RANK_SORT 0
#define TEMO_RANK_SELECT 1
size_t temo_rank_ws_bytes(int64_t N, int m);
int temo_rank(const double *F, int64_t N, int m, int64_t n, int mode, int32_t *rank,
              int32_t *l_out, int32_t *nfronts, int32_t *status, void *ws, size_t ws_bytes,
              temo_stream_t stream);

/* Path selection (diagnostics / A-B comparisons): m = 2 and 3 use the staircase
 * sort (lex-prefix merge-sort tree, ndsort_stair.cuh); temo_rank_force_bitmap(1)
 * (or env TEMO_RANK_BITMAP=1) sends them through the O(N^2) bitmap path like
 * m >= 4.  Both give identical ranks; set it before sizing the workspace. */
void temo_rank_force_bitmap(int on);
/* Diagnostics: per-front phase timestamps (%globaltimer, ns) of the staircase peel's
 * block 0, 8 per front: front start, phase A done, barrier 1 passed, high levels done,
 * high levels done, tile levels done, front written, barrier 2 passed; `on` = 1 + the
 * profiled block (0: off). */
void temo_stair_prof_enable(int on);
int temo_stair_prof_read(uint64_t *host, int64_t count);

/* Dominance bitmap only (ndsort.dominance_matrix, ndsort.py:25-44):
 * D_out is N x ceil(N/32) uint32 words, bit (j%32) of word [i][j/32] set iff
 * row i dominates row j.  For parity tests at small N. */
size_t temo_dominance_ws_bytes(int64_t N, int m);
int temo_dominance(const double *F, int64_t N, int m, uint32_t *D_out, int32_t *status,
                   void *ws, size_t ws_bytes, temo_stream_t stream);

/* --------------------------------------------------- column-sharded ND sort
 * Multi-GPU form of temo_rank.  Every rank passes the same F;
 * rank g owns sorted column tiles [jt_lo, jt_hi) from temo_rank_shard_bounds
 * (multiples of 4 tiles of 256 columns; lo_hi receives 2G values, empty shards
 * possible for tiny N).  Front step k, driven by the host:
 *   temo_rank_shard_detect -> seg (8 (jt_hi - jt_lo) words: own front bits,
 *                             sorted index space), count (device int32)
 *   all-gather of the segments into the full mask (ceil(N/1024)*32 words)
 *   temo_rank_shard_apply  -> ranks the whole front, subtracts its rows from
 *                             the own columns' counts; front_total (device)
 * and temo_rank_shard_finish writes ranks in the original row order (`fill`,
 * a device int32, for rows never ranked in SELECT mode).  All calls of one
 * shard share the workspace and (N, m, jt_lo, jt_hi). */
void temo_rank_shard_bounds(int64_t N, int G, int64_t *lo_hi);
size_t temo_rank_shard_ws_bytes(int64_t N, int m, int64_t jt_lo, int64_t jt_hi);
int temo_rank_shard_build(const double *F, int64_t N, int m, int64_t jt_lo, int64_t jt_hi,
                          int32_t *status, void *ws, size_t ws_bytes, temo_stream_t stream);
int temo_rank_shard_detect(int64_t N, int m, int64_t jt_lo, int64_t jt_hi, uint32_t *seg,
                           int32_t *count, void *ws, size_t ws_bytes, temo_stream_t stream);
int temo_rank_shard_apply(int64_t N, int m, int64_t jt_lo, int64_t jt_hi, const uint32_t *full,
                          int32_t k, int32_t *front_total, void *ws, size_t ws_bytes,
                          temo_stream_t stream);
int temo_rank_shard_finish(int64_t N, int m, int64_t jt_lo, int64_t jt_hi, const int32_t *fill,
                           int32_t *rank, void *ws, size_t ws_bytes, temo_stream_t stream);

/* ---------------------------------------------------------- NSGA-III select
 * Replaces nsga3.py:207-218 (normalize, associate, niche_counts, niche_select,
 * update_rank, keep) on already-shuffled objectives Fs (N x m) whose ranks
 * come from temo_rank(..., TEMO_RANK_SELECT) (`rank` is updated in place to
 * the final ranks; `l` is the device scalar from temo_rank).
 *   W (nr x m) directions; lattice_H > 0 asserts W == das_dennis(m, H) in its
 *   row order (directions.py:64-87) and enables the exact O(1)-per-row lattice
 *   association; 0 = arbitrary direction set (filtered full scan).
 *   keep (n int32) receives flatnonzero(rank < l).
 *   pi, dist (N) association (nsga3.py:96-116; excluded rows pi=0, dist=NaN);
 *   icpt (m), promoted (<= nr, direction order) always written;
 *   Fp (N x m), ideal (m), extreme (m int64), rho/rho_l (nr), counts (8 int32:
 *   n_promoted, n_s, n_dif, -, kept) optional (NULL to skip). */
size_t temo_nsga3_select_ws_bytes(int64_t N, int m, int64_t nr);
int temo_nsga3_select(const double *Fs, int64_t N, int m, const double *W, int64_t nr,
                      int32_t lattice_H, int64_t n, int32_t *rank, const int32_t *l, int32_t *keep, int32_t *pi, double *dist,
                      double *Fp, double *ideal, double *icpt, int64_t *extreme, int32_t *rho,
                      int32_t *rho_l, int32_t *promoted, int32_t *counts, int32_t *status, void *ws,
                      size_t ws_bytes, temo_stream_t stream);

/* Standalone stages (same kernels as temo_nsga3_select), one per reference function:
 *   temo_nsga3_normalize  nsga3.normalize   (nsga3.py:61-93)  rows with NaN are excluded
 *   temo_associate        nsga3.associate   (nsga3.py:96-116)
 *   temo_niche_counts     nsga3.niche_counts (nsga3.py:119-123)
 *   temo_niche_select     nsga3.niche_select (nsga3.py:126-167), counts[0] = #promoted
 *   temo_update_rank      nsga3.update_rank  (nsga3.py:170-183)
 * All share the workspace size temo_nsga3_select_ws_bytes(N, m, nr). */
int temo_nsga3_normalize(const double *F, int64_t N, int m, double *Fp, double *ideal, double *icpt,
                         int64_t *extreme, void *ws, size_t ws_bytes, temo_stream_t stream);
int temo_associate(const double *Fp, int64_t N, int m, const double *W, int64_t nr,
                   int32_t lattice_H, int32_t *pi, double *dist, void *ws, size_t ws_bytes, temo_stream_t stream);
int temo_niche_counts(const int32_t *rank, const int32_t *pi, int64_t N, int32_t l, int64_t nr,
                      int32_t *rho, int32_t *rho_l, void *ws, size_t ws_bytes, temo_stream_t stream);
int temo_niche_select(int32_t *rank, const int32_t *pi, const double *dist, int64_t N, int32_t l,
                      const int32_t *rho, int64_t nr, int32_t *promoted, int32_t *counts, void *ws,
                      size_t ws_bytes, temo_stream_t stream);
int temo_update_rank(int32_t *rank, int64_t N, const int32_t *promoted, int64_t n_promoted,
                     int64_t n_dif, int32_t l, int32_t *status, void *ws, size_t ws_bytes,
                     temo_stream_t stream);

/* Row gathers used to materialise survivors (X[perm][keep]):
 *   dst[r] = src[idx[r]]            (idx32 or idx64, the other NULL)
 *   dst[r] = src[idx_a[idx_b[r]]]   (composed permutation) */
int temo_gather_rows(const double *src, const int32_t *idx32, const int64_t *idx64, int64_t rows,
                     int64_t cols, double *dst, temo_stream_t stream);
int temo_gather_rows2(const double *src, const int64_t *idx_a, const int32_t *idx_b, int64_t rows,
                      int64_t cols, double *dst, temo_stream_t stream);

/* ----------------------------------------------------- RNG, problems, variation
 * NumPy Philox state (np.random.Philox().state: counter, key, buffer,
 * buffer_pos).  Uniform e of a draw that starts `off` raw outputs after this
 * state is bit-identical to the host's Generator.random (rng.py:28-31). */
typedef struct temo_philox_state {
    uint64_t counter[4];
    uint64_t key[2];
    uint64_t buffer[4];
    int32_t buffer_pos;
    int32_t reserved;
} temo_philox_state;

/* Full host state of NumPy's Philox bit generator (Philox.state: counter, key,
 * buffer, buffer_pos, has_uint32, uinteger). */
typedef struct temo_philox_host {
    uint64_t counter[4];
    uint64_t key[2];
    uint64_t buffer[4];
    int32_t buffer_pos;
    int32_t has_uint32;
    uint32_t uinteger;
    uint32_t reserved;
} temo_philox_host;

/* Host (CPU) replica of Generator.permutation(n) (variation.py:52, nsga3.py:204):
 * arange(n) Fisher-Yates-shuffled with NumPy's random_interval draws, bit for bit;
 * `st` is advanced exactly as NumPy advances the Generator.  Native host code,
 * no GPU involved (the reference's sequential shuffle is the host-side bound of
 * the generation loop). */
int temo_host_permutation(temo_philox_host *st, int64_t n, int64_t *out);

#define TEMO_PROB_DTLZ1 1 /* ... TEMO_PROB_DTLZ1 + 6 = DTLZ7 (problems.py:105-136) */
#define TEMO_PROB_LSMOP1 101 /* LSMOP1 ... TEMO_PROB_LSMOP1 + 8 = LSMOP9: Cheng et al. 2017 in the */
#define TEMO_PROB_LSMOP9 109 /* PlatEMO form (no reference; self-oracle oracle/problems.py) */

typedef struct temo_problem {
    int32_t id;          /* TEMO_PROB_* */
    int32_t m;           /* objectives, 2..16 */
    int64_t d;           /* decision variables */
    int32_t nk;          /* LSMOP: subcomponents per objective */
    int32_t sublen[16];  /* LSMOP: subcomponent length per objective */
    int32_t offset[17];  /* LSMOP: start of objective i's groups within x^s */
} temo_problem;

typedef struct temo_variation {
    double eta_c, eta_m, p_m; /* variation.py:17-45 (p_m resolved: None -> 1/d) */
    int32_t gene_swap;
    int32_t reserved;
    const double *lower, *upper; /* device, length d */
} temo_variation;

/* problems.evaluate (problems.py:105-136; LSMOP1-9 new): F (n x m) = f(X (n x d)) */
int temo_evaluate(const temo_problem *prob, const double *X, int64_t n, double *F,
                  temo_stream_t stream);
/* Same, for rows gathered through a map: F[r] = f(X[rows[r]]) (rows NULL = identity); the
 * row-pool layout of the generation loop (children at physical pool rows). */
int temo_evaluate_rows(const temo_problem *prob, const double *X, const int64_t *rows, int64_t n,
                       double *F, temo_stream_t stream);

/* SBX spread factor (variation.py:77-78) for U = mu[t]: beta[t] = pow(2 mu, e) or
 * pow(1 / (2 - 2 mu), e), e = 1 / (eta_c + 1); fast = 1 uses the exp/log form the fused
 * offspring kernel uses (csrc/sbx_pow.cuh), fast = 0 CUDA's pow.  Diagnostic/parity hook. */
int temo_sbx_beta(const double *mu, int64_t n, double eta_c, int fast, double *beta,
                  temo_stream_t stream);

/* Uniform draws: out[e] = Generator.random() element `off + e` of the stream. */
int temo_uniform(const temo_philox_state *st, uint64_t off, int64_t count, double *out,
                 temo_stream_t stream);

/* variation.sbx (variation.py:57-91): C (2q x d) = clip([c1; c2]).  Uniforms
 * come from the Philox stream at off (mu, then swap and crossed when
 * gene_swap; q*d each) unless the u_* arrays are given (injected draws). */
int temo_sbx(const temo_variation *var, const double *X1, const double *X2, int64_t q, int64_t d,
             const temo_philox_state *st, uint64_t off, const double *u_mu, const double *u_swap,
             const double *u_cross, double *C, temo_stream_t stream);

/* variation.polynomial_mutation (variation.py:94-120): Y (rows x d); draws mu
 * then hit (rows*d each) from the stream at off unless injected. */
int temo_pm(const temo_variation *var, const double *X, int64_t rows, int64_t d,
            const temo_philox_state *st, uint64_t off, const double *u_mu, const double *u_hit,
            double *Y, temo_stream_t stream);

/* Fused generation front end for NSGA-III / HypE (harness.py:201-204, 220):
 * pairs (i1[q], i2[q]) of parent rows of X -> SBX -> PM -> evaluate, writing
 * offspring O (2h x d) and objectives FO (2h x m; NULL skips evaluation).
 * Draws follow the reference call order from `off`: SBX mu/swap/crossed
 * (h*d each), PM mu/hit (2h*d each). */
int temo_offspring(const temo_problem *prob, const temo_variation *var, const double *X,
                   const int64_t *i1, const int64_t *i2, int64_t h, const temo_philox_state *st,
                   uint64_t off, double *O, double *FO, temo_stream_t stream);

/* Same result as temo_offspring, computed in two phases through caller workspace
 * (temo_offspring_ws_bytes(h, d) bytes: h*d betas + per-quad flags): a pure-randomness
 * kernel (Philox draws, SBX betas of crossed genes, PM hit bits) and a streaming apply
 * kernel (parents -> children -> objectives).  Row pool (both NULL = plain layout):
 * parent i is row src_map[i] of X, child r (r < 2h) goes to row dst_rows[r] of O.
 * Falls back to the fused kernel when the streams are not congruent mod 4 or d is
 * above the staged-constant limit (row maps are then rejected with TEMO_EINVAL). */
size_t temo_offspring_ws_bytes(int64_t h, int64_t d);
int temo_offspring_ws(const temo_problem *prob, const temo_variation *var, const double *X,
                      const int64_t *i1, const int64_t *i2, int64_t h, const temo_philox_state *st,
                      uint64_t off, double *O, double *FO, const int64_t *src_map,
                      const int64_t *dst_rows, void *ws, size_t ws_bytes, temo_stream_t stream);
/* Row-sharded form: only the pairs [q0, q1) of the h pairs, with exactly the
 * draws and output rows the full call gives them (Philox elements are indexed by the global
 * pair), so G ranks covering [0, h) together produce the full result bit for bit. */
/* The two phases of temo_offspring_ws_range as separate calls (same workspace), so the
 * randomness of the next generation can run on a side stream while this generation's
 * selection runs (it needs no parent data).  Only when temo_offspring_two_phase(h, d).
 * rand_ws writes the spread factors, the flags and (d even, >= 128) the PM hit list;
 * apply_ws consumes them and must follow a rand_ws call with the same (h, q0, q1, st, off, ws). */
int temo_offspring_two_phase(int64_t h, int64_t d);
int temo_offspring_rand_ws(const temo_variation *var, int64_t d, int64_t h, int64_t q0, int64_t q1,
                           const temo_philox_state *st, uint64_t off, void *ws, size_t ws_bytes,
                           temo_stream_t stream);
int temo_offspring_apply_ws(const temo_problem *prob, const temo_variation *var, const double *X,
                            const int64_t *i1, const int64_t *i2, int64_t h, int64_t q0, int64_t q1,
                            const temo_philox_state *st, uint64_t off, double *O, double *FO,
                            const int64_t *src_map, const int64_t *dst_rows, void *ws, size_t ws_bytes,
                            temo_stream_t stream);
int temo_offspring_ws_range(const temo_problem *prob, const temo_variation *var, const double *X,
                            const int64_t *i1, const int64_t *i2, int64_t h, int64_t q0, int64_t q1,
                            const temo_philox_state *st, uint64_t off, double *O, double *FO,
                            const int64_t *src_map, const int64_t *dst_rows, void *ws, size_t ws_bytes,
                            temo_stream_t stream);

/* Row-pool bookkeeping after a selection (replaces the survivor row copy X[perm][keep] of
 * nsga3.py:218 / hype.py:163): phys (N) maps logical merged rows to pool rows; the n
 * survivors are logical rows perm[keep[p]] (perm NULL = identity).  phys_out[p] =
 * phys[perm[keep[p]]] for p < n, and phys_out[n..N) = the other pool rows in logical
 * order (the free rows the next offspring overwrite).  ws: temo_pool_update_ws_bytes(N). */
size_t temo_pool_update_ws_bytes(int64_t N);
int temo_pool_update(const int64_t *phys, const int64_t *perm, const int32_t *keep, int64_t N, int64_t n,
                     int64_t *phys_out, const int32_t *status, void *ws, size_t ws_bytes,
                     temo_stream_t stream);  /* status (nullable): selection status word; when it
                                                is non-zero the pool is left as it is (phys' = phys) */

/* ------------------------------------------------------------------ MOEA/D
 * temo_moead_offspring: moead.moead_offspring (moead.py:127-145) for parents
 *   p1[i], p2[i] (rows of X): SBX child c1 only, PM, evaluate -> O, FO (n rows);
 *   draws from `off`: SBX mu/swap/crossed then PM mu/hit, n*d each.
 * temo_moead_compare: moead.compare_update (moead.py:70-92) without the n x n
 *   matrix: zmin (m), g_new (n x T) and improves (n x T, 0/1).
 * temo_moead_elite: moead.elite_select (moead.py:95-124) in O(n T) via the
 *   reverse CSR (rptr n+1, rcol = i*T + t sorted by i) of I_nb; winner (n,
 *   -1 = incumbent), Xn (n x d), Fn (n x m).
 * temo_aggregate_rows: moead.pbi (moead.py:43-67) / Tchebycheff on aligned rows.
 * kind: TEMO_AGG_PBI (reference) or TEMO_AGG_TCH (new; parity unpinned). */
#define TEMO_AGG_PBI 0
#define TEMO_AGG_TCH 1
/* temo_moead_offspring with the Philox state read from device memory (st_dev: a
 * temo_philox_state in device memory), so the generation can be captured once in a CUDA
 * graph and replayed with each generation's state.  TEMO_EINVAL unless the staged kernel
 * applies (n*d % 4 == 0, d <= 3000). */
int temo_moead_offspring_dev(const temo_problem *prob, const temo_variation *var, const double *X,
                             const int64_t *p1, const int64_t *p2, int64_t n,
                             const temo_philox_state *st_dev, uint64_t off, double *O, double *FO,
                             temo_stream_t stream);
int temo_moead_offspring(const temo_problem *prob, const temo_variation *var, const double *X,
                         const int64_t *p1, const int64_t *p2, int64_t n,
                         const temo_philox_state *st, uint64_t off, double *O, double *FO,
                         temo_stream_t stream);
int temo_moead_compare(const double *F1, const double *F2, const double *W, const int32_t *I_nb,
                       int64_t n, int T, int m, const double *z, double theta, int kind,
                       double *zmin, double *g_new, uint8_t *improves, temo_stream_t stream);
int temo_moead_elite(const double *X, const double *F1, const double *W, const double *O,
                     const double *F2, int64_t n, int64_t d, int T, int m, const double *zmin,
                     double theta, int kind, const int64_t *rptr, const int32_t *rcol,
                     const double *g_new, const uint8_t *improves, int32_t *winner, double *Xn,
                     double *Fn, temo_stream_t stream);
int temo_aggregate_rows(const double *f, const double *w, const double *z, int64_t rows, int m,
                        double theta, int kind, int normalize, double *out, temo_stream_t stream);

/* harness._Stepper.init (harness.py:188-190): X = lower + U (upper - lower), U from the stream. */
int temo_init_population(const temo_philox_state *st, uint64_t off, int64_t rows, int64_t d,
                         const double *lower, const double *upper, double *X, temo_stream_t stream);

/* -------------------------------------------------------------------- HypE
 * temo_hype_alpha: hype.shared_alpha (hype.py:37-51) -> alpha (n1).
 * temo_hv_estimate: hype.hv_estimate (hype.py:54-85) with v_ref (device, m)
 *   and k given; uniforms from the stream at `off` (s*m outputs, consumed iff
 *   *drew == 1 afterwards: the box is non-degenerate) or injected U (s x m).
 *   Sums follow the OpenBLAS dgemv_t order of SURVEY App. A7.
 * temo_hype_select: hype.py:153-163 on ranks from temo_rank (SELECT mode);
 *   v_ref NULL = auto reference (hype.py:129-132); keep (n int32, lexsort
 *   order); v_hv (N); info (4 int32) = {count(r<=l), k, estimated, drew}. */
int temo_hype_alpha(int64_t n1, int64_t k, double *alpha, temo_stream_t stream);
/* hype.auto_reference (hype.py:129-132); scratch: 32 doubles of device memory */
int temo_auto_reference(const double *F, int64_t n, int m, double *out, double *scratch,
                        temo_stream_t stream);
size_t temo_hv_estimate_ws_bytes(int64_t n1, int m, int64_t s);
int temo_hv_estimate(const double *F, int64_t n1, int m, const double *v_ref, int64_t k, int64_t s,
                     const temo_philox_state *st, uint64_t off, const double *U, double *v_hv,
                     int32_t *drew, void *ws, size_t ws_bytes, temo_stream_t stream);
size_t temo_hype_select_ws_bytes(int64_t N, int m, int64_t s);
int temo_hype_select(const double *F, int64_t N, int m, int64_t n, int64_t s, const double *v_ref,
                     const int32_t *rank, const int32_t *l, const temo_philox_state *st,
                     uint64_t off, const double *U, int32_t *keep, double *v_hv, int32_t *info,
                     void *ws, size_t ws_bytes, temo_stream_t stream);

/* temo_hype_select in three phases (same workspace, same results) so the Monte-Carlo work
 * can be sharded over GPUs by exchange column: the s samples fall in 65,536-sample
 * blocks, each giving its 2,048-sample sub-blocks plus one b % 4 tail as columns
 * (temo_hype_columns(s) in total).  begin: k, alpha, box.  columns: the N-row partial sums
 * of columns [c_lo, c_hi) into Tseg (column-major, N per column; NULL = the workspace's own
 * full buffer).  end: combine all columns of Tg (N x temo_hype_columns(s), column-major; NULL =
 * the workspace's buffer) in the reference's summation order, then the lexsort -> keep.
 * Ranks that each fill a column range and all-gather Tg reproduce the single-GPU bits. */
int64_t temo_hype_columns(int64_t s);
int temo_hype_select_begin(const double *F, int64_t N, int m, int64_t n, int64_t s, const double *v_ref,
                           const int32_t *rank, const int32_t *l, void *ws, size_t ws_bytes, temo_stream_t stream);
int temo_hype_select_columns(const double *F, int64_t N, int m, int64_t s, int64_t c_lo, int64_t c_hi,
                             const temo_philox_state *st, uint64_t off, const double *U, double *Tseg, void *ws,
                             size_t ws_bytes, temo_stream_t stream);
int temo_hype_select_end(const double *F, int64_t N, int m, int64_t n, int64_t s, const int32_t *rank,
                         const int32_t *l, const double *Tg, int32_t *keep, double *v_hv, int32_t *info, void *ws,
                         size_t ws_bytes, temo_stream_t stream);

/* The normalize kernel's np.linalg.solve(E, ones) (nsga3.py:86; OpenBLAS getf2 / blocked
 * getrf order, bit-exact for m <= 16) on `count` row-major matrices E + E_off[i] of size
 * m[i] x m[i]; y + y_off[i] receives the solution, ok[i] = 0 on a zero pivot.  Test hook. */
int temo_lu_solve_batch(const double *E, const int64_t *E_off, const int32_t *m, int64_t count,
                        double *y, const int64_t *y_off, int32_t *ok, temo_stream_t stream);

/* ---------------------------------------------------------------- indicators
 * indicators.py:19-100 on the device (csrc/indicators.cu); `out` is one device double.
 * temo_igd : mean over the r reference points Fstar of the distance to the nearest of the
 *            n rows of F (NumPy's last-axis sum and pairwise mean order).
 * temo_hv  : exact dominated volume for m = 2, 3 (sweep / z-slab decomposition, NumPy's
 *            summation orders); rows with any coordinate >= ref are dropped.  Reads two
 *            counts back to the host (data-dependent slab count).
 * temo_hv_mc_hits : m > 3 Monte-Carlo part: hits[s] = 1 iff some row of F <= S[s].
 * temo_eu  : expected utility of U (= -F when minimising) under r weight rows (best
 *            weighted utility per row, or the per-objective `literal` reading), mean. */
size_t temo_igd_ws_bytes(int64_t r);
int temo_igd(const double *F, int64_t n, int m, const double *Fstar, int64_t r, double *out, void *ws,
             size_t ws_bytes, temo_stream_t stream);
size_t temo_hv_ws_bytes(int64_t n, int m);
int temo_hv(const double *F, int64_t n, int m, const double *ref, double *out, void *ws, size_t ws_bytes,
            temo_stream_t stream);
int temo_hv_mc_hits(const double *F, int64_t n, int m, const double *S, int64_t ns, int32_t *hits,
                    temo_stream_t stream);
size_t temo_eu_ws_bytes(int64_t n, int64_t r, int literal);
int temo_eu(const double *U, int64_t n, int m, const double *W, int64_t r, int literal, double *out, void *ws,
            size_t ws_bytes, temo_stream_t stream);

/* -------------------------------------------------------------------- RVEA
 * rvea.apd_select (rvea.py:33-68).  temo_rvea_prep: unit directions Vn (r x m) and the
 * minimal inter-direction angles gamma (r) of W.  temo_rvea_select: one elite per non-empty
 * angle partition of F (N x m) by smallest angle-penalized distance, winners in direction
 * order into keep (<= r, int32 row indices), their number into *count (device);
 * mp = m * (t / t_max)^alpha.  part_out / apd_out (nullable) receive every row's partition
 * and APD. */
int temo_rvea_prep(const double *W, int64_t r, int m, double *Vn, double *gamma, temo_stream_t stream);
size_t temo_rvea_select_ws_bytes(int64_t N, int m, int64_t r);
int temo_rvea_select(const double *F, int64_t N, int m, const double *Vn, const double *gamma, int64_t r,
                     double mp, int32_t *keep, int32_t *count, int32_t *part_out, double *apd_out, void *ws,
                     size_t ws_bytes, temo_stream_t stream);

/* --------------------------------------------------------------- directions
 * directions.neighbors (directions.py:104-114): out (r x T int32) holds the T
 * nearest rows of W (r x m) by Euclidean distance, ties to the lower index.
 * 1 <= T <= min(r, 64), m <= 16. */
int temo_neighbors(const double *W, int64_t r, int m, int T, int32_t *out, temo_stream_t stream);

/* Measured ceilings for bench.py's roofline_compute denominators (probe.cu): the inner-loop
 * instruction mix of a compute-bound kernel on register operands only.
 *   temo_probe_philox_rate : Philox4x64-10 blocks/s (k_offspring_rand's core)
 *   temo_probe_packed_rate : packed dominance pair tests/s (k_dom_rows8's step, m = 3)
 *   temo_probe_dsub_rate   : FP64 add/sub operations/s (k_hv_dom's sample test)
 * scratch: 8 bytes of device memory (written only to keep the work live). */
double temo_probe_philox_rate(int blocks, int iters, uint64_t *scratch, temo_stream_t stream);
double temo_probe_packed_rate(int blocks, int iters, uint64_t *scratch, temo_stream_t stream);
double temo_probe_dsub_rate(int blocks, int iters, uint64_t *scratch, temo_stream_t stream);
/* The offspring apply phase's access pattern alone (two gathered parent rows + one streamed
 * row in, two scattered child rows out, per pair; d even): bytes/s over `iters` launches. */
double temo_probe_rows_rate(const double *X, const int64_t *pa, const int64_t *pb, const double *B,
                            const int64_t *dst, int64_t h, int64_t d, double *O, int iters,
                            temo_stream_t stream);

/* ------------------------------------------------------------ stage timing
 * CUDA-event timing of each kernel stage on its own stream (off by default).
 * temo_timing_read syncs the recorded events, fills ms_out/calls_out
 * (TEMO_STAGE_COUNT entries each) and optionally resets the accumulators. */
#define TEMO_STAGE_COUNT 16
void temo_timing_enable(int on);
const char *temo_timing_name(int stage);
int temo_timing_read(double *ms_out, int64_t *calls_out, int reset);

#ifdef __cplusplus
}
#endif
#endif /* TEMO_B200_H */
