/*
 * detlsh.h -- C ABI of the B200-native DET-LSH hot path (arxiv 2603.24920).
 *
 * The library builds L DE-Trees over n points (Alg. 1 dynamic encoding + Alg. 2
 * index creation) and answers batched c^2-k-ANN queries
 * (Alg. 5) entirely in sm_100a CUDA kernels.  Citations "P:n" are
 * lines of the paper's LaTeX; "AMB-n" are the readings listed in DESIGN.md.
 *
 * Conventions for every entry point
 *  - Pointers may be host or device memory (detected with cudaPointerGetAttributes);
 *    host buffers are copied in/out inside the call.  Arrays are row-major, dense.
 *  - The caller owns every input and output buffer.  An index owns its device
 *    memory (including its own copy of the data unless opts.borrow_data is set).
 *  - Functions return a detlsh_status and never abort.  On error no output is
 *    written (no partial results) and detlsh_last_error() describes the failure.
 *  - All work runs on opts->stream (a cudaStream_t cast to uint64; 0 = legacy
 *    default stream).  Calls return after the stream work has completed unless a
 *    function says otherwise.
 *  - An index is read-only after build: concurrent queries on different streams
 *    are allowed.
 */
#ifndef DETLSH_H
#define DETLSH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct detlsh_index detlsh_index; /* opaque; owns device memory */

typedef enum {
    DETLSH_OK = 0,
    DETLSH_EINVAL = 1,    /* bad argument (see each function) */
    DETLSH_ENOMEM = 2,    /* device or host allocation failed */
    DETLSH_ECUDA = 3,     /* a CUDA runtime/kernel error; also "no CUDA device" */
    DETLSH_ENCCL = 4,     /* reserved for collective glue */
    DETLSH_EINTERNAL = 5  /* an internal invariant failed */
} detlsh_status;

/* Range-query predicate inside partially covered leaves (AMB-12). */
enum { DETLSH_MODE_CELL = 0,     /* point's own region lower bound <= eps r (hot path) */
       DETLSH_MODE_RELAXED = 1,  /* Sec. 6.2.2(1): whole leaf when leaf LB <= eps r */
       DETLSH_MODE_EXACT = 2     /* Alg. 3 as written: the point's true projected
                                    distance ||q'_i - p'_i|| <= eps r; needs an index built with
                                    opts.keep_projections = 1 (n*L*K*4 bytes more) */ };

typedef struct {
    int32_t  max_size;     /* leaf capacity of Alg. 2 (AMB-8), default 128 */
    double   sample_frac;  /* n_s = min(n, max(ceil(f n), 32 N_r)) (AMB-3), default 0.01 */
    int32_t  mode;         /* DETLSH_MODE_*, default CELL */
    int32_t  query_batch;  /* queries per device batch, 0 = sized from free memory */
    uint64_t stream;       /* cudaStream_t, 0 = legacy default stream */
    int32_t  borrow_data;  /* 1: keep the caller's device pointer (d % 8 == 0) instead of copying */
    int32_t  proj_impl;    /* projection kernel: 0 = tcgen05 tensor cores, 1 = SIMT fp32 */
    int64_t  mem_budget;   /* bytes of device scratch for query batches, 0 = auto (60% of the
                              memory free at the first query on this device in the process) */
    int32_t  verify_impl;  /* candidate verification (Alg. 5 l.8): 2 = tcgen05 tensor cores
                              (masked dense X.Q^T: ||x||^2 + ||q||^2 - 2 x.q with 3xTF32 dot
                              products, fp32-level accuracy), 1 = CUDA cores (rows staged once,
                              direct fp32 sum of squares per candidate), 3 = sparse gather (the
                              round's candidates listed, one 8-lane group per candidate reads
                              its row), 0 = per round the cheaper of tensor cores and gather for
                              that round's candidate density (default).
                              Either way the returned distances are recomputed directly in fp32. */
    int32_t  keep_projections; /* build: 1 keeps the fp32 projections of every point (EXACT mode) */
    int32_t  lb_order;     /* query: 1 = Sec. 6.2.2(2): within a tree the qualifying leaves
                              are taken in ascending (lower bound, leaf position) order and the
                              budget is checked after each leaf (Alg. 5 line 7 at leaf granularity);
                              0 = Alg. 5 as written (budget after each tree, default) */
    int32_t  pad1;
} detlsh_opts;

/* Per-query statistics (Alg. 5 bookkeeping). */
typedef struct {
    int32_t rounds;      /* radius rounds started (r = r_min c^(rounds-1) at the end) */
    int32_t trees_last;  /* trees processed in the last round */
    int32_t reason;      /* 0 = budget |S| >= beta n + k (line 7), 1 = radius (line 9), 2 = 64-round cap */
    int32_t pad;
    int64_t n_cand;      /* |S| at termination */
    double  r_final;     /* r of the last round */
    int64_t leaves_tested;   /* box lower bounds evaluated (all rounds, all trees): leaves, and in
                                the two-level filter (DETLSH_TILE_PAIRS) query tiles as well */
    int64_t leaves_passed;   /* boxes with LB <= eps r */
    int64_t points_tested;   /* points of qualifying leaves examined */
    int64_t points_passed;   /* points with cell LB <= eps r (before de-duplication) */
    int64_t subboxes_tested; /* sub-box (runs of 8 leaf points) lower bounds evaluated by the pair kernel */
} detlsh_query_stats;

void detlsh_default_opts(detlsh_opts* opts);

/*
 * Build an index over data[n][d] (fp32).  Steps:
 *  hash family A[L*K][d], a ~ N(0,1) from `seed` (Eq. 1; AMB-1);
 *  sample n_s ids (AMB-3/4); project; breakpoints
 *  B[L*K][N_r+1] from the sorted sample (AMB-5); encode every
 *  coordinate to an 8-bit symbol (Alg. 1; AMB-6/7); per tree sort by the
 *  first-layer key and split segments into leaves (Alg. 2 + SplitNode).
 * Errors (EINVAL): data NULL; n < 1 or n >= 2^31; d < 1; L < 1; K < 1 or K > 32;
 *  N_r not a power of two in [2,256]; max_size < 1; sample_frac not in (0,1];
 *  any non-finite value in data.
 */
detlsh_status detlsh_build(const float* data, int64_t n, int32_t d, int32_t L, int32_t K,
                           int32_t N_r, uint64_t seed, detlsh_index** out);

/*
 * As detlsh_build, for one shard of a larger point-sharded dataset:
 *  id_offset   global id of data row 0 (query outputs report global ids);
 *  n_global    rows of the whole dataset (the sample rule and candidate budget of
 *              each shard use this shard's n; n_global only labels ids);
 *  breakpoints nullable [L*K][N_r+1] fp32 (host or device): use these instead of
 *              this shard's own sample (C1: every shard gets the same breakpoints).
 */
detlsh_status detlsh_build_ex(const float* data, int64_t n, int32_t d, int32_t L, int32_t K,
                              int32_t N_r, uint64_t seed, const detlsh_opts* opts,
                              int64_t id_offset, int64_t n_global, const float* breakpoints,
                              detlsh_index** out);

/*
 * c^2-k-ANN for queries[nq][d] (Alg. 5): rounds r = r_min c^m; each round
 * runs the L range queries at radius eps*r (eps from Eq. 2 for (K, L); AMB-23),
 * unions and de-duplicates candidates in a per-query bitmap, stops after a tree once
 * |S| >= ceil(beta n) + k (AMB-17), else after the round once the k-th smallest exact
 * distance <= c r; at most 64 rounds (AMB-20).  Outputs out_ids[nq][k] (global ids,
 * int64) and out_dists[nq][k] (Euclidean, fp32), ascending by (dist, id) (AMB-21);
 * unfilled slots (fewer than k candidates at the cap) are (-1, +inf).
 * Errors (EINVAL): idx NULL; nq < 0; k < 1 or k > n or k > 4096; c <= 1; beta <= 0;
 *  r_min <= 0 or non-finite; NaN/Inf in queries.  nq == 0 is a no-op.
 */
detlsh_status detlsh_query(const detlsh_index* idx, const float* queries, int64_t nq, int32_t k,
                           double c, double r_min, double beta, int64_t* out_ids, float* out_dists);

/* As detlsh_query with options and optional per-query statistics (host or device, [nq]). */
detlsh_status detlsh_query_ex(const detlsh_index* idx, const float* queries, int64_t nq, int32_t k,
                              double c, double r_min, double beta, const detlsh_opts* opts,
                              int64_t* out_ids, float* out_dists, detlsh_query_stats* stats);

/*
 * Test/debug variant of detlsh_query_ex that also exports each query's candidate set S at
 * termination (the union of Alg. 5 line 6, over every tree the query processed): S is
 * host or device memory [nq][S_words] u32, S_words = ceil(n/32); bit (p % 32) of word p / 32 is
 * set iff local id p is in S.  Other arguments, outputs and errors as detlsh_query_ex; EINVAL if
 * S is NULL or S_words != ceil(n/32).
 */
detlsh_status detlsh_query_candidates(const detlsh_index* idx, const float* queries, int64_t nq, int32_t k,
                                      double c, double r_min, double beta, const detlsh_opts* opts,
                                      int64_t* out_ids, float* out_dists, detlsh_query_stats* stats,
                                      uint32_t* S, int64_t S_words);

/*
 * (r,c)-ANN for queries[nq][d] (Alg. 4): one pass over the L trees at radius
 * eps*r; as soon as |S| >= ceil(beta n) + 1 the point of S closest to q is returned
 * (line 6); after the L trees the closest point of S is returned if it lies within c r
 * (lines 8-9), else nothing (line 10).  Outputs out_ids[nq] (global id, or -1 for
 * nothing) and out_dists[nq] (Euclidean fp32, +inf for nothing); stats as for
 * detlsh_query_ex (reason 0 = budget, 1 = within c r, 2 = nothing).  opts: mode,
 * query_batch, stream, verify_impl as for queries.  Errors (EINVAL): as detlsh_query with
 * k = 1, r_min = r.
 */
detlsh_status detlsh_rc_ann(const detlsh_index* idx, const float* queries, int64_t nq, double r,
                            double c, double beta, const detlsh_opts* opts, int64_t* out_ids,
                            float* out_dists, detlsh_query_stats* stats);

/*
 * "Magic" initial radius (AMB-22): for each of ns sample queries [ns][d] (host or
 * device), r*_q = the smallest radius whose full round (all L range queries) gives
 * |S| >= min(n, ceil(beta n) + k) -- i.e. sqrt of the B-th smallest over points of
 * min_i cellLB_i(p), divided by eps.  Writes r*_q to rstar (host, nullable) and the lower
 * median to *r_min (host).  Sample queries are processed in chunks sized from free device
 * memory (ns * n * 4 bytes are never needed at once).  Errors (EINVAL): NULL idx/queries/r_min;
 * ns < 1; k < 1 or k > n; beta <= 0; a median of 0 (more than B points share the sample
 * queries' own cells in every tree -- e.g. very few regions): rstar and *r_min are still
 * written, but 0 is not a valid r_min for detlsh_query, so the caller must choose one.
 */
detlsh_status detlsh_estimate_rmin(const detlsh_index* idx, const float* queries, int64_t ns, int32_t k,
                                   double beta, const detlsh_opts* opts, double* rstar, double* r_min);

void detlsh_free(detlsh_index* idx);

/* Thread-local description of the last failure; valid until the next call on this thread. */
const char* detlsh_last_error(void);

/* ---------------------------------------------------------------- helpers */

/* eps = sqrt(chi2_{alpha1}(K)), alpha1 = e^{-1/L}; alpha2 = Pr[chi2(K) > eps^2/c^2];
   beta_theory = 2 - 2 alpha2^L (Lemma 3 / Eq. 2).  Host only.  Any out may be NULL. */
detlsh_status detlsh_params(int32_t K, int32_t L, double c, double* eps, double* alpha2,
                            double* beta_theory);

/* n_s = min(n, max(ceil(f n), 32 N_r)) (AMB-3).  Host only. */
int64_t detlsh_sample_size(int64_t n, int32_t N_r, double sample_frac);

/*
 * C1 helper for point-sharded builds: projections of this shard's rows that belong to
 * the global sample (the n_s smallest keyed hashes over [0, n_global), AMB-4).
 * data = this shard's rows [n][d]; rows are global ids id_offset..id_offset+n-1.
 * out = device or host [cap][L*K] fp32; *n_out = rows written.  EINVAL if cap is too small.
 */
detlsh_status detlsh_sample_projections(const float* data, int64_t n, int32_t d, int32_t L,
                                        int32_t K, int32_t N_r, uint64_t seed, double sample_frac,
                                        int64_t id_offset, int64_t n_global, const detlsh_opts* opts,
                                        float* out, int64_t cap, int64_t* n_out);

/* Breakpoints [L*K][N_r+1] from m sample projections [m][L*K] (AMB-5),
   by device radix sort.  Pointers host or device. */
detlsh_status detlsh_breakpoints_from_samples(const float* samples, int64_t m, int32_t LK,
                                              int32_t N_r, const detlsh_opts* opts, float* out);

/*
 * C2 merge: G per-shard top-k lists ids[G][nq][k], dists[G][nq][k], each sorted
 * ascending by (dist, id) with empty slots (id < 0) last (as detlsh_query writes them) -> the k
 * best by (dist, id) (AMB-21); unfilled output slots are (-1, +inf).  Pointers host or device
 * (host inputs are staged); the merge runs on the device (k_merge_topk: rank of each element
 * = its index + binary-searched counts in the other lists), on the legacy default stream.
 * Errors (EINVAL): NULL pointer; G < 1; nq < 0; k < 1.
 */
detlsh_status detlsh_merge_topk(const int64_t* ids, const float* dists, int32_t G, int64_t nq,
                                int32_t k, int64_t* out_ids, float* out_dists);

/* Projection P = X A^T of m rows with the index's hash family, [m][L*K] fp32. */
detlsh_status detlsh_project(const detlsh_index* idx, const float* X, int64_t m, float* out);
/* As detlsh_project with an explicit kernel: proj_impl 0 = tcgen05, 1 = SIMT fp32. */
detlsh_status detlsh_project_ex(const detlsh_index* idx, const float* X, int64_t m, int32_t proj_impl,
                                float* out);

/*
 * Test/debug export of index contents.  what:
 *  0 A [L*K][d] f32          1 breakpoints [L*K][N_r+1] f32    2 codes [n][L*K] u8 (data order)
 *  3 sample ids [n_s] i64    4 tree perm [n] i64 (leaf order)   5 tree leaf_off [nl+1] i64
 *  6 tree leaf lo [nl][K] u8 7 tree leaf hi [nl][K] u8         8 tree leaf bits [nl][K] u8
 *  9 scalars i64[4] = {n, n_s, nl(tree), d}
 * `tree` selects the tree for 4-9.  dst is host memory of `bytes`; *needed gets the size.
 * EINVAL if bytes < needed (nothing written).
 */
detlsh_status detlsh_debug_export(const detlsh_index* idx, int32_t what, int32_t tree, void* dst,
                                  size_t bytes, size_t* needed);

/* Test hook: build only the L trees from given codes[n][L*K] (host or device), so the GPU
   tree builder can be cross-fed the oracle's codes (SURVEY §8(c) acceptance 3). */
detlsh_status detlsh_build_from_codes(const uint8_t* codes, int64_t n, int32_t L, int32_t K,
                                      int32_t N_r, const detlsh_opts* opts, detlsh_index** out);

/* Index persistence.  save writes every device array of the index (the data
   rows included, also when borrowed) to `path` (binary, little-endian, versioned header);
   load reads it back into device memory of the current device and returns a new index the
   caller frees with detlsh_free.  Both are synchronous.  Errors: EINVAL (NULL or unopenable
   path, not an index file, truncated file, unsupported version), ENOMEM, ECUDA. */
detlsh_status detlsh_save(const detlsh_index* idx, const char* path);
detlsh_status detlsh_load(const char* path, detlsh_index** out);

/* Shape of an index: info[8] = {n, d, L, K, N_r, n_global, id_offset, codes_only}.
   Errors: EINVAL on NULL. */
detlsh_status detlsh_index_info(const detlsh_index* idx, int64_t* info);

/* Number of kernels this library has launched in this process (evidence counter). */
int64_t detlsh_launch_count(void);

/* Scratch workspaces.  Every call that launches work bump-allocates its scratch from a
   grow-only device arena owned by the library for its (device, stream), so repeated calls do
   not go through the allocator (and never wait on the driver mapping memory).  The arena
   keeps the high-water scratch of the largest call made on that stream (about 2 GB for a
   1000-query batch at n = 1M).  release frees every arena (call it with no work in flight
   on those streams) and returns the unused memory the library's scratch and index pools hold
   reserved on the current device to the driver; bytes reports what the arenas hold.  Neither
   fails. */
void    detlsh_release_workspace(void);
int64_t detlsh_workspace_bytes(void);

/* Per-kernel device time, measured with CUDA events recorded on each launch's stream while
   enabled (used by bench.py for the live roofline).  read returns the number of kernels and
   fills up to cap records (aggregated since the last reset). */
typedef struct {
    char    name[64];
    int64_t launches;
    double  total_ms;
} detlsh_kernel_time;
void    detlsh_profile_enable(int32_t on);
/* Time only kernels whose name starts with one of the comma-separated prefixes (NULL or "":
   every kernel); fewer event records keep the timed region close to an unprofiled run. */
void    detlsh_profile_filter(const char* prefixes);
void    detlsh_profile_reset(void);
int32_t detlsh_profile_read(detlsh_kernel_time* out, int32_t cap);

#ifdef __cplusplus
}
#endif
#endif /* DETLSH_H */
