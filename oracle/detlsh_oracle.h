/*
 * detlsh_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded fp64 CPU implementation of DET-LSH
 * (arxiv 2603.24920) written step by step from the paper.  It exists to prove
 * the CUDA library right.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  It shares no code, header,
 * table or helper with paper_2603_24920_b200/ (the product), and never includes
 * include/detlsh.h.
 *
 * Citations: "P:n" = line n of the paper's LaTeX; AMB-n = the
 * reading of an ambiguous passage listed in DESIGN.md section "Readings".
 */
#ifndef DETLSH_ORACLE_H
#define DETLSH_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- O1: chi-square quantiles and Lemma 3 / Eq. 2 parameters ---- */
double orc_chi2_sf(double y, int K);              /* Pr[Y > y], Y ~ chi2(K) */
double orc_chi2_isf(double alpha, int K);         /* chi2_alpha(K): upper quantile */
/* eps = sqrt(chi2_{alpha1}(K)), alpha1 = e^{-1/L}; alpha2 = Pr[Y > eps^2/c^2];
   beta_theory = 2 - 2 alpha2^L. */
void   orc_params(int K, int L, double c, double* alpha1, double* eps, double* alpha2, double* beta_theory);

/* ---- O2: hash family (Eq. 1) and projection ---- */
uint64_t orc_splitmix64(uint64_t x);
/* A[(i*K+j)*d + t], L*K rows of d entries (AMB-1). */
void   orc_hash_family(uint64_t seed, int d, int L, int K, float* A);
/* P[p*LK + r] = fl32( sum_t (double)A[r*d+t] * (double)X[p*d+t] ), t ascending (AMB-2). */
void   orc_project(const float* A, int LK, int d, const float* X, int64_t n, float* P);

/* ---- O3: sample and breakpoints ---- */
int64_t orc_sample_size(int64_t n, int N_r, double sample_frac);          /* AMB-3 */
/* The n_s ids in [0,n) with the smallest (key(seed^SALT,id), id); written ascending (AMB-4). */
void   orc_sample_ids(uint64_t seed, int64_t n, int64_t n_s, int64_t* ids);
/* Full sort of m values, then the P:299 formula (AMB-5). out has N_r+1 entries. */
void   orc_breakpoints_sort(const float* v, int64_t m, int N_r, float* out);
/* Same order statistics by log2(N_r) rounds of QuickSelect, divide-and-conquer. */
void   orc_breakpoints_qselect(const float* v, int64_t m, int N_r, float* out);

/* ---- O4: dynamic encoding, Alg. 1, AMB-6/7 ---- */
int    orc_encode_value(float x, const float* b, int N_r);

/* ---- O5: DE-Tree, Alg. 2 and SplitNode ---- */
typedef struct orc_tree orc_tree;
/* codes: row p starts at codes + p*stride, K symbols of log2(N_r) bits.
   builder 0 = literal Alg. 2 (insert ids ascending, split while full);
   builder 1 = the equivalent bulk rule (B6). */
orc_tree* orc_tree_build(const uint8_t* codes, int64_t n, int64_t stride, int K, int N_r,
                         int max_size, int builder);
void      orc_tree_free(orc_tree* t);
int64_t   orc_tree_num_leaves(const orc_tree* t);   /* non-empty leaves */
/* Canonical leaf list: first-layer keys ascending, 0-child first, empty leaves dropped.
   leaf_off[nleaves+1], perm[n] (member ids ascending inside each leaf),
   lo[nleaves*K], hi[nleaves*K] = symbol range of the leaf box, bits[nleaves*K]. */
void      orc_tree_export(const orc_tree* t, int64_t* leaf_off, int64_t* perm,
                          uint8_t* lo, uint8_t* hi, uint8_t* bits);

/* ---- O6: node bounds (Fig. dist), AMB-7 unbounded outer regions ---- */
/* For a box with symbol ranges [lo_j,hi_j] and query coords x (K values):
   squared lower / upper bound distances (upper may be +inf). */
void   orc_box_bounds2(const uint8_t* lo, const uint8_t* hi, const float* x, const float* b,
                       int K, int N_r, double* lb2, double* ub2);

/* ---- Index (O2-O5 together, optionally one shard of a larger dataset: O9) ---- */
typedef struct orc_index orc_index;
/* Builds over rows [row_lo,row_hi) of X (borrowed; must outlive the index), with the
   hash family, sample and breakpoints of the whole n_global-row dataset. */
orc_index* orc_build(const float* X, int64_t n_global, int d, int64_t row_lo, int64_t row_hi,
                     int L, int K, int N_r, uint64_t seed, int max_size, double sample_frac,
                     int builder);
void   orc_index_free(orc_index* ix);
int64_t orc_index_n(const orc_index* ix);
int64_t orc_index_n_sample(const orc_index* ix);
const float*   orc_index_A(const orc_index* ix);          /* [LK][d] */
const float*   orc_index_breakpoints(const orc_index* ix);/* [LK][N_r+1] */
const float*   orc_index_P(const orc_index* ix);          /* [n][LK] (shard rows) */
const uint8_t* orc_index_codes(const orc_index* ix);      /* [n][LK] (shard rows) */
const int64_t* orc_index_sample(const orc_index* ix);     /* [n_s] global ids */
const orc_tree* orc_index_tree(const orc_index* ix, int i);
double orc_index_eps(const orc_index* ix);

/* ---- O7: range query, Alg. 3 ---- */
enum { ORC_CELL = 0, ORC_RELAXED = 1, ORC_EXACT = 2 };
/* Literal traversal of tree i from the first-layer nodes; qp = projected query (K values of
   space i).  Writes local ids (ascending) to out (capacity n), returns the count. */
int64_t orc_range_query(const orc_index* ix, int i, const float* qp, double rho, int mode,
                        int64_t* out);

/* ---- O8: c^2-k-ANN, Alg. 5 ---- */
typedef struct {
    int32_t rounds;      /* rounds started */
    int32_t trees_last;  /* trees processed in the last round */
    int32_t reason;      /* 0 = budget (line 7), 1 = radius (line 9), 2 = round cap */
    int32_t pad;
    int64_t n_cand;      /* |S| at termination */
    double  r_final;     /* r of the last round */
} orc_qstats;
/* ids are global (row_lo added); dists = sqrt(d^2) rounded to fp32; missing -> (-1, +inf). */
void   orc_query(const orc_index* ix, const float* Q, int64_t nq, int k, double c, double r_min,
                 double beta, int mode, int64_t* out_ids, float* out_dists, orc_qstats* stats);
/* ---- O8b: (r,c)-ANN, Alg. 4: one id/dist per query, (-1, +inf) for "nothing" ---- */
void   orc_rc_ann(const orc_index* ix, const float* Q, int64_t nq, double c, double r, double beta, int mode,
                  int64_t* out_ids, float* out_dists);
/* Same with lb_order = 1: §6.2.2(2) -- within each tree the qualifying leaves are taken
   in ascending (lower bound, leaf position) order and the budget |S| >= ceil(beta n)+k is
   checked after each leaf instead of after the tree. */
void   orc_query_ex(const orc_index* ix, const float* Q, int64_t nq, int k, double c, double r_min,
                    double beta, int mode, int lb_order, int64_t* out_ids, float* out_dists, orc_qstats* stats);
/* Projected query (the fp32 K*L vector), exposed for tests. */
void   orc_project_query(const orc_index* ix, const float* q, float* qp);

/* ---- O9: shard merge; O10: exact kNN, metrics ---- */
void   orc_merge_topk(const int64_t* ids, const float* dists, int G, int64_t nq, int k,
                      int64_t* out_ids, float* out_dists);
void   orc_exact_knn(const float* X, int64_t n, int d, const float* Q, int64_t nq, int k,
                     int64_t* out_ids, double* out_dists);
/* "Magic" r_min (AMB-22): per sample query the smallest radius r*_q whose full
   round reaches |S| >= ceil(beta n)+k (written to rstar_out if non-NULL); returns the lower
   median over the sample. */
double orc_estimate_rmin(const orc_index* ix, const float* Qs, int64_t ns, int k, double c,
                         double beta, double* rstar_out);

#ifdef __cplusplus
}
#endif
#endif
