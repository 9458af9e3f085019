/*
 * detlsh_oracle.c -- TEST INFRASTRUCTURE ONLY (see detlsh_oracle.h).
 *
 * Plain single-threaded C, double arithmetic, written in the paper's order and
 * notation.  No blocking, fusion or reordering beyond what a definition states;
 * library primitives used as steps: qsort, exp/log/lgamma/sqrt/cos.
 *
 * Compile with -ffp-contract=off (no FMA contraction) so every sum is the plain
 * left-to-right double sum the comments describe.
 */
#include "detlsh_oracle.h"

#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ORC_MAXK 32

static void* xmalloc(size_t n) {
    void* p = malloc(n ? n : 1);
    if (!p) { fprintf(stderr, "oracle: out of memory (%zu bytes)\n", n); abort(); }
    return p;
}
static void* xcalloc(size_t n, size_t s) {
    void* p = calloc(n ? n : 1, s ? s : 1);
    if (!p) { fprintf(stderr, "oracle: out of memory\n"); abort(); }
    return p;
}

/* ======================================================================== */
/* O1. chi-square upper quantile.  Lemma 2: chi2_alpha(K) is the  */
/* y with Pr[Y > y] = alpha, Y ~ chi2(K).  Pr[Y > y] = Q(K/2, y/2), the       */
/* regularised upper incomplete gamma function.                               */
/* ======================================================================== */

/* Q(a,x) by the power series of P(a,x) for x < a+1, else by the continued
   fraction of Q(a,x) (modified Lentz). */
static double reg_upper_gamma(double a, double x) {
    if (x <= 0.0) return 1.0;
    double lpre = -x + a * log(x) - lgamma(a);
    if (x < a + 1.0) {
        double term = 1.0 / a, sum = term;
        for (int n = 1; n < 100000; ++n) {
            term *= x / (a + n);
            sum += term;
            if (fabs(term) < fabs(sum) * 1e-17) break;
        }
        return 1.0 - sum * exp(lpre);
    }
    const double tiny = 1e-300;
    double b = x + 1.0 - a, c = 1.0 / tiny, d = 1.0 / b, h = d;
    for (int i = 1; i < 100000; ++i) {
        double an = -i * (i - a);
        b += 2.0;
        d = an * d + b;
        if (fabs(d) < tiny) d = tiny;
        c = b + an / c;
        if (fabs(c) < tiny) c = tiny;
        d = 1.0 / d;
        double del = d * c;
        h *= del;
        if (fabs(del - 1.0) < 1e-17) break;
    }
    return exp(lpre) * h;
}

double orc_chi2_sf(double y, int K) { return reg_upper_gamma(0.5 * K, 0.5 * y); }

/* Bisection on the decreasing survival function; bracket [0, K+40 sqrt(2K)],
   widened if needed (SPEC S:143 convention). */
double orc_chi2_isf(double alpha, int K) {
    double lo = 0.0, hi = K + 40.0 * sqrt(2.0 * K);
    while (orc_chi2_sf(hi, K) > alpha) hi *= 2.0;
    for (int it = 0; it < 400; ++it) {
        double mid = 0.5 * (lo + hi);
        if (orc_chi2_sf(mid, K) > alpha) lo = mid; else hi = mid;
        if (hi - lo <= 1e-15 * (hi > 1.0 ? hi : 1.0)) break;
    }
    return 0.5 * (lo + hi);
}

/* Lemma 3 / Eq. 2: L = -1/ln(alpha1)  =>  alpha1 = e^{-1/L};
   eps^2 = chi2_{alpha1}(K) = c^2 chi2_{alpha2}(K)  =>  alpha2 = Pr[Y > eps^2/c^2];
   beta = 2 - 2 alpha2^L. */
void orc_params(int K, int L, double c, double* alpha1, double* eps, double* alpha2,
                double* beta_theory) {
    double a1 = exp(-1.0 / L);
    double e2 = orc_chi2_isf(a1, K);
    double a2 = orc_chi2_sf(e2 / (c * c), K);
    if (alpha1) *alpha1 = a1;
    if (eps) *eps = sqrt(e2);
    if (alpha2) *alpha2 = a2;
    if (beta_theory) *beta_theory = 2.0 - 2.0 * pow(a2, (double)L);
}

/* ======================================================================== */
/* O2. Hash family h(o) = a.o, a_t ~ N(0,1) (Eq. 1).  The paper   */
/* names no generator; AMB-1 fixes a counter-based one (splitmix64 keys,     */
/* Box-Muller) rounded to TF32 precision (11 significant bits).              */
/* ======================================================================== */
uint64_t orc_splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static uint64_t orc_key(uint64_t s, uint64_t c) { return orc_splitmix64(s ^ orc_splitmix64(c)); }

/* Round an fp32 value to nearest-even at mantissa bit 13 (10 explicit bits). */
static float round_to_tf32(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    u += 0xFFFu + ((u >> 13) & 1u);
    u &= ~0x1FFFu;
    memcpy(&f, &u, 4);
    return f;
}

void orc_hash_family(uint64_t seed, int d, int L, int K, float* A) {
    const double two_pi = 6.283185307179586476925286766559;
    int64_t total = (int64_t)L * K * d;
    for (int64_t e = 0; e < total; ++e) {
        double u1 = (double)(orc_key(seed, 2 * (uint64_t)e) >> 11) * (1.0 / 9007199254740992.0);
        double u2 = (double)(orc_key(seed, 2 * (uint64_t)e + 1) >> 11) * (1.0 / 9007199254740992.0);
        double g = sqrt(-2.0 * log(1.0 - u1)) * cos(two_pi * u2);
        A[e] = round_to_tf32((float)g);
    }
}

/* P = X A^T: every output is the double sum over t ascending of A[r][t]*X[p][t],
   rounded once to fp32 (AMB-2).  The t loop is outermost per point only so the
   LK independent sums can proceed together; each sum's order is unchanged. */
void orc_project(const float* A, int LK, int d, const float* X, int64_t n, float* P) {
    double* At = (double*)xmalloc(sizeof(double) * (size_t)LK * d);
    for (int r = 0; r < LK; ++r)
        for (int t = 0; t < d; ++t) At[(size_t)t * LK + r] = (double)A[(size_t)r * d + t];
    double* acc = (double*)xmalloc(sizeof(double) * LK);
    for (int64_t p = 0; p < n; ++p) {
        const float* x = X + (size_t)p * d;
        for (int r = 0; r < LK; ++r) acc[r] = 0.0;
        for (int t = 0; t < d; ++t) {
            double xt = (double)x[t];
            const double* a = At + (size_t)t * LK;
            for (int r = 0; r < LK; ++r) acc[r] += a[r] * xt;
        }
        for (int r = 0; r < LK; ++r) P[(size_t)p * LK + r] = (float)acc[r];
    }
    free(acc);
    free(At);
}

/* ======================================================================== */
/* O3. Sample and breakpoints.                        */
/* ======================================================================== */
#define ORC_SAMPLE_SALT 0x53414D504C45ULL /* "SAMPLE" */

/* AMB-3: n_s = min(n, max(ceil(f n), 32 N_r)).  P:332 uses f = 0.1; the
   configs use a 1% sample. */
int64_t orc_sample_size(int64_t n, int N_r, double sample_frac) {
    int64_t a = (int64_t)ceil(sample_frac * (double)n);
    int64_t floor_ = 32 * (int64_t)N_r;
    int64_t m = a > floor_ ? a : floor_;
    return m < n ? m : n;
}

typedef struct { uint64_t key; int64_t id; } keyid;
static int cmp_keyid(const void* a, const void* b) {
    const keyid* x = (const keyid*)a; const keyid* y = (const keyid*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return (x->id > y->id) - (x->id < y->id);
}
static int cmp_i64(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}
/* AMB-4: "randomly sample n_s points" read as the n_s ids with the
   smallest keyed hash, ties by id: a pure function of (seed, id). */
void orc_sample_ids(uint64_t seed, int64_t n, int64_t n_s, int64_t* ids) {
    keyid* v = (keyid*)xmalloc(sizeof(keyid) * (size_t)n);
    uint64_t s = seed ^ ORC_SAMPLE_SALT;
    for (int64_t i = 0; i < n; ++i) { v[i].key = orc_key(s, (uint64_t)i); v[i].id = i; }
    qsort(v, (size_t)n, sizeof(keyid), cmp_keyid);
    for (int64_t i = 0; i < n_s; ++i) ids[i] = v[i].id;
    free(v);
    qsort(ids, (size_t)n_s, sizeof(int64_t), cmp_i64);
}

static int cmp_f32(const void* a, const void* b) {
    float x = *(const float*)a, y = *(const float*)b;
    return (x > y) - (x < y);
}
/* Position (0-based, in the sorted sample) of breakpoint t, 1 <= t <= N_r-1:
   P:299 B(z) = C^(floor(m/N_r)(z-1)) for z = t+1, 1-based C^ (AMB-5). */
static int64_t bp_pos(int64_t m, int N_r, int t) {
    int64_t stride = m / N_r;
    if (stride < 1) stride = 1;
    int64_t p = (int64_t)t * stride;
    if (p > m) p = m;
    return p - 1;
}
void orc_breakpoints_sort(const float* v, int64_t m, int N_r, float* out) {
    float* s = (float*)xmalloc(sizeof(float) * (size_t)m);
    memcpy(s, v, sizeof(float) * (size_t)m);
    qsort(s, (size_t)m, sizeof(float), cmp_f32);
    out[0] = s[0];                                   /* B(1) = C^(1): minimum */
    for (int t = 1; t < N_r; ++t) out[t] = s[bp_pos(m, N_r, t)];
    out[N_r] = s[m - 1];                             /* B(N_r+1) = C^(n): maximum */
    free(s);
}

/* QuickSelect(start, q, end): place the q-th smallest of a[lo..hi] at
   position q, smaller to its left, larger to its right.  Three-way partition
   around a median-of-three pivot. */
static void quickselect(float* a, int64_t lo, int64_t hi, int64_t q) {
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        float x = a[lo], y = a[mid], z = a[hi];
        float pv = (x < y) ? ((y < z) ? y : ((x < z) ? z : x)) : ((x < z) ? x : ((y < z) ? z : y));
        int64_t lt = lo, i = lo, gt = hi;
        while (i <= gt) {
            if (a[i] < pv) { float t = a[lt]; a[lt] = a[i]; a[i] = t; ++lt; ++i; }
            else if (a[i] > pv) { float t = a[gt]; a[gt] = a[i]; a[i] = t; --gt; }
            else ++i;
        }
        if (q < lt) hi = lt - 1;
        else if (q > gt) lo = gt + 1;
        else return;
    }
}
/* Divide and conquer: round z selects 2^{z-1} breakpoints, each inside
   the sub-range left by the previous round. */
static void dc_select(float* a, int64_t m, int N_r, int t_lo, int t_hi, int64_t lo, int64_t hi,
                      float* out) {
    if (t_hi - t_lo < 2) return;
    int t = (t_lo + t_hi) / 2;
    int64_t p = bp_pos(m, N_r, t);
    quickselect(a, lo, hi, p);
    out[t] = a[p];
    dc_select(a, m, N_r, t_lo, t, lo, p, out);
    dc_select(a, m, N_r, t, t_hi, p, hi, out);
}
void orc_breakpoints_qselect(const float* v, int64_t m, int N_r, float* out) {
    float* a = (float*)xmalloc(sizeof(float) * (size_t)m);
    memcpy(a, v, sizeof(float) * (size_t)m);
    float mn = a[0], mx = a[0];
    for (int64_t i = 1; i < m; ++i) { if (a[i] < mn) mn = a[i]; if (a[i] > mx) mx = a[i]; }
    out[0] = mn;                                     /* min and max are B(1), B(N_r+1) */
    out[N_r] = mx;
    dc_select(a, m, N_r, 0, N_r, 0, m - 1, out);
    free(a);
}

/* ======================================================================== */
/* O4. Alg. 1 line 6: BinarySearch for the region of h.  AMB-6: a    */
/* value equal to an interior breakpoint goes to the lower region; AMB-7:    */
/* values outside [B(1), B(N_r+1)] clamp to the outer symbols.  So the code  */
/* is the number of interior breakpoints b_1..b_{N_r-1} strictly below x.    */
/* ======================================================================== */
int orc_encode_value(float x, const float* b, int N_r) {
    int lo = 1, hi = N_r;          /* search b[1..N_r-1] for the first b_t >= x */
    while (lo < hi) {
        int mid = lo + (hi - lo) / 2;
        if (b[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo - 1;
}

/* ======================================================================== */
/* O5. DE-Tree (Alg. 2; SplitNode P:357-360).                     */
/* ======================================================================== */
typedef struct {
    int32_t child[2];      /* -1 for a leaf */
    int32_t split_dim;
    uint8_t bits[ORC_MAXK];
    uint8_t pre[ORC_MAXK]; /* symbol prefix of bits[j] bits */
    int64_t* ids;          /* leaf entries <ep, pos>; we keep pos (ep is codes[pos]) */
    int64_t size, cap;
} onode;

struct orc_tree {
    int K, N_r, nb, max_size;
    const uint8_t* codes;
    int64_t n, stride;
    onode* nodes;
    int64_t nnodes, capnodes;
    int32_t* first;        /* first-layer node per distinct key, keys ascending */
    uint32_t* first_key;
    int64_t nfirst;
};

static int32_t new_node(orc_tree* t) {
    if (t->nnodes == t->capnodes) {
        t->capnodes = t->capnodes ? 2 * t->capnodes : 1024;
        t->nodes = (onode*)realloc(t->nodes, sizeof(onode) * (size_t)t->capnodes);
        if (!t->nodes) abort();
    }
    onode* nd = &t->nodes[t->nnodes];
    memset(nd, 0, sizeof(onode));
    nd->child[0] = nd->child[1] = -1;
    nd->split_dim = -1;
    return (int32_t)t->nnodes++;
}
static void leaf_push(onode* nd, int64_t id) {
    if (nd->size == nd->cap) {
        nd->cap = nd->cap ? 2 * nd->cap : 8;
        nd->ids = (int64_t*)realloc(nd->ids, sizeof(int64_t) * (size_t)nd->cap);
        if (!nd->ids) abort();
    }
    nd->ids[nd->size++] = id;
}
static inline int sym(const orc_tree* t, int64_t id, int j) { return t->codes[id * t->stride + j]; }
/* Bit of symbol s right below a prefix of `bits` bits (MSB first). */
static inline int next_bit(int s, int bits, int nb) { return (s >> (nb - 1 - bits)) & 1; }

/* First-layer key: one bit (the MSB) per dimension, dimension 0 most significant (AMB-11). */
static uint32_t first_key(const orc_tree* t, int64_t id) {
    uint32_t key = 0;
    for (int j = 0; j < t->K; ++j) key = (key << 1) | (uint32_t)next_bit(sym(t, id, j), 0, t->nb);
    return key;
}

/* SplitNode's choice (AMB-9): among dimensions with bits left, the one
   whose next bit most evenly partitions the node's entries (|n0-n1| minimal),
   ties to the lowest dimension; -1 if no dimension has bits left. */
static int choose_split(const orc_tree* t, const onode* nd, const int64_t* ids, int64_t m) {
    int best = -1;
    int64_t best_imb = INT64_MAX;
    for (int j = 0; j < t->K; ++j) {
        if (nd->bits[j] >= t->nb) continue;
        int64_t ones = 0;
        for (int64_t e = 0; e < m; ++e) ones += next_bit(sym(t, ids[e], j), nd->bits[j], t->nb);
        int64_t imb = m - 2 * ones;
        if (imb < 0) imb = -imb;
        if (imb < best_imb) { best_imb = imb; best = j; }
    }
    return best;
}
static void make_children(orc_tree* t, int32_t ni, int j) {
    int32_t c0 = new_node(t);
    int32_t c1 = new_node(t);
    onode* nd = &t->nodes[ni];
    for (int b = 0; b < 2; ++b) {
        onode* ch = &t->nodes[b ? c1 : c0];
        memcpy(ch->bits, nd->bits, sizeof(nd->bits));
        memcpy(ch->pre, nd->pre, sizeof(nd->pre));
        ch->bits[j] = (uint8_t)(nd->bits[j] + 1);
        ch->pre[j] = (uint8_t)((nd->pre[j] << 1) | b);
    }
    nd->child[0] = c0;
    nd->child[1] = c1;
    nd->split_dim = j;
}
/* SplitNode on a leaf: it becomes internal with two children; the
   entries move in their current (insertion) order.  Returns 0 if unsplittable. */
static int split_leaf(orc_tree* t, int32_t ni) {
    int j = choose_split(t, &t->nodes[ni], t->nodes[ni].ids, t->nodes[ni].size);
    if (j < 0) return 0;
    make_children(t, ni, j);
    onode* nd = &t->nodes[ni];
    int bits = nd->bits[j];
    for (int64_t e = 0; e < nd->size; ++e) {
        int64_t id = nd->ids[e];
        leaf_push(&t->nodes[nd->child[next_bit(sym(t, id, j), bits, t->nb)]], id);
        nd = &t->nodes[ni];   /* realloc-safe: nodes array is not resized here */
    }
    free(nd->ids);
    nd->ids = NULL;
    nd->size = nd->cap = 0;
    return 1;
}

/* simple open-addressing map uint32 key -> node index */
typedef struct { uint32_t* keys; int32_t* vals; uint64_t cap; } kmap;
static void kmap_init(kmap* m, int64_t expect) {
    uint64_t cap = 16;
    while (cap < (uint64_t)(2 * expect)) cap <<= 1;
    m->cap = cap;
    m->keys = (uint32_t*)xmalloc(sizeof(uint32_t) * cap);
    m->vals = (int32_t*)xmalloc(sizeof(int32_t) * cap);
    for (uint64_t i = 0; i < cap; ++i) m->vals[i] = -1;
}
static int32_t* kmap_slot(kmap* m, uint32_t key) {
    uint64_t h = orc_splitmix64(key) & (m->cap - 1);
    while (m->vals[h] >= 0 && m->keys[h] != key) h = (h + 1) & (m->cap - 1);
    m->keys[h] = key;
    return &m->vals[h];
}
static void kmap_free(kmap* m) { free(m->keys); free(m->vals); }

typedef struct { uint32_t key; int32_t node; } keynode;
static int cmp_keynode(const void* a, const void* b) {
    uint32_t x = ((const keynode*)a)->key, y = ((const keynode*)b)->key;
    return (x > y) - (x < y);
}
static void collect_first(orc_tree* t, kmap* m) {
    int64_t cnt = 0;
    for (uint64_t h = 0; h < m->cap; ++h) cnt += m->vals[h] >= 0;
    keynode* kn = (keynode*)xmalloc(sizeof(keynode) * (size_t)(cnt ? cnt : 1));
    int64_t c = 0;
    for (uint64_t h = 0; h < m->cap; ++h)
        if (m->vals[h] >= 0) { kn[c].key = m->keys[h]; kn[c].node = m->vals[h]; ++c; }
    qsort(kn, (size_t)cnt, sizeof(keynode), cmp_keynode);
    t->nfirst = cnt;
    t->first = (int32_t*)xmalloc(sizeof(int32_t) * (size_t)(cnt ? cnt : 1));
    t->first_key = (uint32_t*)xmalloc(sizeof(uint32_t) * (size_t)(cnt ? cnt : 1));
    for (int64_t i = 0; i < cnt; ++i) { t->first[i] = kn[i].node; t->first_key[i] = kn[i].key; }
    free(kn);
}
static int32_t first_layer_node(orc_tree* t, kmap* m, uint32_t key) {
    int32_t* slot = kmap_slot(m, key);
    if (*slot < 0) {
        int32_t ni = new_node(t);
        onode* nd = &t->nodes[ni];
        for (int j = 0; j < t->K; ++j) {
            nd->bits[j] = 1;
            nd->pre[j] = (uint8_t)((key >> (t->K - 1 - j)) & 1u);
        }
        *slot = ni;
    }
    return *slot;
}

/* Literal Alg. 2: insert points z = 1..n (ids ascending, AMB-10); while the
   target leaf holds >= max_size entries, split it and re-route. */
static void build_literal(orc_tree* t) {
    int64_t nk = t->n < ((int64_t)1 << (t->K < 30 ? t->K : 30)) ? t->n : ((int64_t)1 << (t->K < 30 ? t->K : 30));
    kmap m;
    kmap_init(&m, nk);
    for (int64_t z = 0; z < t->n; ++z) {
        int32_t ni = first_layer_node(t, &m, first_key(t, z));
        for (;;) {
            while (t->nodes[ni].child[0] >= 0) {
                const onode* nd = &t->nodes[ni];
                int j = nd->split_dim;
                ni = nd->child[next_bit(sym(t, z, j), nd->bits[j], t->nb)];
            }
            if (t->nodes[ni].size >= t->max_size && split_leaf(t, ni)) continue;  /* re-route */
            break;
        }
        leaf_push(&t->nodes[ni], z);
    }
    collect_first(t, &m);
    kmap_free(&m);
}

/* Bulk rule (B6): a node holding the id-ascending set S, |S| > max_size,
   splits on the dimension chosen from the first max_size ids of S; children get
   the stable partition.  Equivalent to build_literal (proof in DESIGN.md). */
static void bulk_node(orc_tree* t, int32_t ni, int64_t* ids, int64_t m, int64_t* tmp) {
    if (m <= t->max_size) {
        for (int64_t e = 0; e < m; ++e) leaf_push(&t->nodes[ni], ids[e]);
        return;
    }
    int j = choose_split(t, &t->nodes[ni], ids, t->max_size);
    if (j < 0) {
        for (int64_t e = 0; e < m; ++e) leaf_push(&t->nodes[ni], ids[e]);
        return;
    }
    make_children(t, ni, j);
    int bits = t->nodes[ni].bits[j];
    int64_t z = 0;
    for (int64_t e = 0; e < m; ++e)
        if (!next_bit(sym(t, ids[e], j), bits, t->nb)) tmp[z++] = ids[e];
    int64_t o = z;
    for (int64_t e = 0; e < m; ++e)
        if (next_bit(sym(t, ids[e], j), bits, t->nb)) tmp[o++] = ids[e];
    memcpy(ids, tmp, sizeof(int64_t) * (size_t)m);
    int32_t c0 = t->nodes[ni].child[0], c1 = t->nodes[ni].child[1];
    bulk_node(t, c0, ids, z, tmp);
    bulk_node(t, c1, ids + z, m - z, tmp);
}
typedef struct { uint32_t key; int64_t id; } keyid32;
static int cmp_keyid32(const void* a, const void* b) {
    const keyid32* x = (const keyid32*)a; const keyid32* y = (const keyid32*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return (x->id > y->id) - (x->id < y->id);
}
static void build_bulk(orc_tree* t) {
    keyid32* kv = (keyid32*)xmalloc(sizeof(keyid32) * (size_t)t->n);
    for (int64_t z = 0; z < t->n; ++z) { kv[z].key = first_key(t, z); kv[z].id = z; }
    qsort(kv, (size_t)t->n, sizeof(keyid32), cmp_keyid32);
    int64_t* ids = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)t->n);
    int64_t* tmp = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)t->n);
    for (int64_t z = 0; z < t->n; ++z) ids[z] = kv[z].id;
    int64_t nk = t->n < ((int64_t)1 << (t->K < 30 ? t->K : 30)) ? t->n : ((int64_t)1 << (t->K < 30 ? t->K : 30));
    kmap m;
    kmap_init(&m, nk);
    int64_t s = 0;
    while (s < t->n) {
        int64_t e = s;
        while (e < t->n && kv[e].key == kv[s].key) ++e;
        int32_t ni = first_layer_node(t, &m, kv[s].key);
        bulk_node(t, ni, ids + s, e - s, tmp);
        s = e;
    }
    collect_first(t, &m);
    kmap_free(&m);
    free(kv); free(ids); free(tmp);
}

orc_tree* orc_tree_build(const uint8_t* codes, int64_t n, int64_t stride, int K, int N_r,
                         int max_size, int builder) {
    orc_tree* t = (orc_tree*)xcalloc(1, sizeof(orc_tree));
    t->K = K; t->N_r = N_r; t->max_size = max_size; t->codes = codes; t->n = n; t->stride = stride;
    t->nb = 0;
    while ((1 << t->nb) < N_r) ++t->nb;
    if (builder == 0) build_literal(t); else build_bulk(t);
    return t;
}
void orc_tree_free(orc_tree* t) {
    if (!t) return;
    for (int64_t i = 0; i < t->nnodes; ++i) free(t->nodes[i].ids);
    free(t->nodes); free(t->first); free(t->first_key); free(t);
}

static int64_t count_leaves(const orc_tree* t, int32_t ni) {
    const onode* nd = &t->nodes[ni];
    if (nd->child[0] < 0) return nd->size > 0;
    return count_leaves(t, nd->child[0]) + count_leaves(t, nd->child[1]);
}
int64_t orc_tree_num_leaves(const orc_tree* t) {
    int64_t c = 0;
    for (int64_t i = 0; i < t->nfirst; ++i) c += count_leaves(t, t->first[i]);
    return c;
}
static void leaf_box(const orc_tree* t, const onode* nd, uint8_t* lo, uint8_t* hi) {
    for (int j = 0; j < t->K; ++j) {
        int free_bits = t->nb - nd->bits[j];
        int l = nd->pre[j] << free_bits;
        lo[j] = (uint8_t)l;
        hi[j] = (uint8_t)(l + (1 << free_bits) - 1);
    }
}
typedef struct { int64_t leaf, pos; } exp_state;
static void export_node(const orc_tree* t, int32_t ni, exp_state* st, int64_t* leaf_off,
                        int64_t* perm, uint8_t* lo, uint8_t* hi, uint8_t* bits) {
    const onode* nd = &t->nodes[ni];
    if (nd->child[0] >= 0) {
        export_node(t, nd->child[0], st, leaf_off, perm, lo, hi, bits);
        export_node(t, nd->child[1], st, leaf_off, perm, lo, hi, bits);
        return;
    }
    if (nd->size == 0) return;
    int64_t l = st->leaf++;
    leaf_off[l] = st->pos;
    for (int64_t e = 0; e < nd->size; ++e) perm[st->pos++] = nd->ids[e];
    leaf_off[l + 1] = st->pos;
    leaf_box(t, nd, lo + l * t->K, hi + l * t->K);
    for (int j = 0; j < t->K; ++j) bits[l * t->K + j] = nd->bits[j];
}
void orc_tree_export(const orc_tree* t, int64_t* leaf_off, int64_t* perm, uint8_t* lo, uint8_t* hi,
                     uint8_t* bits) {
    exp_state st = {0, 0};
    leaf_off[0] = 0;
    for (int64_t i = 0; i < t->nfirst; ++i) export_node(t, t->first[i], &st, leaf_off, perm, lo, hi, bits);
}

/* ======================================================================== */
/* O6. Bounds (Fig. dist).  Per dimension, a box with symbol range */
/* [lo,hi] spans (l,u] with l = b_lo (or -inf if lo = 0) and u = b_{hi+1} (or */
/* +inf if hi = N_r-1), AMB-7.  LB_j = max(0, l-x, x-u), UB_j = max(|x-l|,    */
/* |x-u|); LB = sqrt(sum LB_j^2), UB = sqrt(sum UB_j^2).  Squares are returned. */
/* ======================================================================== */
static void dim_bounds(int lo, int hi, double x, const float* b, int N_r, double* lbj, double* ubj) {
    double l = lo >= 1 ? (double)b[lo] : -INFINITY;
    double u = hi <= N_r - 2 ? (double)b[hi + 1] : INFINITY;
    double lb = 0.0;
    if (l - x > lb) lb = l - x;
    if (x - u > lb) lb = x - u;
    double a1 = fabs(x - l), a2 = fabs(x - u);
    *lbj = lb;
    *ubj = a1 > a2 ? a1 : a2;
}
void orc_box_bounds2(const uint8_t* lo, const uint8_t* hi, const float* x, const float* b, int K,
                     int N_r, double* lb2, double* ub2) {
    double sl = 0.0, su = 0.0;
    for (int j = 0; j < K; ++j) {
        double lbj, ubj;
        dim_bounds(lo[j], hi[j], (double)x[j], b + (size_t)j * (N_r + 1), N_r, &lbj, &ubj);
        sl += lbj * lbj;
        su += ubj * ubj;
    }
    *lb2 = sl;
    *ub2 = su;
}

/* ======================================================================== */
/* Index                                                                      */
/* ======================================================================== */
struct orc_index {
    const float* X;        /* global rows */
    int64_t n_global, row_lo, n;
    int d, L, K, N_r, LK, max_size;
    uint64_t seed;
    double eps;
    float* A;
    int64_t n_s;
    int64_t* sample;
    float* B;              /* [LK][N_r+1] */
    float* P;              /* [n][LK] */
    uint8_t* codes;        /* [n][LK] */
    orc_tree** trees;
};

orc_index* orc_build(const float* X, int64_t n_global, int d, int64_t row_lo, int64_t row_hi,
                     int L, int K, int N_r, uint64_t seed, int max_size, double sample_frac,
                     int builder) {
    orc_index* ix = (orc_index*)xcalloc(1, sizeof(orc_index));
    ix->X = X; ix->n_global = n_global; ix->row_lo = row_lo; ix->n = row_hi - row_lo;
    ix->d = d; ix->L = L; ix->K = K; ix->N_r = N_r; ix->LK = L * K; ix->max_size = max_size;
    ix->seed = seed;
    orc_params(K, L, 1.5, NULL, &ix->eps, NULL, NULL);   /* eps depends on (K, L) only */
    int LK = ix->LK;
    /* hash family (Eq. 1) */
    ix->A = (float*)xmalloc(sizeof(float) * (size_t)LK * d);
    orc_hash_family(seed, d, L, K, ix->A);
    /* sample of the whole dataset and its projections */
    ix->n_s = orc_sample_size(n_global, N_r, sample_frac);
    ix->sample = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)ix->n_s);
    orc_sample_ids(seed, n_global, ix->n_s, ix->sample);
    float* Xs = (float*)xmalloc(sizeof(float) * (size_t)ix->n_s * d);
    for (int64_t s = 0; s < ix->n_s; ++s)
        memcpy(Xs + (size_t)s * d, X + (size_t)ix->sample[s] * d, sizeof(float) * (size_t)d);
    float* Ps = (float*)xmalloc(sizeof(float) * (size_t)ix->n_s * LK);
    orc_project(ix->A, LK, d, Xs, ix->n_s, Ps);
    free(Xs);
    /* breakpoints per (i,j) */
    ix->B = (float*)xmalloc(sizeof(float) * (size_t)LK * (N_r + 1));
    float* col = (float*)xmalloc(sizeof(float) * (size_t)ix->n_s);
    for (int r = 0; r < LK; ++r) {
        for (int64_t s = 0; s < ix->n_s; ++s) col[s] = Ps[(size_t)s * LK + r];
        orc_breakpoints_sort(col, ix->n_s, N_r, ix->B + (size_t)r * (N_r + 1));
    }
    free(col);
    free(Ps);
    /* projection of this shard's rows and encoding (Alg. 1) */
    ix->P = (float*)xmalloc(sizeof(float) * (size_t)ix->n * LK);
    orc_project(ix->A, LK, d, X + (size_t)row_lo * d, ix->n, ix->P);
    ix->codes = (uint8_t*)xmalloc((size_t)ix->n * LK);
    for (int64_t p = 0; p < ix->n; ++p)
        for (int r = 0; r < LK; ++r)
            ix->codes[(size_t)p * LK + r] =
                (uint8_t)orc_encode_value(ix->P[(size_t)p * LK + r], ix->B + (size_t)r * (N_r + 1), N_r);
    /* L DE-Trees (Alg. 2) over local ids 0..n-1 = global row_lo.. */
    ix->trees = (orc_tree**)xcalloc((size_t)L, sizeof(orc_tree*));
    for (int i = 0; i < L; ++i)
        ix->trees[i] = orc_tree_build(ix->codes + (size_t)i * K, ix->n, LK, K, N_r, max_size, builder);
    return ix;
}
void orc_index_free(orc_index* ix) {
    if (!ix) return;
    for (int i = 0; i < ix->L; ++i) orc_tree_free(ix->trees[i]);
    free(ix->trees); free(ix->A); free(ix->sample); free(ix->B); free(ix->P); free(ix->codes);
    free(ix);
}
int64_t orc_index_n(const orc_index* ix) { return ix->n; }
int64_t orc_index_n_sample(const orc_index* ix) { return ix->n_s; }
const float* orc_index_A(const orc_index* ix) { return ix->A; }
const float* orc_index_breakpoints(const orc_index* ix) { return ix->B; }
const float* orc_index_P(const orc_index* ix) { return ix->P; }
const uint8_t* orc_index_codes(const orc_index* ix) { return ix->codes; }
const int64_t* orc_index_sample(const orc_index* ix) { return ix->sample; }
const orc_tree* orc_index_tree(const orc_index* ix, int i) { return ix->trees[i]; }
double orc_index_eps(const orc_index* ix) { return ix->eps; }

/* ======================================================================== */
/* O7. DET Range Query, Alg. 3 with the traversal of P:446-452:   */
/* prune a node whose LB > r'; take a whole leaf whose UB <= r'; otherwise    */
/* examine its points (AMB-12: CELL = the point's own region lower bound,     */
/* EXACT = its true projected distance; RELAXED = §6.2.2(1), whole leaf when  */
/* LB <= r').  All comparisons are "<=" on squares (AMB-13).                 */
/* ======================================================================== */
typedef struct {
    const orc_index* ix;
    const orc_tree* t;
    int i;
    const float* qp;
    double rho2;
    int mode;
    int64_t* out;
    int64_t cnt;
} rq_state;

static double point_lb2(const orc_index* ix, int i, const float* qp, int64_t id) {
    double s = 0.0;
    for (int j = 0; j < ix->K; ++j) {
        int c = ix->codes[(size_t)id * ix->LK + (size_t)i * ix->K + j];
        double lbj, ubj;
        dim_bounds(c, c, (double)qp[j], ix->B + (size_t)(i * ix->K + j) * (ix->N_r + 1), ix->N_r, &lbj, &ubj);
        s += lbj * lbj;
    }
    return s;
}
static double point_true2(const orc_index* ix, int i, const float* qp, int64_t id) {
    double s = 0.0;
    for (int j = 0; j < ix->K; ++j) {
        double df = (double)qp[j] - (double)ix->P[(size_t)id * ix->LK + (size_t)i * ix->K + j];
        s += df * df;
    }
    return s;
}
static void rq_node(rq_state* st, int32_t ni) {
    const orc_tree* t = st->t;
    const onode* nd = &t->nodes[ni];
    uint8_t lo[ORC_MAXK], hi[ORC_MAXK];
    leaf_box(t, nd, lo, hi);
    double lb2, ub2;
    orc_box_bounds2(lo, hi, st->qp, st->ix->B + (size_t)st->i * st->ix->K * (st->ix->N_r + 1), t->K,
                    t->N_r, &lb2, &ub2);
    if (lb2 > st->rho2) return;                                /* prune */
    if (nd->child[0] >= 0) {                                   /* expand */
        rq_node(st, nd->child[0]);
        rq_node(st, nd->child[1]);
        return;
    }
    if (st->mode == ORC_RELAXED || ub2 <= st->rho2) {          /* whole leaf */
        for (int64_t e = 0; e < nd->size; ++e) st->out[st->cnt++] = nd->ids[e];
        return;
    }
    for (int64_t e = 0; e < nd->size; ++e) {                   /* examine points */
        int64_t id = nd->ids[e];
        double v = st->mode == ORC_EXACT ? point_true2(st->ix, st->i, st->qp, id)
                                         : point_lb2(st->ix, st->i, st->qp, id);
        if (v <= st->rho2) st->out[st->cnt++] = id;
    }
}
/* ---- §6.2.2(2): the qualifying leaves of one tree with their lower bounds, so Alg. 5   */
/* can take them in ascending (LB, leaf) order and stop at the budget.  "leaf" = the leaf's      */
/* position in the tree's canonical order (DFS, 0-child first, first-layer keys ascending; empty */
/* leaves dropped), i.e. the exported leaf order.                                                 */
typedef struct { double lb2, ub2; int64_t ord; int32_t node; } lbleaf;
static int cmp_lbleaf(const void* a, const void* b) {
    const lbleaf* x = (const lbleaf*)a; const lbleaf* y = (const lbleaf*)b;
    if (x->lb2 != y->lb2) return x->lb2 < y->lb2 ? -1 : 1;
    return (x->ord > y->ord) - (x->ord < y->ord);
}
static void ord_node(const orc_tree* t, int32_t ni, int64_t* cnt, int64_t* ord) {
    const onode* nd = &t->nodes[ni];
    if (nd->child[0] >= 0) { ord_node(t, nd->child[0], cnt, ord); ord_node(t, nd->child[1], cnt, ord); return; }
    ord[ni] = nd->size > 0 ? (*cnt)++ : -1;
}
typedef struct { lbleaf* v; int64_t n, cap; const int64_t* ord; } lbset;
static void lq_node(rq_state* st, lbset* out, int32_t ni) {
    const orc_tree* t = st->t;
    const onode* nd = &t->nodes[ni];
    uint8_t lo[ORC_MAXK], hi[ORC_MAXK];
    leaf_box(t, nd, lo, hi);
    double lb2, ub2;
    orc_box_bounds2(lo, hi, st->qp, st->ix->B + (size_t)st->i * st->ix->K * (st->ix->N_r + 1), t->K,
                    t->N_r, &lb2, &ub2);
    if (lb2 > st->rho2) return;                                /* prune */
    if (nd->child[0] >= 0) { lq_node(st, out, nd->child[0]); lq_node(st, out, nd->child[1]); return; }
    if (nd->size == 0) return;
    if (out->n == out->cap) {
        out->cap = out->cap ? 2 * out->cap : 1024;
        out->v = (lbleaf*)realloc(out->v, sizeof(lbleaf) * (size_t)out->cap);
        if (!out->v) { fprintf(stderr, "oracle: out of memory\n"); abort(); }
    }
    lbleaf e = {lb2, ub2, out->ord[ni], ni};
    out->v[out->n++] = e;
}
/* the points one qualifying leaf contributes (same rules as rq_node's leaf case) */
static int64_t leaf_points(rq_state* st, const onode* nd, double ub2, int64_t* out) {
    int64_t cnt = 0;
    if (st->mode == ORC_RELAXED || ub2 <= st->rho2) {
        for (int64_t e = 0; e < nd->size; ++e) out[cnt++] = nd->ids[e];
        return cnt;
    }
    for (int64_t e = 0; e < nd->size; ++e) {
        int64_t id = nd->ids[e];
        double v = st->mode == ORC_EXACT ? point_true2(st->ix, st->i, st->qp, id) : point_lb2(st->ix, st->i, st->qp, id);
        if (v <= st->rho2) out[cnt++] = id;
    }
    return cnt;
}

int64_t orc_range_query(const orc_index* ix, int i, const float* qp, double rho, int mode,
                        int64_t* out) {
    rq_state st = {ix, ix->trees[i], i, qp, rho * rho, mode, out, 0};
    for (int64_t f = 0; f < st.t->nfirst; ++f) rq_node(&st, st.t->first[f]);
    qsort(out, (size_t)st.cnt, sizeof(int64_t), cmp_i64);
    return st.cnt;
}

/* ======================================================================== */
/* O8. c^2-k-ANN, Alg. 5.                                        */
/* ======================================================================== */
void orc_project_query(const orc_index* ix, const float* q, float* qp) {
    orc_project(ix->A, ix->LK, ix->d, q, 1, qp);
}
typedef struct { double d2; int64_t id; } candd;
static int cmp_candd(const void* a, const void* b) {
    const candd* x = (const candd*)a; const candd* y = (const candd*)b;
    if (x->d2 != y->d2) return x->d2 < y->d2 ? -1 : 1;
    return (x->id > y->id) - (x->id < y->id);
}
static double dist2(const float* a, const float* b, int d) {
    double s = 0.0;
    for (int t = 0; t < d; ++t) { double df = (double)a[t] - (double)b[t]; s += df * df; }
    return s;
}
void orc_query(const orc_index* ix, const float* Q, int64_t nq, int k, double c, double r_min,
               double beta, int mode, int64_t* out_ids, float* out_dists, orc_qstats* stats) {
    orc_query_ex(ix, Q, nq, k, c, r_min, beta, mode, 0, out_ids, out_dists, stats);
}
void orc_query_ex(const orc_index* ix, const float* Q, int64_t nq, int k, double c, double r_min,
                  double beta, int mode, int lb_order, int64_t* out_ids, float* out_dists, orc_qstats* stats) {
    int64_t** ords = (int64_t**)xmalloc(sizeof(int64_t*) * (size_t)ix->L);
    for (int i = 0; i < ix->L; ++i) {
        const orc_tree* t = ix->trees[i];
        int64_t cnt = 0;
        ords[i] = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)(t->nnodes ? t->nnodes : 1));
        for (int64_t f = 0; f < t->nfirst; ++f) ord_node(t, t->first[f], &cnt, ords[i]);
    }
    lbset ls = {NULL, 0, 0, NULL};
    int64_t n = ix->n;
    int64_t budget = (int64_t)ceil(beta * (double)n) + k;     /* beta n + k (AMB-17) */
    uint8_t* inS = (uint8_t*)xmalloc((size_t)n);
    int64_t* S = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)n);
    double* d2 = (double*)xmalloc(sizeof(double) * (size_t)n);
    int64_t* buf = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)n);
    float* qp = (float*)xmalloc(sizeof(float) * (size_t)ix->LK);
    for (int64_t qi = 0; qi < nq; ++qi) {
        const float* q = Q + (size_t)qi * ix->d;
        memset(inS, 0, (size_t)n);
        int64_t nS = 0, nver = 0;
        double r = r_min;                                      /* line 1 */
        int rounds = 0, trees_last = 0, reason = 2;
        orc_project_query(ix, q, qp);                          /* line 4: q'_i = H_i(q) */
        for (;;) {                                             /* line 2: while TRUE */
            ++rounds;
            int stop = 0;
            for (int i = 0; i < ix->L; ++i) {                  /* line 3 */
                trees_last = i + 1;
                if (!lb_order) {
                    int64_t cnt = orc_range_query(ix, i, qp + (size_t)i * ix->K, ix->eps * r, mode, buf); /* line 5 */
                    for (int64_t e = 0; e < cnt; ++e)          /* line 6: S <- S u S_i */
                        if (!inS[buf[e]]) { inS[buf[e]] = 1; S[nS++] = buf[e]; }
                    if (nS >= budget) { reason = 0; stop = 1; break; }   /* line 7 */
                } else {
                    /* §6.2.2(2): the tree's qualifying leaves in ascending (LB, leaf) order, the budget
                       checked after each leaf (line 7 at leaf granularity) */
                    rq_state rs = {ix, ix->trees[i], i, qp + (size_t)i * ix->K, (ix->eps * r) * (ix->eps * r), mode, buf, 0};
                    ls.n = 0;
                    ls.ord = ords[i];
                    for (int64_t f = 0; f < rs.t->nfirst; ++f) lq_node(&rs, &ls, rs.t->first[f]);
                    qsort(ls.v, (size_t)ls.n, sizeof(lbleaf), cmp_lbleaf);
                    for (int64_t e = 0; e < ls.n && !stop; ++e) {
                        int64_t cnt = leaf_points(&rs, &rs.t->nodes[ls.v[e].node], ls.v[e].ub2, buf);
                        for (int64_t u = 0; u < cnt; ++u)
                            if (!inS[buf[u]]) { inS[buf[u]] = 1; S[nS++] = buf[u]; }
                        if (nS >= budget) { reason = 0; stop = 1; }
                    }
                    if (stop) break;
                }
            }
            if (stop) break;
            for (; nver < nS; ++nver)                          /* distances of new candidates */
                d2[nver] = dist2(q, ix->X + (size_t)(ix->row_lo + S[nver]) * ix->d, ix->d);
            double cr = c * r;
            int64_t within = 0;
            for (int64_t e = 0; e < nS; ++e) within += d2[e] <= cr * cr;
            if (within >= k) { reason = 1; break; }            /* line 9 */
            if (rounds == 64) { reason = 2; break; }           /* AMB-20 cap */
            r = c * r;                                         /* line 11 */
        }
        for (; nver < nS; ++nver)
            d2[nver] = dist2(q, ix->X + (size_t)(ix->row_lo + S[nver]) * ix->d, ix->d);
        candd* cd = (candd*)xmalloc(sizeof(candd) * (size_t)(nS ? nS : 1));
        for (int64_t e = 0; e < nS; ++e) { cd[e].d2 = d2[e]; cd[e].id = S[e]; }
        qsort(cd, (size_t)nS, sizeof(candd), cmp_candd);       /* top-k by (dist, id), AMB-21 */
        for (int e = 0; e < k; ++e) {
            if (e < nS) {
                out_ids[qi * k + e] = cd[e].id + ix->row_lo;
                out_dists[qi * k + e] = (float)sqrt(cd[e].d2);
            } else {
                out_ids[qi * k + e] = -1;
                out_dists[qi * k + e] = INFINITY;
            }
        }
        free(cd);
        if (stats) {
            stats[qi].rounds = rounds; stats[qi].trees_last = trees_last; stats[qi].reason = reason;
            stats[qi].pad = 0; stats[qi].n_cand = nS; stats[qi].r_final = r;
        }
    }
    free(inS); free(S); free(d2); free(buf); free(qp);
    for (int i = 0; i < ix->L; ++i) free(ords[i]);
    free(ords);
    free(ls.v);
}

/* ======================================================================== */
/* O8b. (r,c)-ANN, Alg. 4: one pass over the L trees at radius    */
/* eps r; return the point of S closest to q (ties by id) as soon as          */
/* |S| >= beta n + 1 (line 6; ceil(beta n) + 1 in double, as AMB-17), else    */
/* after the L trees the closest point if it lies within c r (lines 8-9),     */
/* else nothing (line 10): (-1, +inf).                                        */
/* ======================================================================== */
void orc_rc_ann(const orc_index* ix, const float* Q, int64_t nq, double c, double r, double beta, int mode,
                int64_t* out_ids, float* out_dists) {
    int64_t n = ix->n;
    int64_t budget = (int64_t)ceil(beta * (double)n) + 1;
    uint8_t* inS = (uint8_t*)xmalloc((size_t)n);
    int64_t* S = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)n);
    int64_t* buf = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)n);
    float* qp = (float*)xmalloc(sizeof(float) * (size_t)ix->LK);
    for (int64_t qi = 0; qi < nq; ++qi) {
        const float* q = Q + (size_t)qi * ix->d;
        memset(inS, 0, (size_t)n);
        int64_t nS = 0;                                        /* line 1 */
        int by_budget = 0;
        orc_project_query(ix, q, qp);                          /* line 3 (all i at once) */
        for (int i = 0; i < ix->L; ++i) {                      /* line 2 */
            int64_t cnt = orc_range_query(ix, i, qp + (size_t)i * ix->K, ix->eps * r, mode, buf); /* line 4 */
            for (int64_t e = 0; e < cnt; ++e)                  /* line 5 */
                if (!inS[buf[e]]) { inS[buf[e]] = 1; S[nS++] = buf[e]; }
            if (nS >= budget) { by_budget = 1; break; }        /* line 6 */
        }
        candd best = {INFINITY, -1};
        for (int64_t e = 0; e < nS; ++e) {                     /* the point of S closest to q */
            candd x = {dist2(q, ix->X + (size_t)(ix->row_lo + S[e]) * ix->d, ix->d), S[e]};
            if (best.id < 0 || cmp_candd(&x, &best) < 0) best = x;
        }
        if (best.id >= 0 && (by_budget || best.d2 <= (c * r) * (c * r))) {   /* lines 7, 8-9 */
            out_ids[qi] = best.id + ix->row_lo;
            out_dists[qi] = (float)sqrt(best.d2);
        } else {                                               /* line 10 */
            out_ids[qi] = -1;
            out_dists[qi] = INFINITY;
        }
    }
    free(inS); free(S); free(buf); free(qp);
}

/* ======================================================================== */
/* O9. Merge of per-shard top-k lists by (dist, id).                          */
/* ======================================================================== */
typedef struct { float d; int64_t id; } candf;
static int cmp_candf(const void* a, const void* b) {
    const candf* x = (const candf*)a; const candf* y = (const candf*)b;
    if (x->d != y->d) return x->d < y->d ? -1 : 1;
    return (x->id > y->id) - (x->id < y->id);
}
void orc_merge_topk(const int64_t* ids, const float* dists, int G, int64_t nq, int k,
                    int64_t* out_ids, float* out_dists) {
    candf* v = (candf*)xmalloc(sizeof(candf) * (size_t)G * k);
    for (int64_t q = 0; q < nq; ++q) {
        int m = 0;
        for (int g = 0; g < G; ++g)
            for (int e = 0; e < k; ++e) {
                size_t o = ((size_t)g * nq + q) * k + e;
                if (ids[o] >= 0) { v[m].d = dists[o]; v[m].id = ids[o]; ++m; }
            }
        qsort(v, (size_t)m, sizeof(candf), cmp_candf);
        for (int e = 0; e < k; ++e) {
            out_ids[q * k + e] = e < m ? v[e].id : -1;
            out_dists[q * k + e] = e < m ? v[e].d : INFINITY;
        }
    }
    free(v);
}

/* ======================================================================== */
/* O10. Exact kNN by brute force (double, ties by id): the R* of recall       */
/* (P:812).  A max-heap of the k best (d2, id).                               */
/* ======================================================================== */
static int cand_less(const candd* a, const candd* b) {
    return a->d2 < b->d2 || (a->d2 == b->d2 && a->id < b->id);
}
static void heap_sift_down(candd* h, int m, int i) {
    for (;;) {
        int l = 2 * i + 1, r = l + 1, g = i;
        if (l < m && cand_less(&h[g], &h[l])) g = l;
        if (r < m && cand_less(&h[g], &h[r])) g = r;
        if (g == i) return;
        candd t = h[i]; h[i] = h[g]; h[g] = t; i = g;
    }
}
static void heap_sift_up(candd* h, int i) {
    while (i > 0) {
        int p = (i - 1) / 2;
        if (!cand_less(&h[p], &h[i])) return;
        candd t = h[i]; h[i] = h[p]; h[p] = t; i = p;
    }
}
void orc_exact_knn(const float* X, int64_t n, int d, const float* Q, int64_t nq, int k,
                   int64_t* out_ids, double* out_dists) {
    candd* h = (candd*)xmalloc(sizeof(candd) * (size_t)k);
    for (int64_t q = 0; q < nq; ++q) {
        int m = 0;
        for (int64_t p = 0; p < n; ++p) {
            candd c = {dist2(Q + (size_t)q * d, X + (size_t)p * d, d), p};
            if (m < k) { h[m] = c; heap_sift_up(h, m); ++m; }
            else if (cand_less(&c, &h[0])) { h[0] = c; heap_sift_down(h, m, 0); }
        }
        qsort(h, (size_t)m, sizeof(candd), cmp_candd);
        for (int e = 0; e < k; ++e) {
            out_ids[q * k + e] = e < m ? h[e].id : -1;
            out_dists[q * k + e] = e < m ? sqrt(h[e].d2) : INFINITY;
        }
    }
    free(h);
}

/* ======================================================================== */
/* r_min (AMB-22).  A point enters a full round's S at radius r    */
/* iff min_i cellLB_i <= eps r, so the smallest r with |S| >= B is            */
/* r*_q = t_(B)/eps, t_(B) the B-th smallest min_i cellLB_i: it meets both of */
/* P:719-720's conditions for query q.  One value for all queries: the lower  */
/* median of r*_q over a sample.                                              */
/* ======================================================================== */
static double nth_smallest(double* a, int64_t m, int64_t q) {
    int64_t lo = 0, hi = m - 1;
    while (lo < hi) {
        double pv = a[lo + (hi - lo) / 2];
        int64_t lt = lo, i = lo, gt = hi;
        while (i <= gt) {
            if (a[i] < pv) { double t = a[lt]; a[lt] = a[i]; a[i] = t; ++lt; ++i; }
            else if (a[i] > pv) { double t = a[gt]; a[gt] = a[i]; a[i] = t; --gt; }
            else ++i;
        }
        if (q < lt) hi = lt - 1; else if (q > gt) lo = gt + 1; else return a[q];
    }
    return a[q];
}
static int cmp_f64(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}
double orc_estimate_rmin(const orc_index* ix, const float* Qs, int64_t ns, int k, double c,
                         double beta, double* rstar_out) {
    int64_t n = ix->n;
    int64_t budget = (int64_t)ceil(beta * (double)n) + k;
    if (budget > n) budget = n;
    double* t = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* rq = (double*)xmalloc(sizeof(double) * (size_t)ns);
    float* qp = (float*)xmalloc(sizeof(float) * (size_t)ix->LK);
    for (int64_t s = 0; s < ns; ++s) {
        orc_project_query(ix, Qs + (size_t)s * ix->d, qp);
        for (int64_t p = 0; p < n; ++p) {
            double best = INFINITY;
            for (int i = 0; i < ix->L; ++i) {
                double v = point_lb2(ix, i, qp + (size_t)i * ix->K, p);
                if (v < best) best = v;
            }
            t[p] = best;
        }
        rq[s] = sqrt(nth_smallest(t, n, budget - 1)) / ix->eps;   /* r*_q */
        if (rstar_out) rstar_out[s] = rq[s];
    }
    qsort(rq, (size_t)ns, sizeof(double), cmp_f64);
    double med = rq[(ns - 1) / 2];
    free(t); free(rq); free(qp);
    return med;
}
