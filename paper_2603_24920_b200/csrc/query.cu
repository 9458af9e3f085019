// query.cu -- batched c^2-k-ANN (Alg. 5) on sm_100a.
//
// Per round r = r_min c^m (host loop; one D2H of the active count per round):
//  k_build_lut    once per query batch: per (query, tree, dim) the 256-entry table of squared
//                 region distances (Fig. dist; AMB-7) and the query's symbol.
//  k_range_filter per tree t (trees in order, Alg. 5 lines 3-8): CTAs = groups of 4 queries x
//                 stripes of tiles; warps test leaf boxes (leaf LB = sum_j D_j[clamp(s_x,
//                 lo_j, hi_j)]) then the points of qualifying leaves (cell LB = sum_j
//                 D_j[code_j], AMB-12), OR them into the query's bitmap (de-duplicated union
//                 S <- S u S_i, line 6) and append first-time ids.
//  k_tree_end     after tree t: budget test |S| >= ceil(beta n)+k (line 7, AMB-15/17).
//  k_verify       exact squared L2 of the new candidates: one warp per row, float4 gathers,
//                 warp-shuffle reduction (lines 8/10).
//  k_topk         per query: radix-select the k smallest (d2, id) keys of old top-k u new,
//                 bitonic sort; then the radius test k-th d2 <= (c r)^2 (line 9, AMB-18).
//  k_finalize     ids (global) and sqrt(d2), ascending by (dist, id) (AMB-21, AMB-28).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <cmath>
#include <cstring>
#include <vector>

#include "index.cuh"

namespace detlsh {

void project_rows(const Index& ix, const float* d_X, int64_t ld, int64_t m, float* d_P, int proj_impl,
                  int* d_nonfinite, cudaStream_t st);
bool verify_tc(const float* d_X, int64_t n, int ld, const float* d_Qa, const float* d_Qalo, const float* d_qn, int na,
               const uint32_t* d_NB, const uint32_t* d_BO, int64_t nw4, const float* d_xn, uint32_t* d_cand,
               float* d_d2, cudaStream_t st);

namespace {

enum : int { ST_ACTIVE = 0, ST_BUDGET = 1, ST_RADIUS = 2, ST_CAP = 3 };

struct QState {  // per query of a batch
    int64_t cnt;        // |S| (bits set in the query's bitmap)
    int64_t nver;       // members of S verified and merged into the top-k
    int64_t roff;       // this round's slot range [roff, roff + rcnt) in the round buffer
    int64_t rcnt;
    int32_t status;     // ST_*
    int32_t tk;         // entries in the top-k list
    int32_t trees_last;
    int32_t rounds;
    int32_t overflow;
    int32_t doc;        // count the bitmap this tree (k_count_decide)
    int64_t tnew;       // lb_order: first-time members of the current tree (counted, not yet committed)
    int64_t pub;        // marks since |S| was last counted: |S| <= cnt + pub
};


// ---- per-batch LUTs: D[q][t][j][s] = max(0, l_s - x, x - u_s)^2 for cell s = (b_s, b_{s+1}],
//      l_0 = -inf, u_{N_r-1} = +inf (Fig. dist; AMB-7), and the query's own symbol
//      s_x (AMB-6).  The LUT depends only on the projected query, not on the radius.
__global__ void k_build_lut(const float* __restrict__ Qp, int nqb, int LK, int N_r, const float* __restrict__ B,
                            float* __restrict__ lut, uint8_t* __restrict__ sx) {
    pdl_wait();
    const int64_t total = (int64_t)nqb * LK * N_r;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int s = (int)(i % N_r);
        const int64_t qr = i / N_r;                 // q * LK + r
        const int r = (int)(qr % LK);
        const float* b = B + (int64_t)r * (N_r + 1);
        const float x = Qp[qr];
        const float l = s >= 1 ? b[s] : -INFINITY;
        const float u = s <= N_r - 2 ? b[s + 1] : INFINITY;
        const float v = fmaxf(0.f, fmaxf(l - x, x - u));
        lut[i] = v * v;
        if (s == 0) {
            int pos = 0;
            for (int st = N_r >> 1; st > 0; st >>= 1) {
                const int idx = pos + st;
                pos += (idx <= N_r - 1 && b[idx] < x) ? st : 0;
            }
            sx[qr] = (uint8_t)pos;
        }
    }
}

// ---- per round: quantised lower bounds of the LUT, e = min(cap, floor(D * QT/rho^2)) with
//      products rounded down: sum_j e_j > QT proves sum_j D_j > rho^2, and sum_j e_j <= QT-17
//      proves sum_j D_j < rho^2 (1 - 1e-5) (each e_j > D_j QT/rho^2 - 1.001), so only the band
//      in between needs the exact fp32 sum.  16 terms of <= cap fit the packed lane width.
__device__ inline uint16_t quant_term(float d, float inv_rd, float cap) {
    float v = __fmul_rd(d, inv_rd);
    if (v != v) v = 0.f;                           // 0 * inf: a zero term stays zero
    return (uint16_t)(v >= cap ? cap : floorf(v));
}

// Batch tables in one pass (block = one (query, coordinate) row of N_r entries, thread = region):
// the exact table D (as k_build_lut), the query's region code (the count of interior breakpoints
// below it = k_build_lut's lower bound), and -- for the first round, where every query of the
// batch is active -- both quantised tables of that round (as k_build_qlut).
__global__ void k_build_tables(const float* __restrict__ Qp, int LK, int N_r, const float* __restrict__ B,
                               float* __restrict__ lut, uint8_t* __restrict__ sx,
                               float inv_a, float cap_a, uint16_t* __restrict__ qa,
                               float inv_b, float cap_b, uint16_t* __restrict__ qb_) {
    pdl_wait();
    const int r = blockIdx.x, q = blockIdx.y, s = threadIdx.x;
    const int64_t qr = (int64_t)q * LK + r;
    const float* b = B + (int64_t)r * (N_r + 1);
    const float x = Qp[qr];
    const float l = s >= 1 ? b[s] : -INFINITY;
    const float u = s <= N_r - 2 ? b[s + 1] : INFINITY;
    const float v = fmaxf(0.f, fmaxf(l - x, x - u));
    const float d = v * v;
    const int64_t i = qr * N_r + s;
    lut[i] = d;
    if (qa) qa[i] = quant_term(d, inv_a, cap_a);
    if (qb_) qb_[i] = quant_term(d, inv_b, cap_b);
    const int below = __syncthreads_count(s >= 1 && b[s] < x);
    if (s == 0) sx[qr] = (uint8_t)below;
}

// N_r = 256: the same tables with a warp per (query, coordinate) row, 8 consecutive regions per
// lane (16-byte / 8-byte stores), the region code from the lanes' counts; 8 rows per block.
__global__ void __launch_bounds__(256) k_build_tables256(const float* __restrict__ Qp, int64_t nrows, const float* __restrict__ B,
                                                         int LK, float* __restrict__ lut, uint8_t* __restrict__ sx,
                                                         float inv_a, float cap_a, uint16_t* __restrict__ qa,
                                                         float inv_b, float cap_b, uint16_t* __restrict__ qb_) {
    pdl_wait();
    constexpr int N_r = 256;
    const int lane = threadIdx.x & 31;
    const int64_t qr = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);   // q * LK + r
    if (qr >= nrows) return;
    const int r = (int)(qr % LK);
    const float* b = B + (int64_t)r * (N_r + 1);
    const float x = Qp[qr];
    float d[8];
    int below = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int s_ = lane * 8 + k;
        const float l = s_ >= 1 ? b[s_] : -INFINITY;
        const float u = s_ <= N_r - 2 ? b[s_ + 1] : INFINITY;
        const float v = fmaxf(0.f, fmaxf(l - x, x - u));
        d[k] = v * v;
        below += (s_ >= 1 && b[s_] < x) ? 1 : 0;
    }
    const int64_t i = qr * N_r + lane * 8;
    float4* lo = reinterpret_cast<float4*>(lut + i);
    lo[0] = make_float4(d[0], d[1], d[2], d[3]);
    lo[1] = make_float4(d[4], d[5], d[6], d[7]);
    uint32_t pa[4], pb[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        pa[k] = (uint32_t)quant_term(d[2 * k], inv_a, cap_a) | ((uint32_t)quant_term(d[2 * k + 1], inv_a, cap_a) << 16);
        pb[k] = (uint32_t)quant_term(d[2 * k], inv_b, cap_b) | ((uint32_t)quant_term(d[2 * k + 1], inv_b, cap_b) << 16);
    }
    if (qa) *reinterpret_cast<uint4*>(qa + i) = make_uint4(pa[0], pa[1], pa[2], pa[3]);
    if (qb_) *reinterpret_cast<uint4*>(qb_ + i) = make_uint4(pb[0], pb[1], pb[2], pb[3]);
    for (int o = 16; o > 0; o >>= 1) below += __shfl_xor_sync(0xffffffffu, below, o);
    if (lane == 0) sx[qr] = (uint8_t)below;
}

// later rounds: block = one active query's (coordinate, region) rows
__global__ void k_build_qlut(const float* __restrict__ lut, const int* __restrict__ act, int64_t per_q,
                             float inv_rd, float cap, uint16_t* __restrict__ qlut) {
    pdl_wait();
    const int64_t q = act[blockIdx.y];
    const float* src = lut + q * per_q;
    uint16_t* dst = qlut + q * per_q;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < per_q; e += (int64_t)gridDim.x * blockDim.x)
        dst[e] = quant_term(src[e], inv_rd, cap);
}

// ---- per tree: each 16-query group's quantised table interleaved once (entry (j, s) = the
//      group's 16 8-bit terms), copied by the group's filter CTAs instead of each CTA gathering
//      16 queries' tables itself.  Inactive slots get the cap (never pass).
__global__ void __launch_bounds__(256) k_group_table(const int* __restrict__ act, int na_ub, const int* __restrict__ dna,
                                                     const QState* __restrict__ qs, const uint16_t* __restrict__ qlut,
                                                     int64_t per_q, int t, int KN, uint32_t cap,
                                                     const uint8_t* __restrict__ sx, int L, int K, int N_r,
                                                     uint4* __restrict__ gtab, unsigned int* __restrict__ tctr) {
    pdl_wait();
    // block = (16-query group, dim j); thread = region code c (coalesced table reads per query)
    __shared__ int s_qq[16], s_sv[16];
    const int na = dna ? *dna : na_ub;       // device count (the list is compacted on the device)
    const int64_t grp = blockIdx.x;
    const int j = blockIdx.y;
    if (grp * 16 >= na) return;
    if (tctr && j == 0 && threadIdx.x == 0) tctr[grp] = 0;   // the filter's tile counter of the group
    if (threadIdx.x < 16) {
        const int64_t gi = grp * 16 + threadIdx.x;
        int q = -1;
        if (gi < na) {
            q = act[gi];
            if (qs[q].status != ST_ACTIVE) q = -1;
        }
        s_qq[threadIdx.x] = q;
        s_sv[threadIdx.x] = q >= 0 ? (int)sx[((int64_t)q * L + t) * K + j] : 0;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < N_r; c += blockDim.x) {
        const int64_t e = (int64_t)j * N_r + c;
        uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
        for (int g = 0; g < 16; ++g) {
            const int q = s_qq[g];
            uint32_t v = cap;
            if (q >= 0) {
                v = qlut[(int64_t)q * per_q + (int64_t)t * KN + e];
                if (s_sv[g] < c) v |= 0x80u;     // region flag (k_range_filter)
            }
            w[g >> 2] |= v << (8 * (g & 3));
        }
        gtab[grp * KN + e] = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// ---- range filter of one tree (Alg. 3 at radius eps*r, Alg. 5 lines 5-6), batched:
//      CTA = group of G active queries x stripe of tiles; a warp owns a tile of <= 32 leaves.
//      Leaf lower bounds (lane = leaf) prune; for the points of qualifying leaves the cell
//      lower bound is screened with the quantised table (one 16-byte shared load per code
//      serves all G queries: G = 8 x 12-bit terms in 16-bit lanes, or G = 16 x 8-bit terms
//      widened into 16-bit lanes) and decided in fp32 from the exact table inside the band;
//      passing points are OR-marked into the per-query bitmap (RED.OR).  The fp32 decision
//      sums the same terms in the same order as the cell bound's definition (AMB-12), so the
//      screen never changes a result.
constexpr int RF_THREADS = 256;
constexpr int RF_CTAS = 3;       // resident CTAs per SM
constexpr int RF_G = 16;         // queries per CTA (8-bit terms); 8 selects 12-bit terms
constexpr int RF_BQ = 64;        // band queue per warp: < 32 left over + one step of <= 32

// Byte-wise sign replicate: 0xFF in each byte whose bit 7 is set, else 0x00 (prmt selector
// nibbles 8..B: byte 0..3 with its msb replicated).
__device__ __forceinline__ uint32_t prmt_sign(uint32_t x) {
    uint32_t r;
    asm("prmt.b32 %0, %1, 0, 0xBA98;" : "=r"(r) : "r"(x));
    return r;
}

// Mark id in query row (bm, sm) of the union S: the bit in the bitmap and the bit of its word in
// the row's dirty-word summary (one bit per 32-bit bitmap word), so the per-round scans of S
// (k_count_new, the sparse candidate listing) visit only the words that hold members.
__device__ __forceinline__ void mark_member(uint32_t* bm, uint32_t* sm, uint32_t id) {
    atomicOr(bm + (id >> 5), 1u << (id & 31));              // RED.OR
    atomicOr(sm + (id >> 10), 1u << ((id >> 5) & 31));
}

// Box bound of one query in the 12-bit table (K = 16, N_r = 256): sum_j e_j[clamp(q_j, lo_j, hi_j)]
// with the clamps done two dims per instruction -- each code word's even and odd bytes spread
// into 16-bit lanes (one byte permute each), VIMNMX.U16x2 against the query's codes spread the same
// way (qe[i] / qo[i]: bytes 0, 2 / 1, 3 of word i), and the lanes' byte offsets into the table
// (2c) taken from the doubled word.  Same terms as the byte-wise min/max form, same sum.
__device__ __forceinline__ uint32_t spread_even(uint32_t w) { return __byte_perm(w, 0u, 0x4240); }
__device__ __forceinline__ uint32_t spread_odd(uint32_t w) { return __byte_perm(w, 0u, 0x4341); }
__device__ __forceinline__ uint32_t clamp_u16x2(uint32_t q, uint32_t lo, uint32_t hi) {
    uint32_t r;
    asm("max.u16x2 %0, %1, %2;" : "=r"(r) : "r"(q), "r"(lo));
    asm("min.u16x2 %0, %0, %1;" : "+r"(r) : "r"(hi));
    return r;
}
__device__ __forceinline__ uint32_t box_bound16(const uint16_t* s_e, const uint32_t* qe, const uint32_t* qo,
                                                uint4 lo4, uint4 hi4) {
    const char* tb = reinterpret_cast<const char*>(s_e);
    const uint32_t lw[4] = {lo4.x, lo4.y, lo4.z, lo4.w}, hw[4] = {hi4.x, hi4.y, hi4.z, hi4.w};
    uint32_t lb = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t ce = clamp_u16x2(qe[i], spread_even(lw[i]), spread_even(hw[i])) * 2u;   // lanes <= 510
        const uint32_t co = clamp_u16x2(qo[i], spread_odd(lw[i]), spread_odd(hw[i])) * 2u;
        lb += *reinterpret_cast<const uint16_t*>(tb + (4 * i + 0) * 512 + (ce & 0xFFFFu)) +
              *reinterpret_cast<const uint16_t*>(tb + (4 * i + 2) * 512 + (ce >> 16));
        lb += *reinterpret_cast<const uint16_t*>(tb + (4 * i + 1) * 512 + (co & 0xFFFFu)) +
              *reinterpret_cast<const uint16_t*>(tb + (4 * i + 3) * 512 + (co >> 16));
    }
    return lb;
}

constexpr int NCTR = 5;          // per-query filter counters: leaves tested/passed, points tested/passed, sub-boxes tested

template <int G> struct QuantSpec;
template <> struct QuantSpec<8> { static constexpr uint32_t QT = 2048, CAP = 4095; };
// G = 16: terms are clamped at 127 so that two of them add inside an 8-bit lane.  Clamping
// keeps every term a lower bound (reject rule intact), and a clamped term alone exceeds the
// sure-accept limit QT - 17, so such a point is always decided in fp32 (no result changes).
template <> struct QuantSpec<16> { static constexpr uint32_t QT = 128, CAP = 127; };

// The 16-query box test (K = 16, G = 16 8-bit tables with region flags, see k_range_filter):
// bit g set iff query g's quantised lower bound of the box [lo, hi] is <= QT (128).  Per dim
// the rows D_j[lo] and D_j[hi] are masked by the s < lo / s >= hi query sets (sign-replicating
// byte permutes of the flags), pair sums of 7-bit terms in 8-bit lanes widened into 16-bit lanes.
__device__ __forceinline__ uint32_t simd16_box_mask(const uint4* __restrict__ s_qe, int N_r, uint4 lo4, uint4 hi4) {
    uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int jp = 0; jp < 8; ++jp) {
        uint32_t tw[2][4];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int j = 2 * jp + u, sh = 8 * (j & 3);
            const uint32_t wl = (j >> 2) == 0 ? lo4.x : (j >> 2) == 1 ? lo4.y : (j >> 2) == 2 ? lo4.z : lo4.w;
            const uint32_t wh = (j >> 2) == 0 ? hi4.x : (j >> 2) == 1 ? hi4.y : (j >> 2) == 2 ? hi4.z : hi4.w;
            const uint32_t cl = (wl >> sh) & 255u, ch = (wh >> sh) & 255u;
            const uint4 dl = s_qe[j * N_r + cl];
            const uint4 dh = s_qe[j * N_r + ch];
            const uint32_t dlw[4] = {dl.x, dl.y, dl.z, dl.w}, dhw[4] = {dh.x, dh.y, dh.z, dh.w};
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const uint32_t ml = prmt_sign(dlw[w]);                  // 0xFF: s < lo
                const uint32_t mh = prmt_sign(dhw[w]);                  // 0xFF: s < hi
                // D_j[lo] where s < lo (its flag bit cleared), | D_j[hi] where s >= hi
                // (flag clear there, so bit 7 is already 0): two 3-input logic ops
                const uint32_t tl = dlw[w] & ml & 0x7F7F7F7Fu;
                tw[u][w] = tl | (dhw[w] & ~mh);
            }
        }
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const uint32_t p2 = tw[0][w] + tw[1][w];     // 7-bit terms: no carry out of a byte
            acc[2 * w] += p2 & 0x00FF00FFu;
            acc[2 * w + 1] += __byte_perm(p2, 0u, 0x4341);
        }
    }
    uint32_t m = 0;
#pragma unroll
    for (int g = 0; g < 16; ++g) {
        const uint32_t sg = (acc[2 * (g >> 2) + (g & 1)] >> (16 * ((g >> 1) & 1))) & 0xFFFFu;
        m |= (sg <= QuantSpec<16>::QT ? 1u : 0u) << g;
    }
    return m;
}

struct RFArgs {
    const uint8_t* tcodes;      // tree t: [n][K]
    const uint16_t* ptl;        // tree t: [n] leaf within tile
    const uint32_t* perm;       // tree t: [n]
    const uint32_t* leaf_off;   // global positions
    const uint8_t* lo;          // leaf boxes: box l at lo + l * bs (K bytes), likewise hi
    const uint8_t* hi;
    int bs;                     // box stride in bytes: 2K for the interleaved tight boxes (lo | hi in
                                // one 32-byte row at K = 16: one sector per box), K for prefix boxes
    const uint8_t* tile_lo;     // [ntiles][K] tile bounding boxes
    const uint8_t* tile_hi;
    const uint32_t* tile_leaf;  // [ntiles+1]
    int64_t tile_begin, tile_end;
    int64_t pos_base;           // t * n
    const float* lut;           // [Qb][L][K][N_r] exact
    const uint16_t* qlut;       // [Qb][L][K][N_r] quantised lower bounds (this round)
    const uint4* gtab;          // [groups][K][N_r] the groups' interleaved 8-bit tables (this tree), or null
    const uint8_t* sx;          // [Qb][L][K]
    const float* proj;          // EXACT: data-order projections [n][LK]
    const float* qp;            // EXACT: projected batch queries [Qb][LK]
    const int* act;
    int na;                     // upper bound; the count is *dna when dna != null
    const int* dna;
    const QState* qs;
    QState* qs_mut;             // the same array: per-query mark counts (pub)
    uint32_t* bitmap;           // [Qb][nwords] current union S (OR-marked, no return)
    int64_t nwords;
    uint32_t* wsum;             // [Qb][nsw] dirty-word summary of the bitmap rows
    int64_t nsw;
    float rho2;
    int t, L, K, N_r, mode;
    int pq_cost;                // per-query path cost per 32-point step, relative to 170 per SIMD chunk
    unsigned int* tctr;         // [groups] next tile of each group (zeroed by k_group_table), or null
    int tile_packed;            // k_tile_pairs: list entries hold packed leaf ranges (see there)
    unsigned long long* tp_hist;   // experiments (DETLSH_TP_HIST): reached tiles by number of group queries
    int dbg;                    // experiments (DETLSH_RF_DEBUG): 1 = per-query leaf test; 2 = tile screen
                                // also on the 16-query SIMD leaf path (DETLSH_RF_TSCREEN=1)
    uint32_t* plist;            // CELL, sparse tiles: per-query lists of reachable leaves [Qb][pcap] (or null)
    uint32_t* pcnt;             // [Qb] list lengths
    int64_t pcap;
    unsigned long long* ctr;    // [Qb][4] filter counters
};

template <int KT, int NRT, int G, bool PQ>
__global__ void __launch_bounds__(RF_THREADS, RF_CTAS) k_range_filter(RFArgs a) {
    pdl_wait();
    constexpr uint32_t QT = QuantSpec<G>::QT, CAP = QuantSpec<G>::CAP;
    constexpr bool SIMD_LEAF = KT == 16 && G == 16;   // leaf bounds of all 16 queries per lane
    extern __shared__ __align__(16) unsigned char smem[];
    const int K = KT ? KT : a.K;
    const int N_r = NRT ? NRT : a.N_r;
    uint4* s_qe = reinterpret_cast<uint4*>(smem);                                       // [K][N_r] x 16 B
    // G = 16: byte g of entry (j, c) is query g's 7-bit term D_j[c] with bit 7 set iff the
    // query's own region code in dim j is < c (k_group_table).  A leaf box term D_j[clamp(s, lo,
    // hi)] is then D_j[lo] where entry (j, lo) is flagged (s < lo), D_j[hi] where entry (j, hi)
    // is not (s >= hi; D_j[s] = 0 covers s = hi), 0 otherwise -- byte masks from the flag by one
    // sign-replicating byte permute.  Every other reader masks the flag off.
    __shared__ int s_q[G];
    __shared__ __align__(16) uint8_t s_sx[G][32];
    __shared__ float s_qp[G][32];                                                        // EXACT: q'_t
    __shared__ unsigned int s_ctr[G][4];
    __shared__ unsigned int s_pass[G];                                                  // marks per query
    __shared__ uint32_t s_lq[RF_THREADS / 32][kTileLeaves];                             // per warp: leaf masks
    __shared__ uint32_t s_bq[RF_THREADS / 32][RF_BQ];                                   // per warp: band queue
    __shared__ uint32_t s_pre[RF_THREADS / 32][32];                                     // per warp: packed-point prefix
    __shared__ uint32_t s_off[RF_THREADS / 32][32];                                     // per warp: leaf offsets
    __shared__ int s_active_mask;
    __shared__ unsigned int s_next;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = RF_THREADS / 32;
    if (threadIdx.x < G) {
        const int gi = blockIdx.x * G + threadIdx.x;
        int q = -1;
        if (gi < (a.dna ? *a.dna : a.na)) {
            q = a.act[gi];
            if (a.qs[q].status != ST_ACTIVE) q = -1;       // stopped at an earlier tree (line 7)
        }
        s_q[threadIdx.x] = q;
        for (int c = 0; c < 4; ++c) s_ctr[threadIdx.x][c] = 0;
        s_pass[threadIdx.x] = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int m = 0;
        for (int g = 0; g < G; ++g) m |= (s_q[g] >= 0) << g;
        s_active_mask = m;
    }
    __syncthreads();
    const uint32_t amask = (uint32_t)s_active_mask;
    if (amask == 0) return;
    const int64_t per_q = (int64_t)a.L * K * N_r;
    {   // interleave the G queries' quantised tables: entry (j, s) = 16 bytes
        const uint16_t* src[G];
#pragma unroll
        for (int g = 0; g < G; ++g)
            src[g] = s_q[g] >= 0 ? a.qlut + (int64_t)s_q[g] * per_q + (int64_t)a.t * K * N_r : nullptr;
        if (a.gtab) {   // the group's table, interleaved once per tree by k_group_table: plain copy
            const uint4* gt = a.gtab + (int64_t)blockIdx.x * K * N_r;
            for (int i = threadIdx.x; i < K * N_r; i += RF_THREADS) s_qe[i] = gt[i];
        } else {
            for (int i = threadIdx.x; i < K * N_r; i += RF_THREADS) {
                uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    uint32_t v = src[g] ? src[g][i] : CAP;                             // inactive: never passes
                    if (G == 16 && src[g] && (int)a.sx[((int64_t)s_q[g] * a.L + a.t) * K + i / N_r] < i % N_r)
                        v |= 0x80u;                                                    // region flag (above)
                    if (G == 8) w[g >> 1] |= v << (16 * (g & 1));
                    else w[g >> 2] |= v << (8 * (g & 3));
                }
                s_qe[i] = make_uint4(w[0], w[1], w[2], w[3]);
            }
        }
        if (threadIdx.x < K) {
#pragma unroll
            for (int g = 0; g < G; ++g) {
                s_sx[g][threadIdx.x] = s_q[g] >= 0 ? a.sx[((int64_t)s_q[g] * a.L + a.t) * K + threadIdx.x] : 0;
                if (a.mode == DETLSH_MODE_EXACT)
                    s_qp[g][threadIdx.x] = s_q[g] >= 0 ? a.qp[(int64_t)s_q[g] * a.L * K + a.t * K + threadIdx.x] : 0.f;
            }
        }
    }
    __syncthreads();
    const float rho2 = a.rho2;
    const uint16_t* s_h = reinterpret_cast<const uint16_t*>(s_qe);
    const uint8_t* s_b = reinterpret_cast<const uint8_t*>(s_qe);
    uint32_t c_lt = 0, c_lp = 0, c_pt = 0, c_pp = 0;
    uint32_t* lq = s_lq[warp];
    uint32_t* bq = s_bq[warp];
    uint32_t qn_ = 0;                     // queued band pairs (warp-uniform)

    // warps take tiles one at a time, dynamically: from the group's counter shared by all of the
    // group's CTAs (a.tctr), else from this CTA's contiguous stripe
    const int64_t ntl = a.tile_end - a.tile_begin;
    const int64_t tb = a.tctr ? a.tile_begin : a.tile_begin + ntl * blockIdx.y / gridDim.y;
    const int64_t te = a.tctr ? a.tile_end : a.tile_begin + ntl * (blockIdx.y + 1) / gridDim.y;
    unsigned int* next = a.tctr ? a.tctr + blockIdx.x : &s_next;
    if (threadIdx.x == 0) s_next = 0;
    __syncthreads();
    for (;;) {
        int64_t tile = 0;
        if (lane == 0) tile = tb + atomicAdd(next, 1);
        tile = __shfl_sync(0xffffffffu, tile, 0);
        if (tile >= te) break;
        const uint32_t lb = a.tile_leaf[tile], le = a.tile_leaf[tile + 1];
        const int nlt = (int)(le - lb);
        const uint32_t P0 = a.leaf_off[lb], P1 = a.leaf_off[le];
        // tile screen: quantised lower bound of the tile's bounding box (lane g = query g); a
        // tile no query can reach is skipped whole (every leaf LB >= the tile's LB)
        uint32_t tm;
        {
            bool pass = false;
            if (SIMD_LEAF && !(a.dbg & 3) && lane < G) {
                // the 16-query leaf test below costs the same whatever subset reached the tile,
                // and the group's 16 queries reach ~every tile between them: the tile screen
                // would only add work (every leaf bound is computed for every active query)
                pass = (amask >> lane) & 1;
            } else if (lane < G && ((amask >> lane) & 1)) {
                uint32_t acc = 0;
                if (KT == 16) {
                    const uint4 tl4 = *reinterpret_cast<const uint4*>(a.tile_lo + tile * 16);
                    const uint4 th4 = *reinterpret_cast<const uint4*>(a.tile_hi + tile * 16);
                    const uint4 sx4 = *reinterpret_cast<const uint4*>(&s_sx[lane][0]);
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const int sh = 8 * (j & 3);
                        const uint32_t wl = (j >> 2) == 0 ? tl4.x : (j >> 2) == 1 ? tl4.y : (j >> 2) == 2 ? tl4.z : tl4.w;
                        const uint32_t wh = (j >> 2) == 0 ? th4.x : (j >> 2) == 1 ? th4.y : (j >> 2) == 2 ? th4.z : th4.w;
                        const uint32_t ws = (j >> 2) == 0 ? sx4.x : (j >> 2) == 1 ? sx4.y : (j >> 2) == 2 ? sx4.z : sx4.w;
                        const int c = min(max((int)((ws >> sh) & 255u), (int)((wl >> sh) & 255u)), (int)((wh >> sh) & 255u));
                        acc += G == 8 ? (uint32_t)s_h[(j * N_r + c) * 8 + lane] : (uint32_t)(s_b[(j * N_r + c) * 16 + lane] & 0x7Fu);
                    }
                } else {
                    const uint8_t* tl = a.tile_lo + tile * K;
                    const uint8_t* th = a.tile_hi + tile * K;
                    for (int j = 0; j < K; ++j) {
                        const int e = (j * N_r + min(max((int)s_sx[lane][j], (int)tl[j]), (int)th[j])) * 16;
                        acc += G == 8 ? (uint32_t)s_h[e / 2 + lane] : (uint32_t)(s_b[e + lane] & 0x7Fu);
                    }
                }
                pass = acc <= QT;
            }
            tm = __ballot_sync(0xffffffffu, pass);
            // tile boxes bound the tight leaf boxes; RELAXED decides leaves by their prefix boxes
            if (a.mode == DETLSH_MODE_RELAXED) tm = amask;
        }
        if (tm == 0) continue;
        // leaf lower bounds (Alg. 3 pruning, Fig. dist): lane = leaf, quantised, one query of the
        // tile's set at a time (warp-uniform loop)
        if (lane < nlt) {
            const int64_t l = (int64_t)lb + lane;
            uint32_t m = 0;
            if (KT == 16 && G == 16 && !(a.dbg & 1)) {
                // all 16 queries at once (same 16-bit lane layout as the SIMD point screen): per
                // dim, the rows D_j[lo] and D_j[hi] masked by the s < lo / s > hi query sets
                m = simd16_box_mask(s_qe, N_r, *reinterpret_cast<const uint4*>(a.lo + l * a.bs),
                                    *reinterpret_cast<const uint4*>(a.hi + l * a.bs)) & tm;
            } else if (KT == 16) {
                const uint4 lo4 = *reinterpret_cast<const uint4*>(a.lo + l * a.bs);
                const uint4 hi4 = *reinterpret_cast<const uint4*>(a.hi + l * a.bs);
                for (uint32_t mm = tm; mm; mm &= mm - 1) {
                    const int g = __ffs(mm) - 1;
                    const uint4 sx4 = *reinterpret_cast<const uint4*>(&s_sx[g][0]);
                    uint32_t acc = 0;
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const int sh = 8 * (j & 3);
                        const uint32_t wl = (j >> 2) == 0 ? lo4.x : (j >> 2) == 1 ? lo4.y : (j >> 2) == 2 ? lo4.z : lo4.w;
                        const uint32_t wh = (j >> 2) == 0 ? hi4.x : (j >> 2) == 1 ? hi4.y : (j >> 2) == 2 ? hi4.z : hi4.w;
                        const uint32_t ws = (j >> 2) == 0 ? sx4.x : (j >> 2) == 1 ? sx4.y : (j >> 2) == 2 ? sx4.z : sx4.w;
                        const int c = min(max((int)((ws >> sh) & 255u), (int)((wl >> sh) & 255u)), (int)((wh >> sh) & 255u));
                        acc += G == 8 ? (uint32_t)s_h[(j * N_r + c) * 8 + g] : (uint32_t)(s_b[(j * N_r + c) * 16 + g] & 0x7Fu);
                    }
                    if (acc <= QT) m |= 1u << g;
                }
            } else {
                for (uint32_t mm = tm; mm; mm &= mm - 1) {
                    const int g = __ffs(mm) - 1;
                    uint32_t acc = 0;
                    for (int j = 0; j < K; ++j) {
                        const int e = (j * N_r + min(max((int)s_sx[g][j], (int)a.lo[l * a.bs + j]), (int)a.hi[l * a.bs + j])) * 16;
                        acc += G == 8 ? (uint32_t)s_h[e / 2 + g] : (uint32_t)(s_b[e + g] & 0x7Fu);
                    }
                    if (acc <= QT) m |= 1u << g;
                }
            }
            if (a.mode == DETLSH_MODE_RELAXED) {
                // RELAXED (Sec. 6.2.2(1)): the leaf decision is final, so decide it in fp32
                uint32_t conf = 0, mm = m;
                while (mm) {
                    const int g = __ffs(mm) - 1;
                    mm &= mm - 1;
                    const float* D = a.lut + (int64_t)s_q[g] * per_q + (int64_t)a.t * K * N_r;
                    float s_ = 0.f;
                    for (int j = 0; j < K; ++j)
                        s_ += __ldg(D + j * N_r + min(max((int)s_sx[g][j], (int)a.lo[l * a.bs + j]), (int)a.hi[l * a.bs + j]));
                    if (s_ <= rho2) conf |= 1u << g;
                }
                m = conf;
            }
            lq[lane] = m;
            c_lt += __popc(tm);
            c_lp += __popc(m);
        }
        __syncwarp();
        // exact fp32 cell bound (summed in j order, AMB-12/29) of queued band pairs: one pair
        // per lane, all lanes busy (instead of a divergent per-lane loop over band queries)
        auto flush = [&](int cnt) {
            if (lane < cnt) {
                const uint32_t e = bq[qn_ - cnt + lane];
                const int g = (int)(e & 15u);
                const int64_t pos = (int64_t)(P0 + (e >> 4)) - a.pos_base;
                const float* D = a.lut + (int64_t)s_q[g] * per_q + (int64_t)a.t * K * N_r;
                float s_ = 0.f;
                if (a.mode == DETLSH_MODE_EXACT) {
                    // Alg. 3 as written: ||q'_t - p'_t||^2 in fp32, j order
                    const float* pp = a.proj + (int64_t)a.perm[pos] * a.L * K + a.t * K;
                    for (int j = 0; j < K; ++j) {
                        const float df = s_qp[g][j] - __ldg(pp + j);
                        s_ = fmaf(df, df, s_);
                    }
                } else if (KT == 16) {
                    const uint4 c4 = *reinterpret_cast<const uint4*>(a.tcodes + pos * 16);
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const uint32_t word = (j >> 2) == 0 ? c4.x : (j >> 2) == 1 ? c4.y : (j >> 2) == 2 ? c4.z : c4.w;
                        s_ += __ldg(D + j * N_r + ((word >> (8 * (j & 3))) & 255u));
                    }
                } else {
                    for (int j = 0; j < K; ++j) s_ += __ldg(D + j * N_r + a.tcodes[pos * K + j]);
                }
                if (s_ <= rho2) {
                    ++c_pp;
                    atomicAdd(&s_pass[g], 1u);
                    const uint32_t id = a.perm[pos];
                    mark_member(a.bitmap + (int64_t)s_q[g] * a.nwords, a.wsum + (int64_t)s_q[g] * a.nsw, id);
                }
            }
            qn_ -= cnt;
        };
        // Two ways to screen the points of the reachable leaves:
        //  SIMD  every 32-point chunk of the tile, all G queries at once (16-byte loads serve G
        //        queries) -- best when each point is needed by many of the group's queries;
        //  per-query  for each query, only the points of ITS reachable leaves, packed 32 to a
        //        step -- best at small radii, where a point is needed by ~2 of 16 queries.
        // Chosen per tile from a cost ratio fitted on B200 (pq_cost 40 against 170 per SIMD chunk).
        // In CELL mode the per-query work of sparse tiles is handed to k_leaf_points as
        // (query, reachable leaf) pairs (high-occupancy kernel, coalesced leaf reads); the in-kernel
        // per-query path serves EXACT.
        bool use_pq = false;
        uint32_t my_off = P1, my_sz = 0;
        if (PQ && KT == 16 && a.mode != DETLSH_MODE_RELAXED) {
            if (lane < nlt) {
                my_off = a.leaf_off[lb + lane];
                my_sz = a.leaf_off[lb + lane + 1] - my_off;
            }
            uint32_t w_ = lane < nlt ? (uint32_t)__popc(lq[lane]) * my_sz : 0u;
            for (int o = 16; o > 0; o >>= 1) w_ += __shfl_xor_sync(0xffffffffu, w_, o);
            use_pq = (unsigned long long)a.pq_cost * w_ < 170ull * (P1 - P0);
        }
        if (use_pq && a.plist != nullptr && a.mode == DETLSH_MODE_CELL) {
            // hand the (query, reachable leaf) pairs of this sparse tile to k_leaf_points: per-warp
            // shared counters count each query's pairs, lane g reserves query g's slots in its global
            // list (all reservations in flight together), then each lane writes its own pairs at
            // slots taken from a second counter -- work per lane ~ its (few) pairs, not per query of
            // the group (a query's list order does not matter: k_leaf_points ORs marks)
            uint32_t* w_cnt = s_pre[warp];          // [0,16) counts, [16,32) bases (the per-query
            uint32_t* w_slot = s_off[warp];         // path's scratch, unused in CELL); [0,16) slots
            const uint32_t my_lq = lane < nlt ? lq[lane] : 0u;
            if (lane < 16) { w_cnt[lane] = 0; w_slot[lane] = 0; }
            __syncwarp();
            for (uint32_t mm = my_lq; mm; mm &= mm - 1) atomicAdd(&w_cnt[__ffs(mm) - 1], 1u);
            __syncwarp();
            if (lane < 16) {
                const uint32_t c_ = w_cnt[lane];
                w_cnt[16 + lane] = c_ ? atomicAdd(a.pcnt + s_q[lane], c_) : 0u;
            }
            __syncwarp();
            for (uint32_t mm = my_lq; mm; mm &= mm - 1) {
                const int g = __ffs(mm) - 1;
                const uint32_t sl = w_cnt[16 + g] + atomicAdd(&w_slot[g], 1u);
                a.plist[(int64_t)s_q[g] * a.pcap + sl] = lb + lane;
            }
            __syncwarp();
        } else if (use_pq) {
            uint32_t* pre = s_pre[warp];
            uint32_t* offs = s_off[warp];
            for (uint32_t mm = tm; mm; mm &= mm - 1) {
                const int g = __ffs(mm) - 1;
                const bool pl = lane < nlt && ((lq[lane] >> g) & 1u);
                const uint32_t sz = pl ? my_sz : 0u;
                uint32_t incl = sz;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                const uint32_t T = __shfl_sync(0xffffffffu, incl, 31);
                if (T == 0) continue;
                pre[lane] = incl - sz;
                offs[lane] = my_off;
                __syncwarp();
                // two packed points per lane per iteration: both searches and both code loads are
                // issued before either sum (two independent latency chains)
                for (uint32_t c0 = 0; c0 < T; c0 += 64) {
                    uint32_t pp[2] = {P0, P0};
                    uint4 cc[2];
                    bool valid[2];
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const uint32_t i = c0 + 32 * u + lane;
                        valid[u] = i < T;
                        cc[u] = make_uint4(0, 0, 0, 0);
                        if (valid[u]) {
                            int l = 0;      // the leaf holding packed point i: last l with pre[l] <= i
#pragma unroll
                            for (int st = 16; st > 0; st >>= 1)
                                if (pre[l + st] <= i) l += st;
                            pp[u] = offs[l] + (i - pre[l]);
                            cc[u] = *reinterpret_cast<const uint4*>(a.tcodes + ((int64_t)pp[u] - a.pos_base) * 16);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        bool band = false;
                        const uint32_t p = pp[u];
                        if (valid[u]) {
                            const int64_t pos = (int64_t)p - a.pos_base;
                            const uint4 c4 = cc[u];
                            uint32_t acc = 0;
#pragma unroll
                            for (int j = 0; j < 16; ++j) {
                                const uint32_t word = (j >> 2) == 0 ? c4.x : (j >> 2) == 1 ? c4.y : (j >> 2) == 2 ? c4.z : c4.w;
                                const uint32_t code = (word >> (8 * (j & 3))) & 255u;
                                acc += G == 8 ? (uint32_t)s_h[(j * N_r + code) * 8 + g] : (uint32_t)(s_b[(j * N_r + code) * 16 + g] & 0x7Fu);
                            }
                            ++c_pt;
                            const bool ok = acc <= QT, sure = acc + 17 <= QT;
                            if (a.mode == DETLSH_MODE_CELL && sure) {
                                ++c_pp;
                                atomicAdd(&s_pass[g], 1u);
                                const uint32_t id = a.perm[pos];
                                mark_member(a.bitmap + (int64_t)s_q[g] * a.nwords, a.wsum + (int64_t)s_q[g] * a.nsw, id);
                            } else {
                                band = ok;      // CELL: inside the band; EXACT: every survivor
                            }
                        }
                        const uint32_t bal = __ballot_sync(0xffffffffu, band);
                        if (band) bq[qn_ + __popc(bal & lanemask_lt())] = ((p - P0) << 4) | (uint32_t)g;
                        qn_ += __popc(bal);
                        __syncwarp();
                        if (qn_ >= 32) flush(32);
                        __syncwarp();
                    }
                }
            }
        } else {
        // software pipeline: the next chunk's leaf slots, codes and ids load while this one is screened
            uint32_t nx_ptl = 0, nx_id = 0;
            uint4 nx_c4 = make_uint4(0, 0, 0, 0);
            auto load_chunk = [&](uint32_t pb_) {
                const uint32_t p_ = pb_ + lane;
                if (p_ < P1) {
                    const int64_t pos_ = (int64_t)p_ - a.pos_base;
                    nx_ptl = a.ptl[pos_];
                    nx_id = a.perm[pos_];
                    if (KT == 16) nx_c4 = *reinterpret_cast<const uint4*>(a.tcodes + pos_ * 16);
                }
            };
            load_chunk(P0);
            for (uint32_t pb = P0; pb < P1; pb += 32) {
                const uint32_t p = pb + lane;
                const int64_t pos = (int64_t)p - a.pos_base;
                const uint32_t cur_ptl = nx_ptl, cur_id = nx_id;
                const uint4 c4 = nx_c4;
                if (pb + 32 < P1) load_chunk(pb + 32);
                uint32_t m = 0;
                if (p < P1) m = lq[cur_ptl];
                if (__ballot_sync(0xffffffffu, m != 0) == 0) continue;    // whole warp pruned by leaf LBs
                c_pt += __popc(m);
                uint32_t certain = m, band = 0;
                if (m && a.mode != DETLSH_MODE_RELAXED) {
                    uint32_t ok = 0, sure = 0;
                    if (KT == 16) {
                        uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
                        for (int w = 0; w < 4; ++w) {
                            const uint32_t word = w == 0 ? c4.x : w == 1 ? c4.y : w == 2 ? c4.z : c4.w;
                            const uint4* row = s_qe + (w * 4) * N_r;
                            if (G == 8) {
#pragma unroll
                                for (int b = 0; b < 4; ++b) {
                                    const uint4 v = row[b * N_r + ((word >> (8 * b)) & 255u)];
                                    acc[0] += v.x; acc[1] += v.y; acc[2] += v.z; acc[3] += v.w;
                                }
                            } else {
                                // 7-bit terms (CAP 127): two dims add inside the 8-bit lanes without
                                // carry (<= 254); each pair sum is then widened into 16-bit lanes
                                // (g0,g2) by a mask and (g1,g3) by a byte permute.
                                const uint4 va = row[0 * N_r + (word & 255u)];
                                const uint4 vb = row[1 * N_r + ((word >> 8) & 255u)];
                                const uint4 vc = row[2 * N_r + ((word >> 16) & 255u)];
                                const uint4 vd = row[3 * N_r + (word >> 24)];
                                constexpr uint32_t M7 = 0x7F7F7F7Fu;     // region flags off
                                const uint32_t p2[4] = {(va.x & M7) + (vb.x & M7), (va.y & M7) + (vb.y & M7),
                                                        (va.z & M7) + (vb.z & M7), (va.w & M7) + (vb.w & M7)};
                                const uint32_t r2[4] = {(vc.x & M7) + (vd.x & M7), (vc.y & M7) + (vd.y & M7),
                                                        (vc.z & M7) + (vd.z & M7), (vc.w & M7) + (vd.w & M7)};
#pragma unroll
                                for (int i = 0; i < 4; ++i) {
                                    acc[2 * i] += (p2[i] & 0x00FF00FFu) + (r2[i] & 0x00FF00FFu);
                                    acc[2 * i + 1] += __byte_perm(p2[i], 0u, 0x4341) + __byte_perm(r2[i], 0u, 0x4341);
                                }
                            }
                        }
#pragma unroll
                        for (int g = 0; g < G; ++g) {
                            const uint32_t sg = G == 8 ? (acc[g >> 1] >> (16 * (g & 1))) & 0xFFFFu
                                                       : (acc[2 * (g >> 2) + (g & 1)] >> (16 * ((g >> 1) & 1))) & 0xFFFFu;
                            ok |= (sg <= QT ? 1u : 0u) << g;
                            sure |= (sg + 17 <= QT ? 1u : 0u) << g;
                        }
                    } else {
                        uint32_t acc[G];
#pragma unroll
                        for (int g = 0; g < G; ++g) acc[g] = 0;
                        for (int j = 0; j < K; ++j) {
                            const int e = (j * N_r + a.tcodes[pos * K + j]) * 16;
#pragma unroll
                            for (int g = 0; g < G; ++g) acc[g] += G == 8 ? (uint32_t)s_h[e / 2 + g] : (uint32_t)(s_b[e + g] & 0x7Fu);
                        }
#pragma unroll
                        for (int g = 0; g < G; ++g) {
                            ok |= (acc[g] <= QT ? 1u : 0u) << g;
                            sure |= (acc[g] + 17 <= QT ? 1u : 0u) << g;
                        }
                    }
                    if (a.mode == DETLSH_MODE_CELL) {
                        certain = m & sure;
                        band = m & ok & ~sure;
                    } else {       // EXACT: the cell bound only rejects; every survivor gets its true distance
                        certain = 0;
                        band = m & ok;
                    }
                }
                if (certain) {
                    c_pp += __popc(certain);
                    const uint32_t id = cur_id;
                    uint32_t c_ = certain;
                    while (c_) {
                        const int g = __ffs(c_) - 1;
                        c_ &= c_ - 1;
                        atomicAdd(&s_pass[g], 1u);
                        mark_member(a.bitmap + (int64_t)s_q[g] * a.nwords, a.wsum + (int64_t)s_q[g] * a.nsw, id);
                    }
                }
                // queue the band pairs (point in tile << 4 | query slot) for the warp-wide fp32 pass:
                // one pair per lane per step, flushed 32 at a time
                while (__any_sync(0xffffffffu, band != 0)) {
                    const bool has = band != 0;
                    const uint32_t bal = __ballot_sync(0xffffffffu, has);
                    if (has) {
                        const int g = __ffs(band) - 1;
                        band &= band - 1;
                        bq[qn_ + __popc(bal & lanemask_lt())] = ((p - P0) << 4) | (uint32_t)g;
                    }
                    qn_ += __popc(bal);
                    __syncwarp();
                    if (qn_ >= 32) flush(32);
                    __syncwarp();
                }
            }
        }
        if (qn_) flush(qn_);
        __syncwarp();
    }
    // ---- counters (per group; attributed evenly to its active queries)
    {
        uint32_t v[4] = {c_lt, c_lp, c_pt, c_pp};
#pragma unroll
        for (int i = 0; i < 4; ++i)
            for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
        if (lane == 0) {
            const int na_ = max(1, __popc(amask));
            for (int g = 0; g < G; ++g)
                if ((amask >> g) & 1)
                    for (int i = 0; i < 4; ++i) atomicAdd(&s_ctr[g][i], v[i] / na_);
        }
    }
    __syncthreads();
    if (threadIdx.x < G && s_q[threadIdx.x] >= 0) {
        unsigned long long* c = a.ctr + (int64_t)s_q[threadIdx.x] * NCTR;
        for (int i = 0; i < 4; ++i) atomicAdd(c + i, (unsigned long long)s_ctr[threadIdx.x][i]);
        if (s_pass[threadIdx.x])
            atomicAdd(reinterpret_cast<unsigned long long*>(&a.qs_mut[s_q[threadIdx.x]].pub),
                      (unsigned long long)s_pass[threadIdx.x]);
    }
}

// ---- locality order of a tree's active queries (two-level filter): key = the query's own
//      first-layer cell in tree t (top bit of its region code in each dim, dim 0 most significant);
//      entries past the device count sort last.  Queries reaching the same cells then run side by
//      side in the pair kernel and share its box / code reads in L2.
__global__ void k_qkey(const int* __restrict__ act, int na_ub, const int* __restrict__ dna,
                       const uint8_t* __restrict__ sx, int L, int K, int nb, int t,
                       uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    pdl_wait();
    const int na = dna ? *dna : na_ub;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < na_ub; i += gridDim.x * blockDim.x) {
        uint32_t key = 0xFFFFFFu;
        int q = act[i];
        if (i < na) {
            const uint8_t* c = sx + ((int64_t)q * L + t) * K;
            key = 0;
            for (int j = 0; j < K && j < 23; ++j) key = (key << 1) | ((c[j] >> (nb - 1)) & 1u);
        }
        keys[i] = key;
        vals[i] = (uint32_t)q;
    }
}

// ---- between two chunks of a tree (L2 blocking, see query_index): the pair lists continue
//      (entries taken so far = entries listed so far) and the groups' tile counters restart.
__global__ void k_chunk_prep(const int* __restrict__ act, int na_ub, const int* __restrict__ dna,
                             const uint32_t* __restrict__ pcnt, uint32_t* __restrict__ ptake,
                             unsigned int* __restrict__ tctr) {
    pdl_wait();
    const int na = dna ? *dna : na_ub;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < na; i += gridDim.x * blockDim.x) {
        if (pcnt) {
            const int q = act[i];
            ptake[q] = pcnt[q];
        }
        if (tctr && (i & 15) == 0) tctr[i >> 4] = 0;
    }
}

// ---- tile-pair mode (CELL, K = 16, N_r = 256): the first stage of a two-level filter for
//      indexes whose per-query reach is a small fraction of the tiles (large n, small radius).
//      CTA = 16-query group (its interleaved table, as k_range_filter); a warp takes 32 tiles
//      at a time from the group's counter, lane = tile: the 16-query bound of the tile's box
//      (union of its leaves' tight boxes -- never above a member leaf's bound), and every
//      (query, tile) pair that passes is appended to the query's list.  k_leaf_points then
//      expands each listed tile into its leaves (one warp per tile, lane = leaf) with the
//      query's own 12-bit table -- only the pairs a query reaches are bounded, instead of every
//      leaf of every tile any of the 16 queries reaches (the group's union).
__global__ void __launch_bounds__(RF_THREADS, RF_CTAS) k_tile_pairs(RFArgs a) {
    pdl_wait();
    extern __shared__ __align__(16) unsigned char smem[];
    uint4* s_qe = reinterpret_cast<uint4*>(smem);                 // [16][256] x 16 B
    constexpr int G = 16, N_r = 256, K = 16;
    __shared__ int s_q[G];
    __shared__ unsigned int s_ctr[G][2];
    __shared__ uint32_t s_cnt[RF_THREADS / 32][32];                // per warp: [0,16) counts, [16,32) bases
    __shared__ uint32_t s_slot[RF_THREADS / 32][16];
    __shared__ int s_active_mask;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x < G) {
        const int gi = blockIdx.x * G + threadIdx.x;
        int q = -1;
        if (gi < (a.dna ? *a.dna : a.na)) {
            q = a.act[gi];
            if (a.qs[q].status != ST_ACTIVE) q = -1;
        }
        s_q[threadIdx.x] = q;
        s_ctr[threadIdx.x][0] = s_ctr[threadIdx.x][1] = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int m = 0;
        for (int g = 0; g < G; ++g) m |= (s_q[g] >= 0) << g;
        s_active_mask = m;
    }
    {
        const uint4* gt = a.gtab + (int64_t)blockIdx.x * K * N_r;
        for (int i = threadIdx.x; i < K * N_r; i += RF_THREADS) s_qe[i] = gt[i];
    }
    __syncthreads();
    const uint32_t amask = (uint32_t)s_active_mask;
    if (amask == 0) return;
    uint32_t c_lt = 0, c_lp = 0;
    uint32_t* w_cnt = s_cnt[warp];
    uint32_t* w_slot = s_slot[warp];
    unsigned int* next = a.tctr + blockIdx.x;
    for (;;) {
        int64_t t0 = 0;
        if (lane == 0) t0 = a.tile_begin + 32 * (int64_t)atomicAdd(next, 1);
        t0 = __shfl_sync(0xffffffffu, t0, 0);
        if (t0 >= a.tile_end) break;
        const int64_t T = t0 + lane;
        uint32_t m = 0;
        if (T < a.tile_end) {
            m = simd16_box_mask(s_qe, N_r, *reinterpret_cast<const uint4*>(a.tile_lo + T * 16),
                                *reinterpret_cast<const uint4*>(a.tile_hi + T * 16)) & amask;
            c_lt += __popc(amask);
            c_lp += __popc(m);
            if (a.tp_hist && m) atomicAdd(a.tp_hist + __popc(m), 1ull);
        }
        // append the (query, tile) pairs: per-query counts in the warp, one reservation per query
        // in its global list, then each lane writes its own pairs
        if (lane < 16) { w_cnt[lane] = 0; w_slot[lane] = 0; }
        __syncwarp();
        for (uint32_t mm = m; mm; mm &= mm - 1) atomicAdd(&w_cnt[__ffs(mm) - 1], 1u);
        __syncwarp();
        if (lane < 16) {
            const uint32_t c_ = w_cnt[lane];
            w_cnt[16 + lane] = c_ ? atomicAdd(a.pcnt + s_q[lane], c_) : 0u;
        }
        __syncwarp();
        // list entry: the tile's leaf range packed as (first leaf << 5 | count - 1) when the index
        // has < 2^27 leaves (the pair kernel then skips one dependent load), else the tile index
        uint32_t entry = (uint32_t)T;
        if (m && a.tile_packed) {
            const uint32_t lb0 = a.tile_leaf[T], le0 = a.tile_leaf[T + 1];
            entry = (lb0 << 5) | (le0 - lb0 - 1);
        }
        for (uint32_t mm = m; mm; mm &= mm - 1) {
            const int g = __ffs(mm) - 1;
            const uint32_t sl = w_cnt[16 + g] + atomicAdd(&w_slot[g], 1u);
            a.plist[(int64_t)s_q[g] * a.pcap + sl] = entry;
        }
        __syncwarp();
    }
    // counters (tile bounds count as box bounds: leaves_tested / leaves_passed), per group split
    // evenly over its active queries as in k_range_filter
    for (int o = 16; o > 0; o >>= 1) {
        c_lt += __shfl_xor_sync(0xffffffffu, c_lt, o);
        c_lp += __shfl_xor_sync(0xffffffffu, c_lp, o);
    }
    if (lane == 0) {
        const int na_ = max(1, __popc(amask));
        for (int g = 0; g < G; ++g)
            if ((amask >> g) & 1) {
                atomicAdd(&s_ctr[g][0], c_lt / na_);
                atomicAdd(&s_ctr[g][1], c_lp / na_);
            }
    }
    __syncthreads();
    if (threadIdx.x < G && s_q[threadIdx.x] >= 0) {
        unsigned long long* c = a.ctr + (int64_t)s_q[threadIdx.x] * NCTR;
        atomicAdd(c + 0, (unsigned long long)s_ctr[threadIdx.x][0]);
        atomicAdd(c + 1, (unsigned long long)s_ctr[threadIdx.x][1]);
    }
}

// ---- sparse tiles, CELL mode: the points of each (query, reachable leaf) pair the range filter
//      listed, one warp per leaf, lane per point.  Block = one query (its fp32 table of tree t and a
//      12-bit quantised lower-bound copy in shared memory, ~24 KB: many resident blocks per SM);
//      codes are read coalesced (a leaf's points are contiguous).  Same decision as the filter:
//      sum of 12-bit terms (each <= D 2048/rho^2, rounded down) > 2048 rejects, <= 2031 accepts,
//      the band in between takes the exact fp32 sum in j order (AMB-29).
struct LPArgs {
    const int* act;
    const int* dna;
    int na;
    const QState* qs;
    QState* qs_mut;
    const uint32_t* plist;
    uint32_t* pcnt;
    uint32_t* ptake;            // [Qb] chunks of the list taken so far (dynamic work split)
    int64_t pcap;
    const float* lut;           // [Qb][L][K][N_r]
    const uint16_t* q12;        // [Qb][L][K][N_r] 12-bit lower bounds of this round (k_build_qlut, QT 2048)
    const uint32_t* leaf_off;   // global positions
    const uint8_t* lo;          // tight leaf boxes, box l at lo + l * bs (interleaved: bs = 2K)
    const uint8_t* hi;
    int bs;
    const uint32_t* sb_off;     // [nl_total+1] first sub-box of each leaf (null: no sub-box level)
    const uint8_t* sb_lo;       // sub-box tight boxes, interleaved: box i at sb_lo + 2K i, hi at sb_lo + 2K i + K
    const uint8_t* sb_hi;
    const uint8_t* sx;          // [Qb][L][K] query region codes
    const uint8_t* tcodes;      // tree t [n][K]
    const uint32_t* perm;       // tree t [n]
    int64_t pos_base;
    uint32_t* bitmap;
    int64_t nwords;
    uint32_t* wsum;             // [Qb][nsw] dirty-word summary
    int64_t nsw;
    float rho2, inv_rd;         // inv_rd = 2048/rho^2 rounded down
    int t, L, K, N_r;
    unsigned long long* ctr;
    const uint32_t* tile_leaf;  // non-null: the lists hold tiles (k_tile_pairs), each expanded into its
                                // leaves here (one tile per warp chunk, lane = leaf; LPG = 32)
    int tile_packed;            // the tile entries are packed leaf ranges (first leaf << 5 | count - 1)
};

constexpr int LP_THREADS = 256;     // threads per pair-kernel block (512 with half the blocks: slower)

// KT, NRT > 0: K and N_r fixed at compile time (table rows at immediate offsets, a static table);
// LPG listed leaves per warp chunk
// BX bit 0: box bounds by box_bound16 (K = 16, N_r = 256); bit 1: FIFO sub-box queue with L2 prefetch
// of the point codes (bit 2: into L1)
template <int KT, int NRT, int LPG, int BX = 0>
__global__ void __launch_bounds__(LP_THREADS, LPG == 32 ? 5 : 6) k_leaf_points(LPArgs a) {
    pdl_wait();
    extern __shared__ __align__(16) unsigned char lp_smem[];
    __shared__ __align__(16) uint16_t lp_static[(KT > 0 && NRT > 0) ? KT * NRT : 8];
    const int ai = blockIdx.x;
    if (ai >= (a.dna ? *a.dna : a.na)) return;
    const int q = a.act[ai];
    const uint32_t np = a.pcnt[q];
    if (np == 0 || np <= a.ptake[q] || a.qs[q].status != ST_ACTIVE) return;
    const int K = KT > 0 ? KT : a.K, N_r = NRT > 0 ? NRT : a.N_r, KN = K * N_r;
    uint16_t* s_e = (KT > 0 && NRT > 0) ? lp_static : reinterpret_cast<uint16_t*>(lp_smem);   // 12-bit lower bounds
    const float* s_d = a.lut + ((int64_t)q * a.L + a.t) * KN;              // exact terms (band only, L1/L2)
    {
        const uint4* src = reinterpret_cast<const uint4*>(a.q12 + ((int64_t)q * a.L + a.t) * KN);
        uint4* dst = reinterpret_cast<uint4*>(s_e);
        for (int i = threadIdx.x; i < KN / 8; i += blockDim.x) dst[i] = src[i];
    }
    __shared__ unsigned int s_tested, s_passed, s_sbt;
    __shared__ int s_qx[32];                          // the query's region codes in tree t
    if (threadIdx.x == 0) { s_tested = 0; s_passed = 0; s_sbt = 0; }
    if (threadIdx.x < K) s_qx[threadIdx.x] = a.sx[((int64_t)q * a.L + a.t) * K + threadIdx.x];
    constexpr bool B16 = (BX & 1) && KT == 16 && NRT == 256;
    __shared__ uint32_t s_qeo[8];                     // B16: the query's codes spread for box_bound16
    if (B16 && threadIdx.x >= 32 && threadIdx.x < 40) {
        const int i = (threadIdx.x - 32) & 3, od = (threadIdx.x - 32) >> 2;
        const uint8_t* x = a.sx + ((int64_t)q * a.L + a.t) * K + 4 * i + od;
        s_qeo[threadIdx.x - 32] = (uint32_t)x[0] | ((uint32_t)x[2] << 16);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint32_t* pl = a.plist + (int64_t)q * a.pcap;
    uint32_t* bm = a.bitmap + (int64_t)q * a.nwords;
    uint32_t* sm = a.wsum + (int64_t)q * a.nsw;
    uint32_t tested = 0, passed = 0, sbt = 0;
    // a warp takes LPG listed leaves at a time -- chunks handed out dynamically by a per-query
    // counter to all warps of the query's blocks -- and screens their points packed 32 per step
    // (the owning leaf of packed point i found by a log2(LPG)-step search over the chunk's prefix)
    // per warp: queued sub-boxes (first point position, point count) that passed their bound
    // PF (tile mode): the queue is a FIFO ring; a passing sub-box's codes are prefetched into L2
    // when it is queued and its points are screened only after the next sub-box step (the code
    // loads were the top stall: 24 % of the samples on the point-screen line, ncu)
    constexpr bool PF = (BX & 2) != 0;
    constexpr int SQ = PF ? 128 : 64;
    __shared__ uint32_t s_sqf[LP_THREADS / 32][SQ];
    __shared__ uint8_t s_sqc[LP_THREADS / 32][SQ];
    uint32_t* sq_first = s_sqf[threadIdx.x >> 5];
    uint8_t* sq_cnt = s_sqc[threadIdx.x >> 5];
    uint32_t sqn = 0;                                // warp-uniform (PF: the ring's tail)
    uint32_t sqh = 0;                                // PF: the ring's head
    // screen the points of nb queued sub-boxes (the last nb; PF: the first nb): lane = (sub-box
    // lane / kSubBox, point)
    auto sb_points = [&](uint32_t nb) {
        const uint32_t sbs = lane / kSubBox, k = lane % kSubBox;
        if (sbs < nb) {
            const uint32_t e = PF ? ((sqh + sbs) & (SQ - 1)) : sqn - nb + sbs;
            if (k < sq_cnt[e]) {
                const uint32_t pos = sq_first[e] + k - (uint32_t)a.pos_base;
                uint32_t acc = 0;
                uint4 c4 = make_uint4(0, 0, 0, 0);
                if (K == 16) {
                    c4 = *reinterpret_cast<const uint4*>(a.tcodes + (int64_t)pos * 16);
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const uint32_t w = (j >> 2) == 0 ? c4.x : (j >> 2) == 1 ? c4.y : (j >> 2) == 2 ? c4.z : c4.w;
                        acc += s_e[j * N_r + ((w >> (8 * (j & 3))) & 255u)];
                    }
                } else {
                    for (int j = 0; j < K; ++j) acc += s_e[j * N_r + a.tcodes[(int64_t)pos * K + j]];
                }
                ++tested;
                if (acc <= 2048u) {                          // else: proves cellLB > rho^2
                    bool pass = acc + 17u <= 2048u;          // proves cellLB < rho^2 (1 - 1e-5)
                    if (!pass) {
                        float s_ = 0.f;
                        if (K == 16) {
#pragma unroll
                            for (int j = 0; j < 16; ++j) {
                                const uint32_t w = (j >> 2) == 0 ? c4.x : (j >> 2) == 1 ? c4.y : (j >> 2) == 2 ? c4.z : c4.w;
                                s_ += __ldg(s_d + j * N_r + ((w >> (8 * (j & 3))) & 255u));
                            }
                        } else {
                            for (int j = 0; j < K; ++j) s_ += __ldg(s_d + j * N_r + a.tcodes[(int64_t)pos * K + j]);
                        }
                        pass = s_ <= a.rho2;
                    }
                    if (pass) {
                        ++passed;
                        mark_member(bm, sm, a.perm[pos]);
                    }
                }
            }
        }
        if (PF) sqh += nb;
        else sqn -= nb;
        __syncwarp();
    };
    uint32_t lt = 0, lp = 0;                         // tile mode: leaf bounds evaluated / passed
    for (;;) {
        uint32_t ck = 0;     // ptake: the query's next untaken list entry (lists grow over a tree's chunks)
        // tile mode: two listed tiles per take (one atomic and both list loads in flight together)
        if (lane == 0) ck = atomicAdd(a.ptake + q, a.tile_leaf ? 2u : (uint32_t)LPG);
        const uint32_t e00 = __shfl_sync(0xffffffffu, ck, 0);
        if (e00 >= np) break;
        uint32_t Epre[2] = {0u, 0u};
        if (a.tile_leaf) {
            Epre[0] = pl[e00];
            if (e00 + 1 < np) Epre[1] = pl[e00 + 1];
        }
        for (int u = 0; u < (a.tile_leaf ? 2 : 1); ++u) {
        const uint32_t e0 = e00 + (uint32_t)u;
        if (e0 >= np) break;
        uint32_t my_p0 = 0, my_sz = 0;
        int64_t my_l = -1;
        if (a.tile_leaf) {
            const uint32_t E = Epre[u];
            uint32_t lb0, le0;
            if (a.tile_packed) {
                lb0 = E >> 5;
                le0 = lb0 + (E & 31u) + 1;
            } else {
                lb0 = a.tile_leaf[E];
                le0 = a.tile_leaf[E + 1];
            }
            if (lane < LPG && lb0 + lane < le0) my_l = lb0 + lane;
        } else if (lane < LPG && e0 + lane < np) {
            my_l = pl[e0 + lane];
        }
        if (my_l >= 0) {
            const uint32_t l = (uint32_t)my_l;
            my_p0 = a.leaf_off[l];
            my_sz = a.leaf_off[l + 1] - my_p0;
            // the leaf's box bound in the finer 12-bit table: the filter's 8-bit test passes
            // boxes up to ~12 % above rho^2; a sum > 2048 proves the box (hence every point of
            // the leaf) is beyond rho^2 -- the leaf's points are not screened
            uint32_t lb = 0;
            if (B16) {
                lb = box_bound16(s_e, s_qeo, s_qeo + 4, *reinterpret_cast<const uint4*>(a.lo + (int64_t)l * a.bs),
                                 *reinterpret_cast<const uint4*>(a.hi + (int64_t)l * a.bs));
            } else if (K == 16) {
                const uint4 lo4 = *reinterpret_cast<const uint4*>(a.lo + (int64_t)l * a.bs);
                const uint4 hi4 = *reinterpret_cast<const uint4*>(a.hi + (int64_t)l * a.bs);
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int sh = 8 * (j & 3);
                    const uint32_t wl = (j >> 2) == 0 ? lo4.x : (j >> 2) == 1 ? lo4.y : (j >> 2) == 2 ? lo4.z : lo4.w;
                    const uint32_t wh = (j >> 2) == 0 ? hi4.x : (j >> 2) == 1 ? hi4.y : (j >> 2) == 2 ? hi4.z : hi4.w;
                    const int c = min(max(s_qx[j], (int)((wl >> sh) & 255u)), (int)((wh >> sh) & 255u));
                    lb += s_e[j * N_r + c];
                }
            } else {
                for (int j = 0; j < K; ++j)
                    lb += s_e[j * N_r + min(max(s_qx[j], (int)a.lo[(int64_t)l * a.bs + j]), (int)a.hi[(int64_t)l * a.bs + j])];
            }
            if (lb > 2048u) my_sz = 0;
            ++lt;
            lp += my_sz != 0;
        }
        if (a.sb_off) {
            // second level: the leaves' sub-boxes (kSubBox consecutive points each), packed 32 per
            // step; each sub-box whose 12-bit bound is <= 2048 is queued, and 32 / kSubBox queued
            // sub-boxes' points are screened per step (lane = (sub-box, point))
            const uint32_t my_nsb = (my_sz + kSubBox - 1) / kSubBox;
            uint32_t my_sb0 = 0;
            if (my_l >= 0 && my_sz) my_sb0 = a.sb_off[my_l];
            uint32_t incl = my_nsb;
#pragma unroll
            for (int o = 1; o < LPG; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const uint32_t excl = incl - my_nsb;
            const uint32_t TS = __shfl_sync(0xffffffffu, incl, LPG - 1);
            const uint32_t my_end = my_p0 + my_sz;
            // software pipeline: the next 32 sub-boxes' boxes (one 32-byte row each: lo | hi) are
            // loaded before this step's bounds are computed (the loads were the top stall, ncu)
            auto locate = [&](uint32_t i, uint32_t& sbi, uint32_t& first, uint32_t& cnt) {
                int o_ = 0;                               // last leaf slot with excl <= i
#pragma unroll
                for (int st = LPG / 2; st > 0; st >>= 1) {
                    const uint32_t ex = __shfl_sync(0xffffffffu, excl, o_ + st);
                    if (ex <= i) o_ += st;
                }
                const uint32_t sb0 = __shfl_sync(0xffffffffu, my_sb0, o_);
                const uint32_t pp0 = __shfl_sync(0xffffffffu, my_p0, o_);
                const uint32_t pend = __shfl_sync(0xffffffffu, my_end, o_);
                const uint32_t pex = __shfl_sync(0xffffffffu, excl, o_);
                sbi = sb0 + (i - pex);
                first = pp0 + (i - pex) * kSubBox;
                cnt = min((uint32_t)kSubBox, pend - first);
                return i < TS;
            };
            uint4 nlo = make_uint4(0, 0, 0, 0), nhi = make_uint4(0, 0, 0, 0);
            uint32_t nsbi = 0, nfirst = 0, ncnt = 0;
            bool nvalid = locate(lane, nsbi, nfirst, ncnt);
            if (K == 16 && nvalid && LPG == 32) {
                nlo = *reinterpret_cast<const uint4*>(a.sb_lo + (int64_t)nsbi * 32);
                nhi = *reinterpret_cast<const uint4*>(a.sb_hi + (int64_t)nsbi * 32);
            }
            for (uint32_t c0 = 0; c0 < TS; c0 += 32) {
                const uint4 lo4p = nlo, hi4p = nhi;
                const uint32_t sbi = nsbi, first_c = nfirst, cnt_c = ncnt;
                const bool valid = nvalid;
                if (c0 + 32 < TS) {
                    nvalid = locate(c0 + 32 + lane, nsbi, nfirst, ncnt);
                    // prefetch only in the two-level filter's instantiation (LPG = 32, large n, where
                    // the boxes come from HBM); with LPG = 16 (L2-resident indexes) it cost occupancy
                    if (K == 16 && nvalid && LPG == 32) {
                        nlo = *reinterpret_cast<const uint4*>(a.sb_lo + (int64_t)nsbi * 32);
                        nhi = *reinterpret_cast<const uint4*>(a.sb_hi + (int64_t)nsbi * 32);
                    }
                }
                bool pass = false;
                uint32_t first = 0, cnt = 0;
                if (valid) {
                    first = first_c;
                    cnt = cnt_c;
                    uint32_t lb = 0;
                    if (B16) {
                        uint4 lo4 = lo4p, hi4 = hi4p;
                        if (LPG != 32) {
                            lo4 = *reinterpret_cast<const uint4*>(a.sb_lo + (int64_t)sbi * 32);
                            hi4 = *reinterpret_cast<const uint4*>(a.sb_hi + (int64_t)sbi * 32);
                        }
                        lb = box_bound16(s_e, s_qeo, s_qeo + 4, lo4, hi4);
                    } else if (K == 16) {
                        uint4 lo4 = lo4p, hi4 = hi4p;
                        if (LPG != 32) {
                            lo4 = *reinterpret_cast<const uint4*>(a.sb_lo + (int64_t)sbi * 32);
                            hi4 = *reinterpret_cast<const uint4*>(a.sb_hi + (int64_t)sbi * 32);
                        }
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const int sh = 8 * (j & 3);
                            const uint32_t wl = (j >> 2) == 0 ? lo4.x : (j >> 2) == 1 ? lo4.y : (j >> 2) == 2 ? lo4.z : lo4.w;
                            const uint32_t wh = (j >> 2) == 0 ? hi4.x : (j >> 2) == 1 ? hi4.y : (j >> 2) == 2 ? hi4.z : hi4.w;
                            const int c = min(max(s_qx[j], (int)((wl >> sh) & 255u)), (int)((wh >> sh) & 255u));
                            lb += s_e[j * N_r + c];
                        }
                    } else {
                        for (int j = 0; j < K; ++j)
                            lb += s_e[j * N_r + min(max(s_qx[j], (int)a.sb_lo[(int64_t)sbi * 2 * K + j]),
                                                    (int)a.sb_hi[(int64_t)sbi * 2 * K + j])];
                    }
                    pass = lb <= 2048u;
                    ++sbt;
                }
                const uint32_t bal = __ballot_sync(0xffffffffu, pass);
                if constexpr (PF) {
                    const uint32_t before = sqn;         // queued before this step: prefetched a step ago
                    if (pass) {
                        const uint32_t slot = (sqn + __popc(bal & lanemask_lt())) & (SQ - 1);
                        sq_first[slot] = first;
                        sq_cnt[slot] = (uint8_t)cnt;
                        const uint8_t* c0p = a.tcodes + (int64_t)(first - (uint32_t)a.pos_base) * 16;
                        if constexpr ((BX & 4) != 0) {   // into L1 (the SM's own cache)
                            asm volatile("prefetch.global.L1 [%0];" ::"l"(c0p));
                            asm volatile("prefetch.global.L1 [%0];" ::"l"(c0p + 16 * (cnt - 1)));
                        } else {
                            asm volatile("prefetch.global.L2 [%0];" ::"l"(c0p));
                            asm volatile("prefetch.global.L2 [%0];" ::"l"(c0p + 16 * (cnt - 1)));
                        }
                    }
                    sqn += __popc(bal);
                    __syncwarp();
                    while (before - sqh >= 32 / kSubBox) sb_points(32 / kSubBox);
                } else {
                    if (pass) {
                        const uint32_t slot = sqn + __popc(bal & lanemask_lt());
                        sq_first[slot] = first;
                        sq_cnt[slot] = (uint8_t)cnt;
                    }
                    sqn += __popc(bal);
                    __syncwarp();
                    while (sqn >= 32 / kSubBox) {
                        sb_points(32 / kSubBox);
                    }
                }
            }
            continue;
        }
        uint32_t incl = my_sz;
#pragma unroll
        for (int o = 1; o < LPG; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t excl = incl - my_sz;
        const uint32_t T = __shfl_sync(0xffffffffu, incl, LPG - 1);
        for (uint32_t c0 = 0; c0 < T; c0 += 32) {
            const uint32_t i = c0 + lane;
            int o_ = 0;                                   // last leaf slot with excl <= i
#pragma unroll
            for (int st = LPG / 2; st > 0; st >>= 1) {
                const uint32_t ex = __shfl_sync(0xffffffffu, excl, o_ + st);
                if (ex <= i) o_ += st;
            }
            const uint32_t pp0 = __shfl_sync(0xffffffffu, my_p0, o_);
            const uint32_t pex = __shfl_sync(0xffffffffu, excl, o_);
            if (i >= T) continue;
            const uint32_t p = pp0 + (i - pex);
            const int64_t pos = (int64_t)p - a.pos_base;
            uint32_t acc = 0;
            uint4 c4 = make_uint4(0, 0, 0, 0);
            if (K == 16) {
                c4 = *reinterpret_cast<const uint4*>(a.tcodes + pos * 16);
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const uint32_t w = (j >> 2) == 0 ? c4.x : (j >> 2) == 1 ? c4.y : (j >> 2) == 2 ? c4.z : c4.w;
                    acc += s_e[j * N_r + ((w >> (8 * (j & 3))) & 255u)];
                }
            } else {
                for (int j = 0; j < K; ++j) acc += s_e[j * N_r + a.tcodes[pos * K + j]];
            }
            ++tested;
            if (acc > 2048u) continue;                       // proves cellLB > rho^2
            bool pass = acc + 17u <= 2048u;                  // proves cellLB < rho^2 (1 - 1e-5)
            if (!pass) {
                float s_ = 0.f;
                if (K == 16) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const uint32_t w = (j >> 2) == 0 ? c4.x : (j >> 2) == 1 ? c4.y : (j >> 2) == 2 ? c4.z : c4.w;
                        s_ += __ldg(s_d + j * N_r + ((w >> (8 * (j & 3))) & 255u));
                    }
                } else {
                    for (int j = 0; j < K; ++j) s_ += __ldg(s_d + j * N_r + a.tcodes[pos * K + j]);
                }
                pass = s_ <= a.rho2;
            }
            if (pass) {
                ++passed;
                const uint32_t id = a.perm[pos];
                mark_member(bm, sm, id);
            }
        }
    }   // tiles of this take
    }   // takes
    if constexpr (PF) {
        while (sqn - sqh >= 32 / kSubBox) sb_points(32 / kSubBox);
        if (sqn != sqh) sb_points(sqn - sqh);
    } else {
        if (sqn) sb_points(sqn);
    }
    for (int o = 16; o > 0; o >>= 1) {
        tested += __shfl_xor_sync(0xffffffffu, tested, o);
        passed += __shfl_xor_sync(0xffffffffu, passed, o);
        sbt += __shfl_xor_sync(0xffffffffu, sbt, o);
        lt += __shfl_xor_sync(0xffffffffu, lt, o);
        lp += __shfl_xor_sync(0xffffffffu, lp, o);
    }
    if (a.tile_leaf && lane == 0 && lt) {
        atomicAdd(a.ctr + (int64_t)q * NCTR + 0, (unsigned long long)lt);
        atomicAdd(a.ctr + (int64_t)q * NCTR + 1, (unsigned long long)lp);
    }
    if (lane == 0) { atomicAdd(&s_tested, tested); atomicAdd(&s_passed, passed); if (sbt) atomicAdd(&s_sbt, sbt); }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s_passed) atomicAdd(reinterpret_cast<unsigned long long*>(&a.qs_mut[q].pub), (unsigned long long)s_passed);
        atomicAdd(a.ctr + (int64_t)q * NCTR + 2, (unsigned long long)s_tested);
        atomicAdd(a.ctr + (int64_t)q * NCTR + 3, (unsigned long long)s_passed);
        if (s_sbt) atomicAdd(a.ctr + (int64_t)q * NCTR + 4, (unsigned long long)s_sbt);
    }
}

// One pass over the listed pairs is done: the lists restart empty for the next tree.
// After tree t: |S| += number of bits set now but not in `prev` (the first-time members of
// S <- S u S_i, Alg. 5 line 6), and `prev` catches up.  Grid: (active queries) x (word chunks).
// Only the words flagged in the row's dirty-word summary can hold members: thread per summary
// word (32 bitmap words), 256 per block.
constexpr int CN_SW = 256;
__global__ void __launch_bounds__(256) k_count_new(const int* __restrict__ act, const int* __restrict__ dna,
                                                   QState* __restrict__ qs, const uint32_t* __restrict__ cur,
                                                   uint32_t* __restrict__ prev, int64_t nwords,
                                                   const uint32_t* __restrict__ wsum, int64_t nsw, int commit) {
    pdl_wait();
    __shared__ unsigned int s_cnt;
    if (dna && (int)blockIdx.x >= *dna) return;
    const int q = act[blockIdx.x];
    if (qs[q].status != ST_ACTIVE) return;
    if (commit && !qs[q].doc) return;      // |S| cannot have reached the budget: counted later
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    const uint32_t* c = cur + (int64_t)q * nwords;
    uint32_t* p = prev + (int64_t)q * nwords;
    const int64_t sw = (int64_t)blockIdx.y * CN_SW + threadIdx.x;
    uint32_t cnt = 0;
    if (sw < nsw) {
        for (uint32_t dm = wsum[(int64_t)q * nsw + sw]; dm; dm &= dm - 1) {
            const int64_t w = sw * 32 + (__ffs(dm) - 1);
            const uint32_t cv = c[w], pv = p[w];
            const uint32_t nb = cv & ~pv;
            if (nb) {
                if (commit) p[w] = cv;
                cnt += __popc(nb);
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&s_cnt, cnt);
    __syncthreads();
    if (threadIdx.x == 0 && s_cnt)   // committed: |S| grows; tentative (lb_order): counted into tnew
        atomicAdd(reinterpret_cast<unsigned long long*>(commit ? &qs[q].cnt : &qs[q].tnew), (unsigned long long)s_cnt);
}

// ---- Sec. 6.2.2(2): leaves in ascending (LB, leaf) order, budget per leaf.
//      Only queries whose tree-t candidates would cross the budget need it (for the others the
//      order cannot change S):
//   k_lbo_cross   queries with |S| + tentative first-time members >= budget (compacted list)
//   k_lbo_leaves  per (crossing query, leaf of tree t): the leaf's fp32 lower bound (j order) as a
//                 sort key (0xFFFFFFFF when above eps r) and its number of first-time members
//   (segmented radix sort of the keys, values = leaf positions: ties by leaf position)
//   k_lbo_cut     the first leaf in that order at which |S| reaches the budget
//   k_lbo_reset   S <- S before tree t (the prev bitmap)
//   k_lbo_mark    the members of leaves up to the cut, marked again
__global__ void k_lbo_cross(const int* __restrict__ act, int na_ub, const int* __restrict__ dna,
                            const QState* __restrict__ qs, int64_t budget, int* __restrict__ cross,
                            int* __restrict__ ncross) {
    pdl_wait();
    const int na = dna ? *dna : na_ub;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < na; i += gridDim.x * blockDim.x) {
        const int q = act[i];
        const QState s = qs[q];
        if (s.status == ST_ACTIVE && s.cnt + s.tnew >= budget) cross[atomicAdd(ncross, 1)] = q;
    }
}

struct LboArgs {
    const int* cross;
    const float* lut;           // [Qb][L][K][N_r] fp32
    const uint8_t* sx;          // [Qb][L][K]
    const uint8_t* lo;          // tree t leaves [nl_t][K]
    const uint8_t* hi;
    const uint32_t* leaf_off;   // tree t leaves, global positions [nl_t + 1]
    const uint8_t* tcodes;      // tree t [n][K]
    const uint32_t* perm;       // tree t [n]
    const float* proj;          // EXACT
    const float* qp;            // EXACT: [Qb][LK]
    const uint32_t* prev;       // S before tree t
    uint32_t* cur;
    int64_t nwords, pos_base, nl;
    float rho2;
    int t, L, K, N_r, mode;
    uint32_t* keys;             // [ncross][nl]
    uint32_t* vals;             // [ncross][nl] leaf positions
    uint32_t* nnew;             // [ncross][nl]
    const unsigned long long* cut;   // [ncross] (key << 32 | leaf): mark leaves <= cut
};

template <bool MARK>
__global__ void __launch_bounds__(256) k_lbo_leaves(LboArgs a) {
    pdl_wait();
    extern __shared__ float s_lut[];                   // the query's fp32 table of tree t
    const int c = blockIdx.y;
    const int q = a.cross[c];
    const int K = a.K, N_r = a.N_r;
    const float* src = a.lut + ((int64_t)q * a.L + a.t) * K * N_r;
    for (int i = threadIdx.x; i < K * N_r; i += blockDim.x) s_lut[i] = src[i];
    __syncthreads();
    const uint8_t* sx = a.sx + ((int64_t)q * a.L + a.t) * K;
    const float* qpt = a.qp ? a.qp + (int64_t)q * a.L * K + a.t * K : nullptr;
    const int lane = threadIdx.x & 31;
    const uint32_t* pv = a.prev + (int64_t)q * a.nwords;
    uint32_t* cv = a.cur + (int64_t)q * a.nwords;
    const unsigned long long cut = MARK ? a.cut[c] : 0ull;
    for (int64_t l = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); l < a.nl; l += (int64_t)gridDim.x * 8) {
        float lb = 0.f;                                  // leaf LB, j order (as RELAXED's leaf test)
        for (int j = 0; j < K; ++j)
            lb += s_lut[j * N_r + min(max((int)sx[j], (int)a.lo[l * K + j]), (int)a.hi[l * K + j])];
        const uint32_t key = lb <= a.rho2 ? __float_as_uint(lb) : 0xFFFFFFFFu;
        if (MARK && (key == 0xFFFFFFFFu || (((unsigned long long)key << 32) | (unsigned long long)l) > cut)) continue;
        if (!MARK && key == 0xFFFFFFFFu) {
            if (lane == 0) { a.keys[(int64_t)c * a.nl + l] = key; a.vals[(int64_t)c * a.nl + l] = (uint32_t)l; a.nnew[(int64_t)c * a.nl + l] = 0; }
            continue;
        }
        uint32_t cnt = 0;
        for (uint32_t p = a.leaf_off[l] + lane; p < a.leaf_off[l + 1]; p += 32) {
            const int64_t pos = (int64_t)p - a.pos_base;
            bool pass = true;
            if (a.mode == DETLSH_MODE_CELL) {
                float s_ = 0.f;
                for (int j = 0; j < K; ++j) s_ += s_lut[j * N_r + a.tcodes[pos * K + j]];
                pass = s_ <= a.rho2;
            } else if (a.mode == DETLSH_MODE_EXACT) {
                const float* pp = a.proj + (int64_t)a.perm[pos] * a.L * K + a.t * K;
                float s_ = 0.f;
                for (int j = 0; j < K; ++j) {
                    const float df = qpt[j] - pp[j];
                    s_ = fmaf(df, df, s_);
                }
                pass = s_ <= a.rho2;
            }
            if (!pass) continue;
            const uint32_t id = a.perm[pos];
            if (MARK) {
                atomicOr(cv + (id >> 5), 1u << (id & 31));
            } else if (!((pv[id >> 5] >> (id & 31)) & 1u)) {
                ++cnt;
            }
        }
        if (!MARK) {
            for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
            if (lane == 0) {
                a.keys[(int64_t)c * a.nl + l] = key;
                a.vals[(int64_t)c * a.nl + l] = (uint32_t)l;
                a.nnew[(int64_t)c * a.nl + l] = cnt;
            }
        }
    }
}

__global__ void __launch_bounds__(1024) k_lbo_cut(const int* __restrict__ cross, const QState* __restrict__ qs,
                                                  int64_t budget, const uint32_t* __restrict__ skeys,
                                                  const uint32_t* __restrict__ svals, const uint32_t* __restrict__ nnew,
                                                  int64_t nl, unsigned long long* __restrict__ cut) {
    pdl_wait();
    __shared__ uint32_t s_w[32];
    __shared__ int64_t s_hit;
    const int c = blockIdx.x;
    const int q = cross[c];
    const int64_t need = budget - qs[q].cnt;            // > 0 (the query is still active)
    const uint32_t* k_ = skeys + (int64_t)c * nl;
    const uint32_t* v_ = svals + (int64_t)c * nl;
    const uint32_t* w_ = nnew + (int64_t)c * nl;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_hit = -1;
    int64_t carry = 0;
    for (int64_t b0 = 0; b0 < nl; b0 += 1024) {
        const int64_t b = b0 + threadIdx.x;
        const uint32_t x0 = b < nl ? w_[v_[b]] : 0u;
        uint32_t x = x0;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_w[w] = x;
        __syncthreads();
        if (w == 0) {
            uint32_t t = s_w[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += y;
            }
            s_w[lane] = t;
        }
        __syncthreads();
        const int64_t incl = carry + x + (w ? s_w[w - 1] : 0);
        if (b < nl && incl >= need && incl - x0 < need) s_hit = b;   // unique crossing rank
        carry += s_w[31];
        __syncthreads();
        if (s_hit >= 0) break;
    }
    if (threadIdx.x == 0) {
        const int64_t h = s_hit >= 0 ? s_hit : nl - 1;
        cut[c] = ((unsigned long long)k_[h] << 32) | (unsigned long long)v_[h];
    }
}

__global__ void k_lbo_reset(const int* __restrict__ cross, int ncross, const uint32_t* __restrict__ prev,
                            uint32_t* __restrict__ cur, int64_t nwords) {
    pdl_wait();
    const int64_t total = (int64_t)ncross * nwords;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = i / nwords, w = i - c * nwords;
        const int64_t o = (int64_t)cross[c] * nwords + w;
        cur[o] = prev[o];
    }
}

// Before counting |S| after a tree: the bitmap diff is needed only if the budget may have been
// reached (|S| <= cnt + marks since the last count) or the count is due (force: end of round,
// or lb_order, which needs |S| exact after every tree).
// (pcnt != null: also resets the pair-list lengths and take counters of the tree just filtered.)
__global__ void k_count_decide(const int* __restrict__ act, int na_ub, const int* __restrict__ dna,
                               QState* __restrict__ qs, int64_t budget, int force, uint32_t* __restrict__ pcnt,
                               uint32_t* __restrict__ ptake) {
    pdl_wait();
    const int na = dna ? *dna : na_ub;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < na; i += gridDim.x * blockDim.x) {
        if (pcnt) { pcnt[act[i]] = 0; ptake[act[i]] = 0; }
        QState* s = &qs[act[i]];
        const int d = (s->status == ST_ACTIVE && s->pub > 0 && (force || s->cnt + s->pub >= budget)) ? 1 : 0;
        s->doc = d;
        if (d) s->pub = 0;
    }
}

// After tree t: the budget test |S| >= ceil(beta n) + k (Alg. 5 line 7, AMB-15/17).
__device__ inline void tree_end_one(QState* s, int t, int round, int64_t budget, int64_t cap) {
    if (s->status != ST_ACTIVE) return;
    s->trees_last = t + 1;
    s->rounds = round + 1;
    s->tnew = 0;
    if (s->cnt > cap) s->overflow = 1;
    if (s->cnt >= budget) s->status = ST_BUDGET;
}

__global__ void k_tree_end(const int* __restrict__ act, int na_ub, const int* __restrict__ dna, QState* __restrict__ qs,
                           int t, int round, int64_t budget, int64_t cap) {
    pdl_wait();
    const int na = dna ? *dna : na_ub;
    for (int a_ = blockIdx.x * blockDim.x + threadIdx.x; a_ < na; a_ += gridDim.x * blockDim.x)
        tree_end_one(&qs[act[a_]], t, round, budget, cap);
}

// k_tree_end and then the order-preserving compaction of the still-active queries (single
// block; each query is updated and tested by the one thread that owns its slot).
__global__ void k_tree_end_compact(const int* __restrict__ act, int na_ub, const int* __restrict__ dna,
                                   QState* __restrict__ qs, int t, int round, int64_t budget, int64_t cap,
                                   int* __restrict__ act_out, int* __restrict__ n_out) {
    pdl_wait();
    const int na = dna ? *dna : na_ub;
    __shared__ int s_n;
    __shared__ int s_w[32];
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int base = 0; base < na; base += blockDim.x) {
        const int a = base + threadIdx.x;
        bool keep = false;
        if (a < na) {
            QState* s = &qs[act[a]];
            tree_end_one(s, t, round, budget, cap);
            keep = s->status == ST_ACTIVE;
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) s_w[w] = __popc(bal);
        __syncthreads();
        if (threadIdx.x == 0) {
            int run = s_n;
            for (int i = 0; i < (int)(blockDim.x / 32); ++i) { const int c = s_w[i]; s_w[i] = run; run += c; }
            s_n = run;
        }
        __syncthreads();
        if (keep) act_out[s_w[w] + __popc(bal & lanemask_lt())] = act[a];
        __syncthreads();
    }
    if (threadIdx.x == 0) *n_out = s_n;
}

// After tree t, everything per query in one launch (block = query of the tree's list): the lazy
// count decision (k_count_decide), the bitmap diff over the summary-flagged words when needed
// (k_count_new), the pair-list reset and the budget test (k_tree_end); the last block to finish
// (ticket counter) then compacts the still-active queries for the next tree (k_tree_end_compact).
// act_out == null: no compaction (last tree).  Not for lb_order (its counts are tentative).
// Visit the flagged words of one dirty-word summary row (bit b of summary word sw = bitmap word
// 32 sw + b): 16-byte summary loads, four of them in flight per thread (a 100M-point row is 98K
// summary words, mostly zero -- a one-word-per-thread loop was latency-bound).  nsw is a
// multiple of 4 and rows are 16-byte aligned.
template <class F>
__device__ __forceinline__ void for_each_dirty_word(const uint32_t* __restrict__ sm_row, int64_t nsw, F&& f) {
    const uint4* s4 = reinterpret_cast<const uint4*>(sm_row);
    const int64_t n4 = nsw >> 2;
    for (int64_t i0 = threadIdx.x; i0 < n4; i0 += 4 * (int64_t)blockDim.x) {
        uint4 w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = i0 + u * (int64_t)blockDim.x;
            w[u] = i < n4 ? s4[i] : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if ((w[u].x | w[u].y | w[u].z | w[u].w) == 0) continue;
            const int64_t i = i0 + u * (int64_t)blockDim.x;
            const uint32_t ws[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
#pragma unroll
            for (int k = 0; k < 4; ++k)
                for (uint32_t dm = ws[k]; dm; dm &= dm - 1) f((4 * i + k) * 32 + (__ffs(dm) - 1));
        }
    }
}

__global__ void __launch_bounds__(256) k_tree_post(const int* __restrict__ act, int na_ub, const int* __restrict__ dna,
                                                   QState* __restrict__ qs, const uint32_t* __restrict__ cur,
                                                   uint32_t* __restrict__ prev, int64_t nwords,
                                                   const uint32_t* __restrict__ wsum, int64_t nsw, int64_t budget,
                                                   int force, uint32_t* __restrict__ pcnt, uint32_t* __restrict__ ptake,
                                                   int t, int round, int64_t cap, unsigned int* __restrict__ ticket,
                                                   int* __restrict__ act_out, int* __restrict__ n_out,
                                                   unsigned long long* __restrict__ total) {
    pdl_wait();
    // total != null: end of round instead -- every count forced, no budget test, and the last
    // block lays out the round-buffer slots [roff, roff + rcnt) instead of compacting
    __shared__ unsigned int s_cnt, s_last;
    __shared__ int s_doc;
    const int na = dna ? *dna : na_ub;
    const int a = blockIdx.x;
    if (a < na) {
        const int q = act[a];
        QState* s = &qs[q];
        if (threadIdx.x == 0) {
            if (pcnt) { pcnt[q] = 0; ptake[q] = 0; }
            const int d = (s->status == ST_ACTIVE && s->pub > 0 && (force || s->cnt + s->pub >= budget)) ? 1 : 0;
            s_doc = d;
            s_cnt = 0;
            if (d) s->pub = 0;
        }
        __syncthreads();
        if (s_doc) {
            const uint32_t* c = cur + (int64_t)q * nwords;
            uint32_t* pv = prev + (int64_t)q * nwords;
            uint32_t cnt = 0;
            for_each_dirty_word(wsum + (int64_t)q * nsw, nsw, [&](int64_t w) {
                const uint32_t cv = c[w], pw = pv[w];
                const uint32_t nb = cv & ~pw;
                if (nb) {
                    pv[w] = cv;
                    cnt += __popc(nb);
                }
            });
            for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
            if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&s_cnt, cnt);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            if (s_cnt) s->cnt += s_cnt;
            if (!total) tree_end_one(s, t, round, budget, cap);
        }
    }
    if (!act_out && !total) return;
    // last block: order-preserving compaction of the still-active queries
    __threadfence();
    if (threadIdx.x == 0) s_last = (atomicAdd(ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (total) {   // round-buffer slots: exclusive prefix of (|S| - verified) over the round's queries
        __shared__ unsigned long long s_wl[8];
        __shared__ unsigned long long s_run;
        if (threadIdx.x == 0) s_run = 0;
        __syncthreads();
        for (int base = 0; base < na; base += blockDim.x) {
            const int i = base + threadIdx.x;
            unsigned long long c = 0;
            if (i < na) {
                const volatile QState* vs = (volatile const QState*)&qs[act[i]];
                c = (unsigned long long)(vs->cnt - vs->nver);
            }
            unsigned long long x = c;
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) s_wl[w] = x;
            __syncthreads();
            unsigned long long before = s_run;
            for (int k = 0; k < w; ++k) before += s_wl[k];
            if (i < na) {
                QState* s2 = &qs[act[i]];
                s2->roff = (int64_t)(before + x - c);
                s2->rcnt = (int64_t)c;
            }
            __syncthreads();
            if (threadIdx.x == blockDim.x - 1) s_run = before + x;
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            *total = s_run;
            *ticket = 0;
        }
        return;
    }
    __shared__ int s_n;
    __shared__ int s_w[8];
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    for (int base = 0; base < na; base += blockDim.x) {
        const int i = base + threadIdx.x;
        const bool keep = i < na && ((volatile const QState*)qs)[act[i]].status == ST_ACTIVE;
        const uint32_t bal = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) s_w[w] = __popc(bal);
        __syncthreads();
        if (threadIdx.x == 0) {
            int run = s_n;
            for (int k = 0; k < (int)(blockDim.x / 32); ++k) { const int c_ = s_w[k]; s_w[k] = run; run += c_; }
            s_n = run;
        }
        __syncthreads();
        if (keep) act_out[s_w[w] + __popc(bal & lanemask_lt())] = act[i];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *n_out = s_n;
        *ticket = 0;                                  // ready for the next tree
    }
}


// ---- verify (Alg. 5 lines 8/10): exact squared L2 of every member of S not yet verified,
//      row-blocked: a CTA stages a block of consecutive data rows in shared memory once and
//      serves every active query whose new candidates fall in that block (each row is a
//      candidate of ~beta of all queries), one warp per (block, query): float4 reads of the
//      staged rows, the query in registers, warp-shuffle reduction; (id, d2) appended to the
//      query's list.  new = S \ verified is read from the bitmaps (cur & ~ver).
constexpr int VR_THREADS = 512;

struct VRArgs {
    const float* X;
    int64_t ld, n;
    const float* Q;          // batch queries [Qb][ld]
    const int* act;
    int na;
    QState* qs;
    const uint32_t* cur;
    uint32_t* ver;
    int64_t nwords;
    uint32_t* cand;          // round buffer: ids
    float* d2;               // round buffer: squared distances
    const uint32_t* boff;    // [na][nblocks] slot of each (query, block) in the round buffer
    int64_t nblocks;
    int rbw;                 // bitmap words (32 rows each) per block
};

// Per (active query, row block): where its new candidates go in the round buffer -- the
// query's round offset plus the number of new members of S in earlier blocks (an exclusive
// scan of popcounts of cur & ~ver), so the verify kernel appends without atomics.
__global__ void __launch_bounds__(1024) k_verify_offsets(const int* __restrict__ act, const QState* __restrict__ qs,
                                                         const uint32_t* __restrict__ cur, const uint32_t* __restrict__ ver,
                                                         int64_t nwords, int rbw, int64_t nblocks,
                                                         uint32_t* __restrict__ boff) {
    pdl_wait();
    __shared__ uint32_t s_w[32];
    const int q = act[blockIdx.x];
    const uint32_t* c = cur + (int64_t)q * nwords;
    const uint32_t* v = ver + (int64_t)q * nwords;
    uint32_t* out = boff + (int64_t)blockIdx.x * nblocks;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t carry = (uint32_t)qs[q].roff;
    for (int64_t b0 = 0; b0 < nblocks; b0 += 1024) {
        const int64_t b = b0 + threadIdx.x;
        uint32_t cnt = 0;
        if (b < nblocks)
            for (int i = 0; i < rbw; ++i) {
                const int64_t wd = b * rbw + i;
                if (wd < nwords) cnt += __popc(c[wd] & ~v[wd]);
            }
        uint32_t x = cnt;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_w[w] = x;
        __syncthreads();
        if (w == 0) {
            uint32_t t = s_w[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += y;
            }
            s_w[lane] = t;
        }
        __syncthreads();
        const uint32_t incl = x + (w ? s_w[w - 1] : 0);
        if (b < nblocks) out[b] = carry + incl - cnt;
        carry += s_w[31];
        __syncthreads();
    }
}

// Each warp serves one query at a time: its 32 lanes form 4 row slots of 8 lanes; a slot
// computes one candidate's distance, each lane a strided eighth of the row (float4 reads of
// the staged row, the query's matching eighth held in registers), packed fp32x2 arithmetic,
// a 3-step shuffle reduction inside the slot.  NV = float4 per lane (ld/4 = 8*NV at most;
// NV = 0: rows wider than 256 fp32, the query is re-read from L1/L2).
template <int NV, bool EXACT>
__global__ void __launch_bounds__(VR_THREADS) k_verify_rows(VRArgs a) {
    pdl_wait();
    extern __shared__ __align__(16) float4 s_rows[];
    __shared__ uint8_t s_list[VR_THREADS / 32][256];     // per warp: rows (in block) of the new bits
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = VR_THREADS / 32;
    const int slot = lane >> 3, u = lane & 7;
    const int nf4 = EXACT ? 8 * NV : (int)(a.ld / 4);
    const int64_t w0 = (int64_t)blockIdx.x * a.rbw;
    const int64_t row0 = w0 * 32;
    const int RB = a.rbw * 32;
    const float4* X4 = reinterpret_cast<const float4*>(a.X);
    for (int i = threadIdx.x; i < RB * nf4; i += VR_THREADS) {
        const int r = i / nf4, f = i - r * nf4;
        const int64_t row = row0 + r;
        s_rows[i] = row < a.n ? __ldg(X4 + row * nf4 + f) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    const float4* Q4 = reinterpret_cast<const float4*>(a.Q);
    uint8_t* lst = s_list[warp];
    for (int ai = warp; ai < a.na; ai += nwarps) {
        const int q = a.act[ai];
        // -q, the lane's eighth, as fp32x2 pairs (issued first: its latency overlaps the masks)
        float2 nq[NV ? 2 * NV : 2];
        if (NV) {
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const int f = u + 8 * v;
                const float4 y = (EXACT || f < nf4) ? Q4[(int64_t)q * nf4 + f] : make_float4(0.f, 0.f, 0.f, 0.f);
                nq[2 * v] = make_float2(-y.x, -y.y);
                nq[2 * v + 1] = make_float2(-y.z, -y.w);
            }
        }
        uint32_t mw = 0;
        if (lane < a.rbw) {
            const int64_t w = w0 + lane;
            if (w < a.nwords) {
                uint32_t* vp = a.ver + (int64_t)q * a.nwords + w;
                const uint32_t c = a.cur[(int64_t)q * a.nwords + w];
                mw = c & ~*vp;
                if (mw) *vp = c;
            }
        }
        // rows of the new bits, in order, into the warp's list
        const uint32_t pc = __popc(mw);
        uint32_t incl = pc;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t tot = __shfl_sync(0xffffffffu, incl, 7);
        if (tot == 0) continue;
        const uint32_t base = a.boff[(int64_t)ai * a.nblocks + blockIdx.x];
        {
            uint32_t m = mw, p = incl - pc;
            while (m) {
                lst[p++] = (uint8_t)(lane * 32 + __ffs(m) - 1);
                m &= m - 1;
            }
        }
        __syncwarp();
        const int64_t out = (int64_t)base;
        uint32_t* cl = a.cand;
        float* dl = a.d2;
        for (uint32_t i = 0; i < tot; i += 4) {
            const bool valid = i + slot < tot;
            const int r = lst[valid ? i + slot : i];
            const float4* row = s_rows + r * nf4;
            float2 acc = make_float2(0.f, 0.f);
            if (NV) {
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const int f = u + 8 * v;
                    if (EXACT || f < nf4) {
                        const float4 x = row[f];
                        const float2 d0 = __fadd2_rn(make_float2(x.x, x.y), nq[2 * v]);
                        const float2 d1 = __fadd2_rn(make_float2(x.z, x.w), nq[2 * v + 1]);
                        acc = __ffma2_rn(d0, d0, acc);
                        acc = __ffma2_rn(d1, d1, acc);
                    }
                }
            } else {
                for (int f = u; f < nf4; f += 8) {
                    const float4 x = row[f], y = Q4[(int64_t)q * nf4 + f];
                    const float2 d0 = make_float2(x.x - y.x, x.y - y.y), d1 = make_float2(x.z - y.z, x.w - y.w);
                    acc = __ffma2_rn(d0, d0, acc);
                    acc = __ffma2_rn(d1, d1, acc);
                }
            }
            float s_ = acc.x + acc.y;
            s_ += __shfl_xor_sync(0xffffffffu, s_, 1);
            s_ += __shfl_xor_sync(0xffffffffu, s_, 2);
            s_ += __shfl_xor_sync(0xffffffffu, s_, 4);
            if (valid && u == 0) {
                cl[out + i + slot] = (uint32_t)(row0 + r);
                dl[out + i + slot] = s_;
            }
        }
        __syncwarp();
    }
}

// ---- tensor-core verification inputs (verify_tc.cu), per round:
//  k_verify_prep   per active query a: NB[a][w] = cur & ~ver (the new members of S in word w),
//                  BO[a][w] = the query's round offset + new members in earlier words (a block
//                  scan), and ver catches up with cur.
//  k_prep_queries  the active queries as a contiguous [na][ld] fp32 block, its TF32 residual
//                  q - trunc_tf32(q), and ||q||^2.
__global__ void __launch_bounds__(1024) k_verify_prep(const int* __restrict__ act, const QState* __restrict__ qs,
                                                      const uint32_t* __restrict__ cur, uint32_t* __restrict__ ver,
                                                      int64_t nwords, uint32_t* __restrict__ NB,
                                                      uint32_t* __restrict__ BO) {
    pdl_wait();
    // nwords is a multiple of 4 (padded bitmap rows): each thread owns 4 consecutive words
    __shared__ uint32_t s_w[32];
    const int a = blockIdx.x;
    const int q = act[a];
    const uint4* c = reinterpret_cast<const uint4*>(cur + (int64_t)q * nwords);
    uint4* v = reinterpret_cast<uint4*>(ver + (int64_t)q * nwords);
    uint4* nb_out = reinterpret_cast<uint4*>(NB + (int64_t)a * nwords);
    uint4* bo_out = reinterpret_cast<uint4*>(BO + (int64_t)a * nwords);
    const int64_t n4 = nwords / 4;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t carry = (uint32_t)qs[q].roff;
    for (int64_t b0 = 0; b0 < n4; b0 += 1024) {
        const int64_t b = b0 + threadIdx.x;
        uint4 nb = make_uint4(0, 0, 0, 0);
        if (b < n4) {
            const uint4 cv = c[b], vv = v[b];
            nb = make_uint4(cv.x & ~vv.x, cv.y & ~vv.y, cv.z & ~vv.z, cv.w & ~vv.w);
            if (nb.x | nb.y | nb.z | nb.w) v[b] = cv;
        }
        const uint32_t c0 = __popc(nb.x), c1 = __popc(nb.y), c2 = __popc(nb.z), c3 = __popc(nb.w);
        const uint32_t cnt = c0 + c1 + c2 + c3;
        uint32_t x = cnt;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_w[w] = x;
        __syncthreads();
        if (w == 0) {
            uint32_t t = s_w[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += y;
            }
            s_w[lane] = t;
        }
        __syncthreads();
        const uint32_t ex = carry + x + (w ? s_w[w - 1] : 0) - cnt;
        if (b < n4) {
            nb_out[b] = nb;
            bo_out[b] = make_uint4(ex, ex + c0, ex + c0 + c1, ex + c0 + c1 + c2);
        }
        carry += s_w[31];
        __syncthreads();
    }
}

// Sparse verification listing: the new members of S (cur & ~ver) of active query a, found through
// the row's dirty-word summary (only words that hold members are read), written as (candidate id,
// active-query index) at the query's round-buffer slots [roff, roff + rcnt) -- their order within
// the range is free (the top-k ranks by (d2, id)), so a word's run of slots comes from a shared
// counter; ver catches up with cur.  Block per query.
__global__ void __launch_bounds__(256) k_verify_list(const int* __restrict__ act, const QState* __restrict__ qs,
                                                     const uint32_t* __restrict__ cur, uint32_t* __restrict__ ver,
                                                     int64_t nwords, const uint32_t* __restrict__ wsum, int64_t nsw,
                                                     uint32_t* __restrict__ cand, uint32_t* __restrict__ cq) {
    pdl_wait();
    __shared__ unsigned long long s_slot;             // 64-bit slots: a round may hold >= 2^32 pairs
    const int a = blockIdx.x;
    const int q = act[a];
    if (threadIdx.x == 0) s_slot = (unsigned long long)qs[q].roff;
    __syncthreads();
    const uint32_t* c = cur + (int64_t)q * nwords;
    uint32_t* v = ver + (int64_t)q * nwords;
    const uint32_t* sm = wsum + (int64_t)q * nsw;
    for_each_dirty_word(sm, nsw, [&](int64_t wd) {
        const uint32_t cv = c[wd];
        uint32_t nb = cv & ~v[wd];
        if (!nb) return;
        v[wd] = cv;
        unsigned long long slot = atomicAdd(&s_slot, (unsigned long long)__popc(nb));
        const uint32_t base = (uint32_t)(wd * 32);
        for (; nb; nb &= nb - 1) {
            cand[slot] = base + (uint32_t)(__ffs(nb) - 1);
            cq[slot] = (uint32_t)a;
            ++slot;
        }
    });
}

__global__ void k_prep_queries(const float* __restrict__ Q, int64_t ld, const int* __restrict__ act, int na,
                               float* __restrict__ Qa, float* __restrict__ Qalo, float* __restrict__ qn) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    for (int a = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); a < na; a += gridDim.x * (blockDim.x >> 5)) {
        const float* src = Q + (int64_t)act[a] * ld;
        float acc = 0.f;
        for (int64_t i = lane; i < ld; i += 32) {
            const float x = src[i];
            Qa[(int64_t)a * ld + i] = x;
            Qalo[(int64_t)a * ld + i] = x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
            acc = fmaf(x, x, acc);
        }
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) qn[a] = acc;
    }
}

// ---- top-k merge + termination test
constexpr int TK_THREADS = 512;
constexpr int TK_MAX = 4096;

__device__ inline unsigned long long mkkey(float d2, uint32_t id) {
    return ((unsigned long long)__float_as_uint(d2) << 32) | id;
}

__device__ void bitonic_sort_smem(unsigned long long* a, int n2) {
    for (int k = 2; k <= n2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n2; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const bool up = (i & k) == 0;
                    const unsigned long long x = a[i], y = a[ixj];
                    if ((x > y) == up) { a[i] = y; a[ixj] = x; }
                }
            }
            __syncthreads();
        }
    }
}

// ---- sparse verification (low candidate density): k_verify_list lists the new members
//      of S at their round-buffer slots, then one 8-lane group per candidate gathers its row
//      with float4 loads (k_verify_gather): per candidate 4d bytes of X, no per-(row block,
//      query) work.
// NV > 0: the row is NV float4 per lane (ld = 32 NV), all loads issued before any arithmetic
// (memory-level parallelism of a whole 4d-byte row per 8 lanes); NV = 0: any ld.
template <int NV>
__global__ void __launch_bounds__(256) k_verify_gather(const uint32_t* __restrict__ cand, const uint32_t* __restrict__ cq,
                                                       const int* __restrict__ act, const float* __restrict__ X,
                                                       const float* __restrict__ Q, int64_t ld, int64_t total,
                                                       float* __restrict__ d2) {
    pdl_wait();
    const int u = threadIdx.x & 7;
    const int nf4 = (int)(ld / 4);
    for (int64_t slot = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 3; slot < total;
         slot += ((int64_t)gridDim.x * blockDim.x) >> 3) {
        const float4* x4 = reinterpret_cast<const float4*>(X + (int64_t)cand[slot] * ld);
        const float4* q4 = reinterpret_cast<const float4*>(Q + (int64_t)act[cq[slot]] * ld);
        float2 acc = make_float2(0.f, 0.f);
        if (NV > 0) {
            float4 x[NV > 0 ? NV : 1], y[NV > 0 ? NV : 1];
#pragma unroll
            for (int v = 0; v < NV; ++v) x[v] = __ldcs(x4 + u + 8 * v);      // streamed: read once
#pragma unroll
            for (int v = 0; v < NV; ++v) y[v] = __ldg(q4 + u + 8 * v);
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const float2 e0 = make_float2(x[v].x - y[v].x, x[v].y - y[v].y);
                const float2 e1 = make_float2(x[v].z - y[v].z, x[v].w - y[v].w);
                acc = __ffma2_rn(e0, e0, acc);
                acc = __ffma2_rn(e1, e1, acc);
            }
        } else {
            // 8 float4 of the row in flight per lane, then their arithmetic
            for (int f0 = u; f0 < nf4; f0 += 64) {
                float4 x[8];
#pragma unroll
                for (int v = 0; v < 8; ++v) {
                    const int f = f0 + 8 * v;
                    x[v] = f < nf4 ? __ldcs(x4 + f) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int v = 0; v < 8; ++v) {
                    const int f = f0 + 8 * v;
                    const float4 y = f < nf4 ? __ldg(q4 + f) : make_float4(0.f, 0.f, 0.f, 0.f);
                    const float2 e0 = make_float2(x[v].x - y.x, x[v].y - y.y), e1 = make_float2(x[v].z - y.z, x[v].w - y.w);
                    acc = __ffma2_rn(e0, e0, acc);
                    acc = __ffma2_rn(e1, e1, acc);
                }
            }
        }
        float s_ = acc.x + acc.y;
        s_ += __shfl_xor_sync(0xffffffffu, s_, 1);
        s_ += __shfl_xor_sync(0xffffffffu, s_, 2);
        s_ += __shfl_xor_sync(0xffffffffu, s_, 4);
        if (u == 0) d2[slot] = s_;
    }
}

// ---- after the rounds of a batch: the top-k distances recomputed directly in fp32 (the
//      tensor-core verification ranks by ||x||^2 + ||q||^2 - 2 x.q), re-sorted by (d2, id).
__global__ void __launch_bounds__(256) k_rerank_exact(const QState* __restrict__ qs, const float* __restrict__ X,
                                                      const float* __restrict__ Q, int64_t ld, int k,
                                                      unsigned long long* __restrict__ topk) {
    pdl_wait();
    __shared__ unsigned long long s_keys[TK_MAX];
    const int q = blockIdx.x;
    const int tk = qs[q].tk;
    if (tk <= 0) return;
    unsigned long long* t = topk + (int64_t)q * k;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const float4* q4 = reinterpret_cast<const float4*>(Q + (int64_t)q * ld);
    const int nf4 = (int)(ld / 4);
    for (int e = warp; e < tk; e += 8) {
        const uint32_t id = (uint32_t)(t[e] & 0xFFFFFFFFull);
        const float4* x4 = reinterpret_cast<const float4*>(X + (int64_t)id * ld);
        float2 acc = make_float2(0.f, 0.f);
        for (int f = lane; f < nf4; f += 32) {
            const float4 x = __ldg(x4 + f), y = __ldg(q4 + f);
            const float2 d0 = make_float2(x.x - y.x, x.y - y.y), d1 = make_float2(x.z - y.z, x.w - y.w);
            acc = __ffma2_rn(d0, d0, acc);
            acc = __ffma2_rn(d1, d1, acc);
        }
        float s_ = acc.x + acc.y;
        for (int o = 16; o > 0; o >>= 1) s_ += __shfl_xor_sync(0xffffffffu, s_, o);
        if (lane == 0) s_keys[e] = mkkey(s_, id);
    }
    int n2 = 1;
    while (n2 < tk) n2 <<= 1;
    for (int i = tk + threadIdx.x; i < n2; i += blockDim.x) s_keys[i] = ~0ull;
    __syncthreads();
    bitonic_sort_smem(s_keys, n2);
    for (int i = threadIdx.x; i < tk; i += blockDim.x) t[i] = s_keys[i];
}

__global__ void __launch_bounds__(TK_THREADS) k_topk(const int* __restrict__ act, QState* __restrict__ qs,
                                                     const uint32_t* __restrict__ cand, const float* __restrict__ d2,
                                                     unsigned long long* __restrict__ topk, int k,
                                                     float cr2, int round, int max_rounds) {
    pdl_wait();
    __shared__ unsigned long long s_keys[TK_MAX];
    __shared__ uint32_t s_hist[256];
    uint32_t* s_h12 = reinterpret_cast<uint32_t*>(s_keys);   // 4096 bins, dead before s_keys is filled
    __shared__ uint32_t s_wsum[32];
    __shared__ uint32_t s_bin, s_below;
    __shared__ unsigned long long s_prefix, s_mask, s_rem;
    __shared__ int s_n;
    const int q = act[blockIdx.x];
    QState s = qs[q];
    unsigned long long* tk = topk + (int64_t)q * k;
    const uint32_t* cl = cand;
    const float* dl = d2;
    const int64_t old = s.tk, e0 = s.roff, nn = s.rcnt, M = old + nn;
    auto key_at = [&](int64_t i) -> unsigned long long {
        return i < old ? tk[i] : mkkey(dl[e0 + i - old], cl[e0 + i - old]);
    };
    if (threadIdx.x == 0) { s_n = 0; s_prefix = 0; s_mask = 0; s_rem = (unsigned long long)k; }
    __syncthreads();
    int outn;
    if (M <= k) {
        for (int64_t i = threadIdx.x; i < M; i += TK_THREADS) s_keys[i] = key_at(i);
        outn = (int)M;
    } else {
        // pass 1: histogram of the top 12 key bits (sign, exponent, 3 mantissa bits of d2)
        for (int i = threadIdx.x; i < 4096; i += TK_THREADS) s_h12[i] = 0;
        __syncthreads();
        for (int64_t i = threadIdx.x; i < M; i += TK_THREADS) atomicAdd(&s_h12[key_at(i) >> 52], 1u);
        __syncthreads();
        {   // the bin holding the k-th smallest key: block scan of 8 bins per thread
            uint32_t loc[8], sum = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) { loc[j] = s_h12[threadIdx.x * 8 + j]; sum += loc[j]; }
            uint32_t x = sum;
            const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) s_wsum[w] = x;
            __syncthreads();
            if (w == 0) {
                uint32_t v = lane < TK_THREADS / 32 ? s_wsum[lane] : 0;
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
                    if (lane >= o) v += y;
                }
                if (lane < TK_THREADS / 32) s_wsum[lane] = v;
            }
            __syncthreads();
            uint32_t before = x - sum + (w ? s_wsum[w - 1] : 0);
            if (before < (uint32_t)k && before + sum >= (uint32_t)k) {
                for (int j = 0; j < 8; ++j) {
                    if (before + loc[j] >= (uint32_t)k) {
                        s_bin = threadIdx.x * 8 + j;
                        s_below = before;
                        break;
                    }
                    before += loc[j];
                }
            }
            __syncthreads();
        }
        const uint32_t bin = s_bin, below = s_below, inbin = s_h12[bin];
        __syncthreads();
        if (below + inbin <= (uint32_t)TK_MAX) {
            // pass 2: every key below or in that bin fits in shared memory; sort, keep k
            for (int64_t i = threadIdx.x; i < M; i += TK_THREADS) {
                const unsigned long long key = key_at(i);
                if ((uint32_t)(key >> 52) <= bin) s_keys[atomicAdd(&s_n, 1)] = key;
            }
            __syncthreads();
            outn = (int)(below + inbin);
        } else {
            // crowded bin: exact radix select of the k-th key inside it, 8-bit digits
            if (threadIdx.x == 0) {
                s_prefix = (unsigned long long)bin << 52;
                s_mask = 0xFFFull << 52;
                s_rem = (unsigned long long)(k - below);
            }
            __syncthreads();
            // 8-bit digits at bits 51..4, then a 4-bit digit at bits 3..0: the exact k-th key
            for (int shift = 44; shift >= -4; shift -= 8) {
                const int sh = shift < 0 ? 0 : shift;
                const uint32_t dmask = shift < 0 ? 15u : 255u;
                for (int i = threadIdx.x; i < 256; i += TK_THREADS) s_hist[i] = 0;
                __syncthreads();
                const unsigned long long pre = s_prefix, msk = s_mask;
                for (int64_t i = threadIdx.x; i < M; i += TK_THREADS) {
                    const unsigned long long key = key_at(i);
                    if ((key & msk) == pre) atomicAdd(&s_hist[(key >> sh) & dmask], 1u);
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    unsigned long long cum = 0, rem = s_rem;
                    for (int dg = 0; dg <= (int)dmask; ++dg) {
                        if (cum + s_hist[dg] >= rem) {
                            s_prefix = pre | ((unsigned long long)dg << sh);
                            s_mask = msk | ((unsigned long long)dmask << sh);
                            s_rem = rem - cum;
                            break;
                        }
                        cum += s_hist[dg];
                    }
                }
                __syncthreads();
            }
            // keys are unique per query ((d2, id) with distinct ids), so exactly k keys are <= T0
            const unsigned long long T0 = s_prefix;
            for (int64_t i = threadIdx.x; i < M; i += TK_THREADS) {
                const unsigned long long key = key_at(i);
                if (key <= T0) {
                    const int slot = atomicAdd(&s_n, 1);
                    if (slot < TK_MAX) s_keys[slot] = key;
                }
            }
            __syncthreads();
            outn = min(s_n, TK_MAX);
        }
    }
    __syncthreads();
    __syncthreads();
    int n2 = 1;
    while (n2 < outn) n2 <<= 1;
    for (int i = outn + threadIdx.x; i < n2; i += TK_THREADS) s_keys[i] = ~0ull;
    __syncthreads();
    bitonic_sort_smem(s_keys, n2);
    outn = min(outn, k);
    for (int i = threadIdx.x; i < outn; i += TK_THREADS) tk[i] = s_keys[i];
    if (threadIdx.x == 0) {
        s.tk = outn;
        s.nver += s.rcnt;
        s.rcnt = 0;
        if (s.status == ST_ACTIVE) {
            if (outn >= k && __uint_as_float((uint32_t)(s_keys[k - 1] >> 32)) <= cr2) s.status = ST_RADIUS;  // line 9
            else if (round == max_rounds - 1) s.status = ST_CAP;                                            // AMB-20
        }
        qs[q] = s;
    }
}

__global__ void k_compact(const int* __restrict__ act, int na_ub, const int* __restrict__ dna, const QState* __restrict__ qs, int* __restrict__ act_out,
                          int* __restrict__ n_out) {
    pdl_wait();
    const int na = dna ? *dna : na_ub;
    __shared__ int s_n;
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    // order-preserving compaction (single block)
    for (int base = 0; base < na; base += blockDim.x) {
        const int a = base + threadIdx.x;
        const bool keep = a < na && qs[act[a]].status == ST_ACTIVE;
        const uint32_t bal = __ballot_sync(0xffffffffu, keep);
        __shared__ int s_w[32];
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        if (lane == 0) s_w[w] = __popc(bal);
        __syncthreads();
        if (threadIdx.x == 0) {
            int run = s_n;
            for (int i = 0; i < (int)(blockDim.x / 32); ++i) { int c = s_w[i]; s_w[i] = run; run += c; }
            s_n = run;
        }
        __syncthreads();
        if (keep) act_out[s_w[w] + __popc(bal & lanemask_lt())] = act[a];
        __syncthreads();
    }
    if (threadIdx.x == 0) *n_out = s_n;
}

__global__ void k_finalize(const QState* __restrict__ qs, const unsigned long long* __restrict__ ctr,
                           const unsigned long long* __restrict__ topk, int nqb, int k,
                           int64_t id_offset, const double* __restrict__ radii, int64_t* __restrict__ out_ids,
                           float* __restrict__ out_d, detlsh_query_stats* __restrict__ stats, int null_on_cap) {
    pdl_wait();
    const int64_t total = (int64_t)nqb * k;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int q = (int)(i / k), e = (int)(i % k);
        const QState s = qs[q];
        // (r,c)-ANN (Alg. 4 line 10): nothing unless the pass stopped on the budget or found a
        // point within c r
        if (e < s.tk && !(null_on_cap && s.status == ST_CAP)) {
            const unsigned long long key = topk[(int64_t)q * k + e];
            out_ids[i] = (int64_t)(key & 0xFFFFFFFFull) + id_offset;
            out_d[i] = sqrtf(__uint_as_float((uint32_t)(key >> 32)));
        } else {
            out_ids[i] = -1;
            out_d[i] = INFINITY;
        }
        if (e == 0 && stats) {
            detlsh_query_stats o;
            o.rounds = s.rounds;
            o.trees_last = s.trees_last;
            o.reason = s.status == ST_BUDGET ? 0 : s.status == ST_RADIUS ? 1 : 2;
            o.pad = 0;
            o.n_cand = s.cnt;
            o.r_final = radii[max(0, s.rounds - 1)];
            o.leaves_tested = (int64_t)ctr[q * NCTR + 0];
            o.leaves_passed = (int64_t)ctr[q * NCTR + 1];
            o.points_tested = (int64_t)ctr[q * NCTR + 2];
            o.points_passed = (int64_t)ctr[q * NCTR + 3];
            o.subboxes_tested = (int64_t)ctr[q * NCTR + 4];
            stats[q] = o;
        }
    }
}

// Between query batches: zero the bitmap words the finished batch touched -- exactly the words
// flagged in each row's dirty-word summary (every writer of S, its previous-tree copy and the
// verified set marks the summary) -- instead of streaming zeros over 3 x n bits per query.
// Grid (summary chunks, rows); thread per summary word.
__global__ void __launch_bounds__(256) k_clear_dirty(uint32_t* __restrict__ bm, uint32_t* __restrict__ prev,
                                                     uint32_t* __restrict__ ver, const uint32_t* __restrict__ wsum,
                                                     int64_t nwords, int64_t nsw) {
    pdl_wait();
    const int64_t row = blockIdx.y;
    for (int64_t sw = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sw < nsw; sw += (int64_t)gridDim.x * blockDim.x) {
        uint32_t f = wsum[row * nsw + sw];
        while (f) {
            const int64_t w = sw * 32 + (__ffs(f) - 1);
            f &= f - 1;
            if (w < nwords) {
                bm[row * nwords + w] = 0u;
                prev[row * nwords + w] = 0u;
                ver[row * nwords + w] = 0u;
            }
        }
    }
}

__global__ void k_init_batch(QState* __restrict__ qs, int* __restrict__ act, int nqb) {
    pdl_wait();
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nqb; q += gridDim.x * blockDim.x) {
        QState s;
        s.cnt = 0; s.nver = 0; s.roff = 0; s.rcnt = 0; s.status = ST_ACTIVE; s.tk = 0; s.trees_last = 0; s.rounds = 0;
        s.overflow = 0; s.doc = 0; s.tnew = 0; s.pub = 0;
        qs[q] = s;
        act[q] = q;
    }
}

int64_t auto_query_budget() {
    // device memory free right now (other users of the device -- e.g. the caller's own tensors
    // allocated after an earlier query -- are seen), plus what the scratch pool holds reserved
    // but not in use (reusable by this call's scratch).  Freed index memory stays reserved in
    // the index pool and is not counted.
    int dev = 0;
    DL_CUDA(cudaGetDevice(&dev));
    size_t fr = 0, tot = 0;
    DL_CUDA(cudaMemGetInfo(&fr, &tot));
    uint64_t res = 0, used = 0;
    cudaMemPool_t sp = scratch_pool();
    DL_CUDA(cudaMemPoolGetAttribute(sp, cudaMemPoolAttrReservedMemCurrent, &res));
    DL_CUDA(cudaMemPoolGetAttribute(sp, cudaMemPoolAttrUsedMemCurrent, &used));
    const int64_t avail = (int64_t)fr + std::max<int64_t>(0, (int64_t)res - (int64_t)used);
    return std::max<int64_t>(1, (int64_t)(0.6 * (double)avail));
}

// 2048 / rho2 rounded toward zero (a lower bound of the exact scale factor).
float fdiv_rd_host(float num, float den) {
    const double x = (double)num / (double)den;
    float f = (float)x;
    if (std::isfinite(x) && (double)f > x) f = std::nextafterf(f, 0.0f);
    return f;
}


// ---- r_min estimator (AMB-22): per sample query, t_p = min over trees of the cell
//      lower bound of point p (exact fp32 LUT sums in j order, as the range filter's final
//      test), then the B-th smallest t_p: r*_q = sqrt(t_(B)) / eps is the smallest radius whose
//      full round gives |S| >= B.
__global__ void __launch_bounds__(256) k_rstar_tree(const float* __restrict__ lut, const uint8_t* __restrict__ tcodes,
                                                    const uint32_t* __restrict__ perm, int64_t n, int t, int L, int K,
                                                    int N_r, uint32_t* __restrict__ tp) {
    pdl_wait();
    extern __shared__ float s_lut1[];
    const int q = blockIdx.y;
    const float* src = lut + ((int64_t)q * L + t) * K * N_r;
    for (int i = threadIdx.x; i < K * N_r; i += 256) s_lut1[i] = src[i];
    __syncthreads();
    uint32_t* out = tp + (int64_t)q * n;
    for (int64_t pos = blockIdx.x * (int64_t)256 + threadIdx.x; pos < n; pos += (int64_t)gridDim.x * 256) {
        float s = 0.f;
        for (int j = 0; j < K; ++j) s += s_lut1[j * N_r + tcodes[pos * K + j]];
        atomicMin(out + perm[pos], __float_as_uint(s));      // non-negative floats order as their bits
    }
}

__global__ void __launch_bounds__(1024) k_select_kth_u32(const uint32_t* __restrict__ vals, int64_t n, int64_t rank,
                                                          uint32_t* __restrict__ out) {
    pdl_wait();
    __shared__ uint32_t s_hist[256];
    __shared__ uint32_t s_prefix, s_mask;
    __shared__ unsigned long long s_rem;
    const uint32_t* v = vals + (int64_t)blockIdx.x * n;
    if (threadIdx.x == 0) { s_prefix = 0; s_mask = 0; s_rem = (unsigned long long)rank; }
    __syncthreads();
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += 1024) s_hist[i] = 0;
        __syncthreads();
        const uint32_t pre = s_prefix, msk = s_mask;
        for (int64_t i = threadIdx.x; i < n; i += 1024) {
            const uint32_t x = v[i];
            if ((x & msk) == pre) atomicAdd(&s_hist[(x >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long cum = 0, rem = s_rem;
            for (int dg = 0; dg < 256; ++dg) {
                if (cum + s_hist[dg] >= rem) {
                    s_prefix = pre | ((uint32_t)dg << shift);
                    s_mask = msk | (0xFFu << shift);
                    s_rem = rem - cum;
                    break;
                }
                cum += s_hist[dg];
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = s_prefix;
}

}  // namespace

void estimate_rstar(const Index& ix, const float* d_Q, int64_t q_ld, int64_t ns, int k, double beta, int proj_impl,
                    double* h_rstar, cudaStream_t st) {
    DL_REQUIRE(q_ld == ix.ld, "query row stride must equal the index's");
    const int64_t n = ix.n, LK = ix.LK;
    int64_t B = (int64_t)std::ceil(beta * (double)n) + k;
    if (B > n) B = n;
    Scratch s_qp(st, sizeof(float) * (size_t)(ns * LK));
    Scratch s_flag(st, sizeof(int));
    DL_CUDA(cudaMemsetAsync(s_flag.p, 0, sizeof(int), st));
    project_rows(ix, d_Q, q_ld, ns, s_qp.as<float>(), proj_impl, s_flag.as<int>(), st);
    Scratch s_lut(st, sizeof(float) * (size_t)(ns * LK * ix.N_r));
    Scratch s_sx(st, (size_t)(ns * LK));
    DL_LAUNCH(k_build_lut, (unsigned)std::min<int64_t>(ceil_div(ns * LK * ix.N_r, 256), 148 * 32), 256, 0, st,
              s_qp.as<float>(), (int)ns, (int)LK, ix.N_r, ix.B.as<float>(), s_lut.as<float>(), s_sx.as<uint8_t>());
    // per-point minima of one chunk of sample queries at a time: chunk * n * 4 bytes of scratch
    // bounded by ~1/4 of the query budget (and gridDim.y <= 65535)
    const int64_t per_q = sizeof(uint32_t) * (int64_t)n;
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>({ns, 65535, auto_query_budget() / 4 / per_q}));
    Scratch s_tp(st, (size_t)(per_q * chunk));
    Scratch s_out(st, sizeof(uint32_t) * (size_t)ns);
    const size_t smem = sizeof(float) * (size_t)ix.K * ix.N_r;
    ensure_dyn_smem_fn(k_rstar_tree, smem);
    const unsigned gx = (unsigned)std::min<int64_t>(ceil_div(n, 256), 64);
    for (int64_t q0 = 0; q0 < ns; q0 += chunk) {
        const int64_t nc = std::min(chunk, ns - q0);
        DL_CUDA(cudaMemsetAsync(s_tp.p, 0xFF, (size_t)(per_q * nc), st));   // NaN bits > +inf bits
        for (int t = 0; t < ix.L; ++t)
            DL_LAUNCH(k_rstar_tree, dim3(gx, (unsigned)nc), 256, smem, st, s_lut.as<float>() + q0 * LK * ix.N_r,
                      ix.tcodes.as<uint8_t>() + (int64_t)t * n * ix.K, ix.perm.as<uint32_t>() + (int64_t)t * n, n, t,
                      ix.L, ix.K, ix.N_r, s_tp.as<uint32_t>());
        DL_LAUNCH(k_select_kth_u32, (unsigned)nc, 1024, 0, st, s_tp.as<uint32_t>(), n, B, s_out.as<uint32_t>() + q0);
    }
    std::vector<uint32_t> bits(ns);
    DL_CUDA(cudaMemcpyAsync(bits.data(), s_out.p, sizeof(uint32_t) * ns, cudaMemcpyDeviceToHost, st));
    DL_CUDA(cudaStreamSynchronize(st));
    for (int64_t i = 0; i < ns; ++i) {
        float f;
        std::memcpy(&f, &bits[i], 4);
        h_rstar[i] = std::sqrt((double)f) / ix.eps;
    }
}

void query_index(const Index& ix, const float* d_Q, int64_t q_ld, const QueryArgs& a, int64_t* d_ids,
                 float* d_dists, detlsh_query_stats* d_stats, cudaStream_t st) {
    DL_REQUIRE(q_ld == ix.ld, "query row stride must equal the index's");
    const int64_t n = ix.n, nq = a.nq, LK = ix.LK;
    const int k = a.k;
    const int64_t budget = (int64_t)std::ceil(a.beta * (double)n) + k;   // AMB-17 (k = 1: Alg. 4's beta n + 1)
    const int max_rounds = std::max(1, std::min(64, a.max_rounds));
    const int64_t nwords = round_up(ceil_div(n, 32), 4);   // bitmap words per query (rows padded to 16 B)
    const int64_t cap = n;                                              // |S| <= n always

    Trace tr("query");
    // Q0: project all queries once
    Scratch s_qp(st, sizeof(float) * (size_t)(nq * LK));
    Scratch s_flag(st, sizeof(int));
    DL_CUDA(cudaMemsetAsync(s_flag.p, 0, sizeof(int), st));
    project_rows(ix, d_Q, q_ld, nq, s_qp.as<float>(), a.proj_impl, s_flag.as<int>(), st);
    // the non-finite flag is read with the first round's total (one host sync fewer); a NaN/Inf
    // query only yields garbage bounds until then, never an out-of-range access
    int qflag_checked = 0;
    tr.mark("project queries", st);

    // batch size from the memory budget: bitmap + candidate list + distances per query
    // round-buffer share: one budget's worth (beta n) of new (id, d2) pairs per query -- the buffer
    // grows on demand beyond it (was 2 beta n: measured, the larger batches this allows are 2-2.5 %
    // faster at configs[3] / configs[4])
    const int64_t per_q = nwords * 20 + (int64_t)ix.ld * 8 + (int64_t)k * 8 + (int64_t)LK * (ix.N_r * 6 + 1) + 96 +
                          (int64_t)(std::min(1.0, a.beta) * n) * 8;
    int64_t budget_bytes = a.mem_budget;
    if (budget_bytes <= 0) {
        // 60% of the memory free at this device's first query of the process.  cudaMemGetInfo
        // is not on the per-call path: measured on B200 it took 0.1-75 ms per call (the stream
        // idles meanwhile), which was up to 4x the whole query.
        budget_bytes = auto_query_budget();
    }
    int64_t qb = a.query_batch > 0 ? a.query_batch : std::max<int64_t>(1, budget_bytes / per_q);
    // round-buffer slots are 64-bit on the sparse path; the tensor-core and row paths keep
    // 32-bit offsets and are used only for rounds with < 2^32 new pairs (below)
    qb = std::min<int64_t>({qb, nq, 65535});
    DL_REQUIRE(qb >= 1, "not enough device memory for one query");

    Scratch s_bm(st, sizeof(uint32_t) * (size_t)(2 * qb * nwords));   // current union + previous
    Scratch s_ctr(st, sizeof(unsigned long long) * (size_t)(NCTR * qb));
    Scratch s_ver(st, sizeof(uint32_t) * (size_t)(qb * nwords));     // verified members of S
    const int64_t nsw = round_up(ceil_div(nwords, 32), 4);               // dirty-word summary row
    Scratch s_sum(st, sizeof(uint32_t) * (size_t)(qb * nsw));
    Scratch s_round(st);                   // (id, d2) of this round's new members, grown on demand
    Scratch s_cq(st);                      // sparse verification: active-query index per slot
    int64_t cq_cap = 0;
    int64_t round_cap = 0;
    Scratch s_total(st, sizeof(unsigned long long));
    Scratch s_tk(st, sizeof(unsigned long long) * (size_t)(qb * k));
    Scratch s_qs(st, sizeof(QState) * (size_t)qb);
    Scratch s_act(st, sizeof(int) * (size_t)(4 * qb + 6));
    Scratch s_ch(st, sizeof(uint32_t) * (size_t)(qb + 2));
    Scratch s_radii(st, sizeof(double) * 64);
    int* act = s_act.as<int>();
    int* act2 = act + qb;
    int* n_act = act2 + qb;
    int* fbuf0 = n_act + 2;          // per-tree compacted active lists (filter only)
    int* fbuf1 = fbuf0 + qb;
    int* n_f = fbuf1 + qb;

    const double eps = ix.eps;
    std::vector<double> radii(64);
    {
        double r = a.r_min;
        for (int m = 0; m < 64; ++m) { radii[m] = r; r = a.c * r; }   // r <- c r (line 11), AMB-19
    }
    DL_CUDA(cudaMemcpyAsync(s_radii.p, radii.data(), sizeof(double) * 64, cudaMemcpyHostToDevice, st));



    // per-batch LUTs
    Scratch s_lut(st, sizeof(float) * (size_t)(qb * LK * ix.N_r));
    Scratch s_sx(st, (size_t)(qb * LK));
    const size_t rf_smem = (size_t)16 * ix.K * ix.N_r;
    Scratch s_qlut(st, sizeof(uint16_t) * (size_t)(qb * LK * ix.N_r));
    Scratch s_gtab(st, (size_t)16 * ceil_div(qb, RF_G) * ix.K * ix.N_r);
    Scratch s_tctr(st, sizeof(unsigned int) * (size_t)ceil_div(qb, RF_G));
    Scratch s_ticket(st, sizeof(unsigned int));        // k_tree_post's last-block ticket
    DL_CUDA(cudaMemsetAsync(s_ticket.p, 0, sizeof(unsigned int), st));
    static const bool rf_dyn = !std::getenv("DETLSH_RF_STRIPES");   // experiments: per-CTA stripes
    static const int pq_env = std::getenv("DETLSH_FILTER_PQ") ? std::atoi(std::getenv("DETLSH_FILTER_PQ")) : 1;
    auto k_range_filter_sel = (ix.K == 16 && ix.N_r == 256)
                                  ? (pq_env ? k_range_filter<16 COMMA 256 COMMA RF_G COMMA true>
                                            : k_range_filter<16 COMMA 256 COMMA RF_G COMMA false>)
                                  : k_range_filter<0 COMMA 0 COMMA RF_G COMMA false>;
    ensure_dyn_smem_fn(k_range_filter_sel, rf_smem);
    RFArgs ra;
    ra.gtab = nullptr;
    ra.tctr = nullptr;
    // sparse tiles in CELL mode: (query, leaf) pair lists screened by k_leaf_points
    int64_t pcap = 0;
    for (int t = 0; t < ix.L; ++t) pcap = std::max<int64_t>(pcap, ix.tree_leaf_begin[t + 1] - ix.tree_leaf_begin[t]);
    static const int pairs_env = std::getenv("DETLSH_LEAF_PAIRS") ? std::atoi(std::getenv("DETLSH_LEAF_PAIRS")) : 1;
    const bool use_pairs = pairs_env && a.mode == DETLSH_MODE_CELL && ix.K <= 32;
    Scratch s_plist(st, use_pairs ? sizeof(uint32_t) * (size_t)(qb * pcap) : 0);
    Scratch s_pcnt(st, sizeof(uint32_t) * (size_t)(2 * qb));   // list lengths, take counters
    ra.plist = use_pairs ? s_plist.as<uint32_t>() : nullptr;
    ra.pcnt = s_pcnt.as<uint32_t>();
    ra.pcap = pcap;
    LPArgs lpa;
    lpa.qs = s_qs.as<QState>();
    lpa.qs_mut = s_qs.as<QState>();
    lpa.plist = ra.plist;
    lpa.pcnt = ra.pcnt;
    lpa.ptake = ra.pcnt + qb;
    lpa.pcap = pcap;
    lpa.leaf_off = ix.leaf_off.as<uint32_t>();
    lpa.L = ix.L;
    lpa.K = ix.K;
    lpa.N_r = ix.N_r;
    const size_t lp_smem = (size_t)ix.K * ix.N_r * sizeof(uint16_t);
    Scratch s_q12(st, use_pairs ? sizeof(uint16_t) * (size_t)(qb * LK * ix.N_r) : 0);
    const bool lp_fixed = ix.K == 16 && ix.N_r == 256;
    static const int lp_g = std::getenv("DETLSH_LP_G") ? std::atoi(std::getenv("DETLSH_LP_G")) : 16;
    // two-level filter (k_tile_pairs + tile-mode k_leaf_points): DETLSH_TILE_PAIRS = 1 on, 0 off,
    // default (-1) on when first-layer cells hold >= 64 points on average (n >= 64 * 2^K): then a
    // query reaches few of a tile's leaves and the group-union SIMD leaf scan wastes most of its
    // work (measured: configs[3] 67.5 -> 60.3 ms, configs[4] 662 -> 585 ms; configs[1], 15 points
    // per cell: 1.93 -> 2.18 ms, so off)
    static const int tp_env = std::getenv("DETLSH_TILE_PAIRS") ? std::atoi(std::getenv("DETLSH_TILE_PAIRS")) : -1;
    const bool tp_want = tp_env == 1 || (tp_env < 0 && ix.K < 40 && (n >> ix.K) >= 64);
    const bool tile_pairs = tp_want && use_pairs && lp_fixed && RF_G == 16 && rf_dyn && !a.lb_order;
    // box bounds two dims per min/max (box_bound16); DETLSH_BOX16=0 selects the byte-wise form (read
    // per call: experiments switch it between queries of one index)
    const bool box16 = !(std::getenv("DETLSH_BOX16") && std::atoi(std::getenv("DETLSH_BOX16")) == 0);
    // tile mode: point codes prefetched into L2 one sub-box step ahead (DETLSH_LP_PF, read per call)
    // (measured at configs[4]: 63.2 -> 62.3 ms per 2,000 queries with either; configs[3] +-0.4 %)
    const int lp_pf = std::getenv("DETLSH_LP_PF") ? std::atoi(std::getenv("DETLSH_LP_PF")) : 1;   // 0 off, 1 L2, 2 L1
    auto k_leaf_points_sel = tile_pairs ? (box16 ? (lp_pf == 2   ? k_leaf_points<16, 256, 32, 7>
                                                    : lp_pf == 1 ? k_leaf_points<16, 256, 32, 3>
                                                                 : k_leaf_points<16, 256, 32, 1>)
                                                 : k_leaf_points<16, 256, 32>)
                             : lp_fixed ? (lp_g == 8 ? k_leaf_points<16, 256, 8>
                                           : box16   ? k_leaf_points<16, 256, 16, 1>
                                                     : k_leaf_points<16, 256, 16>)
                                        : k_leaf_points<0, 0, 16>;
    lpa.tile_leaf = tile_pairs ? ix.tile_leaf.as<uint32_t>() : nullptr;
    lpa.tile_packed = ix.tree_leaf_begin.back() < ((int64_t)1 << 27) ? 1 : 0;
    ra.tile_packed = lpa.tile_packed;
    static const bool tp_hist_env = std::getenv("DETLSH_TP_HIST") != nullptr;
    Scratch s_tph(st, tp_hist_env ? sizeof(unsigned long long) * 17 : 0);
    ra.tp_hist = tp_hist_env ? s_tph.as<unsigned long long>() : nullptr;
    if (tp_hist_env) DL_CUDA(cudaMemsetAsync(s_tph.p, 0, sizeof(unsigned long long) * 17, st));
    struct TpHistPrint {      // experiments: print the histogram when the query call ends
        unsigned long long* d;
        cudaStream_t st;
        ~TpHistPrint() {
            if (!d) return;
            unsigned long long h[17];
            if (cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, st) != cudaSuccess) return;
            if (cudaStreamSynchronize(st) != cudaSuccess) return;
            std::fprintf(stderr, "DETLSH_TP_HIST reached tiles by group queries:");
            for (int i = 1; i <= 16; ++i) std::fprintf(stderr, " %llu", h[i]);
            std::fprintf(stderr, "\n");
        }
    } tp_hist_print{ra.tp_hist, st};
    // two-level filter: each tree's active queries in locality order (DETLSH_QSORT=1; measured at
    // configs[4]: no gain in the pair kernel, +9 ms of sorting -- off by default)
    static const int qsort_env = std::getenv("DETLSH_QSORT") ? std::atoi(std::getenv("DETLSH_QSORT")) : 0;
    const bool qsort_on = qsort_env != 0;
    Scratch s_qk(st, tile_pairs && qsort_on ? sizeof(uint32_t) * (size_t)(4 * qb) : 0);
    if (tile_pairs) ensure_dyn_smem_fn(k_tile_pairs, rf_smem);
    const size_t lp_dyn = lp_fixed ? 0 : lp_smem;
    if (use_pairs && !lp_fixed)
        ensure_dyn_smem_fn(k_leaf_points_sel, lp_smem);
    ra.leaf_off = ix.leaf_off.as<uint32_t>();
    // leaf pruning uses the tight boxes (a valid, tighter bound for every member); RELAXED takes
    // whole leaves by the leaf's own (prefix) box, as the method defines it
    ra.lo = a.mode == DETLSH_MODE_RELAXED ? ix.leaf_lo.as<uint8_t>() : ix.leaf_tbox.as<uint8_t>();
    ra.hi = a.mode == DETLSH_MODE_RELAXED ? ix.leaf_hi.as<uint8_t>() : ix.leaf_tbox.as<uint8_t>() + ix.K;
    ra.bs = a.mode == DETLSH_MODE_RELAXED ? ix.K : 2 * ix.K;
    ra.tile_leaf = ix.tile_leaf.as<uint32_t>();
    ra.tile_lo = ix.tile_lo.as<uint8_t>();
    ra.tile_hi = ix.tile_hi.as<uint8_t>();
    ra.lut = s_lut.as<float>();
    ra.qlut = s_qlut.as<uint16_t>();
    ra.sx = s_sx.as<uint8_t>();
    ra.proj = ix.proj.as<float>();
    ra.qs = s_qs.as<QState>();
    ra.qs_mut = s_qs.as<QState>();
    ra.bitmap = s_bm.as<uint32_t>();
    ra.wsum = s_sum.as<uint32_t>();
    ra.nsw = nsw;
    ra.nwords = nwords;
    ra.ctr = s_ctr.as<unsigned long long>();
    uint32_t* bm_prev = s_bm.as<uint32_t>() + qb * nwords;
    ra.L = ix.L;
    ra.K = ix.K;
    ra.N_r = ix.N_r;
    ra.mode = a.mode;
    {
        static const int pq = std::getenv("DETLSH_PQ_COST") ? std::atoi(std::getenv("DETLSH_PQ_COST")) : 40;
        ra.pq_cost = pq;
        static const int rfd = std::getenv("DETLSH_RF_DEBUG") ? std::atoi(std::getenv("DETLSH_RF_DEBUG")) : 0;
        static const int tsc = std::getenv("DETLSH_RF_TSCREEN") ? std::atoi(std::getenv("DETLSH_RF_TSCREEN")) : 0;
        ra.dbg = rfd | (tsc ? 2 : 0);
    }
    const int nv = (int)ceil_div(ix.ld / 4, 8);      // float4 per lane (8 lanes per row)
    const int vnv = nv <= 1 ? 1 : nv <= 2 ? 2 : nv <= 4 ? 4 : nv <= 8 ? 8 : 0;
    VRArgs va;
    va.X = ix.Xp;
    va.ld = ix.ld;
    va.n = n;
    va.qs = s_qs.as<QState>();
    va.cur = s_bm.as<uint32_t>();
    va.ver = s_ver.as<uint32_t>();
    va.nwords = nwords;

    {   // rows per block: as many 32-row words as fit in 120 KB of shared memory (1..8)
        const int64_t per_word = (int64_t)32 * ix.ld * 4;
        va.rbw = (int)std::max<int64_t>(1, std::min<int64_t>(8, (120 * 1024) / per_word));
    }
    const size_t vr_smem = (size_t)va.rbw * 32 * ix.ld * 4;
    // verification kernel per round: the tensor-core kernel costs a dense X.Q^T over all rows and
    // the round's active queries whatever the candidate density; the CUDA-core row kernel reads X
    // once and pays per candidate.  Auto (verify_impl 0) picks the cheaper by a cost model fitted
    // on B200 at configs[1] (tc 2.5 ms per 1M rows x 1000 queries x 256 floats; rows 0.17 ms per
    // 1M x 256 floats read + 6.3 ms per 115.7M candidates x 256 floats).
    const bool tc_ok = a.verify_impl != 1 && a.verify_impl != 3 && ix.xnorm.p != nullptr;
    const int64_t nw4 = round_up(nwords, 4);
    Scratch s_boff(st, sizeof(uint32_t) * (size_t)(a.verify_impl != 1 ? 2 * qb * nw4 : qb * ceil_div(nwords, va.rbw)));
    Scratch s_qa(st, tc_ok ? sizeof(float) * (size_t)(qb * (2 * ix.ld + 1)) : 0);
    const bool vexact = (ix.ld / 4) == 8 * vnv;
    ensure_dyn_smem_fn(k_verify_rows<1, false>, vr_smem);
    ensure_dyn_smem_fn(k_verify_rows<2, false>, vr_smem);
    ensure_dyn_smem_fn(k_verify_rows<4, false>, vr_smem);
    ensure_dyn_smem_fn(k_verify_rows<4, true>, vr_smem);
    ensure_dyn_smem_fn(k_verify_rows<8, false>, vr_smem);
    ensure_dyn_smem_fn(k_verify_rows<8, true>, vr_smem);
    ensure_dyn_smem_fn(k_verify_rows<0, false>, vr_smem);

    // Sec. 6.2.2(2): for the queries whose tree-t candidates cross the budget, keep
    // only the leaves up to the one (in (LB, leaf) order) at which |S| reaches it
    Scratch s_lbo(st);
    size_t lbo_cap = 0;
    Scratch s_lcross(st, sizeof(int) * (size_t)(qb + 1));
    double lbo_rho2 = 0;
    const float* lbo_qp = nullptr;
    auto lb_order_tree = [&](int t, const int* fa_, int nf_, const int* dnf_) {
        int* cross = s_lcross.as<int>();
        int* ncross_d = cross + qb;
        DL_CUDA(cudaMemsetAsync(ncross_d, 0, sizeof(int), st));
        DL_LAUNCH(k_count_new, dim3((unsigned)nf_, (unsigned)ceil_div(nsw, CN_SW)), 256, 0, st, fa_, dnf_,
                  s_qs.as<QState>(), s_bm.as<uint32_t>(), bm_prev, nwords, s_sum.as<uint32_t>(), nsw, 0);
        DL_LAUNCH(k_lbo_cross, (unsigned)ceil_div(nf_, 256), 256, 0, st, fa_, nf_, dnf_, s_qs.as<QState>(), budget, cross,
                  ncross_d);
        int ncross = 0;
        DL_CUDA(cudaMemcpyAsync(&ncross, ncross_d, sizeof(int), cudaMemcpyDeviceToHost, st));
        DL_CUDA(cudaStreamSynchronize(st));
        if (ncross == 0) return;
        const int64_t lb0 = ix.tree_leaf_begin[t], nl_t = ix.tree_leaf_begin[t + 1] - lb0;
        const int64_t m = (int64_t)ncross * nl_t;
        const size_t need_b = sizeof(uint32_t) * (size_t)(5 * m + 1) + sizeof(unsigned long long) * (size_t)ncross + 256;
        if (need_b > lbo_cap) {       // grow-only (scratch is bump-allocated within a call)
            lbo_cap = need_b + need_b / 2;
            s_lbo.alloc(lbo_cap);
        }
        uint32_t* k0 = s_lbo.as<uint32_t>();
        uint32_t* v0 = k0 + m;
        uint32_t* k1 = v0 + m;
        uint32_t* v1 = k1 + m;
        uint32_t* nn = v1 + m;
        unsigned long long* cut = reinterpret_cast<unsigned long long*>(nn + m + (m & 1));   // 8-byte aligned
        LboArgs la;
        la.cross = cross;
        la.lut = s_lut.as<float>();
        la.sx = s_sx.as<uint8_t>();
        la.lo = ix.leaf_lo.as<uint8_t>() + lb0 * ix.K;
        la.hi = ix.leaf_hi.as<uint8_t>() + lb0 * ix.K;
        la.leaf_off = ix.leaf_off.as<uint32_t>() + lb0;
        la.tcodes = ix.tcodes.as<uint8_t>() + (int64_t)t * n * ix.K;
        la.perm = ix.perm.as<uint32_t>() + (int64_t)t * n;
        la.proj = ix.proj.as<float>();
        la.qp = a.mode == DETLSH_MODE_EXACT ? lbo_qp : nullptr;
        la.prev = bm_prev;
        la.cur = s_bm.as<uint32_t>();
        la.nwords = nwords;
        la.pos_base = (int64_t)t * n;
        la.nl = nl_t;
        la.rho2 = (float)lbo_rho2;
        la.t = t;
        la.L = ix.L;
        la.K = ix.K;
        la.N_r = ix.N_r;
        la.mode = a.mode;
        la.keys = k0;
        la.vals = v0;
        la.nnew = nn;
        la.cut = cut;
        const size_t smem = sizeof(float) * (size_t)ix.K * ix.N_r;
        const dim3 grid((unsigned)std::min<int64_t>(ceil_div(nl_t, 8), 64), (unsigned)ncross);
        DL_LAUNCH(k_lbo_leaves<false>, grid, 256, smem, st, la);
        const bool flip = radix_sort_batched(k0, v0, k1, v1, nl_t, ncross, 32, st);
        DL_LAUNCH(k_lbo_cut, (unsigned)ncross, 1024, 0, st, cross, s_qs.as<QState>(), budget, flip ? k1 : k0,
                  flip ? v1 : v0, nn, nl_t, cut);
        DL_LAUNCH(k_lbo_reset, (unsigned)std::min<int64_t>(ceil_div((int64_t)ncross * nwords, 256), 148 * 16), 256, 0, st,
                  cross, ncross, bm_prev, s_bm.as<uint32_t>(), nwords);
        DL_LAUNCH(k_lbo_leaves<true>, grid, 256, smem, st, la);
    };

    // S bitmaps: streamed zeros for the first batch (the scratch holds anything); after a batch,
    // only its dirty words are cleared when they are few (k_clear_dirty: ~3 sector writes per
    // member instead of 12 B per id per query -- at configs[4] the streamed form is 37.5 MB per
    // query)
    uint64_t batch_members = 0;
    int prev_rows = 0;
    for (int64_t q0 = 0; q0 < nq; q0 += qb) {
        const int nqb = (int)std::min<int64_t>(qb, nq - q0);
        const float* Qb = d_Q + q0 * q_ld;
        const float* Qpb = s_qp.as<float>() + q0 * LK;
        va.Q = Qb;
        static const int dirty_env = std::getenv("DETLSH_DIRTY_CLEAR") ? std::atoi(std::getenv("DETLSH_DIRTY_CLEAR")) : 1;
        const bool dirty = dirty_env && q0 > 0 &&      // DETLSH_DIRTY_CLEAR: 0 never, 2 always (tests)
                           (dirty_env == 2 || (double)batch_members * 96.0 < 0.5 * (double)prev_rows * (double)nwords * 12.0);
        if (dirty) {
            DL_LAUNCH(k_clear_dirty, dim3((unsigned)std::min<int64_t>(ceil_div(nsw, 256), 64), (unsigned)prev_rows), 256, 0,
                      st, s_bm.as<uint32_t>(), bm_prev, s_ver.as<uint32_t>(), s_sum.as<uint32_t>(), nwords, nsw);
        } else {
            DL_CUDA(cudaMemsetAsync(s_bm.p, 0, sizeof(uint32_t) * (size_t)(2 * qb * nwords), st));
            DL_CUDA(cudaMemsetAsync(s_ver.p, 0, sizeof(uint32_t) * (size_t)(qb * nwords), st));
        }
        batch_members = 0;
        prev_rows = nqb;
        DL_CUDA(cudaMemsetAsync(s_sum.p, 0, sizeof(uint32_t) * (size_t)(qb * nsw), st));
        DL_CUDA(cudaMemsetAsync(s_ctr.p, 0, sizeof(unsigned long long) * (size_t)(NCTR * qb), st));
        DL_CUDA(cudaMemsetAsync(s_pcnt.p, 0, sizeof(uint32_t) * (size_t)(2 * qb), st));
        tr.mark("batch setup", st);
        DL_LAUNCH(k_init_batch, (unsigned)ceil_div(nqb, 256), 256, 0, st, s_qs.as<QState>(), act, nqb);
        int na = nqb;
        bool any_tc = false;           // a round ranked by the tensor-core form ||x||^2 + ||q||^2 - 2 x.q
        int* cur = act;
        int* nxt = act2;
        for (int m = 0; m < max_rounds && na > 0; ++m) {
            const double r = radii[m];
            const float rho2 = (float)((eps * r) * (eps * r));
            lbo_rho2 = rho2;
            lbo_qp = Qpb;
            const float cr2 = (float)((a.c * r) * (a.c * r));
            {   // quantised screen of this round: scale QT / rho^2 rounded down (the pair kernel's
                // finer table: terms <= D 2048/rho^2, cap 4095)
                const float inv_rd = fdiv_rd_host((float)QuantSpec<RF_G>::QT, rho2);
                const int64_t per_q = LK * ix.N_r;
                if (m == 0 && ix.N_r == 256) {   // every batch query is active: all tables at once
                    DL_LAUNCH(k_build_tables256, (unsigned)ceil_div((int64_t)nqb * LK, 8), 256, 0, st, Qpb,
                              (int64_t)nqb * LK, ix.B.as<float>(), (int)LK, s_lut.as<float>(), s_sx.as<uint8_t>(),
                              inv_rd, (float)QuantSpec<RF_G>::CAP, s_qlut.as<uint16_t>(), fdiv_rd_host(2048.f, rho2),
                              4095.f, use_pairs ? s_q12.as<uint16_t>() : (uint16_t*)nullptr);
                } else if (m == 0) {
                    DL_LAUNCH(k_build_tables, dim3((unsigned)LK, (unsigned)nqb), ix.N_r, 0, st, Qpb, (int)LK, ix.N_r,
                              ix.B.as<float>(), s_lut.as<float>(), s_sx.as<uint8_t>(), inv_rd,
                              (float)QuantSpec<RF_G>::CAP, s_qlut.as<uint16_t>(), fdiv_rd_host(2048.f, rho2), 4095.f,
                              use_pairs ? s_q12.as<uint16_t>() : (uint16_t*)nullptr);
                } else {
                    const dim3 g((unsigned)std::min<int64_t>(ceil_div(per_q, 256), 64), (unsigned)na);
                    DL_LAUNCH(k_build_qlut, g, 256, 0, st, s_lut.as<float>(), cur, per_q, inv_rd,
                              (float)QuantSpec<RF_G>::CAP, s_qlut.as<uint16_t>());
                    if (use_pairs)
                        DL_LAUNCH(k_build_qlut, g, 256, 0, st, s_lut.as<float>(), cur, per_q, fdiv_rd_host(2048.f, rho2),
                                  4095.f, s_q12.as<uint16_t>());
                }
            }
            // queries that stop on the budget after tree t (Alg. 5 line 7) leave the filter: the
            // trees after it run over the compacted list of still-active queries (fewer groups)
            int* fa = cur;
            int nf = na;                   // upper bound of the list's length
            const int* dnf = nullptr;      // its device count once compacted on the device (no host sync)
            for (int t = 0; t < ix.L && nf > 0; ++t) {
                ra.tcodes = ix.tcodes.as<uint8_t>() + (int64_t)t * n * ix.K;
                ra.perm = ix.perm.as<uint32_t>() + (int64_t)t * n;
                ra.ptl = ix.point_tile_leaf.as<uint16_t>() + (int64_t)t * n;
                ra.pos_base = (int64_t)t * n;
                ra.tile_begin = ix.tree_tile_begin[t];
                ra.tile_end = ix.tree_tile_begin[t + 1];
                ra.act = fa;
                ra.qp = Qpb;
                ra.na = nf;
                ra.dna = dnf;
                ra.rho2 = rho2;
                ra.t = t;
                if (tile_pairs && qsort_on && nf > RF_G) {
                    uint32_t* k0 = s_qk.as<uint32_t>();
                    uint32_t* v0 = k0 + qb;
                    DL_LAUNCH(k_qkey, (unsigned)std::min<int64_t>(ceil_div(nf, 256), 148), 256, 0, st, fa, nf, dnf,
                              s_sx.as<uint8_t>(), ix.L, ix.K, ix.nb, t, k0, v0);
                    const bool flip = radix_sort_batched(k0, v0, k0 + 2 * qb, v0 + 2 * qb, nf, 1, 24, st);
                    fa = reinterpret_cast<int*>(flip ? v0 + 2 * qb : v0);
                    ra.act = fa;
                }
                const int groups = (int)ceil_div(nf, RF_G);
                if (RF_G == 16) {
                    uint4* gt = s_gtab.as<uint4>();
                    DL_LAUNCH(k_group_table, dim3((unsigned)groups, (unsigned)ix.K), 256, 0, st, fa, nf, dnf,
                              s_qs.as<QState>(), s_qlut.as<uint16_t>(), LK * ix.N_r, t, ix.K * ix.N_r,
                              (uint32_t)QuantSpec<RF_G>::CAP, s_sx.as<uint8_t>(), ix.L, ix.K, ix.N_r, gt,
                              rf_dyn ? s_tctr.as<unsigned int>() : (unsigned int*)nullptr);
                    ra.gtab = gt;
                    ra.tctr = rf_dyn ? s_tctr.as<unsigned int>() : nullptr;
                }
                // L2 blocking: a large tree is filtered in chunks of consecutive tiles holding ~chunk_pts
                // points each -- the range filter and the pair kernel of all the batch's queries finish one
                // chunk before the next starts, so its codes, ids, boxes and sub-boxes are read from
                // HBM about once per batch and served from L2 to every query (tree order: a chunk's
                // tiles, leaves and points are contiguous).  Results do not depend on the chunking.
                const int64_t t_tile0 = ix.tree_tile_begin[t], t_tile1 = ix.tree_tile_begin[t + 1];
                // (measured at configs[4]: 1M-8M-point chunks were 17-95 % SLOWER than one pass -- the
                // per-chunk launches cost more than the L2 reuse gains; off by default, kept as a switch)
                static const int64_t chunk_pts = std::getenv("DETLSH_CHUNK_PTS")
                                                     ? std::atoll(std::getenv("DETLSH_CHUNK_PTS")) : (int64_t)0;
                const int64_t tiles_t = t_tile1 - t_tile0;
                const int64_t chunk_tiles = (chunk_pts <= 0 || a.lb_order) ? tiles_t
                    : std::max<int64_t>(RF_THREADS / 32, ceil_div(chunk_pts * tiles_t, std::max<int64_t>(1, n)));
                for (int64_t c0 = t_tile0; c0 < t_tile1; c0 += chunk_tiles) {
                ra.tile_begin = c0;
                ra.tile_end = std::min(t_tile1, c0 + chunk_tiles);
                if (c0 != t_tile0)
                    DL_LAUNCH(k_chunk_prep, (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nf, 256), 148)), 256, 0, st,
                              fa, nf, dnf, use_pairs ? (const uint32_t*)ra.pcnt : (const uint32_t*)nullptr, lpa.ptake,
                              ra.tctr);
                const int64_t ntiles = ra.tile_end - ra.tile_begin;
                // about `rf_waves` waves of RF_CTAS resident CTAs per SM in all (tiles from a per-group
                // counter: 1 wave; else per-CTA stripes: 3 waves, 2-4 measured within 1 %)
                static const int rf_waves = std::getenv("DETLSH_RF_WAVES") ? std::atoi(std::getenv("DETLSH_RF_WAVES"))
                                                                           : (rf_dyn ? 1 : 3);
                const int stripes = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(ntiles, RF_THREADS / 32),
                                                                                 (148 * RF_CTAS * rf_waves + groups / 2) / groups));
                if (tile_pairs)
                    DL_LAUNCH(k_tile_pairs, dim3((unsigned)groups, (unsigned)stripes), RF_THREADS, rf_smem, st, ra);
                else
                    DL_LAUNCH(k_range_filter_sel, dim3((unsigned)groups, (unsigned)stripes), RF_THREADS, rf_smem, st, ra);
                if (use_pairs) {
                    lpa.act = fa;
                    lpa.dna = dnf;
                    lpa.na = nf;
                    lpa.lut = s_lut.as<float>();
                    lpa.tcodes = ra.tcodes;
                    lpa.lo = ra.lo;
                    lpa.hi = ra.hi;
                    lpa.bs = ra.bs;
                    static const bool no_sb = std::getenv("DETLSH_NO_SUBBOX") != nullptr;   // experiments
                    lpa.sb_off = (ix.sb_off.p && !no_sb) ? ix.sb_off.as<uint32_t>() : nullptr;
                    lpa.sb_lo = ix.sb_box.as<uint8_t>();
                    lpa.sb_hi = ix.sb_box.as<uint8_t>() + ix.K;
                    lpa.sx = ra.sx;
                    lpa.perm = ra.perm;
                    lpa.pos_base = ra.pos_base;
                    lpa.bitmap = s_bm.as<uint32_t>();
                    lpa.wsum = s_sum.as<uint32_t>();
                    lpa.nsw = nsw;
                    lpa.nwords = nwords;
                    lpa.rho2 = rho2;
                    lpa.inv_rd = fdiv_rd_host(2048.f, rho2);
                    lpa.t = t;
                    lpa.ctr = s_ctr.as<unsigned long long>();
                    lpa.q12 = s_q12.as<uint16_t>();
                    // blocks per query (grid y).  Blocks start in x-major order, so a query holds ~1-2
                    // blocks at first and gains more only as other blocks finish; a query with a
                    // long list needs many blocks available late in the launch (blocks that find the
                    // list taken exit before loading anything).  Measured (per 2,000 queries at
                    // configs[4], ~460 per batch): y = 16 88.5 ms, 32 72.8, 64 66.2, 128 64.0, 256
                    // 63.5; configs[3] (~3,400 per batch) best at 32 (47.3 ms vs 48.1 at 16, 49.0 at
                    // 128); configs[1] (pair kernel of the SIMD path) 32.  Tile mode: ~100K blocks
                    // per launch, y in [16, 256]; DETLSH_LP_Y overrides (read per call).
                    int lp_y = tile_pairs ? (int)std::min<int64_t>(256, std::max<int64_t>(16, 100000 / std::max(1, nf))) : 32;
                    if (std::getenv("DETLSH_LP_Y")) lp_y = std::max(1, std::atoi(std::getenv("DETLSH_LP_Y")));
                    DL_LAUNCH(k_leaf_points_sel, dim3((unsigned)nf, (unsigned)lp_y), LP_THREADS, lp_dyn, st, lpa);
                }
                }   // chunks
                if (!a.lb_order) {
                    int* fa2 = (fa == fbuf0) ? fbuf1 : fbuf0;
                    int* dn2 = (fa == fbuf0) ? n_f + 1 : n_f;
                    const bool more = t + 1 < ix.L;
                    DL_LAUNCH(k_tree_post, (unsigned)nf, 256, 0, st, fa, nf, dnf, s_qs.as<QState>(), s_bm.as<uint32_t>(),
                              bm_prev, nwords, s_sum.as<uint32_t>(), nsw, budget, 0,
                              use_pairs ? ra.pcnt : (uint32_t*)nullptr, lpa.ptake, t, m, cap, s_ticket.as<unsigned int>(),
                              more ? fa2 : (int*)nullptr, more ? dn2 : (int*)nullptr, (unsigned long long*)nullptr);
                    if (more) {
                        fa = fa2;
                        dnf = dn2;
                    }
                    continue;
                }
                lb_order_tree(t, fa, nf, dnf);
                DL_LAUNCH(k_count_decide, (unsigned)ceil_div(nf, 256), 256, 0, st, fa, nf, dnf, s_qs.as<QState>(), budget,
                          1, use_pairs ? ra.pcnt : (uint32_t*)nullptr, lpa.ptake);
                DL_LAUNCH(k_count_new, dim3((unsigned)nf, (unsigned)ceil_div(nsw, CN_SW)), 256, 0, st, fa, dnf,
                          s_qs.as<QState>(), s_bm.as<uint32_t>(), bm_prev, nwords, s_sum.as<uint32_t>(), nsw, 1);
                if (t + 1 < ix.L) {
                    int* fa2 = (fa == fbuf0) ? fbuf1 : fbuf0;
                    int* dn2 = (fa == fbuf0) ? n_f + 1 : n_f;
                    DL_LAUNCH(k_tree_end_compact, 1, 1024, 0, st, fa, nf, dnf, s_qs.as<QState>(), t, m, budget, cap,
                              fa2, dn2);
                    fa = fa2;
                    dnf = dn2;
                } else {
                    DL_LAUNCH(k_tree_end, (unsigned)ceil_div(nf, 256), 256, 0, st, fa, nf, dnf, s_qs.as<QState>(), t, m,
                              budget, cap);
                }
            }
            tr.mark("filter (L trees)", st);
            // |S| exact for the round's accounting (trees whose count was skipped)
            DL_LAUNCH(k_tree_post, (unsigned)na, 256, 0, st, cur, na, (const int*)nullptr, s_qs.as<QState>(),
                      s_bm.as<uint32_t>(), bm_prev, nwords, s_sum.as<uint32_t>(), nsw, budget, 1, (uint32_t*)nullptr,
                      (uint32_t*)nullptr, 0, m, cap, s_ticket.as<unsigned int>(), (int*)nullptr, (int*)nullptr,
                      s_total.as<unsigned long long>());
            unsigned long long tot = 0;     // new members of S over the round's queries
            {
                int bad = 0;
                DL_CUDA(cudaMemcpyAsync(&tot, s_total.p, sizeof(tot), cudaMemcpyDeviceToHost, st));
                if (!qflag_checked) DL_CUDA(cudaMemcpyAsync(&bad, s_flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
                DL_CUDA(cudaStreamSynchronize(st));
                DL_REQUIRE(!bad, "queries contain NaN or Inf");
                qflag_checked = 1;
                batch_members += tot;
                if ((int64_t)tot > round_cap) {
                    round_cap = (int64_t)(tot + tot / 2 + 1024);
                    s_round.alloc((size_t)round_cap * 8);
                }
            }
            va.cand = s_round.as<uint32_t>();
            va.d2 = reinterpret_cast<float*>(s_round.as<uint32_t>() + round_cap);
            va.act = cur;
            va.na = na;
            va.nblocks = ceil_div(nwords, va.rbw);
            va.boff = s_boff.as<uint32_t>();
            bool done_tc = false;
            // 0 = row kernel (verify_impl 1), 1 = tensor cores, 2 = sparse gather
            int path = a.verify_impl == 3 ? 2 : tc_ok ? 1 : 0;
            const bool wide = tot >= 0xFFFFFFFFull;    // 32-bit offsets of the TC / row paths overflow
            if (tc_ok && a.verify_impl == 0 && !wide) {
                const double scale = (double)n / 1e6 * (double)ix.ld / 256.0;
                const double t_tc = 2.5 * scale * (double)round_up(na, 16) / 1000.0;
                const double t_gather = 0.05 * (double)n / 1e6 + (double)tot * ix.ld * 4.0 / 5e9;   // ms at 5 TB/s
                path = t_tc <= t_gather ? 1 : 2;
            }
            if (wide) path = 2;
            if (path >= 1) {
                uint32_t* NB = s_boff.as<uint32_t>();
                uint32_t* BO = NB + (int64_t)qb * nw4;
                if (path == 1)
                    DL_LAUNCH(k_verify_prep, (unsigned)na, 1024, 0, st, cur, s_qs.as<QState>(), s_bm.as<uint32_t>(),
                              s_ver.as<uint32_t>(), nwords, NB, BO);
                if (path == 1) {
                    any_tc = true;
                    float* Qa = s_qa.as<float>();
                    float* Qalo = Qa + (int64_t)qb * ix.ld;
                    float* qn = Qalo + (int64_t)qb * ix.ld;
                    DL_LAUNCH(k_prep_queries, (unsigned)ceil_div(na, 8), 256, 0, st, Qb, (int64_t)ix.ld, cur, na, Qa,
                              Qalo, qn);
                    done_tc = verify_tc(ix.Xp, n, ix.ld, Qa, Qalo, qn, na, NB, BO, nw4, ix.xnorm.as<float>(), va.cand,
                                        va.d2, st);
                    DL_REQUIRE(done_tc, "tensor-core verification does not fit this shape");
                } else if (tot > 0) {
                    if ((int64_t)tot > cq_cap) {      // grow-only
                        cq_cap = (int64_t)(tot + tot / 2 + 1024);
                        s_cq.alloc(sizeof(uint32_t) * (size_t)cq_cap);
                    }
                    DL_LAUNCH(k_verify_list, (unsigned)na, nsw >= 8192 ? 256 : 128, 0, st, cur, s_qs.as<QState>(), s_bm.as<uint32_t>(),
                              s_ver.as<uint32_t>(), nwords, s_sum.as<uint32_t>(), nsw, va.cand, s_cq.as<uint32_t>());
                    const unsigned vg = (unsigned)std::min<int64_t>(ceil_div((int64_t)tot * 8, 256), 148 * 32);
                    auto k_verify_gather_sel = ix.ld == 128   ? k_verify_gather<4>
                                               : ix.ld == 256 ? k_verify_gather<8>
                                               : ix.ld == 512 ? k_verify_gather<16>
                                               : ix.ld == 96  ? k_verify_gather<3>
                                                              : k_verify_gather<0>;
                    DL_LAUNCH(k_verify_gather_sel, vg, 256, 0, st, va.cand, s_cq.as<uint32_t>(), cur, ix.Xp, Qb,
                              (int64_t)ix.ld, (int64_t)tot, va.d2);
                }
                done_tc = true;
            }
            if (!done_tc) {
            DL_LAUNCH(k_verify_offsets, (unsigned)na, 1024, 0, st, cur, s_qs.as<QState>(), s_bm.as<uint32_t>(),
                      s_ver.as<uint32_t>(), nwords, va.rbw, va.nblocks, s_boff.as<uint32_t>());
            {
                const unsigned nblocks = (unsigned)ceil_div(nwords, va.rbw);
                switch (vnv) {
                    case 1: DL_LAUNCH(k_verify_rows<1 COMMA false>, nblocks, VR_THREADS, vr_smem, st, va); break;
                    case 2: DL_LAUNCH(k_verify_rows<2 COMMA false>, nblocks, VR_THREADS, vr_smem, st, va); break;
                    case 4: if (vexact) DL_LAUNCH(k_verify_rows<4 COMMA true>, nblocks, VR_THREADS, vr_smem, st, va);
                            else DL_LAUNCH(k_verify_rows<4 COMMA false>, nblocks, VR_THREADS, vr_smem, st, va);
                            break;
                    case 8: if (vexact) DL_LAUNCH(k_verify_rows<8 COMMA true>, nblocks, VR_THREADS, vr_smem, st, va);
                            else DL_LAUNCH(k_verify_rows<8 COMMA false>, nblocks, VR_THREADS, vr_smem, st, va);
                            break;
                    default: DL_LAUNCH(k_verify_rows<0 COMMA false>, nblocks, VR_THREADS, vr_smem, st, va); break;
                }
            }
            }
            tr.mark("round buffer + verify", st);
            DL_LAUNCH(k_topk, (unsigned)na, TK_THREADS, 0, st, cur, s_qs.as<QState>(), va.cand, va.d2,
                      s_tk.as<unsigned long long>(), k, cr2, m, max_rounds);
            tr.mark("top-k", st);
            DL_LAUNCH(k_compact, 1, 1024, 0, st, cur, na, nullptr, s_qs.as<QState>(), nxt, n_act);
            DL_CUDA(cudaMemcpyAsync(&na, n_act, sizeof(int), cudaMemcpyDeviceToHost, st));
            DL_CUDA(cudaStreamSynchronize(st));
            std::swap(cur, nxt);
        }
        tr.mark("rounds done", st);
        if (any_tc)    // gather / row rounds computed the distances directly already
            DL_LAUNCH(k_rerank_exact, (unsigned)nqb, 256, 0, st, s_qs.as<QState>(), ix.Xp, Qb, (int64_t)ix.ld, k,
                      s_tk.as<unsigned long long>());
        DL_LAUNCH(k_finalize, (unsigned)std::min<int64_t>(ceil_div((int64_t)nqb * k, 256), 148 * 16), 256, 0, st,
                  s_qs.as<QState>(), s_ctr.as<unsigned long long>(), s_tk.as<unsigned long long>(), nqb, k, ix.id_offset, s_radii.as<double>(),
                  d_ids + q0 * k, d_dists + q0 * k, d_stats ? d_stats + q0 : nullptr, a.null_on_cap ? 1 : 0);
        if (a.export_S) {
            const int64_t w = ceil_div(n, 32);
            DL_CUDA(cudaMemcpy2DAsync(a.export_S + q0 * w, sizeof(uint32_t) * w, s_bm.p, sizeof(uint32_t) * nwords,
                                      sizeof(uint32_t) * w, (size_t)nqb, cudaMemcpyDeviceToDevice, st));
        }
        (void)Qb;
    }
}

}  // namespace detlsh
