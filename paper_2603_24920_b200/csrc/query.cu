// query.cu -- batched c^2-k-ANN (Alg. 5) on sm_100a.
//
// Per round r = r_min c^m (host loop; one D2H of the active count per round):
//  k_filter_mark  one CTA per active query walks the L trees in order (Alg. 5 lines 3-8):
//                 per tree a 16x256 LUT of squared region distances (Fig. dist, P:581-584;
//                 AMB-7) in shared memory; warps test leaf boxes (leaf LB = sum_j D_j[clamp(
//                 s_x, lo_j, hi_j)]), then the points of qualifying leaves (cell LB = sum_j
//                 D_j[code_j], AMB-12), OR them into the query's bitmap (de-duplicated union
//                 S <- S u S_i, line 6) and append first-time ids; after each tree the budget
//                 test |S| >= ceil(beta n)+k (line 7, AMB-15/17).
//  k_verify       exact squared L2 of the new candidates: one warp per row, float4 gathers,
//                 warp-shuffle reduction (lines 8/10).
//  k_topk         per query: radix-select the k smallest (d2, id) keys of old top-k u new,
//                 bitonic sort; then the radius test k-th d2 <= (c r)^2 (line 9, AMB-18).
//  k_finalize     ids (global) and sqrt(d2), ascending by (dist, id) (AMB-21, AMB-28).
#include <algorithm>
#include <cmath>
#include <vector>

#include "index.cuh"

namespace detlsh {

void project_rows(const Index& ix, const float* d_X, int64_t ld, int64_t m, float* d_P, int proj_impl,
                  int* d_nonfinite, cudaStream_t st);

namespace {

enum : int { ST_ACTIVE = 0, ST_BUDGET = 1, ST_RADIUS = 2, ST_CAP = 3 };

struct QState {  // per query of a batch
    int64_t cnt;        // |S|
    int64_t nver;       // candidates verified so far (prefix of the list)
    int32_t status;     // ST_*
    int32_t tk;         // entries in the top-k list
    int32_t trees_last;
    int32_t rounds;
    int32_t overflow;
    int32_t pad;
    unsigned long long leaves_tested, leaves_passed, points_tested, points_passed;
};

struct TreeView {
    const float* B;            // [LK][N_r+1]
    const uint32_t* leaf_off;  // [nl+1]
    const uint8_t* lo;         // [nl][K]
    const uint8_t* hi;
    const uint8_t* tcodes;     // [L*n][K]
    const uint32_t* perm;      // [L*n]
    const unsigned long long* tree_begin;  // [L+1]
    int64_t n;
    int L, K, N_r;
};

constexpr int FM_THREADS = 512;
constexpr int FM_LEAVES_PER_THREAD = 4;
constexpr int FM_CHUNK = FM_THREADS * FM_LEAVES_PER_THREAD;

template <int KT>
__global__ void __launch_bounds__(FM_THREADS) k_filter_mark(TreeView tv, const float* __restrict__ Qp,
                                                            const int* __restrict__ act, float rho2,
                                                            int64_t budget, int mode, uint32_t* __restrict__ bitmap,
                                                            int64_t nwords, uint32_t* __restrict__ cand, int64_t cap,
                                                            QState* __restrict__ qs, int round) {
    extern __shared__ float D[];                // [K][N_r] squared region distances
    __shared__ int s_sx[32];
    __shared__ int s_leaves[FM_CHUNK];
    __shared__ int s_nq;
    __shared__ unsigned long long s_new;
    __shared__ unsigned long long s_ctr[4];   // leaves tested / passed, points tested / passed
    const int K = KT ? KT : tv.K;
    const int N_r = tv.N_r, LK = tv.L * K;
    const int q = act[blockIdx.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = FM_THREADS / 32;
    const float* qp = Qp + (int64_t)q * LK;
    uint32_t* bm = bitmap + (int64_t)q * nwords;
    uint32_t* cl = cand + (int64_t)q * cap;
    int64_t cnt = qs[q].cnt;
    int status = ST_ACTIVE, trees = 0;
    const uint32_t lt = lanemask_lt();
    if (threadIdx.x < 4) s_ctr[threadIdx.x] = 0;
    uint32_t c_pt = 0, c_pp = 0;   // per-thread point counters
    for (int t = 0; t < tv.L; ++t) {
        // ---- LUT of tree t: D[j][s] = max(0, l_s - x, x - u_s)^2, cell s = (b_s, b_{s+1}]
        for (int i = threadIdx.x; i < K * N_r; i += FM_THREADS) {
            const int j = i / N_r, s = i - j * N_r;
            const float* b = tv.B + (int64_t)(t * K + j) * (N_r + 1);
            const float x = qp[t * K + j];
            const float l = s >= 1 ? b[s] : -INFINITY;
            const float u = s <= N_r - 2 ? b[s + 1] : INFINITY;
            const float v = fmaxf(0.f, fmaxf(l - x, x - u));
            D[i] = v * v;
        }
        if (threadIdx.x < K) {     // the query's own symbol s_x (AMB-6)
            const float* b = tv.B + (int64_t)(t * K + threadIdx.x) * (N_r + 1);
            const float x = qp[t * K + threadIdx.x];
            int pos = 0;
            for (int s = N_r >> 1; s > 0; s >>= 1) {
                const int idx = pos + s;               // breakpoint b_idx, idx in 1..N_r
                pos += (idx <= N_r - 1 && b[idx] < x) ? s : 0;
            }
            s_sx[threadIdx.x] = pos;
        }
        if (threadIdx.x == 0) { s_nq = 0; s_new = 0; }
        __syncthreads();
        const int64_t lb = (int64_t)tv.tree_begin[t], le = (int64_t)tv.tree_begin[t + 1];
        for (int64_t base = lb; base < le; base += FM_CHUNK) {
            // ---- leaf filter: leaf LB^2 = sum_j D_j[clamp(s_x, lo_j, hi_j)] <= rho^2
#pragma unroll
            for (int i = 0; i < FM_LEAVES_PER_THREAD; ++i) {
                const int64_t l = base + i * FM_THREADS + threadIdx.x;
                if (l < le) {
                    float acc = 0.f;
                    if (KT == 16) {
                        const uint4 lo4 = *reinterpret_cast<const uint4*>(tv.lo + l * 16);
                        const uint4 hi4 = *reinterpret_cast<const uint4*>(tv.hi + l * 16);
                        const uint32_t lw[4] = {lo4.x, lo4.y, lo4.z, lo4.w}, hw[4] = {hi4.x, hi4.y, hi4.z, hi4.w};
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const int lo = (lw[j >> 2] >> ((j & 3) * 8)) & 255, hi = (hw[j >> 2] >> ((j & 3) * 8)) & 255;
                            acc += D[j * N_r + min(max(s_sx[j], lo), hi)];
                        }
                    } else {
                        for (int j = 0; j < K; ++j)
                            acc += D[j * N_r + min(max(s_sx[j], (int)tv.lo[l * K + j]), (int)tv.hi[l * K + j])];
                    }
                    if (acc <= rho2) s_leaves[atomicAdd(&s_nq, 1)] = (int)l;
                }
            }
            __syncthreads();
            // ---- point filter + mark, one warp per qualifying leaf
            const int nq = s_nq;
            if (threadIdx.x == 0) {
                s_ctr[0] += (unsigned long long)((le - base) < FM_CHUNK ? (le - base) : FM_CHUNK);
                s_ctr[1] += (unsigned long long)nq;
            }
            for (int qi = warp; qi < nq; qi += nwarps) {
                const int l = s_leaves[qi];
                const int64_t p0 = tv.leaf_off[l], p1 = tv.leaf_off[l + 1];
                for (int64_t pb = p0; pb < p1; pb += 32) {
                    const int64_t pos = pb + lane;
                    bool isnew = false;
                    uint32_t id = 0;
                    if (pos < p1) {
                        ++c_pt;
                        bool pass = true;
                        if (mode == DETLSH_MODE_CELL) {
                            float acc = 0.f;
                            if (KT == 16) {
                                const uint4 c4 = *reinterpret_cast<const uint4*>(tv.tcodes + pos * 16);
                                const uint32_t cw[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
                                for (int j = 0; j < 16; ++j) acc += D[j * N_r + ((cw[j >> 2] >> ((j & 3) * 8)) & 255)];
                            } else {
                                for (int j = 0; j < K; ++j) acc += D[j * N_r + tv.tcodes[pos * K + j]];
                            }
                            pass = acc <= rho2;
                        }
                        if (pass) {
                            ++c_pp;
                            id = tv.perm[pos];
                            const uint32_t bit = 1u << (id & 31);
                            const uint32_t old = atomicOr(bm + (id >> 5), bit);
                            isnew = !(old & bit);
                        }
                    }
                    const uint32_t nb = __ballot_sync(0xffffffffu, isnew);
                    if (nb) {
                        unsigned long long slot0 = 0;
                        if (lane == 0) slot0 = atomicAdd(&s_new, (unsigned long long)__popc(nb));
                        slot0 = __shfl_sync(0xffffffffu, slot0, 0);
                        if (isnew) {
                            const int64_t at = cnt + (int64_t)slot0 + __popc(nb & lt);
                            if (at < cap) cl[at] = id;
                        }
                    }
                }
            }
            __syncthreads();
            if (threadIdx.x == 0) s_nq = 0;
            __syncthreads();
        }
        cnt += (int64_t)s_new;
        trees = t + 1;
        __syncthreads();
        if (cnt >= budget) { status = ST_BUDGET; break; }   // Alg. 5 line 7
    }
    for (int o = 16; o > 0; o >>= 1) {
        c_pt += __shfl_xor_sync(0xffffffffu, c_pt, o);
        c_pp += __shfl_xor_sync(0xffffffffu, c_pp, o);
    }
    if (lane == 0) {
        atomicAdd(&s_ctr[2], (unsigned long long)c_pt);
        atomicAdd(&s_ctr[3], (unsigned long long)c_pp);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        qs[q].leaves_tested += s_ctr[0];
        qs[q].leaves_passed += s_ctr[1];
        qs[q].points_tested += s_ctr[2];
        qs[q].points_passed += s_ctr[3];
        qs[q].cnt = cnt;
        qs[q].trees_last = trees;
        qs[q].rounds = round + 1;
        if (cnt > cap) qs[q].overflow = 1;
        if (status != ST_ACTIVE) qs[q].status = status;
    }
}

// ---- verify: work = chunks of VCH new candidates per active query
constexpr int VCH = 64;

__global__ void k_verify_prep(const int* __restrict__ act, int na, const QState* __restrict__ qs,
                              uint32_t* __restrict__ choff, uint32_t* __restrict__ work) {
    // single block prefix over active queries of ceil(new / VCH)
    __shared__ uint32_t s_run;
    if (threadIdx.x == 0) s_run = 0;
    __syncthreads();
    for (int base = 0; base < na; base += blockDim.x) {
        const int a = base + threadIdx.x;
        uint32_t c = 0;
        if (a < na) {
            const QState s = qs[act[a]];
            c = (uint32_t)ceil_div(s.cnt - s.nver, VCH);
        }
        // inclusive warp scan then block (blockDim == 1024)
        __shared__ uint32_t s_w[32];
        uint32_t x = c;
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_w[w] = x;
        __syncthreads();
        if (w == 0) {
            uint32_t v = s_w[lane];
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += y;
            }
            s_w[lane] = v;
        }
        __syncthreads();
        const uint32_t incl = x + (w ? s_w[w - 1] : 0);
        if (a < na) choff[a] = s_run + incl - c;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) s_run += incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        choff[na] = s_run;
        work[0] = 0;         // chunk counter
    }
}

template <int NV>
__global__ void __launch_bounds__(256) k_verify(const float* __restrict__ X, int64_t ld, const float* __restrict__ Q,
                                                const int* __restrict__ act, int na, const QState* __restrict__ qs,
                                                const uint32_t* __restrict__ choff, uint32_t* __restrict__ work,
                                                const uint32_t* __restrict__ cand, float* __restrict__ d2,
                                                int64_t cap) {
    const int lane = threadIdx.x & 31;
    const uint32_t total = choff[na];
    const int nf4 = (int)(ld / 4);
    int cur_a = -1;
    float4 qv[NV];
    for (;;) {
        uint32_t c = 0;
        if (lane == 0) c = atomicAdd(work, 1u);
        c = __shfl_sync(0xffffffffu, c, 0);
        if (c >= total) break;
        int lo = 0, hi = na - 1;                   // owner: last a with choff[a] <= c
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (choff[mid] <= c) lo = mid; else hi = mid - 1;
        }
        const int a = lo;
        const int q = act[a];
        if (a != cur_a) {
            cur_a = a;
            const float4* q4 = reinterpret_cast<const float4*>(Q + (int64_t)q * ld);
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const int f = lane + 32 * v;
                qv[v] = f < nf4 ? q4[f] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        const QState s = qs[q];
        const int64_t e0 = s.nver + (int64_t)(c - choff[a]) * VCH;
        const int64_t e1 = min(e0 + VCH, s.cnt);
        const uint32_t* cl = cand + (int64_t)q * cap;
        float* dl = d2 + (int64_t)q * cap;
        for (int64_t e = e0; e < e1; e += 4) {
            uint32_t ids[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) ids[r] = (e + r < e1) ? cl[e + r] : cl[e];
            float4 xv[4][NV];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const float4* x4 = reinterpret_cast<const float4*>(X + (int64_t)ids[r] * ld);
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const int f = lane + 32 * v;
                    xv[r][v] = f < nf4 ? __ldg(x4 + f) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
            float acc[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                float a_ = 0.f;
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const float dx = xv[r][v].x - qv[v].x, dy = xv[r][v].y - qv[v].y;
                    const float dz = xv[r][v].z - qv[v].z, dw = xv[r][v].w - qv[v].w;
                    a_ = fmaf(dx, dx, a_); a_ = fmaf(dy, dy, a_); a_ = fmaf(dz, dz, a_); a_ = fmaf(dw, dw, a_);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) a_ += __shfl_xor_sync(0xffffffffu, a_, o);
                acc[r] = a_;
            }
            if (lane < 4 && e + lane < e1) {
                float v = acc[0];
                if (lane == 1) v = acc[1];
                if (lane == 2) v = acc[2];
                if (lane == 3) v = acc[3];
                dl[e + lane] = v;
            }
        }
    }
}

// Generic-d verify (rows wider than 32*8 float4): loops over float4 columns.
__global__ void __launch_bounds__(256) k_verify_generic(const float* __restrict__ X, int64_t ld,
                                                        const float* __restrict__ Q, const int* __restrict__ act, int na,
                                                        const QState* __restrict__ qs, const uint32_t* __restrict__ choff,
                                                        uint32_t* __restrict__ work, const uint32_t* __restrict__ cand,
                                                        float* __restrict__ d2, int64_t cap) {
    const int lane = threadIdx.x & 31;
    const uint32_t total = choff[na];
    const int nf4 = (int)(ld / 4);
    for (;;) {
        uint32_t c = 0;
        if (lane == 0) c = atomicAdd(work, 1u);
        c = __shfl_sync(0xffffffffu, c, 0);
        if (c >= total) break;
        int lo = 0, hi = na - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (choff[mid] <= c) lo = mid; else hi = mid - 1;
        }
        const int q = act[lo];
        const QState s = qs[q];
        const int64_t e0 = s.nver + (int64_t)(c - choff[lo]) * VCH;
        const int64_t e1 = min(e0 + VCH, s.cnt);
        const float4* q4 = reinterpret_cast<const float4*>(Q + (int64_t)q * ld);
        for (int64_t e = e0; e < e1; ++e) {
            const float4* x4 = reinterpret_cast<const float4*>(X + (int64_t)cand[(int64_t)q * cap + e] * ld);
            float a_ = 0.f;
            for (int f = lane; f < nf4; f += 32) {
                const float4 x = __ldg(x4 + f), y = q4[f];
                const float dx = x.x - y.x, dy = x.y - y.y, dz = x.z - y.z, dw = x.w - y.w;
                a_ = fmaf(dx, dx, a_); a_ = fmaf(dy, dy, a_); a_ = fmaf(dz, dz, a_); a_ = fmaf(dw, dw, a_);
            }
            for (int o = 16; o > 0; o >>= 1) a_ += __shfl_xor_sync(0xffffffffu, a_, o);
            if (lane == 0) d2[(int64_t)q * cap + e] = a_;
        }
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

__global__ void __launch_bounds__(TK_THREADS) k_topk(const int* __restrict__ act, QState* __restrict__ qs,
                                                     const uint32_t* __restrict__ cand, const float* __restrict__ d2,
                                                     int64_t cap, unsigned long long* __restrict__ topk, int k,
                                                     float cr2, int round) {
    __shared__ unsigned long long s_keys[TK_MAX];
    __shared__ uint32_t s_hist[256];
    __shared__ unsigned long long s_prefix, s_mask, s_rem;
    __shared__ int s_n;
    const int q = act[blockIdx.x];
    QState s = qs[q];
    unsigned long long* tk = topk + (int64_t)q * k;
    const uint32_t* cl = cand + (int64_t)q * cap;
    const float* dl = d2 + (int64_t)q * cap;
    const int64_t old = s.tk, e0 = s.nver, nn = s.cnt - s.nver, M = old + nn;
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
        // radix select of the k-th smallest key, 8 digits of 8 bits
        for (int pass = 0; pass < 8; ++pass) {
            const int shift = 56 - 8 * pass;
            for (int i = threadIdx.x; i < 256; i += TK_THREADS) s_hist[i] = 0;
            __syncthreads();
            const unsigned long long pre = s_prefix, msk = s_mask;
            for (int64_t i = threadIdx.x; i < M; i += TK_THREADS) {
                const unsigned long long key = key_at(i);
                if ((key & msk) == pre) atomicAdd(&s_hist[(key >> shift) & 255u], 1u);
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                unsigned long long cum = 0, rem = s_rem;
                for (int dg = 0; dg < 256; ++dg) {
                    if (cum + s_hist[dg] >= rem) {
                        s_prefix = pre | ((unsigned long long)dg << shift);
                        s_mask = msk | (0xFFull << shift);
                        s_rem = rem - cum;
                        break;
                    }
                    cum += s_hist[dg];
                }
            }
            __syncthreads();
        }
        const unsigned long long T = s_prefix;   // keys are unique: exactly k keys <= T
        for (int64_t i = threadIdx.x; i < M; i += TK_THREADS) {
            const unsigned long long key = key_at(i);
            if (key <= T) s_keys[atomicAdd(&s_n, 1)] = key;
        }
        outn = k;
    }
    __syncthreads();
    int n2 = 1;
    while (n2 < outn) n2 <<= 1;
    for (int i = outn + threadIdx.x; i < n2; i += TK_THREADS) s_keys[i] = ~0ull;
    __syncthreads();
    bitonic_sort_smem(s_keys, n2);
    for (int i = threadIdx.x; i < outn; i += TK_THREADS) tk[i] = s_keys[i];
    if (threadIdx.x == 0) {
        s.tk = outn;
        s.nver = s.cnt;
        if (s.status == ST_ACTIVE) {
            if (outn >= k && __uint_as_float((uint32_t)(s_keys[k - 1] >> 32)) <= cr2) s.status = ST_RADIUS;  // line 9
            else if (round == 63) s.status = ST_CAP;                                                        // AMB-20
        }
        qs[q] = s;
    }
}

__global__ void k_compact(const int* __restrict__ act, int na, const QState* __restrict__ qs, int* __restrict__ act_out,
                          int* __restrict__ n_out) {
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

__global__ void k_finalize(const QState* __restrict__ qs, const unsigned long long* __restrict__ topk, int nqb, int k,
                           int64_t id_offset, const double* __restrict__ radii, int64_t* __restrict__ out_ids,
                           float* __restrict__ out_d, detlsh_query_stats* __restrict__ stats) {
    const int64_t total = (int64_t)nqb * k;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int q = (int)(i / k), e = (int)(i % k);
        const QState s = qs[q];
        if (e < s.tk) {
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
            o.leaves_tested = (int64_t)s.leaves_tested;
            o.leaves_passed = (int64_t)s.leaves_passed;
            o.points_tested = (int64_t)s.points_tested;
            o.points_passed = (int64_t)s.points_passed;
            stats[q] = o;
        }
    }
}

__global__ void k_init_batch(QState* __restrict__ qs, int* __restrict__ act, int nqb) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nqb; q += gridDim.x * blockDim.x) {
        QState s;
        s.cnt = 0; s.nver = 0; s.status = ST_ACTIVE; s.tk = 0; s.trees_last = 0; s.rounds = 0;
        s.overflow = 0; s.pad = 0;
        s.leaves_tested = s.leaves_passed = s.points_tested = s.points_passed = 0;
        qs[q] = s;
        act[q] = q;
    }
}

}  // namespace

void query_index(const Index& ix, const float* d_Q, int64_t q_ld, const QueryArgs& a, int64_t* d_ids,
                 float* d_dists, detlsh_query_stats* d_stats, cudaStream_t st) {
    DL_REQUIRE(q_ld == ix.ld, "query row stride must equal the index's");
    const int64_t n = ix.n, nq = a.nq, LK = ix.LK;
    const int k = a.k;
    const int64_t budget = (int64_t)std::ceil(a.beta * (double)n) + k;   // AMB-17
    const int64_t nwords = ceil_div(n, 32);
    const int64_t cap = n;                                              // |S| <= n always

    // Q0: project all queries once
    Scratch s_qp(st, sizeof(float) * (size_t)(nq * LK));
    Scratch s_flag(st, sizeof(int));
    DL_CUDA(cudaMemsetAsync(s_flag.p, 0, sizeof(int), st));
    project_rows(ix, d_Q, q_ld, nq, s_qp.as<float>(), a.proj_impl, s_flag.as<int>(), st);
    {
        int bad = 0;
        DL_CUDA(cudaMemcpyAsync(&bad, s_flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        DL_CUDA(cudaStreamSynchronize(st));
        DL_REQUIRE(!bad, "queries contain NaN or Inf");
    }

    // batch size from the memory budget: bitmap + candidate list + distances per query
    const int64_t per_q = nwords * 4 + cap * 8 + (int64_t)k * 8 + 64;
    int64_t budget_bytes = a.mem_budget;
    if (budget_bytes <= 0) {
        size_t fr = 0, tot = 0;
        DL_CUDA(cudaMemGetInfo(&fr, &tot));
        budget_bytes = (int64_t)(fr * 0.6);
    }
    int64_t qb = a.query_batch > 0 ? a.query_batch : std::max<int64_t>(1, budget_bytes / per_q);
    qb = std::min<int64_t>({qb, nq, 65535});
    DL_REQUIRE(qb >= 1, "not enough device memory for one query");

    Scratch s_bm(st, sizeof(uint32_t) * (size_t)(qb * nwords));
    Scratch s_cand(st, sizeof(uint32_t) * (size_t)(qb * cap));
    Scratch s_d2(st, sizeof(float) * (size_t)(qb * cap));
    Scratch s_tk(st, sizeof(unsigned long long) * (size_t)(qb * k));
    Scratch s_qs(st, sizeof(QState) * (size_t)qb);
    Scratch s_act(st, sizeof(int) * (size_t)(2 * qb + 2));
    Scratch s_ch(st, sizeof(uint32_t) * (size_t)(qb + 2));
    Scratch s_radii(st, sizeof(double) * 64);
    int* act = s_act.as<int>();
    int* act2 = act + qb;
    int* n_act = act2 + qb;
    uint32_t* choff = s_ch.as<uint32_t>();
    uint32_t* work = choff + qb + 1;

    const double eps = ix.eps;
    std::vector<double> radii(64);
    {
        double r = a.r_min;
        for (int m = 0; m < 64; ++m) { radii[m] = r; r = a.c * r; }   // r <- c r (line 11), AMB-19
    }
    DL_CUDA(cudaMemcpyAsync(s_radii.p, radii.data(), sizeof(double) * 64, cudaMemcpyHostToDevice, st));

    TreeView tv;
    tv.B = ix.B.as<float>();
    tv.leaf_off = ix.leaf_off.as<uint32_t>();
    tv.lo = ix.leaf_lo.as<uint8_t>();
    tv.hi = ix.leaf_hi.as<uint8_t>();
    tv.tcodes = ix.tcodes.as<uint8_t>();
    tv.perm = ix.perm.as<uint32_t>();
    Scratch s_tb(st, sizeof(unsigned long long) * (size_t)(ix.L + 1));
    {
        std::vector<unsigned long long> tb(ix.tree_leaf_begin.begin(), ix.tree_leaf_begin.end());
        DL_CUDA(cudaMemcpyAsync(s_tb.p, tb.data(), sizeof(unsigned long long) * tb.size(), cudaMemcpyHostToDevice, st));
    }
    tv.tree_begin = s_tb.as<unsigned long long>();
    tv.n = n;
    tv.L = ix.L;
    tv.K = ix.K;
    tv.N_r = ix.N_r;

    const size_t lut_smem = sizeof(float) * (size_t)ix.K * ix.N_r;
    auto k_filter_mark_sel = ix.K == 16 ? k_filter_mark<16> : k_filter_mark<0>;
    DL_CUDA(cudaFuncSetAttribute(k_filter_mark_sel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lut_smem));
    const int nv = (int)ceil_div(ix.ld / 4, 32);
    int vgrid = 148 * 8;

    for (int64_t q0 = 0; q0 < nq; q0 += qb) {
        const int nqb = (int)std::min<int64_t>(qb, nq - q0);
        const float* Qb = d_Q + q0 * q_ld;
        const float* Qpb = s_qp.as<float>() + q0 * LK;
        DL_CUDA(cudaMemsetAsync(s_bm.p, 0, sizeof(uint32_t) * (size_t)(nqb * nwords), st));
        DL_LAUNCH(k_init_batch, (unsigned)ceil_div(nqb, 256), 256, 0, st, s_qs.as<QState>(), act, nqb);
        int na = nqb;
        int* cur = act;
        int* nxt = act2;
        for (int m = 0; m < 64 && na > 0; ++m) {
            const double r = radii[m];
            const float rho2 = (float)((eps * r) * (eps * r));
            const float cr2 = (float)((a.c * r) * (a.c * r));
            DL_LAUNCH(k_filter_mark_sel, (unsigned)na, FM_THREADS, lut_smem, st, tv, Qpb, cur, rho2, budget, a.mode, s_bm.as<uint32_t>(),
                      nwords, s_cand.as<uint32_t>(), cap, s_qs.as<QState>(), m);
            DL_LAUNCH(k_verify_prep, 1, 1024, 0, st, cur, na, s_qs.as<QState>(), choff, work);
            switch (nv) {
                case 1: DL_LAUNCH(k_verify<1>, vgrid, 256, 0, st, ix.Xp, ix.ld, Qb, cur, na, s_qs.as<QState>(), choff, work,
                                  s_cand.as<uint32_t>(), s_d2.as<float>(), cap); break;
                case 2: DL_LAUNCH(k_verify<2>, vgrid, 256, 0, st, ix.Xp, ix.ld, Qb, cur, na, s_qs.as<QState>(), choff, work,
                                  s_cand.as<uint32_t>(), s_d2.as<float>(), cap); break;
                case 3: case 4: DL_LAUNCH(k_verify<4>, vgrid, 256, 0, st, ix.Xp, ix.ld, Qb, cur, na, s_qs.as<QState>(), choff,
                                  work, s_cand.as<uint32_t>(), s_d2.as<float>(), cap); break;
                case 5: case 6: case 7: case 8:
                    DL_LAUNCH(k_verify<8>, vgrid, 256, 0, st, ix.Xp, ix.ld, Qb, cur, na, s_qs.as<QState>(), choff, work,
                              s_cand.as<uint32_t>(), s_d2.as<float>(), cap); break;
                default:
                    DL_LAUNCH(k_verify_generic, vgrid, 256, 0, st, ix.Xp, ix.ld, Qb, cur, na, s_qs.as<QState>(), choff,
                              work, s_cand.as<uint32_t>(), s_d2.as<float>(), cap);
            }
            DL_LAUNCH(k_topk, (unsigned)na, TK_THREADS, 0, st, cur, s_qs.as<QState>(), s_cand.as<uint32_t>(),
                      s_d2.as<float>(), cap, s_tk.as<unsigned long long>(), k, cr2, m);
            DL_LAUNCH(k_compact, 1, 1024, 0, st, cur, na, s_qs.as<QState>(), nxt, n_act);
            DL_CUDA(cudaMemcpyAsync(&na, n_act, sizeof(int), cudaMemcpyDeviceToHost, st));
            DL_CUDA(cudaStreamSynchronize(st));
            std::swap(cur, nxt);
        }
        DL_LAUNCH(k_finalize, (unsigned)std::min<int64_t>(ceil_div((int64_t)nqb * k, 256), 148 * 16), 256, 0, st,
                  s_qs.as<QState>(), s_tk.as<unsigned long long>(), nqb, k, ix.id_offset, s_radii.as<double>(),
                  d_ids + q0 * k, d_dists + q0 * k, d_stats ? d_stats + q0 : nullptr);
    }
}

}  // namespace detlsh
