// project_tc.cu -- P = X A^T on the 5th-generation tensor cores (tcgen05, kind::tf32),
// the projection of every point onto the L*K Gaussian directions (Eq. 1 P:192-196, P:296;
// Alg. 5 line 4 P:431 for queries).
//
// Precision: A is TF32-exact by construction (AMB-1), so P = X A^T needs only X split into
// hi + lo:  the tensor core reads an fp32 operand as TF32 by dropping the low 13 mantissa
// bits, so MMA(x) = MMA(trunc(x)), and lo = x - trunc(x) (exact in fp32) carries the rest:
// P ~= trunc(x).A + trunc(lo).A with |error| <~ 2^-20 ||x|| ||a||  ("2xTF32").
//
// Kernel (persistent, one CTA per SM, 18 warps = 576 threads, tiles of 128 rows):
//   warp 0          TMA producer: X k-blocks [128 rows x 32 fp32] (SWIZZLE_128B) into a ring of
//                   stages; the whole (L*K_pad x ld) hash matrix once (resident in smem), or one
//                   k-block of it per stage beside the rows when it does not fit (streamA, d = 960).
//   warp 1          TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=L*K_pad, K=8):
//                   per k-block 4 MMAs on x and 4 on lo, accumulating in TMEM; tcgen05.commit
//                   frees the stage and, after the last k-block, hands the tile to the epilogue.
//   warps 2-3, 12-17  8 converter warps: lo = x - trunc_tf32(x) into a twin buffer of the same
//                   swizzled layout (+ ||x||^2 of the rows, the non-finite flag),
//                   fence.proxy.async, arrive.
//   warps 4-11      8 epilogue warps: tcgen05.ld (32x32b) of the double-buffered accumulator ->
//                   projections, or (fused Alg. 1) 8-bit codes by a branch-free Eytzinger search.
#include <cuda.h>

#include <cstdlib>

#include "index.cuh"
#include "tc_util.cuh"

namespace detlsh {

namespace {
using namespace tc;

constexpr int TC_M = 128;           // rows per tile (UMMA M)
constexpr int TC_KB = 32;           // fp32 per k-block (= 128 B, one swizzle row)
constexpr int TC_THREADS = 576;    // 18 warps: producer, MMA, 8 converters (2-3, 12-17), 8 epilogue (4-11)
constexpr int TC_CONV = 256;       // converter threads
constexpr int TC_CM = TC_M * TC_KB / 4 / TC_CONV;   // float4 per converter thread per stage
constexpr int TC_EPI = 256;        // epilogue threads
constexpr int TC_STAGE_BYTES = TC_M * TC_KB * 4;   // 16 KB

struct TcShape {
    int64_t m;        // rows
    int ld;           // row stride (floats), padded columns are zero
    int nkb;          // k-blocks = ceil(ld / 32)
    int LK, npad;     // output columns, padded to a multiple of 16
    int stages;
    uint32_t tmem_cols;
    int N_r;          // > 0: fused Alg. 1 encode, codes instead of projections
    int lgP;          // encode table entries per column = 2^lgP >= N_r (Eytzinger order)
    int streamA;      // 1: the hash matrix does not fit in shared memory -- its k-block is loaded
                      // into every stage beside the rows (re-read from L2 per tile)
    int dbg;          // experiments only (DETLSH_PROJ_DEBUG): 1 no encode search, 2 no conversion, 4 no MMA
    int ta;           // 1: the lo parts go to tensor memory (tcgen05.st by the converters) and the second
                      // MMA of each k-step reads its A operand from there -- no lo buffer in shared
                      // memory (more stages), no shared-memory store / MMA re-read of it
    uint32_t lo_col;  // ta: first TMEM column of the S lo buffers (32 columns each)
};

__global__ void __launch_bounds__(TC_THREADS, 1)
    k_project_tc(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmA, TcShape sh,
                 float* __restrict__ P, int* __restrict__ nonfinite, const float* __restrict__ B,
                 uint8_t* __restrict__ EP, float* __restrict__ xnorm, uint32_t* __restrict__ fkey) {
    pdl_wait();
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte alignment of every swizzled buffer
    // 1024-byte aligned, by pointer arithmetic on the shared array (keeps the shared address
    // space: LDS/STS instead of generic LD/ST)
    unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int S = sh.stages;
    unsigned char* sB = base;                                            // nkb (or S if streamA) x [npad][128 B]
    unsigned char* sX = sB + (size_t)(sh.streamA ? S : sh.nkb) * sh.npad * 128;   // S x 16 KB
    unsigned char* sL = sX + (size_t)S * TC_STAGE_BYTES;                  // S x 16 KB (lo parts; none if ta)
    float* sT = reinterpret_cast<float*>(sL + (sh.ta ? 0 : (size_t)S * TC_STAGE_BYTES));   // encode table [LK][2^lgP] (Eytzinger)
    __shared__ float s_np[2][TC_M];       // ta: ||x||^2 of the second half of each row's columns
    const int tab_floats = sh.N_r > 0 ? sh.LK << sh.lgP : 0;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sT + tab_floats);
    uint64_t* full = bars;              // [S] TMA -> converters, MMA
    uint64_t* conv = bars + S;          // [S] converters -> MMA
    uint64_t* empty = bars + 2 * S;     // [S] MMA commit -> producer
    uint64_t* tfull = bars + 3 * S;     // [2] MMA commit -> epilogue
    uint64_t* tempty = bars + 3 * S + 2;// [2] epilogue -> MMA
    uint64_t* bfull = bars + 3 * S + 4; // hash matrix loaded
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * S + 5);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t ntiles = (sh.m + TC_M - 1) / TC_M;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&conv[s], TC_CONV);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], TC_EPI);
        }
        mbar_init(bfull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {   // TMEM allocation (whole warp), base column written to smem
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(sh.tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            if (!sh.streamA) {   // the hash matrix, once
                mbar_expect_tx(bfull, (uint32_t)(sh.nkb * sh.npad * 128));
                for (int kb = 0; kb < sh.nkb; ++kb) tma_load_2d(sB + (size_t)kb * sh.npad * 128, &tmA, bfull, kb * TC_KB, 0);
            } else {
                mbar_arrive(bfull);
            }
            int s = 0;
            uint32_t ph = 0;
            for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                for (int kb = 0; kb < sh.nkb; ++kb) {
                    mbar_wait(&empty[s], ph ^ 1);
                    mbar_expect_tx(&full[s], TC_STAGE_BYTES + (sh.streamA ? (uint32_t)(sh.npad * 128) : 0u));
                    tma_load_2d(sX + (size_t)s * TC_STAGE_BYTES, &tmX, &full[s], kb * TC_KB, (int)(tile * TC_M));
                    if (sh.streamA) tma_load_2d(sB + (size_t)s * sh.npad * 128, &tmA, &full[s], kb * TC_KB, 0);
                    if (++s == S) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(sh.npad >> 3) << 17) |
                                   ((uint32_t)(TC_M >> 4) << 24);
            mbar_wait(bfull, 0);
            int s = 0;
            uint32_t ph = 0;
            int buf = 0;
            uint32_t tph = 0;
            for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                mbar_wait(&tempty[buf], tph ^ 1);          // epilogue released this accumulator
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + (uint32_t)(buf * sh.npad);
                for (int kb = 0; kb < sh.nkb; ++kb) {
                    mbar_wait(&full[s], ph);
                    mbar_wait(&conv[s], ph);
                    tc_fence_after();
                    const uint32_t ax = smem_u32(sX + (size_t)s * TC_STAGE_BYTES);
                    const uint32_t al = smem_u32(sL + (size_t)s * TC_STAGE_BYTES);
                    const uint32_t bb = smem_u32(sB + (size_t)(sh.streamA ? s : kb) * sh.npad * 128);
                    if (!(sh.dbg & 4)) {
                        if (sh.ta) {
                            const uint32_t ta_lo = tmem_base + sh.lo_col + (uint32_t)(s * TC_KB);
#pragma unroll
                            for (int k = 0; k < TC_KB / 8; ++k) {
                                const uint64_t bd = desc_sw128(bb + k * 32);
                                mma_tf32(d_tmem, desc_sw128(ax + k * 32), bd, idesc, (kb | k) ? 1u : 0u);
                                mma_tf32_ta(d_tmem, ta_lo + (uint32_t)(8 * k), bd, idesc, 1u);
                            }
                        } else {
#pragma unroll
                            for (int k = 0; k < TC_KB / 8; ++k) {        // K = 8 tf32 per MMA = 32 bytes
                                const uint64_t bd = desc_sw128(bb + k * 32);
                                mma_tf32(d_tmem, desc_sw128(ax + k * 32), bd, idesc, (kb | k) ? 1u : 0u);
                                mma_tf32(d_tmem, desc_sw128(al + k * 32), bd, idesc, 1u);
                            }
                        }
                    }
                    mma_commit(&empty[s]);                   // stage free once these MMAs complete
                    if (++s == S) { s = 0; ph ^= 1; }
                }
                mma_commit(&tfull[buf]);                     // accumulator ready
                if (++buf == 2) { buf = 0; tph ^= 1; }
            }
        }
    } else if ((warp < 4 || warp >= 12) && sh.ta) {
        // converters, tensor-memory form: thread = row (32 qd + lane) of its warp's TMEM lane quarter
        // qd, half h of the k-block's 32 columns (the quarter's two converter warps split them):
        // x from the 128B-swizzled stage (chunk c of row r at c ^ (r & 7)), lo = x - trunc_tf32(x)
        // stored to 16 TMEM columns, waited, fenced, then the stage's conversion barrier.
        const int qd = warp & 3, h = warp >= 14 ? 1 : 0;
        const int r = qd * 32 + lane;
        int s = 0;
        uint32_t ph = 0;
        bool bad = false;
        int par = 0;
        const uint32_t trow = tmem_base + ((uint32_t)(qd * 32) << 16) + sh.lo_col + (uint32_t)(16 * h);
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            float nacc = 0.f;
            for (int kb = 0; kb < sh.nkb; ++kb) {
                mbar_wait(&full[s], ph);
                const unsigned char* rowp = sX + (size_t)s * TC_STAGE_BYTES + (size_t)r * 128;
                float lo[16];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const float4 x = *reinterpret_cast<const float4*>(rowp + (((4 * h + c) ^ (r & 7)) << 4));
                    const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        lo[4 * c + e] = xs[e] - __uint_as_float(__float_as_uint(xs[e]) & 0xFFFFE000u);
                        bad |= !isfinite(xs[e]);
                        nacc = fmaf(xs[e], xs[e], nacc);
                    }
                }
                tmem_st16(trow + (uint32_t)(s * TC_KB), lo);
                tc_fence_before();
                mbar_arrive(&conv[s]);
                if (++s == S) { s = 0; ph ^= 1; }
            }
            if (xnorm) {   // the row's two halves: h = 1 hands its sum over, h = 0 writes the norm
                if (h) s_np[par][r] = nacc;
                asm volatile("bar.sync 2, 256;" ::: "memory");   // the 8 converter warps
                const int64_t row = tile * TC_M + r;
                if (!h && row < sh.m) xnorm[row] = nacc + s_np[par][r];
                par ^= 1;
            }
        }
        if (bad) atomicOr(nonfinite, 1);
    } else if (warp < 4 || warp >= 12) {
        // converters (TC_CONV threads): lo = x - trunc_tf32(x), same swizzled offsets.  Thread t sees
        // float4 t + TC_CONV m (m < TC_CM) of every stage, i.e. rows t/8 + (TC_CONV/8) m (swizzling
        // permutes 16-byte chunks only within a row), so it also accumulates those rows' ||x||^2.
        const int t = warp < 4 ? threadIdx.x - 64 : threadIdx.x - 384 + 64;
        int s = 0;
        uint32_t ph = 0;
        bool bad = false;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            float nacc[TC_CM];
#pragma unroll
            for (int m = 0; m < TC_CM; ++m) nacc[m] = 0.f;
            for (int kb = 0; kb < sh.nkb; ++kb) {
                mbar_wait(&full[s], ph);
                const float4* src = reinterpret_cast<const float4*>(sX + (size_t)s * TC_STAGE_BYTES);
                float4* dst = reinterpret_cast<float4*>(sL + (size_t)s * TC_STAGE_BYTES);
#pragma unroll
                for (int m = 0; m < ((sh.dbg & 2) ? 0 : TC_CM); ++m) {
                    const int i = t + TC_CONV * m;
                    const float4 x = src[i];
                    float4 lo;
                    lo.x = x.x - __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
                    lo.y = x.y - __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
                    lo.z = x.z - __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
                    lo.w = x.w - __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
                    bad |= !(isfinite(x.x) && isfinite(x.y) && isfinite(x.z) && isfinite(x.w));
                    dst[i] = lo;
                    nacc[m] = fmaf(x.x, x.x, fmaf(x.y, x.y, fmaf(x.z, x.z, fmaf(x.w, x.w, nacc[m]))));
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive(&conv[s]);
                if (++s == S) { s = 0; ph ^= 1; }
            }
            if (xnorm) {
#pragma unroll
                for (int m = 0; m < TC_CM; ++m) {
                    float v = nacc[m];
                    v += __shfl_xor_sync(0xffffffffu, v, 1);
                    v += __shfl_xor_sync(0xffffffffu, v, 2);
                    v += __shfl_xor_sync(0xffffffffu, v, 4);
                    const int64_t row = tile * TC_M + (t >> 3) + (TC_CONV / 8) * m;
                    if ((t & 7) == 0 && row < sh.m) xnorm[row] = v;
                }
            }
        }
        if (bad) atomicOr(nonfinite, 1);
    } else {
        // epilogue (warps 4-11): TMEM -> registers -> P rows, or (fused Alg. 1) -> 8-bit codes;
        // TMEM lane quarter ew = warp % 4, the two warps of a quarter take alternate 16-column chunks
        const int ew = warp & 3, eh = (warp - 4) >> 2;
        const int row_in_tile = ew * 32 + lane;
        const int N_r = sh.N_r;
        // breakpoint table per column r: c[t] = b_{t+1} (t < N_r-1), +inf beyond (AMB-6/7), padded to
        // NP = 2^lg entries and stored in Eytzinger (breadth-first) order: node k = 2^l + j of level l
        // holds c[j*(P>>l) + (P>>(l+1)) - 1], the element the l-th step of the lower-bound search
        // compares.  The nodes of one level are contiguous, so the 32 lanes of a step (32 rows, one
        // column) hit distinct banks for the first 6 levels instead of colliding on a few.
        const int lg = sh.lgP, NP = 1 << lg;
        if (N_r > 0) {
            for (int i = threadIdx.x - 128; i < tab_floats; i += TC_EPI) {
                const int r = i >> lg, k = i & (NP - 1);
                float c = 0.f;
                if (k > 0) {
                    const int l = 31 - __clz(k), j = k - (1 << l);
                    const int t = j * (NP >> l) + (NP >> (l + 1)) - 1;
                    c = t < N_r - 1 ? B[(int64_t)r * (N_r + 1) + t + 1] : __int_as_float(0x7f800000);
                }
                sT[i] = c;
            }
            asm volatile("bar.sync 1, 256;" ::: "memory");  // epilogue warps only
        }
        int buf = 0;
        uint32_t tph = 0;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            mbar_wait(&tfull[buf], tph);
            tc_fence_after();
            const int64_t row = tile * TC_M + row_in_tile;
            const uint32_t taddr = tmem_base + (uint32_t)(buf * sh.npad) + ((uint32_t)(ew * 32) << 16);
            for (int c0 = 16 * eh; c0 < sh.npad; c0 += 32) {
                float v[16];
                tmem_ld16(taddr + c0, v);
                if (N_r > 0) {
                    // code = #{t in 1..N_r-1 : b_t < x}: branch-free lower bound, k -> 2k + [c_k < x]
                    // down the Eytzinger tree, code = k - NP; the 16 searches advance together
                    // (16 independent shared loads per step)
                    int pos[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) pos[i] = 1;
                    for (int l = (sh.dbg & 1) ? lg : 0; l < lg; ++l) {
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const int r = min(c0 + i, sh.LK - 1);
                            pos[i] = 2 * pos[i] + ((sT[(r << lg) + pos[i]] < v[i]) ? 1 : 0);
                        }
                    }
                    uint32_t packed[4] = {0, 0, 0, 0};
#pragma unroll
                    for (int i = 0; i < 16; ++i) packed[i >> 2] |= (uint32_t)(pos[i] - NP) << (8 * (i & 3));
                    // (K = 16: the chunk is tree c0/16) the tree's first-layer key for the build's
                    // sort, Alg. 2 l.2: the top bit of each dim's symbol, dim 0 most significant
                    if (fkey != nullptr && row < sh.m) {
                        uint32_t key = 0;
#pragma unroll
                        for (int i = 0; i < 16; ++i) key = (key << 1) | (((uint32_t)(pos[i] - NP) >> (lg - 1)) & 1u);
                        fkey[(int64_t)(c0 >> 4) * sh.m + row] = key;
                    }
                    if (row < sh.m) {
                        uint8_t* out = EP + row * sh.LK + c0;
                        if (c0 + 16 <= sh.LK && (sh.LK & 15) == 0) {
                            *reinterpret_cast<uint4*>(out) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
                        } else {
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                if (c0 + i < sh.LK) out[i] = (uint8_t)(packed[i >> 2] >> (8 * (i & 3)));
                        }
                    }
                }
                if (P != nullptr && row < sh.m) {   // projections (also kept beside the codes for EXACT mode)
                    float* out = P + row * sh.LK + c0;
                    if (c0 + 16 <= sh.LK && (sh.LK & 3) == 0) {
#pragma unroll
                        for (int i = 0; i < 16; i += 4)
                            *reinterpret_cast<float4*>(out + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                    } else {
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            if (c0 + i < sh.LK) out[i] = v[i];
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty[buf]);
            if (++buf == 2) { buf = 0; tph ^= 1; }
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(sh.tmem_cols));
    }
}

}  // namespace

// Returns false when the shape does not fit this kernel (resident hash matrix too large).
// B != nullptr: fused encode (Alg. 1) -- writes codes EP[m][LK] instead of P.
static bool launch_tc(const Index& ix, const float* d_X, int64_t ld, int64_t m, float* d_P, int* d_nonfinite,
                      const float* B, uint8_t* EP, float* xnorm, cudaStream_t st, uint32_t* fkey = nullptr) {
    if (m <= 0) return true;
    TcShape sh;
    sh.m = m;
    sh.ld = (int)ld;
    sh.nkb = (int)ceil_div(ld, TC_KB);
    sh.LK = ix.LK;
    sh.npad = (int)round_up(ix.LK, 16);
    sh.N_r = B ? ix.N_r : 0;
    sh.lgP = 0;
    while ((1 << sh.lgP) < ix.N_r) ++sh.lgP;
    if (sh.npad > 256) return false;
    const size_t abytes = (size_t)sh.npad * 128;                 // one k-block of the hash matrix
    const size_t tbytes = B ? sizeof(float) * ((size_t)ix.LK << sh.lgP) : 0;
    const size_t fixed = 1024 /*align*/ + 256 /*barriers*/;
    const size_t budget = 226 * 1024;     // + 1 KB of static shared memory (s_np) within the 227 KB
    static const int force_stream = std::getenv("DETLSH_STREAM_A") ? std::atoi(std::getenv("DETLSH_STREAM_A")) : 0;
    static const int pdbg = std::getenv("DETLSH_PROJ_DEBUG") ? std::atoi(std::getenv("DETLSH_PROJ_DEBUG")) : 0;
    sh.dbg = pdbg;
    // DETLSH_PROJ_TA: 1 = lo parts in tensor memory (default off until measured), 0 = shared memory
    static const int ta_env = std::getenv("DETLSH_PROJ_TA") ? std::atoi(std::getenv("DETLSH_PROJ_TA")) : 0;
    sh.lo_col = (uint32_t)(2 * sh.npad);
    // accumulators (2 x npad columns) + one 32-column lo buffer per stage within 512 columns
    sh.ta = (ta_env && (int)((512 - sh.lo_col) / TC_KB) >= 2) ? 1 : 0;
    const int spb = sh.ta ? 1 : 2;                               // 16 KB stage buffers per stage
    sh.streamA = (force_stream || (size_t)sh.nkb * abytes + tbytes + fixed + 2 * spb * TC_STAGE_BYTES > budget) ? 1 : 0;
    const int max_st = sh.ta ? std::min<int>(8, (int)((512 - sh.lo_col) / TC_KB)) : 6;
    if (!sh.streamA) {
        const size_t bbytes = (size_t)sh.nkb * abytes;
        sh.stages = (int)std::min<size_t>(max_st, (budget - bbytes - tbytes - fixed) / (spb * TC_STAGE_BYTES));
    } else {
        const size_t per = spb * TC_STAGE_BYTES + abytes;
        if (tbytes + fixed + 2 * per > budget) return false;
        sh.stages = (int)std::min<size_t>(max_st, (budget - tbytes - fixed) / per);
    }
    const size_t bbytes = (size_t)(sh.streamA ? sh.stages : sh.nkb) * abytes;
    uint32_t cols = 32;
    while (cols < (uint32_t)(2 * sh.npad + (sh.ta ? TC_KB * sh.stages : 0))) cols <<= 1;
    sh.tmem_cols = cols;
    const size_t smem = bbytes + tbytes + (size_t)sh.stages * spb * TC_STAGE_BYTES + fixed;
    CUtensorMap mx, ma;
    make_map(&mx, d_X, m, (int)ld, TC_M);
    make_map(&ma, ix.A.as<float>(), ix.LK, (int)ld, sh.npad);
    ensure_dyn_smem_fn(k_project_tc, smem);
    int dev = 0, nsm = 148;
    DL_CUDA(cudaGetDevice(&dev));
    DL_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const int64_t ntiles = ceil_div(m, TC_M);
    const int grid = (int)std::min<int64_t>(ntiles, nsm);
    DL_LAUNCH(k_project_tc, grid, TC_THREADS, smem, st, mx, ma, sh, d_P, d_nonfinite, B, EP, xnorm,
              (fkey && ix.K == 16 && (ix.LK & 15) == 0 && (1 << sh.lgP) == ix.N_r) ? fkey : (uint32_t*)nullptr);
    return true;
}

bool project_rows_tc(const Index& ix, const float* d_X, int64_t ld, int64_t m, float* d_P, int* d_nonfinite,
                     cudaStream_t st) {
    return launch_tc(ix, d_X, ld, m, d_P, d_nonfinite, nullptr, nullptr, nullptr, st);
}

bool project_encode_tc(const Index& ix, const float* d_X, int64_t ld, int64_t m, uint8_t* d_EP, int* d_nonfinite,
                       float* d_xnorm, float* d_P, cudaStream_t st, uint32_t* d_fkey) {
    return launch_tc(ix, d_X, ld, m, d_P, d_nonfinite, ix.B.as<float>(), d_EP, d_xnorm, st, d_fkey);
}

}  // namespace detlsh
