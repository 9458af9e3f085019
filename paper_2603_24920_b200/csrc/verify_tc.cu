// verify_tc.cu -- candidate verification (Alg. 5 lines 8/10) on the tcgen05
// tensor cores.
//
// Every member of S not yet verified needs its exact squared distance to the query.  At the
// configurations' radii S covers ~11% of all (point, query) pairs of a round, so the work is
// a masked dense contraction: the kernel computes G = X_tile . Q_tile^T for 128-row x N-query
// tiles on the tensor cores and the epilogue keeps only the pairs whose bit is set in the
// query's "new members of S" bitmap, with
//     d2(x, q) = ||x||^2 + ||q||^2 - 2 x.q .
// The SIMT kernel it replaces (k_verify_rows) was bound by shared-memory bandwidth: every
// candidate re-read its 4d-byte row, 118 GB of shared-memory reads per round at configs[1].
//
// Precision ("3xTF32"): the tensor core reads an fp32 operand as TF32 (low 13 mantissa bits
// dropped), so with x = x_hi + x_lo, q = q_hi + q_lo (lo exact in fp32)
//     x.q ~= MMA(x, q) + MMA(x, q_lo) + MMA(x_lo, q)        (x_lo.q_lo, ~2^-22 |x||q|, dropped)
// with fp32 accumulation in TMEM: fp32-level dot products.  Candidate ordering can differ from
// a direct fp32 sum only at near-ties; the top-k distances returned to the caller are
// recomputed directly in fp32 (k_rerank_exact in query.cu).
//
// Kernel (persistent, one CTA per SM, 8 warps; tile t -> row tile t / nqt, query tile t % nqt,
// so the query tiles of one row tile run back to back and the row tile is read from HBM once):
//   warp 0     TMA producer: per tile the new-member words NB[a][4 rt .. 4 rt + 3] and their
//              round-buffer offsets BO (u32 boxes of 4 words x N queries); per k-block the X
//              rows [128 x 16 fp32] and the query tile (hi = fp32, lo) [N x 16 fp32], 64B-swizzled,
//              on separate barriers (converters start on the rows alone).
//   warp 1     TMEM allocation + single-thread MMA issue (M = 128, N, K = 8; 3 MMAs per k-step)
//              into a double-buffered accumulator.
//   warps 2-3  converters: x_lo = x - trunc_tf32(x) into a twin stage (same swizzled offsets).
//   warps 4-7  epilogue: tcgen05.ld of 16 query columns at a time for the warp's 32 rows; lane
//              i tests bit i of the query's new-member word, writes (row id, d2) at
//              BO + popc(word below lane i).
#include <cstdlib>

#include "index.cuh"
#include "tc_util.cuh"

namespace detlsh {
namespace {
using namespace tc;

constexpr int VT_M = 128;
constexpr int VT_KB = 16;                    // fp32 per k-block (64 B rows, 64-byte swizzle)
constexpr int VT_THREADS = 384;              // 12 warps: producer, MMA, 2 converters, 8 epilogue
constexpr int VT_XSTAGE = VT_M * VT_KB * 4;   // 8 KB

struct VtcShape {
    int64_t n;        // rows of X
    int ld, nkb;      // row stride (floats), k-blocks of 32
    int na;           // active queries of this round
    int N;            // queries per tile (multiple of 16, <= 256)
    int nqt;          // query tiles
    int64_t ntiles;   // row tiles x query tiles
    int stages;
    uint32_t tmem_cols;
    int dbg;          // experiments only (DETLSH_VTC_DEBUG): 1 = no epilogue body, 2 = no MMAs
};

__global__ void __launch_bounds__(VT_THREADS, 1)
    k_verify_tc(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmQ,
                const __grid_constant__ CUtensorMap tmQlo, const __grid_constant__ CUtensorMap tmNB,
                const __grid_constant__ CUtensorMap tmBO, VtcShape sh, const float* __restrict__ xn,
                const float* __restrict__ qn, uint32_t* __restrict__ cand, float* __restrict__ d2) {
    pdl_wait();
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte aligned, by pointer arithmetic on the shared array (keeps the shared address
    // space: LDS/STS instead of generic LD/ST)
    unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int S = sh.stages, N = sh.N;
    const size_t qbytes = (size_t)N * VT_KB * 4;
    const size_t stage_bytes = 2 * (size_t)VT_XSTAGE + 2 * qbytes;
    // stage s: [X 8 KB][X_lo 8 KB][Q N*64 B][Q_lo N*64 B]; then 2 mask buffers [NB N*16][BO N*16]
    unsigned char* sStage = base;
    uint32_t* sMask = reinterpret_cast<uint32_t*>(base + (size_t)S * stage_bytes);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sMask + 2 * 2 * 4 * N);
    uint64_t* full = bars;               // [S] X rows landed -> converters
    uint64_t* conv = bars + S;           // [S] converters -> MMA
    uint64_t* empty = bars + 2 * S;      // [S] MMA commit -> producer
    uint64_t* fullq = bars + 3 * S;      // [S] query tile landed -> MMA
    uint64_t* tfull = bars + 4 * S;      // [2] MMA commit -> epilogue
    uint64_t* tempty = bars + 4 * S + 2; // [2] epilogue -> MMA
    uint64_t* mfull = bars + 4 * S + 4;  // [2] masks loaded
    uint64_t* mempty = bars + 4 * S + 6; // [2] epilogue done with masks
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4 * S + 8);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto sX = [&](int s) { return sStage + (size_t)s * stage_bytes; };
    auto sXl = [&](int s) { return sStage + (size_t)s * stage_bytes + VT_XSTAGE; };
    auto sQ = [&](int s) { return sStage + (size_t)s * stage_bytes + 2 * VT_XSTAGE; };
    auto sQl = [&](int s) { return sStage + (size_t)s * stage_bytes + 2 * VT_XSTAGE + qbytes; };

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&conv[s], 64);
            mbar_init(&empty[s], 1);
            mbar_init(&fullq[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 256);
            mbar_init(&mfull[b], 1);
            mbar_init(&mempty[b], 256);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
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
            int s = 0, mb = 0;
            uint32_t ph = 0, mph = 0;
            const uint32_t txq = (uint32_t)(2 * qbytes);
            for (int64_t tile = blockIdx.x; tile < sh.ntiles; tile += gridDim.x) {
                const int64_t rt = tile / sh.nqt;
                const int qt = (int)(tile - rt * sh.nqt);
                mbar_wait(&mempty[mb], mph ^ 1);
                mbar_expect_tx(&mfull[mb], (uint32_t)(2 * 16 * N));
                uint32_t* m = sMask + (size_t)mb * 8 * N;
                tma_load_2d(m, &tmNB, &mfull[mb], (int)(rt * 4), qt * N);
                tma_load_2d(m + 4 * N, &tmBO, &mfull[mb], (int)(rt * 4), qt * N);
                if (++mb == 2) { mb = 0; mph ^= 1; }
                for (int kb = 0; kb < sh.nkb; ++kb) {
                    mbar_wait(&empty[s], ph ^ 1);
                    mbar_expect_tx(&full[s], (uint32_t)VT_XSTAGE);
                    // k-blocks start at a tile-dependent rotation: the SMs sharing a query tile
                    // then read different parts of it (no L2 hot spot on one k-block)
                    const int kr = (int)((kb + tile) % sh.nkb);
                    tma_load_2d(sX(s), &tmX, &full[s], kr * VT_KB, (int)(rt * VT_M));
                    mbar_expect_tx(&fullq[s], txq);
                    tma_load_2d(sQ(s), &tmQ, &fullq[s], kr * VT_KB, qt * N);
                    tma_load_2d(sQl(s), &tmQlo, &fullq[s], kr * VT_KB, qt * N);
                    if (++s == S) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
                                   ((uint32_t)(VT_M >> 4) << 24);
            int s = 0, buf = 0;
            uint32_t ph = 0, tph = 0;
            for (int64_t tile = blockIdx.x; tile < sh.ntiles; tile += gridDim.x) {
                mbar_wait(&tempty[buf], tph ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + (uint32_t)(buf * N);
                for (int kb = 0; kb < sh.nkb; ++kb) {
                    mbar_wait(&fullq[s], ph);
                    mbar_wait(&conv[s], ph);
                    tc_fence_after();
                    const uint32_t ax = smem_u32(sX(s)), al = smem_u32(sXl(s));
                    const uint32_t bq = smem_u32(sQ(s)), bl = smem_u32(sQl(s));
#pragma unroll
                    if (!(sh.dbg & 2))
                    for (int k = 0; k < VT_KB / 8; ++k) {      // K = 8 tf32 = 32 bytes per MMA
                        const uint64_t dq = desc_sw64(bq + k * 32);
                        const uint64_t dx = desc_sw64(ax + k * 32);
                        mma_tf32(d_tmem, dx, dq, idesc, (kb | k) ? 1u : 0u);       // x_hi q_hi
                        mma_tf32(d_tmem, dx, desc_sw64(bl + k * 32), idesc, 1u);    // x_hi q_lo
                        mma_tf32(d_tmem, desc_sw64(al + k * 32), dq, idesc, 1u);    // x_lo q_hi
                    }
                    mma_commit(&empty[s]);
                    if (++s == S) { s = 0; ph ^= 1; }
                }
                mma_commit(&tfull[buf]);
                if (++buf == 2) { buf = 0; tph ^= 1; }
            }
        }
    } else if (warp < 4) {
        const int t = threadIdx.x - 64;
        int s = 0;
        uint32_t ph = 0;
        for (int64_t tile = blockIdx.x; tile < sh.ntiles; tile += gridDim.x) {
            for (int kb = 0; kb < sh.nkb; ++kb) {
                mbar_wait(&full[s], ph);
                const float4* src = reinterpret_cast<const float4*>(sX(s));
                float4* dst = reinterpret_cast<float4*>(sXl(s));
#pragma unroll
                for (int i = t; i < VT_XSTAGE / 16; i += 64) {
                    const float4 x = src[i];
                    float4 lo;
                    lo.x = x.x - __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
                    lo.y = x.y - __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
                    lo.z = x.z - __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
                    lo.w = x.w - __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
                    dst[i] = lo;
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive(&conv[s]);
                if (++s == S) { s = 0; ph ^= 1; }
            }
        }
    } else {
        // warps 4-11: TMEM lane quarter ew = warp % 4 (rows [32 ew, 32 ew + 32) of the tile);
        // the two warps of a quarter take alternate 16-column chunks
        const int ew = warp & 3, eh = (warp - 4) >> 2;
        const uint32_t below = (1u << lane) - 1u;
        float* s_qn = reinterpret_cast<float*>(tmem_slot + 4) + (warp - 4) * 256;   // per warp: ||q||^2 of the tile
        int buf = 0, mb = 0;
        uint32_t tph = 0, mph = 0;
        int last_qt = -1;
        for (int64_t tile = blockIdx.x; tile < sh.ntiles; tile += gridDim.x) {
            const int64_t rt = tile / sh.nqt;
            const int qt = (int)(tile - rt * sh.nqt);
            const int64_t row = rt * VT_M + ew * 32 + lane;
            const float xr = row < sh.n ? __ldg(xn + row) : 0.f;
            const int a0 = qt * N;
            const int ncols = min(N, sh.na - a0);
            if (qt != last_qt) {
                for (int c = lane; c < ncols; c += 32) s_qn[c] = __ldg(qn + a0 + c);
                __syncwarp();
                last_qt = qt;
            }
            mbar_wait(&mfull[mb], mph);
            mbar_wait(&tfull[buf], tph);
            tc_fence_after();
            const uint32_t* NB = sMask + (size_t)mb * 8 * N;
            const uint32_t* BO = NB + 4 * N;
            const uint32_t taddr = tmem_base + (uint32_t)(buf * N) + ((uint32_t)(ew * 32) << 16);
            for (int c0 = 16 * eh; c0 < ((sh.dbg & 1) ? 0 : ncols); c0 += 32) {
                uint32_t w[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) w[i] = (c0 + i < ncols) ? NB[(c0 + i) * 4 + ew] : 0u;
                uint32_t any = 0;
#pragma unroll
                for (int i = 0; i < 16; ++i) any |= w[i];
                if (!any) continue;   // none of these 16 queries has a new member in the warp's rows
                float v[16];
                tmem_ld16(taddr + c0, v);
                // branch-free: every lane computes all 16 (slot, d2) pairs from broadcast shared
                // loads, then stores predicated on its bit (no divergent per-column branches)
                uint32_t bo[16];
                float qv[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    bo[i] = BO[(c0 + i) * 4 + ew];
                    qv[i] = s_qn[c0 + i];
                }
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const bool hit = (w[i] >> lane) & 1u;
                    const uint32_t slot = bo[i] + __popc(w[i] & below);
                    const float dd = fmaxf(0.f, fmaf(-2.f, v[i], xr + qv[i]));
                    if (hit) {
                        cand[slot] = (uint32_t)row;
                        d2[slot] = dd;
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty[buf]);
            mbar_arrive(&mempty[mb]);
            if (++buf == 2) { buf = 0; tph ^= 1; }
            if (++mb == 2) { mb = 0; mph ^= 1; }
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(sh.tmem_cols));
    }
}

}  // namespace

// d_Qa/d_Qalo: the round's active queries [na][ld] (fp32 and its TF32 residual), d_qn [na]
// their squared norms; d_NB/d_BO [na][nw4] new-member words and their round-buffer offsets;
// d_xn [n] squared row norms of X.  Returns false if the shape does not fit.
bool verify_tc(const float* d_X, int64_t n, int ld, const float* d_Qa, const float* d_Qalo, const float* d_qn, int na,
               const uint32_t* d_NB, const uint32_t* d_BO, int64_t nw4, const float* d_xn, uint32_t* d_cand,
               float* d_d2, cudaStream_t st) {
    if (na <= 0 || n <= 0) return true;
    VtcShape sh;
    sh.n = n;
    sh.ld = ld;
    sh.nkb = (int)ceil_div(ld, VT_KB);
    sh.na = na;
    sh.N = (int)std::min<int64_t>(256, round_up(na, 16));
    sh.nqt = (int)ceil_div(na, sh.N);
    const int64_t nrt = ceil_div(n, VT_M);
    sh.ntiles = nrt * sh.nqt;
    const size_t stage_bytes = 2 * (size_t)VT_XSTAGE + 2 * (size_t)sh.N * VT_KB * 4;
    const size_t fixed = 1024 + 2 * 2 * 16 * (size_t)sh.N + 512 + 8 * 256 * 4;
    const size_t budget = 227 * 1024;
    if (fixed + 2 * stage_bytes > budget) return false;
    sh.stages = (int)std::min<size_t>(8, (budget - fixed) / stage_bytes);
    uint32_t cols = 32;
    while (cols < (uint32_t)(2 * sh.N)) cols <<= 1;
    sh.tmem_cols = cols;
    static const int dbg = std::getenv("DETLSH_VTC_DEBUG") ? std::atoi(std::getenv("DETLSH_VTC_DEBUG")) : 0;
    sh.dbg = dbg;
    const size_t smem = fixed + (size_t)sh.stages * stage_bytes;
    CUtensorMap mx, mq, mql, mnb, mbo;
    make_map_sw64(&mx, d_X, n, ld, VT_M);
    make_map_sw64(&mq, d_Qa, na, ld, sh.N);
    make_map_sw64(&mql, d_Qalo, na, ld, sh.N);
    make_map_u32(&mnb, d_NB, na, nw4, 4, sh.N);
    make_map_u32(&mbo, d_BO, na, nw4, 4, sh.N);
    ensure_dyn_smem_fn(k_verify_tc, smem);
    int dev = 0, nsm = 148;
    DL_CUDA(cudaGetDevice(&dev));
    DL_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const int grid = (int)std::min<int64_t>(sh.ntiles, nsm);
    DL_LAUNCH(k_verify_tc, grid, VT_THREADS, smem, st, mx, mq, mql, mnb, mbo, sh, d_xn, d_qn, d_cand, d_d2);
    return true;
}

}  // namespace detlsh
