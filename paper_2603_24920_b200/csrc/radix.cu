// radix.cu -- hand-written stable LSD radix sort (batched segments) and exclusive scan.
//
// Used by the build for (a) sorting the breakpoint sample per projected coordinate
// and (b) the per-tree first-layer sort of (key, id) pairs (Alg. 2 line 2,
// P:312; B5), and by the leaf finaliser.  No library sort is dispatched.
//
// One pass (8-bit digit): hist (per tile digit counts) -> scan (digit-major, per segment)
// -> scatter (stable rank inside a tile via warp match + per-warp digit counts).
#include "common.cuh"

namespace detlsh {

namespace {

constexpr int RS_THREADS = 256;
constexpr int RS_IPT = 8;                           // items per thread (16: 104 registers, 2 blocks per SM)
constexpr int RS_TILE = RS_THREADS * RS_IPT;        // 2048 keys per tile
constexpr int RS_WARPS = RS_THREADS / 32;

__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const uint32_t* __restrict__ keys, int64_t m,
                                                        int shift, int tiles, uint32_t* __restrict__ hist) {
    pdl_wait();
    __shared__ uint32_t h[256];
    const int seg = blockIdx.y, tile = blockIdx.x;
    h[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t* k = keys + (int64_t)seg * m;
    int64_t base = (int64_t)tile * RS_TILE;
#pragma unroll 4
    for (int j = 0; j < RS_IPT; ++j) {
        int64_t e = base + (int64_t)j * RS_THREADS + threadIdx.x;
        if (e < m) atomicAdd(&h[(k[e] >> shift) & 255u], 1u);
    }
    __syncthreads();
    hist[((int64_t)seg * 256 + threadIdx.x) * tiles + tile] = h[threadIdx.x];
}

// Block-wide exclusive scan of one value per thread (1024 threads max); returns the block total.
template <int NT>
__device__ inline uint32_t block_exclusive_scan(uint32_t v, uint32_t* s_warp, uint32_t& excl) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t t = lane < NT / 32 ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        if (lane < NT / 32) s_warp[lane] = t;  // inclusive warp totals
    }
    __syncthreads();
    uint32_t total = s_warp[NT / 32 - 1];
    excl = x - v + (w ? s_warp[w - 1] : 0);
    __syncthreads();
    return total;
}

// Exclusive scan, in place, of one digit's per-tile counts (warp per (digit, segment); 8 digits
// per block); the digit's total goes to dtot[seg][digit] (the scatter turns those into digit bases).
__global__ void __launch_bounds__(256) k_rs_scan(uint32_t* __restrict__ hist, int tiles, uint32_t* __restrict__ dtot) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int dig = blockIdx.x * 8 + (threadIdx.x >> 5), seg = blockIdx.y;
    uint32_t* h = hist + ((int64_t)seg * 256 + dig) * tiles;
    uint32_t carry = 0;
    for (int base = 0; base < tiles; base += 32) {
        const int e = base + lane;
        const uint32_t v = e < tiles ? h[e] : 0;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (e < tiles) h[e] = carry + x - v;
        carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) dtot[seg * 256 + dig] = carry;
}

// Scatter of one 8-bit digit pass, stable.  Warp w of the block ranks the tile's keys
// [256 w, 256 w + 256) on its own (all its loads issued first): 8 rounds of 32 consecutive keys, warp.match_any groups a
// round's equal digits, the group's lowest lane reads and bumps the warp's private digit counter
// (no block barrier per round).  One block barrier later every key knows its place in the tile
// sorted by (digit, original position); the tile is staged in shared memory in that order and
// written out so that runs of equal digits land on consecutive addresses (coalesced), at the
// digit's global base (this tile's per-digit offset from k_rs_scan + the digits below).
// IOTA: the values are the keys' positions in their segment (not read; the first pass of a sort
// whose values start as 0..m-1 per segment).
template <bool HAS_VALS, bool IOTA = false>
__global__ void __launch_bounds__(RS_THREADS) k_rs_scatter(const uint32_t* __restrict__ kin,
                                                           const uint32_t* __restrict__ vin,
                                                           uint32_t* __restrict__ kout,
                                                           uint32_t* __restrict__ vout, int64_t m,
                                                           int shift, int tiles,
                                                           const uint32_t* __restrict__ offs,
                                                           const uint32_t* __restrict__ dtot) {
    pdl_wait();
    __shared__ uint32_t s_base[256];                 // global position of the tile's first key of digit d
    __shared__ uint32_t s_tds[256];                  // first staged slot of digit d in the sorted tile
    __shared__ uint32_t s_wh[RS_WARPS][256];         // per-warp digit counts -> per-warp digit offsets
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_k[RS_TILE];
    __shared__ uint32_t s_v[HAS_VALS ? RS_TILE : 1];
    const int seg = blockIdx.y, tile = blockIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t* k = kin + (int64_t)seg * m;
    const uint32_t* v = HAS_VALS ? vin + (int64_t)seg * m : nullptr;
    uint32_t* ko = kout + (int64_t)seg * m;
    uint32_t* vo = HAS_VALS ? vout + (int64_t)seg * m : nullptr;
    const int64_t base = (int64_t)tile * RS_TILE;
    for (int i = lane; i < 256; i += 32) s_wh[w][i] = 0;
    __syncwarp();
    constexpr int R = RS_TILE / RS_THREADS;          // rounds of 32 keys per warp
    uint32_t key[R], val[R], loc[R];
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int64_t e = base + (int64_t)w * (32 * R) + 32 * j + lane;
        const bool ok = e < m;
        key[j] = ok ? __ldg(k + e) : 0u;
        val[j] = !HAS_VALS ? 0u : IOTA ? (uint32_t)e : ok ? __ldg(v + e) : 0u;
    }
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int64_t e = base + (int64_t)w * (32 * R) + 32 * j + lane;
        const bool ok = e < m;
        const uint32_t dig = ok ? ((key[j] >> shift) & 255u) : 256u;
        const uint32_t peers = __match_any_sync(0xffffffffu, dig);
        const int leader = __ffs(peers) - 1;
        uint32_t old = 0;
        if (ok && lane == leader) {
            old = s_wh[w][dig];
            s_wh[w][dig] = old + __popc(peers);
        }
        old = __shfl_sync(0xffffffffu, old, leader);
        loc[j] = ok ? old + __popc(peers & lt) : 0xFFFFFFFFu;   // rank among the warp's keys of this digit
        __syncwarp();
    }
    __syncthreads();
    // per digit (thread = digit): warps' exclusive offsets, the tile's count, global base
    {
        const int d = threadIdx.x;
        uint32_t run = 0;
#pragma unroll
        for (int ww = 0; ww < RS_WARPS; ++ww) {
            const uint32_t c = s_wh[ww][d];
            s_wh[ww][d] = run;
            run += c;
        }
        uint32_t tds;
        block_exclusive_scan<RS_THREADS>(run, s_warp, tds);          // slots of the digits below d
        s_tds[d] = tds;
        uint32_t dbase;                                               // this segment's keys of lower digits
        block_exclusive_scan<RS_THREADS>(dtot[seg * 256 + d], s_warp, dbase);
        s_base[d] = dbase + offs[((int64_t)seg * 256 + d) * tiles + tile];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < R; ++j) {
        if (loc[j] != 0xFFFFFFFFu) {
            const uint32_t d = (key[j] >> shift) & 255u;
            const uint32_t slot = s_tds[d] + s_wh[w][d] + loc[j];
            s_k[slot] = key[j];
            if (HAS_VALS) s_v[slot] = val[j];
        }
    }
    __syncthreads();
    const int cnt = (int)(m - base < RS_TILE ? m - base : (int64_t)RS_TILE);
    for (int i = threadIdx.x; i < cnt; i += RS_THREADS) {
        const uint32_t kk = s_k[i];
        const uint32_t d = (kk >> shift) & 255u;
        const uint32_t pos = s_base[d] + (uint32_t)i - s_tds[d];
        ko[pos] = kk;
        if (HAS_VALS) vo[pos] = s_v[i];
    }
}

constexpr int SC_THREADS = 1024;
constexpr int SC_IPT = 8;
constexpr int SC_TILE = SC_THREADS * SC_IPT;

__global__ void __launch_bounds__(SC_THREADS) k_scan_tiles(const uint32_t* __restrict__ in, int64_t n,
                                                           uint32_t* __restrict__ tile_sums) {
    pdl_wait();
    __shared__ uint32_t s_warp[32];
    int64_t base = (int64_t)blockIdx.x * SC_TILE;
    uint32_t s = 0;
#pragma unroll
    for (int j = 0; j < SC_IPT; ++j) {
        int64_t e = base + (int64_t)threadIdx.x * SC_IPT + j;
        if (e < n) s += in[e];
    }
    uint32_t excl;
    uint32_t tot = block_exclusive_scan<SC_THREADS>(s, s_warp, excl);
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(SC_THREADS) k_scan_sums(uint32_t* __restrict__ sums, int64_t nt,
                                                          uint32_t* __restrict__ d_total) {
    pdl_wait();
    __shared__ uint32_t s_warp[32];
    uint32_t carry = 0;
    for (int64_t base = 0; base < nt; base += SC_THREADS) {
        int64_t e = base + threadIdx.x;
        uint32_t v = e < nt ? sums[e] : 0;
        uint32_t excl;
        uint32_t tot = block_exclusive_scan<SC_THREADS>(v, s_warp, excl);
        if (e < nt) sums[e] = carry + excl;
        carry += tot;
    }
    if (threadIdx.x == 0 && d_total) *d_total = carry;
}

__global__ void __launch_bounds__(SC_THREADS) k_scan_apply(const uint32_t* __restrict__ in, int64_t n,
                                                           const uint32_t* __restrict__ tile_offs,
                                                           uint32_t* __restrict__ out) {
    pdl_wait();
    __shared__ uint32_t s_warp[32];
    int64_t base = (int64_t)blockIdx.x * SC_TILE;
    uint32_t v[SC_IPT], s = 0;
#pragma unroll
    for (int j = 0; j < SC_IPT; ++j) {
        int64_t e = base + (int64_t)threadIdx.x * SC_IPT + j;
        v[j] = e < n ? in[e] : 0;
        s += v[j];
    }
    uint32_t excl;
    block_exclusive_scan<SC_THREADS>(s, s_warp, excl);
    uint32_t run = tile_offs[blockIdx.x] + excl;
#pragma unroll
    for (int j = 0; j < SC_IPT; ++j) {
        int64_t e = base + (int64_t)threadIdx.x * SC_IPT + j;
        if (e < n) out[e] = run;
        run += v[j];
    }
}

}  // namespace

bool radix_sort_batched(uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1, int64_t m,
                        int64_t nseg, int bits, cudaStream_t st, bool vals_iota) {
    if (m <= 0 || nseg <= 0 || bits <= 0) return false;
    const int tiles = (int)ceil_div(m, RS_TILE);
    const int64_t len = (int64_t)256 * tiles;
    Scratch hist(st, sizeof(uint32_t) * (size_t)(len * nseg + 256 * nseg));
    uint32_t* dtot = hist.as<uint32_t>() + len * nseg;
    bool flip = false;
    for (int shift = 0; shift < bits; shift += 8) {
        uint32_t* ki = flip ? k1 : k0;
        uint32_t* vi = flip ? v1 : v0;
        uint32_t* ko = flip ? k0 : k1;
        uint32_t* vo = flip ? v0 : v1;
        dim3 grid(tiles, (unsigned)nseg);
        DL_LAUNCH(k_rs_hist, grid, RS_THREADS, 0, st, ki, m, shift, tiles, hist.as<uint32_t>());
        DL_LAUNCH(k_rs_scan, dim3(32, (unsigned)nseg), 256, 0, st, hist.as<uint32_t>(), tiles, dtot);
        if (v0 && vals_iota && shift == 0) {
            DL_LAUNCH(k_rs_scatter<true COMMA true>, grid, RS_THREADS, 0, st, ki, (const uint32_t*)nullptr, ko, vo, m,
                      shift, tiles, hist.as<uint32_t>(), dtot);
        } else if (v0) {
            DL_LAUNCH(k_rs_scatter<true>, grid, RS_THREADS, 0, st, ki, vi, ko, vo, m, shift, tiles,
                      hist.as<uint32_t>(), dtot);
        } else {
            DL_LAUNCH(k_rs_scatter<false>, grid, RS_THREADS, 0, st, ki, (const uint32_t*)nullptr, ko,
                      (uint32_t*)nullptr, m, shift, tiles, hist.as<uint32_t>(), dtot);
        }
        flip = !flip;
    }
    return flip;
}

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* d_total, cudaStream_t st) {
    if (n <= 0) {
        if (d_total) DL_CUDA(cudaMemsetAsync(d_total, 0, sizeof(uint32_t), st));
        return;
    }
    const int64_t nt = ceil_div(n, SC_TILE);
    Scratch sums(st, sizeof(uint32_t) * (size_t)nt);
    DL_LAUNCH(k_scan_tiles, (unsigned)nt, SC_THREADS, 0, st, in, n, sums.as<uint32_t>());
    DL_LAUNCH(k_scan_sums, 1, SC_THREADS, 0, st, sums.as<uint32_t>(), nt, d_total);
    DL_LAUNCH(k_scan_apply, (unsigned)nt, SC_THREADS, 0, st, in, n, sums.as<uint32_t>(), out);
}

}  // namespace detlsh
