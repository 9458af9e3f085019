// build.cu -- index construction on sm_100a.
//
//  B0 hash family A (Eq. 1; AMB-1)      k_hash_family
//  B1 sample: n_s smallest keyed hashes (AMB-3/4)  k_sel_hist / k_sel_pick / k_sel_collect
//  B2 projection P = X A^T                  project_rows (tcgen05 or SIMT, project*.cu)
//  B3 breakpoints from the sorted sample (AMB-5)  radix sort + k_bp_gather
//  B4 encode, Alg. 1 lines 3-8 (AMB-6/7) k_encode
//  B5 first layer, Alg. 2 line 2    k_first_key + batched radix sort
//  B6 splits, Alg. 2 lines 7-10 + SplitNode, bulk rule:
//     a node with more than max_size points splits on the dimension whose next bit most
//     evenly divides its first max_size points (ascending id); children are the stable
//     partition.  Level-synchronous over all L trees at once.
#include <cstring>
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "index.cuh"

namespace detlsh {

namespace {

// ------------------------------------------------------------------ B0
__global__ void k_hash_family(uint64_t seed, int LK, int d, int ld, float* __restrict__ A) {
    pdl_wait();
    const int64_t total = (int64_t)LK * ld;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / ld), t = (int)(i % ld);
        float out = 0.f;
        if (t < d) {
            const uint64_t e = (uint64_t)r * d + t;             // entry index of A[r][t]
            double u1 = (double)(keyed(seed, 2 * e) >> 11) * (1.0 / 9007199254740992.0);
            double u2 = (double)(keyed(seed, 2 * e + 1) >> 11) * (1.0 / 9007199254740992.0);
            double g = sqrt(-2.0 * log(1.0 - u1)) * cos(6.283185307179586476925286766559 * u2);
            uint32_t u = __float_as_uint(__double2float_rn(g));
            u += 0xFFFu + ((u >> 13) & 1u);                     // round to TF32 (nearest even)
            u &= ~0x1FFFu;
            out = __uint_as_float(u);
        }
        A[i] = out;                                             // padded row stride ld, zeros beyond d
    }
}

// ------------------------------------------------------------------ B1 radix select over keyed hashes
struct SelState {
    unsigned long long prefix, mask, remaining, eq_count;
};

__global__ void k_sel_init(SelState* s, int64_t n_s) {
    pdl_wait();
    s->prefix = 0; s->mask = 0; s->remaining = (unsigned long long)n_s; s->eq_count = 0;
}

__global__ void __launch_bounds__(256) k_sel_hist(uint64_t salt, int64_t n_global, int shift,
                                                  const SelState* __restrict__ st,
                                                  uint32_t* __restrict__ hist) {
    pdl_wait();
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t prefix = st->prefix, mask = st->mask;
    for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < n_global;
         id += (int64_t)gridDim.x * blockDim.x) {
        uint64_t key = keyed(salt, (uint64_t)id);
        if ((key & mask) == prefix) atomicAdd(&h[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], h[threadIdx.x]);
}

__global__ void __launch_bounds__(256) k_sel_pick(int shift, SelState* st, uint32_t* hist) {
    pdl_wait();
    __shared__ unsigned long long s_incl[256];
    const unsigned long long v = hist[threadIdx.x];
    s_incl[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 256; o <<= 1) {
        unsigned long long add = threadIdx.x >= o ? s_incl[threadIdx.x - o] : 0ull;
        __syncthreads();
        s_incl[threadIdx.x] += add;
        __syncthreads();
    }
    const unsigned long long incl = s_incl[threadIdx.x], excl = incl - v;
    const unsigned long long rem = st->remaining;
    __syncthreads();
    if (v > 0 && excl < rem && rem <= incl) {
        st->prefix |= (unsigned long long)threadIdx.x << shift;
        st->mask |= 0xFFull << shift;
        st->remaining = rem - excl;
        st->eq_count = v;
    }
    hist[threadIdx.x] = 0;
}

__global__ void __launch_bounds__(256) k_sel_collect(uint64_t salt, int64_t id_lo, int64_t n_range,
                                                     const SelState* __restrict__ st,
                                                     uint32_t* __restrict__ out,
                                                     unsigned long long* __restrict__ counter) {
    pdl_wait();
    const uint64_t T = st->prefix;
    const bool take_eq = st->eq_count == st->remaining;         // all ties needed (the usual case)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_range;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t key = keyed(salt, (uint64_t)(id_lo + i));
        if (key < T || (take_eq && key == T)) out[atomicAdd(counter, 1ull)] = (uint32_t)i;
    }
}

// Ties at the threshold beyond what is needed: take the lowest ids (AMB-4), serially.
// Only reachable when two 64-bit keys collide exactly at the n_s-th position.
__global__ void k_sel_ties(uint64_t salt, int64_t id_lo, int64_t n_range, int64_t n_global,
                           const SelState* __restrict__ st, uint32_t* __restrict__ out,
                           unsigned long long* __restrict__ counter) {
    pdl_wait();
    if (st->eq_count == st->remaining) return;
    const uint64_t T = st->prefix;
    unsigned long long need = st->remaining;
    for (int64_t id = 0; id < n_global && need; ++id) {
        if (keyed(salt, (uint64_t)id) == T) {
            --need;
            if (id >= id_lo && id < id_lo + n_range) out[atomicAdd(counter, 1ull)] = (uint32_t)(id - id_lo);
        }
    }
}

// Fast path of the same selection: one 16-bit histogram of the keys' top bits finds the bin b
// holding the n_s-th smallest key; keys in lower bins are all taken, and the few keys in bin b
// (~n/65536) are ranked exactly by (key, id) -- ties to the lowest id (AMB-4).  Identical set
// to the 8-pass radix select above, which remains the fallback if bin b overflows its buffer.
struct Sel16 {
    uint32_t bin, need, ncand, overflow;
};

__global__ void __launch_bounds__(256) k_sel16_hist(uint64_t salt, int64_t n_global, uint32_t* __restrict__ hist) {
    pdl_wait();
    for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < n_global;
         id += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&hist[keyed(salt, (uint64_t)id) >> 48], 1u);
}

// one CTA of 1024 threads, 64 bins each
__global__ void __launch_bounds__(1024) k_sel16_pick(const uint32_t* __restrict__ hist, int64_t n_s, Sel16* __restrict__ st) {
    pdl_wait();
    __shared__ uint32_t s_warp[32];
    __shared__ unsigned long long s_tot[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t* h = hist + threadIdx.x * 64;
    unsigned long long sum = 0;
    {
        const uint4* h4 = reinterpret_cast<const uint4*>(h);   // 16 loads of 16 B, all in flight
        uint4 v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = h4[j];
#pragma unroll
        for (int j = 0; j < 16; ++j) sum += (unsigned long long)v[j].x + v[j].y + v[j].z + v[j].w;
    }
    unsigned long long x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_tot[w] = x;
    __syncthreads();
    unsigned long long before = x - sum;
    for (int ww = 0; ww < w; ++ww) before += s_tot[ww];
    (void)s_warp;
    const unsigned long long want = (unsigned long long)n_s;
    if (before < want && want <= before + sum) {      // exactly one thread
        unsigned long long run = before;
        for (int j = 0; j < 64; ++j) {
            if (run + h[j] >= want) {
                st->bin = (uint32_t)(threadIdx.x * 64 + j);
                st->need = (uint32_t)(want - run);
                st->ncand = 0;
                st->overflow = 0;
                break;
            }
            run += h[j];
        }
    }
}

__global__ void __launch_bounds__(256) k_sel16_collect(uint64_t salt, int64_t id_lo, int64_t n_range, int64_t n_global,
                                                       Sel16* __restrict__ st, uint32_t* __restrict__ out,
                                                       unsigned long long* __restrict__ counter,
                                                       unsigned long long* __restrict__ ckey, uint32_t* __restrict__ cid,
                                                       uint32_t ccap) {
    pdl_wait();
    const uint32_t b = st->bin;
    for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < n_global;
         id += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t key = keyed(salt, (uint64_t)id);
        const uint32_t top = (uint32_t)(key >> 48);
        if (top < b) {
            if (id >= id_lo && id < id_lo + n_range) out[atomicAdd(counter, 1ull)] = (uint32_t)(id - id_lo);
        } else if (top == b) {
            const uint32_t i = atomicAdd(&st->ncand, 1u);
            if (i < ccap) { ckey[i] = key; cid[i] = (uint32_t)id; }
        }
    }
}

// one CTA: rank every candidate of bin b by (key, id); the `need` smallest are taken
__global__ void __launch_bounds__(1024) k_sel16_finish(int64_t id_lo, int64_t n_range, Sel16* __restrict__ st,
                                                       const unsigned long long* __restrict__ ckey,
                                                       const uint32_t* __restrict__ cid, uint32_t ccap,
                                                       uint32_t* __restrict__ out, unsigned long long* __restrict__ counter) {
    pdl_wait();
    extern __shared__ unsigned long long s_key[];
    uint32_t* s_id = reinterpret_cast<uint32_t*>(s_key + ccap);
    const uint32_t nc = st->ncand;
    if (nc > ccap) {
        if (threadIdx.x == 0) st->overflow = 1;
        return;
    }
    for (uint32_t i = threadIdx.x; i < nc; i += blockDim.x) { s_key[i] = ckey[i]; s_id[i] = cid[i]; }
    __syncthreads();
    const uint32_t need = st->need;
    for (uint32_t i = threadIdx.x; i < nc; i += blockDim.x) {
        const unsigned long long k = s_key[i];
        const uint32_t id = s_id[i];
        uint32_t rank = 0;
        for (uint32_t j = 0; j < nc; ++j) rank += (s_key[j] < k || (s_key[j] == k && s_id[j] < id)) ? 1u : 0u;
        if (rank < need && (int64_t)id >= id_lo && (int64_t)id < id_lo + n_range)
            out[atomicAdd(counter, 1ull)] = (uint32_t)(id - id_lo);
    }
}

__global__ void k_gather_rows(const float* __restrict__ X, int64_t ld, const uint32_t* __restrict__ ids,
                              int64_t m, float* __restrict__ out) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < m; r += nwarps) {
        const float4* src = reinterpret_cast<const float4*>(X + (int64_t)ids[r] * ld);
        float4* dst = reinterpret_cast<float4*>(out + r * ld);
        for (int64_t f = lane; f < ld / 4; f += 32) dst[f] = src[f];
    }
}

// ------------------------------------------------------------------ B3
__global__ void k_transpose_keys(const float* __restrict__ Ps, int64_t m, int LK, uint32_t* __restrict__ keys) {
    pdl_wait();
    const int64_t total = m * LK;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = i / LK;
        const int r = (int)(i % LK);
        keys[(int64_t)r * m + s] = f2key(Ps[i]);
    }
}

// B(1) = C^(1), B(z) = C^(floor(m/N_r)(z-1)) (1-based, z=2..N_r), B(N_r+1) = C^(m)  (AMB-5)
__global__ void k_bp_gather(const uint32_t* __restrict__ sorted, int64_t m, int LK, int N_r, float* __restrict__ B) {
    pdl_wait();
    const int64_t total = (int64_t)LK * (N_r + 1);
    const int64_t stride = m / N_r > 0 ? m / N_r : 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / (N_r + 1)), t = (int)(i % (N_r + 1));
        int64_t pos;
        if (t == 0) pos = 0;
        else if (t == N_r) pos = m - 1;
        else pos = min((int64_t)t * stride, m) - 1;
        B[i] = key2f(sorted[(int64_t)r * m + pos]);
    }
}

// ------------------------------------------------------------------ B4 encode (Alg. 1)
// code = #{t in 1..N_r-1 : b_t < x}: branch-free lower_bound over the interior breakpoints
// with a +inf sentinel (AMB-6: ties go to the lower region; AMB-7: clamp to 0 / N_r-1).
__global__ void __launch_bounds__(256) k_encode(const float* __restrict__ P, int64_t m, int LK, int N_r,
                                                const float* __restrict__ B, uint8_t* __restrict__ EP) {
    pdl_wait();
    extern __shared__ float tab[];  // [LK][N_r]
    for (int i = threadIdx.x; i < LK * N_r; i += blockDim.x) {
        const int r = i / N_r, t = i % N_r;
        tab[i] = (t < N_r - 1) ? B[(int64_t)r * (N_r + 1) + t + 1] : __int_as_float(0x7f800000);
    }
    __syncthreads();
    if (LK & 3) {  // generic path
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m * LK;
             i += (int64_t)gridDim.x * blockDim.x) {
            const float* t = tab + (int)(i % LK) * N_r;
            const float x = P[i];
            int pos = 0;
            for (int s = N_r >> 1; s > 0; s >>= 1) pos += (t[pos + s - 1] < x) ? s : 0;
            EP[i] = (uint8_t)pos;
        }
        return;
    }
    const int64_t total4 = m * LK / 4;
    const float4* P4 = reinterpret_cast<const float4*>(P);
    uchar4* E4 = reinterpret_cast<uchar4*>(EP);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total4;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float4 v = P4[i];
        const int r0 = (int)((i * 4) % LK);
        const float xs[4] = {v.x, v.y, v.z, v.w};
        uint8_t c[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float* t = tab + (r0 + q) * N_r;
            int pos = 0;
            for (int s = N_r >> 1; s > 0; s >>= 1) pos += (t[pos + s - 1] < xs[q]) ? s : 0;
            c[q] = (uint8_t)pos;
        }
        E4[i] = make_uchar4(c[0], c[1], c[2], c[3]);
    }
}

// ------------------------------------------------------------------ B5/B6 trees
struct __align__(16) Node {
    uint4 bits;       // 4-bit symbol-prefix length per dimension (32 dims)
    uint32_t start;   // global position in the [L*n] perm array (tree = start / n)
    uint32_t len;
    uint32_t pad0, pad1;
};

__device__ inline int nib(const uint4& b, int j) {
    const uint32_t w = j < 8 ? b.x : j < 16 ? b.y : j < 24 ? b.z : b.w;
    return (int)((w >> ((j & 7) * 4)) & 15u);
}
__device__ inline void nib_inc(uint4& b, int j) {
    const uint32_t add = 1u << ((j & 7) * 4);
    if (j < 8) b.x += add; else if (j < 16) b.y += add; else if (j < 24) b.z += add; else b.w += add;
}
__device__ inline bool splittable(const uint4& b, int K, int nb) {
    for (int j = 0; j < K; ++j)
        if (nib(b, j) < nb) return true;
    return false;
}

// First-layer key of point id in tree t: MSB of each of the K symbols, dim 0 most significant (AMB-11).
__global__ void k_first_key(const uint8_t* __restrict__ EP, int64_t n, int L, int K, int nb,
                            uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    pdl_wait();
    const int LK = L * K;
    const int64_t total = n * L;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int t = (int)(g / n);
        const int64_t id = g - (int64_t)t * n;
        const uint8_t* c = EP + id * LK + t * K;
        uint32_t key = 0;
        if (K == 16 && (LK & 15) == 0) {          // one 16-byte load of the tree's codes
            const uint4 c4 = *reinterpret_cast<const uint4*>(c);
            const uint32_t w[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
            for (int j = 0; j < 16; ++j) key = (key << 1) | ((w[j >> 2] >> (8 * (j & 3) + nb - 1)) & 1u);
        } else {
            for (int j = 0; j < K; ++j) key = (key << 1) | ((c[j] >> (nb - 1)) & 1u);
        }
        keys[g] = key;
        vals[g] = (uint32_t)id;
    }
}


__global__ void k_seg_flags(const uint32_t* __restrict__ keys, int64_t n, int64_t total, uint32_t* __restrict__ flags) {
    pdl_wait();
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
         g += (int64_t)gridDim.x * blockDim.x)
        flags[g] = (g % n == 0 || keys[g] != keys[g - 1]) ? 1u : 0u;
}

__global__ void k_seg_write(const uint32_t* __restrict__ flags, const uint32_t* __restrict__ idx, int64_t total,
                            uint32_t* __restrict__ starts) {
    pdl_wait();
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
         g += (int64_t)gridDim.x * blockDim.x)
        if (flags[g]) starts[idx[g]] = (uint32_t)g;
}

// Append with a capacity guard: the count keeps growing past cap so the host can detect
// overflow and retry with more room.
__device__ inline void push_node(Node* arr, uint32_t* cnt, uint32_t cap, const Node& nd) {
    const uint32_t i = atomicAdd(cnt, 1u);
    if (i < cap) arr[i] = nd;
}

// Where a node goes: a leaf (<= max_size points or no bits left), the block-local list (small
// enough for k_local_finish to split it to the end in shared memory), or the next global level.
// Local nodes in two size tiers sharing one array: <= local_max1 points from the front,
// (local_max1, local_max] from the back (each tier's k_local_finish launch sizes its shared memory
// for its own largest node; both tiers' nodes are disjoint, > max_size points: <= cap_local in all).
struct Sinks {
    Node* active; uint32_t* n_active; uint32_t cap_active;
    Node* local; uint32_t* n_local; uint32_t cap_local; int local_max;
    Node* leaves; uint32_t* n_leaves; uint32_t cap_leaves;
    uint32_t* n_local2; int local_max1;
};
__device__ inline void route_node(const Sinks& k, const Node& nd, int K, int nb, int max_size) {
    if ((int64_t)nd.len <= max_size || !splittable(nd.bits, K, nb)) {
        push_node(k.leaves, k.n_leaves, k.cap_leaves, nd);
    } else if ((int64_t)nd.len <= k.local_max1) {
        push_node(k.local, k.n_local, k.cap_local, nd);
    } else if ((int64_t)nd.len <= k.local_max) {
        const uint32_t i = atomicAdd(k.n_local2, 1u);
        if (i < k.cap_local) k.local[k.cap_local - 1 - i] = nd;
    } else {
        push_node(k.active, k.n_active, k.cap_active, nd);
    }
}

__global__ void k_init_nodes(const uint32_t* __restrict__ starts, const uint32_t* __restrict__ nseg_p,
                             int64_t total, int K, int nb, int max_size, Sinks sk) {
    pdl_wait();
    const uint32_t nseg = *nseg_p;
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nseg;
         s += (int64_t)gridDim.x * blockDim.x) {
        Node nd;
        uint32_t w[4];
        for (int q = 0; q < 4; ++q) {
            uint32_t x = 0;
            for (int e = 0; e < 8; ++e) x |= (uint32_t)((q * 8 + e) < K ? 1 : nb) << (4 * e);
            w[q] = x;
        }
        nd.bits = make_uint4(w[0], w[1], w[2], w[3]);
        nd.start = starts[s];
        nd.len = (uint32_t)((s + 1 < nseg ? (int64_t)starts[s + 1] : total) - nd.start);
        nd.pad0 = nd.pad1 = 0;
        route_node(sk, nd, K, nb, max_size);
    }
}

// SplitNode's dimension (AMB-9): over the node's first max_size points, the dim with bits
// left whose next bit minimises |n0 - n1|; ties to the lowest dim.  One warp per node.
__global__ void k_choose_split(const Node* __restrict__ nodes, const uint32_t* __restrict__ n_nodes_p,
                               const uint32_t* __restrict__ perm, const uint8_t* __restrict__ EP,
                               int64_t n, int LK, int K, int nb, int max_size, int chunk,
                               int* __restrict__ split, uint32_t* __restrict__ nch) {
    pdl_wait();
    const uint32_t n_nodes = *n_nodes_p;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t a = warp; a < n_nodes; a += nwarps) {
        const Node nd = nodes[a];
        const int t = (int)(nd.start / n);
        int ones[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) ones[j] = 0;
        for (int e = lane; e < max_size; e += 32) {
            const uint8_t* c = EP + (int64_t)perm[nd.start + e] * LK + t * K;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                if (j < K) {
                    const int b = nib(nd.bits, j);
                    if (b < nb) ones[j] += (c[j] >> (nb - 1 - b)) & 1;
                }
            }
        }
        int best = -1, best_imb = 0x7fffffff;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            int v = ones[j];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (j < K && nib(nd.bits, j) < nb) {
                int imb = abs(max_size - 2 * v);
                if (imb < best_imb) { best_imb = imb; best = j; }
            }
        }
        if (lane == 0) {
            split[a] = best;
            nch[a] = best >= 0 ? (uint32_t)ceil_div(nd.len, chunk) : 0u;
        }
    }
}

__device__ inline int64_t chunk_owner(const uint32_t* __restrict__ choff, int64_t n_nodes, uint32_t c) {
    int64_t lo = 0, hi = n_nodes - 1;   // last a with choff[a] <= c
    while (lo < hi) {
        int64_t mid = (lo + hi + 1) >> 1;
        if (choff[mid] <= c) lo = mid; else hi = mid - 1;
    }
    return lo;
}

constexpr int PART_THREADS = 256;
constexpr int PART_IPT = 8;
constexpr int PART_CHUNK = PART_THREADS * PART_IPT;

__device__ inline int next_bit_of(const uint8_t* __restrict__ EP, uint32_t id, int64_t LK, int off, int shift) {
    return (EP[(int64_t)id * LK + off] >> shift) & 1;
}

__global__ void __launch_bounds__(PART_THREADS) k_part_count(const Node* __restrict__ nodes, const int* __restrict__ split,
                                                             const uint32_t* __restrict__ choff, const uint32_t* __restrict__ n_nodes_p,
                                                             const uint32_t* __restrict__ total_ch_p,
                                                             const uint32_t* __restrict__ perm, const uint8_t* __restrict__ EP,
                                                             int64_t n, int LK, int K, int nb, uint32_t* __restrict__ zc) {
    pdl_wait();
    __shared__ uint32_t s_cnt;
    const uint32_t c = blockIdx.x;
    if (c >= *total_ch_p) return;
    const int64_t a = chunk_owner(choff, *n_nodes_p, c);
    const Node nd = nodes[a];
    const int j = split[a];
    const int t = (int)(nd.start / n);
    const int shift = nb - 1 - nib(nd.bits, j);
    const int64_t base = (int64_t)(c - choff[a]) * PART_CHUNK;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    uint32_t z = 0;
    for (int q = 0; q < PART_IPT; ++q) {
        const int64_t e = base + q * PART_THREADS + threadIdx.x;
        if (e < nd.len) z += 1 - next_bit_of(EP, perm[nd.start + e], LK, t * K + j, shift);
    }
    for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&s_cnt, z);
    __syncthreads();
    if (threadIdx.x == 0) zc[c] = s_cnt;
}

__global__ void k_part_offsets(const uint32_t* __restrict__ choff, const uint32_t* __restrict__ nch,
                               const uint32_t* __restrict__ n_nodes_p, uint32_t* __restrict__ zc,
                               uint32_t* __restrict__ zeros) {
    pdl_wait();
    const uint32_t n_nodes = *n_nodes_p;
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n_nodes;
         a += (int64_t)gridDim.x * blockDim.x) {
        uint32_t run = 0;
        for (uint32_t c = choff[a]; c < choff[a] + nch[a]; ++c) {
            uint32_t v = zc[c];
            zc[c] = run;
            run += v;
        }
        zeros[a] = run;
    }
}

__global__ void __launch_bounds__(PART_THREADS) k_part_scatter(const Node* __restrict__ nodes, const int* __restrict__ split,
                                                               const uint32_t* __restrict__ choff, const uint32_t* __restrict__ n_nodes_p,
                                                               const uint32_t* __restrict__ total_ch_p,
                                                               const uint32_t* __restrict__ zoff, const uint32_t* __restrict__ zeros,
                                                               const uint32_t* __restrict__ perm, const uint8_t* __restrict__ EP,
                                                               int64_t n, int LK, int K, int nb, uint32_t* __restrict__ perm_out) {
    pdl_wait();
    __shared__ uint32_t s_warp[PART_THREADS / 32];
    const uint32_t c = blockIdx.x;
    if (c >= *total_ch_p) return;
    const int64_t a = chunk_owner(choff, *n_nodes_p, c);
    const Node nd = nodes[a];
    const int j = split[a];
    const int t = (int)(nd.start / n);
    const int shift = nb - 1 - nib(nd.bits, j);
    const int64_t base = (int64_t)(c - choff[a]) * PART_CHUNK;
    const uint32_t Z = zeros[a], z0 = zoff[c];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t run0 = 0;  // zeros before this round inside the chunk
    for (int q = 0; q < PART_IPT; ++q) {
        const int64_t e = base + q * PART_THREADS + threadIdx.x;
        const bool ok = e < nd.len;
        uint32_t id = 0;
        int bit = 1;
        if (ok) {
            id = perm[nd.start + e];
            bit = next_bit_of(EP, id, LK, t * K + j, shift);
        }
        const uint32_t is0 = ok && bit == 0;
        const uint32_t bal = __ballot_sync(0xffffffffu, is0);
        if (lane == 0) s_warp[w] = __popc(bal);
        __syncthreads();
        uint32_t before = run0, tot = 0;
        for (int ww = 0; ww < PART_THREADS / 32; ++ww) {
            if (ww < w) before += s_warp[ww];
            tot += s_warp[ww];
        }
        before += __popc(bal & lanemask_lt());
        if (ok) {
            const int64_t pos_in_chunk = q * PART_THREADS + threadIdx.x;
            const uint32_t r0 = before;                                   // zeros before me in chunk
            const uint32_t r1 = (uint32_t)(pos_in_chunk) - (r0 - 0);       // ones before me in chunk
            uint32_t dst;
            if (is0) dst = nd.start + z0 + r0;
            else dst = nd.start + Z + ((uint32_t)base - z0) + r1;
            perm_out[dst] = id;
        }
        run0 += tot;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(PART_THREADS) k_part_copy(const Node* __restrict__ nodes,
                                                            const uint32_t* __restrict__ choff,
                                                            const uint32_t* __restrict__ n_nodes_p,
                                                            const uint32_t* __restrict__ total_ch_p,
                                                            const uint32_t* __restrict__ src, uint32_t* __restrict__ dst) {
    pdl_wait();
    const uint32_t c = blockIdx.x;
    if (c >= *total_ch_p) return;
    const int64_t a = chunk_owner(choff, *n_nodes_p, c);
    const Node nd = nodes[a];
    const int64_t base = (int64_t)(c - choff[a]) * PART_CHUNK;
    for (int q = 0; q < PART_IPT; ++q) {
        const int64_t e = base + q * PART_THREADS + threadIdx.x;
        if (e < nd.len) dst[nd.start + e] = src[nd.start + e];
    }
}

__global__ void k_make_children(const Node* __restrict__ nodes, const uint32_t* __restrict__ n_nodes_p,
                                const int* __restrict__ split, const uint32_t* __restrict__ zeros,
                                int K, int nb, int max_size, Sinks sk) {
    pdl_wait();
    const uint32_t n_nodes = *n_nodes_p;
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n_nodes;
         a += (int64_t)gridDim.x * blockDim.x) {
        const Node nd = nodes[a];
        const int j = split[a];
        if (j < 0) {                          // unsplittable: an oversized leaf (AMB-9)
            push_node(sk.leaves, sk.n_leaves, sk.cap_leaves, nd);
            continue;
        }
        const uint32_t Z = zeros[a];
        for (int b = 0; b < 2; ++b) {
            Node ch = nd;
            nib_inc(ch.bits, j);
            ch.start = b ? nd.start + Z : nd.start;
            ch.len = b ? nd.len - Z : Z;
            if (ch.len == 0) continue;        // empty children are dropped (AMB-11)
            route_node(sk, ch, K, nb, max_size);
        }
    }
}

// The rest of B6 for one node of <= LM points, entirely in shared memory: the same SplitNode
// rule and stable partition as k_choose_split / k_part_* above, applied level by level to the
// node's sub-nodes until every piece is a leaf.  Codes are staged once (gathered from EP);
// partitions move 16-bit positions only; perm is written back at the end.  One CTA per node
// (grid-stride over the local list).
constexpr int LF_MAXSEG = 64;       // live sub-nodes per level (each > max_size points: LM / (max_size+1))

template <int KM, int LF_THREADS>   // KM >= K: 16 or 32 (split-count registers)
__global__ void __launch_bounds__(LF_THREADS, 1024 / LF_THREADS) k_local_finish(const Node* __restrict__ loc, const uint32_t* __restrict__ n_loc_p,
                                                             int LM, uint32_t* __restrict__ perm, const uint8_t* __restrict__ EP,
                                                             int64_t n, int LK, int K, int nb, int max_size,
                                                             Node* __restrict__ leaves, uint32_t* __restrict__ n_leaves,
                                                             uint32_t cap_leaves, int64_t rev_cap) {
    pdl_wait();
    extern __shared__ __align__(16) unsigned char lf_smem[];
    const int CB = K <= 16 ? 16 : 32;                                     // code bytes per point
    uint8_t* s_code = lf_smem;                                            // [LM][CB], load order
    uint32_t* s_id = reinterpret_cast<uint32_t*>(s_code + (size_t)LM * CB);   // [LM] point ids, load order
    uint16_t* s_ixa = reinterpret_cast<uint16_t*>(s_id + LM);             // [LM] current order -> load slot
    uint16_t* s_ixb = s_ixa + LM;
    uint16_t* s_pz = s_ixb + LM;                                          // [LM+1] exclusive prefix of zeros
    uint8_t* s_seg = reinterpret_cast<uint8_t*>(s_pz + LM + 8);           // [LM] live sub-node of each position
    __shared__ Node s_act[2][LF_MAXSEG];
    __shared__ int s_dim[LF_MAXSEG], s_shift[LF_MAXSEG];
    __shared__ uint32_t s_ones[LF_MAXSEG * KM];                          // per live sub-node: ones per dim
    __shared__ uint32_t s_nact[2], s_wsum[LF_THREADS / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = LF_THREADS / 32;
    const uint32_t n_loc = *n_loc_p;
    for (uint32_t a = blockIdx.x; a < n_loc; a += gridDim.x) {
        const Node nd = loc[rev_cap ? rev_cap - 1 - (int64_t)a : (int64_t)a];   // rev_cap: the back tier
        const int t = (int)(nd.start / n);
        const int m = (int)nd.len;
        const uint32_t base = nd.start;
        for (int i = tid; i < m; i += LF_THREADS) {
            const uint32_t id = perm[base + i];
            s_id[i] = id;
            s_ixa[i] = (uint16_t)i;
            const uint8_t* c = EP + (int64_t)id * LK + t * K;
            if (K == 16 && (LK & 15) == 0) {
                *reinterpret_cast<uint4*>(s_code + i * 16) = *reinterpret_cast<const uint4*>(c);
            } else {
                for (int j = 0; j < K; ++j) s_code[i * CB + j] = c[j];
            }
        }
        if (tid == 0) { s_act[0][0] = nd; s_nact[0] = 1; }
        for (int i = tid; i < KM; i += LF_THREADS) s_ones[i] = 0;
        __syncthreads();
        uint16_t* ix = s_ixa;
        uint16_t* ix2 = s_ixb;
        const int IT = (m + LF_THREADS - 1) / LF_THREADS;   // positions per thread in the scan (<= 8)
        for (int cur = 0;; cur ^= 1) {
            const int nact = (int)s_nact[cur];
            if (nact == 0) break;
            // SplitNode dimension of each live sub-node (AMB-9), block-wide: warp items are
            // (sub-node, 32 of its first max_size points); per dim a ballot counts the item's ones and
            // lane j adds dim j's count to the sub-node's tally (s_ones, zeroed a phase earlier); then
            // a thread per sub-node takes the dim with bits left whose next bit most evenly divides
            // those points, ties to the lowest dim -- as k_choose_split.  (A warp per sub-node left
            // the other warps at the next barrier: 34 % of the stall samples, ncu.)
            {
                const int CH = (max_size + 31) / 32;
                for (int wi = warp; wi < nact * CH; wi += nwarps) {
                    const int sg = wi / CH, e = (wi - sg * CH) * 32 + lane;
                    const Node sn = s_act[cur][sg];
                    const int st = (int)(sn.start - base);
                    const bool ok = e < max_size;
                    const uint8_t* c = s_code + (int)ix[st + (ok ? e : 0)] * CB;
                    uint32_t my = 0;
                    if (KM == 16 && CB == 16) {
                        // the 16 codes in 4 words; dim j's next bit at 8 (j & 3) + nb - 1 - b_j of
                        // word j / 4; one REDUX per dim
                        const uint4 c4 = *reinterpret_cast<const uint4*>(c);
                        const uint32_t wv[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            if (j < K) {
                                const int b = nib(sn.bits, j);
                                const uint32_t bit = (ok && b < nb) ? (wv[j >> 2] >> (8 * (j & 3) + nb - 1 - b)) & 1u : 0u;
                                const uint32_t cnt = __reduce_add_sync(0xffffffffu, bit);
                                my = lane == j ? cnt : my;
                            }
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < KM; ++j) {
                            if (j < K) {
                                const int b = nib(sn.bits, j);
                                const bool bit = ok && b < nb && ((c[j] >> (nb - 1 - b)) & 1);
                                const uint32_t cnt = __popc(__ballot_sync(0xffffffffu, bit));
                                if (lane == j) my = cnt;
                            }
                        }
                    }
                    if (lane < K && my) atomicAdd(&s_ones[sg * KM + lane], my);
                }
            }
            __syncthreads();
            for (int sg = tid; sg < nact; sg += LF_THREADS) {   // live sub-nodes are splittable: best >= 0
                const Node sn = s_act[cur][sg];
                int best = -1, best_imb = 0x7fffffff;
                for (int j = 0; j < K; ++j)
                    if (nib(sn.bits, j) < nb) {
                        const int imb = abs(max_size - 2 * (int)s_ones[sg * KM + j]);
                        if (imb < best_imb) { best_imb = imb; best = j; }
                    }
                s_dim[sg] = best;
                s_shift[sg] = nb - 1 - nib(sn.bits, best);
            }
            for (int i = tid; i < m; i += LF_THREADS) s_seg[i] = 0xFF;
            if (tid == 0) s_nact[cur ^ 1] = 0;
            __syncthreads();
            for (int sg = warp; sg < nact; sg += nwarps) {
                const int st = (int)(s_act[cur][sg].start - base), len = (int)s_act[cur][sg].len;
                for (int e = lane; e < len; e += 32) s_seg[st + e] = (uint8_t)sg;
            }
            // next level's tallies (at most two live children per live sub-node)
            for (int i = tid; i < min(2 * nact, LF_MAXSEG) * KM; i += LF_THREADS) s_ones[i] = 0;
            __syncthreads();
            // zero flags of positions in live sub-nodes, block-wide exclusive scan
            uint32_t fl = 0, cnt = 0;
            for (int q = 0; q < IT; ++q) {
                const int i = tid * IT + q;
                if (i < m && s_seg[i] != 0xFF) {
                    const int sg = s_seg[i];
                    const uint32_t z = 1u - ((s_code[(int)ix[i] * CB + s_dim[sg]] >> s_shift[sg]) & 1u);
                    fl |= z << q;
                    cnt += z;
                }
            }
            uint32_t inc = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += v;
            }
            if (lane == 31) s_wsum[warp] = inc;
            __syncthreads();
            uint32_t wpre = 0;
            for (int w = 0; w < warp; ++w) wpre += s_wsum[w];
            uint32_t run = wpre + inc - cnt;
            for (int q = 0; q < IT; ++q) {
                const int i = tid * IT + q;
                if (i < m) s_pz[i] = (uint16_t)run;
                run += (fl >> q) & 1u;
            }
            if (tid == LF_THREADS - 1) s_pz[m] = (uint16_t)run;
            __syncthreads();
            // stable partition of every live sub-node: zeros first, then ones
            for (int i = tid; i < m; i += LF_THREADS) {
                const int sg = s_seg[i];
                if (sg == 0xFF) { ix2[i] = ix[i]; continue; }
                const int st = (int)(s_act[cur][sg].start - base), len = (int)s_act[cur][sg].len;
                const int pst = s_pz[st], Zs = (int)s_pz[st + len] - pst, zb = (int)s_pz[i] - pst;
                const bool is0 = s_pz[i + 1] != s_pz[i];
                const int dst = is0 ? st + zb : st + Zs + (i - st - zb);
                ix2[dst] = ix[i];
            }
            // children, as k_make_children: leaves out, the rest live at the next level
            for (int sg = tid; sg < nact; sg += LF_THREADS) {
                const Node sn = s_act[cur][sg];
                const int st = (int)(sn.start - base);
                const uint32_t Z = (uint32_t)(s_pz[st + sn.len] - s_pz[st]);
                for (int b = 0; b < 2; ++b) {
                    Node ch = sn;
                    nib_inc(ch.bits, s_dim[sg]);
                    ch.start = b ? sn.start + Z : sn.start;
                    ch.len = b ? sn.len - Z : Z;
                    if (ch.len == 0) continue;
                    if ((int64_t)ch.len <= max_size || !splittable(ch.bits, K, nb)) {
                        push_node(leaves, n_leaves, cap_leaves, ch);
                    } else {
                        const uint32_t k = atomicAdd(&s_nact[cur ^ 1], 1u);
                        s_act[cur ^ 1][k] = ch;
                    }
                }
            }
            __syncthreads();
            uint16_t* tmp = ix; ix = ix2; ix2 = tmp;
        }
        for (int i = tid; i < m; i += LF_THREADS) perm[base + i] = s_id[ix[i]];
        __syncthreads();
    }
}

size_t local_finish_smem(int LM, int K) {
    return (size_t)LM * ((K <= 16 ? 16 : 32) + 4 + 2 + 2 + 2 + 1) + 16 + 64;
}

// Canonical leaf order (ascending start) without a sort: leaves tile [0, L*n) disjointly, so a
// leaf's rank is the number of leaf starts before its own -- a bitmap of starts plus a prefix
// count of its words.
__global__ void k_leaf_starts(const Node* __restrict__ leaves, const uint32_t* __restrict__ nl_p,
                              uint32_t* __restrict__ bitmap) {
    pdl_wait();
    const uint32_t nl = *nl_p;
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < nl;
         l += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t s = leaves[l].start;
        atomicOr(&bitmap[s >> 5], 1u << (s & 31));
    }
}

__global__ void k_word_popc(const uint32_t* __restrict__ bitmap, int64_t nw, uint32_t* __restrict__ cnt) {
    pdl_wait();
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nw;
         w += (int64_t)gridDim.x * blockDim.x)
        cnt[w] = __popc(bitmap[w]);
}

__global__ void k_leaf_rank(const Node* __restrict__ leaves, const uint32_t* __restrict__ nl_p,
                            const uint32_t* __restrict__ bitmap, const uint32_t* __restrict__ pre,
                            uint32_t* __restrict__ order) {
    pdl_wait();
    const uint32_t nl = *nl_p;
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < nl;
         l += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t s = leaves[l].start;
        const uint32_t r = pre[s >> 5] + __popc(bitmap[s >> 5] & ((1u << (s & 31)) - 1u));
        order[r] = (uint32_t)l;
    }
}

__global__ void k_leaf_finalize(const Node* __restrict__ leaves, const uint32_t* __restrict__ order, int64_t nl,
                                const uint32_t* __restrict__ perm, const uint8_t* __restrict__ EP, int64_t n,
                                int LK, int K, int nb, uint32_t* __restrict__ leaf_off, uint8_t* __restrict__ lo,
                                uint8_t* __restrict__ hi, uint8_t* __restrict__ bits, int64_t total) {
    pdl_wait();
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < nl;
         l += (int64_t)gridDim.x * blockDim.x) {
        const Node nd = leaves[order[l]];
        leaf_off[l] = nd.start;
        const int t = (int)(nd.start / n);
        const uint8_t* c = EP + (int64_t)perm[nd.start] * LK + t * K;
        for (int j = 0; j < K; ++j) {
            const int b = nib(nd.bits, j), fr = nb - b;
            const int l0 = (c[j] >> fr) << fr;
            lo[l * K + j] = (uint8_t)l0;
            hi[l * K + j] = (uint8_t)(l0 + (1 << fr) - 1);
            bits[l * K + j] = (uint8_t)b;
        }
        if (l == nl - 1) leaf_off[nl] = (uint32_t)total;
    }
}

__global__ void k_tree_begin(const uint32_t* __restrict__ leaf_off, int64_t nl, int64_t n, int L,
                             unsigned long long* __restrict__ begin) {
    pdl_wait();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t > L) return;
    const uint64_t target = (uint64_t)t * n;   // first leaf with start >= t*n
    int64_t lo = 0, hi = nl;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (leaf_off[mid] < target) lo = mid + 1; else hi = mid;
    }
    begin[t] = (unsigned long long)lo;
}

__global__ void k_gather_tcodes(const uint32_t* __restrict__ perm, const uint8_t* __restrict__ EP, int64_t n,
                                int L, int K, uint8_t* __restrict__ tcodes) {
    pdl_wait();
    const int LK = L * K;
    const int64_t total = n * L;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int t = (int)(g / n);
        const uint8_t* src = EP + (int64_t)perm[g] * LK + t * K;
        uint8_t* dst = tcodes + g * K;
        if ((K & 15) == 0) {
            for (int j = 0; j < K; j += 16)
                *reinterpret_cast<uint4*>(dst + j) = *reinterpret_cast<const uint4*>(src + j);
        } else {
            for (int j = 0; j < K; ++j) dst[j] = src[j];
        }
    }
}

__global__ void k_gather_rows_strided(const float* __restrict__ src, int64_t src_ld, int d,
                                      const uint32_t* __restrict__ ids, int64_t m, float* __restrict__ dst,
                                      int64_t dst_ld) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < m; r += nwarps) {
        const float* s = src + (int64_t)ids[r] * src_ld;
        float* o = dst + r * dst_ld;
        for (int64_t f = lane; f < dst_ld; f += 32) o[f] = f < d ? s[f] : 0.f;
    }
}

// Query tiles: runs of kTileLeaves consecutive leaves of one
// tree (the last tile of a tree may be shorter); one warp of the range filter owns a tile.
__global__ void k_tile_flags(const uint32_t* __restrict__ leaf_off, int64_t nl, int64_t n, int tl,
                             const unsigned long long* __restrict__ tree_begin, uint32_t* __restrict__ flags) {
    pdl_wait();
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < nl;
         l += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = leaf_off[l] / n;
        flags[l] = ((l - (int64_t)tree_begin[t]) % tl == 0) ? 1u : 0u;
    }
}

// Within each leaf, the points reordered by a locality key: the top bits of the K codes
// interleaved bit-plane by bit-plane (Morton / z-order; min(8, 64 / K) bits per dim), ties by the
// original (id) order.  A leaf is a set (Alg. 3 takes its points by their own bounds), so the
// order is free; consecutive points then lie close in every dim and the sub-boxes of kSubBox
// consecutive points (k_sb_boxes) get tight boxes -- measured on a configs[4]-like tree, half the
// points behind passing sub-boxes.  Warp per leaf of <= 128 points (bitonic sort in shared
// memory); larger (unsplittable) leaves keep their order.  perm and tcodes move together.
constexpr int LM_WARPS = 8;
// Bits b (7 >= b > 7 - 4) of the four code bytes of w gathered into a nibble (byte 0 lowest):
// the bits sit at positions 0, 8, 16, 24 and one multiply moves them to 24..27 without carries.
__device__ __forceinline__ uint32_t plane_nibble(uint32_t w, int b) {
    return ((((w >> b) & 0x01010101u) * 0x01020408u) >> 24) & 0xFu;
}
__global__ void __launch_bounds__(LM_WARPS * 32) k_leaf_morton(const uint32_t* __restrict__ leaf_off, int64_t nl, int K,
                                                               uint32_t* __restrict__ perm, uint8_t* __restrict__ tcodes) {
    pdl_wait();
    __shared__ unsigned long long s_key[LM_WARPS][128];
    __shared__ uint32_t s_idx[LM_WARPS][128];
    __shared__ uint32_t s_perm[LM_WARPS][128];
    __shared__ __align__(16) uint8_t s_codes[LM_WARPS][128 * 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int bpd = K >= 8 ? (64 / K > 8 ? 8 : 64 / K) : 8;       // key bits per dim (generic K)
    for (int64_t l = (int64_t)blockIdx.x * LM_WARPS + w; l < nl; l += (int64_t)gridDim.x * LM_WARPS) {
        const uint32_t p0 = leaf_off[l];
        const int m = (int)(leaf_off[l + 1] - p0);
        if (m <= 2 || m > 128) continue;
        int P2 = 4;                                   // sort size: next power of two >= m
        while (P2 < m) P2 <<= 1;
        for (int e = lane; e < P2; e += 32) {
            unsigned long long key = ~0ull;
            if (e < m) {
                const uint8_t* c = tcodes + (int64_t)(p0 + e) * K;
                s_perm[w][e] = perm[p0 + e];
                if (K == 16) {
                    const uint4 c4 = *reinterpret_cast<const uint4*>(c);
                    *reinterpret_cast<uint4*>(&s_codes[w][e * 16]) = c4;
                    key = 0;
#pragma unroll
                    for (int b = 7; b > 3; --b)           // 4 bit-planes x 16 dims = 64 bits
                        key = (key << 16) | (plane_nibble(c4.x, b) << 12) | (plane_nibble(c4.y, b) << 8) |
                              (plane_nibble(c4.z, b) << 4) | plane_nibble(c4.w, b);
                } else {
                    key = 0;
                    for (int b = 0; b < bpd; ++b)
                        for (int j = 0; j < K; ++j) key = (key << 1) | ((c[j] >> (7 - b)) & 1u);
                    for (int j = 0; j < K; ++j) s_codes[w][e * K + j] = c[j];
                }
            }
            s_key[w][e] = key;
            s_idx[w][e] = (uint32_t)e;
        }
        __syncwarp();
        // bitonic sort of the P2 (key, idx) pairs, ascending
        for (int size = 2; size <= P2; size <<= 1) {
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int t = lane; t < (P2 >> 1); t += 32) {
                    const int i = 2 * t - (t & (stride - 1)), j = i + stride;
                    const bool up = (i & size) == 0;
                    const unsigned long long ki = s_key[w][i], kj = s_key[w][j];
                    const uint32_t ii = s_idx[w][i], ij = s_idx[w][j];
                    const bool gt = ki > kj || (ki == kj && ii > ij);
                    if (gt == up) {
                        s_key[w][i] = kj; s_key[w][j] = ki;
                        s_idx[w][i] = ij; s_idx[w][j] = ii;
                    }
                }
                __syncwarp();
            }
        }
        for (int e = lane; e < m; e += 32) {
            const uint32_t src = s_idx[w][e];
            perm[p0 + e] = s_perm[w][src];
            uint8_t* dst = tcodes + (int64_t)(p0 + e) * K;
            if (K == 16) {
                *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(&s_codes[w][src * 16]);
            } else {
                for (int j = 0; j < K; ++j) dst[j] = s_codes[w][src * K + j];
            }
        }
        __syncwarp();
    }
}

// Fused leaf layout for K = 16 (the Morton path): per leaf (warp per leaf), the points' codes
// are gathered from the data-order codes EP (the k_gather_tcodes step), the points sorted by
// their Morton key in registers (bitonic network over 32 / 64 / 128 elements, shuffles for
// strides < 32, register swaps above; the key's low 7 bits carry the element's original slot,
// so keys are distinct and the order deterministic), perm and tcodes written in that order, and
// the sub-boxes (runs of kSubBox = 8 positions: one 8-lane group per register) and the leaf's
// tight box reduced on the fly (k_sb_boxes + k_leaf_tight_sb).  Leaves of > 128 points
// (unsplittable duplicates) keep their order and take the plain loops.
__device__ __forceinline__ uint4 vmin4(uint4 a, uint4 b) {
    return make_uint4(__vminu4(a.x, b.x), __vminu4(a.y, b.y), __vminu4(a.z, b.z), __vminu4(a.w, b.w));
}
__device__ __forceinline__ uint4 vmax4(uint4 a, uint4 b) {
    return make_uint4(__vmaxu4(a.x, b.x), __vmaxu4(a.y, b.y), __vmaxu4(a.z, b.z), __vmaxu4(a.w, b.w));
}
__device__ __forceinline__ uint4 shfl_xor4(uint4 v, int m) {
    return make_uint4(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m),
                      __shfl_xor_sync(0xffffffffu, v.z, m), __shfl_xor_sync(0xffffffffu, v.w, m));
}
// 16 code bytes spread into 8 words of 16-bit lanes (even bytes of word i in e[i], odd in o[i]):
// byte-wise min / max of two such boxes is 8 VIMNMX.U16x2 (the packed __vminu4 is emulated, ~6
// instructions per word), packed back into bytes once at the end.
struct Spread16 { uint32_t v[8]; };
__device__ __forceinline__ Spread16 spread16(uint4 c) {
    const uint32_t w[4] = {c.x, c.y, c.z, c.w};
    Spread16 r;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        r.v[2 * i] = __byte_perm(w[i], 0u, 0x4240);
        r.v[2 * i + 1] = __byte_perm(w[i], 0u, 0x4341);
    }
    return r;
}
__device__ __forceinline__ uint4 pack16(const Spread16& a) {   // inverse of spread16
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = __byte_perm(a.v[2 * i], a.v[2 * i + 1], 0x6240);
    return make_uint4(w[0], w[1], w[2], w[3]);
}
__device__ __forceinline__ void min16x2_into(Spread16& a, const Spread16& b) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm("min.u16x2 %0, %0, %1;" : "+r"(a.v[i]) : "r"(b.v[i]));
}
__device__ __forceinline__ void max16x2_into(Spread16& a, const Spread16& b) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm("max.u16x2 %0, %0, %1;" : "+r"(a.v[i]) : "r"(b.v[i]));
}
__device__ __forceinline__ Spread16 shfl_xor16(const Spread16& a, int m) {
    Spread16 r;
#pragma unroll
    for (int i = 0; i < 8; ++i) r.v[i] = __shfl_xor_sync(0xffffffffu, a.v[i], m);
    return r;
}
constexpr int LL_WARPS = 8;
__global__ void __launch_bounds__(LL_WARPS * 32) k_leaf_layout16(const uint32_t* __restrict__ leaf_off, int64_t nl,
                                                                 const uint32_t* __restrict__ sb_off,
                                                                 uint32_t* __restrict__ perm, const uint8_t* __restrict__ EP,
                                                                 int64_t n, int LK, uint8_t* __restrict__ tcodes,
                                                                 uint8_t* __restrict__ sbox, uint8_t* __restrict__ tbox) {
    pdl_wait();
    __shared__ uint4 s_c[LL_WARPS][128];
    __shared__ uint32_t s_p[LL_WARPS][128];
    __shared__ uint8_t s_srt[LL_WARPS][128];          // sorted position -> gathered slot
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint4 NEUT_LO = make_uint4(~0u, ~0u, ~0u, ~0u), NEUT_HI = make_uint4(0, 0, 0, 0);
    for (int64_t l = (int64_t)blockIdx.x * LL_WARPS + w; l < nl; l += (int64_t)gridDim.x * LL_WARPS) {
        const uint32_t p0 = leaf_off[l];
        const int m = (int)(leaf_off[l + 1] - p0);
        const int t = (int)(p0 / n);
        const int64_t cb = (int64_t)t * 16;
        uint32_t sb0 = sb_off[l];
        if (m > 128) {     // unsplittable oversized leaf: gather in place, boxes by plain loops
            for (int e = lane; e < m; e += 32) {
                const uint4 c = *reinterpret_cast<const uint4*>(EP + (int64_t)perm[p0 + e] * LK + cb);
                *reinterpret_cast<uint4*>(tcodes + (int64_t)(p0 + e) * 16) = c;
            }
            __syncwarp();
            uint4 tl = NEUT_LO, th = NEUT_HI;
            for (int s = lane; s < (m + kSubBox - 1) / kSubBox; s += 32) {
                uint4 lo = NEUT_LO, hi = NEUT_HI;
                for (int e = s * kSubBox; e < min(m, (s + 1) * kSubBox); ++e) {
                    const uint4 c = *reinterpret_cast<const uint4*>(tcodes + (int64_t)(p0 + e) * 16);
                    lo = vmin4(lo, c);
                    hi = vmax4(hi, c);
                }
                *reinterpret_cast<uint4*>(sbox + (int64_t)(sb0 + s) * 32) = lo;
                *reinterpret_cast<uint4*>(sbox + (int64_t)(sb0 + s) * 32 + 16) = hi;
                tl = vmin4(tl, lo);
                th = vmax4(th, hi);
            }
            for (int o = 16; o > 0; o >>= 1) {
                tl = vmin4(tl, shfl_xor4(tl, o));
                th = vmax4(th, shfl_xor4(th, o));
            }
            if (lane == 0) {
                *reinterpret_cast<uint4*>(tbox + l * 32) = tl;
                *reinterpret_cast<uint4*>(tbox + l * 32 + 16) = th;
            }
            continue;
        }
        const int R = m <= 32 ? 1 : m <= 64 ? 2 : 4;          // elements per lane (P2 = 32 R)
        unsigned long long key[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int e = r * 32 + lane;
            key[r] = ~0ull;
            if (r < R && e < m) {
                const uint32_t id = perm[p0 + e];
                const uint4 c = *reinterpret_cast<const uint4*>(EP + (int64_t)id * LK + cb);
                s_c[w][e] = c;
                s_p[w][e] = id;
                unsigned long long k = 0;
#pragma unroll
                for (int b = 7; b > 3; --b)
                    k = (k << 16) | (plane_nibble(c.x, b) << 12) | (plane_nibble(c.y, b) << 8) |
                        (plane_nibble(c.z, b) << 4) | plane_nibble(c.w, b);
                key[r] = ((k >> 1) & ~127ull) | (unsigned long long)e;     // real keys < 2^63
            } else if (r < R) {
                key[r] = (1ull << 63) | (unsigned long long)e;             // padding: after every real key
            }
        }
        // bitonic sort, ascending, element e = r * 32 + lane (compile-time register indices only)
        const int P2 = 32 * R;
        auto cmpx = [](unsigned long long& x, unsigned long long& y, bool asc) {   // x: lower slot
            const unsigned long long mn = x < y ? x : y, mx = x < y ? y : x;
            x = asc ? mn : mx;
            y = asc ? mx : mn;
        };
        for (int size = 2; size <= P2; size <<= 1) {
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                if (stride >= 64) {                       // pairs (0,2), (1,3)
                    cmpx(key[0], key[2], ((0 * 32 + lane) & size) == 0);
                    cmpx(key[1], key[3], ((1 * 32 + lane) & size) == 0);
                } else if (stride == 32) {                // pairs (0,1), (2,3)
                    cmpx(key[0], key[1], ((0 * 32 + lane) & size) == 0);
                    if (R == 4) cmpx(key[2], key[3], ((2 * 32 + lane) & size) == 0);
                } else {
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        if (r >= R) continue;
                        const int e = r * 32 + lane;
                        const unsigned long long other = __shfl_xor_sync(0xffffffffu, key[r], stride);
                        const bool asc = (e & size) == 0, lower = (e & stride) == 0;
                        const unsigned long long mn = key[r] < other ? key[r] : other;
                        const unsigned long long mx = key[r] < other ? other : key[r];
                        key[r] = (lower == asc) ? mn : mx;
                    }
                }
            }
        }
        __syncwarp();
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (r >= R) continue;
            const int e = r * 32 + lane;
            if (e < m) {
                const int src = (int)(key[r] & 127ull);
                s_srt[w][e] = (uint8_t)src;
                perm[p0 + e] = s_p[w][src];
                *reinterpret_cast<uint4*>(tcodes + (int64_t)(p0 + e) * 16) = s_c[w][src];
            }
        }
        __syncwarp();
        // sub-box s = sorted positions [8 s, 8 s + 8) on lane s (<= 16 of them), byte-wise min / max
        // in the spread form; then the leaf's tight box as the union of its sub-boxes' boxes
        const int nsb = (m + kSubBox - 1) / kSubBox;
        Spread16 lo, hi;
#pragma unroll
        for (int i = 0; i < 8; ++i) { lo.v[i] = 0x00FF00FFu; hi.v[i] = 0u; }
        if (lane < nsb) {
            const int e0 = lane * kSubBox, e1 = min(m, e0 + kSubBox);
            for (int e = e0; e < e1; ++e) {
                const Spread16 c = spread16(s_c[w][s_srt[w][e]]);
                min16x2_into(lo, c);
                max16x2_into(hi, c);
            }
            const uint32_t sidx = sb0 + (uint32_t)lane;
            *reinterpret_cast<uint4*>(sbox + (int64_t)sidx * 32) = pack16(lo);
            *reinterpret_cast<uint4*>(sbox + (int64_t)sidx * 32 + 16) = pack16(hi);
        }
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) {             // nsb <= 16: lanes 0-15 hold every sub-box
            min16x2_into(lo, shfl_xor16(lo, o));
            max16x2_into(hi, shfl_xor16(hi, o));
        }
        if (lane == 0) {
            *reinterpret_cast<uint4*>(tbox + l * 32) = pack16(lo);
            *reinterpret_cast<uint4*>(tbox + l * 32 + 16) = pack16(hi);
        }
        __syncwarp();
    }
}

// Sub-boxes: each leaf's points cut into runs of kSubBox consecutive points (leaf order); per
// run the min/max code per dim.  A valid lower bound for every member, tighter than the leaf's
// (a few points span less of each dim): the pair kernel screens runs before their points.
__global__ void k_sb_count(const uint32_t* __restrict__ leaf_off, int64_t nl, uint32_t* __restrict__ cnt) {
    pdl_wait();
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < nl; l += (int64_t)gridDim.x * blockDim.x)
        cnt[l] = (leaf_off[l + 1] - leaf_off[l] + kSubBox - 1) / kSubBox;
}

// thread per sub-box (its leaf by binary search over sb_off); consecutive threads read
// consecutive runs of points
// Boxes are interleaved: box i = lo (K bytes) then hi (K bytes) at box + 2K i.
__global__ void k_sb_boxes(const uint32_t* __restrict__ leaf_off, const uint32_t* __restrict__ sb_off, int64_t nl, int K,
                           const uint8_t* __restrict__ tcodes, uint8_t* __restrict__ box) {
    pdl_wait();
    const uint32_t nsb = sb_off[nl];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nsb; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t a_ = 0, b_ = nl - 1;                  // last leaf l with sb_off[l] <= i
        while (a_ < b_) {
            const int64_t m = (a_ + b_ + 1) >> 1;
            if (sb_off[m] <= (uint32_t)i) a_ = m; else b_ = m - 1;
        }
        const uint32_t p0 = leaf_off[a_] + (uint32_t)(i - sb_off[a_]) * kSubBox;
        const uint32_t e = min(p0 + (uint32_t)kSubBox, leaf_off[a_ + 1]);
        if (K == 16) {
            uint4 mn = make_uint4(~0u, ~0u, ~0u, ~0u), mx = make_uint4(0, 0, 0, 0);
            for (uint32_t p = p0; p < e; ++p) {
                const uint4 c = *reinterpret_cast<const uint4*>(tcodes + (int64_t)p * 16);
                mn = make_uint4(__vminu4(mn.x, c.x), __vminu4(mn.y, c.y), __vminu4(mn.z, c.z), __vminu4(mn.w, c.w));
                mx = make_uint4(__vmaxu4(mx.x, c.x), __vmaxu4(mx.y, c.y), __vmaxu4(mx.z, c.z), __vmaxu4(mx.w, c.w));
            }
            *reinterpret_cast<uint4*>(box + i * 32) = mn;
            *reinterpret_cast<uint4*>(box + i * 32 + 16) = mx;
        } else {
            for (int j = 0; j < K; ++j) {
                int mn = 255, mx = 0;
                for (uint32_t p = p0; p < e; ++p) {
                    const int c = tcodes[(int64_t)p * K + j];
                    mn = min(mn, c);
                    mx = max(mx, c);
                }
                box[i * 2 * K + j] = (uint8_t)mn;
                box[i * 2 * K + K + j] = (uint8_t)mx;
            }
        }
    }
}

// Tight box of each leaf as the union of its sub-boxes' boxes (same min/max over the same points).
__global__ void k_leaf_tight_sb(const uint32_t* __restrict__ sb_off, int64_t nl, int K, const uint8_t* __restrict__ sbox,
                                uint8_t* __restrict__ tbox) {
    pdl_wait();
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < nl; l += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t a = sb_off[l], e = sb_off[l + 1];
        if (K == 16) {
            uint4 mn = make_uint4(~0u, ~0u, ~0u, ~0u), mx = make_uint4(0, 0, 0, 0);
            for (uint32_t b = a; b < e; ++b) {
                const uint4 x = *reinterpret_cast<const uint4*>(sbox + (int64_t)b * 32);
                const uint4 y = *reinterpret_cast<const uint4*>(sbox + (int64_t)b * 32 + 16);
                mn = make_uint4(__vminu4(mn.x, x.x), __vminu4(mn.y, x.y), __vminu4(mn.z, x.z), __vminu4(mn.w, x.w));
                mx = make_uint4(__vmaxu4(mx.x, y.x), __vmaxu4(mx.y, y.y), __vmaxu4(mx.z, y.z), __vmaxu4(mx.w, y.w));
            }
            *reinterpret_cast<uint4*>(tbox + l * 32) = mn;
            *reinterpret_cast<uint4*>(tbox + l * 32 + 16) = mx;
        } else {
            for (int j = 0; j < K; ++j) {
                int mn = 255, mx = 0;
                for (uint32_t b = a; b < e; ++b) {
                    mn = min(mn, (int)sbox[(int64_t)b * 2 * K + j]);
                    mx = max(mx, (int)sbox[(int64_t)b * 2 * K + K + j]);
                }
                tbox[l * 2 * K + j] = (uint8_t)mn;
                tbox[l * 2 * K + K + j] = (uint8_t)mx;
            }
        }
    }
}

// Box of each query tile: per dim the smallest lo and largest hi over its leaves (the union's
// bounding box, so its lower bound never exceeds a member leaf's -- the filter skips whole tiles).
__global__ void k_tile_boxes(const uint32_t* __restrict__ tile_leaf, const uint32_t* __restrict__ ntiles_p, int K, const uint8_t* __restrict__ lo,
                             const uint8_t* __restrict__ hi, uint8_t* __restrict__ tlo, uint8_t* __restrict__ thi) {
    pdl_wait();
    const int64_t ntiles = *ntiles_p;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ntiles * K;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = i / K;
        const int j = (int)(i - t * K);
        int a = 255, b = 0;
        for (uint32_t l = tile_leaf[t]; l < tile_leaf[t + 1]; ++l) {     // leaf boxes interleaved (2K per box)
            a = min(a, (int)lo[(int64_t)l * 2 * K + j]);
            b = max(b, (int)hi[(int64_t)l * 2 * K + j]);
        }
        tlo[i] = (uint8_t)a;
        thi[i] = (uint8_t)b;
    }
}

__global__ void k_tile_write(const uint32_t* __restrict__ flags, const uint32_t* __restrict__ idx, int64_t nl,
                             uint32_t* __restrict__ tile_leaf) {
    pdl_wait();
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < nl;
         l += (int64_t)gridDim.x * blockDim.x)
        if (flags[l]) tile_leaf[idx[l]] = (uint32_t)l;
}

// Per point (tree order): index of its leaf within its query tile (< kTileLeaves).
// warp per tile: lane l holds the start of the tile's leaf l; each point's leaf slot by a
// 5-step shuffle search, written coalesced
__global__ void k_point_tile_leaf(const uint32_t* __restrict__ leaf_off, const uint32_t* __restrict__ tile_leaf,
                                  const uint32_t* __restrict__ ntiles_p, int64_t nl, uint16_t* __restrict__ ptl) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int64_t ntiles = *ntiles_p;
    for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < ntiles;
         t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const uint32_t lb = tile_leaf[t], le = tile_leaf[t + 1];
        const int nlt = (int)(le - lb);
        const uint32_t start = lane < nlt ? leaf_off[lb + lane] : 0xFFFFFFFFu;
        const uint32_t P0 = leaf_off[lb], P1 = leaf_off[le];
        for (uint32_t b = P0; b < P1; b += 32) {      // warp-uniform (shuffles below)
            const uint32_t p = b + lane;
            int o_ = 0;                               // last leaf slot with start <= p
#pragma unroll
            for (int sd = 16; sd > 0; sd >>= 1) {
                const uint32_t ex = __shfl_sync(0xffffffffu, start, o_ + sd);
                if (ex <= p) o_ += sd;
            }
            if (p < P1) ptl[p] = (uint16_t)o_;
        }
    }
    (void)nl;
}

// tile_begin[t] = first tile of tree t (tile_begin[L] = ntiles), and the tile list's end marker
// tile_leaf[ntiles] = nl -- all from device counts (no host round trip)
__global__ void k_tree_tiles(const uint32_t* __restrict__ idx, const unsigned long long* __restrict__ leaf_begin,
                             int L, const uint32_t* __restrict__ ntiles_p, uint32_t nl, uint32_t* __restrict__ tile_leaf,
                             unsigned long long* __restrict__ tile_begin) {
    pdl_wait();
    const int t = threadIdx.x;
    const uint32_t ntiles = *ntiles_p;
    if (t < L) tile_begin[t] = leaf_begin[t] < nl ? idx[leaf_begin[t]] : ntiles;
    if (t == L) {
        tile_begin[t] = ntiles;
        tile_leaf[ntiles] = nl;
    }
}

// ||x||^2 of every row, warp per row (used when the projection ran on the CUDA cores).
__global__ void k_row_norms(const float* __restrict__ X, int64_t ld, int64_t n, float* __restrict__ out) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < n;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const float* x = X + r * ld;
        float acc = 0.f;
        for (int64_t i = lane; i < ld; i += 32) acc = fmaf(x[i], x[i], acc);
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) out[r] = acc;
    }
}

int grid_for(int64_t work, int threads, int cap = 148 * 16) {
    int64_t g = ceil_div(std::max<int64_t>(work, 1), threads);
    return (int)std::min<int64_t>(g, cap);
}

template <class T> T d2h(const T* d, cudaStream_t st) {
    T h;
    DL_CUDA(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, st));
    DL_CUDA(cudaStreamSynchronize(st));
    return h;
}

}  // namespace

// ====================================================================== host drivers

// B1: ids in [id_lo, id_lo+n_range) among the n_s smallest keyed hashes of [0, n_global).
void sample_ids_device(uint64_t seed, int64_t id_lo, int64_t n_range, int64_t n_global, int64_t n_s,
                       uint32_t* d_out_local, int64_t* n_out_host, cudaStream_t st) {
    const uint64_t salt = seed ^ kSampleSalt;
    // fast path: 16-bit histogram + exact ranking of the threshold bin
    if (n_s <= 0) {
        *n_out_host = 0;
        return;
    }
    static const int cap_env = std::getenv("DETLSH_SEL16_CAP") ? std::atoi(std::getenv("DETLSH_SEL16_CAP")) : 0;  // tests
    const uint32_t ccap = cap_env > 0 ? (uint32_t)cap_env : (uint32_t)std::min<int64_t>(8192, 1024 + 2 * (n_global >> 16));
    Scratch s16(st, sizeof(uint32_t) * 65536 + sizeof(Sel16) + 2 * sizeof(unsigned long long) +
                        (sizeof(unsigned long long) + sizeof(uint32_t)) * (size_t)ccap + 64);
    uint32_t* hist = s16.as<uint32_t>();
    unsigned long long* ckey = reinterpret_cast<unsigned long long*>(hist + 65536);
    unsigned long long* counter = ckey + ccap;
    Sel16* state = reinterpret_cast<Sel16*>(counter + 1);
    uint32_t* cid = reinterpret_cast<uint32_t*>(state + 1);
    DL_CUDA(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * 65536, st));
    DL_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned long long) + sizeof(Sel16), st));
    const int g = grid_for(n_global, 256, 148 * 8);
    DL_LAUNCH(k_sel16_hist, g, 256, 0, st, salt, n_global, hist);
    DL_LAUNCH(k_sel16_pick, 1, 1024, 0, st, hist, n_s, state);
    DL_LAUNCH(k_sel16_collect, g, 256, 0, st, salt, id_lo, n_range, n_global, state, d_out_local, counter, ckey, cid, ccap);
    const size_t fsm = (sizeof(unsigned long long) + sizeof(uint32_t)) * (size_t)ccap;
    ensure_dyn_smem_fn(k_sel16_finish, fsm);
    DL_LAUNCH(k_sel16_finish, 1, 1024, fsm, st, id_lo, n_range, state, ckey, cid, ccap, d_out_local, counter);
    struct {
        unsigned long long got;
        Sel16 s;
    } h;
    DL_CUDA(cudaMemcpyAsync(&h.got, counter, sizeof(unsigned long long) + sizeof(Sel16), cudaMemcpyDeviceToHost, st));
    DL_CUDA(cudaStreamSynchronize(st));
    if (!h.s.overflow) {
        *n_out_host = (int64_t)h.got;
        return;
    }
    // fallback: 8-pass radix select over the 64-bit keys
    Scratch s_state(st, sizeof(SelState) + 256 * sizeof(uint32_t) + 16);
    SelState* sstate = s_state.as<SelState>();
    uint32_t* hist8 = reinterpret_cast<uint32_t*>(sstate + 1);
    DL_CUDA(cudaMemsetAsync(hist8, 0, 256 * sizeof(uint32_t), st));
    DL_LAUNCH(k_sel_init, 1, 1, 0, st, sstate, n_s);
    for (int pass = 0; pass < 8; ++pass) {
        const int shift = 56 - 8 * pass;
        DL_LAUNCH(k_sel_hist, g, 256, 0, st, salt, n_global, shift, sstate, hist8);
        DL_LAUNCH(k_sel_pick, 1, 256, 0, st, shift, sstate, hist8);
    }
    Scratch s_cnt(st, sizeof(unsigned long long));
    DL_CUDA(cudaMemsetAsync(s_cnt.p, 0, sizeof(unsigned long long), st));
    DL_LAUNCH(k_sel_collect, grid_for(n_range, 256, 148 * 8), 256, 0, st, salt, id_lo, n_range, sstate, d_out_local,
              s_cnt.as<unsigned long long>());
    DL_LAUNCH(k_sel_ties, 1, 1, 0, st, salt, id_lo, n_range, n_global, sstate, d_out_local,
              s_cnt.as<unsigned long long>());
    *n_out_host = (int64_t)d2h(s_cnt.as<unsigned long long>(), st);
}

void breakpoints_from_projections(const float* d_Ps, int64_t m, int LK, int N_r, float* d_B, cudaStream_t st) {
    Scratch keys(st, sizeof(uint32_t) * (size_t)(2 * m * LK));
    uint32_t* k0 = keys.as<uint32_t>();
    uint32_t* k1 = k0 + m * LK;
    DL_LAUNCH(k_transpose_keys, grid_for(m * LK, 256), 256, 0, st, d_Ps, m, LK, k0);
    bool flip = radix_sort_batched(k0, nullptr, k1, nullptr, m, LK, 32, st);
    DL_LAUNCH(k_bp_gather, grid_for((int64_t)LK * (N_r + 1), 256), 256, 0, st, flip ? k1 : k0, m, LK, N_r, d_B);
}

static void encode_all(const Index& ix, const float* d_P, int64_t m, uint8_t* d_EP, cudaStream_t st) {
    const size_t smem = sizeof(float) * (size_t)ix.LK * ix.N_r;
    ensure_dyn_smem_fn(k_encode, smem);
    DL_LAUNCH(k_encode, grid_for(m * ix.LK / 4, 256, 148 * 4), 256, smem, st, d_P, m, ix.LK, ix.N_r,
              ix.B.as<float>(), d_EP);
}

// B5 + B6 for all L trees at once, from codes EP[n][LK] (data order).  Returns false if the
// leaf list overflowed its capacity (the caller retries with a larger factor).
static bool build_trees_try(Index& ix, const uint8_t* d_EP, int64_t leaf_factor, cudaStream_t st,
                            const int* d_flag = nullptr, int* h_flag = nullptr, uint32_t* d_fkey = nullptr) {
    Trace tr("trees");
    const int64_t n = ix.n, L = ix.L, total = n * L;
    const int K = ix.K, nb = ix.nb, LK = ix.LK, max_size = ix.max_size;
    DL_REQUIRE(total < (int64_t)0xFFFFFFFF, "L*n must be < 2^32");

    ix.perm.alloc(sizeof(uint32_t) * (size_t)total, st);
    Scratch s_sort(st, sizeof(uint32_t) * (size_t)((d_fkey ? 2 : 3) * total));
    uint32_t* keys0 = d_fkey ? d_fkey : s_sort.as<uint32_t>() + 2 * total;
    uint32_t* keys1 = s_sort.as<uint32_t>();
    uint32_t* vals1 = keys1 + total;
    uint32_t* perm = ix.perm.as<uint32_t>();

    // B5: first-layer keys (from the projection epilogue, or from the codes), stable (key, id)
    // sort per tree
    // (the values start as the ids 0..n-1 of every tree: the sort's first pass generates them)
    if (!d_fkey)
        DL_LAUNCH(k_first_key, grid_for(total, 256), 256, 0, st, d_EP, n, (int)L, K, nb, keys0, perm);
    bool flip = radix_sort_batched(keys0, perm, keys1, vals1, n, L, K, st, true);
    const uint32_t* skeys = flip ? keys1 : keys0;
    if (flip) DL_CUDA(cudaMemcpyAsync(perm, vals1, sizeof(uint32_t) * total, cudaMemcpyDeviceToDevice, st));

    // first-layer segments
    Scratch s_seg(st, sizeof(uint32_t) * (size_t)(2 * total + 8));
    uint32_t* flags = s_seg.as<uint32_t>();
    uint32_t* idx = flags + total;
    uint32_t* counters = idx + total;  // [0]=nseg [1]=n_active [2]=n_next [3]=n_leaves [4]=total_chunks [5]=n_local [6]=n_local2
    DL_CUDA(cudaMemsetAsync(counters, 0, 8 * sizeof(uint32_t), st));
    DL_LAUNCH(k_seg_flags, grid_for(total, 256), 256, 0, st, skeys, n, total, flags);
    exclusive_scan_u32(flags, idx, total, counters + 0, st);
    // the segment count stays on the device: first-layer nodes of one tree <= min(n, 2^K)
    const int64_t nseg_ub = std::min<int64_t>(total, K >= 40 ? total : L * ((int64_t)1 << std::min(K, 39)));
    Scratch s_starts(st, sizeof(uint32_t) * (size_t)std::max<int64_t>(nseg_ub, 1));
    DL_LAUNCH(k_seg_write, grid_for(total, 256), 256, 0, st, flags, idx, total, s_starts.as<uint32_t>());

    // node storage: active nodes of one level are disjoint and hold > max_size points each;
    // leaves are disjoint and non-empty (<= total); start from a typical size and grow on overflow
    const int64_t cap_active = total / std::max(1, max_size) + 1;
    const int64_t cap_leaves = std::min<int64_t>(total, nseg_ub + leaf_factor * (total / std::max(1, max_size)) + 1024);
    Scratch s_nodes(st, sizeof(Node) * (size_t)(3 * cap_active + cap_leaves));
    Node* act = s_nodes.as<Node>();
    Node* nxt = act + cap_active;
    Node* loc = nxt + cap_active;
    Node* leaves = loc + cap_active;
    uint32_t* n_act = counters + 1;
    uint32_t* n_nxt = counters + 2;
    uint32_t* n_leaves = counters + 3;
    uint32_t* total_ch = counters + 4;
    uint32_t* n_loc = counters + 5;
    // nodes of <= LM points finish in shared memory (k_local_finish); LM keeps the live
    // sub-nodes of one level within LF_MAXSEG and the positions within 16 bits
    const int lm_env = std::getenv("DETLSH_LOCAL_MAX") ? std::atoi(std::getenv("DETLSH_LOCAL_MAX")) : 3072;   // read per build
    // (scan flags of one thread fit 32 bits: LM <= 32 * 256; staged codes + indices fit shared memory)
    const int64_t lm_smem = (int64_t)(200 * 1024) / ((K <= 16 ? 16 : 32) + 11);
    const int LM = (int)std::min<int64_t>(std::min<int64_t>(std::min<int64_t>(lm_env, 8192), lm_smem),
                                          (int64_t)(LF_MAXSEG - 1) * (max_size + 1));
    // two local tiers: nodes of <= LM1 points in CTAs sized for LM1 (4 per SM), larger ones up to LM
    // in CTAs of 512 threads sized for LM (measured at configs[4]: one LM = 1536 tier 170.1 ms of
    // build, LM = 3072 in one tier 162.7 ms but slower at configs[1] / configs[3])
    const int LM1 = std::min(LM, 1536);
    uint32_t* n_loc2 = counters + 6;
    Sinks sk{act, n_act, (uint32_t)cap_active, loc, n_loc, (uint32_t)cap_active, LM > max_size ? LM : 0,
             leaves, n_leaves, (uint32_t)cap_leaves, n_loc2, LM1};
    DL_LAUNCH(k_init_nodes, grid_for(nseg_ub, 256), 256, 0, st, s_starts.as<uint32_t>(), counters + 0, total, K, nb,
              max_size, sk);
    s_starts.free_();

    tr.mark("first layer sort+segments", st);
    // B6: level loop
    Scratch s_level(st, sizeof(uint32_t) * (size_t)(4 * cap_active + 4));
    int* split = s_level.as<int>();
    uint32_t* nch = reinterpret_cast<uint32_t*>(split + cap_active);
    uint32_t* choff = nch + cap_active;
    uint32_t* zeros = choff + cap_active;
    Scratch s_tmp(st, sizeof(uint32_t) * (size_t)total);
    // chunks of one level <= total / PART_CHUNK + one partial chunk per active node
    const int64_t nc_ub = total / PART_CHUNK + cap_active + 1;
    Scratch s_zc(st, sizeof(uint32_t) * (size_t)nc_ub);
    int64_t na = d2h(n_act, st);
    int level = 0;
    while (na > 0) {
        DL_REQUIRE(++level < 4096, "tree build: too many split levels");
        DL_LAUNCH(k_choose_split, grid_for(na * 32, 256), 256, 0, st, act, n_act, perm, d_EP, n, LK, K, nb,
                  max_size, PART_CHUNK, split, nch);
        exclusive_scan_u32(nch, choff, na, total_ch, st);
        const int64_t nc = std::min<int64_t>(nc_ub, total / PART_CHUNK + na + 1);   // grid bound; *total_ch exact
        {
            DL_LAUNCH(k_part_count, (unsigned)nc, PART_THREADS, 0, st, act, split, choff, n_act, total_ch, perm, d_EP,
                      n, LK, K, nb, s_zc.as<uint32_t>());
            DL_LAUNCH(k_part_offsets, grid_for(na, 256), 256, 0, st, choff, nch, n_act, s_zc.as<uint32_t>(), zeros);
            DL_LAUNCH(k_part_scatter, (unsigned)nc, PART_THREADS, 0, st, act, split, choff, n_act, total_ch,
                      s_zc.as<uint32_t>(), zeros, perm, d_EP, n, LK, K, nb, s_tmp.as<uint32_t>());
            DL_LAUNCH(k_part_copy, (unsigned)nc, PART_THREADS, 0, st, act, choff, n_act, total_ch, s_tmp.as<uint32_t>(),
                      perm);
        }
        DL_CUDA(cudaMemsetAsync(n_nxt, 0, sizeof(uint32_t), st));
        sk.active = nxt;
        sk.n_active = n_nxt;
        DL_LAUNCH(k_make_children, grid_for(na, 256), 256, 0, st, act, n_act, split, zeros, K, nb, max_size, sk);
        std::swap(act, nxt);
        std::swap(n_act, n_nxt);
        na = d2h(n_act, st);
        DL_REQUIRE(na <= cap_active, "tree build: active-node capacity exceeded");
    }
    if (sk.local_max > 0) {
        int dev = 0, nsm = 148;
        DL_CUDA(cudaGetDevice(&dev));
        DL_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        const int lf_nt = std::getenv("DETLSH_LF_THREADS") ? std::atoi(std::getenv("DETLSH_LF_THREADS")) : 0;
        for (int tier = 0; tier < 2; ++tier) {
            const int lm_t = tier == 0 ? LM1 : LM;
            if (tier == 1 && LM <= LM1) break;
            const size_t lsm = local_finish_smem(lm_t, K);
            const int LF_THREADS = lf_nt == 256 ? 256 : lf_nt == 512 ? 512 : (tier == 0 ? 256 : 512);
            auto k_local_finish_sel = K <= 16 ? (LF_THREADS == 256 ? k_local_finish<16, 256> : k_local_finish<16, 512>)
                                              : (LF_THREADS == 256 ? k_local_finish<32, 256> : k_local_finish<32, 512>);
            ensure_dyn_smem_fn(k_local_finish_sel, lsm);
            int per_sm = 1;
            DL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_local_finish_sel, LF_THREADS, lsm));
            DL_LAUNCH(k_local_finish_sel, nsm * std::max(1, per_sm), LF_THREADS, lsm, st, loc, tier == 0 ? n_loc : n_loc2,
                      lm_t, perm, d_EP, n, LK, K, nb, max_size, leaves, n_leaves, (uint32_t)cap_leaves,
                      tier == 0 ? (int64_t)0 : cap_active);
        }
    }
    s_tmp.free_();
    s_zc.free_();
    s_level.free_();
    tr.mark("split levels", st);

    // leaves in canonical order = ascending start position (DFS, 0-child first, keys ascending)
    const int64_t nl = d2h(n_leaves, st);
    if (nl > cap_leaves) return false;
    const int64_t nw = ceil_div(total, 32);
    Scratch s_lsort(st, sizeof(uint32_t) * (size_t)(nl + 3 * nw));
    uint32_t* order = s_lsort.as<uint32_t>();
    uint32_t* bitmap = order + nl;
    uint32_t* wcnt = bitmap + nw;
    uint32_t* wpre = wcnt + nw;
    DL_CUDA(cudaMemsetAsync(bitmap, 0, sizeof(uint32_t) * (size_t)nw, st));
    DL_LAUNCH(k_leaf_starts, grid_for(nl, 256), 256, 0, st, leaves, n_leaves, bitmap);
    DL_LAUNCH(k_word_popc, grid_for(nw, 256), 256, 0, st, bitmap, nw, wcnt);
    exclusive_scan_u32(wcnt, wpre, nw, nullptr, st);
    DL_LAUNCH(k_leaf_rank, grid_for(nl, 256), 256, 0, st, leaves, n_leaves, bitmap, wpre, order);
    ix.leaf_off.alloc(sizeof(uint32_t) * (size_t)(nl + 1), st);
    ix.leaf_lo.alloc((size_t)nl * K, st);
    ix.leaf_hi.alloc((size_t)nl * K, st);
    ix.leaf_bits.alloc((size_t)nl * K, st);
    DL_LAUNCH(k_leaf_finalize, grid_for(nl, 256), 256, 0, st, leaves, order, nl, perm, d_EP, n, LK, K, nb,
              ix.leaf_off.as<uint32_t>(), ix.leaf_lo.as<uint8_t>(), ix.leaf_hi.as<uint8_t>(),
              ix.leaf_bits.as<uint8_t>(), total);
    // per tree: first leaf (k_tree_begin) and first tile (k_tree_tiles), read back together with
    // the caller's flag in the single host round trip at the end
    Scratch s_begin(st, sizeof(unsigned long long) * (size_t)(2 * (L + 1)) + 16);
    unsigned long long* d_lbeg = s_begin.as<unsigned long long>();
    unsigned long long* d_tbeg = d_lbeg + (L + 1);
    DL_LAUNCH(k_tree_begin, 1, 64, 0, st, ix.leaf_off.as<uint32_t>(), nl, n, (int)L, d_lbeg);
    ix.tcodes.alloc((size_t)total * K, st);
    // DETLSH_LEAF_MORTON: 1 always, 0 never, default when leaves are large (first-layer cells of
    // >= 64 points on average: configs[3], configs[4]; at configs[1] the ~19-point leaves have 2-3
    // sub-boxes, and the sort cost 0.23 ms of build for 0.03 ms of query)
    static const int morton_env = std::getenv("DETLSH_LEAF_MORTON") ? std::atoi(std::getenv("DETLSH_LEAF_MORTON")) : -1;
    static const int fused_env = std::getenv("DETLSH_LEAF_FUSED") ? std::atoi(std::getenv("DETLSH_LEAF_FUSED")) : 1;
    const bool morton = K <= 32 && (morton_env == 1 || (morton_env < 0 && (n >> K) >= 64));
    ix.leaf_tbox.alloc((size_t)nl * 2 * K, st);
    if (morton && K == 16 && (LK & 15) == 0 && fused_env) {
        // gather + Morton order + sub-boxes + tight boxes in one pass (k_leaf_layout16)
        build_subboxes(ix, nl, st, false);
        DL_LAUNCH(k_leaf_layout16, grid_for(nl, LL_WARPS, 148 * 16), LL_WARPS * 32, 0, st, ix.leaf_off.as<uint32_t>(), nl,
                  ix.sb_off.as<uint32_t>(), perm, d_EP, n, LK, ix.tcodes.as<uint8_t>(), ix.sb_box.as<uint8_t>(),
                  ix.leaf_tbox.as<uint8_t>());
    } else {
        DL_LAUNCH(k_gather_tcodes, grid_for(total, 256), 256, 0, st, perm, d_EP, n, (int)L, K, ix.tcodes.as<uint8_t>());
        if (morton)
            DL_LAUNCH(k_leaf_morton, grid_for(nl, LM_WARPS, 148 * 16), LM_WARPS * 32, 0, st, ix.leaf_off.as<uint32_t>(), nl,
                      K, perm, ix.tcodes.as<uint8_t>());
        build_subboxes(ix, nl, st, true);
        DL_LAUNCH(k_leaf_tight_sb, grid_for(nl, 256), 256, 0, st, ix.sb_off.as<uint32_t>(), nl, K, ix.sb_box.as<uint8_t>(),
                  ix.leaf_tbox.as<uint8_t>());
    }
    tr.mark("leaf finalize+codes", st);
    // query tiles: runs of kTileLeaves leaves of one tree; the tile count stays on the device
    // (arrays sized by its bound: each tree adds at most one partial tile)
    {
        const int64_t nt_ub = nl / kTileLeaves + L + 1;
        Scratch s_tf(st, sizeof(uint32_t) * (size_t)(2 * nl + 2));
        uint32_t* tf = s_tf.as<uint32_t>();
        uint32_t* tidx = tf + nl;
        uint32_t* ntiles_d = tidx + nl;
        DL_LAUNCH(k_tile_flags, grid_for(nl, 256), 256, 0, st, ix.leaf_off.as<uint32_t>(), nl, n, kTileLeaves, d_lbeg, tf);
        exclusive_scan_u32(tf, tidx, nl, ntiles_d, st);
        ix.tile_leaf.alloc(sizeof(uint32_t) * (size_t)(nt_ub + 1), st);
        DL_LAUNCH(k_tile_write, grid_for(nl, 256), 256, 0, st, tf, tidx, nl, ix.tile_leaf.as<uint32_t>());
        DL_LAUNCH(k_tree_tiles, 1, 64, 0, st, tidx, d_lbeg, (int)L, ntiles_d, (uint32_t)nl, ix.tile_leaf.as<uint32_t>(),
                  d_tbeg);
        ix.tile_lo.alloc((size_t)nt_ub * K, st);
        ix.tile_hi.alloc((size_t)nt_ub * K, st);
        DL_LAUNCH(k_tile_boxes, grid_for(nt_ub * K, 256), 256, 0, st, ix.tile_leaf.as<uint32_t>(), ntiles_d, K,
                  ix.leaf_tbox.as<uint8_t>(), ix.leaf_tbox.as<uint8_t>() + K, ix.tile_lo.as<uint8_t>(), ix.tile_hi.as<uint8_t>());
        ix.point_tile_leaf.alloc(sizeof(uint16_t) * (size_t)total, st);
        DL_LAUNCH(k_point_tile_leaf, grid_for(nt_ub * 32, 256), 256, 0, st, ix.leaf_off.as<uint32_t>(),
                  ix.tile_leaf.as<uint32_t>(), ntiles_d, nl, ix.point_tile_leaf.as<uint16_t>());
        std::vector<unsigned long long> h(2 * (L + 1) + 1, 0);
        DL_CUDA(cudaMemcpyAsync(h.data(), d_lbeg, sizeof(unsigned long long) * 2 * (L + 1), cudaMemcpyDeviceToHost, st));
        if (d_flag) DL_CUDA(cudaMemcpyAsync(&h[2 * (L + 1)], d_flag, sizeof(int), cudaMemcpyDeviceToHost, st));
        DL_CUDA(cudaStreamSynchronize(st));
        ix.tree_leaf_begin.assign(h.begin(), h.begin() + (L + 1));
        ix.tree_leaf_begin[L] = nl;
        ix.tree_tile_begin.assign(h.begin() + (L + 1), h.begin() + 2 * (L + 1));
        if (h_flag) std::memcpy(h_flag, &h[2 * (L + 1)], sizeof(int));
    }
    tr.mark("tiles", st);
    return true;
}

// Sub-box offsets (k_sb_count + scan) and storage; boxes = true also fills them from tcodes.
void build_subboxes(Index& ix, int64_t nl, cudaStream_t st, bool boxes) {
    if (nl <= 0) return;
    ix.sb_off.alloc(sizeof(uint32_t) * (size_t)(nl + 1), st);
    Scratch s_cnt(st, sizeof(uint32_t) * (size_t)(nl + 1));
    DL_LAUNCH(k_sb_count, grid_for(nl, 256), 256, 0, st, ix.leaf_off.as<uint32_t>(), nl, s_cnt.as<uint32_t>());
    exclusive_scan_u32(s_cnt.as<uint32_t>(), ix.sb_off.as<uint32_t>(), nl, ix.sb_off.as<uint32_t>() + nl, st);
    const int64_t nsb_ub = (int64_t)ix.n * ix.L / kSubBox + nl;   // each leaf adds at most one partial run
    ix.sb_box.alloc((size_t)nsb_ub * 2 * ix.K, st);
    if (boxes)
        DL_LAUNCH(k_sb_boxes, grid_for(nsb_ub, 256), 256, 0, st, ix.leaf_off.as<uint32_t>(), ix.sb_off.as<uint32_t>(), nl,
                  ix.K, ix.tcodes.as<uint8_t>(), ix.sb_box.as<uint8_t>());
}

// d_flag (optional): a device int read back (into *h_flag) with the build's last host round trip
static void build_trees(Index& ix, const uint8_t* d_EP, cudaStream_t st, const int* d_flag = nullptr,
                        int* h_flag = nullptr, uint32_t* d_fkey = nullptr) {
    for (int64_t f = 4;; f *= 4) {
        // first-layer keys from the projection epilogue serve the first attempt only (its sort
        // overwrites them; a retry recomputes them from the codes)
        if (build_trees_try(ix, d_EP, f, st, d_flag, h_flag, f == 4 ? d_fkey : nullptr)) return;
        DL_REQUIRE(f < (int64_t)1 << 40, "tree build: leaf list overflow");
    }
}

bool project_encode_tc(const Index& ix, const float* d_X, int64_t ld, int64_t m, uint8_t* d_EP, int* d_nonfinite,
                       float* d_xnorm, float* d_P, cudaStream_t st, uint32_t* d_fkey);

void build_index(Index& ix, const float* d_data, int64_t data_ld, const float* bp_given, double sample_frac,
                 int proj_impl, cudaStream_t st) {
    Trace tr("build");
    const int64_t n = ix.n;
    // B0: hash family
    ix.A.alloc(sizeof(float) * (size_t)ix.LK * ix.ld, st);
    DL_LAUNCH(k_hash_family, grid_for((int64_t)ix.LK * ix.ld, 256), 256, 0, st, ix.seed, ix.LK, ix.d, ix.ld,
              ix.A.as<float>());
    Scratch s_flag(st, sizeof(int));
    DL_CUDA(cudaMemsetAsync(s_flag.p, 0, sizeof(int), st));
    // B1-B3: breakpoints
    ix.B.alloc(sizeof(float) * (size_t)ix.LK * (ix.N_r + 1), st);
    if (bp_given) {
        DL_CUDA(cudaMemcpyAsync(ix.B.p, bp_given, ix.B.bytes, cudaMemcpyDefault, st));
        ix.n_s = 0;
    } else {
        const int64_t n_s = detlsh_sample_size(n, ix.N_r, sample_frac);
        ix.sample.alloc(sizeof(uint32_t) * (size_t)n_s, st);
        int64_t got = 0;
        sample_ids_device(ix.seed, 0, n, n, n_s, ix.sample.as<uint32_t>(), &got, st);
        DL_REQUIRE(got == n_s, "sample selection returned the wrong count");
        ix.n_s = n_s;
        Scratch s_xs(st, sizeof(float) * (size_t)(n_s * data_ld));
        Scratch s_ps(st, sizeof(float) * (size_t)(n_s * ix.LK));
        DL_LAUNCH(k_gather_rows, grid_for(n_s * 32, 256), 256, 0, st, d_data, data_ld, ix.sample.as<uint32_t>(), n_s,
                  s_xs.as<float>());
        project_rows(ix, s_xs.as<float>(), data_ld, n_s, s_ps.as<float>(), proj_impl, s_flag.as<int>(), st);
        tr.mark("sample+sample projection", st);
        breakpoints_from_projections(s_ps.as<float>(), n_s, ix.LK, ix.N_r, ix.B.as<float>(), st);
    }
    tr.mark("breakpoints", st);
    // B2 + B4: project every row and encode -- fused in the tensor-core epilogue when the
    // shape fits, else projection (chunked so P stays bounded) + k_encode
    Scratch s_ep(st, (size_t)n * ix.LK);
    ix.xnorm.alloc(sizeof(float) * (size_t)n, st);     // ||x||^2 per row (tensor-core verification)
    if (ix.keep_proj) ix.proj.alloc(sizeof(float) * (size_t)n * ix.LK, st);   // EXACT mode: p' of every point
    // the tensor-core epilogue also writes each tree's first-layer keys (K = 16, N_r a power of two):
    // the tree build's sort starts from them instead of re-reading the codes (k_first_key)
    const bool fk_ok = proj_impl == 0 && ix.K == 16 && (ix.LK & 15) == 0 && (ix.N_r & (ix.N_r - 1)) == 0 &&
                       (int64_t)n * ix.L < (int64_t)0xFFFFFFFF;
    Scratch s_fkey(st, fk_ok ? sizeof(uint32_t) * (size_t)(n * ix.L) : 0);
    bool fk_written = false;
    if (proj_impl == 0 && project_encode_tc(ix, d_data, data_ld, n, s_ep.as<uint8_t>(), s_flag.as<int>(),
                                            ix.xnorm.as<float>(), ix.keep_proj ? ix.proj.as<float>() : nullptr, st,
                                            fk_ok ? s_fkey.as<uint32_t>() : nullptr)) {
        fk_written = fk_ok;
    } else {
        DL_LAUNCH(k_row_norms, grid_for(n * 32, 256), 256, 0, st, d_data, data_ld, n, ix.xnorm.as<float>());
        const int64_t chunk = std::min<int64_t>(n, std::max<int64_t>(1 << 16, (int64_t)(1ll << 30) / (4 * ix.LK)));
        Scratch s_p(st, sizeof(float) * (size_t)(chunk * ix.LK));
        for (int64_t r0 = 0; r0 < n; r0 += chunk) {
            const int64_t m = std::min(chunk, n - r0);
            project_rows(ix, d_data + r0 * data_ld, data_ld, m, s_p.as<float>(), proj_impl, s_flag.as<int>(), st);
            encode_all(ix, s_p.as<float>(), m, s_ep.as<uint8_t>() + r0 * ix.LK, st);
            if (ix.keep_proj)
                DL_CUDA(cudaMemcpyAsync(ix.proj.as<float>() + r0 * ix.LK, s_p.p, sizeof(float) * (size_t)(m * ix.LK),
                                        cudaMemcpyDeviceToDevice, st));
        }
    }
    tr.mark("project+encode", st);
    // B5 + B6; the non-finite flag of the projection is read with the trees' last round trip
    // (a NaN/Inf row makes the whole build fail -- after the trees, not before)
    int nonfinite = 0;
    build_trees(ix, s_ep.as<uint8_t>(), st, s_flag.as<int>(), &nonfinite, fk_written ? s_fkey.as<uint32_t>() : nullptr);
    DL_REQUIRE(!nonfinite, "data contains NaN or Inf");
    tr.mark("trees", st);
}

void build_trees_from_codes(Index& ix, const uint8_t* d_codes, cudaStream_t st) { build_trees(ix, d_codes, st); }

void build_index_hash_only(Index& ix, cudaStream_t st) {
    ix.A.alloc(sizeof(float) * (size_t)ix.LK * ix.ld, st);
    DL_LAUNCH(k_hash_family, grid_for((int64_t)ix.LK * ix.ld, 256), 256, 0, st, ix.seed, ix.LK, ix.d, ix.ld,
              ix.A.as<float>());
}

void gather_rows_strided(const float* d_src, int64_t src_ld, int d, const uint32_t* d_ids, int64_t m, float* d_dst,
                         int64_t dst_ld, cudaStream_t st) {
    if (m <= 0) return;
    DL_LAUNCH(k_gather_rows_strided, grid_for(m * 32, 256), 256, 0, st, d_src, src_ld, d, d_ids, m, d_dst, dst_ld);
}

}  // namespace detlsh
