// merge.cu -- C2 of the point-sharded query: the G per-shard top-k lists of
// each query merged into the k best by (dist, id) (AMB-21), on the device.
//
// Each list is sorted ascending by (dist, id) with empty slots (id < 0) at its tail (what
// detlsh_query writes).  Merge by ranking: an element's place in the merged order is its index
// in its own list plus, for every other list, the number of that list's elements that order
// before it (binary search; equal keys -- only possible for repeated ids -- order by list
// index).  Every element of rank < k writes itself; no sort, no atomics, one block per query.
#include <cmath>

#include "index.cuh"

namespace detlsh {
namespace {

struct MKey {
    float d;
    int64_t id;
};

__device__ __forceinline__ MKey mkey_at(const int64_t* ids, const float* dists, int64_t o) {
    const int64_t id = ids[o];
    return id < 0 ? MKey{INFINITY, INT64_MAX} : MKey{dists[o], id};
}
__device__ __forceinline__ bool mk_less(const MKey& a, const MKey& b) {
    return a.d < b.d || (a.d == b.d && a.id < b.id);
}

// Number of elements of list [base, base + k) ordering before x (strictly, or also equal
// when `or_equal`: lists with a smaller index than x's own).
__device__ int mrank(const int64_t* ids, const float* dists, int64_t base, int k, const MKey& x, bool or_equal) {
    int lo = 0, hi = k;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const MKey y = mkey_at(ids, dists, base + mid);
        const bool before = or_equal ? !mk_less(x, y) : mk_less(y, x);
        if (before) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(256) k_merge_topk(const int64_t* __restrict__ ids, const float* __restrict__ dists,
                                                    int G, int64_t nq, int k, int64_t* __restrict__ out_ids,
                                                    float* __restrict__ out_dists) {
    pdl_wait();
    for (int64_t q = blockIdx.x; q < nq; q += gridDim.x) {
        for (int e = threadIdx.x; e < k; e += blockDim.x) {
            out_ids[q * k + e] = -1;
            out_dists[q * k + e] = INFINITY;
        }
        __syncthreads();
        for (int64_t e = threadIdx.x; e < (int64_t)G * k; e += blockDim.x) {
            const int g = (int)(e / k), i = (int)(e % k);
            const int64_t o = ((int64_t)g * nq + q) * k + i;
            if (ids[o] < 0) continue;
            const MKey x = mkey_at(ids, dists, o);
            int64_t rank = i;
            for (int h = 0; h < G && rank < k; ++h)
                if (h != g) rank += mrank(ids, dists, ((int64_t)h * nq + q) * k, k, x, h < g);
            if (rank < k) {
                out_ids[q * k + rank] = x.id;
                out_dists[q * k + rank] = x.d;
            }
        }
        __syncthreads();
    }
}

}  // namespace

void merge_topk_device(const int64_t* d_ids, const float* d_dists, int G, int64_t nq, int k, int64_t* d_out_ids,
                       float* d_out_dists, cudaStream_t st) {
    if (nq <= 0) return;
    const unsigned grid = (unsigned)std::min<int64_t>(nq, 148 * 16);
    DL_LAUNCH(k_merge_topk, grid, 256, 0, st, d_ids, d_dists, G, nq, k, d_out_ids, d_out_dists);
}

}  // namespace detlsh
