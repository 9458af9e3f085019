// index.cuh -- device layout of a DET-LSH index.
#pragma once

#include <atomic>
#include <vector>

#include "common.cuh"

namespace detlsh {

// Pool for index-owned (long-lived) buffers, separate from the scratch pool (workspace.cu), so
// the two lifetimes do not fragment each other (api.cu).  The query batch budget subtracts
// what this pool has reserved since its free-memory snapshot (query.cu).
cudaMemPool_t index_pool();
// Bytes held by live index buffers (all devices), kept by DevBuf.
extern std::atomic<int64_t> g_index_bytes;

// Index-owned device memory, stream-ordered from index_pool() (no device-wide sync on
// allocate/free); freed on the legacy default stream.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { reset(); }
    void alloc(size_t b, cudaStream_t st = 0) {
        reset();
        if (b) DL_CUDA(cudaMallocFromPoolAsync(&p, b, index_pool(), st));
        bytes = b;
        g_index_bytes += (int64_t)b;
    }
    void reset() {
        if (p) cudaFreeAsync(p, 0);
        g_index_bytes -= (int64_t)bytes;
        p = nullptr;
        bytes = 0;
    }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

constexpr int kTileLeaves = 32;     // leaves per query tile (one warp of the range filter)
constexpr int kSubBox = 8;          // points per leaf sub-box (consecutive in leaf order)

struct Index {
    // shape / parameters
    int64_t n = 0;          // points in this index (shard)
    int64_t n_global = 0;
    int64_t id_offset = 0;
    int32_t d = 0, ld = 0;  // dimension, padded row stride (floats, multiple of 8)
    int32_t L = 0, K = 0, LK = 0, N_r = 0, nb = 0;
    int32_t max_size = 128;
    uint64_t seed = 0;
    double eps = 0;         // sqrt(chi2_{e^{-1/L}}(K)) (Eq. 2)
    int64_t n_s = 0;        // sample size used for the breakpoints (0 if given)
    bool codes_only = false;

    // device arrays
    DevBuf X;               // [n][ld] fp32 (owned copy) -- unless borrowed
    const float* Xp = nullptr;  // points to X or the borrowed buffer
    DevBuf A;               // [LK][d] fp32 hash family (TF32-exact values, AMB-1)
    DevBuf B;               // [LK][N_r+1] fp32 breakpoints
    DevBuf sample;          // [n_s] u32 sample ids (local), unordered
    DevBuf perm;            // [L*n] u32: tree t's point ids in leaf order at [t*n, (t+1)*n)
    DevBuf tcodes;          // [L*n][K] u8: codes of perm in leaf order (per tree)
    DevBuf leaf_off;        // [nl_total+1] u32 global positions into perm (tree-major)
    DevBuf leaf_lo, leaf_hi;// [nl_total][K] u8 symbol range of each leaf box
    DevBuf leaf_bits;       // [nl_total][K] u8 bits per dim of each leaf
    std::vector<int64_t> tree_leaf_begin;  // [L+1] leaf index range of each tree (host copy)
    DevBuf tile_leaf;       // [ntiles+1] first leaf of each query tile (tree-major; see build.cu)
    std::vector<int64_t> tree_tile_begin;  // [L+1] tile index range of each tree (host copy)
    DevBuf point_tile_leaf; // [L*n] u16: leaf of each point (tree order) within its tile (< 32)
    DevBuf leaf_tbox;           // [nl_total][2K] u8 tight box: min code (K bytes) then max code (K bytes)
                                // of the leaf's points -- lo and hi in one row (one 32 B sector at K = 16)
    DevBuf tile_lo, tile_hi;// [ntiles][K] u8 bounding box of each tile's tight leaf boxes
    DevBuf sb_off;          // [nl_total+1] u32 first sub-box of each leaf (sub-box = kSubBox consecutive points)
    DevBuf sb_box;          // [nsb][2K] u8 tight box (lo | hi) of each sub-box (the pair kernel's second-level bound)
    DevBuf xnorm;           // [n] fp32 ||x||^2 of every row (tensor-core verification, verify_tc.cu)
    bool keep_proj = false; // build option: keep the projections (EXACT mode)
    DevBuf proj;            // [n][LK] fp32 projections p' in data order (EXACT mode only)

    int64_t nl_total() const { return tree_leaf_begin.empty() ? 0 : tree_leaf_begin.back(); }
};

// build.cu
void build_index(Index& ix, const float* d_data, int64_t data_ld, const float* bp_given,
                 double sample_frac, int proj_impl, cudaStream_t st);
void build_trees_from_codes(Index& ix, const uint8_t* d_codes, cudaStream_t st);
// Sub-box tight boxes of the nl leaves (derived from tcodes + leaf_off; also rebuilt on load).
void build_subboxes(Index& ix, int64_t nl, cudaStream_t st, bool boxes = true);
void build_index_hash_only(Index& ix, cudaStream_t st);
void gather_rows_strided(const float* d_src, int64_t src_ld, int d, const uint32_t* d_ids, int64_t m, float* d_dst,
                         int64_t dst_ld, cudaStream_t st);
void project_rows(const Index& ix, const float* d_X, int64_t ld, int64_t m, float* d_P, int proj_impl,
                  int* d_nonfinite, cudaStream_t st);
void sample_ids_device(uint64_t seed, int64_t id_lo, int64_t n_range, int64_t n_global, int64_t n_s,
                       uint32_t* d_out_local, int64_t* n_out_host, cudaStream_t st);
void breakpoints_from_projections(const float* d_Ps, int64_t m, int LK, int N_r, float* d_B,
                                  cudaStream_t st);

// merge.cu: C2 merge of G per-shard top-k lists [G][nq][k] (device pointers)
void merge_topk_device(const int64_t* d_ids, const float* d_dists, int G, int64_t nq, int k, int64_t* d_out_ids,
                       float* d_out_dists, cudaStream_t st);

// persist.cu
void save_index(const Index& ix, const char* path);
Index* load_index(const char* path);

// query.cu
struct QueryArgs {
    int64_t nq;
    int k;
    double c, r_min, beta;
    int mode;
    int query_batch;
    int64_t mem_budget;
    int proj_impl;
    int verify_impl;
    int lb_order = 0;           // Sec. 6.2.2(2): leaves in (LB, leaf) order, budget checked per leaf
    int max_rounds = 64;        // AMB-20 round cap; 1 for (r,c)-ANN (Alg. 4)
    bool null_on_cap = false;   // (r,c)-ANN: return nothing when the single pass neither hit the
                                // budget nor found a point within c r
    uint32_t* export_S = nullptr;   // test export: device [nq][ceil(n/32)] copy of each query's final
                                    // candidate-set bitmap S (bit p%32 of word p/32 = local id p)
};
void query_index(const Index& ix, const float* d_Q, int64_t q_ld, const QueryArgs& a, int64_t* d_ids,
                 float* d_dists, detlsh_query_stats* d_stats, cudaStream_t st);

void estimate_rstar(const Index& ix, const float* d_Q, int64_t q_ld, int64_t ns, int k, double beta, int proj_impl,
                    double* h_rstar, cudaStream_t st);

// host_math.cpp
double chi2_upper_quantile(double alpha, int K);
double chi2_survival(double y, int K);

}  // namespace detlsh
