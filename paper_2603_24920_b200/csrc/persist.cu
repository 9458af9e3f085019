// persist.cu -- index save/load: the device layout of an Index (index.cuh)
// written field by field to a little-endian binary file and read back into fresh device
// buffers.  Host-side marshalling only; no method arithmetic happens here.
//
// File: "DETLSH\0\1" | u32 version | header (fixed-width scalars) | the two host vectors
// (tree leaf / tile ranges) | device arrays, each as u64 byte count + bytes, in the order
// X, A, B, sample, perm, tcodes, leaf_off, leaf_lo, leaf_hi, leaf_bits, tile_leaf,
// point_tile_leaf, xnorm, proj (EXACT-mode projections; empty if not kept), tile_lo, tile_hi, leaf_tbox.  The data rows are always stored (a borrowed X is copied out), so
// a loaded index owns everything it needs.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "index.cuh"

namespace detlsh {
namespace {

constexpr char kMagic[8] = {'D', 'E', 'T', 'L', 'S', 'H', 0, 1};
constexpr uint32_t kVersion = 2;     // 2: tight leaf boxes interleaved (leaf_tbox)

struct Header {
    int64_t n, n_global, id_offset, n_s;
    int32_t d, ld, L, K, LK, N_r, nb, max_size;
    uint64_t seed;
    double eps;
    int32_t codes_only, ntl, ntt, pad;   // sizes of the two host vectors
};

struct File {
    FILE* f = nullptr;
    ~File() {
        if (f) std::fclose(f);
    }
};

void wr(FILE* f, const void* p, size_t b) {
    if (b && std::fwrite(p, 1, b, f) != b) throw Error(DETLSH_EINVAL, "write failed");
}
void rd(FILE* f, void* p, size_t b) {
    if (b && std::fread(p, 1, b, f) != b) throw Error(DETLSH_EINVAL, "truncated or corrupt index file");
}

// device buffer -> file (u64 size + bytes), staged through a host buffer in 64 MB chunks
void put_dev(FILE* f, const void* d, size_t b) {
    const uint64_t n = b;
    wr(f, &n, 8);
    std::vector<char> h(std::min<size_t>(b, (size_t)64 << 20));
    for (size_t o = 0; o < b; o += h.size()) {
        const size_t c = std::min(h.size(), b - o);
        DL_CUDA(cudaMemcpy(h.data(), static_cast<const char*>(d) + o, c, cudaMemcpyDeviceToHost));
        wr(f, h.data(), c);
    }
}
void get_dev(FILE* f, DevBuf& buf, size_t expect) {
    uint64_t n = 0;
    rd(f, &n, 8);
    if (n < expect) throw Error(DETLSH_EINVAL, "index file array size mismatch");
    buf.alloc((size_t)n, 0);
    std::vector<char> h(std::min<size_t>((size_t)n, (size_t)64 << 20));
    for (size_t o = 0; o < n; o += h.size()) {
        const size_t c = std::min(h.size(), (size_t)n - o);
        rd(f, h.data(), c);
        DL_CUDA(cudaMemcpy(static_cast<char*>(buf.p) + o, h.data(), c, cudaMemcpyHostToDevice));
    }
}

}  // namespace

void save_index(const Index& ix, const char* path) {
    DL_REQUIRE(path && *path, "path is empty");
    File fh;
    fh.f = std::fopen(path, "wb");
    DL_REQUIRE(fh.f, std::string("cannot open for writing: ") + path);
    DL_CUDA(cudaDeviceSynchronize());
    wr(fh.f, kMagic, 8);
    wr(fh.f, &kVersion, 4);
    Header h{};
    h.n = ix.n; h.n_global = ix.n_global; h.id_offset = ix.id_offset; h.n_s = ix.n_s;
    h.d = ix.d; h.ld = ix.ld; h.L = ix.L; h.K = ix.K; h.LK = ix.LK; h.N_r = ix.N_r; h.nb = ix.nb;
    h.max_size = ix.max_size; h.seed = ix.seed; h.eps = ix.eps; h.codes_only = ix.codes_only ? 1 : 0;
    h.ntl = (int32_t)ix.tree_leaf_begin.size();
    h.ntt = (int32_t)ix.tree_tile_begin.size();
    wr(fh.f, &h, sizeof(h));
    wr(fh.f, ix.tree_leaf_begin.data(), sizeof(int64_t) * ix.tree_leaf_begin.size());
    wr(fh.f, ix.tree_tile_begin.data(), sizeof(int64_t) * ix.tree_tile_begin.size());
    const size_t xbytes = ix.codes_only ? 0 : sizeof(float) * (size_t)ix.n * ix.ld;
    put_dev(fh.f, ix.Xp, xbytes);
    const DevBuf* arr[] = {&ix.A, &ix.B, &ix.sample, &ix.perm, &ix.tcodes, &ix.leaf_off, &ix.leaf_lo,
                           &ix.leaf_hi, &ix.leaf_bits, &ix.tile_leaf, &ix.point_tile_leaf, &ix.xnorm, &ix.proj, &ix.tile_lo, &ix.tile_hi, &ix.leaf_tbox};
    for (const DevBuf* b : arr) put_dev(fh.f, b->p, b->bytes);
    if (std::fflush(fh.f) != 0) throw Error(DETLSH_EINVAL, "write failed");
}

Index* load_index(const char* path) {
    DL_REQUIRE(path && *path, "path is empty");
    File fh;
    fh.f = std::fopen(path, "rb");
    DL_REQUIRE(fh.f, std::string("cannot open: ") + path);
    char magic[8];
    uint32_t ver = 0;
    rd(fh.f, magic, 8);
    DL_REQUIRE(std::memcmp(magic, kMagic, 8) == 0, "not a DET-LSH index file");
    rd(fh.f, &ver, 4);
    DL_REQUIRE(ver == kVersion, "unsupported index file version");
    Header h{};
    rd(fh.f, &h, sizeof(h));
    DL_REQUIRE(h.n >= 1 && h.L >= 1 && h.K >= 1 && h.K <= 32 && h.LK == h.L * h.K && h.ntl == h.L + 1 &&
                   h.ntt == h.L + 1 && h.ld >= h.d && h.d >= 1,
               "corrupt index header");
    auto ix = std::make_unique<Index>();
    ix->n = h.n; ix->n_global = h.n_global; ix->id_offset = h.id_offset; ix->n_s = h.n_s;
    ix->d = h.d; ix->ld = h.ld; ix->L = h.L; ix->K = h.K; ix->LK = h.LK; ix->N_r = h.N_r; ix->nb = h.nb;
    ix->max_size = h.max_size; ix->seed = h.seed; ix->eps = h.eps; ix->codes_only = h.codes_only != 0;
    ix->tree_leaf_begin.resize(h.ntl);
    ix->tree_tile_begin.resize(h.ntt);
    rd(fh.f, ix->tree_leaf_begin.data(), sizeof(int64_t) * h.ntl);
    rd(fh.f, ix->tree_tile_begin.data(), sizeof(int64_t) * h.ntt);
    const int64_t nl = ix->tree_leaf_begin.back(), nt = ix->tree_tile_begin.back();
    const size_t xbytes = ix->codes_only ? 0 : sizeof(float) * (size_t)h.n * h.ld;
    get_dev(fh.f, ix->X, xbytes);
    ix->Xp = ix->X.as<float>();
    const size_t nLK = (size_t)h.LK;
    get_dev(fh.f, ix->A, ix->codes_only ? 0 : sizeof(float) * nLK * h.ld);
    get_dev(fh.f, ix->B, ix->codes_only ? 0 : sizeof(float) * nLK * (h.N_r + 1));
    get_dev(fh.f, ix->sample, 0);
    get_dev(fh.f, ix->perm, sizeof(uint32_t) * (size_t)h.n * h.L);
    get_dev(fh.f, ix->tcodes, (size_t)h.n * h.L * h.K);
    get_dev(fh.f, ix->leaf_off, sizeof(uint32_t) * (size_t)(nl + 1));
    get_dev(fh.f, ix->leaf_lo, (size_t)nl * h.K);
    get_dev(fh.f, ix->leaf_hi, (size_t)nl * h.K);
    get_dev(fh.f, ix->leaf_bits, (size_t)nl * h.K);
    get_dev(fh.f, ix->tile_leaf, sizeof(uint32_t) * (size_t)(nt + 1));
    get_dev(fh.f, ix->point_tile_leaf, sizeof(uint16_t) * (size_t)h.n * h.L);
    get_dev(fh.f, ix->xnorm, ix->codes_only ? 0 : sizeof(float) * (size_t)h.n);
    get_dev(fh.f, ix->proj, 0);                        // empty unless built with keep_projections
    ix->keep_proj = ix->proj.p != nullptr;
    get_dev(fh.f, ix->tile_lo, (size_t)nt * h.K);
    get_dev(fh.f, ix->tile_hi, (size_t)nt * h.K);
    get_dev(fh.f, ix->leaf_tbox, (size_t)nl * 2 * h.K);
    build_subboxes(*ix, nl, 0);                        // derived from tcodes + leaf_off (not stored)
    DL_CUDA(cudaDeviceSynchronize());
    return ix.release();
}

}  // namespace detlsh
