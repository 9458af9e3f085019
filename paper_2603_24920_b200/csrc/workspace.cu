// workspace.cu -- grow-only per-(device, stream) scratch arenas behind Scratch (common.cuh).
//
// Measured on B200 (configs[1], 1000 queries): with per-call cudaMallocAsync scratch the
// query wall time varied 19 -> 80 ms from call to call (stalls of 9-60 ms in the stream
// while the driver (re)mapped ~2 GB of pool memory); the kernels themselves are constant.
// The arena keeps the memory mapped across calls.
#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"
#include "index.cuh"

namespace detlsh {
namespace {

struct Arena {
    std::mutex mu;
    char* base = nullptr;
    size_t cap = 0;
    size_t used = 0;      // bytes bumped in the current call
    size_t vused = 0;     // bytes the call would have bumped had the arena been large enough
    size_t need = 0;      // high-water mark of vused in the current call
    cudaStream_t st = nullptr;
};

std::mutex g_mu;
std::map<std::pair<int, cudaStream_t>, Arena*> g_arenas;
thread_local Arena* t_ws = nullptr;

constexpr size_t kAlign = 256;
// Arenas are kept mapped only up to this size: a call that needs more (very large query
// batches) takes its scratch stream-ordered from the default pool instead, which returns it
// after the call, so a huge arena never starves later index builds.
constexpr size_t kArenaMax = (size_t)16 << 30;
inline size_t align_up(size_t b) { return (b + kAlign - 1) / kAlign * kAlign; }

}  // namespace

void* ws_alloc(size_t bytes, cudaStream_t st, bool* from_arena) {
    Arena* a = t_ws;
    const size_t b = align_up(bytes);
    if (a && a->st == st) {
        a->vused += b;
        if (a->vused > a->need) a->need = a->vused;
        if (a->used + b <= a->cap && a->used == a->vused - b) {
            void* p = a->base + a->used;
            a->used += b;
            *from_arena = true;
            return p;
        }
    }
    void* p = nullptr;
    DL_CUDA(cudaMallocFromPoolAsync(&p, bytes, scratch_pool(), st));
    *from_arena = false;
    return p;
}

cudaMemPool_t scratch_pool() {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    int dev = 0;
    DL_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (!pools[dev]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        DL_CUDA(cudaMemPoolCreate(&pools[dev], &props));
        uint64_t thr = UINT64_MAX;    // no unmap/remap between calls
        DL_CUDA(cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr));
    }
    return pools[dev];
}

void ensure_dyn_smem(const void* fn, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> done;
    int dev = 0;
    DL_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    size_t& have = done[{dev, fn}];
    if (have >= bytes) return;
    DL_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    have = bytes;
}

WorkspaceScope::WorkspaceScope(cudaStream_t st) {
    if (t_ws) return;   // nested entry point: the outer scope owns the arena
    int dev = 0;
    DL_CUDA(cudaGetDevice(&dev));
    Arena* a;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        Arena*& slot = g_arenas[{dev, st}];
        if (!slot) slot = new Arena();
        a = slot;
    }
    a->mu.lock();
    a->st = st;
    a->used = a->vused = a->need = 0;
    t_ws = a;
    impl = a;
    owner = true;
}

WorkspaceScope::~WorkspaceScope() {
    if (!owner) return;
    Arena* a = static_cast<Arena*>(impl);
    t_ws = nullptr;
    if (a->need > a->cap && a->need <= kArenaMax) {
        // regrow to the call's high-water mark (+25%); in-flight work may still use the old block
        cudaStreamSynchronize(a->st);
        if (a->base) cudaFree(a->base);
        a->base = nullptr;
        a->cap = 0;
        const size_t want = align_up(a->need + a->need / 4);
        void* p = nullptr;
        if (cudaMalloc(&p, want) == cudaSuccess) {
            a->base = static_cast<char*>(p);
            a->cap = want;
        } else {
            cudaGetLastError();   // stay on the fallback path; the call already succeeded
        }
    }
    a->mu.unlock();
}

void ws_release_all() {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto& kv : g_arenas) {
        Arena* a = kv.second;
        std::lock_guard<std::mutex> al(a->mu);
        if (a->base) {
            int cur = 0;
            cudaGetDevice(&cur);
            cudaSetDevice(kv.first.first);
            cudaStreamSynchronize(a->st);
            cudaFree(a->base);
            cudaSetDevice(cur);
        }
        a->base = nullptr;
        a->cap = 0;
    }
    // return the pools' unused reserved memory to the device (current device)
    cudaDeviceSynchronize();
    cudaMemPoolTrimTo(scratch_pool(), 0);
    cudaMemPoolTrimTo(index_pool(), 0);
}

int64_t ws_bytes_held() {
    std::lock_guard<std::mutex> lk(g_mu);
    int64_t s = 0;
    for (auto& kv : g_arenas) s += (int64_t)kv.second->cap;
    return s;
}

}  // namespace detlsh

extern "C" {
void detlsh_release_workspace(void) { detlsh::ws_release_all(); }
int64_t detlsh_workspace_bytes(void) { return detlsh::ws_bytes_held(); }
}
