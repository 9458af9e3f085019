// common.cuh -- shared helpers of the DET-LSH sm_100a library (product code).
// Nothing here is shared with oracle/ (the test oracle has its own C code).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/detlsh.h"

namespace detlsh {

// ------------------------------------------------------------------ errors
struct Error : std::runtime_error {
    detlsh_status code;
    Error(detlsh_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define DL_CUDA(expr)                                                                          \
    do {                                                                                       \
        cudaError_t _e = (expr);                                                               \
        if (_e != cudaSuccess) {                                                               \
            throw ::detlsh::Error(_e == cudaErrorMemoryAllocation ? DETLSH_ENOMEM : DETLSH_ECUDA, \
                                  std::string(#expr) + ": " + cudaGetErrorString(_e) + " (" +    \
                                      __FILE__ + ":" + std::to_string(__LINE__) + ")");         \
        }                                                                                      \
    } while (0)

#define DL_REQUIRE(cond, msg)                                                                  \
    do {                                                                                       \
        if (!(cond)) throw ::detlsh::Error(DETLSH_EINVAL, msg);                                \
    } while (0)

extern std::atomic<int64_t> g_launches;
extern std::atomic<int> g_profile;
// Kernel timing (bench.py's live roofline): CUDA events recorded on the launch stream
// around each launch while profiling is enabled (detlsh_profile_enable).
void profile_begin(cudaStream_t st, const char* name, int* slot);
void profile_end(cudaStream_t st, int slot);

// Every kernel launch goes through this macro: counts launches (the evidence counter
// behind detlsh_launch_count), optionally times it, and checks the launch error.
// Every launch allows programmatic dependent launch (PDL): the next kernel on the stream is
// launched while this one drains, and every kernel of the library begins with pdl_wait()
// (griddepcontrol.wait: returns once the preceding grid has completed and its memory is visible;
// a no-op for a launch without the attribute), so results are those of plain stream order and
// only the launch latency between dependent kernels overlaps.  DETLSH_PDL=0 turns it off.
bool pdl_enabled();
#define DL_LAUNCH(kernel, grid, block, smem, strm_, ...)                                         \
    do {                                                                                       \
        int _slot = -1;                                                                        \
        if (::detlsh::g_profile.load(std::memory_order_relaxed))                               \
            ::detlsh::profile_begin((strm_), #kernel, &_slot);                                \
        cudaLaunchConfig_t _cfg = {};                                                          \
        _cfg.gridDim = dim3(grid);                                                             \
        _cfg.blockDim = dim3(block);                                                           \
        _cfg.dynamicSmemBytes = (size_t)(smem);                                                \
        _cfg.stream = (strm_);                                                                  \
        cudaLaunchAttribute _attr[1];                                                          \
        _attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                      \
        _attr[0].val.programmaticStreamSerializationAllowed = 1;                               \
        _cfg.attrs = _attr;                                                                    \
        _cfg.numAttrs = ::detlsh::pdl_enabled() ? 1 : 0;                                       \
        DL_CUDA(cudaLaunchKernelEx(&_cfg, kernel, __VA_ARGS__));                               \
        ::detlsh::g_launches.fetch_add(1, std::memory_order_relaxed);                          \
        if (_slot >= 0) ::detlsh::profile_end((strm_), _slot);                                \
        DL_CUDA(cudaGetLastError());                                                           \
    } while (0)

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

#define COMMA ,

// ------------------------------------------------------------------ math helpers
__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// splitmix64 output for state x, and the keyed hash key(s, c) = splitmix64(s ^ splitmix64(c))
// that AMB-1 (hash family) and AMB-4 (sample) are defined with.
__host__ __device__ inline uint64_t mix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__host__ __device__ inline uint64_t keyed(uint64_t s, uint64_t c) { return mix64(s ^ mix64(c)); }

constexpr uint64_t kSampleSalt = 0x53414D504C45ULL;  // AMB-4

#if defined(__CUDACC__)
// Order-preserving fp32 <-> u32 maps (radix sorting floats).
__device__ inline uint32_t f2key(float f) {
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ inline float key2f(uint32_t k) {
    uint32_t u = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
    return __uint_as_float(u);
}

__device__ inline uint32_t lanemask_lt() {
    uint32_t m;
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}
#endif

// ------------------------------------------------------------------ primitives (radix.cu)
// Stable batched LSD radix sort: nseg independent segments of m u32 keys (segment s at
// keys + s*m), optional u32 values; sorts on key bits [0, bits).  Ping-pongs between
// (k0,v0) and (k1,v1); returns true if the result ended in (k1,v1).  vals_iota: the values
// start as 0..m-1 in every segment and v0 is not read.
bool radix_sort_batched(uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1, int64_t m,
                        int64_t nseg, int bits, cudaStream_t st, bool vals_iota = false);
// Exclusive scan of n u32 values; writes the total to *d_total (device) if non-null.
void exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* d_total,
                        cudaStream_t st);

// ------------------------------------------------------------------ host phase trace
// DETLSH_TRACE=1: print host wall time per phase (synchronising the stream at each mark).
struct Trace {
    bool on;
    double t0, last;
    const char* what;
    explicit Trace(const char* w);
    void mark(const char* phase, cudaStream_t st);
};

// ------------------------------------------------------------------ scratch allocation
// Per-call device scratch.  Inside a WorkspaceScope (every C-ABI entry point that launches
// work opens one for its stream) requests are bump-allocated from a grow-only arena owned by
// that (device, stream): no allocator traffic between calls, so a query or build never
// waits on the driver mapping memory.  A request the arena cannot hold yet is served by
// the scratch pool (stream-ordered) and counted; when the call ends the arena is regrown to the call's
// high-water mark, so from the second call of a given shape on everything is bumped.
// Outside a scope Scratch falls back to stream-ordered allocations from scratch_pool().
void* ws_alloc(size_t bytes, cudaStream_t st, bool* from_arena);

struct WorkspaceScope {
    explicit WorkspaceScope(cudaStream_t st);
    ~WorkspaceScope();
    WorkspaceScope(const WorkspaceScope&) = delete;
    WorkspaceScope& operator=(const WorkspaceScope&) = delete;
    void* impl = nullptr;
    bool owner = false;
};
void ws_release_all();
int64_t ws_bytes_held();
// Pool for per-call scratch that the arena cannot hold (private: the device's default pool and
// its release threshold are left as the process set them).  Keeps freed memory mapped.
cudaMemPool_t scratch_pool();

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) for `fn` on the current device, once per
// (device, kernel) and only when `bytes` exceeds what was set before (thread-safe).
void ensure_dyn_smem(const void* fn, size_t bytes);
template <class F> inline void ensure_dyn_smem_fn(F* fn, size_t bytes) {
    ensure_dyn_smem(reinterpret_cast<const void*>(fn), bytes);
}

struct Scratch {
    cudaStream_t st;
    void* p = nullptr;
    bool arena = false;
    explicit Scratch(cudaStream_t s) : st(s) {}
    Scratch(cudaStream_t s, size_t bytes) : st(s) { alloc(bytes); }
    void alloc(size_t bytes) {
        free_();
        if (bytes) p = ws_alloc(bytes, st, &arena);
    }
    void free_() {
        if (p && !arena) cudaFreeAsync(p, st);
        p = nullptr;
        arena = false;
    }
    ~Scratch() { free_(); }
    template <class T> T* as() const { return static_cast<T*>(p); }
    Scratch(const Scratch&) = delete;
    Scratch& operator=(const Scratch&) = delete;
};

}  // namespace detlsh
