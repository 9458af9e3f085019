// profile.cu -- per-kernel CUDA-event timing behind detlsh_profile_* (bench.py's live
// roofline numbers).  Off by default; when on, every DL_LAUNCH records an event pair on
// its own stream.
#include <chrono>
#include <cstring>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace detlsh {

std::atomic<int> g_profile{0};

namespace {
struct Rec {
    const char* name;
    cudaEvent_t a, b;
    bool done;
};
std::mutex g_mu;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;
struct Agg {
    int64_t launches = 0;
    double ms = 0;
};
std::map<std::string, Agg> g_agg;
std::vector<std::string> g_filter;   // name prefixes to time (empty: every kernel)

cudaEvent_t take_event() {
    if (!g_pool.empty()) {
        cudaEvent_t e = g_pool.back();
        g_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

void drain_locked() {
    // DETLSH_PROFILE_RAW=1: also print every launch as (start, duration) relative to the first
    // launch of the batch (a device timeline for finding gaps between kernels).
    static const bool raw = std::getenv("DETLSH_PROFILE_RAW") != nullptr;
    for (auto& r : g_recs) {
        cudaEventSynchronize(r.b);
        float ms = 0;
        cudaEventElapsedTime(&ms, r.a, r.b);
        if (raw) {
            float t0 = 0;
            cudaEventElapsedTime(&t0, g_recs.front().a, r.a);
            std::fprintf(stderr, "[detlsh launch] %10.3f %8.3f %s\n", t0, ms, r.name);
        }
        Agg& g = g_agg[r.name];
        g.launches += 1;
        g.ms += ms;
    }
    for (auto& r : g_recs) {
        g_pool.push_back(r.a);
        g_pool.push_back(r.b);
    }
    g_recs.clear();
}
}  // namespace

void profile_begin(cudaStream_t st, const char* name, int* slot) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_filter.empty()) {
        bool hit = false;
        for (const auto& f : g_filter) hit |= std::strncmp(name, f.c_str(), f.size()) == 0;
        if (!hit) return;
    }
    if (g_recs.size() > 100000) drain_locked();
    Rec r{name, take_event(), take_event(), false};
    cudaEventRecord(r.a, st);
    g_recs.push_back(r);
    *slot = (int)g_recs.size() - 1;
}

void profile_end(cudaStream_t st, int slot) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (slot < (int)g_recs.size()) cudaEventRecord(g_recs[slot].b, st);
}

static double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

Trace::Trace(const char* w) : on(std::getenv("DETLSH_TRACE") != nullptr), t0(now_ms()), last(t0), what(w) {}

void Trace::mark(const char* phase, cudaStream_t st) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const double t = now_ms();
    std::fprintf(stderr, "[detlsh %s] %-28s %8.3f ms (total %8.3f)\n", what, phase, t - last, t - t0);
    last = t;
}

}  // namespace detlsh

using namespace detlsh;

extern "C" {

void detlsh_profile_enable(int32_t on) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_profile.store(on ? 1 : 0);
}

void detlsh_profile_filter(const char* prefixes) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_filter.clear();
    if (!prefixes) return;
    std::string cur;
    for (const char* c = prefixes;; ++c) {
        if (*c == ',' || *c == 0) {
            if (!cur.empty()) g_filter.push_back(cur);
            cur.clear();
            if (*c == 0) break;
        } else {
            cur.push_back(*c);
        }
    }
}

void detlsh_profile_reset(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    drain_locked();
    g_agg.clear();
}

int32_t detlsh_profile_read(detlsh_kernel_time* out, int32_t cap) {
    std::lock_guard<std::mutex> lk(g_mu);
    drain_locked();
    int32_t i = 0;
    for (auto& kv : g_agg) {
        if (out && i < cap) {
            std::snprintf(out[i].name, sizeof(out[i].name), "%s", kv.first.c_str());
            out[i].launches = kv.second.launches;
            out[i].total_ms = kv.second.ms;
        }
        ++i;
    }
    return i;
}

}  // extern "C"
