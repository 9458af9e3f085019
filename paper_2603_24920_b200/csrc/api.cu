// api.cu -- the C ABI (include/detlsh.h): argument validation, host/device marshalling,
// error capture.  Every step of the method runs in the kernels of build.cu / query.cu /
// project_*.cu / radix.cu; this file only moves buffers and checks arguments.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "index.cuh"

namespace detlsh {

std::atomic<int64_t> g_launches{0};
// PDL on every launch unless DETLSH_PDL=0 (read per call: experiments switch it between calls)
bool pdl_enabled() {
    const char* e = std::getenv("DETLSH_PDL");
    return !(e && std::atoi(e) == 0);
}
static thread_local std::string g_err;

void project_rows_simt(const Index& ix, const float* d_X, int64_t ld, int64_t m, float* d_P, int* d_nonfinite,
                       cudaStream_t st);
bool project_rows_tc(const Index& ix, const float* d_X, int64_t ld, int64_t m, float* d_P, int* d_nonfinite,
                     cudaStream_t st);

void project_rows(const Index& ix, const float* d_X, int64_t ld, int64_t m, float* d_P, int proj_impl,
                  int* d_nonfinite, cudaStream_t st) {
    DL_REQUIRE(ld == ix.ld, "projection row stride mismatch");
    if (m <= 0) return;
    // proj_impl 0: tensor cores (tcgen05) for every shape whose hash matrix fits in shared
    // memory; other shapes (and proj_impl 1) use the CUDA-core kernel.
    if (proj_impl == 0 && project_rows_tc(ix, d_X, ld, m, d_P, d_nonfinite, st)) return;
    project_rows_simt(ix, d_X, ld, m, d_P, d_nonfinite, st);
}

std::atomic<int64_t> g_index_bytes{0};

cudaMemPool_t index_pool() {
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
        uint64_t thr = UINT64_MAX;
        DL_CUDA(cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr));
    }
    return pools[dev];
}

namespace {

template <class F> detlsh_status guard(F&& f) {
    try {
        f();
        return DETLSH_OK;
    } catch (const Error& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return DETLSH_ENOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return DETLSH_EINTERNAL;
    }
}

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes at;
    cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

void require_device() {
    int cnt = 0;
    cudaError_t e = cudaGetDeviceCount(&cnt);
    if (e != cudaSuccess || cnt == 0) {
        cudaGetLastError();
        throw Error(DETLSH_ECUDA, "no CUDA device available");
    }
    // scratch and index memory come from the library's own pools (scratch_pool, index_pool),
    // which keep freed memory mapped; the device's default pool is left alone
}

cudaStream_t stream_of(const detlsh_opts* o) { return o ? reinterpret_cast<cudaStream_t>(o->stream) : (cudaStream_t)0; }

detlsh_opts opts_or_default(const detlsh_opts* o) {
    detlsh_opts d;
    detlsh_default_opts(&d);
    return o ? *o : d;
}

void validate_shape(int64_t n, int32_t d, int32_t L, int32_t K, int32_t N_r) {
    DL_REQUIRE(n >= 1 && n < ((int64_t)1 << 31), "n must be in [1, 2^31)");
    DL_REQUIRE(d >= 1, "d must be >= 1");
    DL_REQUIRE(L >= 1, "L must be >= 1");
    DL_REQUIRE(K >= 1 && K <= 32, "K must be in [1, 32]");
    DL_REQUIRE(N_r >= 2 && N_r <= 256 && (N_r & (N_r - 1)) == 0, "N_r must be a power of two in [2, 256]");
    DL_REQUIRE((int64_t)n * L < 0xFFFFFFFFll, "n * L must be < 2^32");
}

// Copy rows[m][d] (host or device) into a device buffer [m][ld] (zero padded).
void stage_rows(const float* src, int64_t m, int32_t d, int32_t ld, float* dst, cudaStream_t st) {
    if (ld != d) DL_CUDA(cudaMemsetAsync(dst, 0, sizeof(float) * (size_t)m * ld, st));
    if (m > 0)
        DL_CUDA(cudaMemcpy2DAsync(dst, sizeof(float) * ld, src, sizeof(float) * d, sizeof(float) * d, (size_t)m,
                                  cudaMemcpyDefault, st));
}

void init_index_params(Index& ix, int64_t n, int32_t d, int32_t L, int32_t K, int32_t N_r, uint64_t seed,
                       const detlsh_opts& o) {
    ix.n = n;
    ix.n_global = n;
    ix.d = d;
    ix.ld = (int32_t)round_up(d, 8);
    ix.L = L;
    ix.K = K;
    ix.LK = L * K;
    ix.N_r = N_r;
    ix.nb = 0;
    while ((1 << ix.nb) < N_r) ++ix.nb;
    ix.max_size = o.max_size;
    ix.seed = seed;
    ix.eps = std::sqrt(chi2_upper_quantile(std::exp(-1.0 / L), K));   // Eq. 2
}

struct DevOut {  // a device view of a caller buffer (host buffers are staged)
    void* user;
    size_t bytes;
    bool host;
    Scratch tmp;
    DevOut(void* u, size_t b, cudaStream_t st) : user(u), bytes(b), host(!is_device_ptr(u)), tmp(st) {
        if (host && bytes) tmp.alloc(bytes);
    }
    void* dev() { return host ? tmp.p : user; }
    void finish(cudaStream_t st) {
        if (host && bytes) DL_CUDA(cudaMemcpyAsync(user, tmp.p, bytes, cudaMemcpyDeviceToHost, st));
    }
};

}  // namespace
}  // namespace detlsh

using namespace detlsh;

extern "C" {

void detlsh_default_opts(detlsh_opts* o) {
    if (!o) return;
    std::memset(o, 0, sizeof(*o));
    o->max_size = 128;
    o->sample_frac = 0.01;
    o->mode = DETLSH_MODE_CELL;
    o->query_batch = 0;
    o->stream = 0;
    o->borrow_data = 0;
    o->proj_impl = 0;
    o->mem_budget = 0;
    o->verify_impl = 0;
    o->keep_projections = 0;
    o->lb_order = 0;
    o->pad1 = 0;
}

const char* detlsh_last_error(void) { return g_err.c_str(); }

int64_t detlsh_launch_count(void) { return g_launches.load(); }

int64_t detlsh_sample_size(int64_t n, int32_t N_r, double f) {
    int64_t a = (int64_t)std::ceil(f * (double)n);
    int64_t m = std::max<int64_t>(a, 32 * (int64_t)N_r);
    return std::min<int64_t>(m, n);
}

detlsh_status detlsh_params(int32_t K, int32_t L, double c, double* eps, double* alpha2, double* beta_theory) {
    return guard([&] {
        DL_REQUIRE(K >= 1 && L >= 1 && c > 1.0, "need K >= 1, L >= 1, c > 1");
        const double e2 = chi2_upper_quantile(std::exp(-1.0 / L), K);
        const double a2 = chi2_survival(e2 / (c * c), K);
        if (eps) *eps = std::sqrt(e2);
        if (alpha2) *alpha2 = a2;
        if (beta_theory) *beta_theory = 2.0 - 2.0 * std::pow(a2, (double)L);
    });
}

detlsh_status detlsh_build_ex(const float* data, int64_t n, int32_t d, int32_t L, int32_t K, int32_t N_r,
                              uint64_t seed, const detlsh_opts* opts, int64_t id_offset, int64_t n_global,
                              const float* breakpoints, detlsh_index** out) {
    return guard([&] {
        DL_REQUIRE(out, "out is NULL");
        DL_REQUIRE(data, "data is NULL");
        validate_shape(n, d, L, K, N_r);
        const detlsh_opts o = opts_or_default(opts);
        DL_REQUIRE(o.max_size >= 1, "max_size must be >= 1");
        DL_REQUIRE(o.sample_frac > 0.0 && o.sample_frac <= 1.0, "sample_frac must be in (0, 1]");
        DL_REQUIRE(id_offset >= 0, "id_offset must be >= 0");
        require_device();
        cudaStream_t st = stream_of(&o);
        WorkspaceScope ws(st);
        auto ix = std::make_unique<Index>();
        init_index_params(*ix, n, d, L, K, N_r, seed, o);
        ix->keep_proj = o.keep_projections != 0;
        ix->id_offset = id_offset;
        ix->n_global = std::max<int64_t>(n_global, n);
        const bool dev = is_device_ptr(data);
        if (o.borrow_data && dev && d % 8 == 0) {
            ix->Xp = data;
        } else {
            ix->X.alloc(sizeof(float) * (size_t)n * ix->ld, st);
            stage_rows(data, n, d, ix->ld, ix->X.as<float>(), st);
            ix->Xp = ix->X.as<float>();
        }
        const float* bp = nullptr;
        Scratch s_bp(st);
        if (breakpoints) {
            const size_t bytes = sizeof(float) * (size_t)ix->LK * (N_r + 1);
            s_bp.alloc(bytes);
            DL_CUDA(cudaMemcpyAsync(s_bp.p, breakpoints, bytes, cudaMemcpyDefault, st));
            bp = s_bp.as<float>();
        }
        build_index(*ix, ix->Xp, ix->ld, bp, o.sample_frac, o.proj_impl, st);
        DL_CUDA(cudaStreamSynchronize(st));
        *out = reinterpret_cast<detlsh_index*>(ix.release());
    });
}

detlsh_status detlsh_build(const float* data, int64_t n, int32_t d, int32_t L, int32_t K, int32_t N_r,
                           uint64_t seed, detlsh_index** out) {
    return detlsh_build_ex(data, n, d, L, K, N_r, seed, nullptr, 0, n, nullptr, out);
}

static detlsh_status run_query(const detlsh_index* idx, const float* queries, int64_t nq, int32_t k, double c,
                               double r_min, double beta, const detlsh_opts* opts, int64_t* out_ids, float* out_dists,
                               detlsh_query_stats* stats, int max_rounds, bool null_on_cap,
                               uint32_t* export_S = nullptr, int64_t S_words = 0) {
    return guard([&] {
        DL_REQUIRE(idx, "index is NULL");
        const Index& ix = *reinterpret_cast<const Index*>(idx);
        DL_REQUIRE(!ix.codes_only, "index was built from codes only (no data to verify against)");
        DL_REQUIRE(nq >= 0, "nq must be >= 0");
        if (nq == 0) return;
        DL_REQUIRE(queries && out_ids && out_dists, "NULL buffer");
        DL_REQUIRE(k >= 1 && k <= ix.n && k <= 4096, "k must be in [1, min(n, 4096)]");
        DL_REQUIRE(c > 1.0 && std::isfinite(c), "c must be > 1");
        DL_REQUIRE(beta > 0.0 && std::isfinite(beta), "beta must be > 0");
        DL_REQUIRE(r_min > 0.0 && std::isfinite(r_min), "r_min must be > 0 and finite");
        const detlsh_opts o = opts_or_default(opts);
        DL_REQUIRE(o.mode == DETLSH_MODE_CELL || o.mode == DETLSH_MODE_RELAXED || o.mode == DETLSH_MODE_EXACT,
                   "unknown mode");
        DL_REQUIRE(o.mode != DETLSH_MODE_EXACT || ix.proj.p != nullptr,
                   "EXACT mode needs an index built with opts.keep_projections = 1");
        require_device();
        cudaStream_t st = stream_of(&o);
        WorkspaceScope ws(st);
        Scratch s_q(st, sizeof(float) * (size_t)nq * ix.ld);
        stage_rows(queries, nq, ix.d, ix.ld, s_q.as<float>(), st);
        DevOut oi(out_ids, sizeof(int64_t) * (size_t)(nq * k), st);
        DevOut od(out_dists, sizeof(float) * (size_t)(nq * k), st);
        std::unique_ptr<DevOut> os;
        if (stats) os.reset(new DevOut(stats, sizeof(detlsh_query_stats) * (size_t)nq, st));
        std::unique_ptr<DevOut> oS;
        if (export_S) {
            DL_REQUIRE(S_words == ceil_div(ix.n, 32), "S_words must be ceil(n / 32)");
            oS.reset(new DevOut(export_S, sizeof(uint32_t) * (size_t)(nq * S_words), st));
        }
        DL_REQUIRE(o.verify_impl >= 0 && o.verify_impl <= 3, "verify_impl must be 0..3");
        QueryArgs a{nq, k, c, r_min, beta, o.mode, o.query_batch, o.mem_budget, o.proj_impl, o.verify_impl};
        a.max_rounds = max_rounds;
        a.null_on_cap = null_on_cap;
        a.lb_order = o.lb_order ? 1 : 0;
        a.export_S = oS ? static_cast<uint32_t*>(oS->dev()) : nullptr;
        query_index(ix, s_q.as<float>(), ix.ld, a, static_cast<int64_t*>(oi.dev()), static_cast<float*>(od.dev()),
                    os ? static_cast<detlsh_query_stats*>(os->dev()) : nullptr, st);
        oi.finish(st);
        od.finish(st);
        if (os) os->finish(st);
        if (oS) oS->finish(st);
        DL_CUDA(cudaStreamSynchronize(st));
    });
}

detlsh_status detlsh_query_ex(const detlsh_index* idx, const float* queries, int64_t nq, int32_t k, double c,
                              double r_min, double beta, const detlsh_opts* opts, int64_t* out_ids, float* out_dists,
                              detlsh_query_stats* stats) {
    return run_query(idx, queries, nq, k, c, r_min, beta, opts, out_ids, out_dists, stats, 64, false);
}

detlsh_status detlsh_query_candidates(const detlsh_index* idx, const float* queries, int64_t nq, int32_t k, double c,
                                      double r_min, double beta, const detlsh_opts* opts, int64_t* out_ids,
                                      float* out_dists, detlsh_query_stats* stats, uint32_t* S, int64_t S_words) {
    if (!S) {
        g_err = "S is NULL";
        return DETLSH_EINVAL;
    }
    return run_query(idx, queries, nq, k, c, r_min, beta, opts, out_ids, out_dists, stats, 64, false, S, S_words);
}

detlsh_status detlsh_rc_ann(const detlsh_index* idx, const float* queries, int64_t nq, double r, double c,
                            double beta, const detlsh_opts* opts, int64_t* out_ids, float* out_dists,
                            detlsh_query_stats* stats) {
    return run_query(idx, queries, nq, 1, c, r, beta, opts, out_ids, out_dists, stats, 1, true);
}

detlsh_status detlsh_query(const detlsh_index* idx, const float* queries, int64_t nq, int32_t k, double c,
                           double r_min, double beta, int64_t* out_ids, float* out_dists) {
    return detlsh_query_ex(idx, queries, nq, k, c, r_min, beta, nullptr, out_ids, out_dists, nullptr);
}

detlsh_status detlsh_estimate_rmin(const detlsh_index* idx, const float* queries, int64_t ns, int32_t k, double beta,
                                   const detlsh_opts* opts, double* rstar, double* r_min) {
    return guard([&] {
        DL_REQUIRE(idx && queries && r_min, "NULL argument");
        const Index& ix = *reinterpret_cast<const Index*>(idx);
        DL_REQUIRE(!ix.codes_only, "index was built from codes only");
        DL_REQUIRE(ns >= 1, "need at least one sample query");
        DL_REQUIRE(k >= 1 && k <= ix.n, "k must be in [1, n]");
        DL_REQUIRE(beta > 0.0 && std::isfinite(beta), "beta must be > 0");
        const detlsh_opts o = opts_or_default(opts);
        require_device();
        cudaStream_t st = stream_of(&o);
        WorkspaceScope ws(st);
        Scratch s_q(st, sizeof(float) * (size_t)ns * ix.ld);
        stage_rows(queries, ns, ix.d, ix.ld, s_q.as<float>(), st);
        std::vector<double> rs((size_t)ns);
        estimate_rstar(ix, s_q.as<float>(), ix.ld, ns, k, beta, o.proj_impl, rs.data(), st);
        if (rstar) std::memcpy(rstar, rs.data(), sizeof(double) * (size_t)ns);
        std::vector<double> sorted = rs;
        std::sort(sorted.begin(), sorted.end());
        *r_min = sorted[(size_t)(ns - 1) / 2];      // lower median (AMB-22)
        DL_REQUIRE(*r_min > 0.0, "estimated r_min is 0 (more than beta n + k points share the sample queries' "
                                 "cells in every tree); choose a positive r_min");
    });
}

detlsh_status detlsh_save(const detlsh_index* idx, const char* path) {
    return guard([&] {
        DL_REQUIRE(idx, "index is NULL");
        require_device();
        save_index(*reinterpret_cast<const Index*>(idx), path);
    });
}

detlsh_status detlsh_load(const char* path, detlsh_index** out) {
    return guard([&] {
        DL_REQUIRE(out, "out is NULL");
        require_device();
        *out = reinterpret_cast<detlsh_index*>(load_index(path));
    });
}

detlsh_status detlsh_index_info(const detlsh_index* idx, int64_t* info) {
    return guard([&] {
        DL_REQUIRE(idx && info, "NULL argument");
        const Index& ix = *reinterpret_cast<const Index*>(idx);
        const int64_t v[8] = {ix.n, ix.d, ix.L, ix.K, ix.N_r, ix.n_global, ix.id_offset, ix.codes_only ? 1 : 0};
        std::memcpy(info, v, sizeof(v));
    });
}

void detlsh_free(detlsh_index* idx) {
    if (!idx) return;
    delete reinterpret_cast<Index*>(idx);
}

detlsh_status detlsh_project(const detlsh_index* idx, const float* X, int64_t m, float* out) {
    return guard([&] {
        DL_REQUIRE(idx && X && out, "NULL argument");
        const Index& ix = *reinterpret_cast<const Index*>(idx);
        DL_REQUIRE(!ix.codes_only, "index has no hash family");
        DL_REQUIRE(m >= 0, "m must be >= 0");
        if (m == 0) return;
        require_device();
        cudaStream_t st = 0;
        WorkspaceScope ws(st);
        Scratch s_x(st, sizeof(float) * (size_t)m * ix.ld);
        stage_rows(X, m, ix.d, ix.ld, s_x.as<float>(), st);
        Scratch s_flag(st, sizeof(int));
        DL_CUDA(cudaMemsetAsync(s_flag.p, 0, sizeof(int), st));
        DevOut o(out, sizeof(float) * (size_t)(m * ix.LK), st);
        project_rows(ix, s_x.as<float>(), ix.ld, m, static_cast<float*>(o.dev()), 0, s_flag.as<int>(), st);
        o.finish(st);
        DL_CUDA(cudaStreamSynchronize(st));
    });
}

detlsh_status detlsh_project_ex(const detlsh_index* idx, const float* X, int64_t m, int32_t proj_impl, float* out) {
    return guard([&] {
        DL_REQUIRE(idx && X && out, "NULL argument");
        const Index& ix = *reinterpret_cast<const Index*>(idx);
        DL_REQUIRE(!ix.codes_only, "index has no hash family");
        if (m <= 0) return;
        require_device();
        cudaStream_t st = 0;
        WorkspaceScope ws(st);
        Scratch s_x(st, sizeof(float) * (size_t)m * ix.ld);
        stage_rows(X, m, ix.d, ix.ld, s_x.as<float>(), st);
        Scratch s_flag(st, sizeof(int));
        DL_CUDA(cudaMemsetAsync(s_flag.p, 0, sizeof(int), st));
        DevOut o(out, sizeof(float) * (size_t)(m * ix.LK), st);
        project_rows(ix, s_x.as<float>(), ix.ld, m, static_cast<float*>(o.dev()), proj_impl, s_flag.as<int>(), st);
        o.finish(st);
        DL_CUDA(cudaStreamSynchronize(st));
    });
}

detlsh_status detlsh_sample_projections(const float* data, int64_t n, int32_t d, int32_t L, int32_t K, int32_t N_r,
                                        uint64_t seed, double sample_frac, int64_t id_offset, int64_t n_global,
                                        const detlsh_opts* opts, float* out, int64_t cap, int64_t* n_out) {
    return guard([&] {
        DL_REQUIRE(data && out && n_out, "NULL argument");
        validate_shape(n, d, L, K, N_r);
        DL_REQUIRE(n_global >= id_offset + n && id_offset >= 0, "shard range outside [0, n_global)");
        DL_REQUIRE(sample_frac > 0.0 && sample_frac <= 1.0, "sample_frac must be in (0, 1]");
        const detlsh_opts o = opts_or_default(opts);
        require_device();
        cudaStream_t st = stream_of(&o);
        WorkspaceScope ws(st);
        Index ix;
        init_index_params(ix, n, d, L, K, N_r, seed, o);
        const int64_t n_s = detlsh_sample_size(n_global, N_r, sample_frac);
        Scratch s_ids(st, sizeof(uint32_t) * (size_t)std::min<int64_t>(n_s, n));
        int64_t got = 0;
        sample_ids_device(seed, id_offset, n, n_global, n_s, s_ids.as<uint32_t>(), &got, st);
        DL_REQUIRE(got <= cap, "cap too small for this shard's sample rows");
        // the sampled rows, padded to the index row stride
        Scratch s_x(st, sizeof(float) * (size_t)std::max<int64_t>(got, 1) * ix.ld);
        if (is_device_ptr(data)) {
            gather_rows_strided(data, d, d, s_ids.as<uint32_t>(), got, s_x.as<float>(), ix.ld, st);
        } else {
            std::vector<uint32_t> ids(got);
            DL_CUDA(cudaMemcpyAsync(ids.data(), s_ids.p, sizeof(uint32_t) * got, cudaMemcpyDeviceToHost, st));
            DL_CUDA(cudaStreamSynchronize(st));
            std::vector<float> rows((size_t)got * ix.ld, 0.f);
            for (int64_t i = 0; i < got; ++i)
                std::memcpy(rows.data() + i * ix.ld, data + (int64_t)ids[i] * d, sizeof(float) * d);
            DL_CUDA(cudaMemcpyAsync(s_x.p, rows.data(), sizeof(float) * rows.size(), cudaMemcpyHostToDevice, st));
            DL_CUDA(cudaStreamSynchronize(st));
        }
        Index full;
        init_index_params(full, n, d, L, K, N_r, seed, o);
        build_index_hash_only(full, st);
        Scratch s_flag(st, sizeof(int));
        DL_CUDA(cudaMemsetAsync(s_flag.p, 0, sizeof(int), st));
        DevOut po(out, sizeof(float) * (size_t)std::max<int64_t>(got, 1) * ix.LK, st);
        project_rows(full, s_x.as<float>(), full.ld, got, static_cast<float*>(po.dev()), o.proj_impl,
                     s_flag.as<int>(), st);
        if (got) po.finish(st);
        DL_CUDA(cudaStreamSynchronize(st));
        *n_out = got;
    });
}

detlsh_status detlsh_breakpoints_from_samples(const float* samples, int64_t m, int32_t LK, int32_t N_r,
                                              const detlsh_opts* opts, float* out) {
    return guard([&] {
        DL_REQUIRE(samples && out, "NULL argument");
        DL_REQUIRE(m >= 1 && LK >= 1, "need m >= 1, LK >= 1");
        DL_REQUIRE(N_r >= 2 && N_r <= 256 && (N_r & (N_r - 1)) == 0, "N_r must be a power of two in [2, 256]");
        require_device();
        const detlsh_opts o = opts_or_default(opts);
        cudaStream_t st = stream_of(&o);
        WorkspaceScope ws(st);
        Scratch s_in(st, sizeof(float) * (size_t)(m * LK));
        DL_CUDA(cudaMemcpyAsync(s_in.p, samples, sizeof(float) * (size_t)(m * LK), cudaMemcpyDefault, st));
        DevOut bo(out, sizeof(float) * (size_t)LK * (N_r + 1), st);
        breakpoints_from_projections(s_in.as<float>(), m, LK, N_r, static_cast<float*>(bo.dev()), st);
        bo.finish(st);
        DL_CUDA(cudaStreamSynchronize(st));
    });
}

detlsh_status detlsh_merge_topk(const int64_t* ids, const float* dists, int32_t G, int64_t nq, int32_t k,
                                int64_t* out_ids, float* out_dists) {
    return guard([&] {
        DL_REQUIRE(ids && dists && out_ids && out_dists, "NULL argument");
        DL_REQUIRE(G >= 1 && nq >= 0 && k >= 1, "need G >= 1, nq >= 0, k >= 1");
        if (nq == 0) return;
        require_device();
        cudaStream_t st = 0;
        WorkspaceScope ws(st);
        const size_t ni = sizeof(int64_t) * (size_t)G * nq * k, nd = sizeof(float) * (size_t)G * nq * k;
        Scratch s_i(st), s_d(st);
        const int64_t* di = ids;
        const float* dd = dists;
        if (!is_device_ptr(ids)) {
            s_i.alloc(ni);
            DL_CUDA(cudaMemcpyAsync(s_i.p, ids, ni, cudaMemcpyHostToDevice, st));
            di = s_i.as<int64_t>();
        }
        if (!is_device_ptr(dists)) {
            s_d.alloc(nd);
            DL_CUDA(cudaMemcpyAsync(s_d.p, dists, nd, cudaMemcpyHostToDevice, st));
            dd = s_d.as<float>();
        }
        DevOut oi(out_ids, sizeof(int64_t) * (size_t)(nq * k), st);
        DevOut od(out_dists, sizeof(float) * (size_t)(nq * k), st);
        merge_topk_device(di, dd, G, nq, k, static_cast<int64_t*>(oi.dev()), static_cast<float*>(od.dev()), st);
        oi.finish(st);
        od.finish(st);
        DL_CUDA(cudaStreamSynchronize(st));
    });
}

detlsh_status detlsh_build_from_codes(const uint8_t* codes, int64_t n, int32_t L, int32_t K, int32_t N_r,
                                      const detlsh_opts* opts, detlsh_index** out) {
    return guard([&] {
        DL_REQUIRE(codes && out, "NULL argument");
        validate_shape(n, 1, L, K, N_r);
        const detlsh_opts o = opts_or_default(opts);
        DL_REQUIRE(o.max_size >= 1, "max_size must be >= 1");
        require_device();
        cudaStream_t st = stream_of(&o);
        WorkspaceScope ws(st);
        auto ix = std::make_unique<Index>();
        init_index_params(*ix, n, 1, L, K, N_r, 0, o);
        ix->codes_only = true;
        Scratch s_c(st, (size_t)n * ix->LK);
        DL_CUDA(cudaMemcpyAsync(s_c.p, codes, (size_t)n * ix->LK, cudaMemcpyDefault, st));
        build_trees_from_codes(*ix, s_c.as<uint8_t>(), st);
        DL_CUDA(cudaStreamSynchronize(st));
        *out = reinterpret_cast<detlsh_index*>(ix.release());
    });
}

detlsh_status detlsh_debug_export(const detlsh_index* idx, int32_t what, int32_t tree, void* dst, size_t bytes,
                                  size_t* needed) {
    return guard([&] {
        DL_REQUIRE(idx, "index is NULL");
        const Index& ix = *reinterpret_cast<const Index*>(idx);
        DL_REQUIRE(what == 0 || what == 1 || what == 2 || what == 3 || what == 9 || (tree >= 0 && tree < ix.L),
                   "tree out of range");
        const int64_t n = ix.n, K = ix.K, LK = ix.LK;
        const int64_t lb = (what >= 4 && what <= 9 && tree >= 0 && tree < ix.L) ? ix.tree_leaf_begin[tree] : 0;
        const int64_t le = (what >= 4 && what <= 9 && tree >= 0 && tree < ix.L) ? ix.tree_leaf_begin[tree + 1] : 0;
        const int64_t nl = le - lb;
        size_t need = 0;
        switch (what) {
            case 0: need = sizeof(float) * (size_t)(LK * ix.d); break;
            case 1: need = sizeof(float) * (size_t)(LK * (ix.N_r + 1)); break;
            case 2: need = (size_t)(n * LK); break;
            case 3: need = sizeof(int64_t) * (size_t)ix.n_s; break;
            case 4: need = sizeof(int64_t) * (size_t)n; break;
            case 5: need = sizeof(int64_t) * (size_t)(nl + 1); break;
            case 6: case 7: case 8: need = (size_t)(nl * K); break;
            case 9: need = sizeof(int64_t) * 4; break;
            default: throw Error(DETLSH_EINVAL, "unknown export id");
        }
        if (needed) *needed = need;
        if (!dst) return;
        DL_REQUIRE(bytes >= need, "destination too small");
        DL_REQUIRE(!(ix.codes_only && (what == 0 || what == 1 || what == 3)), "not available for a codes-only index");
        cudaStream_t st = 0;
        auto d2h = [&](void* h, const void* d, size_t b) {
            if (b) DL_CUDA(cudaMemcpy(h, d, b, cudaMemcpyDeviceToHost));
        };
        switch (what) {
            case 0: {
                std::vector<float> a((size_t)LK * ix.ld);
                d2h(a.data(), ix.A.p, a.size() * 4);
                float* o = static_cast<float*>(dst);
                for (int64_t r = 0; r < LK; ++r) std::memcpy(o + r * ix.d, a.data() + r * ix.ld, sizeof(float) * ix.d);
                break;
            }
            case 1: d2h(dst, ix.B.p, need); break;
            case 2: {   // reconstruct data-order codes from tree-order codes of every tree
                std::vector<uint32_t> perm((size_t)n * ix.L);
                std::vector<uint8_t> tc((size_t)n * ix.L * K);
                d2h(perm.data(), ix.perm.p, perm.size() * 4);
                d2h(tc.data(), ix.tcodes.p, tc.size());
                uint8_t* o = static_cast<uint8_t*>(dst);
                for (int64_t t = 0; t < ix.L; ++t)
                    for (int64_t p = 0; p < n; ++p)
                        std::memcpy(o + (int64_t)perm[t * n + p] * LK + t * K, tc.data() + (t * n + p) * K, K);
                break;
            }
            case 3: {
                std::vector<uint32_t> s((size_t)ix.n_s);
                d2h(s.data(), ix.sample.p, s.size() * 4);
                std::sort(s.begin(), s.end());
                int64_t* o = static_cast<int64_t*>(dst);
                for (size_t i = 0; i < s.size(); ++i) o[i] = (int64_t)s[i] + ix.id_offset;
                break;
            }
            case 4: {
                // canonical order: a leaf's points by ascending id (the device layout orders them by a
                // locality key for the sub-box bounds, build.cu k_leaf_morton)
                std::vector<uint32_t> p((size_t)n), off((size_t)nl + 1);
                d2h(p.data(), ix.perm.as<uint32_t>() + (size_t)tree * n, p.size() * 4);
                d2h(off.data(), ix.leaf_off.as<uint32_t>() + lb, off.size() * 4);
                for (int64_t l = 0; l < nl; ++l)
                    std::sort(p.begin() + (off[l] - (int64_t)tree * n), p.begin() + (off[l + 1] - (int64_t)tree * n));
                int64_t* o = static_cast<int64_t*>(dst);
                for (int64_t i = 0; i < n; ++i) o[i] = p[i];
                break;
            }
            case 5: {
                std::vector<uint32_t> p((size_t)nl + 1);
                d2h(p.data(), ix.leaf_off.as<uint32_t>() + lb, p.size() * 4);
                int64_t* o = static_cast<int64_t*>(dst);
                for (int64_t i = 0; i <= nl; ++i) o[i] = (int64_t)p[i] - (int64_t)tree * n;
                break;
            }
            case 6: d2h(dst, ix.leaf_lo.as<uint8_t>() + lb * K, need); break;
            case 7: d2h(dst, ix.leaf_hi.as<uint8_t>() + lb * K, need); break;
            case 8: d2h(dst, ix.leaf_bits.as<uint8_t>() + lb * K, need); break;
            case 9: {
                int64_t* o = static_cast<int64_t*>(dst);
                o[0] = n; o[1] = ix.n_s; o[2] = nl; o[3] = ix.d;
                break;
            }
        }
        (void)st;
    });
}

}  // extern "C"
