// lightcache.hpp -- header-only C++ mirror of the reference's operator and
// config API (namespace stagecache, /root/reference/proj/include/stagecache)
// over the C-ABI of liblightcache.so.  Same names, argument meaning and
// error behaviour: every failure rethrows the reference exception type for
// the status code (proj/include/stagecache/common.hpp:33-57).
//
// A reference user switches by replacing
//     #include "stagecache/pipeline.hpp"      stagecache::run_pipeline(cfg)
// with
//     #include "lightcache.hpp"               stagecache_b200::run_pipeline(text)
// where `text` is the reference's own config grammar (config_to_text output
// or a config file's contents), so existing configs and --set overrides
// carry over unchanged.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "lightcache.h"

namespace stagecache_b200 {

struct Error : std::runtime_error {
    explicit Error(const std::string& m) : std::runtime_error(m) {}
};
struct ShapeError : Error {
    using Error::Error;
};
struct ConfigError : Error {
    using Error::Error;
};
struct BudgetError : Error {
    int stage;  // 0 setup, 1 encode, 2 denoise, 3 decode (BudgetError::stage)
    BudgetError(int st, const std::string& m) : Error(m), stage(st) {}
};
struct InvariantError : Error {
    using Error::Error;
};
struct DeviceError : Error {
    using Error::Error;
};

inline void check(int rc) {
    if (rc == 0) return;
    const std::string m = lc_last_error();
    switch (rc) {
        case 1: throw ShapeError(m);
        case 2: throw ConfigError(m);
        case 3: throw BudgetError(lc_last_error_stage(), m);
        case 4: throw InvariantError(m);
        default: throw DeviceError(m);
    }
}

// StepPlan / plan_steps (proj/include/stagecache/cache.hpp:27-40).
struct StepPlan {
    std::vector<int8_t> kinds, flags;
    bool is_full(int64_t s) const { return kinds[static_cast<size_t>(s)] != 0; }
    bool has_consumers(int64_t s) const { return (flags[static_cast<size_t>(s)] & 1) != 0; }
    bool is_last_consumer(int64_t s) const { return (flags[static_cast<size_t>(s)] & 2) != 0; }
};
inline StepPlan plan_steps(int64_t total, int64_t interval_n) {
    StepPlan p;
    p.kinds.resize(static_cast<size_t>(total > 0 ? total : 0));
    p.flags.resize(p.kinds.size());
    check(lc_plan_steps(total, interval_n, p.kinds.data(), p.flags.data()));
    return p;
}

// StageWall / StageReport / TimelineEvent / RunResult
// (proj/include/stagecache/pipeline.hpp:11-39, ledger.hpp:49-63,
// swap.hpp:16-31) -- the typed result of lc_get_run_result plus the video.
struct StageWall {
    double setup = 0, encode = 0, denoise = 0, decode = 0, total = 0;
};
struct StageReport {
    std::array<std::array<int64_t, 2>, 4> peak{};  // [stage][tier]
    std::array<int64_t, 2> current{};
    std::array<int64_t, 4> events_per_stage{};
    uint64_t event_count = 0;
    int64_t stage_peak(int s, int t) const { return peak[static_cast<size_t>(s)][static_cast<size_t>(t)]; }
    int64_t overall_peak(int t) const {
        int64_t m = 0;
        for (const auto& row : peak) m = row[static_cast<size_t>(t)] > m ? row[static_cast<size_t>(t)] : m;
        return m;
    }
};
struct TimelineEvent {
    int kind = 0;  // TimelineEventKind: 0 compute_start .. 5 await_end
    int64_t step = -1, bytes = 0, clock_ns = 0;
};
struct RunResult {
    std::vector<float> video;  // b = 1, {t,c,h,w}
    StageWall wall;
    StageReport mem;
    std::vector<TimelineEvent> timeline;
    int64_t denoiser_macs = 0, macs_per_full_step = 0, macs_per_cached_step = 0;
    int64_t full_steps = 0, cached_steps = 0, cache_bytes_planned = 0;
    double makespan_s = 0, stall_s = 0;
    bool simulated = false;
    std::string report_json;  // the engine's JSON report (device ms, swap bytes, arena, ...)
};

// One GPU context (weights, buffers, streams).
class Context {
public:
    explicit Context(int device = 0) { check(lc_ctx_create(device, &ctx_)); }
    ~Context() { lc_ctx_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;

    // run_pipeline (proj/src/pipeline.cpp:64) for a config in the reference grammar.
    RunResult run_pipeline(const std::string& config_text) {
        check(lc_configure(ctx_, config_text.c_str()));
        RunResult r;
        r.video.resize(static_cast<size_t>(lc_video_elems(ctx_)));
        std::vector<char> rep(1 << 22);
        check(lc_run_pipeline(ctx_, nullptr, r.video.data(), nullptr, rep.data(),
                              static_cast<int64_t>(rep.size())));
        r.report_json = rep.data();
        fill_result(&r);
        return r;
    }
    // typed fields of the last run (lc_get_run_result)
    void fill_result(RunResult* r) {
        lc_run_result t{};
        check(lc_get_run_result(ctx_, &t, nullptr, 0));
        std::vector<int64_t> rows(static_cast<size_t>(4 * t.n_timeline));
        check(lc_get_run_result(ctx_, &t, rows.data(), t.n_timeline));
        r->wall = {t.wall_setup, t.wall_encode, t.wall_denoise, t.wall_decode, t.wall_total};
        for (size_t s = 0; s < 4; ++s) {
            r->mem.peak[s] = {t.peak_fast[s], t.peak_slow[s]};
            r->mem.events_per_stage[s] = t.events_per_stage[s];
        }
        r->mem.current = {t.current_fast, t.current_slow};
        r->mem.event_count = static_cast<uint64_t>(t.event_count);
        r->timeline.resize(static_cast<size_t>(t.n_timeline));
        for (size_t i = 0; i < r->timeline.size(); ++i)
            r->timeline[i] = {static_cast<int>(rows[4 * i]), rows[4 * i + 1], rows[4 * i + 2], rows[4 * i + 3]};
        r->denoiser_macs = t.denoiser_macs;
        r->macs_per_full_step = t.macs_per_full_step;
        r->macs_per_cached_step = t.macs_per_cached_step;
        r->full_steps = t.full_steps;
        r->cached_steps = t.cached_steps;
        r->cache_bytes_planned = t.cache_bytes_planned;
        r->makespan_s = t.makespan_s;
        r->stall_s = t.stall_s;
        r->simulated = t.simulated != 0;
    }
    // Throughput form with caller-owned (pinned) buffers: queue runs, then wait().
    void run_pipeline_async(const float* x0, float* video) { check(lc_run_pipeline_async(ctx_, x0, video)); }
    std::string wait() {
        std::vector<char> rep(1 << 22);
        check(lc_wait(ctx_, rep.data(), static_cast<int64_t>(rep.size())));
        return rep.data();
    }

    // video_series(psnr / ssim) (proj/src/metrics.cpp:81-104) of two b=1
    // videos {t,c,h,w}; host or device pointers.
    void video_metrics(const float* a, const float* b, int64_t t, int64_t c, int64_t h, int64_t w,
                       double data_range, std::vector<double>* psnr, std::vector<double>* ssim) {
        psnr->resize(static_cast<size_t>(t));
        ssim->resize(static_cast<size_t>(t));
        check(lc_video_metrics(ctx_, a, b, t, c, h, w, data_range, psnr->data(), ssim->data()));
    }

    // cfg_combine + reverse_step_{ancestral,ddim,euler} (proj/src/sampler.cpp:
    // 95-133) at index t of the configured schedule; kind follows SamplerKind
    // (0 ancestral, 1 ddim, 2 euler).  Returns x'.
    std::vector<float> sampler_step(int kind, int64_t t, const std::vector<float>& x,
                                    const std::vector<float>& eps_uncond, const std::vector<float>& eps_cond,
                                    double guidance, uint64_t noise_seed = 0) {
        if (eps_uncond.size() != x.size() || eps_cond.size() != x.size())
            throw ShapeError("cfg_combine: operand shapes differ");
        std::vector<float> eps2(eps_uncond);
        eps2.insert(eps2.end(), eps_cond.begin(), eps_cond.end());
        std::vector<float> out(x.size());
        check(lc_sampler_step(ctx_, kind, t, x.data(), eps2.data(), static_cast<int64_t>(x.size()), guidance,
                              noise_seed, out.data(), nullptr));
        return out;
    }

    // all_finite (proj/src/tensor.cpp:376) on the device.
    bool all_finite(const std::vector<float>& x) {
        int f = 0;
        check(lc_all_finite(ctx_, x.data(), static_cast<int64_t>(x.size()), &f));
        return f != 0;
    }

    // write_ledger_csv content (proj/src/ledger.cpp:224-242) of this engine.
    std::string ledger_csv() {
        int64_t need = 0;
        check(lc_ledger_csv(ctx_, nullptr, 0, &need));
        std::vector<char> buf(static_cast<size_t>(need) + 16);
        check(lc_ledger_csv(ctx_, buf.data(), static_cast<int64_t>(buf.size()), &need));
        return buf.data();
    }

    lc_ctx* raw() { return ctx_; }

private:
    lc_ctx* ctx_ = nullptr;
};

inline void validate_config(const std::string& config_text) { check(lc_config_check(config_text.c_str())); }

}  // namespace stagecache_b200
