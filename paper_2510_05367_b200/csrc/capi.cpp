// extern "C" boundary of liblightcache.so; see include/lightcache.h.
#include "../../include/lightcache.h"

#include <nccl.h>

#include <cmath>
#include <cstring>
#include <sstream>
#include <string>

#include "engine.hpp"
#include "metrics.cuh"

struct lc_ctx {
    explicit lc_ctx(int dev) : device(dev), engine(dev) {}
    int device;
    lc::Engine engine;
    ncclComm_t comm = nullptr;
    int world = 1, rank = 0;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    lc::ConvProfiler prof;
};

namespace {

thread_local std::string g_err;
thread_local int g_err_stage = -1;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const lc::LcError& e) {
        g_err = e.what();
        g_err_stage = e.code == lc::kBudgetError ? e.stage : -1;
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        g_err_stage = -1;
        return lc::kShapeError;
    }
}

// Entry points that take a context make its GPU current first: one context
// per GPU, several contexts per process (lightcache.h).
template <typename F>
int guarded_on(lc_ctx* ctx, F&& f) {
    return guarded([&] {
        if (!ctx) lc::throw_config("null lc_ctx");
        LC_CUDA(cudaSetDevice(ctx->device));
        f();
    });
}

void put(char* dst, int64_t cap, const std::string& s) {
    if (!dst || cap <= 0) return;
    const size_t n = std::min<size_t>(s.size(), static_cast<size_t>(cap - 1));
    std::memcpy(dst, s.data(), n);
    dst[n] = 0;
}

std::string report_json(const lc::Engine& e, const lc::RunStats& st) {
    static const char* stages[4] = {"setup", "encode", "denoise", "decode"};
    static const char* kinds[9] = {"compute_start", "compute_end", "xfer_start",     "xfer_end",       "await_start",
                                   "await_end",     "origin",      "await_part_start", "await_part_end"};
    std::ostringstream os;
    os.precision(10);
    os << "{\"device_ms\":{\"denoise\":" << st.ms_denoise << ",\"decode\":" << st.ms_decode
       << ",\"total\":" << st.ms_total << "},";
    os << "\"peaks\":{";
    for (int s = 0; s < 4; ++s)
        os << (s ? "," : "") << "\"" << stages[s] << "\":{\"fast\":" << st.peak[s][0]
           << ",\"slow\":" << st.peak[s][1] << "}";
    os << "},\"hbm_peak_bytes\":" << st.hbm_peak << ",";
    os << "\"mac\":{\"denoiser_total\":" << st.denoiser_macs << ",\"per_full_step\":" << st.macs_full
       << ",\"per_cached_step\":" << st.macs_cached << ",\"full_steps\":" << st.full_steps
       << ",\"cached_steps\":" << st.cached_steps << "},";
    os << "\"cache_bytes\":" << st.cache_bytes_planned << ",\"cache_bytes_physical\":"
       << st.cache_bytes_physical << ",";
    os << "\"swap\":{\"bytes\":" << st.swap_bytes << ",\"bytes_moved\":" << st.swap_bytes_moved
       << ",\"calls\":" << st.swap_calls << "},";
    os << "\"timeline\":{\"simulated\":" << (st.simulated ? "true" : "false")
       << ",\"makespan_ms\":" << st.makespan_ms << ",\"stall_ms\":" << st.stall_ms
       << ",\"events\":[";
    for (size_t i = 0; i < st.timeline.size(); ++i) {
        const auto& t = st.timeline[i];
        os << (i ? "," : "") << "[\"" << kinds[static_cast<int>(t[0])] << "\"," << static_cast<int64_t>(t[1])
           << "," << static_cast<int64_t>(t[2]) << "," << t[3] << "]";
    }
    os << "]},\"kernel_launches\":" << st.kernel_launches << ",";
    {
        const auto ai = e.arena_info();
        os << "\"arena\":{\"bytes\":" << ai.arena << ",\"activations\":" << ai.act << ",\"cache\":" << ai.cache
           << ",\"decode\":" << ai.dec << ",\"encode\":" << ai.enc
           << ",\"decode_overlaps_cache\":" << (ai.dec_overlaps_cache ? "true" : "false") << "},";
        os << "\"swap_schedule\":{\"link_gbs_probe\":" << e.link_gbs()
           << ",\"branch_deep\":" << e.branch_deep() << ",\"branch_seam\":" << (e.branch_seam() ? "true" : "false")
           << "},";
    }
    const auto& c = e.config();
    os << "\"video\":{\"frames\":" << c.frames << ",\"channels\":" << c.image_channels
       << ",\"height\":" << c.height << ",\"width\":" << c.width << "}}";
    return os.str();
}

// fp32 NCHW (n,c,h,w) -> fp16 NHWC with channel stride cs
std::vector<__half> to_nhwc(const float* x, int n, int c, int h, int w, int cs) {
    std::vector<__half> out(static_cast<size_t>(n) * h * w * cs, __float2half_rn(0.0f));
    for (int i = 0; i < n; ++i)
        for (int ch = 0; ch < c; ++ch)
            for (int y = 0; y < h; ++y)
                for (int xx = 0; xx < w; ++xx)
                    out[((static_cast<size_t>(i) * h + y) * w + xx) * cs + ch] =
                        __float2half_rn(x[((static_cast<size_t>(i) * c + ch) * h + y) * w + xx]);
    return out;
}
void from_nhwc(const std::vector<__half>& in, int n, int c, int h, int w, int cs, float* out) {
    for (int i = 0; i < n; ++i)
        for (int ch = 0; ch < c; ++ch)
            for (int y = 0; y < h; ++y)
                for (int xx = 0; xx < w; ++xx)
                    out[((static_cast<size_t>(i) * c + ch) * h + y) * w + xx] =
                        __half2float(in[((static_cast<size_t>(i) * h + y) * w + xx) * cs + ch]);
}
lc::Act upload_act(lc::DevBuf& buf, const float* x, int n, int c, int h, int w) {
    lc::Act a;
    a.n = n;
    a.c = c;
    a.h = h;
    a.w = w;
    a.cs = (c + 63) / 64 * 64;
    const auto hv = to_nhwc(x, n, c, h, w, a.cs);
    buf = lc::dev_alloc(nullptr, static_cast<int64_t>(hv.size()) * 2, false);
    lc::h2d_blocking(buf.p, hv.data(), hv.size() * 2);
    a.p = buf.as<__half>();
    return a;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw lc::LcError(lc::kCudaError, std::string("NCCL error ") + ncclGetErrorString(r) + " at " + what);
}

}  // namespace

extern "C" {

int lc_version(void) { return 1; }
const char* lc_last_error(void) { return g_err.c_str(); }
int lc_last_error_stage(void) { return g_err_stage; }

int lc_get_run_result(lc_ctx* ctx, lc_run_result* out, int64_t* timeline, int64_t cap_rows) {
    return guarded_on(ctx, [&] {
        const lc::RunStats& st = ctx->engine.last_stats();
        const lc::Ledger& l = ctx->engine.ledger();
        lc_run_result r{};
        r.wall_setup = st.setup_s;
        r.wall_encode = st.ms_encode * 1e-3;
        r.wall_denoise = st.ms_denoise * 1e-3;
        r.wall_decode = st.ms_decode * 1e-3;
        r.wall_total = st.ms_total * 1e-3;
        for (int s = 0; s < 4; ++s) {
            r.peak_fast[s] = st.peak[s][0];
            r.peak_slow[s] = st.peak[s][1];
            r.events_per_stage[s] = l.events_per_stage[s];
        }
        r.current_fast = l.occ[0];
        r.current_slow = l.occ[1];
        r.event_count = static_cast<int64_t>(l.events.size());
        r.denoiser_macs = st.denoiser_macs;
        r.macs_per_full_step = st.macs_full;
        r.macs_per_cached_step = st.macs_cached;
        r.full_steps = st.full_steps;
        r.cached_steps = st.cached_steps;
        r.cache_bytes_planned = st.cache_bytes_planned;
        r.makespan_s = st.makespan_ms * 1e-3;
        r.stall_s = st.stall_ms * 1e-3;
        r.simulated = st.simulated ? 1 : 0;
        // the reference's TimelineEventKind rows (the partial seam awaits,
        // kinds 7/8, are this engine's refinement and stay in the JSON report)
        int64_t n = 0;
        for (const auto& t : st.timeline) {
            const int kind = static_cast<int>(t[0]);
            if (kind > 5) continue;
            if (timeline) {
                if (n >= cap_rows) lc::throw_shape("timeline buffer too small");
                timeline[4 * n + 0] = kind;
                timeline[4 * n + 1] = static_cast<int64_t>(t[1]);
                timeline[4 * n + 2] = static_cast<int64_t>(t[2]);
                timeline[4 * n + 3] = static_cast<int64_t>(std::llround(t[3] * 1e6));
            }
            ++n;
        }
        r.n_timeline = n;
        if (out) *out = r;
    });
}

int lc_ctx_create(int device, lc_ctx** out) {
    return guarded([&] { *out = new lc_ctx(device); });
}
int lc_ctx_destroy(lc_ctx* ctx) {
    if (!ctx) return 0;
    return guarded_on(ctx, [&] {
        if (ctx->comm) ncclCommDestroy(ctx->comm);
        delete ctx;
    });
}

int lc_config_check(const char* text) {
    return guarded([&] { lc::parse_config_text(text ? text : "").validate(); });
}
int lc_config_to_text(const char* text, char* out, int64_t cap) {
    return guarded([&] { put(out, cap, lc::config_to_text(lc::parse_config_text(text ? text : ""))); });
}
int lc_configure(lc_ctx* ctx, const char* text) {
    return guarded_on(ctx, [&] { ctx->engine.configure(lc::parse_config_text(text ? text : "")); });
}
int64_t lc_latent_elems(lc_ctx* ctx) { return ctx->engine.latent_elems(); }
int64_t lc_video_elems(lc_ctx* ctx) { return ctx->engine.video_elems(); }

int lc_run_pipeline(lc_ctx* ctx, const float* x0, float* video, float* latent_out, char* report,
                    int64_t cap) {
    return guarded_on(ctx, [&] {
        const lc::RunStats st = ctx->engine.run(x0, video, latent_out, false);
        put(report, cap, report_json(ctx->engine, st));
    });
}
// Both copies are ordered on the engine's compute stream after any queued
// async runs (which read the staged latent / write the device video) and
// complete before returning.
int lc_upload_latent(lc_ctx* ctx, const float* x0) {
    return guarded_on(ctx, [&] {
        (void)ctx->engine.wait();
        ctx->engine.run_prepare();
        LC_CUDA(cudaMemcpyAsync(ctx->engine.latent_dev(), x0, static_cast<size_t>(ctx->engine.latent_elems()) * 4,
                                cudaMemcpyHostToDevice, ctx->engine.stream()));
        LC_CUDA(cudaStreamSynchronize(ctx->engine.stream()));
    });
}
int lc_run_resident(lc_ctx* ctx, char* report, int64_t cap) {
    return guarded_on(ctx, [&] {
        const lc::RunStats st = ctx->engine.run(nullptr, nullptr, nullptr, true);
        put(report, cap, report_json(ctx->engine, st));
    });
}
int lc_run_resident_async(lc_ctx* ctx) {
    return guarded_on(ctx, [&] { ctx->engine.run_resident_async(); });
}
int lc_run_pipeline_async(lc_ctx* ctx, const float* x0, float* video) {
    return guarded_on(ctx, [&] { ctx->engine.run_e2e_async(x0, video); });
}
int lc_wait(lc_ctx* ctx, char* report, int64_t cap) {
    return guarded_on(ctx, [&] {
        const lc::RunStats st = ctx->engine.wait();
        put(report, cap, report_json(ctx->engine, st));
    });
}
int lc_download_video(lc_ctx* ctx, float* video) {
    return guarded_on(ctx, [&] {
        (void)ctx->engine.wait();
        LC_CUDA(cudaMemcpyAsync(video, ctx->engine.video_dev(), static_cast<size_t>(ctx->engine.video_elems()) * 4,
                                cudaMemcpyDeviceToHost, ctx->engine.stream()));
        LC_CUDA(cudaStreamSynchronize(ctx->engine.stream()));
    });
}
int lc_set_decode_slice(lc_ctx* ctx, int64_t frames) {
    return guarded_on(ctx, [&] {
        if (frames < 1) lc::throw_config("decode slice must be >= 1");
        ctx->engine.decode_slice = frames;
    });
}

int lc_timer_start(lc_ctx* ctx) {
    return guarded_on(ctx, [&] {
        if (!ctx->t0) {
            LC_CUDA(cudaEventCreate(&ctx->t0));
            LC_CUDA(cudaEventCreate(&ctx->t1));
        }
        LC_CUDA(cudaEventRecord(ctx->t0, ctx->engine.stream()));
    });
}
int lc_timer_stop(lc_ctx* ctx, float* ms) {
    return guarded_on(ctx, [&] {
        LC_CUDA(cudaEventRecord(ctx->t1, ctx->engine.stream()));
        LC_CUDA(cudaEventSynchronize(ctx->t1));
        LC_CUDA(cudaEventElapsedTime(ms, ctx->t0, ctx->t1));
    });
}
int lc_set_conv_profile(lc_ctx* ctx, int on) {
    return guarded_on(ctx, [&] {
        ctx->prof.clear();
        lc::set_conv_profiler(on ? &ctx->prof : nullptr);
    });
}
int lc_conv_profile(lc_ctx* ctx, int64_t* launches, double* ms, double* alg, double* exec) {
    return guarded_on(ctx, [&] { ctx->prof.summarize(launches, ms, alg, exec); });
}
int lc_conv_profile_records(lc_ctx* ctx, char* buf, int64_t cap) {
    return guarded_on(ctx, [&] { put(buf, cap, ctx->prof.records_json()); });
}
void* lc_alloc_pinned(int64_t bytes) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, static_cast<size_t>(bytes), cudaHostAllocDefault) != cudaSuccess) {
        g_err = "cudaHostAlloc failed";
        return nullptr;
    }
    return p;
}
int lc_free_pinned(void* p) {
    return guarded([&] { LC_CUDA(cudaFreeHost(p)); });
}

int lc_forward(lc_ctx* ctx, const float* x, int64_t T, int64_t timestep, const float* deep_in,
               float* deep_out, float* eps) {
    return guarded_on(ctx, [&] { ctx->engine.forward(x, T, timestep, deep_in, deep_out, eps); });
}
int lc_ledger_csv(lc_ctx* ctx, char* buf, int64_t cap, int64_t* needed) {
    return guarded_on(ctx, [&] {
        static const char* kinds[5] = {"alloc", "free", "move_start", "move_end", "stage_enter"};
        static const char* stages[4] = {"setup", "encode", "denoise", "decode"};
        const lc::Ledger& l = ctx->engine.ledger();
        std::ostringstream os;
        os << "seq,clock,kind,tier,bytes,alloc_id,occupancy_bytes,stage\n";
        int64_t occ[2] = {0, 0};
        for (const lc::LedgerEvent& e : l.events) {
            // replay as write_ledger_csv does (ledger.cpp:224-242): a move's
            // start row carries the destination tier, its end the source
            if (e.kind == 0 || e.kind == 2) occ[e.tier] += e.bytes;
            if (e.kind == 1 || e.kind == 3) occ[e.tier] -= e.bytes;
            os << e.seq << ',' << e.clock << ',' << kinds[e.kind] << ',' << (e.tier ? "slow" : "fast") << ','
               << e.bytes << ',' << e.alloc_id << ',' << occ[e.tier] << ',' << stages[e.stage] << "\n";
        }
        const std::string t = os.str();
        if (needed) *needed = static_cast<int64_t>(t.size()) + 1;
        put(buf, cap, t);
    });
}
int lc_ledger_summary(lc_ctx* ctx, char* buf, int64_t cap) {
    return guarded_on(ctx, [&] {
        static const char* stages[4] = {"setup", "encode", "denoise", "decode"};
        const lc::Ledger& l = ctx->engine.ledger();
        std::ostringstream os;
        int64_t over[2] = {0, 0};
        os << "{\"clock\":\"" << (ctx->engine.config().swap_simulate ? "virtual" : "monotonic")
           << "\",\"stages\":{";
        for (int s = 0; s < 4; ++s) {
            over[0] = std::max(over[0], l.peak[s][0]);
            over[1] = std::max(over[1], l.peak[s][1]);
            os << (s ? "," : "") << "\"" << stages[s] << "\":{\"fast_peak_bytes\":" << l.peak[s][0]
               << ",\"slow_peak_bytes\":" << l.peak[s][1] << ",\"events\":" << l.events_per_stage[s] << "}";
        }
        os << "},\"overall\":{\"fast_peak_bytes\":" << over[0] << ",\"slow_peak_bytes\":" << over[1]
           << "},\"current\":{\"fast_bytes\":" << l.occ[0] << ",\"slow_bytes\":" << l.occ[1]
           << "},\"event_count\":" << l.events.size() << "}";
        put(buf, cap, os.str());
    });
}
int lc_video_metrics(lc_ctx* ctx, const float* a, const float* b, int64_t t, int64_t c, int64_t h, int64_t w,
                     double data_range, double* psnr, double* ssim) {
    return guarded_on(ctx, [&] {
        if (!(data_range > 0.0)) lc::throw_config("psnr: data_range must be positive");
        if (h < 7 || w < 7) lc::throw_shape("ssim: frame smaller than the 7x7 window");
        if (t < 1 || c < 1) lc::throw_shape("video_metrics: empty video");
        const size_t bytes = static_cast<size_t>(t * c * h * w) * 4;
        auto on_device = [](const void* p) {
            cudaPointerAttributes pa{};
            const bool dev = cudaPointerGetAttributes(&pa, p) == cudaSuccess &&
                             (pa.type == cudaMemoryTypeDevice || pa.type == cudaMemoryTypeManaged);
            cudaGetLastError();
            return dev;
        };
        lc::DevBuf da, db;
        const float* pa = a;
        const float* pb = b;
        cudaStream_t st = ctx->engine.stream();
        if (!on_device(a)) {
            da = lc::dev_alloc(nullptr, static_cast<int64_t>(bytes), false);
            LC_CUDA(cudaMemcpyAsync(da.p, a, bytes, cudaMemcpyHostToDevice, st));
            pa = da.as<float>();
        }
        if (!on_device(b)) {
            db = lc::dev_alloc(nullptr, static_cast<int64_t>(bytes), false);
            LC_CUDA(cudaMemcpyAsync(db.p, b, bytes, cudaMemcpyHostToDevice, st));
            pb = db.as<float>();
        }
        LC_CUDA(lc::video_metrics(pa, pb, t, c, h, w, data_range, psnr, ssim, st));
    });
}
int lc_decode(lc_ctx* ctx, const float* latents, int64_t n, int64_t c, int64_t h, int64_t w, int64_t slice,
              float* video) {
    return guarded_on(ctx, [&] { ctx->engine.decode(latents, n, c, h, w, video, slice); });
}

int lc_conv2d(lc_ctx* ctx, const float* x, int64_t b, int64_t t, int64_t c_in, int64_t h, int64_t w,
              const float* taps, const float* bias, int64_t c_out, int64_t k, float s, float o, int silu,
              float* out) {
    return guarded_on(ctx, [&] {
        if (k < 1 || k % 2 == 0) lc::throw_shape("kernel size must be odd");
        lc::Bank bank;
        bank.c_in = c_in;
        bank.c_out = c_out;
        bank.k = k;
        bank.taps.assign(taps, taps + c_out * c_in * k * k);
        bank.bias.assign(bias, bias + c_out);
        auto L = lc::pack_tc_layer(nullptr, bank, static_cast<int>(c_in), 0);
        const int n = static_cast<int>(b * t);
        lc::DevBuf xb, ob;
        const lc::Act xa = upload_act(xb, x, n, static_cast<int>(c_in), static_cast<int>(h), static_cast<int>(w));
        lc::Act oa;
        oa.n = n;
        oa.c = static_cast<int>(c_out);
        oa.h = static_cast<int>(h);
        oa.w = static_cast<int>(w);
        oa.cs = (oa.c + 63) / 64 * 64;
        ob = lc::dev_alloc(nullptr, oa.elems() * 2, true);
        oa.p = ob.as<__half>();
        const int H = static_cast<int>(h), W = static_cast<int>(w);
        lc::run_tc_conv(*L, &xa, oa, lc::Window{0, H, 0, W, 0, H, 0, W}, s, o, silu != 0,
                        ctx->engine.stream());
        LC_CUDA(cudaStreamSynchronize(ctx->engine.stream()));
        std::vector<__half> hv(static_cast<size_t>(oa.elems()));
        LC_CUDA(cudaMemcpy(hv.data(), oa.p, hv.size() * 2, cudaMemcpyDeviceToHost));
        from_nhwc(hv, n, oa.c, H, W, oa.cs, out);
    });
}

int lc_up_conv2d(lc_ctx* ctx, const float* skip, const float* u, int64_t b, int64_t t, int64_t c_a,
                 int64_t c_b, int64_t h, int64_t w, const float* taps, const float* bias, int64_t c_out,
                 float s, float o, float* out) {
    return guarded_on(ctx, [&] {
        if (h % 2 || w % 2) lc::throw_shape("up block needs even extents");
        lc::Bank bank;
        bank.c_in = c_a + c_b;
        bank.c_out = c_out;
        bank.k = 3;
        bank.taps.assign(taps, taps + c_out * (c_a + c_b) * 9);
        bank.bias.assign(bias, bias + c_out);
        auto L = lc::pack_tc_layer(nullptr, bank, static_cast<int>(c_a), 1);
        const int n = static_cast<int>(b * t), H = static_cast<int>(h), W = static_cast<int>(w);
        lc::DevBuf sb, ub, ob;
        lc::Act srcs[2];
        srcs[0] = upload_act(sb, skip, n, static_cast<int>(c_a), H, W);
        srcs[1] = upload_act(ub, u, n, static_cast<int>(c_b), H / 2, W / 2);
        lc::Act oa;
        oa.n = n;
        oa.c = static_cast<int>(c_out);
        oa.h = H;
        oa.w = W;
        oa.cs = (oa.c + 63) / 64 * 64;
        ob = lc::dev_alloc(nullptr, oa.elems() * 2, true);
        oa.p = ob.as<__half>();
        lc::run_tc_conv(*L, srcs, oa, lc::Window{0, H, 0, W, 0, H, 0, W}, s, o, true, ctx->engine.stream());
        LC_CUDA(cudaStreamSynchronize(ctx->engine.stream()));
        std::vector<__half> hv(static_cast<size_t>(oa.elems()));
        LC_CUDA(cudaMemcpy(hv.data(), oa.p, hv.size() * 2, cudaMemcpyDeviceToHost));
        from_nhwc(hv, n, oa.c, H, W, oa.cs, out);
    });
}

int lc_sampler_step(lc_ctx* ctx, int sampler, int64_t t, const float* x, const float* eps2, int64_t n,
                    double guidance, uint64_t noise_seed, float* x_out, int* nonfinite) {
    return guarded_on(ctx, [&] {
        if (sampler < 0 || sampler > 2) lc::throw_config("sampler must be 0 (ancestral), 1 (ddim) or 2 (euler)");
        if (n < 0) lc::throw_shape("sampler step: negative element count");
        // cfg_combine's check first, then reverse_step's check_t (pipeline order)
        if (guidance < 0.0) lc::throw_config("cfg_combine: guidance scale must be >= 0");
        const lc::Schedule sc = lc::make_schedule(ctx->engine.config());
        const lc::StepCoeffs k = lc::step_coeffs_at(static_cast<lc::Sampler>(sampler), sc, t, noise_seed);
        if (nonfinite) *nonfinite = 0;
        if (n == 0) return;
        std::vector<float> z;
        if (k.has_noise) {
            z.resize(static_cast<size_t>(n));
            lc::randn(k.noise_seed, n, z.data());
        }
        // one buffer: e_u e_c | x | z | x' | flag, each 16-byte aligned
        const int64_t seg = (n + 3) / 4 * 4;
        lc::DevBuf d = lc::dev_alloc(nullptr, (5 * seg + 4) * 4, false);
        float* e_d = d.as<float>();
        float* x_d = e_d + 2 * seg;
        float* z_d = x_d + seg;
        float* o_d = z_d + seg;
        int* bad_d = reinterpret_cast<int*>(o_d + seg);
        cudaStream_t st = ctx->engine.stream();
        LC_CUDA(cudaMemcpyAsync(e_d, eps2, n * 4, cudaMemcpyHostToDevice, st));
        LC_CUDA(cudaMemcpyAsync(e_d + n, eps2 + n, n * 4, cudaMemcpyHostToDevice, st));
        LC_CUDA(cudaMemcpyAsync(x_d, x, n * 4, cudaMemcpyHostToDevice, st));
        if (k.has_noise) LC_CUDA(cudaMemcpyAsync(z_d, z.data(), n * 4, cudaMemcpyHostToDevice, st));
        LC_CUDA(cudaMemsetAsync(bad_d, 0, 4, st));
        lc::StepArgs a{};
        a.eps2 = e_d;
        a.x = x_d;
        a.x_out = o_d;
        a.z = k.has_noise ? z_d : nullptr;
        a.n = n;
        a.g = static_cast<float>(guidance);
        a.a = k.a;
        a.b = k.b;
        a.c = k.noise;
        a.bad = bad_d;
        LC_CUDA(lc::launch_step(a, st));
        int bad = 0;
        LC_CUDA(cudaMemcpyAsync(x_out, o_d, n * 4, cudaMemcpyDeviceToHost, st));
        LC_CUDA(cudaMemcpyAsync(&bad, bad_d, 4, cudaMemcpyDeviceToHost, st));
        LC_CUDA(cudaStreamSynchronize(st));
        if (nonfinite) *nonfinite = bad;
    });
}

int lc_all_finite(lc_ctx* ctx, const float* x, int64_t n, int* finite) {
    return guarded_on(ctx, [&] {
        if (n < 0 || !finite) lc::throw_shape("all_finite: negative element count or null result");
        *finite = 1;
        if (n == 0) return;
        lc::DevBuf d = lc::dev_alloc(nullptr, (n + 3) / 4 * 16 + 4, false);
        float* x_d = d.as<float>();
        int* bad_d = reinterpret_cast<int*>(x_d + (n + 3) / 4 * 4);
        cudaStream_t st = ctx->engine.stream();
        LC_CUDA(cudaMemcpyAsync(x_d, x, n * 4, cudaMemcpyHostToDevice, st));
        LC_CUDA(cudaMemsetAsync(bad_d, 0, 4, st));
        LC_CUDA(lc::launch_isfinite(x_d, n, bad_d, st));
        int bad = 0;
        LC_CUDA(cudaMemcpyAsync(&bad, bad_d, 4, cudaMemcpyDeviceToHost, st));
        LC_CUDA(cudaStreamSynchronize(st));
        *finite = !bad;
    });
}

int lc_plan_steps(int64_t total, int64_t n, int8_t* kinds, int8_t* flags) {
    return guarded([&] {
        const lc::StepPlan p = lc::plan_steps(total, n);
        for (int64_t s = 0; s < total; ++s) {
            kinds[s] = p.is_full(s) ? 1 : 0;
            if (flags)
                flags[s] = static_cast<int8_t>((p.has_consumers(s) ? 1 : 0) | (p.is_last_consumer(s) ? 2 : 0));
        }
    });
}

int lc_split(int64_t h, int64_t w, int64_t eta, int64_t omega, int halo_kind, int64_t halo_px, int64_t k,
             int64_t* regions, int64_t* halo_out) {
    return guarded([&] {
        if (halo_kind < 0 || halo_kind > 2) lc::throw_config("halo kind must be 0, 1 or 2");
        const auto tiles = lc::split(h, w, eta, omega, static_cast<lc::HaloKind>(halo_kind), halo_px, k, halo_out);
        int64_t i = 0;
        for (const auto& t : tiles)
            for (const lc::Region* r : {&t.core, &t.padded, &t.out_window}) {
                regions[i++] = r->y0;
                regions[i++] = r->y1;
                regions[i++] = r->x0;
                regions[i++] = r->x1;
            }
    });
}

int lc_model_numbers(const char* text, int64_t* macs_full, int64_t* macs_cached, int64_t* cache_bytes) {
    return guarded([&] {
        const lc::RunConfig c = lc::parse_config_text(text ? text : "");
        c.validate();
        const int64_t lh = c.latent_h(), lw = c.latent_w();
        if (macs_full) *macs_full = lc::flops_estimate(c, 2, c.frames, lh, lw, false);
        if (macs_cached) *macs_cached = lc::flops_estimate(c, 2, c.frames, lh, lw, true);
        if (cache_bytes)
            *cache_bytes = 2 * c.frames * lc::cache_channels(c) * (lh >> c.cache_depth) * (lw >> c.cache_depth) * 4;
    });
}

int lc_plan_arena(const char* text, char* out, int64_t cap) {
    return guarded([&] {
        const lc::RunConfig c = lc::parse_config_text(text ? text : "");
        c.validate();
        const lc::ArenaPlan p = lc::plan_arena(c);
        std::ostringstream os;
        os << "{\"cache_bytes\":" << p.cache_bytes << ",\"act_end\":" << p.act_end << ",\"ops\":" << p.steps_ops
           << ",\"buffers\":[";
        bool first = true;
        for (const lc::ArenaBuf& b : p.bufs) {
            os << (first ? "" : ",") << "{\"name\":\"" << b.name << "\",\"bytes\":" << b.bytes << ",\"t0\":" << b.t0
               << ",\"t1\":" << b.t1 << ",\"off\":" << b.off << ",\"c\":" << b.c << ",\"cs\":" << b.cs << "}";
            first = false;
        }
        os << "]}";
        put(out, cap, os.str());
    });
}

int lc_simulate_timeline(const char* text, int64_t* events, int64_t cap_events, int64_t* n_events,
                         int64_t* makespan_ns, int64_t* stall_ns) {
    return guarded([&] {
        const lc::RunConfig c = lc::parse_config_text(text ? text : "");
        const auto tl = lc::simulate_timeline(c);
        if (n_events) *n_events = static_cast<int64_t>(tl.size());
        if (makespan_ns) *makespan_ns = lc::sim_makespan_ns(tl);
        if (stall_ns) *stall_ns = lc::sim_stall_ns(tl);
        if (events) {
            if (static_cast<int64_t>(tl.size()) > cap_events) lc::throw_shape("timeline buffer too small");
            for (size_t i = 0; i < tl.size(); ++i) {
                events[4 * i + 0] = tl[i].kind;
                events[4 * i + 1] = tl[i].step;
                events[4 * i + 2] = tl[i].bytes;
                events[4 * i + 3] = tl[i].clock_ns;
            }
        }
    });
}

uint64_t lc_derive_seed(uint64_t seed, uint64_t stream) { return lc::derive_seed(seed, stream); }
int lc_randn(uint64_t seed, int64_t n, float* out) {
    return guarded([&] { lc::randn(seed, n, out); });
}

int lc_shard_frames(int64_t T, int world, int rank, int64_t* first, int64_t* count) {
    return guarded([&] {
        const lc::ShardSpan sp = lc::shard_frames(T, world, rank);
        *first = sp.first;
        *count = sp.count;
    });
}

int lc_gather_plan(int64_t T, int world, int64_t slice, int64_t* rows, int64_t cap_rows, int64_t* n_rows) {
    return guarded([&] {
        const auto plan = lc::gather_plan(T, world, slice);
        if (n_rows) *n_rows = static_cast<int64_t>(plan.size());
        if (!rows) return;
        if (static_cast<int64_t>(plan.size()) > cap_rows) lc::throw_shape("gather plan buffer too small");
        for (size_t i = 0; i < plan.size(); ++i) {
            rows[4 * i + 0] = plan[i].round;
            rows[4 * i + 1] = plan[i].rank;
            rows[4 * i + 2] = plan[i].first;
            rows[4 * i + 3] = plan[i].count;
        }
    });
}

int lc_mem_info(lc_ctx* ctx, int64_t* free_bytes, int64_t* total_bytes) {
    return guarded_on(ctx, [&] {
        size_t f = 0, t = 0;
        LC_CUDA(cudaMemGetInfo(&f, &t));
        if (free_bytes) *free_bytes = static_cast<int64_t>(f);
        if (total_bytes) *total_bytes = static_cast<int64_t>(t);
    });
}

int lc_host_register(void* p, int64_t bytes) {
    return guarded([&] { LC_CUDA(cudaHostRegister(p, static_cast<size_t>(bytes), cudaHostRegisterPortable)); });
}
int lc_host_unregister(void* p) {
    return guarded([&] { LC_CUDA(cudaHostUnregister(p)); });
}

int lc_nccl_unique_id(uint8_t* id128) {
    return guarded([&] {
        ncclUniqueId id;
        nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(id128, &id, sizeof(id));
    });
}

int lc_nccl_init(lc_ctx* ctx, const uint8_t* id128, int world, int rank) {
    return guarded_on(ctx, [&] {
        ncclUniqueId id;
        std::memcpy(&id, id128, sizeof(id));
        LC_CUDA(cudaSetDevice(ctx->device));
        nccl_check(ncclCommInitRank(&ctx->comm, world, id, rank), "ncclCommInitRank");
        ctx->world = world;
        ctx->rank = rank;
    });
}

int lc_kernel_launches(lc_ctx* ctx, int64_t* n) {
    return guarded_on(ctx, [&] { *n = ctx->engine.launches; });
}
int lc_decode_sharded(lc_ctx* ctx, const float* latents, int64_t T, int64_t c, int64_t h, int64_t w,
                      int64_t slice, float* video, int flags, float* ms_out) {
    return guarded_on(ctx, [&] {
        if (!ctx->comm && ctx->world > 1) lc::throw_config("lc_nccl_init first");
        ctx->engine.decode_sharded(latents, T, c, h, w, slice, video, (flags & LC_SHARD_HOST_SHARED) != 0,
                                   ctx->comm, ctx->world, ctx->rank, ms_out);
    });
}

}  // extern "C"
