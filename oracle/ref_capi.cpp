// C-ABI shim over the UNMODIFIED reference library (stagecache, compiled in
// place from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).
// TEST INFRASTRUCTURE ONLY: used by tests/ (golden-vector generation and
// cross-checks of oracle/lc_oracle.c) and by bench.py's reference arm.  The
// product library never links or loads this file.
//
// Every entry point returns 0 on success, or the reference CLI's exit code
// for the exception type it caught (proj/tools/main.cpp:157-169):
// ConfigError 2, BudgetError 3, InvariantError 4, anything else 1.
#include <cstring>
#include <sstream>
#include <string>

#include "stagecache/cache.hpp"
#include "stagecache/chunk.hpp"
#include "stagecache/codec.hpp"
#include "stagecache/config.hpp"
#include "stagecache/metrics.hpp"
#include "stagecache/pipeline.hpp"
#include "stagecache/sampler.hpp"
#include "stagecache/unet.hpp"

using namespace stagecache;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 2;
    } catch (const BudgetError& e) {
        g_err = e.what();
        return 3;
    } catch (const InvariantError& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// "key = value" lines (the config-file grammar, proj/src/config.cpp:206-224)
// applied on top of default_config().
RunConfig parse_text(const char* text) {
    RunConfig cfg = default_config();
    std::istringstream is(text ? text : "");
    std::string line;
    while (std::getline(is, line)) {
        const auto hash = line.find('#');
        if (hash != std::string::npos) line = line.substr(0, hash);
        const auto eq = line.find('=');
        auto trim = [](std::string s) {
            const auto b = s.find_first_not_of(" \t\r\n");
            if (b == std::string::npos) return std::string();
            const auto e = s.find_last_not_of(" \t\r\n");
            return s.substr(b, e - b + 1);
        };
        if (trim(line).empty()) continue;
        if (eq == std::string::npos) throw ConfigError("expected key = value");
        apply_override(cfg, trim(line.substr(0, eq)), trim(line.substr(eq + 1)));
    }
    return cfg;
}

void copy_out(const Tensor5& t, float* dst) {
    std::memcpy(dst, t.data(), static_cast<size_t>(t.bytes()));
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Full run_pipeline (proj/src/pipeline.cpp:64).  `video` receives the b=1
// video {t,c,h,w}; `report` the run_report_json text; `macs` (4 int64):
// denoiser_total, per_full, per_cached, cache_bytes_planned.
int ref_run_pipeline(const char* config_text, float* video, int64_t video_cap_elems,
                     char* report, int64_t report_cap, int64_t* macs) {
    return guarded([&] {
        RunConfig cfg = parse_text(config_text);
        cfg.out_dir = "";
        RunResult r = run_pipeline(cfg);
        if (video) {
            if (r.video.elems() > video_cap_elems) throw ShapeError("video buffer too small");
            copy_out(r.video, video);
        }
        if (report) {
            const std::string js = run_report_json(r);
            std::strncpy(report, js.c_str(), static_cast<size_t>(report_cap - 1));
            report[report_cap - 1] = 0;
        }
        if (macs) {
            macs[0] = r.denoiser_macs;
            macs[1] = r.macs_per_full_step;
            macs[2] = r.macs_per_cached_step;
            macs[3] = r.cache_bytes_planned;
        }
    });
}

// run_pipeline's engine timeline (proj/src/pipeline.cpp:209, swap.hpp:26-31)
// as (kind, step, bytes, clock_ns) rows; `info` (3 int64): event count,
// makespan_ns, stall_total_ns (swap.cpp:59-79).  With swap.simulate = true
// the clocks are the simulated engine's virtual nanoseconds.
int ref_timeline(const char* config_text, int64_t* events, int64_t cap_events, int64_t* info) {
    return guarded([&] {
        RunConfig cfg = parse_text(config_text);
        cfg.out_dir = "";
        RunResult r = run_pipeline(cfg);
        const auto& tl = r.timeline;
        info[0] = static_cast<int64_t>(tl.size());
        info[1] = makespan_ns(tl);
        info[2] = stall_total_ns(tl);
        if (static_cast<int64_t>(tl.size()) > cap_events) throw ShapeError("timeline buffer too small");
        for (size_t i = 0; i < tl.size(); ++i) {
            events[4 * i + 0] = static_cast<int64_t>(tl[i].kind);
            events[4 * i + 1] = tl[i].step;
            events[4 * i + 2] = tl[i].bytes;
            events[4 * i + 3] = tl[i].clock_ns;
        }
    });
}

// Config validation only (reference grammar + RunConfig::validate).
int ref_check_config(const char* config_text) {
    return guarded([&] { parse_text(config_text).validate(); });
}

// forward_full (proj/src/unet.cpp:188) on x (2,T,C,h,w) using the config's
// U-Net and chunk settings.  eps has x's shape; deep receives u_next.
int ref_forward_full(const char* config_text, const float* x, int64_t t, int64_t h, int64_t w,
                     int64_t timestep, float* eps, float* deep) {
    return guarded([&] {
        RunConfig cfg = parse_text(config_text);
        const UNetWeights wts = init_weights(cfg.unet);
        Tensor5 xin = Tensor5::uninit({2, t, cfg.unet.in_channels, h, w});
        std::memcpy(xin.data(), x, static_cast<size_t>(xin.bytes()));
        FullForwardResult r = forward_full(xin, timestep, wts, cfg.unet,
                                           cfg.chunk_enabled ? &cfg.chunk : nullptr, nullptr);
        copy_out(r.eps, eps);
        if (deep) copy_out(r.deep.u_next, deep);
    });
}

// forward_cached (proj/src/unet.cpp:232) consuming `deep` at the seam.
int ref_forward_cached(const char* config_text, const float* x, int64_t t, int64_t h, int64_t w,
                       int64_t timestep, const float* deep, float* eps) {
    return guarded([&] {
        RunConfig cfg = parse_text(config_text);
        const UNetWeights wts = init_weights(cfg.unet);
        Tensor5 xin = Tensor5::uninit({2, t, cfg.unet.in_channels, h, w});
        std::memcpy(xin.data(), x, static_cast<size_t>(xin.bytes()));
        DeepFeatures d;
        d.u_next = Tensor5::uninit(cache_feature_shape(cfg.unet, xin.shape()));
        std::memcpy(d.u_next.data(), deep, static_cast<size_t>(d.u_next.bytes()));
        Tensor5 e = forward_cached(xin, timestep, wts, cfg.unet, std::move(d),
                                   cfg.chunk_enabled ? &cfg.chunk : nullptr, nullptr);
        copy_out(e, eps);
    });
}

// decode_batch / decode_sliced (proj/src/codec.cpp:117-145) of latents
// (n,1,C,h,w) -> (n,1,3,h*s,w*s).
int ref_decode(const char* config_text, const float* lat, int64_t n, int64_t h, int64_t w,
               int sliced, float* video) {
    return guarded([&] {
        RunConfig cfg = parse_text(config_text);
        const CodecWeights cw = init_codec(cfg.codec);
        Tensor5 l = Tensor5::uninit({1, n, cfg.codec.latent_channels, h, w});
        std::memcpy(l.data(), lat, static_cast<size_t>(l.bytes()));
        LatentBatch lb = merge_bt(std::move(l));
        Tensor5 v = sliced ? decode_sliced(lb, cw, cfg.codec) : decode_batch(lb, cw, cfg.codec);
        copy_out(v, video);
    });
}

// cfg_combine + reverse_step_{ancestral,ddim,euler} (proj/src/sampler.cpp:
// 95-133) at index t of the config's spaced schedule (pipeline.cpp:90-93);
// kind follows SamplerKind (0 ancestral, 1 ddim, 2 euler); x, eps_u, eps_c
// and out hold n floats.
int ref_sampler_step(const char* config_text, int kind, int64_t t, const float* x, const float* eps_u,
                     const float* eps_c, int64_t n, double guidance, uint64_t noise_seed, float* out) {
    return guarded([&] {
        RunConfig cfg = parse_text(config_text);
        const NoiseSchedule train = make_linear_schedule(cfg.train_steps, cfg.beta_min, cfg.beta_max);
        const SampledSchedule sub = spaced_schedule(train, cfg.inference_steps);
        auto load = [n](const float* src) {
            Tensor5 v = Tensor5::uninit({1, 1, 1, 1, n});
            std::memcpy(v.data(), src, static_cast<size_t>(v.bytes()));
            return v;
        };
        const Tensor5 xt = load(x), eu = load(eps_u), ec = load(eps_c);
        const Tensor5 eps = cfg_combine({eu, ec, guidance});
        Tensor5 r;
        switch (kind) {
            case 0: r = reverse_step_ancestral(xt, t, eps, sub.schedule, noise_seed); break;
            case 1: r = reverse_step_ddim(xt, t, eps, sub.schedule); break;
            case 2: r = reverse_step_euler(xt, t, eps, sub.schedule); break;
            default: throw ConfigError("sampler kind");
        }
        copy_out(r, out);
    });
}

// conv2d_window (proj/src/tensor.cpp:155) with explicit taps/bias.
int ref_conv2d_window(const float* x, int64_t b, int64_t t, int64_t c, int64_t h, int64_t w,
                      const float* taps, const float* bias, int64_t c_out, int64_t k, int64_t y0,
                      int64_t y1, int64_t x0, int64_t x1, float* out) {
    return guarded([&] {
        Tensor5 xin = Tensor5::uninit({b, t, c, h, w});
        std::memcpy(xin.data(), x, static_cast<size_t>(xin.bytes()));
        KernelBank bank;
        bank.c_in = c;
        bank.c_out = c_out;
        bank.k = k;
        bank.taps.assign(taps, taps + c_out * c * k * k);
        bank.bias.assign(bias, bias + c_out);
        Tensor5 o = conv2d_window(xin, bank, y0, y1, x0, x1);
        copy_out(o, out);
    });
}

// plan_steps (proj/src/cache.cpp:25): kinds[s] = 1 for Full, 0 for Cached;
// flags[s] bit0 has_consumers, bit1 is_last_consumer.
int ref_plan_steps(int64_t total, int64_t n, int8_t* kinds, int8_t* flags) {
    return guarded([&] {
        const StepPlan p = plan_steps(total, {n, 0});
        for (int64_t s = 0; s < total; ++s) {
            kinds[s] = p.is_full(s) ? 1 : 0;
            flags[s] = static_cast<int8_t>((p.has_consumers(s) ? 1 : 0) |
                                           (p.is_last_consumer(s) ? 2 : 0));
        }
    });
}

// split (proj/src/chunk.cpp:145) for a single-conv chain of kernel k.
// regions: 12 int64 per tile (core, padded, out_window as y0,y1,x0,x1).
int ref_split(int64_t h, int64_t w, int64_t eta, int64_t omega, int halo_kind, int64_t halo_px,
              int64_t k, int64_t* regions, int64_t* halo_out) {
    return guarded([&] {
        KernelBank bank;
        bank.c_in = 1;
        bank.c_out = 1;
        bank.k = k;
        bank.taps.assign(static_cast<size_t>(k * k), 0.0f);
        bank.bias.assign(1, 0.0f);
        ChunkSpec spec;
        spec.eta = eta;
        spec.omega = omega;
        spec.halo = halo_kind == 0   ? HaloMode::exact()
                    : halo_kind == 1 ? HaloMode::fixed_px(halo_px)
                                     : HaloMode::none();
        const TileGrid g = split({1, 1, 1, h, w}, spec, BlockChain{ChainOp::conv(bank)});
        *halo_out = g.halo_px;
        int64_t i = 0;
        for (const Tile& t : g.tiles) {
            for (const SpatialRegion* r : {&t.core, &t.padded, &t.out_window}) {
                regions[i++] = r->y0;
                regions[i++] = r->y1;
                regions[i++] = r->x0;
                regions[i++] = r->x1;
            }
        }
    });
}

// flops_estimate / cache_feature_shape / cache_bytes (proj/src/unet.cpp:287-309,
// proj/src/cache.cpp:124) for the config's model input.
int ref_model_numbers(const char* config_text, int64_t* out) {
    return guarded([&] {
        RunConfig cfg = parse_text(config_text);
        const Shape5 in = cfg.model_input_shape();
        out[0] = flops_estimate(cfg.unet, in, ForwardMode::Full);
        out[1] = flops_estimate(cfg.unet, in, ForwardMode::Cached);
        const Shape5 cs = cache_feature_shape(cfg.unet, in);
        out[2] = cs.b;
        out[3] = cs.t;
        out[4] = cs.c;
        out[5] = cs.h;
        out[6] = cs.w;
        out[7] = cache_bytes(cfg.cache_policy(), cfg.unet, in);
    });
}

// video_series(psnr/ssim) over two b=1 videos {t,c,h,w} (proj/src/metrics.cpp:10-104).
int ref_video_metrics(const float* a, const float* b, int64_t t, int64_t c, int64_t h, int64_t w,
                      double data_range, double* psnr_out, double* ssim_out) {
    return guarded([&] {
        Tensor5 ta = Tensor5::uninit({1, t, c, h, w});
        Tensor5 tb = Tensor5::uninit({1, t, c, h, w});
        std::memcpy(ta.data(), a, static_cast<size_t>(ta.bytes()));
        std::memcpy(tb.data(), b, static_cast<size_t>(tb.bytes()));
        const MetricSeries ps = video_series(&psnr, ta, tb, data_range);
        const MetricSeries ss = video_series(&ssim, ta, tb, data_range);
        for (int64_t i = 0; i < t; ++i) {
            psnr_out[i] = ps.per_frame[static_cast<size_t>(i)];
            ssim_out[i] = ss.per_frame[static_cast<size_t>(i)];
        }
    });
}

// write_video_raw (proj/src/codec.cpp:172-182): the artifact format.
int ref_write_video_raw(const char* path, const float* video, int64_t t, int64_t c, int64_t h, int64_t w) {
    return guarded([&] {
        Tensor5 v = Tensor5::uninit({1, t, c, h, w});
        std::memcpy(v.data(), video, static_cast<size_t>(v.bytes()));
        write_video_raw(path, v);
    });
}

}  // extern "C"
