// Host-side model; see host.hpp.  Each function cites the reference code it
// restates (paths relative to /root/reference/proj).
#include "host.hpp"

#include <algorithm>
#include <cctype>
#include <cmath>
#include <sstream>

namespace lc {

namespace {

std::string trim(const std::string& s) {
    const auto b = s.find_first_not_of(" \t\r\n");
    if (b == std::string::npos) return "";
    const auto e = s.find_last_not_of(" \t\r\n");
    return s.substr(b, e - b + 1);
}

// src/config.cpp:16-63 value parsers
int64_t parse_int(const std::string& key, const std::string& v) {
    try {
        size_t pos = 0;
        const int64_t out = std::stoll(v, &pos);
        if (pos != v.size()) throw std::invalid_argument(v);
        return out;
    } catch (const std::exception&) {
        throw_config("key '" + key + "': expected an integer, got '" + v + "'");
    }
}
uint64_t parse_uint(const std::string& key, const std::string& v) {
    try {
        size_t pos = 0;
        const uint64_t out = std::stoull(v, &pos);
        if (pos != v.size()) throw std::invalid_argument(v);
        return out;
    } catch (const std::exception&) {
        throw_config("key '" + key + "': expected an unsigned integer, got '" + v + "'");
    }
}
double parse_double(const std::string& key, const std::string& v) {
    try {
        size_t pos = 0;
        const double out = std::stod(v, &pos);
        if (pos != v.size()) throw std::invalid_argument(v);
        return out;
    } catch (const std::exception&) {
        throw_config("key '" + key + "': expected a number, got '" + v + "'");
    }
}
bool parse_bool(const std::string& key, const std::string& v) {
    if (v == "true" || v == "on" || v == "1") return true;
    if (v == "false" || v == "off" || v == "0") return false;
    throw_config("key '" + key + "': expected a boolean, got '" + v + "'");
}
std::vector<std::string> split_list(const std::string& v) {
    std::vector<std::string> out;
    std::string item;
    std::istringstream is(v);
    while (std::getline(is, item, ',')) {
        item = trim(item);
        if (!item.empty()) out.push_back(item);
    }
    return out;
}
Sampler sampler_from_string(const std::string& s) {  // sampler.cpp:143-148
    if (s == "ancestral") return Sampler::Ancestral;
    if (s == "ddim") return Sampler::Ddim;
    if (s == "euler") return Sampler::Euler;
    throw_config("unknown sampler '" + s + "'");
}
const char* to_string(Sampler s) {
    return s == Sampler::Ancestral ? "ancestral" : s == Sampler::Ddim ? "ddim" : "euler";
}
SwapMode swap_from_string(const std::string& s) {  // swap.cpp:21-26
    if (s == "off") return SwapMode::Off;
    if (s == "sync") return SwapMode::Sync;
    if (s == "async") return SwapMode::Async;
    throw_config("unknown swap mode '" + s + "'");
}
const char* to_string(SwapMode m) {
    return m == SwapMode::Off ? "off" : m == SwapMode::Sync ? "sync" : "async";
}
const char* to_string(HaloKind h) {
    return h == HaloKind::Exact ? "exact" : h == HaloKind::None ? "none" : "fixed";
}

}  // namespace

// src/config.cpp:100-141 (+ UNetConfig::validate unet.cpp:139-146,
// CodecConfig::validate codec.cpp:39-43)
void RunConfig::validate() const {
    if (frames < 1) throw_config("run.frames must be >= 1");
    if (height < 1 || width < 1) throw_config("run.height/run.width must be >= 1");
    if (mode != "text" && mode != "image") throw_config("run.mode must be 'text' or 'image'");
    if (depth < 1) throw_config("unet depth must be >= 1");
    if (base_channels < 1) throw_config("base_channels must be >= 1");
    if (kernel < 1 || kernel % 2 == 0) throw_config("kernel must be odd");
    if (cache_depth < 0 || cache_depth >= depth) throw_config("cache_depth must lie in [0, depth)");
    if (in_channels < 1) throw_config("in_channels must be >= 1");
    if (latent_channels < 1 || image_channels < 1 || codec_width < 1)
        throw_config("codec channel counts must be >= 1");
    if (stages < 1) throw_config("codec upsample_stages must be >= 1");
    if (in_channels != latent_channels)
        throw_config("unet.in_channels must equal codec.latent_channels");
    if (height % scale() != 0 || width % scale() != 0)
        throw_config("pixel extents must be divisible by the codec scale " + std::to_string(scale()));
    const int64_t lh = latent_h(), lw = latent_w();
    const int64_t div = int64_t(1) << depth;
    if (lh % div != 0 || lw % div != 0)
        throw_config("latent extents must be divisible by 2^unet.depth = " + std::to_string(div));
    if (train_steps < 1) throw_config("schedule.train_steps must be >= 1");
    if (!(beta_min > 0.0) || !(beta_min <= beta_max) || !(beta_max < 1.0))
        throw_config("schedule betas must satisfy 0 < beta_min <= beta_max < 1");
    if (steps < 1 || steps > train_steps)
        throw_config("sampler.steps must lie in [1, schedule.train_steps]");
    if (guidance < 0.0) throw_config("sampler.guidance must be >= 0");
    if (cache_enabled && cache_n < 1) throw_config("cache.n must be >= 1");
    if (chunk_enabled) {
        if (eta < 1 || omega < 1) throw_config("chunk.eta/omega must be >= 1");
        for (const std::string& t : targets) {
            int64_t level = 0;
            if ((t[0] == 'u' || t[0] == 'd') && t.size() > 1 && isdigit(static_cast<unsigned char>(t[1])))
                level = parse_int("chunk.targets", t.substr(1));
            else if (t == "mid")
                level = depth;
            const int64_t h = lh >> level, w = lw >> level;
            if (h % eta != 0 || w % omega != 0)
                throw_config("chunk target '" + t + "' extent " + std::to_string(h) + "x" +
                             std::to_string(w) + " not divisible by eta x omega");
        }
    }
    if (budget_fast_bytes < 0) throw_config("budget.fast_bytes must be >= 0");
    if (swap_simulate && !(swap_bandwidth > 0))  // swap.cpp:117-120
        throw_config("simulated transfer engine needs bandwidth > 0");
    if (swap_simulate && !(swap_mac_rate > 0))
        throw_config("simulated transfer engine needs a positive MAC rate");
}

RunConfig RunConfig::baseline() const {
    RunConfig b = *this;
    b.cache_enabled = false;
    b.chunk_enabled = false;
    b.slice_decode = false;
    b.swap_mode = SwapMode::Off;
    b.budget_fast_bytes = 0;
    return b;
}

// src/config.cpp:158-204
void apply_override(RunConfig& cfg, const std::string& key, const std::string& value) {
    const std::string v = trim(value);
    if (key == "run.frames") cfg.frames = parse_int(key, v);
    else if (key == "run.height") cfg.height = parse_int(key, v);
    else if (key == "run.width") cfg.width = parse_int(key, v);
    else if (key == "run.seed") cfg.seed = parse_uint(key, v);
    else if (key == "run.mode") cfg.mode = v;
    else if (key == "run.out_dir") cfg.out_dir = v;
    else if (key == "unet.depth") cfg.depth = parse_int(key, v);
    else if (key == "unet.base_channels") cfg.base_channels = parse_int(key, v);
    else if (key == "unet.kernel") cfg.kernel = parse_int(key, v);
    else if (key == "unet.cache_depth") cfg.cache_depth = parse_int(key, v);
    else if (key == "unet.weight_seed") cfg.unet_seed = parse_uint(key, v);
    else if (key == "codec.latent_channels") {
        cfg.latent_channels = parse_int(key, v);
        cfg.in_channels = cfg.latent_channels;
    } else if (key == "codec.stages") cfg.stages = parse_int(key, v);
    else if (key == "codec.width") cfg.codec_width = parse_int(key, v);
    else if (key == "codec.weight_seed") cfg.codec_seed = parse_uint(key, v);
    else if (key == "schedule.train_steps") cfg.train_steps = parse_int(key, v);
    else if (key == "schedule.beta_min") cfg.beta_min = parse_double(key, v);
    else if (key == "schedule.beta_max") cfg.beta_max = parse_double(key, v);
    else if (key == "sampler.kind") cfg.sampler = sampler_from_string(v);
    else if (key == "sampler.steps") cfg.steps = parse_int(key, v);
    else if (key == "sampler.guidance") cfg.guidance = parse_double(key, v);
    else if (key == "cache.enabled") cfg.cache_enabled = parse_bool(key, v);
    else if (key == "cache.n") cfg.cache_n = parse_int(key, v);
    else if (key == "swap.mode") cfg.swap_mode = swap_from_string(v);
    else if (key == "swap.simulate") cfg.swap_simulate = parse_bool(key, v);
    else if (key == "swap.bandwidth") cfg.swap_bandwidth = parse_double(key, v);
    else if (key == "swap.latency") cfg.swap_latency = parse_double(key, v);
    else if (key == "swap.mac_rate") cfg.swap_mac_rate = parse_double(key, v);
    else if (key == "chunk.enabled") cfg.chunk_enabled = parse_bool(key, v);
    else if (key == "chunk.eta") cfg.eta = parse_int(key, v);
    else if (key == "chunk.omega") cfg.omega = parse_int(key, v);
    else if (key == "chunk.halo") {
        // HaloMode::exact()/none() reset the pixel count; "fixed" keeps it.
        if (v == "exact") cfg.halo = HaloKind::Exact, cfg.halo_px = 0;
        else if (v == "none") cfg.halo = HaloKind::None, cfg.halo_px = 0;
        else if (v == "fixed") cfg.halo = HaloKind::Fixed;
        else throw_config("chunk.halo must be exact, none or fixed");
    } else if (key == "chunk.halo_px") cfg.halo_px = parse_int(key, v);
    else if (key == "chunk.targets") cfg.targets = split_list(v);
    else if (key == "decode.sliced") cfg.slice_decode = parse_bool(key, v);
    else if (key == "budget.fast_bytes") cfg.budget_fast_bytes = parse_int(key, v);
    else throw_config("unknown config key '" + key + "'");
}

// src/config.cpp:206-224
RunConfig parse_config_text(const std::string& text) {
    RunConfig cfg;
    std::istringstream is(text);
    std::string line;
    int lineno = 0;
    while (std::getline(is, line)) {
        lineno++;
        const auto hash = line.find('#');
        if (hash != std::string::npos) line = line.substr(0, hash);
        line = trim(line);
        if (line.empty()) continue;
        const auto eq = line.find('=');
        if (eq == std::string::npos)
            throw_config("<config>:" + std::to_string(lineno) + ": expected key = value");
        apply_override(cfg, trim(line.substr(0, eq)), trim(line.substr(eq + 1)));
    }
    return cfg;
}

// src/config.cpp:226-264
std::string config_to_text(const RunConfig& c) {
    std::ostringstream os;
    os << "run.frames = " << c.frames << "\n"
       << "run.height = " << c.height << "\n"
       << "run.width = " << c.width << "\n"
       << "run.seed = " << c.seed << "\n"
       << "run.mode = " << c.mode << "\n"
       << "run.out_dir = " << c.out_dir << "\n"
       << "unet.depth = " << c.depth << "\n"
       << "unet.base_channels = " << c.base_channels << "\n"
       << "unet.kernel = " << c.kernel << "\n"
       << "unet.cache_depth = " << c.cache_depth << "\n"
       << "unet.weight_seed = " << c.unet_seed << "\n"
       << "codec.latent_channels = " << c.latent_channels << "\n"
       << "codec.stages = " << c.stages << "\n"
       << "codec.width = " << c.codec_width << "\n"
       << "codec.weight_seed = " << c.codec_seed << "\n"
       << "schedule.train_steps = " << c.train_steps << "\n"
       << "schedule.beta_min = " << c.beta_min << "\n"
       << "schedule.beta_max = " << c.beta_max << "\n"
       << "sampler.kind = " << to_string(c.sampler) << "\n"
       << "sampler.steps = " << c.steps << "\n"
       << "sampler.guidance = " << c.guidance << "\n"
       << "cache.enabled = " << (c.cache_enabled ? "true" : "false") << "\n"
       << "cache.n = " << c.cache_n << "\n"
       << "swap.mode = " << to_string(c.swap_mode) << "\n"
       << "swap.simulate = " << (c.swap_simulate ? "true" : "false") << "\n"
       << "swap.bandwidth = " << c.swap_bandwidth << "\n"
       << "swap.latency = " << c.swap_latency << "\n"
       << "swap.mac_rate = " << c.swap_mac_rate << "\n"
       << "chunk.enabled = " << (c.chunk_enabled ? "true" : "false") << "\n"
       << "chunk.eta = " << c.eta << "\n"
       << "chunk.omega = " << c.omega << "\n"
       << "chunk.halo = " << to_string(c.halo) << "\n"
       << "chunk.halo_px = " << c.halo_px << "\n"
       << "chunk.targets = ";
    for (size_t i = 0; i < c.targets.size(); ++i) os << (i ? "," : "") << c.targets[i];
    os << "\n"
       << "decode.sliced = " << (c.slice_decode ? "true" : "false") << "\n"
       << "budget.fast_bytes = " << c.budget_fast_bytes << "\n";
    return os.str();
}

// ------------------------------------------------------------------ plans
bool StepPlan::has_consumers(int64_t s) const {
    if (!full[s]) return false;
    return s + 1 < size() && !full[s + 1];
}
bool StepPlan::is_last_consumer(int64_t s) const {
    if (full[s]) return false;
    return s + 1 >= size() || full[s + 1];
}
StepPlan plan_steps(int64_t total_steps, int64_t n) {
    if (n < 1) throw_config("cache interval must be >= 1");
    if (total_steps < 1) throw_config("plan_steps needs total_steps >= 1");
    StepPlan p;
    p.full.resize(static_cast<size_t>(total_steps));
    for (int64_t s = 0; s < total_steps; ++s) p.full[s] = (s % n == 0);
    return p;
}

std::vector<Tile> split(int64_t h, int64_t w, int64_t eta, int64_t omega, HaloKind halo_kind,
                        int64_t halo_px, int64_t k, int64_t* halo_out) {
    if (h < 1 || w < 1) throw_shape("all extents must be >= 1");
    if (eta < 1 || omega < 1) throw_config("eta and omega must be >= 1");
    if (h % eta != 0)
        throw_shape("height " + std::to_string(h) + " not divisible by eta " + std::to_string(eta));
    if (w % omega != 0)
        throw_shape("width " + std::to_string(w) + " not divisible by omega " + std::to_string(omega));
    const int64_t r = (k - 1) / 2;  // receptive_radius of {conv} (chunk.cpp:124-143)
    const int64_t halo = halo_kind == HaloKind::Exact ? r : halo_kind == HaloKind::Fixed ? halo_px : 0;
    if (halo_out) *halo_out = halo;
    const int64_t th = h / eta, tw = w / omega;
    std::vector<Tile> tiles;
    for (int64_t i = 0; i < eta; ++i)
        for (int64_t j = 0; j < omega; ++j) {
            Tile t;
            t.core = {i * th, (i + 1) * th, j * tw, (j + 1) * tw};
            t.padded = {std::max<int64_t>(t.core.y0 - halo, 0), std::min(t.core.y1 + halo, h),
                        std::max<int64_t>(t.core.x0 - halo, 0), std::min(t.core.x1 + halo, w)};
            t.out_window = t.core;
            tiles.push_back(t);
        }
    return tiles;
}

// ------------------------------------------------------------------ model
std::vector<BlockPlan> block_plans(const RunConfig& c) {
    std::vector<BlockPlan> plan;
    const int64_t M = c.depth;
    auto ch = [&](int64_t l) { return c.base_channels << l; };
    plan.push_back({"stem", c.in_channels, c.base_channels, false, true, 0});
    plan.push_back({"d0", c.base_channels, c.base_channels, false, true, 0});
    for (int64_t i = 1; i < M; ++i) plan.push_back({"d" + std::to_string(i), ch(i - 1), ch(i), true, true, i});
    plan.push_back({"mid", ch(M - 1), ch(M - 1), true, true, M});
    for (int64_t i = M - 1; i >= 0; --i) {
        const int64_t c_next = (i + 1 == M) ? ch(M - 1) : ch(i + 1);
        plan.push_back({"u" + std::to_string(i), ch(i) + c_next, ch(i), false, true, i});
    }
    plan.push_back({"head", c.base_channels, c.in_channels, false, false, 0});
    return plan;
}

int64_t block_index(const RunConfig& c, const std::string& name) {
    const auto plan = block_plans(c);
    for (size_t i = 0; i < plan.size(); ++i)
        if (plan[i].name == name) return static_cast<int64_t>(i);
    return -1;
}

int64_t flops_estimate(const RunConfig& c, int64_t b, int64_t t, int64_t h, int64_t w, bool cached) {
    const auto plan = block_plans(c);
    const int64_t M = c.depth, m = c.cache_depth;
    std::vector<std::string> names{"stem"};
    const int64_t deepest = cached ? m : M - 1;
    for (int64_t i = 0; i <= deepest; ++i) names.push_back("d" + std::to_string(i));
    if (!cached) names.push_back("mid");
    for (int64_t i = deepest; i >= 0; --i) names.push_back("u" + std::to_string(i));
    names.push_back("head");
    int64_t total = 0;
    for (const auto& n : names) {
        const BlockPlan& bp = plan[static_cast<size_t>(block_index(c, n))];
        total += b * t * bp.c_out * (h >> bp.level) * (w >> bp.level) * c.kernel * c.kernel * bp.c_in;
    }
    return total;
}

int64_t cache_channels(const RunConfig& c) {
    const int64_t m = c.cache_depth;
    return (m + 1 == c.depth) ? (c.base_channels << (c.depth - 1)) : (c.base_channels << (m + 1));
}

// ------------------------------------------------------------------ simulated swap
namespace {

// Virtual transfer engine state for the two cache entries (one per CFG
// branch, cache.cpp:43-60).  Jobs carry their virtual [start, end).
struct SimJob {
    int entry;
    bool to_fast;
    int64_t step, bytes, start, end;
    int id;
};
struct SimEntry {
    bool present = false;
    bool on_fast = true;   // physical tier (Tensor5::tier)
    int heading = -1;      // swap.cpp heading_: -1 none, 0 fast, 1 slow
    int ticket = -1;       // job id of the entry's last ticket; -1 = no-op ticket
};

struct SimEngine {
    const RunConfig& c;
    bool swap_on;
    int64_t now = 0, channel_free = 0;
    std::vector<SimJob> pending;
    std::vector<bool> done;      // per job id
    std::vector<int64_t> ends;   // per job id
    std::vector<SimEvent> tl;
    SimEntry entries[2];

    explicit SimEngine(const RunConfig& cfg) : c(cfg), swap_on(cfg.swap_mode != SwapMode::Off) {}

    void rec(int kind, int64_t step, int64_t bytes, int64_t clock) { tl.push_back({kind, step, bytes, clock}); }
    void macs(int64_t m) {  // mac_hook_tramp, swap.cpp:161-165
        now += static_cast<int64_t>(std::llround(static_cast<double>(m) / c.swap_mac_rate * 1e9));
    }
    int64_t transfer_ns(int64_t bytes) const {  // swap.cpp:149-153
        const double secs = c.swap_latency + static_cast<double>(bytes) / c.swap_bandwidth;
        return static_cast<int64_t>(std::llround(secs * 1e9));
    }
    void finish(const SimJob& j) {  // finish_move, swap.cpp:195-213
        rec(2, j.step, j.bytes, j.start);
        SimEntry& e = entries[j.entry];
        e.on_fast = j.to_fast;
        if (e.heading == (j.to_fast ? 0 : 1)) e.heading = -1;
        rec(3, j.step, j.bytes, j.end);
        done[static_cast<size_t>(j.id)] = true;
    }
    void flush(int64_t up_to) {  // sim_flush, swap.cpp:351-364
        std::stable_sort(pending.begin(), pending.end(),
                         [](const SimJob& a, const SimJob& b) { return a.end < b.end; });
        std::vector<SimJob> kept;
        for (const SimJob& j : pending) {
            if (j.end <= up_to) finish(j);
            else kept.push_back(j);
        }
        pending.swap(kept);
    }
    int submit(int entry, bool to_fast, int64_t step, int64_t bytes) {  // swap.cpp:215-250
        SimJob j{entry, to_fast, step, bytes, std::max(now, channel_free), 0, static_cast<int>(done.size())};
        j.end = j.start + transfer_ns(bytes);
        channel_free = j.end;
        done.push_back(false);
        ends.push_back(j.end);
        entries[entry].heading = to_fast ? 0 : 1;
        if (c.swap_mode == SwapMode::Sync) {
            now = std::max(now, j.end);
            finish(j);
        } else {
            pending.push_back(j);
        }
        return j.id;
    }
    int heading_tier(int entry) const {  // 0 fast, 1 slow
        const SimEntry& e = entries[entry];
        return e.heading >= 0 ? e.heading : (e.on_fast ? 0 : 1);
    }
    void await(int entry, int64_t step_of_ticket) {  // await_ready, swap.cpp:306-316
        const int id = entries[entry].ticket;
        if (id < 0) return;
        rec(4, step_of_ticket, 0, now);
        if (!done[static_cast<size_t>(id)]) {
            now = std::max(now, ends[static_cast<size_t>(id)]);
            flush(now);
        }
        rec(5, step_of_ticket, 0, now);
    }
    void drain() {  // swap.cpp:326-333
        int64_t horizon = now;
        for (const SimJob& j : pending) horizon = std::max(horizon, j.end);
        now = horizon;
        flush(horizon);
    }
};

}  // namespace

namespace {

// Virtual-clock run of the denoising loop; returns the clock after the
// loop's drain (pipeline.cpp:187).  Decode MACs advance the clock after the
// last event and never reach the timeline.
int64_t run_sim(const RunConfig& c, std::vector<SimEvent>* out) {
    c.validate();
    if (!(c.swap_bandwidth > 0) || !(c.swap_mac_rate > 0))
        throw_config("simulated transfer engine needs bandwidth > 0 and a positive MAC rate");
    SimEngine E(c);
    const int64_t S = c.steps, T = c.frames, lh = c.latent_h(), lw = c.latent_w();
    const int64_t M = c.depth, m = c.cache_depth;
    StepPlan plan;
    if (c.cache_enabled) plan = plan_steps(S, c.cache_n);
    else plan.full.assign(static_cast<size_t>(S), true);
    const auto blocks = block_plans(c);
    const bool store_on = E.swap_on;  // CacheStore gets the engine only when swapping
    const int64_t entry_bytes = T * cache_channels(c) * (lh >> m) * (lw >> m) * 4;
    std::vector<int64_t> job_step;

    // One block's convolution calls (unet.cpp:78-123, chunk.cpp:194-223,
    // :274-316): a chunked block runs one conv2d_window per tile core.
    auto block = [&](const std::string& name) {
        const BlockPlan& bp = blocks[static_cast<size_t>(block_index(c, name))];
        const int64_t h = lh >> bp.level, w = lw >> bp.level;
        const int64_t per_px = 2 * T * bp.c_out * c.kernel * c.kernel * bp.c_in;
        const bool chunked = c.chunk_enabled &&
                             std::find(c.targets.begin(), c.targets.end(), name) != c.targets.end();
        if (chunked && (c.eta > 1 || c.omega > 1)) {
            const auto tiles = split(h, w, c.eta, c.omega, c.halo, c.halo_px, c.kernel);
            for (const Tile& t : tiles)
                E.macs(per_px * (t.core.y1 - t.core.y0) * (t.core.x1 - t.core.x0));
        } else {
            E.macs(per_px * h * w);
        }
    };
    auto submit = [&](int entry, bool to_fast, int64_t step) {
        job_step.push_back(step);
        return E.submit(entry, to_fast, step, entry_bytes);
    };
    auto await_entry = [&](int b) {
        const int id = E.entries[b].ticket;
        if (id >= 0) E.await(b, job_step[static_cast<size_t>(id)]);
    };
    auto pending = [&](int b) {
        const int id = E.entries[b].ticket;
        return id >= 0 && !E.done[static_cast<size_t>(id)];
    };
    auto evict_all = [&](int64_t s) {  // cache.cpp:92-98, swap.cpp:284-289
        for (int b = 0; b < 2; ++b) {
            if (!E.entries[b].present) continue;
            if (E.heading_tier(b) == 1) throw_invariant("evict: entry already on (or heading to) the Slow tier");
            E.entries[b].ticket = submit(b, false, s);
        }
    };
    auto prefetch_all = [&](int64_t needed) {  // cache.cpp:100-106, swap.cpp:291-298
        for (int b = 0; b < 2; ++b) {
            if (!E.entries[b].present) continue;
            E.entries[b].ticket = E.heading_tier(b) == 0 ? -1 : submit(b, true, needed);
        }
    };

    for (int64_t s = 0; s < S; ++s) {
        E.rec(0, s, 0, E.now);  // compute_begin (the MAC hook installs here)
        block("stem");
        if (plan.is_full(s)) {
            for (int64_t i = 0; i < M; ++i) block("d" + std::to_string(i));
            block("mid");
            for (int64_t i = M - 1; i >= 0; --i) block("u" + std::to_string(i));
            block("head");
            E.rec(1, s, 0, E.now);
            E.flush(E.now);
            if (c.cache_enabled) {
                for (int b = 0; b < 2; ++b) {  // CacheStore::store, cache.cpp:43-60
                    SimEntry& e = E.entries[b];
                    if (e.present && store_on && pending(b)) await_entry(b);
                    e.present = true;
                    e.on_fast = true;
                    e.ticket = -1;
                }
                if (E.swap_on) {
                    evict_all(s);
                    if (plan.has_consumers(s)) prefetch_all(s + 1);
                }
            }
        } else {
            for (int64_t i = 0; i <= m; ++i) block("d" + std::to_string(i));
            // seam: CacheStore::assemble -> fetch(uncond), fetch(cond) (cache.cpp:62-90)
            if (store_on) {
                for (int b = 0; b < 2; ++b) {
                    await_entry(b);
                    if (!E.entries[b].on_fast) {  // recall, swap.cpp:300-304
                        E.entries[b].ticket = E.heading_tier(b) == 0 ? -1 : submit(b, true, s);
                        await_entry(b);
                    }
                }
                if (plan.is_last_consumer(s)) evict_all(s);
            }
            for (int64_t i = m; i >= 0; --i) block("u" + std::to_string(i));
            block("head");
            E.rec(1, s, 0, E.now);
            E.flush(E.now);
        }
    }
    E.drain();
    // TransferEngine::timeline() returns the log stably sorted by clock
    // (swap.cpp:366-374).
    std::stable_sort(E.tl.begin(), E.tl.end(),
                     [](const SimEvent& a, const SimEvent& b) { return a.clock_ns < b.clock_ns; });
    if (out) *out = std::move(E.tl);
    return E.now;
}

}  // namespace

std::vector<SimEvent> simulate_timeline(const RunConfig& c) {
    std::vector<SimEvent> tl;
    run_sim(c, &tl);
    return tl;
}
int64_t sim_denoise_end_ns(const RunConfig& c) { return run_sim(c, nullptr); }

int64_t sim_makespan_ns(const std::vector<SimEvent>& tl) {
    if (tl.empty()) return 0;
    int64_t lo = tl.front().clock_ns, hi = lo;
    for (const SimEvent& e : tl) {
        lo = std::min(lo, e.clock_ns);
        hi = std::max(hi, e.clock_ns);
    }
    return hi - lo;
}
int64_t sim_stall_ns(const std::vector<SimEvent>& tl) {
    int64_t total = 0, open = 0;
    for (const SimEvent& e : tl) {
        if (e.kind == 4) open = e.clock_ns;
        else if (e.kind == 5) total += e.clock_ns - open;
    }
    return total;
}

// ------------------------------------------------------------------ rng
uint64_t splitmix64_at(uint64_t seed, uint64_t counter) {
    uint64_t z = seed + (counter + 1) * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
uint64_t derive_seed(uint64_t seed, uint64_t stream) {
    return splitmix64_at(seed, 0x5ca1ab1e00000000ull ^ stream);
}
static double uniform_unit(uint64_t seed, uint64_t counter) {
    return static_cast<double>((splitmix64_at(seed, counter) >> 11) + 1) * 0x1.0p-53;
}
float normal_at(uint64_t seed, uint64_t i) {
    const uint64_t pair = i / 2;
    const double u1 = uniform_unit(seed, 2 * pair);
    const double u2 = uniform_unit(seed, 2 * pair + 1);
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 6.283185307179586476925286766559 * u2;
    return static_cast<float>(i % 2 == 0 ? r * std::cos(a) : r * std::sin(a));
}
void randn(uint64_t seed, int64_t n, float* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = normal_at(seed, static_cast<uint64_t>(i));
}

// ------------------------------------------------------------------ weights
UNetWeights init_unet(const RunConfig& c) {
    UNetWeights w;
    uint64_t stream = 0;
    for (const BlockPlan& bp : block_plans(c)) {
        Bank b;
        b.c_in = bp.c_in;
        b.c_out = bp.c_out;
        b.k = c.kernel;
        const int64_t fan_in = c.kernel * c.kernel * bp.c_in;
        const float gain = 1.0f / std::sqrt(static_cast<float>(fan_in));
        const uint64_t st = derive_seed(c.unet_seed, stream++);
        b.taps.resize(static_cast<size_t>(bp.c_out * fan_in));
        for (size_t i = 0; i < b.taps.size(); ++i) b.taps[i] = gain * normal_at(st, i);
        const uint64_t sb = derive_seed(c.unet_seed, stream++);
        b.bias.resize(static_cast<size_t>(bp.c_out));
        for (size_t i = 0; i < b.bias.size(); ++i) b.bias[i] = 0.02f * normal_at(sb, i);
        const uint64_t sc = derive_seed(c.unet_seed, stream++);
        std::vector<float> cs(8), co(8);
        for (int k = 0; k < 8; ++k) {
            cs[k] = 0.02f * normal_at(sc, static_cast<uint64_t>(k));
            co[k] = 0.02f * normal_at(sc, static_cast<uint64_t>(8 + k));
        }
        w.banks.push_back(std::move(b));
        w.cs.push_back(std::move(cs));
        w.co.push_back(std::move(co));
    }
    return w;
}

static Bank draw_bank(int64_t c_in, int64_t c_out, int64_t k, uint64_t seed) {  // codec.cpp:14-30
    Bank b;
    b.c_in = c_in;
    b.c_out = c_out;
    b.k = k;
    const int64_t fan_in = k * k * c_in;
    const float gain = 1.0f / std::sqrt(static_cast<float>(fan_in));
    b.taps.resize(static_cast<size_t>(c_out * fan_in));
    for (size_t i = 0; i < b.taps.size(); ++i) b.taps[i] = gain * normal_at(seed, i);
    const uint64_t sb = derive_seed(seed, 0xb1a5);
    b.bias.resize(static_cast<size_t>(c_out));
    for (size_t i = 0; i < b.bias.size(); ++i) b.bias[i] = 0.02f * normal_at(sb, i);
    return b;
}

CodecWeights init_codec(const RunConfig& c) {
    CodecWeights w;
    uint64_t stream = 0;
    auto seed = [&] { return derive_seed(c.codec_seed, stream++); };
    w.enc.push_back(draw_bank(c.image_channels, c.codec_width, 3, seed()));
    for (int64_t i = 1; i <= c.stages; ++i)
        w.enc.push_back(draw_bank(c.codec_width, i == c.stages ? c.latent_channels : c.codec_width, 3, seed()));
    w.dec.push_back(draw_bank(c.latent_channels, c.codec_width, 3, seed()));
    for (int64_t i = 1; i <= c.stages; ++i)
        w.dec.push_back(draw_bank(c.codec_width, i == c.stages ? c.image_channels : c.codec_width, 3, seed()));
    return w;
}

void block_conditioning(const UNetWeights& w, int64_t block, int64_t timestep, float* s, float* o) {
    float e[8];
    for (int k = 0; k < 4; ++k) {
        const double freq = std::pow(10000.0, -static_cast<double>(k) / 4);
        e[2 * k] = static_cast<float>(std::sin(static_cast<double>(timestep) * freq));
        e[2 * k + 1] = static_cast<float>(std::cos(static_cast<double>(timestep) * freq));
    }
    float ss = 1.0f, oo = 0.0f;
    for (int k = 0; k < 8; ++k) {
        ss += w.cs[block][k] * e[k];
        oo += w.co[block][k] * e[k];
    }
    *s = ss;
    *o = oo;
}

// ------------------------------------------------------------------ schedule
Schedule make_schedule(const RunConfig& c) {
    const int64_t T = c.train_steps, S = c.steps;
    if (T < 1) throw_config("train_steps must be >= 1");
    if (!(c.beta_min > 0.0) || !(c.beta_min <= c.beta_max) || !(c.beta_max < 1.0))
        throw_config("need 0 < beta_min <= beta_max < 1");
    std::vector<double> betas(static_cast<size_t>(T)), abar(static_cast<size_t>(T));
    if (T == 1) betas[0] = c.beta_min;
    else {  // Eigen 3.4 LinSpaced (linspaced_op_impl, non-integer scalar)
        const double step = (c.beta_max - c.beta_min) / static_cast<double>(T - 1);
        const bool flip = std::fabs(c.beta_max) < std::fabs(c.beta_min);
        for (int64_t i = 0; i < T; ++i) {
            if (flip) betas[i] = i == 0 ? c.beta_min : c.beta_max - static_cast<double>(T - 1 - i) * step;
            else betas[i] = i == T - 1 ? c.beta_max : c.beta_min + static_cast<double>(i) * step;
        }
    }
    double prod = 1.0;
    for (int64_t i = 0; i < T; ++i) {
        prod *= 1.0 - betas[i];
        abar[i] = prod;
    }
    if (S < 1 || S > T) throw_config("inference steps must lie in [1, train_steps]");
    Schedule s;
    s.betas.resize(S);
    s.alphas.resize(S);
    s.abar.resize(S);
    s.src.resize(S);
    if (S == T) {
        for (int64_t i = 0; i < T; ++i) {
            s.betas[i] = betas[i];
            s.alphas[i] = 1.0 - betas[i];
            s.abar[i] = abar[i];
            s.src[i] = i;
        }
        return s;
    }
    double prev = 1.0;
    for (int64_t i = 0; i < S; ++i) {
        const int64_t src = S == 1 ? T - 1
                                   : static_cast<int64_t>(std::llround(static_cast<double>(i) *
                                                                       static_cast<double>(T - 1) /
                                                                       static_cast<double>(S - 1)));
        s.src[i] = src;
        s.abar[i] = abar[src];
        s.alphas[i] = s.abar[i] / prev;
        s.betas[i] = 1.0 - s.alphas[i];
        prev = s.abar[i];
    }
    return s;
}

StepCoeffs step_coeffs_at(Sampler kind, const Schedule& sc, int64_t j, uint64_t noise_seed) {
    if (j < 0 || j >= static_cast<int64_t>(sc.betas.size()))  // check_t, sampler.cpp:78-83
        throw_config("reverse_step: t=" + std::to_string(j) + " outside [0, " +
                     std::to_string(sc.betas.size()) + ")");
    StepCoeffs k;
    switch (kind) {
        case Sampler::Euler: {  // sampler.cpp:119-125
            const double drift = 2.0 - std::sqrt(sc.alphas[j]);
            const double diff = -0.5 * sc.betas[j] / std::sqrt(1.0 - sc.abar[j]);
            k.a = static_cast<float>(drift);
            k.b = static_cast<float>(diff);
            break;
        }
        case Sampler::Ddim: {  // sampler.cpp:108-117
            const double ab = sc.abar[j];
            const double abp = j > 0 ? sc.abar[j - 1] : 1.0;
            const double a = std::sqrt(abp / ab);
            const double b = std::sqrt(1.0 - abp) - a * std::sqrt(1.0 - ab);
            k.a = static_cast<float>(a);
            k.b = static_cast<float>(b);
            break;
        }
        case Sampler::Ancestral: {  // sampler.cpp:95-106
            const double alpha = sc.alphas[j], ab = sc.abar[j];
            const double mean_x = 1.0 / std::sqrt(alpha);
            const double mean_e = -mean_x * (1.0 - alpha) / std::sqrt(1.0 - ab);
            k.a = static_cast<float>(mean_x);
            k.b = static_cast<float>(mean_e);
            if (j != 0) {
                k.has_noise = true;
                k.noise = static_cast<float>(std::sqrt(sc.betas[j]));
                k.noise_seed = noise_seed;
            }
            break;
        }
    }
    return k;
}

StepCoeffs step_coeffs(const RunConfig& c, const Schedule& sc, int64_t s) {
    // step s of the loop runs schedule index S-1-s (pipeline.cpp:160-185)
    return step_coeffs_at(c.sampler, sc, c.steps - 1 - s, derive_seed(c.seed, 0x1000 + static_cast<uint64_t>(s)));
}

// ------------------------------------------------------------------ arena plan
ArenaPlan plan_arena(const RunConfig& cfg) {
    auto al = [](int64_t b) { return (b + 255) / 256 * 256; };
    auto r64 = [](int64_t v) { return static_cast<int>((v + 63) / 64 * 64); };
    const int n = static_cast<int>(2 * cfg.frames);
    const int M = static_cast<int>(cfg.depth), m = static_cast<int>(cfg.cache_depth);
    const int lh = static_cast<int>(cfg.latent_h()), lw = static_cast<int>(cfg.latent_w());
    auto ch = [&](int l) { return static_cast<int>(cfg.base_channels << l); };
    const int kp = r64(cfg.in_channels * cfg.kernel * cfg.kernel);
    ArenaPlan plan;
    std::vector<ArenaBuf>& B = plan.bufs;
    auto def = [&](const std::string& name, int h, int w, int c, int cs) {
        B.push_back({name, n, h, w, c, cs, al(static_cast<int64_t>(n) * h * w * cs * 2), 1 << 30, -1, 0});
    };
    if (cfg.cache_enabled) {
        const int cc = static_cast<int>(cache_channels(cfg));
        def("cache", lh >> (m + 1), lw >> (m + 1), cc, r64(cc));
    }
    def("patch", lh, lw, kp, kp);
    def("stem", lh, lw, ch(0), r64(ch(0)));
    for (int i = 0; i < M; ++i) {
        const int h = lh >> i, w = lw >> i;
        def("D" + std::to_string(i), h, w, ch(i), r64(ch(i)));
        if (i >= 1) def("P" + std::to_string(i), h, w, ch(i - 1), r64(ch(i - 1)));
        if (!(cfg.cache_enabled && i == m + 1)) def("U" + std::to_string(i), h, w, ch(i), r64(ch(i)));
        const int cu = (i == M - 1) ? ch(M - 1) : ch(i + 1);
        if (cfg.kernel != 3 || (cfg.chunk_enabled && cfg.halo != HaloKind::Exact))
            def("UP" + std::to_string(i), h, w, cu, r64(cu));
    }
    def("P" + std::to_string(M), lh >> M, lw >> M, ch(M - 1), r64(ch(M - 1)));
    if (!(cfg.cache_enabled && m + 1 == M)) def("mid", lh >> M, lw >> M, ch(M - 1), r64(ch(M - 1)));
    auto use = [&](const std::string& name, int t) {
        for (ArenaBuf& b : B)
            if (b.name == name) {
                b.t0 = std::min(b.t0, t);
                b.t1 = std::max(b.t1, t);
            }
    };
    auto U_at = [&](int l) -> std::string {
        if (cfg.cache_enabled && l == m + 1) return "cache";
        return l == M ? "mid" : "U" + std::to_string(l);
    };
    auto has = [&](const std::string& name) {
        for (const ArenaBuf& b : B)
            if (b.name == name) return true;
        return false;
    };
    int t = 0;
    use("patch", t++);
    use("patch", t), use("stem", t++);
    use("stem", t), use("D0", t++);
    for (int i = 1; i <= M; ++i) {
        use("D" + std::to_string(i - 1), t), use("P" + std::to_string(i), t++);  // down2
        use("P" + std::to_string(i), t), use(i == M ? U_at(M) : "D" + std::to_string(i), t++);
    }
    for (int i = M - 1; i >= 0; --i) {
        const std::string up = "UP" + std::to_string(i);
        if (has(up)) use(U_at(i + 1), t), use(up, t++);
        use("D" + std::to_string(i), t), use(U_at(i + 1), t), use(up, t), use(U_at(i), t++);
    }
    use("U0", t++);  // head
    plan.steps_ops = t;
    // the cache lives across steps at [0, cache)
    int64_t base = 0;
    if (cfg.cache_enabled) {
        B[0].t0 = 0, B[0].t1 = t;
        B[0].off = 0;
        base = plan.cache_bytes = B[0].bytes;
    }
    std::vector<size_t> order;
    for (size_t i = 0; i < B.size(); ++i)
        if (B[i].name != "cache") order.push_back(i);
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return B[a].bytes > B[b].bytes; });
    std::vector<size_t> placed;
    int64_t top = base;
    for (size_t k : order) {
        ArenaBuf& L = B[k];
        if (L.t1 < 0) continue;  // not used in this configuration
        int64_t o = base;
        for (bool moved = true; moved;) {
            moved = false;
            for (size_t j : placed) {
                const ArenaBuf& P = B[j];
                const bool live_both = !(P.t1 < L.t0 || L.t1 < P.t0);
                const bool overlap = !(P.off + P.bytes <= o || o + L.bytes <= P.off);
                if (live_both && overlap) {
                    o = P.off + P.bytes;
                    moved = true;
                }
            }
        }
        L.off = o;
        placed.push_back(k);
        top = std::max(top, o + L.bytes);
    }
    plan.act_end = top;
    return plan;
}

// ------------------------------------------------------------------ sharded decode
ShardSpan shard_frames(int64_t T, int world, int rank) {
    if (world < 1 || rank < 0 || rank >= world) throw_config("bad world/rank");
    if (T < 0) throw_shape("negative frame count");
    const int64_t base = T / world, extra = T % world;
    ShardSpan s;
    s.first = rank * base + std::min<int64_t>(rank, extra);
    s.count = base + (rank < extra ? 1 : 0);
    return s;
}

std::vector<GatherRow> gather_plan(int64_t T, int world, int64_t slice) {
    if (slice < 1) throw_config("decode slice must be >= 1");
    std::vector<GatherRow> rows;
    for (int64_t round = 0;; ++round) {
        bool any = false;
        for (int r = 0; r < world; ++r) {
            const ShardSpan sp = shard_frames(T, world, r);
            const int64_t g0 = round * slice;
            if (g0 >= sp.count) continue;
            any = true;
            rows.push_back({round, r, sp.first + g0, std::min(slice, sp.count - g0)});
        }
        if (!any) break;
    }
    return rows;
}

}  // namespace lc
