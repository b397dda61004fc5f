// proj/src/pipeline_b200.cpp -- the binding a stagecache maintainer adds to
// the reference tree (INTEGRATION.md section 1 embeds this file verbatim).
// Drop-in for run_pipeline (proj/src/pipeline.cpp:64): the same RunConfig
// in, a fully typed RunResult out (video, StageWall, StageReport, timeline,
// MAC counters, cache bytes, makespan / stall), the same exception types.
#include <cstring>
#include <memory>

#include "lightcache.hpp"
#include "stagecache/pipeline.hpp"

namespace stagecache {

RunResult run_pipeline_b200(const RunConfig& cfg) {
    cfg.validate();
    static stagecache_b200::Context gpu(0);  // weights / buffers cached per config
    stagecache_b200::RunResult g;
    try {
        g = gpu.run_pipeline(config_to_text(cfg));
    } catch (const stagecache_b200::ConfigError& e) {
        throw ConfigError(e.what());
    } catch (const stagecache_b200::BudgetError& e) {
        throw BudgetError(static_cast<StageTag>(e.stage), e.what());
    } catch (const stagecache_b200::InvariantError& e) {
        throw InvariantError(e.what());
    } catch (const stagecache_b200::ShapeError& e) {
        throw ShapeError(e.what());
    }
    RunResult res;
    res.config = cfg;
    res.ledger = std::make_shared<MemLedger>();
    {
        LedgerScope scope(*res.ledger);  // the video is the run's one live allocation
        res.video = Tensor5::uninit({1, cfg.frames, cfg.codec.image_channels, cfg.height, cfg.width});
    }
    std::memcpy(res.video.data(), g.video.data(), static_cast<size_t>(res.video.bytes()));
    res.wall = {g.wall.setup, g.wall.encode, g.wall.denoise, g.wall.decode, g.wall.total};
    for (size_t s = 0; s < 4; ++s) {
        res.mem.peak[s] = g.mem.peak[s];  // [stage][tier]: HBM / pinned host bytes
        res.mem.events_per_stage[s] = g.mem.events_per_stage[s];
    }
    res.mem.current = g.mem.current;
    res.mem.event_count = g.mem.event_count;
    for (const auto& e : g.timeline)
        res.timeline.push_back({static_cast<TimelineEventKind>(e.kind), e.step, e.bytes, e.clock_ns});
    res.denoiser_macs = g.denoiser_macs;
    res.macs_per_full_step = g.macs_per_full_step;
    res.macs_per_cached_step = g.macs_per_cached_step;
    res.full_steps = g.full_steps;
    res.cached_steps = g.cached_steps;
    res.cache_bytes_planned = g.cache_bytes_planned;
    res.makespan_s = g.makespan_s;
    res.stall_s = g.stall_s;
    res.simulated = g.simulated;
    return res;
}

}  // namespace stagecache
