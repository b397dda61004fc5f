// Host-side model of the LightCache path: run configuration (same keys,
// grammar and validation as the reference), step plans, tile grids,
// schedules and deterministic weight initialisation.  Pure integer/double
// logic; bit-exact with the reference (pinned by tests/test_host.py).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace lc {

// ------------------------------------------------------------------ errors
// Status codes shared with the C-ABI; they equal the reference CLI exit
// codes for the corresponding exception (proj/tools/main.cpp:157-169,
// proj/include/stagecache/common.hpp:33-57).
enum Status : int {
    kOk = 0,
    kShapeError = 1,      // ShapeError / other std::exception -> exit 1
    kConfigError = 2,     // ConfigError
    kBudgetError = 3,     // BudgetError
    kInvariantError = 4,  // InvariantError
    kCudaError = 5,       // device failure (no reference analogue)
};

struct LcError : std::runtime_error {
    int code;
    int stage = -1;  // BudgetError: the stage it was raised in (BudgetError::stage, common.hpp:43-46)
    LcError(int c, const std::string& m, int st = -1) : std::runtime_error(m), code(c), stage(st) {}
};
[[noreturn]] inline void throw_config(const std::string& m) { throw LcError(kConfigError, m); }
[[noreturn]] inline void throw_shape(const std::string& m) { throw LcError(kShapeError, m); }
[[noreturn]] inline void throw_invariant(const std::string& m) { throw LcError(kInvariantError, m); }

// ------------------------------------------------------------------ config
enum class Sampler { Ancestral = 0, Ddim = 1, Euler = 2 };
enum class SwapMode { Off = 0, Sync = 1, Async = 2 };
enum class HaloKind { Exact = 0, Fixed = 1, None = 2 };

// Mirror of stagecache::RunConfig (proj/include/stagecache/config.hpp:16-71)
// with default_config() values (proj/src/config.cpp:90-98).
struct RunConfig {
    int64_t frames = 8, height = 64, width = 64;
    uint64_t seed = 42;
    std::string mode = "text";
    std::string out_dir = "out";
    // unet.*
    int64_t depth = 3, base_channels = 8, kernel = 3, cache_depth = 0, in_channels = 4;
    uint64_t unet_seed = 1234;
    // codec.*
    int64_t latent_channels = 4, stages = 2, image_channels = 3, codec_width = 8;
    uint64_t codec_seed = 77;
    // schedule.*
    int64_t train_steps = 50;
    double beta_min = 0.002, beta_max = 0.25;
    // sampler.*
    Sampler sampler = Sampler::Euler;
    int64_t steps = 25;
    double guidance = 1.5;
    // cache.*
    bool cache_enabled = true;
    int64_t cache_n = 2;
    // swap.*
    SwapMode swap_mode = SwapMode::Async;
    bool swap_simulate = false;
    double swap_bandwidth = 4e9, swap_latency = 20e-6, swap_mac_rate = 5e7;
    // chunk.*
    bool chunk_enabled = true;
    int64_t eta = 2, omega = 2;
    HaloKind halo = HaloKind::Exact;
    int64_t halo_px = 0;
    std::vector<std::string> targets{"u0"};
    // decode.*
    bool slice_decode = true;
    // budget.*
    int64_t budget_fast_bytes = 0;

    int64_t scale() const { return int64_t(1) << stages; }
    int64_t latent_h() const { return height / scale(); }
    int64_t latent_w() const { return width / scale(); }
    void validate() const;         // config.cpp:100-141
    RunConfig baseline() const;    // config.cpp:148-156
};

// apply_override (config.cpp:158-204): identical key set and parse errors.
void apply_override(RunConfig& cfg, const std::string& key, const std::string& value);
// load_config_file grammar (config.cpp:206-224) on an in-memory text.
RunConfig parse_config_text(const std::string& text);
std::string config_to_text(const RunConfig& cfg);  // config.cpp:226-264

// ------------------------------------------------------------------ plans
// plan_steps (proj/src/cache.cpp:25-33); kinds: true = Full.
struct StepPlan {
    std::vector<bool> full;
    bool is_full(int64_t s) const { return full[s]; }
    int64_t size() const { return static_cast<int64_t>(full.size()); }
    bool has_consumers(int64_t s) const;     // cache.cpp:19-23
    bool is_last_consumer(int64_t s) const;  // cache.cpp:15-18
};
StepPlan plan_steps(int64_t total_steps, int64_t interval_n);

struct Region {
    int64_t y0 = 0, y1 = 0, x0 = 0, x1 = 0;
    bool operator==(const Region&) const = default;
};
struct Tile {
    Region core, padded, out_window;
};
// split (proj/src/chunk.cpp:145-181) for a single-conv chain of kernel k.
std::vector<Tile> split(int64_t h, int64_t w, int64_t eta, int64_t omega, HaloKind halo,
                        int64_t halo_px, int64_t k, int64_t* halo_out = nullptr);

// ------------------------------------------------------------------ model
struct BlockPlan {
    std::string name;
    int64_t c_in, c_out;
    bool down_before, has_silu;
    int64_t level;
};
// block_plans (proj/src/unet.cpp:33-50)
std::vector<BlockPlan> block_plans(const RunConfig& cfg);
int64_t block_index(const RunConfig& cfg, const std::string& name);

// flops_estimate (unet.cpp:287-300), MACs for model input (b,t,c,h,w).
int64_t flops_estimate(const RunConfig& cfg, int64_t b, int64_t t, int64_t h, int64_t w,
                       bool cached);
// cache_feature_shape channel count at the seam (unet.cpp:302-309).
int64_t cache_channels(const RunConfig& cfg);

// ------------------------------------------------------------------ simulated swap
// One timeline event (swap.hpp:16-30): kind 0 compute_start, 1 compute_end,
// 2 xfer_start, 3 xfer_end, 4 await_start, 5 await_end; clock in virtual ns.
struct SimEvent {
    int kind;
    int64_t step, bytes, clock_ns;
};
// The reference's simulated transfer engine (swap.simulate = true,
// proj/src/swap.cpp:141-364) driven by the denoising loop of run_pipeline
// (pipeline.cpp:119-207) and the cache store (cache.cpp:43-122): a virtual
// nanosecond clock advanced by every convolution call's MAC count at
// swap.mac_rate (tensor.cpp:21-24, :194), one transfer channel of
// latency + bytes / bandwidth per job.  Returns the event list in the
// reference's recording order; bit-exact with it (tests/test_simulate.py).
std::vector<SimEvent> simulate_timeline(const RunConfig& cfg);
int64_t sim_makespan_ns(const std::vector<SimEvent>& tl);  // swap.cpp:59-68
int64_t sim_stall_ns(const std::vector<SimEvent>& tl);     // swap.cpp:70-79
// Virtual clock after the denoising loop's drain (pipeline.cpp:187).
int64_t sim_denoise_end_ns(const RunConfig& cfg);

// ------------------------------------------------------------------ arena plan
// The denoise activations' lifetimes within one full step (whole-batch op
// order: patch, stem, d0, [down2, d_i]..., down2, mid, [up2, u_i]...,
// head) and their first-fit packing by lifetime (Engine::alloc_activations
// lays the arena out from this plan).  Buffers: "patch", "stem", "D<i>",
// "P<i>", "U<i>", "UP<i>", "mid"; the cache entries ("cache", U_{m+1}) keep
// [0, cache_bytes) for the whole run.  Sizes are fp16 NHWC with 64-channel
// strides, 256-byte aligned; t0/t1 the first write and last read.
struct ArenaBuf {
    std::string name;
    int n, h, w, c, cs;
    int64_t bytes;
    int t0, t1;
    int64_t off;
};
struct ArenaPlan {
    std::vector<ArenaBuf> bufs;  // "cache" first when caching is on
    int64_t cache_bytes = 0;     // [0, cache_bytes): the entries
    int64_t act_end = 0;         // end of the packed activations
    int steps_ops = 0;           // op slots of a full step (lifetime axis)
};
ArenaPlan plan_arena(const RunConfig& cfg);

// ------------------------------------------------------------------ sharded decode
// Multi-GPU sliced decode (the unit of work is
// decode_sliced, proj/src/codec.cpp:126-145): rank r of g owns a contiguous
// frame block, balanced (the first T % g ranks take one frame more: 25 on 8
// GPUs = 4,3,3,3,3,3,3,3), decoded in slices of `slice` frames.  Gather
// round i moves the i-th slice of every rank that has one to rank 0; the
// GPU engine executes the rounds with NCCL and the CPU tests with gloo, so
// both consume this one plan.
struct ShardSpan {
    int64_t first = 0, count = 0;
};
ShardSpan shard_frames(int64_t T, int world, int rank);
struct GatherRow {
    int64_t round, rank, first, count;  // frames [first, first+count) of `rank`
};
std::vector<GatherRow> gather_plan(int64_t T, int world, int64_t slice);

// ------------------------------------------------------------------ rng
uint64_t splitmix64_at(uint64_t seed, uint64_t counter);  // rng.hpp:11-16
uint64_t derive_seed(uint64_t seed, uint64_t stream);     // rng.hpp:24-26
float normal_at(uint64_t seed, uint64_t i);               // rng.hpp:34-41
void randn(uint64_t seed, int64_t n, float* out);         // tensor.cpp:142-149

// ------------------------------------------------------------------ weights
struct Bank {
    int64_t c_in = 0, c_out = 0, k = 0;
    std::vector<float> taps;  // [c_out][c_in][k][k]
    std::vector<float> bias;  // [c_out]
};
struct UNetWeights {
    std::vector<Bank> banks;                  // block_plans order
    std::vector<std::vector<float>> cs, co;   // [block][8]
};
UNetWeights init_unet(const RunConfig& cfg);   // unet.cpp:153-186
struct CodecWeights {
    std::vector<Bank> enc, dec;
};
CodecWeights init_codec(const RunConfig& cfg);  // codec.cpp:45-62

// Per-block conditioning scalars for a timestep (unet.cpp:14-22, :67-74).
void block_conditioning(const UNetWeights& w, int64_t block, int64_t timestep, float* s, float* o);

// ------------------------------------------------------------------ schedule
struct Schedule {
    std::vector<double> betas, alphas, abar;
    std::vector<int64_t> src;  // source timestep per index
};
Schedule make_schedule(const RunConfig& cfg);  // sampler.cpp:26-75

// Per-step scalar coefficients of the sampler update (sampler.cpp:95-133),
// already cast to float exactly as the reference casts them.
struct StepCoeffs {
    float a = 0, b = 0;      // x' = a*x + b*eps  (mean for ancestral)
    float noise = 0;         // ancestral sqrt(beta) (0: no noise)
    bool has_noise = false;
    uint64_t noise_seed = 0;
};
StepCoeffs step_coeffs(const RunConfig& cfg, const Schedule& sc, int64_t s);
// The same at schedule index t (the reference's reverse_step_* t argument),
// ancestral noise drawn from noise_seed; ConfigError outside [0, steps).
StepCoeffs step_coeffs_at(Sampler kind, const Schedule& sc, int64_t t, uint64_t noise_seed);

}  // namespace lc
