// GPU execution engine for the LightCache path: packed weights, device
// buffers, streams, the denoise loop with the feature cache and its
// asynchronous host swap, chunked execution and sliced decode.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <array>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "conv_tc.cuh"
#include "host.hpp"
#include "kernels.cuh"
#include "subpix_tc.cuh"

namespace lc {

void cuda_check(cudaError_t e, const char* what);
#define LC_CUDA(x) ::lc::cuda_check((x), #x)

// ---------------------------------------------------------------- ledger
// Physical memory accounting per (stage, tier): Fast = HBM bytes allocated
// by the engine, Slow = pinned host bytes (cf. MemLedger,
// proj/include/stagecache/ledger.hpp:69-146; peaks per stage, fast budget).
enum Stage { kSetup = 0, kEncode = 1, kDenoise = 2, kDecode = 3 };
// Memory ledger of the engine (the reference's MemLedger,
// proj/src/ledger.cpp:35-123): every HBM (fast) and pinned-host (slow)
// allocation and free is an event with an id, the stage it happened in and
// a clock; stage entries are events too.  Besides the persistent
// allocations (weights, latents, video: real cudaMalloc / cudaHostAlloc),
// the per-run working sets live in ONE device arena (Engine::alloc_arena)
// and are logged as regions with lifetimes: the denoise activations and the
// feature-cache entries for the denoise stage, the decode (and encode)
// workspace for its stage, each alloc / free at the stage boundary, and the
// swap's tier moves of the cache entries (move_start adds the destination
// tier's bytes -- double residency -- move_end releases the source,
// ledger.cpp:93-123).  The arena is sized to the peak of those lifetimes, so
// the ledger's fast-tier peak is the physical HBM the engine holds.
// Peaks per (stage, tier), the fast-tier budget (BudgetError naming the
// stage) and the CSV / JSON writers' content (proj/src/ledger.cpp:200-242)
// come from it.
struct LedgerEvent {
    int kind;  // 0 alloc, 1 free, 2 move_start, 3 move_end, 4 stage_enter (ledger.hpp MemEventKind)
    int64_t bytes;
    int tier;  // 0 fast (HBM), 1 slow (pinned host)
    int stage;
    uint64_t alloc_id, seq;
    double clock;  // seconds since the ledger was created
};
struct Ledger {
    int stage = kSetup;
    int64_t occ[2] = {0, 0};
    int64_t peak[4][2] = {};
    int64_t events_per_stage[4] = {};
    int64_t budget_fast = 0;
    std::vector<LedgerEvent> events;
    uint64_t next_id = 1;
    double t0 = now();
    // swap.simulate: events carry the simulated engine's virtual clock
    // (pipeline.cpp:79-82) at the enclosing step boundary; < 0 = monotonic.
    double virt = -1;
    struct Live {
        int64_t bytes;
        int tier;
        bool moving;
        int dst;
    };
    std::map<uint64_t, Live> live;  // arena regions (persistent buffers are not tracked here)
    static double now();
    void enter(int s);
    uint64_t alloc(int tier, int64_t bytes);
    void free(int tier, int64_t bytes, uint64_t id);
    void record(int kind, int tier, int64_t bytes, uint64_t id);
    void check_budget(int64_t extra) const;
    // arena regions with lifetimes (see above)
    uint64_t region_alloc(int tier, int64_t bytes);
    void region_free(uint64_t id);
    void move_start(uint64_t id, int dst);
    void move_end(uint64_t id);
    int region_tier(uint64_t id) const;
};

struct DevBuf {
    void* p = nullptr;
    int64_t bytes = 0;
    Ledger* ledger = nullptr;
    int tier = 0;  // 0 device, 1 pinned host
    uint64_t id = 0;  // ledger allocation id
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept { *this = std::move(o); }
    DevBuf& operator=(DevBuf&& o) noexcept;
    ~DevBuf() { reset(); }
    void reset();
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};
DevBuf dev_alloc(Ledger* l, int64_t bytes, bool zero = true);
// Host -> device copy that has LANDED when it returns.  A legacy-stream
// cudaMemcpy from pageable memory may return before its DMA completes, and
// the engine's kernels run on non-blocking streams that do not order after
// the legacy stream, so every setup upload goes through this.
void h2d_blocking(void* dst, const void* src, size_t bytes);
DevBuf host_alloc(Ledger* l, int64_t bytes);

// fp16 NHWC activation view.
struct Act {
    __half* p = nullptr;
    int n = 0, h = 0, w = 0, cs = 0, c = 0;
    int64_t elems() const { return static_cast<int64_t>(n) * h * w * cs; }
};

// ------------------------------------------------------- tensor-core layer
// One conv bank packed for conv_tc: fp16 weights [P][n_pad][K], bias, and
// the conditioning-shift border tables.  mode 0: regular taps (segments =
// channel split of c_in); mode 1: sub-pixel nearest-upsample fusion (k=3):
// seg0 = full-res skip read with stride 2 (absent when c_skip == 0), seg1 =
// low-res operand with merged 2x2 taps; P = 4 parity classes.
struct TcLayer {
    int mode = 0;
    int k = 3, r = 1;
    int c_out = 0, n_pad = 0, BN = 0, P = 1, k_total = 0;
    int nseg = 0;
    int seg_c[2] = {0, 0};      // real channels per segment
    int seg_cpad[2] = {0, 0};   // channels read per segment (multiple of 64)
    int seg_ntaps[2] = {0, 0};
    int seg_kbase[2] = {0, 0};
    int seg_m[2] = {1, 1};      // lattice->source multiplier
    int8_t ox[2][4][kMaxTaps] = {}, oy[2][4][kMaxTaps] = {};
    int rc = 1;                 // class radius in lattice units
    float wscale = 1.0f;        // weights stored as fp16(w * wscale)
    DevBuf w, bias, corr;
};
// c_split: channels of segment 0 (the skip operand for up blocks; c_in for
// a single-source conv).
// m_tiles_hint: M tiles per parity class of the launches this layer will
// serve (0 = unknown) -- steers the choice of BN (see pack_tc_layer).
std::unique_ptr<TcLayer> pack_tc_layer(Ledger* l, const Bank& b, int c_split, int mode, int m_tiles_hint = 0);
int est_m_tiles(int n, int h, int w);

// Thin (CUDA-core) layer: fp32 weights on device.
struct ThinLayer {
    int c_in = 0, c_out = 0, k = 3;
    DevBuf w, bias;
};
std::unique_ptr<ThinLayer> pack_thin_layer(Ledger* l, const Bank& b);

// Optional per-launch timing of the tensor-core conv (bench roofline):
// CUDA events on the launching stream around each launch.
struct ConvProfiler {
    struct Rec {
        double alg_flops = 0, exec_flops = 0;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        std::string desc;  // shape / schedule of the launch (per-layer report)
    };
    std::vector<Rec> recs;
    void clear();
    // totals: launches, ms, algorithmic FLOPs, executed MMA FLOPs
    void summarize(int64_t* n, double* ms, double* alg, double* exec) const;
    std::string records_json() const;  // [{"ms","alg_flops","exec_flops","desc"}, ...]
};
ConvProfiler* conv_profiler();
void set_conv_profiler(ConvProfiler* p);

// Launch one tensor-core conv (all tiles of one region).  `srcs` are the
// segment operands in source coordinates; `win` the valid window of the
// operand of segment 0 in ITS coordinates ({0,h,0,w} = whole image) and the
// output region in output-pixel coordinates.
// out32 non-null: write fp32 NCHW (out.n, c_out, out.h, out.w) instead of
// fp16 NHWC into out.p.
// nhwc32 (with out32): raw fp32 NHWC s*conv(x) into out32 with the channel
// stride out.cs (tap-to-N GEMMs, no offsets / activation); planar: the same
// values channel-planar [out.cs][out.n][out.h][out.w] (coalesced gathers).
void run_tc_conv(const TcLayer& L, const Act* srcs, const Act& out, const Window& win, float s,
                 float o, bool silu, cudaStream_t st, float* out32 = nullptr, int shuffle_c = 0,
                 bool nhwc32 = false, bool planar = false);

// Bank of a thin-input conv re-expressed as a 1x1 conv over gathered
// patches (see launch_patch): c_in' = roundup64(c_in*k*k).
Bank patch_bank(const Bank& b);
// Last decoder conv (nearest upsample + 3x3, c_out small) re-expressed as a
// 3x3 conv on the low-res image with 4*c_out outputs (one per parity) --
// the sub-pixel form -- followed by depth-to-space in the epilogue.
Bank subpixel_shuffle_bank(const Bank& b);

// ---------------------------------------------------------------- engine
struct RunStats {
    double ms_encode = 0, ms_denoise = 0, ms_decode = 0, ms_total = 0;  // device-timed
    double setup_s = 0;  // host wall time of the configure() that prepared the weights
    double stall_ms = 0, makespan_ms = 0;
    int64_t full_steps = 0, cached_steps = 0;
    int64_t macs_full = 0, macs_cached = 0, denoiser_macs = 0;
    int64_t swap_bytes = 0, swap_calls = 0;  // logical (reference) transfer bytes and calls
    int64_t swap_bytes_moved = 0;             // bytes that crossed the host link (clean evictions elided)
    int64_t cache_bytes_planned = 0, cache_bytes_physical = 0;
    int64_t peak[4][2] = {};
    int64_t hbm_peak = 0;
    std::vector<std::array<double, 4>> timeline;  // kind, step, bytes, t_ms
    bool simulated = false;  // timeline is the swap.simulate virtual clock
    int64_t kernel_launches = 0;
};

class Engine {
public:
    explicit Engine(int device);
    ~Engine();

    // Prepare weights/buffers for a config (no-op when unchanged).
    void configure(const RunConfig& cfg);
    const RunConfig& config() const { return cfg_; }

    // Whole pipeline.  x0_host: initial latent (1,T,C,h,w) fp32 or nullptr
    // to generate it (text mode: randn(derive_seed(seed,1)),
    // pipeline.cpp:115).  video_host may be nullptr (video stays on device
    // in video_dev()).  latent_host receives the final latent if non-null.
    RunStats run(const float* x0_host, float* video_host, float* latent_host, bool resident_input);
    // Throughput loops: enqueue one resident run (graph replay) without
    // waiting; wait() completes the queued runs and reports the last one.
    void run_resident_async();
    void run_e2e_async(const float* x0_pinned, float* video_pinned);
    RunStats wait();

    // Operator-level entry points (for unit parity).
    // forward_full / forward_cached on x (2,T,C,h,w) host fp32.
    void forward(const float* x_host, int64_t T, int64_t timestep, const float* deep_in_ref,
                 float* deep_out_ref, float* eps_host);
    // decode n latents (n,C,h,w) -> (n,3,H,W); C, h, w are checked against
    // the configured codec geometry (ShapeError, codec.cpp:129-131).
    void decode(const float* lat_host, int64_t n, int64_t c, int64_t h, int64_t w, float* video_host,
                int64_t slice);
    // Sliced decode sharded over `world` ranks (balanced contiguous frame
    // blocks, host.hpp shard_frames); each decoded slice is sent to rank 0
    // over NCCL as soon as it is final (gather_plan rounds) while the next
    // slice decodes.  video_host: rank 0's full video (after the gather);
    // with `host_shared` every rank instead writes ITS frames straight into
    // `video_host`, one host buffer mapped by all ranks (parallel host links).
    void decode_sharded(const float* lat_host, int64_t T, int64_t c, int64_t h, int64_t w, int64_t slice,
                        float* video_host, bool host_shared, ncclComm_t comm, int world, int rank,
                        float* ms_out);
    // Allocate run buffers for the configured frame count.
    void run_prepare() { alloc_activations(cfg_.frames); }

    // Device-resident helpers for the bench.
    // Staged initial latent for resident runs (copied into the trajectory
    // buffer at the start of every run).
    float* latent_dev() { return x0_.as<float>(); }
    float* video_dev() { return video_.as<float>(); }
    int64_t latent_elems() const;
    int64_t video_elems() const;
    cudaStream_t stream() const { return s_compute_; }
    Ledger& ledger() { return ledger_; }

    const RunStats& last_stats() const { return last_stats_; }
    double configure_s_ = 0;

    int64_t decode_slice = 4;  // frames per decode launch group (tool flag)
    int64_t launches = 0;
    bool use_graphs = true;    // replay the denoise+decode body as a CUDA graph

    // Stage arena (see Ledger): sizes of the run's working sets this config
    // needs, in bytes (for reports and tests).
    struct ArenaInfo {
        int64_t arena = 0, act = 0, cache = 0, dec = 0, enc = 0;
        bool dec_overlaps_cache = false;
    };
    ArenaInfo arena_info() const { return arena_info_; }
    double link_gbs() const { return link_gbs_; }  // host-link probe (GB/s per direction, 0 = not probed)
    int branch_deep() const { return branch_deep_; }
    bool branch_seam() const { return branch_seam_; }

private:
    // Decode workspace: per-stage activations of one slice of G frames, the
    // first conv's patch rows and the tap-to-N partial sums (fallback path).
    struct DecWs {
        Act act[8];
        Act patch;
        float* y = nullptr;
        int G = 0;
    };
    DecWs dec_ws_run_;              // carved from the arena (runs)
    DecWs dec_ws_op_;               // operator-level decode / decode_sharded
    std::vector<DevBuf> dec_bufs_op_;
    const DecWs* dec_ws_ = nullptr;  // the workspace decode_dev uses
    void ensure_op_dec_ws(int G);
    int64_t dec_ws_bytes(int G, bool want_y) const;
    DevBuf arena_;                  // one device allocation for every per-run working set
    ArenaInfo arena_info_;
    double link_gbs_ = 0;
    int64_t arena_G_ = -1;
    bool act_padding_ = false, dec_padding_ = false, enc_padding_ = false;
    uint64_t rid_act_ = 0, rid_dec_ = 0, rid_enc_ = 0, rid_cache_[2] = {0, 0};
    struct Level {
        Act D;     // skip output of d_i
        Act P;     // pooled input of d_i (i >= 1) / mid
        Act U;     // output of u_i
        Act UP;    // materialised upsample (fallback path only)
    };
    void alloc_activations(int64_t T);
    void enqueue_body(RunStats& st);
    void prepare_noise();
    void invalidate_graph();
    RunStats finish_run(RunStats st, float* video_host, float* latent_host);
    static void copy_out_parallel(float* dst, const float* src, int64_t n);
    bool async_pending_ = false;
    bool host_valid_ = false;  // the pinned host copy equals the device cache (clean entries)
    RunStats last_async_;
    RunStats last_stats_;  // the last completed run (typed RunResult, lc_run_result)
    bool body_enqueued_ = false;  // this run's body was enqueued on the host (eager or capture)
    int64_t body_peak_[4][2] = {};  // ledger peaks of that run (graph replays report them)
    void ensure_buf(DevBuf* b, int64_t bytes);  // grow-only scratch (invalidates the graph when it grows)
    // seam: 0 no swap, 1 await the prefetch at the seam, 2 await + evict
    // (last consumer), 3 full step with swap (record the cache-ready event
    // after the U_{m+1} producer).  stacked: x_dev holds the explicit (2,T,...) CFG
    // stack instead of the b=1 latent.
    // fuse (nullable): the sampler step of this denoising step; when the
    // head runs as K8 it applies it in its epilogue (eps never reaches HBM)
    // and step_fused_ is set, otherwise eps2_dev is written.
    void forward_dev(const float* x_dev, bool stacked, int64_t T, int64_t timestep, bool full,
                     float* eps2_dev, int step, int seam, const StepArgs* fuse = nullptr);
    bool step_fused_ = false;
    // per-branch deep path in full steps that evict (forward_dev): chosen
    // from the measured host-link bandwidth (LC_BRANCH_DEEP=0/1 forces it)
    int branch_deep_ = 0;  // 0 whole batch, 1 per-branch deep path, 2 per-branch up path
    bool branch_seam_ = true;  // cached steps: seam block per CFG entry (see decide_branch_deep)
    void decide_branch_deep();
    double probe_link_gbs();
    void conv_block(int j, const Act& in, const Act& out, float s, float o, bool silu);
    void up_block(int i, const Act& skip, const Act& u, const Act& out, float s, float o);
    void decode_dev(const float* lat_dev, int64_t n, float* video_dev);
    void issue_evict(int step);
    void issue_prefetch(int issued, int needed);
    void seam_await(int step);
    void record(int kind, int step, int64_t bytes, cudaStream_t st);

    int device_;
    RunConfig cfg_;
    bool configured_ = false;
    std::string cfg_key_;
    std::string cfg_prev_mode_;       // arena layout depends on these too
    bool cfg_prev_sliced_ = true;
    Ledger ledger_;
    UNetWeights uw_;
    CodecWeights cw_;
    std::vector<std::unique_ptr<TcLayer>> tc_;     // per block (nullptr for thin)
    std::vector<std::unique_ptr<TcLayer>> tc_fb_;  // up blocks: materialised-upsample fallback
    std::unique_ptr<ThinLayer> stem_, head_;
    std::unique_ptr<TcLayer> head_tc_;  // head on the tensor cores (N padded to 16)
    std::unique_ptr<TcLayer> stem_tc_, dec0_tc_, dec_last_tc_;
    // tap-to-N forms of the thin-output convs: 1x1 GEMM over (tap, channel)
    // columns + a gather kernel (launch_tap_gather / launch_subpix_gather)
    std::unique_ptr<TcLayer> head_tap_tc_, dec_last_tap_tc_;
    DevBuf head_wsum_, head_bias_, dec_last_bias_, head_y_buf_;
    DevBuf dec_last_w16_, head_w16_;  // K8 tap banks, fp16 [N][kb*64]
    int dec_last_kb_ = 0, dec_last_n_ = 0, head_kb_ = 0, head_n_ = 0;
    float dec_last_wscale_ = 1.0f, head_wscale_ = 1.0f;
    DevBuf shard_lat_, shard_vid_;  // decode_sharded buffers
    // encoder (image mode, codec.cpp:64-81): patch GEMM + [down2 + conv]xS
    std::unique_ptr<TcLayer> enc0_tc_;
    std::vector<std::unique_ptr<TcLayer>> enc_tc_;
    int enc0_kp_ = 64;
    DevBuf frames_dev_, eps0_dev_;
    std::string img_key_;
    Act enc_patch_, enc_e_[8], enc_p_[8];  // encode workspace (arena)
    void prepare_image();
    void encode_dev(float* lat_dev);
    int stem_kp_ = 64, dec0_kp_ = 64;
    Act patch_;                          // stem patch rows (2T, h, w, kp)
    std::vector<std::unique_ptr<TcLayer>> dec_tc_;  // decoder stages 1..S-1
    std::unique_ptr<ThinLayer> dec0_, dec_last_;
    int64_t run_dec_group() const;  // frames per decoder slice of a run
    std::vector<Level> lv_;
    Act stem_out_, mid_;
    Act cache_;        // U_{m+1} (b=2 stacked: images [0,T) uncond, [T,2T) cond)
    DevBuf cache_buf_, cache_host_;
    std::vector<DevBuf> act_bufs_;
    DevBuf x0_, x_, xn_, eps2_, video_, z_, bad_;
    int64_t T_alloc_ = -1;

    cudaStream_t s_compute_ = nullptr, s_d2h_ = nullptr, s_h2d_ = nullptr;
    cudaStream_t s_comm_ = nullptr;  // NCCL gather of decoded slices (decode_sharded)
    cudaEvent_t ev_base_ = nullptr;
    std::vector<cudaEvent_t> ev_pool_;
    size_t ev_next_ = 0;
    struct Mark {
        int kind;
        int step;
        int64_t bytes;
        cudaEvent_t ev;
    };
    std::vector<Mark> marks_;
    // swap.simulate: virtual timeline of the config (host.cpp
    // simulate_timeline), each step's virtual compute start and the clock
    // after the denoising drain, in seconds.
    std::vector<SimEvent> sim_tl_;
    std::vector<double> sim_step_s_;
    double sim_decode_s_ = 0;
    cudaEvent_t ev_prefetch_part_[2] = {nullptr, nullptr};  // first half of an entry's images landed
    cudaEvent_t ev_evict_[2] = {nullptr, nullptr}, ev_prefetch_[2] = {nullptr, nullptr},
                ev_cache_ready_[2] = {nullptr, nullptr};  // per CFG entry: U_{m+1} half complete
    bool evict_pending_ = false, prefetch_pending_ = false, cache_ready_recorded_ = false;
    bool d2h_used_ = false, h2d_used_ = false;
    cudaEvent_t ev_start_ = nullptr, ev_den0_ = nullptr, ev_den1_ = nullptr, ev_end_ = nullptr;
    cudaEvent_t ev_join_[2] = {nullptr, nullptr};
    cudaEvent_t ev_vid_done_ = nullptr;               // last video byte downloaded (see enqueue_video_out)
    bool out_slices_ = false;                         // decode_dev inside the run body
    std::vector<std::pair<int64_t, int64_t>> slice_spans_;  // decoded slices (first frame, frames)
    void enqueue_video_out(float* pinned);
    float* x_final_ = nullptr;
    // Deferred video download (pipelined e2e): run k's video is copied to its
    // pinned destination by a memcpy node inside run k+1's graph, released at
    // a gate point of k+1's body (compute-bound blocks, away from the
    // memory-bound ones the host-link DMA slows down); the node is re-pointed
    // (or disabled) before each launch, wait() flushes the last one.
    cudaStream_t s_vid_ = nullptr;
    cudaEvent_t ev_dl_gate_ = nullptr, ev_dl_done_ = nullptr, ev_dl_src_ = nullptr;
    bool dl_capture_ = false, dl_fired_ = false;
    int dl_gate_step_ = 0;
    std::string dl_gate_where_ = "stem";  // measured: 0:stem ~ 0:d0 > off > later gates (B e2e)
    DevBuf dl_scratch_;                    // pinned capture placeholder of the node's destination
    DevBuf vid_stage_;                     // pinned staging of a pageable run() video destination
    cudaGraph_t graph_ = nullptr;          // kept alive: dl_node_ belongs to it
    cudaGraphNode_t dl_node_ = nullptr;
    float* dl_pending_ = nullptr;          // pinned destination of a not yet issued download
    void dl_gate(int step, const char* where);
    void fire_download();
    void flush_pending_download();
    void arm_download_node();              // before a graph launch
    cudaGraphExec_t graph_exec_ = nullptr;
    RunStats graph_stats_;
    int eager_runs_ = 0;
    int64_t graph_slice_ = -1;
    float* video_host_pinned_ = nullptr;  // current run's pinned destination (or null)
    std::string z_key_;
    std::vector<cudaEvent_t> ev_chunk_[3];  // [0,1] swap chunks per branch, [2] decoded slices
    cudaEvent_t chunk_event(int b, size_t i);
    int prefetch_tag_ = -1;
    RunStats* stats_ = nullptr;
    cudaEvent_t next_event();
};

}  // namespace lc
