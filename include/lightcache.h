/*
 * lightcache.h -- C-ABI of the B200-native LightCache hot path
 * (paper_2510_05367_b200/liblightcache.so).
 *
 * The reference ("stagecache", /root/reference/proj) exposes this path only
 * as C++ API of a static library; it has no plugin registry or FFI.  Each
 * entry point below is the flat C form of the reference call it replaces
 * (cited as proj/<file>:<line>), with plain pointers and sizes.  All
 * functions return 0 on success or the reference CLI exit code of the
 * exception the reference would throw (proj/tools/main.cpp:157-169):
 *   1 ShapeError (and other std::exception), 2 ConfigError,
 *   3 BudgetError, 4 InvariantError; 5 = CUDA failure (no reference analogue).
 * lc_last_error() returns the thread-local message of the last failure.
 *
 * Config text uses the reference grammar (proj/src/config.cpp:206-224):
 * one "key = value" per line over default_config(), '#' comments, every key
 * of apply_override (proj/src/config.cpp:158-204); unknown keys -> 2.
 *
 * Host tensors are row-major {b,t,c,h,w} fp32 exactly as stagecache::Tensor5
 * (proj/include/stagecache/tensor.hpp:60-62).
 */
#ifndef LIGHTCACHE_H
#define LIGHTCACHE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lc_ctx lc_ctx;

/* Library / context ------------------------------------------------------ */
int lc_version(void);
const char* lc_last_error(void);
/* One context per GPU: streams, packed weights, device buffers. */
int lc_ctx_create(int device, lc_ctx** out);
int lc_ctx_destroy(lc_ctx* ctx);

/* Configuration (host only) ---------------------------------------------- */
/* RunConfig parse + validate (proj/src/config.cpp:100-141, :158-224). */
int lc_config_check(const char* config_text);
/* config_to_text (proj/src/config.cpp:226-264) of the parsed config. */
int lc_config_to_text(const char* config_text, char* out, int64_t cap);
/* Prepare a context for a config: weights (init_weights, proj/src/unet.cpp:153;
 * init_codec, proj/src/codec.cpp:45), packed for the tensor cores, and buffers. */
int lc_configure(lc_ctx* ctx, const char* config_text);
int64_t lc_latent_elems(lc_ctx* ctx); /* T*C*h*w of the b=1 latent */
int64_t lc_video_elems(lc_ctx* ctx);  /* T*3*H*W of the b=1 video */

/* Whole pipeline: replaces run_pipeline (proj/include/stagecache/pipeline.hpp:42,
 * proj/src/pipeline.cpp:64-228).  x0: initial latent (1,T,C,h,w) or NULL to
 * draw it as the reference does (randn(derive_seed(seed,1)), pipeline.cpp:115).
 * video (1,T,3,H,W) and latent_out (final x) may be NULL.  report receives a
 * JSON object (device-timed stage ms, MAC counters, cache bytes, swap
 * timeline makespan/stall, per-stage HBM/pinned peaks). */
int lc_run_pipeline(lc_ctx* ctx, const float* x0, float* video, float* latent_out,
                    char* report, int64_t report_cap);

/* Typed RunResult of the last completed run (run_pipeline's result,
 * proj/include/stagecache/pipeline.hpp:18-39), without the video (passed to
 * lc_run_pipeline) and the config (the caller's).  wall_*: StageWall in
 * seconds -- setup is the host time of the lc_configure that initialised
 * and packed the weights, encode / denoise / decode / total are device
 * (CUDA event) times of the run.  peak_* / current_* / events_per_stage /
 * event_count: StageReport of the engine's ledger (stage order setup,
 * encode, denoise, decode).  Timeline rows (kind, step, bytes, clock_ns) in
 * TimelineEventKind order (swap.hpp:16-31), clock from the run's start;
 * pass timeline = NULL to query n_timeline. */
typedef struct lc_run_result {
    double wall_setup, wall_encode, wall_denoise, wall_decode, wall_total;
    int64_t peak_fast[4], peak_slow[4];
    int64_t current_fast, current_slow;
    int64_t events_per_stage[4];
    int64_t event_count;
    int64_t denoiser_macs, macs_per_full_step, macs_per_cached_step, full_steps, cached_steps;
    int64_t cache_bytes_planned;
    double makespan_s, stall_s;
    int simulated;
    int64_t n_timeline;
} lc_run_result;
int lc_get_run_result(lc_ctx* ctx, lc_run_result* out, int64_t* timeline, int64_t cap_rows);
/* Stage (0 setup, 1 encode, 2 denoise, 3 decode) of the last BudgetError
 * on this thread (BudgetError::stage, proj/include/stagecache/common.hpp:43),
 * -1 when the last error was of another kind. */
int lc_last_error_stage(void);

/* Device-resident variant for throughput measurement: the initial latent
 * must have been staged with lc_upload_latent; the video stays in HBM
 * (fetch with lc_download_video). */
int lc_upload_latent(lc_ctx* ctx, const float* x0);
int lc_run_resident(lc_ctx* ctx, char* report, int64_t report_cap);
/* Throughput loops: enqueue one resident run without a host round trip
 * (steady state: a CUDA-graph replay; runs queue back to back), then
 * lc_wait completes everything queued and reports the last run.  The first
 * runs after lc_configure execute synchronously (graph capture). */
int lc_run_resident_async(lc_ctx* ctx);
/* Same with pinned host buffers (the lc_run_pipeline contract): the H2D of
 * x0, the run and the per-slice D2H of the video are queued without a host
 * round trip, so run k+1 computes while run k's video downloads; lc_wait
 * completes them.  x0 / video must stay valid until lc_wait returns.
 * Pageable buffers are accepted but run synchronously (lc_run_pipeline). */
int lc_run_pipeline_async(lc_ctx* ctx, const float* x0, float* video);
int lc_wait(lc_ctx* ctx, char* report, int64_t report_cap);
int lc_download_video(lc_ctx* ctx, float* video);
/* Frames decoded per launch group in sliced decode (tool flag, not a config
 * key; the output is identical for every value). */
int lc_set_decode_slice(lc_ctx* ctx, int64_t frames);

/* Memory ledger: the engine's physical event log in the
 * reference's ledger.csv format (write_ledger_csv, proj/src/ledger.cpp:224-242:
 * seq,clock,kind,tier,bytes,alloc_id,occupancy_bytes,stage), and its summary
 * (write_ledger_json content: per-stage fast/slow peaks and event counts,
 * overall peaks, current occupancy, event count) as JSON.  `needed` receives
 * the full text length; text beyond `cap` is truncated. */
int lc_ledger_csv(lc_ctx* ctx, char* buf, int64_t cap, int64_t* needed);
int lc_ledger_summary(lc_ctx* ctx, char* buf, int64_t cap);

/* Measurement helpers (bench.py) ------------------------------------------ */
/* CUDA events on the context's compute stream bracketing any number of
 * calls; lc_timer_stop synchronises and returns the elapsed device ms. */
int lc_timer_start(lc_ctx* ctx);
int lc_timer_stop(lc_ctx* ctx, float* ms);
/* Per-launch CUDA-event timing of the tensor-core conv kernel (on/off);
 * lc_conv_profile returns launches, device ms, algorithmic FLOPs (the
 * reference's conv MAC count x2) and executed MMA FLOPs since the last reset. */
int lc_set_conv_profile(lc_ctx* ctx, int on);
int lc_conv_profile(lc_ctx* ctx, int64_t* launches, double* ms, double* alg_flops,
                    double* exec_flops);
/* Per-launch records of the conv profile: JSON [{ms, alg_flops, exec_flops, desc}]. */
int lc_conv_profile_records(lc_ctx* ctx, char* buf, int64_t cap);
/* Kernels this library launched for the last run / decode call. */
int lc_kernel_launches(lc_ctx* ctx, int64_t* n);
/* Pinned host buffers for end-to-end copies. */
void* lc_alloc_pinned(int64_t bytes);
int lc_free_pinned(void* p);

/* Operators -------------------------------------------------------------- */
/* forward_full (deep_in == NULL; proj/src/unet.cpp:188-230) or
 * forward_cached (proj/src/unet.cpp:232-276) on x (2,T,C,h,w).  deep_in /
 * deep_out use the reference geometry u_next = upsample2(U_{m+1})
 * (cache_feature_shape, proj/src/unet.cpp:302-309).  eps has x's shape. */
int lc_forward(lc_ctx* ctx, const float* x, int64_t T, int64_t timestep, const float* deep_in,
               float* deep_out, float* eps);
/* decode_batch / decode_sliced (proj/src/codec.cpp:117-145) of n latents
 * (n,1,c,h,w) -> (n,1,3,H,W); `slice` frames per launch group.  c must be
 * the codec's latent channel count (ShapeError, as codec.cpp:129-131) and
 * h x w the configured latent geometry (ShapeError otherwise). */
int lc_decode(lc_ctx* ctx, const float* latents, int64_t n, int64_t c, int64_t h, int64_t w,
              int64_t slice, float* video);
/* Quality metrics: per-frame PSNR (dB, capped at 99) and
 * mean 7x7-window SSIM of two b=1 videos {t,c,h,w} fp32 (host or device
 * pointers), data range L.  Replaces psnr / ssim / video_series
 * (proj/src/metrics.cpp:10-104).  Errors: data_range <= 0 -> 2 (ConfigError),
 * h or w < 7 -> 1 (ShapeError). */
int lc_video_metrics(lc_ctx* ctx, const float* a, const float* b, int64_t t, int64_t c, int64_t h,
                     int64_t w, double data_range, double* psnr, double* ssim);
/* conv2d (proj/src/tensor.cpp:151-197) of affine(x, s, o) with optional SiLU
 * on the tensor-core kernel: x (b,t,c_in,h,w), taps [c_out][c_in][k][k]. */
int lc_conv2d(lc_ctx* ctx, const float* x, int64_t b, int64_t t, int64_t c_in, int64_t h,
              int64_t w, const float* taps, const float* bias, int64_t c_out, int64_t k,
              float s, float o, int silu, float* out);
/* Up block (proj/src/unet.cpp:101-122): silu(conv3x3(concat(affine(skip),
 * affine(upsample2(u))))) with the upsample fused (sub-pixel).  skip
 * (b,t,c_a,h,w), u (b,t,c_b,h/2,w/2), taps [c_out][c_a+c_b][3][3]. */
int lc_up_conv2d(lc_ctx* ctx, const float* skip, const float* u, int64_t b, int64_t t,
                 int64_t c_a, int64_t c_b, int64_t h, int64_t w, const float* taps,
                 const float* bias, int64_t c_out, float s, float o, float* out);
/* cfg_combine + reverse_step_{ancestral,ddim,euler} (proj/src/sampler.cpp:
 * 95-133) as one device update at index t of the context's configured
 * (spaced) schedule, the t argument of the reference's reverse_step_*:
 *   eps = (1-g) e_u + g e_c;  x' = a x + b eps  [+ sqrt(beta_t) z,
 *   z = randn(n, noise_seed), ancestral with t > 0 only].
 * sampler: 0 ancestral, 1 ddim, 2 euler (SamplerKind).  eps2 holds e_u then
 * e_c (2n floats, select_batch(eps2, 0/1)); x, x_out n floats (host).
 * *nonfinite (nullable) = 1 if x' holds a non-finite value.  Errors:
 * guidance < 0, then t outside [0, steps) -> 2 (ConfigError, sampler.cpp:130,
 * :79-84). */
int lc_sampler_step(lc_ctx* ctx, int sampler, int64_t t, const float* x, const float* eps2, int64_t n,
                    double guidance, uint64_t noise_seed, float* x_out, int* nonfinite);
/* all_finite (proj/src/tensor.cpp:376) of n host floats on the device:
 * *finite = 1 when every value is finite. */
int lc_all_finite(lc_ctx* ctx, const float* x, int64_t n, int* finite);

/* Host logic (bit-exact contracts) ---------------------------------------- */
/* plan_steps (proj/src/cache.cpp:25-33): kinds[s] 1 = Full; flags bit0
 * has_consumers (cache.cpp:19-23), bit1 is_last_consumer (cache.cpp:15-18). */
int lc_plan_steps(int64_t total, int64_t interval_n, int8_t* kinds, int8_t* flags);
/* split (proj/src/chunk.cpp:145-181) for a single-conv chain of kernel k;
 * halo_kind 0 exact, 1 fixed, 2 none; regions 12 int64 per tile:
 * core, padded, out_window as (y0,y1,x0,x1). */
int lc_split(int64_t h, int64_t w, int64_t eta, int64_t omega, int halo_kind, int64_t halo_px,
             int64_t k, int64_t* regions, int64_t* halo_out);
/* flops_estimate (proj/src/unet.cpp:287-300) MACs for the config's model
 * input, Full (cached=0) or Cached (cached=1); cache_bytes
 * (proj/src/cache.cpp:124-130) in the reference fp32 geometry. */
int lc_model_numbers(const char* config_text, int64_t* macs_full, int64_t* macs_cached,
                     int64_t* cache_bytes);
/* The simulated transfer engine (swap.simulate = true,
 * proj/src/swap.cpp:141-364, driven by pipeline.cpp:119-207 and
 * cache.cpp:43-122): the virtual-clock timeline of the config's denoising
 * loop.  Host-only (no device work).  `events` receives n_events rows of
 * (kind, step, bytes, clock_ns), kind as TimelineEventKind
 * (proj/include/stagecache/swap.hpp:16-23); makespan and stall as
 * makespan_ns / stall_total_ns (swap.cpp:59-79).  Pass events = NULL to
 * query n_events. */
int lc_simulate_timeline(const char* config_text, int64_t* events, int64_t cap_events,
                         int64_t* n_events, int64_t* makespan_ns, int64_t* stall_ns);
/* The denoise activations' arena plan (host only): every buffer's bytes,
 * lifetime [t0, t1] within a full step and offset, packed first-fit by
 * lifetime (the layout lc_run_pipeline uses), as JSON
 * {cache_bytes, act_end, ops, buffers: [{name, bytes, t0, t1, off, c, cs}]}. */
int lc_plan_arena(const char* config_text, char* out, int64_t cap);
/* derive_seed / NormalStream (proj/include/stagecache/rng.hpp:11-45). */
uint64_t lc_derive_seed(uint64_t seed, uint64_t stream);
int lc_randn(uint64_t seed, int64_t n, float* out);

/* Multi-GPU sliced decode (one process per GPU) --------------------------- */
/* Frame shard of rank r out of g for T frames: balanced contiguous blocks
 * (the first T % g ranks take one more frame; 25 on
 * 8 GPUs = 4,3,3,3,3,3,3,3). */
int lc_shard_frames(int64_t T, int world, int rank, int64_t* first, int64_t* count);
/* The gather schedule lc_decode_sharded executes: rows of (round, rank,
 * first_frame, count); round i moves the i-th decoded slice of every rank
 * that has one to rank 0.  rows = NULL queries n_rows. */
int lc_gather_plan(int64_t T, int world, int64_t slice, int64_t* rows, int64_t cap_rows,
                   int64_t* n_rows);
/* NCCL communicator for the decode gather.  lc_nccl_unique_id writes
 * 128 bytes; the caller distributes them (e.g. over torch.distributed). */
int lc_nccl_unique_id(uint8_t* id128);
int lc_nccl_init(lc_ctx* ctx, const uint8_t* id128, int world, int rank);
/* Decode this rank's shard of `latents` (T,1,c,h,w, replicated on every
 * rank) slice by slice (decode_sliced, proj/src/codec.cpp:126-145) and
 * gather every frame into rank 0's HBM over NVLink: each slice is sent with
 * ncclSend as soon as it is decoded, rank 0 receives round by round
 * (lc_gather_plan) while its own slices decode.  video (T,1,3,H,W host,
 * nullable): without flags rank 0 writes the whole video (other ranks may
 * pass NULL); with LC_SHARD_HOST_SHARED `video` is ONE host buffer mapped by
 * every rank (e.g. a shared-memory segment registered with
 * lc_host_register) and each rank downloads its own frames into it over its
 * own host link.  ms_out (nullable): device time of H2D + decode + gather
 * (+ download) on this rank. */
#define LC_SHARD_HOST_SHARED 1
int lc_decode_sharded(lc_ctx* ctx, const float* latents, int64_t T, int64_t c, int64_t h, int64_t w,
                      int64_t slice, float* video, int flags, float* ms_out);
/* cudaMemGetInfo of the context's device (cross-check of the ledger's
 * physical HBM peak). */
int lc_mem_info(lc_ctx* ctx, int64_t* free_bytes, int64_t* total_bytes);
/* Page-lock caller memory (cudaHostRegister, portable) for fast copies. */
int lc_host_register(void* p, int64_t bytes);
int lc_host_unregister(void* p);

#ifdef __cplusplus
}
#endif

#endif /* LIGHTCACHE_H */
