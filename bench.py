#!/usr/bin/env python
"""Benchmark of the B200-native LightCache path.

Metric (BASELINE.json): end-to-end video frames/sec (+ peak HBM GB) against
the uncached GPU run and the CPU reference.  One "step" is one whole video
generation -- run_pipeline (proj/src/pipeline.cpp:64): the denoise loop with
the feature cache / async swap / chunked execution, then sliced decode --
on the LARGEST single-GPU configuration of BASELINE.json (configs[2],
config C): SVD-XT-shaped U-Net, 25 frames, latent 4x72x128 (1024x576
video), 25 Euler steps, cache N=2 with the async swap, base 320, synthetic
latent and random-init weights (B, A and the decode workload D on request).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C|B|A|D]
  python bench.py --impl reference ...     (CPU reference arm: oracle/_ref)
  python bench.py --gpus N ...             (spawns N local ranks itself)
  torchrun --nproc-per-node N bench.py --gpus N   (same, launched by torchrun)

At N > 1 every rank runs one replica of the workload (denoising does not
shard: batch 1 per GPU) and the line adds
`decode_sharded`: workload D's sliced decode sharded over the N GPUs with
the NCCL gather of the decoded slices (strong scaling).

Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
# default_config() (proj/src/config.cpp:90-98): the workloads override it
DEFAULT_TEXT = ""

WORKLOADS = {
    # configs[1] of BASELINE.json
    "B": {"run.frames": 16, "run.height": 512, "run.width": 512, "codec.stages": 3, "codec.width": 128,
          "unet.base_channels": 320, "unet.depth": 3, "sampler.steps": 4, "cache.n": 2},
    # configs[2]: SVD-XT-shaped with async cache swap
    "C": {"run.frames": 25, "run.height": 576, "run.width": 1024, "codec.stages": 3, "codec.width": 128,
          "unet.base_channels": 320, "unet.depth": 3, "sampler.steps": 25, "cache.n": 2, "swap.mode": "async"},
    # configs[0]: tiny desk config
    "A": {"run.height": 128, "run.width": 128, "cache.n": 3, "chunk.eta": 2, "chunk.omega": 1},
    # configs[3]: SVD-XT VAE decode alone (latent 25x4x72x128 -> 25 frames of 1024x576),
    # latent slices sharded over the GPUs, NCCL gather to rank 0
    "D": {"run.frames": 25, "run.height": 576, "run.width": 1024, "codec.stages": 3, "codec.width": 128,
          "unet.base_channels": 320, "unet.depth": 3},
}
DESCR = {
    "B": "AnimateDiff-Lightning-shaped U-Net: 16 frames, latent 4x64x64 (512x512 video), 4 Euler steps, "
         "cache N=2 at seam m=0, async swap, chunk u0 2x2 exact halo, sliced decode (4 frames/slice), "
         "base 320, depth 3, codec W=128 S=3",
    "C": "SVD-XT-shaped U-Net: 25 frames, latent 4x72x128 (1024x576 video), 25 Euler steps, cache N=2 at "
         "seam m=0 (13 full + 12 cached steps), async swap, chunk u0 2x2 exact halo, sliced decode, base 320, "
         "depth 3, codec W=128 S=3",
    "A": "tiny desk config: 8 frames, latent 4x32x32, 25 steps, N=3, chunk u0 2x1",
    "D": "SVD-XT VAE decode: latent 25x4x72x128 -> 25 frames 1024x576, codec W=128 S=3, 5-frame slices, "
         "contiguous frame blocks per GPU, NCCL gather of the decoded frames to rank 0",
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------- helpers
def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # host-side plumbing only (barriers, max over ranks, the NCCL id);
        # the data path's collective is the library's own NCCL gather
        dist.init_process_group("gloo", rank=rank, world_size=world)
    return world, rank, local


def spawn_ranks(n: int) -> int:
    """`--gpus N` without torchrun: start N local ranks of this script (one
    per GPU, RANK/LOCAL_RANK/WORLD_SIZE/MASTER_* set as torchrun sets them)
    and wait; rank 0's stdout is the JSON line."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable] + sys.argv, env=env,
                                      stdout=None if r == 0 else subprocess.DEVNULL))
    rc = 0
    for p in procs:
        rc = rc or p.wait()
    return rc


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def allmax(world, v: float) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        time.sleep(0.05)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        if "bf16_tflops_sustained" in d:
            return d["bf16_tflops_sustained"], "measured (MEASURED_PEAKS.json bf16 sustained; fp16 same rate)"
    return 1400.0, "fallback (B200_PROFILING.md sustained)"


def decode_macs(kv: dict, frames: int) -> int:
    """Decoder MACs (proj/src/codec.cpp:103-113, counted by tensor.cpp:194)."""
    S = int(kv["codec.stages"])
    W = int(kv["codec.width"])
    C = int(kv["codec.latent_channels"])
    h = int(kv["run.height"]) >> S
    w = int(kv["run.width"]) >> S
    tot = C * W * h * w
    for i in range(1, S + 1):
        co = 3 if i == S else W
        tot += W * co * (h << i) * (w << i)
    return 9 * tot * frames


def _plan_counts(kv: dict):
    """(full, cached) step counts of plan_steps (proj/src/cache.cpp:25-33)."""
    S, N = int(kv["sampler.steps"]), int(kv["cache.n"])
    enabled = kv["cache.enabled"] in ("true", "on", "1")
    nf = sum(1 for s in range(S) if (not enabled) or s % N == 0)
    return nf, S - nf


def ref_run_macs(lib, kv: dict) -> int:
    """MACs of one whole run_pipeline of `kv` from the REFERENCE's own
    closed forms: flops_estimate per Full / Cached step
    (proj/src/unet.cpp:287-300, via oracle/_ref or the restatement) over the
    plan, plus the decoder's convs (proj/src/codec.cpp:103-113)."""
    import lco
    if isinstance(lib, lco.Reference):
        nums = lib.model_numbers(kv)
        mf, mc = nums[0], nums[1]
    else:
        mf, mc = lib.flops_estimate(kv, False), lib.flops_estimate(kv, True)
    nf, nc = _plan_counts(kv)
    return nf * mf + nc * mc + decode_macs(kv, int(kv["run.frames"]))


# ---------------------------------------------------------------- CPU arm
# Bounded sample of a workload for the reference's CPU path: one frame (the
# toy model has no cross-frame ops), the smallest latent the
# U-Net depth admits with the workload's aspect (C: 8x16 = 1/72 of 72x128),
# the same channels / depth / kernel / codec, and one refresh period of the
# cache plan (N steps: 1 Full + N-1 Cached); the swap and chunking settings
# stay.  The reference's work is linear in frames x pixels and per step, so
# frames/s of the full workload = sample MACs / full-frame MACs x samples/s,
# with both MAC counts from the reference's own closed forms.
SAMPLES = {
    "C": {"run.frames": 1, "run.height": 64, "run.width": 128, "sampler.steps": 2},
    # B at latent 8x16 like C (tools/ref_crosscheck.py: an 8x8 sample ran the
    # reference at 0.73x, a 16x16 one at 1.20x its full-frame MAC rate)
    "B": {"run.frames": 1, "run.height": 64, "run.width": 128, "sampler.steps": 2},
    "A": {"run.frames": 1, "run.height": 32, "run.width": 32, "sampler.steps": 3},
    "D": {"run.frames": 1, "run.height": 64, "run.width": 128},
}


def _kv(over: dict) -> dict:
    import lco
    kv = lco.parse_text(DEFAULT_TEXT)
    kv.update({k: str(v) for k, v in over.items()})
    return kv


def _cpu_lib():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import lco
    if lco.Reference.available():
        return lco.Reference(), "reference"
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    return lco.Restatement(), "port"


def _cpu_worker(args):
    """One bounded sample through the reference's public API (run_pipeline,
    or decode_sliced for workload D); returns its wall seconds."""
    text, decode_only = args
    lib, _ = _cpu_lib()
    import lco
    kv = lco.parse_text(text)
    t = time.time()
    if decode_only:
        import numpy as np
        s = 1 << int(kv["codec.stages"])
        lat = np.random.default_rng(0).standard_normal(
            (1, 1, int(kv["codec.latent_channels"]), int(kv["run.height"]) // s,
             int(kv["run.width"]) // s)).astype(np.float32)
        lib.decode(kv, lat)
    else:
        lib.run_pipeline(kv)
    return time.time() - t


def cpu_sample(workload: str):
    """(sample config kv, sample MACs, full-workload MACs per frame, kind)."""
    lib, kind = _cpu_lib()
    full = _kv(WORKLOADS[workload])
    samp = _kv(dict(WORKLOADS[workload], **SAMPLES[workload]))
    T = int(full["run.frames"])
    if workload == "D":
        return samp, decode_macs(samp, 1), decode_macs(full, T) / T, kind
    return samp, ref_run_macs(lib, samp), ref_run_macs(lib, full) / T, kind


def _sample_desc(workload, samp, macs_s, macs_f, kind):
    s = 1 << int(samp["codec.stages"])
    what = "decode of 1 frame" if workload == "D" else (
        f"run_pipeline of 1 frame, {samp['sampler.steps']} steps (one N={samp['cache.n']} cache period)")
    return (f"{kind} CPU path ({'oracle/_ref, the unmodified reference' if kind == 'reference' else 'oracle port'}): "
            f"{what} at latent {int(samp['run.height']) // s}x{int(samp['run.width']) // s}, same channels/depth/codec; "
            f"{macs_s / 1e9:.2f} GMAC per sample vs {macs_f / 1e9:.1f} GMAC per full-workload frame "
            f"(reference flops_estimate + decoder MACs); frames/s = sample MACs / frame MACs x samples/s")


def cpu_measure(workload: str, reps: int = 1):
    """Single-core reference sample for the GPU arm's cpu_baseline."""
    samp, macs_s, macs_f, kind = cpu_sample(workload)
    import lco
    times = [_cpu_worker((lco.to_text(samp), workload == "D")) for _ in range(reps)]
    per = statistics.median(times)
    fps = macs_s / macs_f / per
    return {"value": fps, "unit": "frames/s", "cores": 1, "kind": kind,
            "sample": _sample_desc(workload, samp, macs_s, macs_f, kind) + f"; {per:.1f} s per sample, 1 core "
                      "(not size-calibrated: the --impl reference arm measures the full-resolution / sample rate "
                      "ratio, 1.24 on C in profiles/ref_crosscheck_r02.json)"}


# Full-resolution calibration job of the reference arm: one frame of the
# real workload over one cache refresh period (the sample's step mix).  The
# reference's MAC rate depends on the image size (tools/ref_crosscheck.py,
# profiles/ref_crosscheck_r02.json: C at full resolution 1.22 GMAC/s per
# core vs 0.98 for the 8x16 sample; B 0.96 vs 0.97), so the sample's
# extrapolated frames/s is scaled by the ratio measured in the same run.
CALIB = {"C": {"run.frames": 1, "sampler.steps": 2}, "B": {"run.frames": 1, "sampler.steps": 2}}


def reference_arm(args, world, rank):
    """The reference's own CPU implementation of the path (oracle/_ref:
    the unmodified proj/src compiled in place; run_pipeline,
    proj/src/pipeline.cpp:64-228) on all host cores: each step runs one
    bounded sample per core in a persistent process pool; the warm-up runs
    the full-resolution calibration job (CALIB) once per core.  Nothing of
    the product (paper_2510_05367_b200) is imported or loaded here."""
    if rank != 0:
        return
    import multiprocessing as mp
    import lco
    samp, macs_s, macs_f, kind = cpu_sample(args.workload)
    workers = max(1, min(os.cpu_count() or 1, 256))
    job = (lco.to_text(samp), args.workload == "D")
    calib = None
    with mp.get_context("spawn").Pool(workers) as pool:
        if args.workload in CALIB and args.warmup > 0:
            lib, _ = _cpu_lib()
            ckv = _kv(dict(WORKLOADS[args.workload], **CALIB[args.workload]))
            cmacs = ref_run_macs(lib, ckv)
            cwalls = pool.map(_cpu_worker, [(lco.to_text(ckv), False)] * workers)
            calib = {"full_res_gmac_per_s_per_core": cmacs / 1e9 / statistics.median(cwalls),
                     "job": f"1 frame at {ckv['run.height']}x{ckv['run.width']}, {ckv['sampler.steps']} steps, "
                            f"{cmacs / 1e9:.1f} GMAC, {statistics.median(cwalls):.0f} s per core"}
        for _ in range(max(0, args.warmup - (1 if calib else 0))):
            pool.map(_cpu_worker, [job] * workers)
        walls, per_proc = [], []
        for _ in range(args.steps):
            t0 = time.time()
            per_proc += pool.map(_cpu_worker, [job] * workers)
            walls.append(time.time() - t0)
    total = sum(walls)
    frames = workers * args.steps * macs_s / macs_f  # full-workload frame equivalents
    fps_raw = frames / total
    fps = fps_raw
    desc = _sample_desc(args.workload, samp, macs_s, macs_f, kind) + (
        f"; {workers} processes x {args.steps} steps, {total / args.steps:.2f} s per step")
    if calib:
        calib["sample_gmac_per_s_per_core"] = macs_s / 1e9 / statistics.median(per_proc)
        calib["ratio"] = calib["full_res_gmac_per_s_per_core"] / calib["sample_gmac_per_s_per_core"]
        fps = fps_raw * calib["ratio"]
        desc += (f"; scaled by the reference's full-resolution / sample MAC-rate ratio {calib['ratio']:.3f} "
                 f"measured in the warm-up ({calib['job']})")
    line = {"metric": "video_frames_per_sec", "value": fps, "unit": "frames/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * total / args.steps,
            "higher_is_better": True, "scaling": "weak" if args.workload != "D" else "strong",
            "vs_baseline": None, "dtype": "fp32",
            "data": "synthetic (seeded randn latent, random-init weights of the reference architecture)",
            "config": workload_config(args, world), "impl": "reference",
            "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": workers, "kind": kind, "sample": desc,
                             "uncalibrated_value": fps_raw, "calibration": calib},
            "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def swap_summary(rep: dict) -> dict:
    """Logical / moved bytes, seam stall, host-link GB/s of the transfers
    that moved bytes, and the fraction of that transfer time hidden behind
    compute (1 - stall / transfer time)."""
    open_x, xfer_ms, xfer_bytes = {}, 0.0, 0
    for kind, step, nbytes, t in rep["timeline"]["events"]:
        if kind == "xfer_start":
            open_x.setdefault(step, []).append(t)
        elif kind == "xfer_end" and open_x.get(step):
            dt = t - open_x[step].pop(0)
            if dt > 0.02:  # clean evictions move nothing (~0 ms)
                xfer_ms += dt
                xfer_bytes += nbytes
    stall = rep["timeline"]["stall_ms"]
    return {"bytes_per_step": rep["swap"]["bytes"], "bytes_moved_per_step": rep["swap"]["bytes_moved"],
            "stall_ms": stall, "transfer_ms": xfer_ms,
            "link_gbs": xfer_bytes / (xfer_ms * 1e6) if xfer_ms > 0 else None,
            "overlap_frac": 1.0 - stall / xfer_ms if xfer_ms > 0 else None}


def _traffic(workload):
    """Mean DRAM bytes per conv_tc launch of the workload from the round's
    ncu launch list (tools/conv_traffic.py -> profiles/conv_traffic.json)."""
    tpath = os.path.join(ROOT, "profiles", "conv_traffic.json")
    return json.load(open(tpath)).get(workload) if os.path.exists(tpath) else None


def workload_config(args, world) -> dict:
    """`config` of the JSON line -- identical for both arms (the reference
    arm times a bounded sample of this same workload, see SAMPLES)."""
    T = int(WORKLOADS[args.workload].get("run.frames", 8))
    return {"workload": DESCR[args.workload], "frames_per_step": T,
            "parallelism": (f"decode sharded x{world}" if args.workload == "D" else
                            (f"{world} replicas (one video per GPU)" if world > 1 else "single GPU")),
            "l2": "working set per step > 126 MB L2 (inputs larger than L2)",
            "decode_slice_frames": args.decode_slice}


# ---------------------------------------------------------------- GPU arm
def gpu_arm(args, world, rank, local):
    import numpy as np

    import paper_2510_05367_b200 as lc
    over = WORKLOADS[args.workload]
    text = lc.config_text(over, base=lc.DEFAULT_CONFIG)
    kv = lc.parse_config(text)
    T = int(kv["run.frames"])
    ctx = lc.Context(local)
    free0, total_mem = ctx.mem_info()
    ctx.configure(text)
    ctx.set_decode_slice(args.decode_slice)
    n_lat, n_vid = ctx.latent_elems(), ctx.video_elems()
    x0 = lc.PinnedArray(n_lat)
    x0.array[:] = lc.randn(lc.derive_seed(int(kv["run.seed"]), 1), n_lat)  # pipeline.cpp:115
    vid = lc.PinnedArray(n_vid)
    clocks = ClockSampler(local).start()

    # ---- device-resident throughput (value)
    ctx.upload_latent(x0.array)
    for _ in range(args.warmup):
        rep = ctx.run_resident()
    free1, _ = ctx.mem_info()
    barrier(world)
    ctx.timer_start()
    for _ in range(args.steps):
        ctx.run_resident_async()  # graph replays queued back to back
    rep = ctx.wait()
    launches = rep["kernel_launches"] * args.steps
    ms = ctx.timer_stop()
    ms = allmax(world, ms)
    barrier(world)
    value = world * T * args.steps / (ms / 1000.0)

    # ---- end to end through the C-ABI with pinned host buffers
    for _ in range(max(1, args.warmup // 2)):
        ctx.run_e2e(x0, vid)
    barrier(world)
    ctx.timer_start()
    for _ in range(args.steps):
        ctx.run_e2e_async(x0, vid)  # H2D latent + run + D2H video, queued back to back
    rep_e = ctx.wait()
    ms_e = allmax(world, ctx.timer_stop())
    e2e = world * T * args.steps / (ms_e / 1000.0)
    clk = clocks.stop()
    finite = bool(np.isfinite(vid.array).all())

    # ---- roofline of the dominant kernel (tensor-core conv), CUDA events
    # around every conv launch of one extra step (not part of the timing)
    ctx.set_conv_profile(True)
    ctx.run_resident()
    prof = ctx.conv_profile()
    ctx.set_conv_profile(False)
    peak, peak_src = peaks()
    achieved = prof["alg_flops"] / (prof["ms"] / 1000.0) / 1e12 if prof["ms"] > 0 else 0.0
    executed = prof["exec_flops"] / (prof["ms"] / 1000.0) / 1e12 if prof["ms"] > 0 else 0.0
    traffic = _traffic(args.workload)

    # ---- uncached GPU anchor: RunConfig::baseline() (config.cpp:148-156)
    base_text = lc.config_text(dict(over, **{"cache.enabled": "false", "chunk.enabled": "false",
                                             "decode.sliced": "false", "swap.mode": "off"}), base=lc.DEFAULT_CONFIG)
    ctx.configure(base_text)
    ctx.upload_latent(x0.array)
    for _ in range(max(3, args.warmup)):  # eager, graph capture, replay
        ctx.run_resident()
    ctx.timer_start()
    nb = max(1, args.steps // 2)
    for _ in range(nb):
        ctx.run_resident_async()
    rep_b = ctx.wait()
    ms_b = allmax(world, ctx.timer_stop())
    uncached = {"value": world * T * nb / (ms_b / 1000.0), "unit": "frames/s",
                "hbm_peak_gb": rep_b["hbm_peak_bytes"] / 1e9, "denoiser_macs": rep_b["mac"]["denoiser_total"]}
    x0.free()
    vid.free()
    ctx.close()

    sharded = decode_sharded_leg(args, world, rank, local) if world > 1 and not args.plumbing_test else None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_measure(args.workload)
        line = {
            "metric": "video_frames_per_sec", "value": value, "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "fp16 (fp32 accumulate; fp32 latent, sampler and video)",
            "data": "synthetic (seeded randn latent, random-init weights of the reference architecture)",
            "config": workload_config(args, world),
            "hbm_peak_gb": rep["hbm_peak_bytes"] / 1e9,
            "hbm_peaks_by_stage_gb": {k: v["fast"] / 1e9 for k, v in rep["peaks"].items()},
            "cuda_mem_in_use_gb": (free0 - free1) / 1e9,
            "cuda_mem_note": "cudaMemGetInfo drop from context creation to after warm-up (ledger buffers + "
                             "CUDA graph and allocator overhead); hbm_peak_gb is the engine ledger's peak",
            "uncached": uncached,
            "speedup_vs_uncached": value / uncached["value"],
            "denoise_ms": rep["device_ms"]["denoise"], "decode_ms": rep["device_ms"]["decode"],
            "swap": dict(swap_summary(rep), **{"schedule": rep.get("swap_schedule")}),
            "e2e": {"value": e2e, "unit": "frames/s", "h2d_bytes_per_step": n_lat * 4,
                    "d2h_bytes_per_step": n_vid * 4},
            "roofline": {"bound": "tensor", "kernel": "conv_tc_kernel (tcgen05 implicit-GEMM conv)",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "executed_mma_tflops": executed, "executed_frac": executed / peak,
                         "note": "achieved counts the reference's MACs (9-tap conv over the upsampled "
                                 "concat); the sub-pixel and tap-to-N forms issue fewer MMA FLOPs, so "
                                 "frac can exceed 1 -- executed_frac is the hardware-side figure",
                         "launches_per_step": prof["launches"],
                         "conv_ms_per_step": prof["ms"],
                         "conv_share_of_step": prof["ms"] / (ms / args.steps)},
            "gpu_launches": launches,
            "clocks": clk,
            "video_finite": finite,
        }
        if sharded:
            line["decode_sharded"] = sharded
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)


def _nccl_ctx(lc, ctx, world, rank):
    import torch.distributed as dist
    uid = [lc.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    ctx.nccl_init(uid[0], world, rank)


def decode_sharded_leg(args, world, rank, local, steps=None):
    """Workload D over all ranks: lc_decode_sharded (balanced frame blocks,
    per-slice NCCL sends to rank 0).  value: frames / device time of (shard
    H2D + decode + gather), max over ranks; e2e: every rank also downloads
    its frames into one shared pinned host video (parallel host links)."""
    import numpy as np

    import paper_2510_05367_b200 as lc
    steps = steps or args.steps
    text = lc.config_text(WORKLOADS["D"], base=lc.DEFAULT_CONFIG)
    kv = lc.parse_config(text)
    T, s = int(kv["run.frames"]), 1 << int(kv["codec.stages"])
    H, W = int(kv["run.height"]), int(kv["run.width"])
    ctx = lc.Context(local)
    ctx.configure(text)
    if world > 1:
        _nccl_ctx(lc, ctx, world, rank)
    lat = lc.randn(lc.derive_seed(int(kv["run.seed"]), 1), T * 4 * (H // s) * (W // s))
    lat_p = lc.PinnedArray(lat.size)
    lat_p.array[:] = lat
    name = f"lc_bench_video_{os.environ.get('MASTER_PORT', '0')}"
    host_shared = False
    if world > 1:
        import shutil
        import torch.distributed as dist
        # one shared page-locked video (every rank downloads its own frames)
        # when /dev/shm can hold it; otherwise rank 0 downloads the gathered
        # video into its own pinned buffer
        try:
            host_shared = shutil.disk_usage("/dev/shm").free > 2 * T * 3 * H * W * 4
        except OSError:
            host_shared = False
        if host_shared:
            if rank == 0:
                shared = lc.SharedVideo(name, T * 3 * H * W, create=True)
            dist.barrier()
            if rank != 0:
                shared = lc.SharedVideo(name, T * 3 * H * W, create=False)
        else:
            shared = lc.PinnedArray(T * 3 * H * W) if rank == 0 else None
    else:
        shared = lc.PinnedArray(T * 3 * H * W)
    sl = max(d for d in range(1, 6) if T % d == 0) if args.workload != "D" else args.decode_slice
    for _ in range(max(3, args.warmup)):
        ctx.decode_sharded(lat_p, sl)
    barrier(world)
    dev_ms = 0.0
    launches = 0
    for _ in range(steps):
        _, ms = ctx.decode_sharded(lat_p, sl)  # device resident: the gathered video stays in rank 0's HBM
        dev_ms += ms
        launches += ctx.kernel_launches()
    dev_ms = allmax(world, dev_ms)
    for _ in range(2):
        ctx.decode_sharded(lat_p, sl, out=shared, host_shared=host_shared)
    barrier(world)
    e2e_ms = 0.0
    for _ in range(steps):
        _, ms = ctx.decode_sharded(lat_p, sl, out=shared, host_shared=host_shared)
        e2e_ms += ms
    e2e_ms = allmax(world, e2e_ms)
    barrier(world)
    finite = bool(np.isfinite(shared.array).all()) if rank == 0 else None
    barrier(world)
    if shared is not None:
        shared.free()
    lat_p.free()
    ctx.close()
    return {"workload": DESCR["D"], "n_gpus": world, "steps": steps, "decode_slice_frames": sl,
            "value": T * steps / (dev_ms / 1e3), "unit": "frames/s", "ms_per_step": dev_ms / steps,
            "scaling": "strong",
            "e2e": {"value": T * steps / (e2e_ms / 1e3), "unit": "frames/s",
                    "h2d_bytes_per_step": T * 4 * (H // s) * (W // s) * 4, "d2h_bytes_per_step": T * 3 * H * W * 4,
                    "note": ("each rank H2Ds its latent block and D2Hs its own frames into one shared pinned video"
                             if host_shared else "each rank H2Ds its latent block; rank 0 D2Hs the gathered video")},
            "gpu_launches": launches, "video_finite": finite}


def decode_arm(args, world, rank, local):
    """Workload D (BASELINE.json configs[3]) as the headline workload: the
    sharded sliced decode over the launch's N GPUs (strong scaling)."""
    import paper_2510_05367_b200 as lc
    clocks = ClockSampler(local).start()
    d = decode_sharded_leg(args, world, rank, local)
    clk = clocks.stop()
    # roofline: the decoder convs of one single-GPU 5-frame decode, event-timed
    text = lc.config_text(WORKLOADS["D"], base=lc.DEFAULT_CONFIG)
    kv = lc.parse_config(text)
    s = 1 << int(kv["codec.stages"])
    ctx = lc.Context(local)
    ctx.configure(text)
    lat = lc.randn(7, 5 * 4 * (int(kv["run.height"]) // s) * (int(kv["run.width"]) // s)).reshape(
        1, 5, 4, int(kv["run.height"]) // s, int(kv["run.width"]) // s)
    ctx.set_conv_profile(True)
    ctx.decode(lat, args.decode_slice)
    prof = ctx.conv_profile()
    ctx.set_conv_profile(False)
    ctx.close()
    peak, peak_src = peaks()
    achieved = prof["alg_flops"] / (prof["ms"] / 1e3) / 1e12 if prof["ms"] > 0 else 0.0
    if rank == 0:
        line = {
            "metric": "video_frames_per_sec", "value": d["value"], "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": d["ms_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "fp16 (fp32 accumulate; fp32 latent and video)",
            "data": "synthetic (seeded randn latent, random-init codec weights of the reference architecture)",
            "config": workload_config(args, world), "e2e": d["e2e"],
            "roofline": {"bound": "tensor", "kernel": "conv_tc_kernel (decoder convs)", "achieved": achieved,
                         "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                         "traffic": _traffic("D"), "peak_source": peak_src},
            "gpu_launches": d["gpu_launches"], "clocks": clk, "video_finite": d["video_finite"],
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_measure("D")
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="lightcache", choices=["lightcache", "reference"])
    ap.add_argument("--workload", default="C", choices=sorted(WORKLOADS),
                    help="C (default): the largest single-GPU configuration of BASELINE.json")
    ap.add_argument("--decode-slice", type=int, default=None,
                    help="frames per decoder slice (default: config A's 4 slices of 2 frames; otherwise the "
                         "largest divisor of the frame count <= 5: B 4, C/D 5 -- even slices, no 1-frame tail)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--plumbing-test", action="store_true",
                    help="(testing only) every rank on GPU 0 and no NCCL leg: exercises the N > 1 host plumbing "
                         "(spawn, barriers, max over ranks) on a one-GPU box; not a measurement")
    args = ap.parse_args()
    if args.decode_slice is None:
        T = int(WORKLOADS[args.workload].get("run.frames", 8))
        args.decode_slice = 2 if args.workload == "A" else max(d for d in range(1, 6) if T % d == 0)
    if args.warmup < 3 and args.impl != "reference":
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    world, rank, local = dist_init()
    if args.plumbing_test:
        local = 0
    if args.impl == "reference":
        reference_arm(args, world, rank)
    elif args.workload == "D":
        decode_arm(args, world, rank, local)
    else:
        gpu_arm(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
