#!/usr/bin/env python
"""Benchmark of the B200-native LightCache path.

Metric (BASELINE.json): end-to-end video frames/sec (+ peak HBM GB) against
the uncached GPU run and the CPU reference.  One "step" is one whole video
generation -- run_pipeline (proj/src/pipeline.cpp:64): the denoise loop with
the feature cache / async swap / chunked execution, then sliced decode --
on the workload BASELINE.json quotes at one GPU (configs[1], config B):
AnimateDiff-Lightning-shaped U-Net, 16 frames, latent 4x64x64, 4 Euler
steps, N=2, base 320, synthetic latent and random-init weights.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload B|C|A]
  python bench.py --impl reference ...     (CPU reference arm)
  torchrun --nproc-per-node N bench.py --gpus N   (N replicas, weak scaling)

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
    "C": "SVD-XT-shaped U-Net: 25 frames, latent 4x72x128 (1024x576 video), 25 Euler steps, cache N=2, "
         "async swap, chunk u0 2x2, sliced decode, base 320, depth 3, codec W=128 S=3",
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
        dist.init_process_group("gloo", rank=rank, world_size=world)
    return world, rank, local


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
        return d.get("bf16_tflops_sustained", 1392.2), "measured (MEASURED_PEAKS.json bf16 sustained; fp16 same rate)"
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


def run_macs(lc, text: str, kv: dict) -> int:
    mf, mc, _ = lc.model_numbers(text)
    S, N = int(kv["sampler.steps"]), int(kv["cache.n"])
    enabled = kv["cache.enabled"] in ("true", "on", "1")
    nf = sum(1 for s in range(S) if (not enabled) or s % N == 0)
    return nf * mf + (S - nf) * mc + decode_macs(kv, int(kv["run.frames"]))


# ---------------------------------------------------------------- CPU arm
def cpu_sample_config(over: dict) -> dict:
    """Bounded sample of the workload: one frame at 1/16 of the latent area
    (latent 16x16 for B), same channels/depth/steps/cache plan; the work
    is linear in frames x pixels, so frames/s is extrapolated by the exact
    MAC ratio (conv MACs per tensor.cpp:194-195, decode per codec.cpp)."""
    s = dict(over)
    s["run.frames"] = 1
    scale = 1 << int(s.get("codec.stages", 2))
    depth = 1 << int(s.get("unet.depth", 3))
    # 16x16 latent (>= 2^depth and divisible by eta/omega of the chunk)
    s["run.height"] = 16 * scale
    s["run.width"] = 16 * scale
    return s


def _cpu_worker(args):
    text, kind = args
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import lco
    kv = lco.parse_text(text)
    t = time.time()
    if kind == "reference":
        lco.Reference().run_pipeline(kv)
    else:
        os.environ.setdefault("OMP_NUM_THREADS", "1")
        lco.Restatement().run_pipeline(kv)
    return time.time() - t


def cpu_measure(lc, over: dict, workers: int, reps: int):
    """Time the reference CPU path on the bounded sample; returns
    (frames/s extrapolated to the full workload, kind, sample description)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import lco
    kind = "reference" if lco.Reference.available() else "port"
    full_text = lc.config_text(over, base=lc.DEFAULT_CONFIG)
    samp = cpu_sample_config(over)
    samp_text = lc.config_text(samp, base=lc.DEFAULT_CONFIG)
    kv_full = lco.parse_text(full_text)
    kv_s = lco.parse_text(samp_text)
    macs_full = run_macs(lc, full_text, kv_full) / int(kv_full["run.frames"])
    macs_s = run_macs(lc, samp_text, kv_s)
    times = []
    if workers <= 1:
        for _ in range(reps):
            times.append(_cpu_worker((lco.to_text(kv_s), kind)))
        per_sample = statistics.median(times)
        fps_sample = 1.0 / per_sample
    else:
        import multiprocessing as mp
        with mp.get_context("fork").Pool(workers) as pool:
            t0 = time.time()
            for _ in range(reps):
                pool.map(_cpu_worker, [(lco.to_text(kv_s), kind)] * workers)
            wall = time.time() - t0
        fps_sample = workers * reps / wall
        per_sample = wall / reps
    fps = fps_sample * macs_s / macs_full
    desc = (f"1 frame at latent {kv_s['run.height']}x{kv_s['run.width']} pixels/{1 << int(kv_s['codec.stages'])} "
            f"(same channels, depth, {kv_s['sampler.steps']} steps, N={kv_s['cache.n']}), "
            f"{macs_s / 1e9:.2f} GMAC vs {macs_full / 1e9:.1f} GMAC per full-size frame; "
            f"{per_sample:.1f} s per sample; frames/s extrapolated by the MAC ratio")
    return fps, kind, desc


def _cpu_decode_worker(text):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np

    import lco
    kv = lco.parse_text(text)
    s = 1 << int(kv["codec.stages"])
    lat = np.random.default_rng(0).standard_normal(
        (1, 1, 4, int(kv["run.height"]) // s, int(kv["run.width"]) // s)).astype(np.float32)
    lib = lco.Reference() if lco.Reference.available() else lco.Restatement()
    t = time.time()
    lib.decode(kv, lat)
    return time.time() - t


def reference_arm(args, world, rank):
    import paper_2510_05367_b200 as lc
    if rank != 0:
        return
    over = WORKLOADS[args.workload]
    workers = min(os.cpu_count() or 1, 64)
    if args.workload == "D":
        # the reference's decode of one frame per host process (decode is frame-wise)
        import multiprocessing as mp
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import lco
        kind = "reference" if lco.Reference.available() else "port"
        text = lc.config_text(over, base=lc.DEFAULT_CONFIG)
        with mp.get_context("fork").Pool(workers) as pool:
            t0 = time.time()
            for _ in range(max(1, args.steps // 10)):
                pool.map(_cpu_decode_worker, [text] * workers)
            wall = time.time() - t0
        fps = workers * max(1, args.steps // 10) / wall
        desc = f"1 frame decoded per host process, {workers} processes, {max(1, args.steps // 10)} rounds"
    else:
        # each round = one bounded sample per host process (~10 s); capped so
        # the arm ends within a few minutes whatever --steps is
        fps, kind, desc = cpu_measure(lc, over, workers, min(args.steps, 8))
    line = {"metric": "video_frames_per_sec", "value": fps, "unit": "frames/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * WORKLOADS_FRAMES(over) / fps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
            "data": "synthetic (seeded randn latent, random-init weights)",
            "config": {"workload": DESCR[args.workload], "parallelism": f"{workers} CPU processes"},
            "impl": "reference",
            "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": workers, "kind": kind, "sample": desc},
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


def WORKLOADS_FRAMES(over):
    return int(over.get("run.frames", 8))


# ---------------------------------------------------------------- GPU arm
def gpu_arm(args, world, rank, local):
    import numpy as np

    import paper_2510_05367_b200 as lc
    over = WORKLOADS[args.workload]
    text = lc.config_text(over, base=lc.DEFAULT_CONFIG)
    kv = lc.parse_config(text)
    T = int(kv["run.frames"])
    ctx = lc.Context(local)
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
    barrier(world)
    ctx.timer_start()
    launches = 0
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
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "conv_traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(args.workload)

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

    line = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            fps, kind, desc = cpu_measure(lc, over, 1, 1)
            cpu = {"value": fps, "unit": "frames/s", "cores": 1, "kind": kind, "sample": desc}
        line = {
            "metric": "video_frames_per_sec", "value": value, "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "fp16 (fp32 accumulate; fp32 latent, sampler and video)",
            "data": "synthetic (seeded randn latent, random-init weights of the reference architecture)",
            "config": {"workload": DESCR[args.workload], "frames_per_step": T,
                       "parallelism": "replicas" if world > 1 else "single GPU",
                       "l2": "working set per step ~0.9 GB > 126 MB L2 (inputs larger than L2)",
                       "decode_slice_frames": args.decode_slice},
            "hbm_peak_gb": rep["hbm_peak_bytes"] / 1e9,
            "uncached": uncached,
            "speedup_vs_uncached": value / uncached["value"],
            "denoise_ms": rep["device_ms"]["denoise"], "decode_ms": rep["device_ms"]["decode"],
            "swap": swap_summary(rep),
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
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    x0.free()
    vid.free()
    ctx.close()


def decode_arm(args, world, rank, local):
    """Workload D (BASELINE.json configs[3]): sliced decode sharded over N
    GPUs (lc_decode_sharded: contiguous frame blocks, grouped NCCL
    send/recv to rank 0).  A step decodes the whole 25-frame latent video;
    value = frames / device time of (latent shard H2D + decode + gather),
    max over ranks; e2e adds the D2H of the full video on rank 0."""
    import numpy as np

    import paper_2510_05367_b200 as lc
    over = WORKLOADS["D"]
    text = lc.config_text(over, base=lc.DEFAULT_CONFIG)
    kv = lc.parse_config(text)
    T, s = int(kv["run.frames"]), 1 << int(kv["codec.stages"])
    H, W = int(kv["run.height"]), int(kv["run.width"])
    ctx = lc.Context(local)
    ctx.configure(text)
    if world > 1:
        import torch.distributed as dist
        uid = [lc.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.nccl_init(uid[0], world, rank)
    lat = lc.randn(lc.derive_seed(int(kv["run.seed"]), 1), T * 4 * (H // s) * (W // s)).reshape(
        1, T, 4, H // s, W // s)
    lat_p = lc.PinnedArray(lat.size)  # pinned host buffers: the API's fast path
    lat_p.array[:] = lat.reshape(-1)
    vid_p = lc.PinnedArray(T * 3 * H * W)
    clocks = ClockSampler(local).start()
    for _ in range(args.warmup):
        ctx.decode_sharded(lat_p, args.decode_slice, out=vid_p)
    barrier(world)
    ctx.timer_start()
    dev_ms = 0.0
    launches = 0
    for _ in range(args.steps):
        video, ms = ctx.decode_sharded(lat_p, args.decode_slice, out=vid_p)
        dev_ms += ms
        launches += ctx.kernel_launches()
    ms_e = allmax(world, ctx.timer_stop())
    dev_ms = allmax(world, dev_ms)
    clk = clocks.stop()
    value = T * args.steps / (dev_ms / 1e3)
    e2e = T * args.steps / (ms_e / 1e3)
    # roofline: the decoder convs of one single-GPU decode, event-timed
    ctx.set_conv_profile(True)
    ctx.decode(lat[:, :min(T, 4)], args.decode_slice)
    prof = ctx.conv_profile()
    ctx.set_conv_profile(False)
    peak, peak_src = peaks()
    achieved = prof["alg_flops"] / (prof["ms"] / 1e3) / 1e12 if prof["ms"] > 0 else 0.0
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            import lco
            kind = "reference" if lco.Reference.available() else "port"
            lib = lco.Reference() if kind == "reference" else lco.Restatement()
            t0 = time.time()
            lib.decode(lco.parse_text(text), lat[:, :1])
            dt = time.time() - t0
            cpu = {"value": 1.0 / dt, "unit": "frames/s", "cores": 1, "kind": kind,
                   "sample": f"1 frame decoded by the {kind} CPU decoder ({dt:.1f} s)"}
        line = {
            "metric": "video_frames_per_sec", "value": value, "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "fp16 (fp32 accumulate; fp32 latent and video)",
            "data": "synthetic (seeded randn latent, random-init codec weights of the reference architecture)",
            "config": {"workload": DESCR["D"], "frames_per_step": T, "parallelism": f"decode sharded x{world}",
                       "l2": "video 177 MB > 126 MB L2 (outputs larger than L2)",
                       "decode_slice_frames": args.decode_slice},
            "e2e": {"value": e2e, "unit": "frames/s", "h2d_bytes_per_step": int(lat.nbytes) // world,
                    "d2h_bytes_per_step": int(video.nbytes)},
            "roofline": {"bound": "tensor", "kernel": "conv_tc_kernel (decoder convs)", "achieved": achieved,
                         "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                         "traffic": None, "peak_source": peak_src},
            "gpu_launches": launches,
            "clocks": clk,
            "video_finite": bool(np.isfinite(video).all()) if rank == 0 else None,
        }
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    lat_p.free()
    vid_p.free()
    ctx.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="lightcache", choices=["lightcache", "reference"])
    ap.add_argument("--workload", default="B", choices=sorted(WORKLOADS))
    ap.add_argument("--decode-slice", type=int, default=None,
                    help="frames per decoder slice (default: config A's 4 slices of 2 frames; otherwise the "
                         "largest divisor of the frame count <= 5: B 4, C/D 5 -- even slices, no 1-frame tail)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.decode_slice is None:
        T = int(WORKLOADS[args.workload].get("run.frames", 8))
        args.decode_slice = 2 if args.workload == "A" else max(d for d in range(1, 6) if T % d == 0)
    if args.warmup < 3 and args.impl != "reference":
        args.warmup = 3
    world, rank, local = dist_init()
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
