"""Run artifacts, CLI commands and the comparison harness (SURVEY.md §8 f2,
f4) on the GPU engine.

Mirrors the reference's drivers and writers over the C-ABI:

* ``write_run_artifacts`` -- report.json (``run_report_json``,
  proj/src/pipeline.cpp:230-259), ledger.json / ledger.csv
  (``write_ledger_json`` / ``write_ledger_csv``, proj/src/ledger.cpp:200-242),
  video.raw + video.raw.hdr (``write_video_raw``, proj/src/codec.cpp:172-182);
* ``compare`` / ``ablate`` / ``sweep_n`` / ``export_plots``
  (proj/src/pipeline.cpp:278-376) with per-frame PSNR / SSIM computed on the
  GPU (``Context.video_metrics``);
* JSON layouts of ``compare_row_json`` / ``ablation_table_json`` /
  ``sweep_table_json`` (proj/src/pipeline.cpp:378-420): nlohmann's ``dump(2)``
  with its sorted keys.

Timing columns (``wall_seconds``, ``speed_up``, ``wall_total``) are the
engine's device-timed stage times of the measured run (CUDA events), after
one warm-up run of the same configuration (graph capture); the reference
uses host wall clock of its single run.
"""
import json
import os
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import (DEFAULT_CONFIG, ConfigError, Context, check_config, config_text, lib, normalize_config, parse_config,
               _check, I64)
import ctypes

STAGES = ("setup", "encode", "denoise", "decode")

# config_to_json (proj/src/config.cpp:267-301): section, JSON name, type
_SCHEMA = {
    "run.frames": ("run", "frames", int), "run.height": ("run", "height", int),
    "run.width": ("run", "width", int), "run.seed": ("run", "seed", int), "run.mode": ("run", "mode", str),
    "run.out_dir": ("run", "out_dir", str),
    "unet.depth": ("unet", "depth", int), "unet.base_channels": ("unet", "base_channels", int),
    "unet.kernel": ("unet", "kernel", int), "unet.cache_depth": ("unet", "cache_depth", int),
    "unet.weight_seed": ("unet", "weight_seed", int),
    "codec.latent_channels": ("codec", "latent_channels", int), "codec.stages": ("codec", "stages", int),
    "codec.width": ("codec", "width", int), "codec.weight_seed": ("codec", "weight_seed", int),
    "schedule.train_steps": ("schedule", "train_steps", int),
    "schedule.beta_min": ("schedule", "beta_min", float), "schedule.beta_max": ("schedule", "beta_max", float),
    "sampler.kind": ("sampler", "kind", str), "sampler.steps": ("sampler", "steps", int),
    "sampler.guidance": ("sampler", "guidance", float),
    "cache.enabled": ("cache", "enabled", bool), "cache.n": ("cache", "n", int),
    "swap.mode": ("swap", "mode", str), "swap.simulate": ("swap", "simulate", bool),
    "swap.bandwidth": ("swap", "bandwidth", float), "swap.latency": ("swap", "latency", float),
    "swap.mac_rate": ("swap", "mac_rate", float),
    "chunk.enabled": ("chunk", "enabled", bool), "chunk.eta": ("chunk", "eta", int),
    "chunk.omega": ("chunk", "omega", int), "chunk.halo": ("chunk", "halo", str),
    "chunk.halo_px": ("chunk", "halo_px", int), "chunk.targets": ("chunk", "targets", list),
    "decode.sliced": ("decode", "sliced", bool), "budget.fast_bytes": ("budget", "fast_bytes", int),
}


def config_json(text: str) -> dict:
    """config_to_json of a config text (every key typed as the reference)."""
    out: Dict[str, dict] = {}
    for k, v in parse_config(text).items():
        if k not in _SCHEMA:
            continue
        sec, name, typ = _SCHEMA[k]
        if typ is bool:
            val = v.lower() in ("true", "1", "yes", "on")
        elif typ is list:
            val = [t.strip() for t in v.split(",") if t.strip()]
        else:
            val = typ(v)
        out.setdefault(sec, {})[name] = val
    return out


def baseline_text(text: str) -> str:
    """RunConfig::baseline() (proj/src/config.cpp:148-156)."""
    return config_text({"cache.enabled": "false", "chunk.enabled": "false", "decode.sliced": "false",
                        "swap.mode": "off", "budget.fast_bytes": "0"}, base=normalize_config(text))


def dumps(obj) -> str:
    """nlohmann::json::dump(2): two-space indent, keys sorted."""
    return json.dumps(obj, indent=2, sort_keys=True)


class RunResult:
    """What run_pipeline returns on the host side (pipeline.hpp:18-39)."""

    def __init__(self, text: str, video: np.ndarray, rep: dict):
        self.text, self.video, self.rep = text, video, rep
        dm = rep["device_ms"]
        self.wall = {"setup": 0.0, "encode": max(0.0, dm["total"] - dm["denoise"] - dm["decode"]) / 1e3,
                     "denoise": dm["denoise"] / 1e3, "decode": dm["decode"] / 1e3, "total": dm["total"] / 1e3}
        self.peaks = rep["peaks"]
        self.denoiser_macs = rep["mac"]["denoiser_total"]


def run_pipeline(ctx: Context, text: str, repeats: int = 2) -> RunResult:
    """run_pipeline on the GPU; the last of `repeats` runs is reported (the
    first run of a new configuration captures the CUDA graph)."""
    ctx.configure(text)
    video = rep = None
    for _ in range(max(1, repeats)):
        video, _, rep = ctx.run_pipeline()
    return RunResult(text, video, rep)


def ledger_csv(ctx: Context) -> str:
    need = I64()
    _check(lib().lc_ledger_csv(ctx._h, None, I64(0), ctypes.byref(need)))
    buf = ctypes.create_string_buffer(int(need.value) + 16)
    _check(lib().lc_ledger_csv(ctx._h, buf, I64(len(buf)), ctypes.byref(need)))
    return buf.value.decode()


def ledger_summary(ctx: Context) -> dict:
    buf = ctypes.create_string_buffer(1 << 16)
    _check(lib().lc_ledger_summary(ctx._h, buf, I64(len(buf))))
    return json.loads(buf.value.decode())


def run_report(res: RunResult) -> dict:
    """run_report_json (proj/src/pipeline.cpp:230-259)."""
    rep = res.rep
    j = {
        "config": config_json(res.text),
        "wall_seconds": res.wall,
        "peaks": {s: {"fast": rep["peaks"][s]["fast"], "slow": rep["peaks"][s]["slow"]} for s in STAGES},
        "overall_peak": {t: max(rep["peaks"][s][t] for s in STAGES) for t in ("fast", "slow")},
        "mac": {k: rep["mac"][k] for k in ("denoiser_total", "per_full_step", "per_cached_step", "full_steps",
                                           "cached_steps")},
        "cache_bytes": rep["cache_bytes"],
        "timeline": {"makespan_seconds": rep["timeline"]["makespan_ms"] / 1e3,
                     "stall_seconds": rep["timeline"]["stall_ms"] / 1e3,
                     "simulated": bool(rep["timeline"].get("simulated", False))},
        "video": {"frames": rep["video"]["frames"], "channels": rep["video"]["channels"],
                  "height": rep["video"]["height"], "width": rep["video"]["width"]},
    }
    return j


def write_video_raw(path: str, video: np.ndarray) -> None:
    """write_video_raw (proj/src/codec.cpp:172-182): raw fp32 {t,c,h,w} and a
    "t c h w" header next to it."""
    v = np.ascontiguousarray(video, dtype=np.float32)
    if v.ndim == 5:
        if v.shape[0] != 1:
            raise ValueError("write_video_raw expects b == 1")
        v = v[0]
    v.tofile(path)
    with open(path + ".hdr", "w") as f:
        f.write(f"{v.shape[0]} {v.shape[1]} {v.shape[2]} {v.shape[3]}\n")


def read_video_raw(path: str) -> np.ndarray:
    """read_video_raw (proj/src/codec.cpp:184-196) -> (1,t,c,h,w)."""
    with open(path + ".hdr") as f:
        t, c, h, w = (int(x) for x in f.read().split())
    v = np.fromfile(path, np.float32)
    if v.size != t * c * h * w:
        raise ValueError("short read from " + path)
    return v.reshape(1, t, c, h, w)


def write_run_artifacts(ctx: Context, res: RunResult, out_dir: str) -> None:
    """write_run_artifacts (proj/src/pipeline.cpp:261-276)."""
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, "report.json"), "w") as f:
        f.write(dumps(run_report(res)) + "\n")
    led = ledger_summary(ctx)
    led["run"] = {"makespan_seconds": res.rep["timeline"]["makespan_ms"] / 1e3,
                  "stall_seconds": res.rep["timeline"]["stall_ms"] / 1e3, "denoiser_macs": res.denoiser_macs}
    with open(os.path.join(out_dir, "ledger.json"), "w") as f:
        f.write(dumps(led) + "\n")
    with open(os.path.join(out_dir, "ledger.csv"), "w") as f:
        f.write(ledger_csv(ctx))
    write_video_raw(os.path.join(out_dir, "video.raw"), res.video)


# ------------------------------------------------------------- harness
def _series(ctx: Context, a: np.ndarray, b: np.ndarray):
    ps, ss = ctx.video_metrics(a[0], b[0], 1.0)
    return ps, ss


def compare(ctx: Context, baseline: str, variant: str) -> dict:
    """compare (proj/src/pipeline.cpp:278-297) -> compare_row_json."""
    kb, kv = parse_config(baseline), parse_config(variant)
    for k in ("run.frames", "run.height", "run.width", "run.mode", "codec.latent_channels", "codec.stages",
              "codec.width"):
        if kb[k] != kv[k]:
            raise ConfigError(f"compare: configs differ in {k}")
    base = run_pipeline(ctx, baseline)
    var = run_pipeline(ctx, variant)
    ps, ss = _series(ctx, base.video, var.video)
    return {
        "speed_up": base.wall["total"] / var.wall["total"],
        "psnr_mean": float(ps.mean()), "ssim_mean": float(ss.mean()),
        "psnr_per_frame": [float(x) for x in ps], "ssim_per_frame": [float(x) for x in ss],
        "variant_macs": var.denoiser_macs, "baseline_macs": base.denoiser_macs,
        "identical_video": base.video.tobytes() == var.video.tobytes(),
        "peak_delta_fast": {s: var.peaks[s]["fast"] - base.peaks[s]["fast"] for s in STAGES},
    }


def ablate(ctx: Context, text: str) -> List[dict]:
    """ablate (proj/src/pipeline.cpp:299-331) -> ablation_table_json rows."""
    kv = parse_config(text)
    on = lambda k: kv[k].lower() in ("true", "1", "yes", "on")  # noqa: E731
    if not (on("cache.enabled") and on("chunk.enabled") and on("decode.sliced") and kv["swap.mode"] != "off"):
        raise ConfigError("ablate: base config must enable cache, swap, chunk and slicing")
    baseline = run_pipeline(ctx, baseline_text(text))
    rows = []
    norm = normalize_config(text)
    for label, over in [("all-on", {}), ("-swapping", {"swap.mode": "off"}), ("-slicing", {"decode.sliced": "false"}),
                        ("-chunk", {"chunk.enabled": "false"}),
                        ("cache-only", {"swap.mode": "off", "decode.sliced": "false", "chunk.enabled": "false"})]:
        r = run_pipeline(ctx, config_text(over, base=norm))
        ps, ss = _series(ctx, baseline.video, r.video)
        rows.append({"label": label, "wall_total": r.wall["total"], "psnr_mean": float(ps.mean()),
                     "ssim_mean": float(ss.mean()), "peak_fast": {s: r.peaks[s]["fast"] for s in STAGES}})
    return rows


def sweep_n(ctx: Context, text: str, ns: Sequence[int]) -> dict:
    """sweep_n (proj/src/pipeline.cpp:333-360) -> sweep_table_json."""
    for i in range(1, len(ns)):
        if ns[i] <= ns[i - 1]:
            raise ConfigError("sweep-n: N values must be ascending")
    baseline = run_pipeline(ctx, baseline_text(text))
    norm = normalize_config(text)
    rows = []
    for n in ns:
        r = run_pipeline(ctx, config_text({"cache.enabled": "true", "cache.n": n}, base=norm))
        ps, ss = _series(ctx, baseline.video, r.video)
        rows.append({"n": int(n), "speed_up": baseline.wall["total"] / r.wall["total"],
                     "psnr_mean": float(ps.mean()), "ssim_mean": float(ss.mean()), "macs": r.denoiser_macs})
    speed_mono = all(rows[i]["speed_up"] >= rows[i - 1]["speed_up"] for i in range(1, len(rows)))
    qual_mono = all(rows[i]["psnr_mean"] <= rows[i - 1]["psnr_mean"] and
                    rows[i]["ssim_mean"] <= rows[i - 1]["ssim_mean"] for i in range(1, len(rows)))
    return {"rows": rows, "speed_monotone": speed_mono, "quality_monotone": qual_mono}


def metrics_csv(ps, ss) -> str:
    """write_metrics_csv (proj/src/metrics.cpp:106-117): precision(10)."""
    lines = ["frame_index,psnr,ssim"]
    lines += [f"{i},{p:.10g},{s:.10g}" for i, (p, s) in enumerate(zip(ps, ss))]
    return "\n".join(lines) + "\n"


def export_plots(ctx: Context, text: str, ns: Sequence[int], out_dir: str) -> List[str]:
    """export_plots (proj/src/pipeline.cpp:362-376)."""
    os.makedirs(out_dir, exist_ok=True)
    baseline = run_pipeline(ctx, baseline_text(text))
    norm = normalize_config(text)
    paths = []
    for n in ns:
        r = run_pipeline(ctx, config_text({"cache.enabled": "true", "cache.n": n}, base=norm))
        ps, ss = _series(ctx, baseline.video, r.video)
        path = os.path.join(out_dir, f"metrics_n{int(n)}.csv")
        with open(path, "w") as f:
            f.write(metrics_csv(ps, ss))
        paths.append(path)
    return paths


def build_config(config_path: Optional[str], overrides: Sequence[str], out_dir: Optional[str]) -> str:
    """build_config (proj/tools/main.cpp:16-29): default_config(), the file,
    --set key=value overrides, --out; validated like the reference."""
    text = DEFAULT_CONFIG
    if config_path:
        with open(config_path) as f:
            text = text + "\n" + f.read()
    over = {}
    for kv in overrides or []:
        if "=" not in kv:
            raise ConfigError(f"--set expects key=value, got '{kv}'")
        k, v = kv.split("=", 1)
        over[k] = v
    if out_dir:
        over["run.out_dir"] = out_dir
    text = normalize_config(config_text(over, base=text))
    check_config(text)  # RunConfig::validate (proj/src/config.cpp:100-146)
    return text
