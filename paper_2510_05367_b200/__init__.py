"""B200-native LightCache hot path (arXiv 2510.05367) behind the reference's
operator and config API.

The product is the native library ``liblightcache.so`` (CUDA kernels for
sm_100a + C++ host runtime) with the C-ABI declared in ``include/lightcache.h``.
This module is a thin ctypes binding over that C-ABI for tests and the
benchmark; it contains no compute and no fallback: if the shared object is
missing or the GPU is unavailable, calls raise.

Error classes mirror the reference exception hierarchy
(proj/include/stagecache/common.hpp:33-57) and its CLI exit codes
(proj/tools/main.cpp:157-169).
"""
from __future__ import annotations

import ctypes
import json
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblightcache.so")
REPO_ROOT = os.path.dirname(_HERE)
HEADER_PATH = os.path.join(REPO_ROOT, "include", "lightcache.h")


class LightCacheError(RuntimeError):
    code = 1


class ShapeError(LightCacheError):
    code = 1


class ConfigError(LightCacheError):
    code = 2


class BudgetError(LightCacheError):
    code = 3


class InvariantError(LightCacheError):
    code = 4


class DeviceError(LightCacheError):
    code = 5


_ERRORS = {1: ShapeError, 2: ConfigError, 3: BudgetError, 4: InvariantError, 5: DeviceError}

_lib = None


def lib() -> ctypes.CDLL:
    """Load liblightcache.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() (make -C "
                              f"paper_2510_05367_b200/csrc)")
        L = ctypes.CDLL(LIB_PATH)
        L.lc_last_error.restype = ctypes.c_char_p
        L.lc_latent_elems.restype = ctypes.c_int64
        L.lc_video_elems.restype = ctypes.c_int64
        L.lc_derive_seed.restype = ctypes.c_uint64
        L.lc_derive_seed.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        msg = lib().lc_last_error().decode()
        raise _ERRORS.get(rc, LightCacheError)(msg)


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


I64 = ctypes.c_int64

# Every symbol include/lightcache.h declares (checked by tests/test_capi.py).
EXPORTS = [
    "lc_version", "lc_last_error", "lc_ctx_create", "lc_ctx_destroy", "lc_config_check",
    "lc_config_to_text", "lc_configure", "lc_latent_elems", "lc_video_elems", "lc_run_pipeline",
    "lc_upload_latent", "lc_run_resident", "lc_run_resident_async", "lc_run_pipeline_async", "lc_wait", "lc_download_video",
    "lc_set_decode_slice",
    "lc_forward", "lc_decode", "lc_video_metrics", "lc_ledger_csv", "lc_ledger_summary", "lc_conv2d", "lc_up_conv2d", "lc_plan_steps", "lc_split",
    "lc_model_numbers", "lc_simulate_timeline", "lc_derive_seed", "lc_randn", "lc_shard_frames", "lc_nccl_unique_id",
    "lc_nccl_init", "lc_decode_sharded", "lc_gather_plan", "lc_host_register", "lc_host_unregister", "lc_mem_info",
    "lc_get_run_result", "lc_last_error_stage", "lc_plan_arena",
    "lc_timer_start", "lc_timer_stop", "lc_set_conv_profile",
    "lc_conv_profile", "lc_conv_profile_records", "lc_kernel_launches", "lc_alloc_pinned", "lc_free_pinned",
    "lc_sampler_step", "lc_all_finite",
]

# ----------------------------------------------------------------- config
DEFAULT_CONFIG = """\
run.frames = 8
run.height = 64
run.width = 64
run.seed = 42
run.mode = text
unet.depth = 3
unet.base_channels = 8
unet.kernel = 3
unet.cache_depth = 0
unet.weight_seed = 1234
codec.latent_channels = 4
codec.stages = 2
codec.width = 8
codec.weight_seed = 77
schedule.train_steps = 50
schedule.beta_min = 0.002
schedule.beta_max = 0.25
sampler.kind = euler
sampler.steps = 25
sampler.guidance = 1.5
cache.enabled = true
cache.n = 2
swap.mode = async
swap.simulate = false
chunk.enabled = true
chunk.eta = 2
chunk.omega = 2
chunk.halo = exact
chunk.targets = u0
decode.sliced = true
budget.fast_bytes = 0
"""


def config_text(overrides: Optional[dict] = None, base: str = "") -> str:
    """Reference-grammar config text: `base` lines then `key = value` overrides."""
    lines = [base] if base else []
    for k, v in (overrides or {}).items():
        lines.append(f"{k} = {v}")
    return "\n".join(lines) + "\n"


def check_config(text: str) -> None:
    _check(lib().lc_config_check(text.encode()))


def normalize_config(text: str) -> str:
    buf = ctypes.create_string_buffer(1 << 16)
    _check(lib().lc_config_to_text(text.encode(), buf, I64(1 << 16)))
    return buf.value.decode()


def parse_config(text: str) -> dict:
    out = {}
    for line in normalize_config(text).splitlines():
        k, v = line.split("=", 1)
        out[k.strip()] = v.strip()
    return out


def model_numbers(text: str):
    mf, mc, cb = I64(), I64(), I64()
    _check(lib().lc_model_numbers(text.encode(), ctypes.byref(mf), ctypes.byref(mc), ctypes.byref(cb)))
    return mf.value, mc.value, cb.value


TIMELINE_KINDS = ("compute_start", "compute_end", "xfer_start", "xfer_end", "await_start", "await_end")


def simulate_timeline(text: str):
    """Virtual-clock timeline of the simulated transfer engine
    (proj/src/swap.cpp:141-364): (events int64[n, 4] of kind, step, bytes,
    clock_ns; makespan_ns; stall_ns)."""
    n, mk, st = I64(), I64(), I64()
    _check(lib().lc_simulate_timeline(text.encode(), None, I64(0), ctypes.byref(n), None, None))
    ev = np.empty((max(1, n.value), 4), np.int64)
    _check(lib().lc_simulate_timeline(text.encode(), _p(ev), I64(n.value), ctypes.byref(n), ctypes.byref(mk),
                                      ctypes.byref(st)))
    return ev[:n.value], mk.value, st.value


def plan_arena(text: str) -> dict:
    """lc_plan_arena: the lifetime-packed layout of the denoise activations."""
    buf = ctypes.create_string_buffer(1 << 16)
    _check(lib().lc_plan_arena(text.encode(), buf, I64(1 << 16)))
    return json.loads(buf.value.decode())


def plan_steps(total: int, n: int):
    kinds = np.empty(total, np.int8)
    flags = np.empty(total, np.int8)
    _check(lib().lc_plan_steps(I64(total), I64(n), _p(kinds), _p(flags)))
    return kinds, flags


HALO = {"exact": 0, "fixed": 1, "none": 2}


def split(h: int, w: int, eta: int, omega: int, halo: str = "exact", halo_px: int = 0, k: int = 3):
    regions = np.empty(12 * max(1, eta * omega), np.int64)
    halo_out = I64()
    _check(lib().lc_split(I64(h), I64(w), I64(eta), I64(omega), ctypes.c_int(HALO[halo]), I64(halo_px),
                          I64(k), _p(regions), ctypes.byref(halo_out)))
    return regions.reshape(-1, 3, 4), halo_out.value


def derive_seed(seed: int, stream: int) -> int:
    return lib().lc_derive_seed(seed, stream)


def randn(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.float32)
    _check(lib().lc_randn(ctypes.c_uint64(seed), I64(n), _p(out)))
    return out


def shard_frames(T: int, world: int, rank: int):
    f0, cnt = I64(), I64()
    _check(lib().lc_shard_frames(I64(T), ctypes.c_int(world), ctypes.c_int(rank), ctypes.byref(f0),
                                 ctypes.byref(cnt)))
    return f0.value, cnt.value


def gather_plan(T: int, world: int, slice_frames: int) -> np.ndarray:
    """The slice-by-slice gather schedule of lc_decode_sharded: int64 rows of
    (round, rank, first_frame, count)."""
    n = I64()
    _check(lib().lc_gather_plan(I64(T), ctypes.c_int(world), I64(slice_frames), None, I64(0), ctypes.byref(n)))
    rows = np.empty((max(1, n.value), 4), np.int64)
    _check(lib().lc_gather_plan(I64(T), ctypes.c_int(world), I64(slice_frames), _p(rows), I64(n.value),
                                ctypes.byref(n)))
    return rows[:n.value]


SHARD_HOST_SHARED = 1


# ----------------------------------------------------------------- context
class Context:
    """One GPU: streams, packed weights and device buffers (lc_ctx)."""

    def __init__(self, device: int = 0):
        self._h = ctypes.c_void_p()
        _check(lib().lc_ctx_create(ctypes.c_int(device), ctypes.byref(self._h)))
        self.device = device
        self._text = None

    def close(self):
        if self._h:
            lib().lc_ctx_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- configuration
    def configure(self, text: str):
        _check(lib().lc_configure(self._h, text.encode()))
        self._text = text
        return self

    def latent_elems(self) -> int:
        return lib().lc_latent_elems(self._h)

    def video_elems(self) -> int:
        return lib().lc_video_elems(self._h)

    def mem_info(self):
        """(free, total) device bytes (cudaMemGetInfo)."""
        f, t = I64(), I64()
        _check(lib().lc_mem_info(self._h, ctypes.byref(f), ctypes.byref(t)))
        return f.value, t.value

    def set_decode_slice(self, frames: int):
        _check(lib().lc_set_decode_slice(self._h, I64(frames)))

    # -- run_pipeline (proj/src/pipeline.cpp:64)
    def run_pipeline(self, x0: Optional[np.ndarray] = None, want_video=True, want_latent=False):
        cfg = parse_config(self._text)
        T, H, W = int(cfg["run.frames"]), int(cfg["run.height"]), int(cfg["run.width"])
        video = np.empty((1, T, 3, H, W), np.float32) if want_video else None
        lat = np.empty(self.latent_elems(), np.float32) if want_latent else None
        x = None if x0 is None else _f32(x0)
        rep = self._report_buf()
        _check(lib().lc_run_pipeline(self._h, _p(x), _p(video), _p(lat), rep, I64(1 << 22)))
        report = json.loads(rep.value.decode())
        if lat is not None:
            s = 1 << int(cfg["codec.stages"])
            lat = lat.reshape(1, T, int(cfg["codec.latent_channels"]), H // s, W // s)
        return video, lat, report

    def run_result(self) -> dict:
        """Typed RunResult of the last completed run (lc_get_run_result;
        proj/include/stagecache/pipeline.hpp:18-39): StageWall (s),
        StageReport peaks, timeline rows (kind, step, bytes, clock_ns), MAC
        counters, cache_bytes_planned, makespan / stall (s), simulated."""
        class _R(ctypes.Structure):
            _fields_ = ([(n, ctypes.c_double) for n in ("wall_setup", "wall_encode", "wall_denoise", "wall_decode",
                                                        "wall_total")] +
                        [("peak_fast", ctypes.c_int64 * 4), ("peak_slow", ctypes.c_int64 * 4),
                         ("current_fast", ctypes.c_int64), ("current_slow", ctypes.c_int64),
                         ("events_per_stage", ctypes.c_int64 * 4), ("event_count", ctypes.c_int64)] +
                        [(n, ctypes.c_int64) for n in ("denoiser_macs", "macs_per_full_step", "macs_per_cached_step",
                                                       "full_steps", "cached_steps", "cache_bytes_planned")] +
                        [("makespan_s", ctypes.c_double), ("stall_s", ctypes.c_double), ("simulated", ctypes.c_int),
                         ("n_timeline", ctypes.c_int64)])
        r = _R()
        _check(lib().lc_get_run_result(self._h, ctypes.byref(r), None, I64(0)))
        rows = np.empty((max(1, r.n_timeline), 4), np.int64)
        _check(lib().lc_get_run_result(self._h, ctypes.byref(r), _p(rows), I64(r.n_timeline)))
        out = {f: getattr(r, f) for f, _ in _R._fields_}
        for f in ("peak_fast", "peak_slow", "events_per_stage"):
            out[f] = list(out[f])
        out["simulated"] = bool(out["simulated"])
        out["timeline"] = rows[:r.n_timeline]
        return out

    def upload_latent(self, x0: np.ndarray):
        _check(lib().lc_upload_latent(self._h, _p(_f32(x0))))

    def _report_buf(self):
        if getattr(self, "_rep", None) is None:
            self._rep = ctypes.create_string_buffer(1 << 22)
        return self._rep

    def run_resident(self) -> dict:
        rep = self._report_buf()
        _check(lib().lc_run_resident(self._h, rep, I64(1 << 22)))
        return json.loads(rep.value.decode())

    def run_resident_async(self) -> None:
        """Queue one resident run (graph replay) without waiting; see wait()."""
        _check(lib().lc_run_resident_async(self._h))

    def run_e2e_async(self, x0_pinned: "PinnedArray", video_pinned: "PinnedArray") -> None:
        """Queue one run with pinned host input/output (H2D + D2H inside);
        consecutive runs overlap compute with the previous video download."""
        _check(lib().lc_run_pipeline_async(self._h, x0_pinned.ptr, video_pinned.ptr))

    def wait(self) -> dict:
        """Complete the queued resident runs; report of the last one."""
        rep = self._report_buf()
        _check(lib().lc_wait(self._h, rep, I64(1 << 22)))
        return json.loads(rep.value.decode())

    def download_video(self) -> np.ndarray:
        out = np.empty(self.video_elems(), np.float32)
        _check(lib().lc_download_video(self._h, _p(out)))
        return out

    # -- measurement
    def timer_start(self):
        _check(lib().lc_timer_start(self._h))

    def timer_stop(self) -> float:
        ms = ctypes.c_float()
        _check(lib().lc_timer_stop(self._h, ctypes.byref(ms)))
        return ms.value

    def set_conv_profile(self, on: bool):
        _check(lib().lc_set_conv_profile(self._h, ctypes.c_int(int(on))))

    def conv_profile(self) -> dict:
        n, ms, alg, exe = I64(), ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        _check(lib().lc_conv_profile(self._h, ctypes.byref(n), ctypes.byref(ms), ctypes.byref(alg),
                                     ctypes.byref(exe)))
        return {"launches": n.value, "ms": ms.value, "alg_flops": alg.value, "exec_flops": exe.value}

    def kernel_launches(self) -> int:
        """Kernels launched by the last run / decode call."""
        n = I64()
        _check(lib().lc_kernel_launches(self._h, ctypes.byref(n)))
        return n.value

    def conv_profile_records(self) -> list:
        buf = ctypes.create_string_buffer(1 << 20)
        _check(lib().lc_conv_profile_records(self._h, buf, I64(1 << 20)))
        return json.loads(buf.value.decode())

    def run_e2e(self, x0_pinned: "PinnedArray", video_pinned: "PinnedArray") -> dict:
        """run_pipeline with pinned host input/output buffers (H2D + D2H inside)."""
        rep = self._report_buf()
        _check(lib().lc_run_pipeline(self._h, x0_pinned.ptr, video_pinned.ptr, None, rep, I64(1 << 22)))
        return json.loads(rep.value.decode())

    # -- operators
    def forward(self, x: np.ndarray, timestep: int, deep_in: Optional[np.ndarray] = None,
                want_deep: bool = False, deep_shape=None):
        """forward_full / forward_cached (proj/src/unet.cpp:188-276) on x (2,T,C,h,w)."""
        x = _f32(x)
        T = x.shape[1]
        eps = np.empty_like(x)
        deep_out = np.empty(deep_shape, np.float32) if want_deep else None
        din = None if deep_in is None else _f32(deep_in)
        _check(lib().lc_forward(self._h, _p(x), I64(T), I64(timestep), _p(din), _p(deep_out), _p(eps)))
        return eps, deep_out

    def decode(self, latents: np.ndarray, slice_frames: int = 1) -> np.ndarray:
        """decode_sliced (proj/src/codec.cpp:126-145) of latents (b,t,c,h,w)."""
        lat = _f32(latents)
        if lat.ndim != 5:
            raise ShapeError("decode: latents must be (b, t, c, h, w)")
        cfg = parse_config(self._text)
        s = 1 << int(cfg["codec.stages"])
        ic = int(cfg.get("codec.image_channels", 3))
        b, t, c, h, w = lat.shape
        out = np.empty((b, t, ic, h * s, w * s), np.float32)
        # c / h / w are validated by the library against the configured codec
        _check(lib().lc_decode(self._h, _p(lat), I64(b * t), I64(c), I64(h), I64(w), I64(slice_frames), _p(out)))
        return out

    def video_metrics(self, a, b, data_range: float = 1.0):
        """Per-frame PSNR and SSIM of two b=1 videos (t,c,h,w) on the GPU
        (psnr / ssim / video_series, proj/src/metrics.cpp:10-104)."""
        a, b = _f32(a), _f32(b)
        if a.shape != b.shape:
            raise ShapeError("video_metrics: shape mismatch")
        t, c, h, w = a.shape[-4:]
        ps, ss = np.empty(t, np.float64), np.empty(t, np.float64)
        _check(lib().lc_video_metrics(self._h, _p(a), _p(b), I64(t), I64(c), I64(h), I64(w),
                                      ctypes.c_double(data_range), _p(ps), _p(ss)))
        return ps, ss

    def conv2d(self, x, taps, bias, s=1.0, o=0.0, silu=False):
        x, taps, bias = _f32(x), _f32(taps), _f32(bias)
        b, t, c, h, w = x.shape
        c_out, k = taps.shape[0], taps.shape[-1]
        out = np.empty((b, t, c_out, h, w), np.float32)
        _check(lib().lc_conv2d(self._h, _p(x), I64(b), I64(t), I64(c), I64(h), I64(w), _p(taps), _p(bias),
                               I64(c_out), I64(k), ctypes.c_float(s), ctypes.c_float(o), ctypes.c_int(int(silu)),
                               _p(out)))
        return out

    def up_conv2d(self, skip, u, taps, bias, s=1.0, o=0.0):
        skip, u, taps, bias = _f32(skip), _f32(u), _f32(taps), _f32(bias)
        b, t, ca, h, w = skip.shape
        cb = u.shape[2]
        c_out = taps.shape[0]
        out = np.empty((b, t, c_out, h, w), np.float32)
        _check(lib().lc_up_conv2d(self._h, _p(skip), _p(u), I64(b), I64(t), I64(ca), I64(cb), I64(h), I64(w),
                                  _p(taps), _p(bias), I64(c_out), ctypes.c_float(s), ctypes.c_float(o), _p(out)))
        return out

    SAMPLER_KINDS = {"ancestral": 0, "ddim": 1, "euler": 2}  # SamplerKind order

    def sampler_step(self, sampler, t: int, x, eps_uncond, eps_cond, guidance: float, noise_seed: int = 0):
        """cfg_combine + reverse_step_<sampler> (proj/src/sampler.cpp:95-133) at
        index t of the configured (spaced) schedule, on the device.  Returns
        (x', nonfinite)."""
        kind = self.SAMPLER_KINDS[sampler] if isinstance(sampler, str) else int(sampler)
        x, eu, ec = _f32(x), _f32(eps_uncond), _f32(eps_cond)
        if eu.shape != x.shape or ec.shape != x.shape:
            raise ShapeError("cfg_combine: operand shapes differ")
        eps2 = np.ascontiguousarray(np.concatenate([eu.ravel(), ec.ravel()]))
        out = np.empty_like(x)
        bad = ctypes.c_int(0)
        _check(lib().lc_sampler_step(self._h, ctypes.c_int(kind), I64(t), _p(x), _p(eps2), I64(x.size),
                                     ctypes.c_double(guidance), ctypes.c_uint64(noise_seed), _p(out),
                                     ctypes.byref(bad)))
        return out, bool(bad.value)

    def all_finite(self, x) -> bool:
        """all_finite (proj/src/tensor.cpp:376) on the device."""
        x = _f32(x)
        f = ctypes.c_int(0)
        _check(lib().lc_all_finite(self._h, _p(x), I64(x.size), ctypes.byref(f)))
        return bool(f.value)

    # -- multi-GPU sliced decode
    def nccl_init(self, uid: bytes, world: int, rank: int):
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        _check(lib().lc_nccl_init(self._h, buf, ctypes.c_int(world), ctypes.c_int(rank)))

    def decode_sharded(self, latents, slice_frames: int = 4, out=None, host_shared: bool = False):
        """lc_decode_sharded; `latents` may be a PinnedArray (the whole
        (1,T,C,h,w) latent video of the config) or a numpy array (b,t,c,h,w);
        `out` a PinnedArray / SharedVideo / numpy array or None (device
        only: the gathered video stays in rank 0's HBM).  Returns (video or
        None, device ms)."""
        cfg = parse_config(self._text)
        s = 1 << int(cfg["codec.stages"])
        C = int(cfg["codec.latent_channels"])
        if isinstance(latents, PinnedArray):
            T = int(cfg["run.frames"])
            h, w = int(cfg["run.height"]) // s, int(cfg["run.width"]) // s
            if latents.n != T * C * h * w:
                raise ShapeError("decode_sharded: pinned latent size does not match the config")
            lat_ptr, c = latents.ptr, C
        else:
            lat = _f32(latents)
            if lat.ndim != 5:
                raise ShapeError("decode_sharded: latents must be (b, t, c, h, w)")
            lat_ptr, T, c, h, w = _p(lat), lat.shape[0] * lat.shape[1], lat.shape[2], lat.shape[3], lat.shape[4]
        nvid = T * 3 * h * s * w * s
        out_ptr = None
        if out is not None:
            n_out = out.n if hasattr(out, "n") else out.size
            if n_out < nvid:
                raise ShapeError("decode_sharded: output buffer too small")
            out_ptr = out.ptr if hasattr(out, "ptr") else _p(out)
        ms = ctypes.c_float()
        _check(lib().lc_decode_sharded(self._h, lat_ptr, I64(T), I64(c), I64(h), I64(w), I64(slice_frames), out_ptr,
                                       ctypes.c_int(SHARD_HOST_SHARED if host_shared else 0), ctypes.byref(ms)))
        if out is None:
            return None, ms.value
        arr = out.array if hasattr(out, "array") else out
        return arr.reshape(-1)[:nvid].reshape(1, T, 3, h * s, w * s), ms.value


class PinnedArray:
    """fp32 array in page-locked host memory (lc_alloc_pinned)."""

    def __init__(self, n: int):
        L = lib()
        L.lc_alloc_pinned.restype = ctypes.c_void_p
        self.ptr = ctypes.c_void_p(L.lc_alloc_pinned(I64(max(1, n) * 4)))
        if not self.ptr:
            raise DeviceError(L.lc_last_error().decode())
        self.n = n
        self.array = np.ctypeslib.as_array(ctypes.cast(self.ptr, ctypes.POINTER(ctypes.c_float)), shape=(n,))

    def free(self):
        if self.ptr:
            lib().lc_free_pinned(self.ptr)
            self.ptr = None


class SharedVideo:
    """fp32 host buffer in a POSIX shared-memory segment, page-locked with
    lc_host_register, so every rank of one box maps the same video and
    downloads its own frames into it (LC_SHARD_HOST_SHARED)."""

    def __init__(self, name: str, n: int, create: bool):
        from multiprocessing import shared_memory
        self.shm = shared_memory.SharedMemory(name=name, create=create, size=max(1, n) * 4)
        self.n = n
        self.array = np.ndarray((n,), np.float32, buffer=self.shm.buf)
        self.ptr = ctypes.c_void_p(self.array.ctypes.data)
        _check(lib().lc_host_register(self.ptr, I64(max(1, n) * 4)))
        self._owner = create

    def free(self):
        if self.ptr is not None:
            lib().lc_host_unregister(self.ptr)
            self.ptr = None
            self.array = None
            try:
                self.shm.close()
            except BufferError:  # a caller still holds a view of the video: unmapped at exit
                pass
            if self._owner:
                self.shm.unlink()


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(lib().lc_nccl_unique_id(buf))
    return bytes(buf)


def rel_l2(a: np.ndarray, b: np.ndarray) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
