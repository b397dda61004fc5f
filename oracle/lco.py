"""ctypes front-end for the CPU oracles.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
arm import this module; the product package never does.

Two oracles are exposed:

* ``Restatement`` -- oracle/liblc_oracle.so, the plain-C restatement
  (oracle/lc_oracle.c) of the reference algorithm.  Always built by
  ``__graft_entry__.build()`` from committed source.
* ``Reference`` -- oracle/_ref/libstagecache_ref.so, the unmodified
  reference sources compiled in place (oracle/Makefile).  Present where
  /root/reference was available at build time (and on GPU boxes that receive
  the prebuilt file).

Config text uses the reference grammar (proj/src/config.cpp:158-224): one
``key = value`` per line over ``default_config()``.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATE_SO = os.path.join(HERE, "liblc_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libstagecache_ref.so")

# default_config() (proj/src/config.cpp:90-98 over config.hpp:16-71)
DEFAULTS = {
    "run.frames": "8", "run.height": "64", "run.width": "64", "run.seed": "42",
    "run.mode": "text", "run.out_dir": "out",
    "unet.depth": "3", "unet.base_channels": "8", "unet.kernel": "3",
    "unet.cache_depth": "0", "unet.weight_seed": "1234",
    "codec.latent_channels": "4", "codec.stages": "2", "codec.width": "8",
    "codec.weight_seed": "77",
    "schedule.train_steps": "50", "schedule.beta_min": "0.002", "schedule.beta_max": "0.25",
    "sampler.kind": "euler", "sampler.steps": "25", "sampler.guidance": "1.5",
    "cache.enabled": "true", "cache.n": "2",
    "swap.mode": "async", "swap.simulate": "false", "swap.bandwidth": "4e9",
    "swap.latency": "2e-05", "swap.mac_rate": "5e7",
    "chunk.enabled": "true", "chunk.eta": "2", "chunk.omega": "2", "chunk.halo": "exact",
    "chunk.halo_px": "0", "chunk.targets": "u0",
    "decode.sliced": "true", "budget.fast_bytes": "0",
}


def parse_text(text: str) -> dict:
    kv = dict(DEFAULTS)
    for line in text.splitlines():
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        k, v = line.split("=", 1)
        kv[k.strip()] = v.strip()
    return kv


def to_text(kv: dict) -> str:
    return "".join(f"{k} = {v}\n" for k, v in kv.items())


def _bool(v: str) -> int:
    return 1 if v in ("true", "on", "1") else 0


class LcoConfig(ctypes.Structure):
    _fields_ = [
        ("frames", ctypes.c_int64), ("height", ctypes.c_int64), ("width", ctypes.c_int64),
        ("seed", ctypes.c_uint64), ("mode_image", ctypes.c_int32),
        ("depth", ctypes.c_int64), ("base_channels", ctypes.c_int64), ("kernel", ctypes.c_int64),
        ("cache_depth", ctypes.c_int64), ("in_channels", ctypes.c_int64),
        ("unet_seed", ctypes.c_uint64),
        ("latent_channels", ctypes.c_int64), ("stages", ctypes.c_int64),
        ("image_channels", ctypes.c_int64), ("codec_width", ctypes.c_int64),
        ("codec_seed", ctypes.c_uint64),
        ("train_steps", ctypes.c_int64), ("beta_min", ctypes.c_double), ("beta_max", ctypes.c_double),
        ("sampler", ctypes.c_int32), ("steps", ctypes.c_int64), ("guidance", ctypes.c_double),
        ("cache_enabled", ctypes.c_int32), ("cache_n", ctypes.c_int64),
        ("chunk_enabled", ctypes.c_int32), ("eta", ctypes.c_int64), ("omega", ctypes.c_int64),
        ("halo_kind", ctypes.c_int32), ("halo_px", ctypes.c_int64),
        ("chunk_targets", ctypes.c_uint64), ("slice_decode", ctypes.c_int32),
    ]


def block_index(name: str, depth: int) -> int:
    """Position in block_plans order (proj/src/unet.cpp:33-50)."""
    if name == "stem":
        return 0
    if name == "mid":
        return 1 + depth
    if name == "head":
        return 2 + 2 * depth
    if name[0] == "d":
        return 1 + int(name[1:])
    if name[0] == "u":
        return 2 + depth + (depth - 1 - int(name[1:]))
    raise ValueError(name)


def make_config(kv: dict) -> LcoConfig:
    c = LcoConfig()
    c.frames, c.height, c.width = int(kv["run.frames"]), int(kv["run.height"]), int(kv["run.width"])
    c.seed = int(kv["run.seed"])
    c.mode_image = 1 if kv["run.mode"] == "image" else 0
    c.depth = int(kv["unet.depth"])
    c.base_channels = int(kv["unet.base_channels"])
    c.kernel = int(kv["unet.kernel"])
    c.cache_depth = int(kv["unet.cache_depth"])
    c.latent_channels = int(kv["codec.latent_channels"])
    c.in_channels = c.latent_channels
    c.unet_seed = int(kv["unet.weight_seed"])
    c.stages = int(kv["codec.stages"])
    c.image_channels = 3
    c.codec_width = int(kv["codec.width"])
    c.codec_seed = int(kv["codec.weight_seed"])
    c.train_steps = int(kv["schedule.train_steps"])
    c.beta_min, c.beta_max = float(kv["schedule.beta_min"]), float(kv["schedule.beta_max"])
    c.sampler = {"ancestral": 0, "ddim": 1, "euler": 2}[kv["sampler.kind"]]
    c.steps = int(kv["sampler.steps"])
    c.guidance = float(kv["sampler.guidance"])
    c.cache_enabled = _bool(kv["cache.enabled"])
    c.cache_n = int(kv["cache.n"])
    c.chunk_enabled = _bool(kv["chunk.enabled"])
    c.eta, c.omega = int(kv["chunk.eta"]), int(kv["chunk.omega"])
    c.halo_kind = {"exact": 0, "fixed": 1, "none": 2}[kv["chunk.halo"]]
    c.halo_px = int(kv["chunk.halo_px"])
    mask = 0
    for t in [s.strip() for s in kv["chunk.targets"].split(",") if s.strip()]:
        mask |= 1 << block_index(t, c.depth)
    c.chunk_targets = mask
    c.slice_decode = _bool(kv["decode.sliced"])
    return c


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class Shapes:
    latent: tuple
    video: tuple
    model_input: tuple


def shapes_of(kv: dict) -> Shapes:
    s = 1 << int(kv["codec.stages"])
    T, H, W = int(kv["run.frames"]), int(kv["run.height"]), int(kv["run.width"])
    C = int(kv["codec.latent_channels"])
    return Shapes((1, T, C, H // s, W // s), (1, T, 3, H, W), (2, T, C, H // s, W // s))


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Restatement:
    """oracle/lc_oracle.c via ctypes."""

    def __init__(self, path: str = RESTATE_SO):
        self.lib = ctypes.CDLL(path)
        self.lib.lco_last_error.restype = ctypes.c_char_p
        self.lib.lco_normal_at.restype = ctypes.c_float
        self.lib.lco_normal_at.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        self.lib.lco_derive_seed.restype = ctypes.c_uint64
        self.lib.lco_derive_seed.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        self.lib.lco_flops_estimate.restype = ctypes.c_int64

    def _chk(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.lco_last_error().decode())

    def derive_seed(self, seed, stream):
        return self.lib.lco_derive_seed(seed, stream)

    def randn(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, np.float32)
        self.lib.lco_randn(ctypes.c_uint64(seed), ctypes.c_int64(n), _p(out))
        return out

    def run_pipeline(self, kv: dict):
        sh = shapes_of(kv)
        cfg = make_config(kv)
        video = np.empty(sh.video, np.float32)
        lat = np.empty(sh.latent, np.float32)
        self._chk(self.lib.lco_run_pipeline(ctypes.byref(cfg), _p(video), _p(lat)))
        return video, lat

    def forward(self, kv: dict, x: np.ndarray, timestep: int, deep_in=None, want_deep=False):
        cfg = make_config(kv)
        x = _f32(x)
        B, T, C, H, W = x.shape
        eps = np.empty_like(x)
        deep_out = None
        m, M, base = cfg.cache_depth, cfg.depth, cfg.base_channels
        c_next = base << (M - 1) if m + 1 == M else base << (m + 1)
        dshape = (B, T, c_next, H >> m, W >> m)
        if want_deep:
            deep_out = np.empty(dshape, np.float32)
        din = None if deep_in is None else _f32(deep_in)
        self._chk(self.lib.lco_forward(
            ctypes.byref(cfg), _p(x), ctypes.c_int64(B), ctypes.c_int64(T), ctypes.c_int64(H),
            ctypes.c_int64(W), ctypes.c_int64(timestep), _p(din) if din is not None else None,
            _p(deep_out) if deep_out is not None else None, _p(eps)))
        return eps, deep_out

    def decode(self, kv: dict, lat: np.ndarray) -> np.ndarray:
        cfg = make_config(kv)
        lat = _f32(lat)
        n, C, h, w = lat.shape[0] * lat.shape[1], lat.shape[2], lat.shape[3], lat.shape[4]
        s = 1 << cfg.stages
        out = np.empty((lat.shape[0], lat.shape[1], 3, h * s, w * s), np.float32)
        self._chk(self.lib.lco_decode(ctypes.byref(cfg), _p(lat), ctypes.c_int64(n),
                                      ctypes.c_int64(h), ctypes.c_int64(w), _p(out)))
        return out

    def conv2d_window(self, x, taps, bias, k, win=None):
        x = _f32(x)
        taps, bias = _f32(taps), _f32(bias)
        b, t, c, h, w = x.shape
        c_out = bias.shape[0]
        y0, y1, x0, x1 = win if win is not None else (0, h, 0, w)
        out = np.empty((b, t, c_out, y1 - y0, x1 - x0), np.float32)
        i64 = ctypes.c_int64
        self._chk(self.lib.lco_conv2d_window(
            _p(x), i64(b), i64(t), i64(c), i64(h), i64(w), _p(taps), _p(bias), i64(c_out), i64(k),
            i64(y0), i64(y1), i64(x0), i64(x1), _p(out)))
        return out

    def plan_steps(self, total: int, n: int):
        kinds = np.empty(total, np.int8)
        flags = np.empty(total, np.int8)
        self._chk(self.lib.lco_plan_steps(ctypes.c_int64(total), ctypes.c_int64(n), _p(kinds), _p(flags)))
        return kinds, flags

    def split(self, h, w, eta, omega, halo_kind, halo_px, k):
        regions = np.empty(12 * eta * omega, np.int64)
        halo = ctypes.c_int64()
        self._chk(self.lib.lco_split(
            ctypes.c_int64(h), ctypes.c_int64(w), ctypes.c_int64(eta), ctypes.c_int64(omega),
            ctypes.c_int32(halo_kind), ctypes.c_int64(halo_px), ctypes.c_int64(k), _p(regions),
            ctypes.byref(halo)))
        return regions.reshape(-1, 3, 4), halo.value

    def unet_bank(self, kv: dict, j: int, c_in: int, c_out: int, k: int):
        cfg = make_config(kv)
        taps = np.empty((c_out, c_in, k, k), np.float32)
        bias = np.empty(c_out, np.float32)
        cs = np.empty(8, np.float32)
        co = np.empty(8, np.float32)
        self._chk(self.lib.lco_unet_bank(ctypes.byref(cfg), ctypes.c_int64(j), _p(taps), _p(bias),
                                         _p(cs), _p(co)))
        return taps, bias, cs, co

    def flops_estimate(self, kv: dict, cached: bool) -> int:
        cfg = make_config(kv)
        B, T, C, h, w = shapes_of(kv).model_input
        return self.lib.lco_flops_estimate(ctypes.byref(cfg), ctypes.c_int64(B), ctypes.c_int64(T),
                                           ctypes.c_int64(h), ctypes.c_int64(w), ctypes.c_int(int(cached)))

    def video_metrics(self, a, b, data_range=1.0):
        """psnr/ssim video_series (proj/src/metrics.cpp:10-104) of two b=1 videos."""
        a, b = _f32(a), _f32(b)
        t, c, h, w = a.shape[-4:]
        ps, ss = np.empty(t, np.float64), np.empty(t, np.float64)
        i64 = ctypes.c_int64
        self._chk(self.lib.lco_video_metrics(_p(a), _p(b), i64(t), i64(c), i64(h), i64(w), ctypes.c_double(data_range),
                                _p(ps), _p(ss)))
        return ps, ss


class Reference:
    """The reference itself (oracle/_ref) via its C shim oracle/ref_capi.cpp."""

    def __init__(self, path: str = REF_SO):
        self.lib = ctypes.CDLL(path)
        self.lib.ref_last_error.restype = ctypes.c_char_p

    @staticmethod
    def available(path: str = REF_SO) -> bool:
        return os.path.exists(path)

    def _chk(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def run_pipeline(self, kv: dict):
        import json
        sh = shapes_of(kv)
        video = np.empty(sh.video, np.float32)
        rep = ctypes.create_string_buffer(1 << 20)
        macs = (ctypes.c_int64 * 4)()
        self._chk(self.lib.ref_run_pipeline(to_text(kv).encode(), _p(video), ctypes.c_int64(video.size),
                                            rep, ctypes.c_int64(1 << 20), macs))
        return video, json.loads(rep.value.decode()), list(macs)

    def timeline(self, kv: dict, cap: int = 1 << 14):
        """run_pipeline's timeline rows (kind, step, bytes, clock_ns), makespan_ns, stall_ns."""
        ev = np.empty((cap, 4), np.int64)
        info = (ctypes.c_int64 * 3)()
        self._chk(self.lib.ref_timeline(to_text(kv).encode(), _p(ev), ctypes.c_int64(cap), info))
        return ev[:info[0]].copy(), info[1], info[2]

    def check_config(self, kv: dict) -> int:
        return self.lib.ref_check_config(to_text(kv).encode())

    def forward(self, kv: dict, x: np.ndarray, timestep: int, deep_in=None, want_deep=False):
        x = _f32(x)
        B, T, C, H, W = x.shape
        eps = np.empty_like(x)
        nums = self.model_numbers(kv, (T, H, W))
        dshape = tuple(nums[2:7])
        i64 = ctypes.c_int64
        if deep_in is None:
            deep = np.empty(dshape, np.float32) if want_deep else np.empty(dshape, np.float32)
            self._chk(self.lib.ref_forward_full(to_text(kv).encode(), _p(x), i64(T), i64(H), i64(W),
                                                i64(timestep), _p(eps), _p(deep)))
            return eps, (deep if want_deep else None)
        d = _f32(deep_in)
        self._chk(self.lib.ref_forward_cached(to_text(kv).encode(), _p(x), i64(T), i64(H), i64(W),
                                              i64(timestep), _p(d), _p(eps)))
        return eps, None

    def model_numbers(self, kv: dict, thw=None):
        kv2 = dict(kv)
        if thw is not None:
            s = 1 << int(kv["codec.stages"])
            kv2["run.frames"], kv2["run.height"], kv2["run.width"] = str(thw[0]), str(thw[1] * s), str(thw[2] * s)
        out = (ctypes.c_int64 * 8)()
        self._chk(self.lib.ref_model_numbers(to_text(kv2).encode(), out))
        return list(out)

    def decode(self, kv: dict, lat: np.ndarray, sliced=True) -> np.ndarray:
        lat = _f32(lat)
        n, h, w = lat.shape[0] * lat.shape[1], lat.shape[3], lat.shape[4]
        s = 1 << int(kv["codec.stages"])
        out = np.empty((lat.shape[0], lat.shape[1], 3, h * s, w * s), np.float32)
        i64 = ctypes.c_int64
        self._chk(self.lib.ref_decode(to_text(kv).encode(), _p(lat), i64(n), i64(h), i64(w),
                                      ctypes.c_int(int(sliced)), _p(out)))
        return out

    def sampler_step(self, kv: dict, kind: int, t: int, x, eps_u, eps_c, guidance: float, noise_seed: int = 0):
        """cfg_combine + reverse_step_* (proj/src/sampler.cpp:95-133) at index t
        of the config's spaced schedule; kind 0 ancestral, 1 ddim, 2 euler."""
        x, eps_u, eps_c = _f32(x), _f32(eps_u), _f32(eps_c)
        out = np.empty_like(x)
        self._chk(self.lib.ref_sampler_step(to_text(kv).encode(), ctypes.c_int(kind), ctypes.c_int64(t), _p(x),
                                            _p(eps_u), _p(eps_c), ctypes.c_int64(x.size), ctypes.c_double(guidance),
                                            ctypes.c_uint64(noise_seed), _p(out)))
        return out

    def conv2d_window(self, x, taps, bias, k, win=None):
        x = _f32(x)
        taps, bias = _f32(taps), _f32(bias)
        b, t, c, h, w = x.shape
        c_out = bias.shape[0]
        y0, y1, x0, x1 = win if win is not None else (0, h, 0, w)
        out = np.empty((b, t, c_out, y1 - y0, x1 - x0), np.float32)
        i64 = ctypes.c_int64
        self._chk(self.lib.ref_conv2d_window(
            _p(x), i64(b), i64(t), i64(c), i64(h), i64(w), _p(taps), _p(bias), i64(c_out), i64(k),
            i64(y0), i64(y1), i64(x0), i64(x1), _p(out)))
        return out

    def plan_steps(self, total: int, n: int):
        kinds = np.empty(total, np.int8)
        flags = np.empty(total, np.int8)
        self._chk(self.lib.ref_plan_steps(ctypes.c_int64(total), ctypes.c_int64(n), _p(kinds), _p(flags)))
        return kinds, flags

    def split(self, h, w, eta, omega, halo_kind, halo_px, k):
        regions = np.empty(12 * eta * omega, np.int64)
        halo = ctypes.c_int64()
        self._chk(self.lib.ref_split(
            ctypes.c_int64(h), ctypes.c_int64(w), ctypes.c_int64(eta), ctypes.c_int64(omega),
            ctypes.c_int(halo_kind), ctypes.c_int64(halo_px), ctypes.c_int64(k), _p(regions),
            ctypes.byref(halo)))
        return regions.reshape(-1, 3, 4), halo.value

    def video_metrics(self, a, b, data_range=1.0):
        """psnr/ssim video_series (proj/src/metrics.cpp:10-104) of two b=1 videos."""
        a, b = _f32(a), _f32(b)
        t, c, h, w = a.shape[-4:]
        ps, ss = np.empty(t, np.float64), np.empty(t, np.float64)
        i64 = ctypes.c_int64
        self._chk(self.lib.ref_video_metrics(_p(a), _p(b), i64(t), i64(c), i64(h), i64(w), ctypes.c_double(data_range),
                                _p(ps), _p(ss)))
        return ps, ss

    def write_video_raw(self, path, video):
        v = _f32(video)
        t, c, h, w = v.shape[-4:]
        i64 = ctypes.c_int64
        self._chk(self.lib.ref_write_video_raw(path.encode(), _p(v), i64(t), i64(c), i64(h), i64(w)))
