"""Config E (BASELINE.json configs[4]): cache interval N x chunk count sweep on
the SVD-XT shape -- frames/s vs peak HBM, plus video quality (PSNR / SSIM,
the reference's definitions, proj/src/metrics.cpp:10-71) against the
uncached run.  Writes a JSON table (profiles/sweep_<round>.json)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2510_05367_b200 as lc  # noqa: E402


def psnr(a, b, peak=1.0):
    """proj/src/metrics.cpp:10-24: 10 log10(peak^2 / MSE), capped at 99 dB."""
    mse = float(np.mean((a.astype(np.float64) - b.astype(np.float64)) ** 2))
    return 99.0 if mse <= 0 else min(99.0, 10.0 * np.log10(peak * peak / mse))


def ssim(a, b, peak=1.0):
    """proj/src/metrics.cpp:26-71: mean SSIM over 7x7 uniform windows per channel."""
    from numpy.lib.stride_tricks import sliding_window_view as win
    c1, c2 = (0.01 * peak) ** 2, (0.03 * peak) ** 2
    vals = []
    for ch in range(a.shape[0]):
        x = win(a[ch].astype(np.float64), (7, 7))
        y = win(b[ch].astype(np.float64), (7, 7))
        mx, my = x.mean(axis=(-1, -2)), y.mean(axis=(-1, -2))
        vx, vy = x.var(axis=(-1, -2)), y.var(axis=(-1, -2))
        cov = ((x - mx[..., None, None]) * (y - my[..., None, None])).mean(axis=(-1, -2))
        s = ((2 * mx * my + c1) * (2 * cov + c2)) / ((mx ** 2 + my ** 2 + c1) * (vx + vy + c2))
        vals.append(s.mean())
    return float(np.mean(vals))


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "C"
    out_path = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "sweep.json")
    steps = int(os.environ.get("SWEEP_STEPS", "3"))
    base = dict(bench.WORKLOADS[wl])
    ctx = lc.Context(0)
    rows = []

    def measure(over, label):
        text = lc.config_text(over, base=lc.DEFAULT_CONFIG)
        ctx.configure(text)
        kv = lc.parse_config(text)
        ctx.upload_latent(lc.randn(lc.derive_seed(int(kv["run.seed"]), 1), ctx.latent_elems()))
        for _ in range(2):
            ctx.run_resident()
        ctx.timer_start()
        for _ in range(steps):
            rep = ctx.run_resident()
        ms = ctx.timer_stop() / steps
        video = ctx.download_video().reshape(int(kv["run.frames"]), 3, int(kv["run.height"]), int(kv["run.width"]))
        return {"label": label, "frames_per_s": int(kv["run.frames"]) / (ms / 1e3), "ms_per_video": ms,
                "hbm_peak_gb": rep["hbm_peak_bytes"] / 1e9, "swap_stall_ms": rep["timeline"]["stall_ms"],
                "denoiser_tmac": rep["mac"]["denoiser_total"] / 1e12}, video

    ref_row, ref_video = measure(dict(base, **{"cache.enabled": "false", "chunk.enabled": "false",
                                               "decode.sliced": "false", "swap.mode": "off"}), "uncached")
    ref_row.update({"psnr_db": 99.0, "ssim": 1.0})
    rows.append(ref_row)
    print(json.dumps(ref_row), flush=True)
    for n in (1, 2, 3, 4, 8):
        for eta, omega in ((1, 1), (1, 2), (2, 2)):
            over = dict(base, **{"cache.n": n, "chunk.eta": eta, "chunk.omega": omega})
            row, video = measure(over, f"N={n} chunk={eta}x{omega}")
            row["psnr_db"] = float(np.mean([psnr(video[t], ref_video[t]) for t in range(video.shape[0])]))
            row["ssim"] = float(np.mean([ssim(video[t], ref_video[t]) for t in range(0, video.shape[0], 6)]))
            row.update({"n": n, "eta": eta, "omega": omega})
            rows.append(row)
            print(json.dumps(row), flush=True)
    json.dump({"workload": bench.DESCR[wl], "rows": rows}, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main()
