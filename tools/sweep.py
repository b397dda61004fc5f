"""Config E (BASELINE.json configs[4]): cache interval N x chunk count sweep on
the SVD-XT shape -- frames/s vs peak HBM, plus video quality against the
uncached run: per-frame PSNR / SSIM on the GPU (lc_video_metrics, the
reference's definitions, proj/src/metrics.cpp:10-104), averaged over all
frames as video_series does.  Writes a JSON table (profiles/sweep_<round>.json)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2510_05367_b200 as lc  # noqa: E402


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "C"
    out_path = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "sweep.json")
    steps = int(os.environ.get("SWEEP_STEPS", "3"))
    base = dict(bench.WORKLOADS[wl])
    ctx = lc.Context(0)
    rows = []

    def measure(over, label):
        # a fresh engine per row: its ledger peak is this configuration's alone
        nonlocal ctx
        ctx.close()
        ctx = lc.Context(0)
        text = lc.config_text(over, base=lc.DEFAULT_CONFIG)
        ctx.configure(text)
        kv = lc.parse_config(text)
        ctx.upload_latent(lc.randn(lc.derive_seed(int(kv["run.seed"]), 1), ctx.latent_elems()))
        for _ in range(2):
            ctx.run_resident()
        ctx.timer_start()
        for _ in range(steps):
            ctx.run_resident_async()
        rep = ctx.wait()
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
            ps, ss = ctx.video_metrics(ref_video, video, 1.0)
            row["psnr_db"], row["ssim"] = float(ps.mean()), float(ss.mean())
            row.update({"n": n, "eta": eta, "omega": omega})
            rows.append(row)
            print(json.dumps(row), flush=True)
    json.dump({"workload": bench.DESCR[wl], "rows": rows}, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main()
