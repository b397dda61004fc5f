"""Cross-check of bench.py's reference arm: every host core
runs the reference's own run_pipeline (oracle/_ref) at FULL resolution --
one frame of config B, and one frame of config C over the sample's 2-step
refresh period -- and then the bench's bounded sample, in the same process
pool; the two per-core MAC rates tell how far the sample's extrapolation is
from the reference's speed at the real image size.  Writes a JSON summary.
Nothing of the product is imported."""
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import bench  # noqa: E402


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "ref_crosscheck.json")
    import lco
    workers = max(1, min(os.cpu_count() or 1, 256))
    res = {"cores": workers}
    lib, _ = bench._cpu_lib()
    with mp.get_context("spawn").Pool(workers) as pool:
        for wl, full_over in (("B", {"run.frames": 1}),
                              # C at full resolution over the sample's 2-step refresh period (a 25-step
                              # C frame is ~55 min per core): the same work per step as the headline
                              ("C", {"run.frames": 1, "sampler.steps": 2})):
            full = bench._kv(dict(bench.WORKLOADS[wl], **full_over))
            samp, macs_s, macs_f, kind = bench.cpu_sample(wl)
            macs_full = bench.ref_run_macs(lib, full)
            t0 = time.time()
            pool.map(bench._cpu_worker, [(lco.to_text(full), False)] * workers)
            wall_full = time.time() - t0
            t0 = time.time()
            pool.map(bench._cpu_worker, [(lco.to_text(samp), False)] * workers)
            wall_samp = time.time() - t0
            r = {"kind": kind,
                 "full_resolution": {"gmac_per_s_per_core": macs_full / 1e9 / wall_full, "wall_s": wall_full,
                                     "gmac": macs_full / 1e9, "config": {k: full[k] for k in full_over} |
                                     {"run.height": full["run.height"], "run.width": full["run.width"]}},
                 "sample": {"gmac_per_s_per_core": macs_s / 1e9 / wall_samp, "wall_s": wall_samp,
                            "gmac": macs_s / 1e9, "latent": f"{samp['run.height']}x{samp['run.width']} px"}}
            r["rate_ratio_sample_over_full"] = r["sample"]["gmac_per_s_per_core"] / r["full_resolution"]["gmac_per_s_per_core"]
            res[wl] = r
    json.dump(res, open(out_path, "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
