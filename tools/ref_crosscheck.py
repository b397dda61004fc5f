"""Un-extrapolated cross-check of bench.py's reference arm:
every host core runs the reference's own run_pipeline (oracle/_ref) on ONE
full-resolution frame of config B (frame 0 is bit-identical to the T-frame
run's), so frames/s = cores / wall with no MAC scaling; the
bench's bounded-sample estimate for B is measured in the same process pool
beside it.  Writes a JSON summary.  Nothing of the product is imported."""
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
    full = bench._kv(dict(bench.WORKLOADS["B"], **{"run.frames": 1}))
    samp, macs_s, macs_f, kind = bench.cpu_sample("B")
    with mp.get_context("spawn").Pool(workers) as pool:
        t0 = time.time()
        pool.map(bench._cpu_worker, [(lco.to_text(full), False)] * workers)
        wall_full = time.time() - t0
        t0 = time.time()
        pool.map(bench._cpu_worker, [(lco.to_text(samp), False)] * workers)
        wall_samp = time.time() - t0
    res = {"kind": kind, "cores": workers,
           "full_frame": {"frames_per_s": workers / wall_full, "wall_s": wall_full,
                          "what": "one full-resolution frame of config B per core (512x512, 4 steps, N=2)"},
           "sample_extrapolated": {"frames_per_s": workers * macs_s / macs_f / wall_samp, "wall_s": wall_samp,
                                   "sample_gmac": macs_s / 1e9, "frame_gmac": macs_f / 1e9},
           }
    res["ratio_sample_over_full"] = res["sample_extrapolated"]["frames_per_s"] / res["full_frame"]["frames_per_s"]
    json.dump(res, open(out_path, "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
