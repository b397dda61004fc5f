"""Copy one tools/refresh_profiles_r02.sh run (gpurun_out/) into profiles/:
bench lines (C headline, reference arm, D, B), the C launch list (share per
kernel, DRAM bytes per launch, the per-kernel HBM table), the `ncu --set
full` summaries of C's stem GEMM, d0, head (K8 + fused sampler step) and
the decoder's last stage, the per-layer event timing and swap timeline of C.
Usage: python tools/collect_profiles_r02.py [round]"""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
rnd = sys.argv[1] if len(sys.argv) > 1 else "r02"


def last_json(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


def run(args):
    return subprocess.run(args, capture_output=True, text=True).stdout


for name in ("b", "c", "d", "ref"):
    src = os.path.join(G, f"bench_{name}.json")
    if os.path.exists(src):
        try:
            json.dump(last_json(src), open(os.path.join(P, f"bench_{name}_{rnd}.json"), "w"), indent=1)
        except Exception as e:  # noqa: BLE001
            print("skip", src, e)
src = os.path.join(G, "launch_c.csv")
if os.path.exists(src):
    shutil.copy(src, os.path.join(P, f"ncu_launches_c_{rnd}.csv"))
    out = run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), src, "2", "-v"])
    open(os.path.join(P, f"ncu_launches_c_{rnd}.txt"), "w").write(
        "# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
        "python tools/profile_step.py C 2\n# (serialized, cold-ish caches: per-launch SHARES are meaningful, "
        "absolute sums are not)\n" + out)
    out = run([sys.executable, os.path.join(ROOT, "tools", "membound_report.py"), src, "2"])
    open(os.path.join(P, f"membound_c_{rnd}.txt"), "w").write(out)
src = os.path.join(G, "launch_d.csv")
if os.path.exists(src):
    shutil.copy(src, os.path.join(P, f"ncu_launches_d_{rnd}.csv"))
    print(run([sys.executable, os.path.join(ROOT, "tools", "conv_traffic.py"), src, "D", "2"]))
    out = run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), src, "2", "-v"])
    open(os.path.join(P, f"ncu_launches_d_{rnd}.txt"), "w").write(
        "# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
        "python tools/profile_step.py D 2\n" + out)
src = os.path.join(G, "launch_c.csv")
if os.path.exists(src):
    print(run([sys.executable, os.path.join(ROOT, "tools", "conv_traffic.py"), src, "C", "2"]))
KEEP = ("sm__pipe_tc_cycles_active.avg.pct", "sm__pipe_tensor_cycles_active.avg.pct", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "lts__t_bytes.sum",
        "smsp__average_warps_issue_stalled_", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed")
WHAT = {
    "stem": ("-k regex:conv_tc --launch-skip 0", "C stem GEMM (K = 64 patch rows -> 320 ch, SiLU, TMA store), "
             "run 1 step 0", "conv_tc_kernel<1, 1>"),
    "d0": ("-k regex:conv_tc --launch-skip 1", "C d0 (3x3 320 -> 320 on 72x128, halo ring, CTA pairs), run 1 "
           "step 0", "conv_tc_kernel<2, 1>"),
    "head": ("-k regex:tap_tc --launch-skip 0", "C head: K8 tap_tc_kernel<1> with the fused CFG + Euler step, "
             "run 1 step 0", "tap_tc_kernel<1"),
    "dec": ("-k regex:tap_tc --launch-skip 25", "C decoder last stage: K8 tap_tc_kernel<0> (nearest 2x + 3x3 "
            "128 -> 3), 5-frame slice", "tap_tc_kernel<0"),
}
WHAT["d_dec2"] = ("-k regex:conv_tc --launch-skip 2", "D dec2: sub-pixel up-conv 128 -> 128 to 288x512, "
                   "halo-staged, weight-stationary, 5-frame slice (profile_step D 1)", "conv_tc_kernel<1, 1>")
for tag, (sel, desc, kname) in WHAT.items():
    rep = os.path.join(G, f"full_c_{tag}.ncu-rep" if not tag.startswith("d_") else f"full_{tag}.ncu-rep")
    if not os.path.exists(rep):
        continue
    det = run(["ncu", "-i", rep, "--page", "details"])
    if kname not in det:  # the capture must be the kernel the file is named after
        print(f"skip {tag}: captured kernel is not {kname}")
        continue
    raw = run(["ncu", "-i", rep, "--page", "raw", "--csv"])
    rows = list(csv.reader(raw.splitlines()))
    sel_rows = [f"{h} ({u}) = {v}" for h, u, v in zip(rows[0], rows[1], rows[2]) if h.startswith(KEEP)]
    name = f"ncu_full_c_{tag}_{rnd}.txt" if not tag.startswith("d_") else f"ncu_full_{tag}_{rnd}.txt"
    wl = "D" if tag.startswith("d_") else "C"
    open(os.path.join(P, name), "w").write(
        f"# ncu --set full --clock-control none --import-source on {sel} --launch-count 1 "
        f"python tools/profile_step.py {wl} 1\n# {desc}\n\n" + det + "\n# selected raw metrics\n" +
        "\n".join(sel_rows) + "\n")
for name in ("layers_c.txt", "swap_timeline_c.txt", "parity.json", "sweep.json", "ref_crosscheck.json"):
    src = os.path.join(G, name)
    if os.path.exists(src):
        base, ext = os.path.splitext(name)
        shutil.copy(src, os.path.join(P, f"{'sweep_c' if base == 'sweep' else base}_{rnd}{ext}"))
print("collected", rnd)
