"""Copy one refresh_profiles.sh run (gpurun_out/) into profiles/<round>:
bench lines, parity, launch-list summaries, conv DRAM traffic and the
`ncu --set full` summary of the top conv launch."""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"


def last_json(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


for name in ("b", "c", "d", "ref"):
    src = os.path.join(G, f"bench_{name}.json")
    if os.path.exists(src):
        json.dump(last_json(src), open(os.path.join(P, f"bench_{name}_{rnd}.json"), "w"), indent=1)
if os.path.exists(os.path.join(G, "parity.json")):
    shutil.copy(os.path.join(G, "parity.json"), os.path.join(P, f"parity_{rnd}.json"))
for wl, steps in (("b", 3), ("c", 2)):
    src = os.path.join(G, f"launch_{wl}.csv")
    if not os.path.exists(src):
        continue
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), src, str(steps), "-v"],
                         capture_output=True, text=True).stdout
    open(os.path.join(P, f"ncu_launches_{wl}_{rnd}.txt"), "w").write(
        f"# ncu --metrics gpu__time_duration.sum --clock-control none python tools/profile_step.py {wl.upper()} "
        f"{steps}\n# (serialized, cold-ish caches: per-launch SHARES are meaningful, absolute sums are not)\n" + out)
    if wl == "b":
        shutil.copy(src, os.path.join(P, f"ncu_launches_b_{rnd}.csv"))
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "conv_traffic.py"), src, "B", "3"])
rep = os.path.join(G, "full_top.ncu-rep")
if os.path.exists(rep):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    keep = ("sm__pipe_tc_cycles_active", "sm__pipe_tensor", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "lts__t_bytes.sum",
            "smsp__average_warps_issue_stalled_", "l1tex__m_xbar2l1tex_read_bytes.sum")
    sel = [f"{h} = {v}" for h, v in zip(rows[0], rows[2]) if h.startswith(keep) and not h.endswith("pct_of_peak_sustained_elapsed")]
    open(os.path.join(P, f"ncu_full_conv_b_{rnd}.txt"), "w").write(
        "# ncu --set full --clock-control none --import-source on -k regex:conv_tc --launch-skip 92 "
        "--launch-count 1 python tools/profile_step.py B 3\n# (u0 of a full step: cg=2, BN=160, K=5440)\n\n" +
        det + "\n# selected raw metrics\n" + "\n".join(sel) + "\n")
rep = os.path.join(G, "full_tap.ncu-rep")
if os.path.exists(rep):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
    open(os.path.join(P, f"ncu_full_tap_b_{rnd}.txt"), "w").write(
        "# ncu --set full --clock-control none --import-source on -k regex:tap_tc --launch-skip 4 "
        "--launch-count 1 python tools/profile_step.py B 1\n# (K8, the decoder's fused last stage of the "
        "first 4-frame slice)\n\n" + det)
rep = os.path.join(G, "full_halo.ncu-rep")
if os.path.exists(rep):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
    open(os.path.join(P, f"ncu_full_halo_b_{rnd}.txt"), "w").write(
        "# ncu --set full --clock-control none --import-source on -k regex:conv_tc --launch-skip 116 "
        "--launch-count 1 python tools/profile_step.py B 3\n# (decoder dec2: P4 sub-pixel up-conv 128->128 at "
        "256x256, halo-staged, weight-stationary, first 4-frame slice of run 3)\n\n" + det)
src = os.path.join(G, "launch_d.csv")
if os.path.exists(src):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), src, "4", "-v"],
                         capture_output=True, text=True).stdout
    open(os.path.join(P, f"ncu_launches_d_{rnd}.txt"), "w").write(
        "# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
        "python bench.py --workload D --steps 1 --warmup 3\n# (last of 4 decodes; serialized: per-launch SHARES "
        "are meaningful, absolute sums are not)\n" + out)
for name in ("layers_b", "layers_c", "swap_timeline_b"):
    src = os.path.join(G, f"{name}.txt")
    if os.path.exists(src):
        shutil.copy(src, os.path.join(P, f"{name}_{rnd}.txt"))
src = os.path.join(G, "launch_b.csv")
if os.path.exists(src):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "membound_report.py"), src, "3"],
                         capture_output=True, text=True).stdout
    open(os.path.join(P, f"membound_b_{rnd}.txt"), "w").write(out)
print("collected into", P)
