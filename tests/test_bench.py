"""bench.py's host-side contract on CPU: `--gpus N` without torchrun spawns
N local ranks (RANK / LOCAL_RANK / WORLD_SIZE / MASTER_* as torchrun sets
them, gloo plumbing), rank 0 alone runs the reference arm and prints ONE
JSON line with the GPU arm's metric / config; the reference arm never
loads the product library."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_self_spawned_ranks(tmp_path):
    env = dict(os.environ)
    for k in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    # a tiny workload keeps the CPU sample short
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0", "--workload", "A"], capture_output=True, text=True,
                       timeout=600, env=env, cwd=str(tmp_path))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["metric"] == "video_frames_per_sec" and d["n_gpus"] == 2
    assert d["value"] > 0 and d["steps"] == 1 and d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_reference_arm_does_not_load_the_product():
    code = ("import sys, bench; bench.cpu_sample('C'); "
            "assert 'paper_2510_05367_b200' not in sys.modules, 'product imported'; print('ok')")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
