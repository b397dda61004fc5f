"""CLI, run artifacts and the comparison harness:
the reference's subcommands, exit codes (proj/tools/main.cpp:157-169),
artifact formats (report.json, ledger.json/.csv, video.raw + .hdr) and the
compare / sweep-n / export-plots tables."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import lco
import paper_2510_05367_b200 as lc
from paper_2510_05367_b200 import harness as H

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
TINY = ["run.frames=2", "run.height=32", "run.width=32", "sampler.steps=6"]


def _cli(*args, cwd=None):
    return subprocess.run([sys.executable, "-m", "paper_2510_05367_b200", *args], cwd=cwd or ROOT,
                          capture_output=True, text=True, timeout=600)


# ---------------------------------------------------------------- CPU
@pytest.mark.parametrize("args,code", [
    (["--set", "badkv", "run"], 2),                       # --set expects key=value
    (["--set", "foo.bar=1", "run"], 2),                   # unknown key
    (["--set", "run.frames=0", "run"], 2),                # validate()
    (["--set", "run.height=65", "run"], 2),               # codec-scale divisibility
    (["--set", "sampler.kind=heun", "run"], 2),           # bad enum
    (["sweep-n", "--n", "3,2"], 2),                       # N ascending
    (["sweep-n", "--n", ","], 2),                         # empty N list
])
def test_cli_config_errors_exit_like_the_reference(args, code):
    r = _cli(*args)
    assert r.returncode == code, r.stderr
    assert r.stderr.startswith("config error:")


def test_cli_config_file_and_overrides(tmp_path):
    cfg = tmp_path / "c.cfg"
    cfg.write_text("# comment\nrun.frames = 3\nsampler.kind = ddim\n")
    text = H.build_config(str(cfg), ["sampler.steps=7"], str(tmp_path / "o"))
    kv = lc.parse_config(text)
    assert kv["run.frames"] == "3" and kv["sampler.kind"] == "ddim" and kv["sampler.steps"] == "7"
    assert kv["run.out_dir"] == str(tmp_path / "o")


def test_config_json_matches_reference_report():
    """config_to_json (proj/src/config.cpp:267-301) of the golden tiny run."""
    g = np.load(os.path.join(GOLD, "tiny.npz"))
    want = json.loads(str(g["report"]))["config"]
    got = H.config_json(str(g["config"]))
    want["run"].pop("out_dir")
    got["run"].pop("out_dir")
    assert got == want


def test_video_raw_is_byte_identical_to_reference_writer(tmp_path, reference):
    v = np.random.default_rng(1).standard_normal((1, 3, 3, 8, 12)).astype(np.float32)
    H.write_video_raw(str(tmp_path / "ours.raw"), v)
    reference.write_video_raw(str(tmp_path / "ref.raw"), v[0])
    assert (tmp_path / "ours.raw").read_bytes() == (tmp_path / "ref.raw").read_bytes()
    assert (tmp_path / "ours.raw.hdr").read_text() == (tmp_path / "ref.raw.hdr").read_text()
    assert np.array_equal(H.read_video_raw(str(tmp_path / "ours.raw")), v)


def test_metrics_csv_format():
    """write_metrics_csv (proj/src/metrics.cpp:106-117), precision(10)."""
    txt = H.metrics_csv([99.0, 31.234567891234], [1.0, 0.91234567891])
    assert txt == "frame_index,psnr,ssim\n0,99,1\n1,31.23456789,0.9123456789\n"


# ---------------------------------------------------------------- GPU
def _keys(d):
    return {k: _keys(v) for k, v in d.items()} if isinstance(d, dict) else None


@pytest.mark.gpu
def test_cli_run_writes_reference_artifacts(tmp_path):
    out = tmp_path / "run"
    r = _cli("--out", str(out), *sum((["--set", kv] for kv in TINY), []), "run")
    assert r.returncode == 0, r.stderr
    rep = json.loads((out / "report.json").read_text())
    g = np.load(os.path.join(GOLD, "tiny.npz"))
    want = json.loads(str(g["report"]))
    assert _keys(rep) == _keys(want)  # run_report_json layout
    assert rep["mac"] == want["mac"] and rep["cache_bytes"] == want["cache_bytes"]
    assert rep["video"] == want["video"]
    video = H.read_video_raw(str(out / "video.raw"))
    assert lc.rel_l2(video, g["video"]) < 1e-3
    led = json.loads((out / "ledger.json").read_text())
    assert set(led) == {"clock", "stages", "overall", "current", "event_count", "run"}
    rows = (out / "ledger.csv").read_text().splitlines()
    assert rows[0] == "seq,clock,kind,tier,bytes,alloc_id,occupancy_bytes,stage"
    assert len(rows) - 1 == led["event_count"]
    # replaying the log reproduces the peaks (replay_csv_peaks, ledger.cpp:244-283)
    occ, peak = {"fast": 0, "slow": 0}, {}
    for row in rows[1:]:
        _, _, kind, tier, nbytes, _, occ_after, stage = row.split(",")
        if kind in ("alloc", "move_start"):  # a move's start row carries the destination tier
            occ[tier] += int(nbytes)
        elif kind in ("free", "move_end"):  # its end row the source tier
            occ[tier] -= int(nbytes)
        assert occ[tier] == int(occ_after)
        peak[(stage, tier)] = max(peak.get((stage, tier), 0), occ[tier])
    assert occ["fast"] == led["current"]["fast_bytes"] and occ["slow"] == led["current"]["slow_bytes"]
    for s in H.STAGES:
        for t in ("fast", "slow"):
            assert peak.get((s, t), 0) <= led["stages"][s][f"{t}_peak_bytes"]


@pytest.mark.gpu
def test_compare_and_sweep_tables(ctx, oracle, tmp_path):
    text = H.build_config(None, TINY, str(tmp_path))
    row = H.compare(ctx, H.baseline_text(text), text)
    assert set(row) == {"speed_up", "psnr_mean", "ssim_mean", "psnr_per_frame", "ssim_per_frame", "variant_macs",
                        "baseline_macs", "identical_video", "peak_delta_fast"}
    assert row["baseline_macs"] > row["variant_macs"] and not row["identical_video"]
    base = H.run_pipeline(ctx, H.baseline_text(text))
    var = H.run_pipeline(ctx, text)
    ps, ss = oracle.video_metrics(base.video[0], var.video[0], 1.0)
    np.testing.assert_allclose(row["psnr_per_frame"], ps, rtol=1e-12)
    np.testing.assert_allclose(row["ssim_per_frame"], ss, rtol=1e-12)
    same = H.compare(ctx, H.baseline_text(text), H.baseline_text(text))
    assert same["identical_video"] and same["psnr_mean"] == 99.0 and same["ssim_mean"] == 1.0
    table = H.sweep_n(ctx, text, [1, 2, 3])
    assert [r["n"] for r in table["rows"]] == [1, 2, 3]
    assert table["rows"][0]["psnr_mean"] == 99.0  # N=1 == cache off, bit-identical
    paths = H.export_plots(ctx, text, [2], str(tmp_path))
    lines = open(paths[0]).read().splitlines()
    assert lines[0] == "frame_index,psnr,ssim" and len(lines) == 3


@pytest.mark.gpu
def test_cli_ablate(tmp_path):
    r = _cli("--out", str(tmp_path), *sum((["--set", kv] for kv in TINY), []), "ablate")
    assert r.returncode == 0, r.stderr
    rows = json.loads((tmp_path / "ablate.json").read_text())
    assert [x["label"] for x in rows] == ["all-on", "-swapping", "-slicing", "-chunk", "cache-only"]
    r = _cli("--out", str(tmp_path), "--set", "swap.mode=off", "ablate")
    assert r.returncode == 2
