"""The committed frame-0 goldens at the B / C shapes are the reference's own
output: tests/golden/make_golden.py `pin` ran oracle/_ref's run_pipeline on
each config and found the restatement's video bit-identical, and stored the
reference's video, its MAC counter and wall time."""
import os

import numpy as np
import pytest

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FRAME0 = ["b_frame0", "c_frame0", "b_frame0_ancestral", "b_frame0_ddim", "b_frame0_image", "b_frame0_fixed_k5",
          "c_frame0_none_s2", "c_frame0_fixed_k5_s2", "b_frame0_none"]


@pytest.mark.parametrize("name", FRAME0)
def test_frame0_golden_is_pinned_to_the_reference(name):
    import lco
    g = np.load(os.path.join(HERE, f"{name}.npz"))
    assert str(g["video_source"]) == "oracle/_ref"
    kv = lco.parse_text(str(g["config"]))
    s = 1 << int(kv["codec.stages"])
    T, H, W = int(kv["run.frames"]), int(kv["run.height"]), int(kv["run.width"])
    assert T == 1 and g["video"].shape == (1, 1, 3, H, W) and g["latent"].shape == (1, 1, 4, H // s, W // s)
    assert np.isfinite(g["video"]).all() and np.isfinite(g["latent"]).all()
    assert int(g["macs"][0]) > 0 and float(g["ref_seconds"]) > 0


SAMPLER_CASES = ["euler_t24", "euler_t0", "ddim_t12", "ddim_t0", "ancestral_t7", "ancestral_t0", "euler_s6_t5",
                 "ancestral_s6_t3"]


@pytest.mark.parametrize("name", SAMPLER_CASES)
def test_sampler_golden_matches_live_reference(reference, name):
    """tests/golden/sampler.npz (cfg_combine + reverse_step_*,
    proj/src/sampler.cpp:95-133) equals a live oracle/_ref call bit for bit."""
    import lco
    g = np.load(os.path.join(HERE, "sampler.npz"))
    kind, t, seed = (int(v) for v in g[name + "_args"])
    out = reference.sampler_step(lco.parse_text(str(g[name + "_config"])), kind, t, g[name + "_x"],
                                 g[name + "_eu"], g[name + "_ec"], float(g[name + "_g"]), seed)
    assert np.array_equal(out, g[name + "_out"])


def test_sampler_reference_errors(reference):
    """check_t (sampler.cpp:79-84) and the guidance check (sampler.cpp:130)
    raise ConfigError (exit code 2)."""
    import lco
    kv = lco.parse_text("")
    x = np.zeros(8, np.float32)
    for kind, t, g in [(2, 25, 1.5), (1, -1, 1.5), (0, 3, -0.5)]:
        with pytest.raises(lco.OracleError) as e:
            reference.sampler_step(kv, kind, t, x, x, x, g)
        assert e.value.code == 2
