"""Multi-GPU sliced decode: the host-side partition and the frame gather.

* world_size 2 over gloo on CPU: each rank decodes its contiguous frame
  block (lc_shard_frames) with the oracle decoder, the blocks are gathered
  to rank 0 and must equal the single-process decode bit-exactly (decode is
  frame-wise, proj/src/codec.cpp:126-145).
* On one GPU: lc_decode_sharded with world 1 equals lc_decode.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TINY = {"run.frames": 5, "run.height": 32, "run.width": 32, "sampler.steps": 2}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, lat, out_path):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch

    import lco
    import paper_2510_05367_b200 as lc
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    kv = lco.parse_text(lc.DEFAULT_CONFIG)
    kv.update({k: str(v) for k, v in TINY.items()})
    T = lat.shape[1]
    f0, cnt = lc.shard_frames(T, world, rank)
    part = lco.Restatement().decode(kv, lat[:, f0:f0 + cnt]) if cnt else np.zeros((1, 0, 3, 32, 32), np.float32)
    # pad to equal chunks for all_gather (ncclAllGather-style)
    per = -(-T // world)
    buf = np.zeros((per, 3, 32, 32), np.float32)
    buf[:cnt] = part[0]
    out = [torch.zeros(per, 3, 32, 32) for _ in range(world)]
    dist.all_gather(out, torch.from_numpy(buf))
    if rank == 0:
        frames = []
        for r in range(world):
            g0, gc = lc.shard_frames(T, world, r)
            frames.append(out[r][:gc].numpy())
        np.save(out_path, np.concatenate(frames)[None])
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_decode_gather_gloo(tmp_path, oracle, world):
    import lco
    import paper_2510_05367_b200 as lc
    kv = lco.parse_text(lc.DEFAULT_CONFIG)
    kv.update({k: str(v) for k, v in TINY.items()})
    lat = np.random.default_rng(0).standard_normal((1, 5, 4, 8, 8)).astype(np.float32)
    out_path = str(tmp_path / "video.npy")
    mp.start_processes(_worker, args=(world, _free_port(), lat, out_path), nprocs=world, start_method="fork")
    got = np.load(out_path)
    want = oracle.decode(kv, lat)
    assert np.array_equal(got, want)


@pytest.mark.gpu
def test_decode_sharded_single_rank_equals_decode(ctx):
    import paper_2510_05367_b200 as lc
    ctx.configure(lc.config_text(TINY, base=lc.DEFAULT_CONFIG))
    lat = np.random.default_rng(1).standard_normal((1, 5, 4, 8, 8)).astype(np.float32)
    a = ctx.decode(lat, slice_frames=2)
    b, ms = ctx.decode_sharded(lat, slice_frames=2)
    assert np.array_equal(a, b) and ms > 0


@pytest.mark.gpu
def test_decode_sharded_repeated_calls_and_pinned_buffers(ctx):
    """The shard buffers persist across calls (bench workload D): repeated
    calls, a shorter latent after a longer one, and pinned host buffers all
    give the single-device decode bit for bit."""
    import paper_2510_05367_b200 as lc
    over = dict(TINY, **{"run.frames": 6})
    ctx.configure(lc.config_text(over, base=lc.DEFAULT_CONFIG))
    rng = np.random.default_rng(2)
    lat6 = rng.standard_normal((1, 6, 4, 8, 8)).astype(np.float32)
    want6 = ctx.decode(lat6, slice_frames=4)
    for _ in range(3):
        got, _ = ctx.decode_sharded(lat6, slice_frames=4)
        assert np.array_equal(got, want6)
    lat3 = lat6[:, :3].copy()
    got3, _ = ctx.decode_sharded(lat3, slice_frames=4)
    assert np.array_equal(got3, want6[:, :3])
    lp, vp = lc.PinnedArray(lat6.size), lc.PinnedArray(want6.size)
    lp.array[:] = lat6.reshape(-1)
    vid, _ = ctx.decode_sharded(lp, slice_frames=4, out=vp)
    assert np.array_equal(vid, want6)
    lp.free()
    vp.free()
