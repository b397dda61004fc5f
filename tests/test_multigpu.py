"""Multi-GPU sliced decode: the host-side partition and the frame gather.

* world_size 2/3/4/8 over gloo on CPU: every rank takes its balanced frame
  block (lc_shard_frames), decodes it slice by slice with the oracle
  decoder, and the ranks execute the product's gather schedule
  (lc_gather_plan: round i sends the i-th slice of every rank to rank 0)
  with point-to-point send/recv -- the same rows lc_decode_sharded issues as
  ncclSend / grouped ncclRecv on the GPU.  Rank 0's assembled video must
  equal the single-process decode bit-exactly (decode is frame-wise,
  proj/src/codec.cpp:126-145).
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


def _worker(rank, world, port, lat, slice_frames, out_path):
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
    H = W = 32
    f0, cnt = lc.shard_frames(T, world, rank)
    plan = lc.gather_plan(T, world, slice_frames)
    # this rank's slices, decoded one at a time (decode_sliced per slice)
    mine = [r for r in plan if r[1] == rank]
    assert sum(int(r[3]) for r in mine) == cnt
    decoded = {}
    for rnd, _, first, count in mine:
        assert f0 <= first and first + count <= f0 + cnt
        decoded[int(first)] = lco.Restatement().decode(kv, lat[:, first:first + count])[0]
    video = np.full((T, 3, H, W), np.nan, np.float32) if rank == 0 else None
    for rnd, r, first, count in plan:
        first, count = int(first), int(count)
        if r == 0:
            if rank == 0:
                video[first:first + count] = decoded[first]
        elif rank == 0:
            buf = torch.empty(count, 3, H, W)
            dist.recv(buf, src=int(r))
            video[first:first + count] = buf.numpy()
        elif rank == r:
            dist.send(torch.from_numpy(decoded[first]), dst=0)
    if rank == 0:
        np.save(out_path, video[None])
    dist.destroy_process_group()


@pytest.mark.parametrize("world,slice_frames", [(2, 2), (3, 1), (4, 2), (8, 1)])
def test_sharded_decode_gather_gloo(tmp_path, oracle, world, slice_frames):
    import lco
    import paper_2510_05367_b200 as lc
    kv = lco.parse_text(lc.DEFAULT_CONFIG)
    kv.update({k: str(v) for k, v in TINY.items()})
    lat = np.random.default_rng(0).standard_normal((1, 5, 4, 8, 8)).astype(np.float32)
    out_path = str(tmp_path / "video.npy")
    # spawn, not fork: the parent's OpenMP pool (the oracle decoder) does
    # not survive a fork (libgomp hangs in the child)
    mp.start_processes(_worker, args=(world, _free_port(), lat, slice_frames, out_path), nprocs=world,
                       start_method="spawn")
    got = np.load(out_path)
    want = oracle.decode(kv, lat)
    assert np.array_equal(got, want)


def test_gather_plan_rounds():
    """Every frame is moved exactly once, slices never exceed the slice
    size, and round i holds the i-th slice of each rank that has one."""
    import paper_2510_05367_b200 as lc
    for T in (1, 5, 16, 25):
        for world in (1, 2, 3, 4, 8):
            for sl in (1, 2, 4, 5):
                plan = lc.gather_plan(T, world, sl)
                frames = sorted(f for _, _, a, c in plan for f in range(a, a + c))
                assert frames == list(range(T))
                assert all(1 <= c <= sl for *_, c in plan)
                for r in range(world):
                    f0, cnt = lc.shard_frames(T, world, r)
                    rows = [row for row in plan if row[1] == r]
                    assert [int(x[0]) for x in rows] == list(range(len(rows)))
                    assert [int(x[2]) for x in rows] == list(range(f0, f0 + cnt, sl))


@pytest.mark.gpu
def test_decode_sharded_single_rank_equals_decode(ctx):
    import paper_2510_05367_b200 as lc
    ctx.configure(lc.config_text(TINY, base=lc.DEFAULT_CONFIG))
    lat = np.random.default_rng(1).standard_normal((1, 5, 4, 8, 8)).astype(np.float32)
    a = ctx.decode(lat, slice_frames=2)
    b, ms = ctx.decode_sharded(lat, slice_frames=2, out=np.empty(a.size, np.float32))
    assert np.array_equal(a, b) and ms > 0
    # device-only form (the gathered video stays in HBM): same call, no output
    none, ms2 = ctx.decode_sharded(lat, slice_frames=2)
    assert none is None and ms2 > 0


@pytest.mark.gpu
def test_decode_rejects_wrong_latent_geometry(ctx):
    """decode_batch / decode_sliced raise ShapeError on a channel mismatch
    (proj/src/codec.cpp:129-131); the engine also rejects a latent h x w
    other than the configured one (no host overrun)."""
    import paper_2510_05367_b200 as lc
    ctx.configure(lc.config_text(TINY, base=lc.DEFAULT_CONFIG))
    with pytest.raises(lc.ShapeError):
        ctx.decode(np.zeros((1, 2, 3, 8, 8), np.float32))
    with pytest.raises(lc.ShapeError):
        ctx.decode(np.zeros((1, 2, 4, 16, 8), np.float32))
    with pytest.raises(lc.ShapeError):
        ctx.decode_sharded(np.zeros((1, 2, 5, 8, 8), np.float32), out=np.empty(2 * 3 * 32 * 32, np.float32))


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
        got, _ = ctx.decode_sharded(lat6, slice_frames=4, out=np.empty(want6.size, np.float32))
        assert np.array_equal(got, want6)
    lat3 = lat6[:, :3].copy()
    got3, _ = ctx.decode_sharded(lat3, slice_frames=4, out=np.empty(want6.size // 2, np.float32))
    assert np.array_equal(got3, want6[:, :3])
    lp, vp = lc.PinnedArray(lat6.size), lc.PinnedArray(want6.size)
    lp.array[:] = lat6.reshape(-1)
    vid, _ = ctx.decode_sharded(lp, slice_frames=4, out=vp)
    assert np.array_equal(vid, want6)
    lp.free()
    vp.free()


@pytest.mark.gpu
def test_decode_sharded_into_shared_host_video(ctx):
    """LC_SHARD_HOST_SHARED: the rank writes its frames straight into one
    page-locked shared-memory video (the multi-rank e2e path of bench.py);
    at world 1 that is every frame, bit-identical to lc_decode."""
    import paper_2510_05367_b200 as lc
    over = dict(TINY, **{"run.frames": 6})
    ctx.configure(lc.config_text(over, base=lc.DEFAULT_CONFIG))
    lat = np.random.default_rng(4).standard_normal((1, 6, 4, 8, 8)).astype(np.float32)
    want = ctx.decode(lat, slice_frames=4)
    name = f"lc_test_video_{os.getpid()}"
    shared = lc.SharedVideo(name, want.size, create=True)
    try:
        shared.array[:] = np.nan
        got, ms = ctx.decode_sharded(lat, slice_frames=4, out=shared, host_shared=True)
        assert ms > 0 and np.array_equal(got, want)
        # a second mapping of the same segment sees the frames (another rank's view)
        other = lc.SharedVideo(name, want.size, create=False)
        assert np.array_equal(other.array.reshape(want.shape), want)
        other.free()
    finally:
        shared.free()
