"""World-size-2 gloo tests (CPU) of the multi-GPU plumbing:
frame partitioning, scene broadcast, key-frame mask sharing, frame gather and
the max-over-ranks timing."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_16422_b200 import dist as fdist
from paper_2503_16422_b200.api import bracket, keyframes


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _fake_mask(k, words):
    """Deterministic stand-in for fdgs_keyframe_mask (no GPU here)."""
    rng = np.random.default_rng(1000 + k)
    return rng.integers(0, 2 ** 32, words, dtype=np.uint64).astype(np.uint32).view(np.int32)


def _fake_render(frame, shape):
    f, ti, ci = frame
    return torch.full(shape, float(f * 7 + ti * 3 + ci), dtype=torch.float32)


def _worker(rank, world_size, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    try:
        # scene broadcast: rank 0 owns the data
        shapes = {"mean": (10, 4), "sh": (10, 16, 3), "opacity": (10,)}
        tens = {k: (torch.arange(int(np.prod(s)), dtype=torch.float32).reshape(s) if rank == 0
                    else torch.zeros(s)) for k, s in shapes.items()}
        fdist.broadcast_scene(tens)
        ok_scene = all(torch.equal(tens[k], torch.arange(int(np.prod(s)), dtype=torch.float32).reshape(s))
                       for k, s in shapes.items())
        # key-frame masks: rank k mod N builds row k
        built = []

        def build(k, out):
            built.append(k)
            out.copy_(torch.from_numpy(_fake_mask(k, out.numel())))

        kf = keyframes(300, 20)
        masks = fdist.share_keyframe_masks(len(kf), 37, build, "cpu")
        want = np.stack([_fake_mask(k, 37) for k in range(len(kf))])
        ok_masks = np.array_equal(masks.numpy(), want)
        # frame partition + gather to rank 0
        seq = [(f, f // 20, f % 20) for f in range(40)]
        mine = fdist.shard_frames(seq, rank, world_size)
        batch = torch.stack([_fake_render(x, (3, 2, 2)) for x in mine[:8]])
        got = fdist.gather_frames(batch)
        ok_gather = True
        if rank == 0:
            for r in range(world_size):
                exp = torch.stack([_fake_render(x, (3, 2, 2)) for x in fdist.shard_frames(seq, r, world_size)[:8]])
                ok_gather &= torch.equal(got[r], exp)
        # slowest rank defines the job time
        t = fdist.max_over_ranks(10.0 + rank, "cpu")
        total = fdist.sum_over_ranks(len(mine), "cpu")
        results[rank] = dict(scene=ok_scene, masks=ok_masks, built=built, mine=[x[0] for x in mine],
                             gather=ok_gather, tmax=t, total=total,
                             brackets=[bracket(kf, x[1]) for x in mine[:5]])
    finally:
        dist.destroy_process_group()


def test_two_rank_plumbing():
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(2, port, results), nprocs=2, join=True)
    r0, r1 = results[0], results[1]
    assert r0["scene"] and r1["scene"]
    assert r0["masks"] and r1["masks"]
    assert r0["built"] == list(range(0, 16, 2)) and r1["built"] == list(range(1, 16, 2))
    assert sorted(r0["mine"] + r1["mine"]) == list(range(40))
    assert all(f % 2 == 0 for f in r0["mine"]) and all(f % 2 == 1 for f in r1["mine"])
    assert r0["gather"]
    assert r0["tmax"] == r1["tmax"] == 11.0
    assert r0["total"] == 40.0
