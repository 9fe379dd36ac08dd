"""World-size-2/3 gloo tests (CPU) of the multi-GPU plumbing:
frame partitioning, scene broadcast, key-frame mask sharing, the chunked
frame gather to rank 0 and the max-over-ranks timing -- and bench.py's own
multi-rank orchestration (self-spawned under torch.distributed.run, with the
CPU stand-in renderer of --fake-render)."""
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
        # frame partition + chunked gather to rank 0 (7 frames, chunks of 3: a ragged tail)
        seq = [(f, f // 20, f % 20) for f in range(40)]
        mine = fdist.shard_frames(seq, rank, world_size)
        g = fdist.FrameGather((3, 2, 2), 3, "cpu", ring=4)
        frames = [_fake_render(x, (3, 2, 2)) for x in mine[:7]]
        g.begin_step(7)
        for k, fr in enumerate(frames):
            g.frame_done(k, fr, None)
        g.end_step()
        ok_gather = True
        if rank == 0:
            assert g.chunks == 3 and g.bytes_received == (world_size - 1) * 7 * 48
            for r in range(1, world_size):
                exp = [_fake_render(x, (3, 2, 2)) for x in fdist.shard_frames(seq, r, world_size)[:7]]
                for k in range(7):
                    ok_gather &= torch.equal(g.ring[k // 3, r - 1, k % 3], exp[k])
        else:
            assert g.bytes_sent == 7 * 48
        chk = g.validate(frames)
        ok_gather &= (rank != 0) or (chk["ok"] and chk["frames"] == (world_size - 1) * 7)
        # slowest rank defines the job time
        t = fdist.max_over_ranks(10.0 + rank, "cpu")
        total = fdist.sum_over_ranks(len(mine), "cpu")
        results[rank] = dict(scene=ok_scene, masks=ok_masks, built=built, mine=[x[0] for x in mine],
                             gather=ok_gather, tmax=t, total=total,
                             brackets=[bracket(kf, x[1]) for x in mine[:5]])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world_size", [2, 3])
def test_multi_rank_plumbing(world_size):
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world_size, port, results), nprocs=world_size, join=True)
    rs = [results[r] for r in range(world_size)]
    assert all(r["scene"] and r["masks"] for r in rs)
    for r in range(world_size):
        assert rs[r]["built"] == list(range(r, 16, world_size))
        assert all(f % world_size == r for f in rs[r]["mine"])
    assert sorted(sum((r["mine"] for r in rs), [])) == list(range(40))
    assert all(r["gather"] for r in rs)
    assert all(r["tmax"] == 10.0 + world_size - 1 for r in rs)
    assert rs[0]["total"] == 40.0


def test_bench_orchestration_two_ranks():
    """bench.py --gpus 2 without a launcher spawns its own two ranks (gloo here,
    --fake-render) and runs exactly its multi-rank path: scene broadcast, mask
    sharing, frame partition, per-step barrier + timing, the chunked frame
    gather to rank 0 inside the timed steps, validation on rank 0, max-over-
    ranks reduction; rank 0 alone prints the JSON line."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--fake-render", "--steps", "3", "--warmup", "1",
                        "--frames-per-step", "13", "--gather-chunk", "4"], cwd=root, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1                       # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["config"]["frames_per_rank"] == 39
    fk = d["fake_render"]
    assert fk["scene_broadcast_ok"] and fk["masks_ok"] and fk["frames_rank0"] == [0, 2, 4, 6]
    g = d["gather"]
    assert g["validated_ok"] and g["validated_frames"] == 13 and g["fake_content_ok"]
    assert g["bytes_into_rank0_per_step"] == 13 * 3 * 6 * 8 * 4
    # value = all frames / the slowest rank's total time
    tmax = max(fk["per_rank_total_ms"])
    assert abs(d["value"] - 2 * 39 / (tmax / 1e3)) <= 1e-4 * d["value"]  # (totals rounded to 0.1 us)
    # per-step statistics over the max-over-ranks step times, outliers listed
    st = d["step_stats"]
    assert st["min_ms"] <= st["median_ms"] <= st["max_ms"] and isinstance(st["outliers"], list)
    assert all(o["ms"] > 1.5 * st["median_ms"] for o in st["outliers"])
    assert d["config"]["submission"].startswith("per frame: one CUDA-graph launch")
