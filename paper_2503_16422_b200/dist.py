"""Multi-GPU plumbing of the frame-parallel render.

Frames (distinct (camera, t) pairs of a sequence, "render the images
from any viewpoint at a given timestamp") are independent given a replicated
scene and replicated key-frame masks, so the render itself has no collective:
frame f goes to rank f mod N (one process per GPU).  torch.distributed (NCCL
over NVLink on GPUs, gloo in the CPU tests) carries what BASELINE.json's
north_star names -- the scene and masks out, the frames and timings back:

* ``broadcast_scene``       scene arrays from rank 0 to every rank;
* ``share_keyframe_masks``  key-frame k built by rank k mod N, one all-reduce
                            (disjoint rows summed);
* ``FrameGather``           every rank's rendered frames to rank 0, in chunks
                            of grouped P2P send/recv issued on a side stream as
                            soon as a chunk's blends finish, so the transfer
                            overlaps the rendering of later frames; rank 0
                            receives into a bounded ring buffer and validates a
                            sample against the senders' checksums;
* ``max_over_ranks``        the job time is the slowest rank's device time.

``launch_self`` re-executes a script under torch.distributed.run when a
multi-GPU run is requested without a launcher (``bench.py --gpus N``).
"""
from __future__ import annotations

import os
import socket
import sys

import torch
import torch.distributed as dist


def world():
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def env_ranks():
    """(rank, world_size, local_rank) from the launcher's environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launch_self(n: int, argv=None):
    """Re-execute the running script as n ranks under torch.distributed.run
    (rendezvous on 127.0.0.1).  Does not return."""
    argv = list(sys.argv if argv is None else argv)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), *argv]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def init(backend: str, device=None):
    """init_process_group from the launcher's environment (no-op at world 1)."""
    rank, n, _ = env_ranks()
    if n > 1 and not dist.is_initialized():
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group(backend)
    return world()


def barrier():
    if world()[1] > 1:
        dist.barrier()


def shutdown():
    if dist.is_available() and dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


def shard_frames(frames: list, rank: int, world_size: int) -> list:
    """Round-robin partition of the sequence: frame f -> rank f mod N."""
    return [x for i, x in enumerate(frames) if i % world_size == rank]


_NCCL_NATIVE = {torch.float32, torch.float64, torch.float16, torch.bfloat16, torch.int32, torch.int64,
                torch.uint8, torch.int8}


def broadcast_scene(tensors: dict, src: int = 0) -> dict:
    """In-place broadcast of every scene tensor from `src` (sorted keys are the
    protocol: all ranks pass the same keys with the same shapes and dtypes).
    Dtypes NCCL lacks (the uint16 VQ index) travel as bytes."""
    _, n = world()
    if n > 1:
        for k in sorted(tensors):
            t = tensors[k]
            dist.broadcast(t if t.dtype in _NCCL_NATIVE else t.view(torch.uint8), src=src)
    return tensors


def share_keyframe_masks(n_keyframes: int, words: int, build, device) -> torch.Tensor:
    """masks[k] = build(k, out) computed on rank k mod N, replicated everywhere.

    `build(k, out)` fills the int32 row `out` (ceil(N/32) words).  Rows are
    disjoint across ranks, so a SUM all-reduce reproduces every row exactly."""
    rank, n = world()
    masks = torch.zeros((n_keyframes, words), dtype=torch.int32, device=device)
    for k in range(n_keyframes):
        if k % n == rank:
            build(k, masks[k])
    if n > 1:
        # int32 sum of one non-zero row and zeros is exact for every bit pattern
        dist.all_reduce(masks, op=dist.ReduceOp.SUM)
    return masks


def max_over_ranks(value: float, device) -> float:
    _, n = world()
    if n == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device) -> float:
    _, n = world()
    if n == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_timings(values, device) -> list:
    """Per-rank lists of floats (equal lengths) on every rank: [rank][k]."""
    rank, n = world()
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    if n == 1:
        return [t.tolist()]
    out = [torch.empty_like(t) for _ in range(n)]
    dist.all_gather(out, t)
    return [x.tolist() for x in out]


class FrameGather:
    """Every rank's frames to rank `dst` (BASELINE north_star: "NCCL ... to
    gather frames"), chunked and overlapped with rendering.

    Protocol, identical on every rank (all ranks render the same number of
    frames per step, in submission order):
      begin_step(n)            n frames follow in this step;
      frame_done(k, out, st, ev) frame k's output `out` is complete once stream
                               `st` reaches this point, or once event `ev`
                               completes (None, None on CPU);
      end_step(main)           issues the last partial chunk and makes stream
                               `main` wait for every transfer of the step, so
                               a step's time includes its gather.
    Every `chunk` frames, senders issue one group of `chunk` sends (grouped
    NCCL P2P, one kernel) on a side stream that waited for those frames;
    rank `dst` issues the matching group of receives from every other rank
    into a ring of `ring` chunk slots (bounded memory; a slot is reused once
    the receives before it on the NCCL stream completed).  Rank dst's own
    frames stay where they are.
    """

    def __init__(self, frame_shape, chunk: int, device, dst: int = 0, ring: int = 2, dtype=torch.float32):
        self.rank, self.world = world()
        self.dst = dst
        self.chunk = max(1, int(chunk))
        self.device = torch.device(device)
        self.cuda = self.device.type == "cuda"
        self.frame_shape = tuple(frame_shape)
        self.frame_bytes = int(torch.Size(frame_shape).numel()) * torch.tensor([], dtype=dtype).element_size()
        self.stream = torch.cuda.Stream(self.device) if self.cuda else None
        self.ring = None
        if self.rank == dst and self.world > 1:
            self.ring = torch.empty((ring, self.world - 1, self.chunk, *frame_shape), dtype=dtype, device=self.device)
        self.slot = 0
        self._pending = []    # frames of the open chunk
        self._works = []      # outstanding P2P works of this step
        self._n = 0
        self._events = []
        self.bytes_sent = 0
        self.bytes_received = 0
        self.chunks = 0
        self.last = None      # (slot, count) of the last chunk received on dst

    # -------------------------------------------------------------- steps
    def begin_step(self, n_frames: int):
        self._n = int(n_frames)
        self._k = 0
        self._pending = []
        self._works = []

    def _event(self, i):
        while len(self._events) <= i:
            self._events.append(torch.cuda.Event())
        return self._events[i]

    def frame_done(self, k: int, out: torch.Tensor, stream=None, event=None):
        """Frame k's output is complete once `stream` reaches this point, or
        once `event` (already recorded) completes."""
        if self.world == 1:
            return
        if self.cuda and event is not None:
            self.stream.wait_event(event)
        elif self.cuda and stream is not None:
            ev = self._event(len(self._pending))
            ev.record(stream)
            self.stream.wait_event(ev)
        self._pending.append(out)
        if len(self._pending) == self.chunk:
            self._flush()

    def _flush(self):
        if not self._pending:
            return
        cnt = len(self._pending)
        ops = []
        if self.rank == self.dst:
            slot = self.slot % self.ring.shape[0]
            for r in range(self.world):
                if r == self.dst:
                    continue
                ri = r if r < self.dst else r - 1
                for g in range(cnt):
                    ops.append(dist.P2POp(dist.irecv, self.ring[slot, ri, g], r))
            self.bytes_received += (self.world - 1) * cnt * self.frame_bytes
            self.last = (slot, cnt)
            self.slot += 1
        else:
            for t in self._pending:
                ops.append(dist.P2POp(dist.isend, t, self.dst))
            self.bytes_sent += cnt * self.frame_bytes
        if self.cuda:
            with torch.cuda.stream(self.stream):
                self._works += dist.batch_isend_irecv(ops)
        else:
            self._works += dist.batch_isend_irecv(ops)
        self.chunks += 1
        self._pending = []

    def end_step(self, main_stream=None):
        """Issue the partial chunk; `main_stream` (or the host, on CPU) waits
        for every transfer of the step."""
        if self.world == 1:
            return
        self._flush()
        if self.cuda:
            with torch.cuda.stream(main_stream or torch.cuda.current_stream(self.device)):
                for w in self._works:
                    w.wait()      # stream-ordered: main waits for the NCCL stream
        else:
            for w in self._works:
                w.wait()
        self._works = []

    # ---------------------------------------------------------- validation
    def validate(self, frames: list) -> dict:
        """Gather `frames` (this rank's, equal count on every rank) once more,
        synchronously, and compare on rank dst each received frame's float64
        sum with the sender's (a second small message).  Returns
        {"frames": checked, "ok": bool} on dst, {} elsewhere."""
        if self.world == 1:
            return {"frames": 0, "ok": True}
        n = len(frames)
        sums = torch.stack([f.double().sum() for f in frames]) if n else torch.zeros(0, dtype=torch.float64,
                                                                                      device=self.device)
        ok, checked = True, 0
        for c0 in range(0, n, self.chunk):
            part = frames[c0:c0 + self.chunk]
            self.begin_step(len(part))
            for k, f in enumerate(part):
                self.frame_done(k, f, torch.cuda.current_stream(self.device) if self.cuda else None)
            self.end_step()
            if self.cuda:
                torch.cuda.current_stream(self.device).synchronize()
            ps = sums[c0:c0 + len(part)].contiguous()
            if self.rank == self.dst:
                slot, cnt = self.last
                got = torch.empty((self.world - 1, cnt), dtype=torch.float64, device=self.device)
                ops = [dist.P2POp(dist.irecv, got[r if r < self.dst else r - 1], r)
                       for r in range(self.world) if r != self.dst]
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
                # same shape and reduction as the sender's sums: bit-identical iff the bytes are
                mine = torch.stack([torch.stack([self.ring[slot, ri, g].double().sum() for g in range(cnt)])
                                    for ri in range(self.world - 1)])
                ok &= bool(torch.equal(mine, got))
                checked += (self.world - 1) * cnt
            else:
                for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, ps, self.dst)]):
                    w.wait()
        return {"frames": checked, "ok": ok} if self.rank == self.dst else {}
