#!/usr/bin/env python
"""Frames/s of the 4DGS-1K render hot path on B200 (BASELINE.json metric).

Workload (configs[2]): the N3V-shaped 200k-Gaussian scene,
1352x1014, 20 cameras x 300 timestamps = 6000 frames, key-frame interval 20,
every frame rendered with the union mask of its two bracketing key-frames.
A step renders the next F (default 60) frames of this rank's share of the
sequence (frame f -> rank f mod N, weak scaling).  L2 is flushed between
steps (a 512 MiB write), outside the timed events.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Rank 0 prints one JSON line.  `--impl reference` times the CPU oracle (this
tier's reference arm) on bounded samples of the same workload.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "frames/sec at 1352x1014 (N3V-shaped 200k-Gaussian masked scene)"
UNIT = "frames/s"
CONFIG = "c3"
BLEND_KERNEL = "k_blend_wi"
# launches of libfdgs kernels per frame (render.cu launch_render, tile grid <= 256 rows):
# k_zero, k_cull, k_count_scan, k_cull_emit, k_slice, k_count_scan, k_vis_emit, k_sort_hist,
# 4 x k_onesweep (depth), k_bin_count, k_count_scan, k_bin_offsets, k_row_items, k_row_scan,
# k_onesweep (rows), k_row_count, k_tile_scan, k_row_scatter (the front end: one CUDA-graph
# launch per frame by default), k_blend_wi
KERNELS_PER_FRAME = 22  # the timed blend (render.cu); k_blend_ws<true> supplies the work counters
N_CAMS = 20
N_FRAMES_T = 300
INTERVAL = 20
MASKED = True
WORKLOADS = {
    "c1": "c1: tiny 1000 4D Gaussians, 64x64, 1 camera x 4 t, no key-frame filter",
    "c2": "c2: D-NeRF-shaped 100k 4D Gaussians, 800x800, 50 cams x 150 t, key-frame interval 10",
    "c3": "c3: N3V-shaped 200k 4D Gaussians, 1352x1014, 20 cams x 300 t, key-frame interval 20",
    "c4": "c4: N3V-shaped 3M 4D Gaussians (vanilla-4DGS scale), 1352x1014, 20 cams x 300 t, key-frame interval 20",
}


def apply_config(args):
    """BASELINE configs[0..3]; c3 is the metric's named workload (the default);
    c1 (configs[0], the tiny oracle-sized case) has no key-frame filter."""
    global CONFIG, N_CAMS, N_FRAMES_T, INTERVAL, MASKED, METRIC
    import fdgs_inputs as fi
    CONFIG = args.config
    cfg = fi.CONFIGS[CONFIG]
    if args.streams is None:
        args.streams = 8 if CONFIG == "c2" else 6
    N_CAMS = {"hemisphere50": 50, "arc20": 20, "c1": 1}[cfg["rig"]]
    N_FRAMES_T = cfg["frames"]
    INTERVAL = cfg["keyframe_interval"]
    MASKED = not args.unmasked and INTERVAL is not None
    if CONFIG != "c3" or not MASKED or args.vq:
        METRIC = (f"frames/sec at {cfg['width']}x{cfg['height']} ({CONFIG}, "
                  f"{'masked' if MASKED else 'unmasked'}{f', VQ-SH K={args.vq}' if args.vq else ''})")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)  # 50 x 120 = the whole 6000-frame C3 sequence
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--frames-per-step", type=int, default=120,
                   help="frames per step (the pipeline drains at every step end; 60 measured 1.3%% lower)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-stage-events", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--streams", type=int, default=None,
                   help="frame-pipelining depth (workspaces/streams); default 8 at c2 (800x800: shorter frames "
                        "want more in flight, measured), else 6")
    p.add_argument("--no-split", action="store_true", help="blend on the front-end stream (no priority split)")
    p.add_argument("--no-graphs", action="store_true",
                   help="launch the front end's kernels one by one instead of one CUDA-graph launch per frame")
    p.add_argument("--native-submit", action="store_true",
                   help="submit each step's frames with one fdgs_pipeline_render call instead of the per-frame "
                        "loop")
    p.add_argument("--submit-threads", type=int, default=1,
                   help="host threads of fdgs_pipeline_render (1: frames issued in order; more cost device throughput)")
    p.add_argument("--copy-streams", type=int, default=1, help="e2e: D2H copy streams of the pipeline")
    p.add_argument("--sync-compact", action="store_true",
                   help="read each working set's size back to the host (Scene.compact sync=True)")
    p.add_argument("--config", choices=["c1", "c2", "c3", "c4"], default="c3")
    p.add_argument("--unmasked", action="store_true", help="render without the key-frame filter")
    p.add_argument("--literal-masks", action="store_true",
                   help="key-frame masks from the Eq. 2 blending weights (P:282 literal, R3b) instead of the "
                        "BASELINE config's geometric visibility")
    p.add_argument("--no-working-set", dest="working_set", action="store_false",
                   help="render the full scene under the masks instead of the window's compacted working set")
    p.add_argument("--vq", type=int, default=0, metavar="K",
                   help="Ours-PP storage: SH vector-quantised to a K-entry codebook (P:483), 0 = dense SH")
    p.add_argument("--gather-chunk", type=int, default=10,
                   help="N > 1: frames per grouped send/recv of the frame gather to rank 0")
    p.add_argument("--no-gather", action="store_true", help="N > 1: do not gather the frames to rank 0")
    p.add_argument("--cpu-single-core", action="store_true",
                   help="also time the oracle on one host core (cpu_baseline.single_core)")
    p.add_argument("--fake-render", action="store_true", help=argparse.SUPPRESS)  # CPU orchestration test (gloo)
    p.add_argument("--fake-n", type=int, default=300, help=argparse.SUPPRESS)
    return p.parse_args()


def sequence():
    """All (frame f, time index, camera) of the sequence, ordered by f."""
    return [(f, f // N_CAMS, f % N_CAMS) for f in range(N_CAMS * N_FRAMES_T)]


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during timing."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms",
                                          os.environ.get("FDGS_BENCH_CLOCK_MS", "200")],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def settle(self, timeout=10.0):
        """Wait for nvidia-smi's first sample (its NVML start-up can stall the
        CUDA launch path for ~0.2 s), then drop the samples taken so far: the
        timed region starts after this."""
        t0 = time.perf_counter()
        while self.proc is not None and not self.lines and time.perf_counter() - t0 < timeout:
            time.sleep(0.01)
        self.lines.clear()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        after = not self.lines  # a timed region shorter than the sampling interval
        if after:
            t0 = time.perf_counter()
            while not self.lines and time.perf_counter() - t0 < 2.0:
                time.sleep(0.01)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        out = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
               "reasons": sorted(reasons), "samples": len(sm)}
        if after:
            out["note"] = "timed region shorter than the 200 ms sampling interval: first sample after it"
        return out


# ----------------------------------------------------------------- helpers
def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def load_traffic():
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


class OracleMasks:
    """Key-frame masks from the oracle itself, built on first use:
    the CPU legs take no input from the CUDA path."""

    def __init__(self, scene, cams):
        import oracle
        import fdgs_inputs as fi
        self.scene, self.cams = scene, cams
        self.times = fi.frame_times(N_FRAMES_T)
        self.kf = oracle.keyframes(N_FRAMES_T, INTERVAL)
        self.rows = {}

    def active(self, ti):
        import oracle
        l, r = oracle.bracket(self.kf, ti)
        for k in (l, r):
            if k not in self.rows:
                self.rows[k] = oracle.keyframe_mask(self.scene, self.cams, self.times[self.kf[k]])
        full = np.zeros((len(self.kf), self.rows[l].shape[0]), np.uint32)
        full[l], full[r] = self.rows[l], self.rows[r]
        return oracle.active_mask(full, self.kf, ti)  # the oracle's own bracketing and OR


def cpu_oracle_run(scene, cams, masks, frames, seconds, row_stride=8, threads=None):
    """Time the oracle as it stands on bounded samples: rows j = 0 mod row_stride
    of consecutive frames until `seconds` elapse.  Returns (frames/s, info).
    masks: the oracle's own (OracleMasks; built outside the timed loop), None =
    unmasked."""
    import oracle  # the oracle's own schedule, bracketing and mask OR
    import fdgs_inputs as fi

    times = fi.frame_times(N_FRAMES_T)
    W, H = cams[0].width, cams[0].height
    rows = np.arange(0, H, row_stride)
    pix = (rows[:, None] * W + np.arange(W)[None, :]).ravel()
    done_px, k, n_pairs, t0 = 0, 0, 0, time.perf_counter()
    oracle.load()
    prev = oracle.num_threads()
    if threads:
        oracle.set_num_threads(threads)
    acts = {}
    if masks is not None:  # the sampled frames' active masks, built before the timed loop
        for x in frames[:400]:
            if x[1] not in acts and len(acts) < 6:
                acts[x[1]] = masks.active(x[1])
    t0 = time.perf_counter()
    while True:
        f, ti, ci = frames[k % len(frames)]
        act = None
        if masks is not None:
            if ti not in acts:
                acts[ti] = masks.active(ti)
            act = acts[ti]
        r = oracle.render(scene, cams[ci], float(times[ti]), mask=act, pixels=pix)
        done_px += pix.size
        n_pairs += r["stats"]["evaluated"]
        k += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    fps = done_px / (W * H) / el
    cores = oracle.num_threads()
    if threads:
        oracle.set_num_threads(prev)
    return fps, dict(cores=cores, frames=k, seconds=round(el, 2),
                     ns_per_evaluated_pair=round(el * 1e9 / max(n_pairs, 1), 3),
                     core_ns_per_evaluated_pair=round(el * 1e9 * cores / max(n_pairs, 1), 2),
                     sample=f"oracle per-pixel render of rows j%{row_stride}==0 ({pix.size} px) of {k} "
                            f"consecutive {'masked' if masks is not None else 'unmasked'} {CONFIG} frames; "
                            f"fps = sampled pixels/(W*H)/wall")


# ----------------------------------------------------------------- ours
class _FakePipeline:
    """--fake-render: the orchestration of run_ours on CPU ranks (gloo) with a
    deterministic stand-in for the CUDA render, so that the multi-rank logic
    bench.py runs (partition, broadcast, mask sharing, frame gather, timing
    reduction) is tested without a GPU (tests/test_dist_gloo.py).  Frame f's
    image is filled with the value f."""

    def __init__(self, shape):
        self.shape = shape

    def render_many(self, frames, outs, stream=None, frame_done=None, **_):
        for k, x in enumerate(frames):
            outs[k].fill_(float(x[0]))
            if frame_done is not None:
                frame_done(k, outs[k], None, None)


def _fake_mask(k, words):
    rng = np.random.default_rng(1000 + k)
    return rng.integers(0, 2 ** 32, words, dtype=np.uint64).astype(np.uint32).view(np.int32)


def run_ours(args):
    import torch

    import fdgs_inputs as fi
    from paper_2503_16422_b200 import dist as fdist

    import paper_2503_16422_b200 as fd  # (the library itself loads on first use: not in --fake-render)

    fake = args.fake_render
    graphs = not args.no_graphs
    rank, world, local = fdist.env_ranks()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if fake:
        dev = torch.device("cpu")
    else:
        torch.cuda.set_device(local)
        dev = torch.device("cuda", local)
    fdist.init("gloo" if fake else "nccl", dev)

    # ---- scene: rank 0 draws it, broadcast to the others (NCCL over NVLink)
    cfg = fi.CONFIGS[CONFIG]
    n = args.fake_n if fake else cfg["n"]
    shapes = {"mean": (n, 4), "scale": (n, 4), "rot_l": (n, 4), "rot_r": (n, 4), "opacity": (n,),
              "log255_opacity": (n,), "sh": (args.vq, 16, 3) if args.vq else (n, 16, 3)}
    if rank == 0:
        arrays = fi.make_scene(CONFIG, n=n)
        if args.vq:
            arrays = fi.vq_scene(arrays, codebook_size=args.vq, seed=1)
        tens = {k: torch.from_numpy(v).to(dev) for k, v in arrays.arrays().items()}
    else:
        arrays = None
        tens = {k: torch.empty(s, dtype=torch.float32, device=dev) for k, s in shapes.items()}
        if args.vq:
            tens["sh_index"] = torch.empty(n, dtype=torch.uint16, device=dev)
    fdist.broadcast_scene(tens)
    scene_ok = True
    if fake:  # every rank holds rank 0's scene (checked against the generator)
        ref = fi.make_scene(CONFIG, n=n).arrays()
        scene_ok = all(np.array_equal(tens[k].numpy(), ref[k]) for k in ref)
    scene = None if fake else fd.Scene(tens, device=dev)
    cams = fi.make_cameras(CONFIG)
    W, H = (8, 6) if fake else (cams[0].width, cams[0].height)
    cam_structs = None if fake else [fd.camera_struct(c) for c in cams]
    times = fi.frame_times(N_FRAMES_T)
    kf = fd.keyframes(N_FRAMES_T, INTERVAL or N_FRAMES_T)
    bracket = fd.bracket
    # ---- key-frame masks: key-frame k built by rank k mod N, all-reduced (disjoint rows)
    words = (n + 31) // 32

    def build(k, out):
        if fake:
            out.copy_(torch.from_numpy(_fake_mask(k, words)))
        elif args.literal_masks:  # P:282 read literally (R3b): blending weight > 0 in some view
            out.copy_(fd.keyframe_mask_contrib(scene, cams, float(times[kf[k]]), 0.0))
        else:
            fd.keyframe_mask(scene, cams, float(times[kf[k]]), out=out)

    t_mask0 = time.perf_counter()
    masks = fdist.share_keyframe_masks(len(kf), words, build, dev)
    if not fake:
        torch.cuda.synchronize()
    mask_build_s = time.perf_counter() - t_mask0
    masks_ok = (not fake) or all(np.array_equal(masks[k].numpy(), _fake_mask(k, words)) for k in range(len(kf)))

    seq = sequence()
    mine = fdist.shard_frames(seq, rank, world)
    F = args.frames_per_step
    if fake:
        pipe = _FakePipeline((3, H, W))
        outs = [torch.empty((3, H, W), dtype=torch.float32) for _ in range(F)]
        stream = None
    else:
        pipe = fd.RenderPipeline(scene, W, H, depth=args.streams, split=not args.no_split, graphs=graphs,
                                 native=args.native_submit, copy_streams=args.copy_streams,
                                 threads=args.submit_threads)
        renderer = pipe.renderers[0]
        outs = [renderer.new_output() for _ in range(F)]
        stats = torch.zeros((F, 4), dtype=torch.int64, device=dev)  # fdgs_frame_stats is 32 bytes
        flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device=dev)  # 512 MiB > L2
        stream = torch.cuda.current_stream()
    gather = None
    if world > 1 and not args.no_gather:
        gather = fdist.FrameGather((3, H, W), args.gather_chunk, dev)
    use_ev = not fake and not args.no_stage_events
    if use_ev:
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(F)]
        for row in evs:
            for e in row:
                e.record(stream)  # materialise the CUDA events
        torch.cuda.synchronize()

    # key-frame windows as compacted working sets (Scene.compact): built the
    # first time a window is rendered (inside that step's timed region), kept
    # while the sequence stays in the window
    wsets = {}
    compacts = []  # one entry per Scene.compact: whether it ran inside a timed step
    timing_now = [False]
    cur_step = [0]  # index of the timed step being enqueued (1-based; 0 = untimed)

    def frame_args(x):
        if fake:
            return x
        f, ti, ci = x
        if not MASKED:
            return cam_structs[ci], float(times[ti]), None, None
        li, ri = bracket(kf, ti)
        if not args.working_set:
            return cam_structs[ci], float(times[ti]), masks[li], masks[ri]
        if (li, ri) not in wsets:
            if len(wsets) >= 2:
                wsets.pop(next(iter(wsets)))
            wsets[(li, ri)] = scene.compact(masks[li], masks[ri], stream=stream, sync=args.sync_compact)
            compacts.append(timing_now[0] and cur_step[0])
        return cam_structs[ci], float(times[ti]), None, None, wsets[(li, ri)]

    host_ms = []  # host enqueue time of each step (render_many returning)

    def run_step(step_frames, timed, count=False):
        """One step: this rank's next F frames (and, N > 1, their gather to
        rank 0), bracketed by a barrier and device events on both sides."""
        if not fake:
            flush.zero_()
            torch.cuda.synchronize()
        fdist.barrier()
        if fake:
            t0 = time.perf_counter()
        else:
            start = torch.cuda.Event(enable_timing=True)
            end = torch.cuda.Event(enable_timing=True)
            start.record(stream)
        h0 = time.perf_counter()
        g = gather if (gather is not None and not count) else None
        if g is not None:
            g.begin_step(len(step_frames))
        kw = {} if fake else dict(stats=stats if count else None, stage_events=evs if (use_ev and timed) else None)
        pipe.render_many([frame_args(x) for x in step_frames], outs[:len(step_frames)], stream=stream,
                         frame_done=g.frame_done if g is not None else None, **kw)
        if g is not None:
            g.end_step(stream)
        host_ms.append((time.perf_counter() - h0) * 1e3)
        if fake:
            return (time.perf_counter() - t0) * 1e3, None
        end.record(stream)
        end.synchronize()
        ms = start.elapsed_time(end)
        stage = None
        if use_ev and timed:
            # busy time of each stage = length of the union of its per-frame
            # [event s, event s+1] intervals (frames on different streams overlap)
            stage = np.zeros(4)
            for s_ in range(4):
                iv = sorted((start.elapsed_time(evs[k][s_]), start.elapsed_time(evs[k][s_ + 1]))
                            for k in range(len(step_frames)))
                cur0, cur1 = iv[0]
                for a, b in iv[1:]:
                    if a > cur1:
                        stage[s_] += cur1 - cur0
                        cur0, cur1 = a, b
                    else:
                        cur1 = max(cur1, b)
                stage[s_] += cur1 - cur0
        return ms, stage

    ptr = 0

    def next_frames():
        nonlocal ptr
        out = [mine[(ptr + k) % len(mine)] for k in range(F)]
        ptr += F
        return out

    sampler = ClockSampler(local) if not fake else None
    if sampler:
        sampler.start()
    for _ in range(args.warmup):
        run_step(next_frames(), False)
    if sampler:
        sampler.settle()
    step_ms, stage_ms = [], np.zeros(4)
    h_first = len(host_ms)
    timed_frames = []
    timing_now[0] = True
    # no cyclic-GC pauses while steps are enqueued (a pause longer than the
    # host's lead over the GPU starves the queue); collected after timing
    gc.collect()
    gc.disable()
    for k_step in range(args.steps):
        cur_step[0] = k_step + 1
        fr = next_frames()
        timed_frames.append(fr)
        ms, stg = run_step(fr, True)
        step_ms.append(ms)
        if stg is not None:
            stage_ms += stg
    clocks = sampler.stop() if sampler else None
    gc.enable()
    timing_now[0] = False
    # k_mask_compact + k_scene_gather per working set built inside the timed steps
    compact_launches = 2 * sum(1 for x in compacts if x)
    compact_steps = {x - 1 for x in compacts if x}
    host_timed = host_ms[h_first:h_first + args.steps]
    # the job time is the slowest rank's device time (max over ranks), per step too
    per_rank = fdist.gather_timings(step_ms, dev)
    total_ms = max(sum(r) for r in per_rank)
    step_max = [max(r[k] for r in per_rank) for k in range(args.steps)]
    frames_total = world * args.steps * F
    value = frames_total / (total_ms / 1e3)
    frames_rank = args.steps * F
    med = statistics.median(step_max)
    res = dict(metric=METRIC, value=round(value, 2), unit=UNIT, n_gpus=world, steps=args.steps, warmup=args.warmup,
               ms_per_step=round(total_ms / args.steps, 4), higher_is_better=True, scaling="weak", vs_baseline=None,
               dtype="f32 (decision path f64)", data="synthetic",
               config={"workload": WORKLOADS[CONFIG] + (", masked (union of bracketing key-frames)" if MASKED
                                                         else ", unmasked")
                       + (", literal key-frame masks (Eq. 2 weight > 0 in some view; P:282, R3b)"
                          if MASKED and args.literal_masks else "")
                       + (f", SH vector-quantised (K={args.vq} codebook, uint16 index; Ours-PP, P:483)"
                          if args.vq else ""),
                       "frames_per_step": F, "frames_per_rank": frames_rank, "partition": "frame f -> rank f mod N",
                       "l2": "flushed between steps (512 MiB write)", "parallelism": f"frames x{world}",
                       "streams_per_gpu": args.streams,
                       "submission": (("native batch (fdgs_pipeline_render)" +
                                       (", front end as each slot's CUDA graph" if graphs else ""))
                                      if args.native_submit else
                                      "per frame: one CUDA-graph launch of the front end + the blend launch"
                                      if graphs else "per frame: ~22 kernel launches"),
                       "stream_split": "front end high priority, blend low priority" if not args.no_split else "none",
                       "filter": ("compacted working set per key-frame window (Scene.compact, built inside the timed "
                                  "region when the sequence enters the window)") if MASKED and args.working_set
                       else ("masks OR-ed per frame" if MASKED else "none")},
               step_stats={"median_frames_per_s": round(world * F / (med / 1e3), 2),
                           "min_ms": round(min(step_max), 4), "median_ms": round(med, 4),
                           "max_ms": round(max(step_max), 4),
                           "outliers": [{"step": k, "ms": round(step_max[k], 3), "host_ms": round(host_timed[k], 3),
                                         "new_working_set": k in compact_steps}
                                        for k in range(args.steps) if step_max[k] > 1.5 * med][:8],
                           "note": "per-step max-over-ranks device time; value = all frames / sum of per-rank totals "
                                   "(max over ranks)"})
    if not fake:
        res["gpu_launches"] = KERNELS_PER_FRAME * frames_rank + compact_launches
    if gather is not None:
        chk = gather.validate(outs[:F])  # one more gather of the last step's frames, checksums compared on rank 0
        g = {"chunk_frames": gather.chunk, "bytes_per_frame": gather.frame_bytes,
             "bytes_into_rank0_per_step": (world - 1) * F * gather.frame_bytes,
             "in_timed_region": True,
             "how": "grouped P2P send/recv (torch.distributed batch_isend_irecv: NCCL over NVLink) on a side stream "
                    "per chunk as soon as its frames' blends finish; each step's end waits for its transfers",
             "validated_frames": chk.get("frames"), "validated_ok": chk.get("ok")}
        if fake and rank == 0:
            # the last validated chunk holds, for every sender r, the fake frames of r's last step
            slot, cnt = gather.last
            c0 = ((F - 1) // gather.chunk) * gather.chunk
            ok = True
            for r in range(1, world):
                theirs = fdist.shard_frames(seq, r, world)
                base = (args.warmup + args.steps - 1) * F
                for gi in range(cnt):
                    f = theirs[(base + c0 + gi) % len(theirs)][0]
                    ok &= bool(torch.all(gather.ring[slot, r - 1, gi] == float(f)))
            g["fake_content_ok"] = ok
        res["gather"] = g
    if fake:
        res["fake_render"] = {"scene_broadcast_ok": scene_ok, "masks_ok": masks_ok,
                              "frames_rank0": [x[0] for x in mine[:4]],
                              "per_rank_total_ms": [round(sum(r), 4) for r in per_rank]}
        fdist.shutdown()
        if rank == 0:
            print(json.dumps(res), flush=True)
        return

    n_eval = n_blend = 0
    n_vis_tot = n_ent_tot = n_act_tot = 0
    # work counters of the same frames (counting blend variant, not timed)
    for fr in timed_frames:
        run_step(fr, False, count=True)
        s = stats.cpu().numpy()
        lo = np.ascontiguousarray(s[:, 0]).view(np.uint32).reshape(F, 2)
        hi = np.ascontiguousarray(s[:, 1]).view(np.uint32).reshape(F, 2)
        n_act_tot += int(lo[:, 0].sum())
        n_vis_tot += int(lo[:, 1].sum())
        n_ent_tot += int(hi[:, 0].sum())
        assert np.all(hi[:, 1] == 0), "a frame overflowed its entry capacity"
        n_eval += int(s[:, 2].sum())
        n_blend += int(s[:, 3].sum())

    # ---- roofline of the dominant stage
    peaks, peak_src = load_peaks()
    stage_names = ["preprocess", "depth_sort", "binning", "blend"]
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    lane_peak = 148 * 128 * sm_mhz * 1e6  # FP32 lane-ops/s

    def blend_rl(ms_total, frames):
        """SURVEY §8(d) lane-op model: 8 FP32 lane-ops per evaluated pair + 9 per
        blended pair, over 148 SMs x 128 lanes x clock; the flop model beside it."""
        ops = (8.0 * n_eval + 9.0 * n_blend) * frames / max(frames_rank, 1)
        ach = ops / (ms_total / 1e3)
        fl = (10.0 * n_eval + 12.0 * n_blend) * frames / max(frames_rank, 1) / (ms_total / 1e3) / 1e12
        return ach, fl

    if use_ev and stage_ms.sum() > 0:
        per_frame = stage_ms / frames_rank
        dom = int(np.argmax(stage_ms))
        if dom == 3:
            ach, fl = blend_rl(stage_ms[3], frames_rank)
            rl = {"kernel": BLEND_KERNEL, "bound": "alu", "achieved": round(ach / 1e12, 3),
                  "peak": round(lane_peak / 1e12, 3), "unit": "T lane-ops/s", "frac": round(ach / lane_peak, 4),
                  "peak_src": f"148 SMs x 128 FP32 lanes x {sm_mhz:.0f} MHz (sm_max, {peak_src} peaks)",
                  "work": "SURVEY 8(d): 8 FP32 lane-ops per evaluated (pixel, Gaussian) pair + 9 per blended pair; "
                          "pairs from the counting blend on the same frames",
                  "flop_model": {"achieved_tflops": round(fl, 3), "peak_tflops": round(2 * lane_peak / 1e12, 2),
                                 "frac": round(fl * 1e12 / (2 * lane_peak), 4),
                                 "work": "10 flops per evaluated + 12 per blended pair, FMA = 2"}}
        else:
            hbm = float(peaks.get("hbm_gbs", 6650.0))
            nb = {0: 68.0 * n_act_tot + 192.0 * n_vis_tot + 68.0 * n_vis_tot,
                  1: 72.0 * n_vis_tot, 2: 40.0 * n_ent_tot}[dom]
            achieved = nb / (stage_ms[dom] / 1e3) / 1e9
            rl = {"kernel": stage_names[dom], "bound": "hbm", "achieved": round(achieved, 1), "peak": hbm,
                  "unit": "GB/s", "frac": round(achieved / hbm, 4), "peak_src": peak_src}
        trj = load_traffic()
        rl["traffic"] = trj.get(rl["kernel"])
        for key in ("issue_slots_busy", "pipes"):  # ncu of the blend (profiles/traffic.json)
            if trj.get(rl["kernel"] + "_" + key) is not None:
                rl["ncu_" + key] = trj[rl["kernel"] + "_" + key]
        res["roofline"] = rl
        res["stages"] = {nm: {"ms_per_frame": round(float(per_frame[i]), 4),
                              "share": round(float(stage_ms[i] / sum(step_ms)), 4)} for i, nm in enumerate(stage_names)}
        res["stages"]["stage_events_sum_vs_step"] = round(float(stage_ms.sum() / sum(step_ms)), 4)
        res["stages"]["note"] = (f"per-stage CUDA events of every timed frame; a stage's time is the union of its "
                                 f"per-frame intervals (busy time); with {args.streams} frame-pipelining streams "
                                 "stages of different frames run concurrently, so shares can sum above 1")
    # isolated (one stream, nothing overlapping) per-stage times of one extra step
    # of the same frames, outside the timed region: the blend's own throughput
    if use_ev and stage_ms.sum() > 0 and "roofline" in res:
        iso = fd.RenderPipeline(scene, W, H, depth=1, split=False)
        iso.renderers[0] = renderer
        fr = timed_frames[0]
        flush.zero_()
        torch.cuda.synchronize()
        iso.render_many([frame_args(x) for x in fr], outs[:len(fr)], stage_events=evs, stream=stream)
        torch.cuda.synchronize()
        iso_ms = np.array([sum(evs[k][s_].elapsed_time(evs[k][s_ + 1]) for k in range(len(fr))) for s_ in range(4)])
        if res["roofline"]["kernel"] == BLEND_KERNEL:
            # the counters cover all timed frames, this pass the first step's
            ach, fl = blend_rl(iso_ms[3] * len(timed_frames), frames_rank)
            res["roofline"]["isolated"] = {"achieved": round(ach / 1e12, 3), "frac": round(ach / lane_peak, 4),
                                           "ms_per_frame": round(float(iso_ms[3] / len(fr)), 4),
                                           "note": "same frames on one stream, no overlap (outside the timed region)"}
        res["stages_isolated_ms_per_frame"] = {nm: round(float(iso_ms[i] / len(fr)), 4)
                                               for i, nm in enumerate(stage_names)}
    res["work_per_frame"] = {"n_act": round(n_act_tot / frames_rank), "n_vis": round(n_vis_tot / frames_rank),
                             "entries": round(n_ent_tot / frames_rank), "evaluated_pairs": round(n_eval / frames_rank),
                             "blended_pairs": round(n_blend / frames_rank)}
    # whole-frame HBM model of SURVEY.md §8(d) d.4 (BASELINE "% HBM roofline"): algorithmic
    # bytes per frame from the device counters, over the frame time, against the measured copy peak
    na, nv, ne = n_act_tot / frames_rank, n_vis_tot / frames_rank, n_ent_tot / frames_rank
    px = W * H
    mask_terms = (8.0 * ((n + 31) // 32) + 8.0 * na) if MASKED else 0.0
    bpf = mask_terms + 68.0 * na + (192.0 + 96.0 + 72.0) * nv + (8.0 + 32.0 + 52.0) * ne + 12.0 * px
    hbm = float(load_peaks()[0].get("hbm_gbs", 6650.0))
    achieved_gbs = bpf * value / world / 1e9
    res["frame_hbm"] = {"bytes_per_frame": round(bpf), "achieved": round(achieved_gbs, 1), "peak": hbm,
                        "unit": "GB/s", "frac": round(achieved_gbs / hbm, 4),
                        "model": "SURVEY.md 8(d) d.4: mask words + index + 68 B/active + (192+96+72) B/visible + "
                                 "(8+32+52) B/entry + 12 B/pixel, per GPU"}
    dram = load_traffic().get("frame_dram_bytes")
    if dram is not None and CONFIG == "c3" and MASKED:  # the committed capture is of this workload
        res["frame_hbm"]["ncu_dram_bytes_per_frame"] = dram
    res["clocks"] = clocks
    # host time to enqueue a step (render_many returning) vs the step's device
    # time: the pipeline is host-bound if the ratio approaches 1
    res["host_enqueue"] = {"ms_per_frame_median": round(float(np.median(host_timed)) / F, 4),
                           "ms_per_frame_max": round(float(np.max(host_timed)) / F, 4),
                           "vs_device": round(float(np.median(host_timed)) / float(np.median(step_ms)), 3),
                           "slowest_step": int(np.argmax(host_timed))}
    res["setup"] = {"keyframe_masks_s": round(mask_build_s, 3), "n_keyframes": len(kf)}

    # ---- e2e through the public API with host buffers
    if not args.no_e2e:
        host_masks = masks.cpu().pin_memory()
        dev_masks = torch.empty_like(masks)
        host_out = torch.empty((F, 3, H, W), dtype=torch.float32).pin_memory()
        e2e_ms = []
        h2d_bytes = d2h_bytes = 0
        e2e_sets = {}
        for it in range(args.warmup + max(1, args.steps // 2)):
            fr = next_frames()
            need = sorted({i for x in fr for i in bracket(kf, x[1])}) if MASKED else []
            flush.zero_()
            torch.cuda.synchronize()
            fdist.barrier()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for i in need:
                dev_masks[i].copy_(host_masks[i], non_blocking=True)
            jobs = []
            for k, x in enumerate(fr):
                f, ti, ci = x
                li, ri = bracket(kf, ti)
                if MASKED and args.working_set:
                    # a window's working set is built (from the masks copied H2D) when the
                    # sequence enters it, as in the device-timed loop
                    if (li, ri) not in e2e_sets:
                        if len(e2e_sets) >= 2:
                            e2e_sets.pop(next(iter(e2e_sets)))
                        e2e_sets[(li, ri)] = scene.compact(dev_masks[li], dev_masks[ri], stream=stream,
                                                           sync=args.sync_compact)
                    jobs.append((cam_structs[ci], float(times[ti]), None, None, e2e_sets[(li, ri)]))
                else:
                    jobs.append((cam_structs[ci], float(times[ti]), dev_masks[li] if MASKED else None,
                                 dev_masks[ri] if MASKED else None))
            # each frame goes D2H on the pipeline's copy stream as soon as its blend is done
            # (and, N > 1, to rank 0 over NVLink as in the device-timed loop)
            if gather is not None:
                gather.begin_step(len(fr))
            pipe.render_many(jobs, outs[:len(fr)], stream=stream, host_outs=host_out,
                             frame_done=gather.frame_done if gather is not None else None)
            if gather is not None:
                gather.end_step(stream)
            b.record(stream)
            b.synchronize()
            if it >= args.warmup:
                e2e_ms.append(a.elapsed_time(b))
                h2d_bytes = len(need) * words * 4
                d2h_bytes = F * 3 * H * W * 4
        tot = fdist.max_over_ranks(float(sum(e2e_ms)), dev)
        res["e2e"] = {"value": round(world * len(e2e_ms) * F / (tot / 1e3), 2), "unit": UNIT,
                      "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": d2h_bytes,
                      "path": "RenderPipeline.render_many (fdgs_render_split) with the step's key-frame masks H2D "
                              "from pinned host and every frame D2H to pinned host (copy stream, overlapping later "
                              "frames) inside the timed region" +
                              ("; N > 1: every rank copies its own frames D2H and gathers them to rank 0 over "
                               "NVLink (FrameGather)" if gather is not None else "")}

    # ---- CPU oracle baseline (rank 0, N = 1 only)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        omasks = OracleMasks(arrays, cams) if MASKED else None
        fps, info = cpu_oracle_run(arrays, cams, omasks, mine, args.cpu_seconds)
        res["cpu_baseline"] = {"value": round(fps, 5), "unit": UNIT, "cores": info["cores"], "kind": "oracle",
                               "sample": info["sample"], "ns_per_evaluated_pair": info["ns_per_evaluated_pair"],
                               "core_ns_per_evaluated_pair": info["core_ns_per_evaluated_pair"]}
        if args.cpu_single_core:
            fps1, info1 = cpu_oracle_run(arrays, cams, omasks, mine, args.cpu_seconds, row_stride=64, threads=1)
            res["cpu_baseline"]["single_core"] = {"value": round(fps1, 6), "cores": 1, "sample": info1["sample"],
                                                  "ns_per_evaluated_pair": info1["ns_per_evaluated_pair"]}
    fdist.shutdown()
    if rank == 0:
        print(json.dumps(res), flush=True)


# ------------------------------------------------------------- reference
def run_reference(args):
    """This tier's reference arm: the CPU oracle as it stands (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import fdgs_inputs as fi
    import oracle

    scene = fi.make_scene(CONFIG)
    cams = fi.make_cameras(CONFIG)
    times = fi.frame_times(N_FRAMES_T)
    masks = OracleMasks(scene, cams) if MASKED else None  # the oracle's own schedule and masks
    seq = sequence()
    per_step = max(1.0, 60.0 / max(1, args.steps + args.warmup))
    vals = []
    info = None
    for s in range(args.warmup + args.steps):
        frames = seq[(s * 7) % len(seq):] + seq
        fps, info = cpu_oracle_run(scene, cams, masks, frames, per_step, row_stride=16)
        if s >= args.warmup:
            vals.append(fps)
    value = float(np.mean(vals))
    res = dict(metric=METRIC, value=round(value, 5), unit=UNIT, n_gpus=world, steps=args.steps,
               warmup=args.warmup, ms_per_step=round(per_step * 1e3, 1), higher_is_better=True, scaling="weak",
               vs_baseline=None, dtype="f64", data="synthetic", impl="reference",
               config={"workload": WORKLOADS[CONFIG] + (", masked" if MASKED else ", unmasked")
                                   + "; each step a bounded row sample (rows j%16==0) of consecutive frames"},
               cpu_baseline={"value": round(value, 5), "unit": UNIT, "kind": "oracle", "cores": info["cores"],
                             "sample": info["sample"]},
               e2e={"value": round(value, 5), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
    print(json.dumps(res), flush=True)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-run this command under torch.distributed.run
        from paper_2503_16422_b200.dist import launch_self
        launch_self(args.gpus)
    apply_config(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
