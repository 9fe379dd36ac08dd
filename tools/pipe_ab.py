"""Interleaved A/B of frame-submission variants on the C3 bench workload (GPU box).

One process builds the scene, the key-frame masks and the working sets once,
then times each variant's steps (60 frames, device events, L2 flushed between
steps) in rounds A B C A B C ..., so slow drifts and one-off stalls hit every
variant alike; prints the median frames/s per variant and its host enqueue
time per frame.

    python tools/pipe_ab.py --rounds 5 --steps 6 py native:3 native:1 native:6
"""
import argparse
import json
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import fdgs_inputs as fi  # noqa: E402
import paper_2503_16422_b200 as fd  # noqa: E402
from paper_2503_16422_b200 import _lib  # noqa: E402

_LIBS = {}


def use_lib(name):
    """Route the binding to tools/variants/libfdgs_<name>.so ('' = the in-tree
    build): every variant library is loaded once, side by side."""
    if name not in _LIBS:
        saved_path, saved = _lib.LIB_PATH, _lib._lib
        _lib._lib = None
        if name:
            _lib.LIB_PATH = f"tools/variants/libfdgs_{name}.so"
            _lib.CHECK_ABI = name != "r01"  # the round-1 library predates ABI version 2
        _LIBS[name] = _lib.lib()
        _lib.LIB_PATH, _lib._lib, _lib.CHECK_ABI = saved_path, saved, True
    _lib._lib = _LIBS[name]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("variants", nargs="+",
                    help="py | native:T | graphs | gnative:T (native with graphs), optionally @depth (native:3@8), "
                         "#lib variant (native:1#sleep200)")
    ap.add_argument("--config", default="c3")
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--frames", type=int, default=60)
    a = ap.parse_args()
    cfg = fi.CONFIGS[a.config]
    scene = fi.make_scene(a.config)
    cams = fi.make_cameras(a.config)
    F, D = cfg["frames"], cfg["keyframe_interval"]
    times = fi.frame_times(F)
    kf = fd.keyframes(F, D)
    use_lib("")
    sc = fd.Scene.from_arrays(scene)
    masks = [fd.keyframe_mask(sc, cams, float(times[k])) for k in kf]
    cs = [fd.camera_struct(c) for c in cams]
    seq = [(f, f // len(cams), f % len(cams)) for f in range(len(cams) * F)]
    wsets = {}
    sync_now = [False]

    def frame(x):
        f, ti, ci = x
        li, ri = fd.bracket(kf, ti)
        key = (li, ri, sync_now[0])
        if key not in wsets:
            wsets[key] = sc.compact(masks[li], masks[ri], sync=sync_now[0])
        return cs[ci], float(times[ti]), None, None, wsets[key]

    flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device="cuda")
    pipes = {}
    use_lib("")
    libs = {}
    syncs = {}
    for v in a.variants:
        spec, _, libname = v.partition("#")
        syncs[v] = spec.endswith("+sync") or libname == "r01"   # r01: no device-count working sets
        spec = spec.replace("+sync", "")
        libs[v] = libname
        use_lib(libname)
        name, _, rest = spec.partition("@")
        depth = int(rest or 6)
        kind, _, thr = name.partition(":")
        pipes[v] = fd.RenderPipeline(sc, cams[0].width, cams[0].height, depth=depth,
                                     graphs=kind in ("graphs", "gnative"), native=kind in ("native", "gnative"),
                                     threads=int(thr or 3))
        if kind == "pyswap":  # experiment: blend streams high priority, front-end streams low
            pp = pipes[v]
            pp.front = [torch.cuda.Stream(priority=0) for _ in range(depth)]
            pp.blend = [torch.cuda.Stream(priority=-1) for _ in range(depth)]
    outs = [pipes[a.variants[0]].renderers[0].new_output() for _ in range(a.frames)]
    res = {v: [] for v in a.variants}
    host = {v: [] for v in a.variants}
    ptr = [0]

    def step(p, timed):
        fr = [seq[(ptr[0] + k) % len(seq)] for k in range(a.frames)]
        ptr[0] += a.frames
        jobs = [frame(x) for x in fr]
        flush.zero_()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        h0 = time.perf_counter()
        p.render_many(jobs, outs)
        h = time.perf_counter() - h0
        e.record()
        e.synchronize()
        return s.elapsed_time(e), h

    for v in a.variants:  # warm every variant
        use_lib(libs[v])
        sync_now[0] = syncs[v]
        for _ in range(2):
            step(pipes[v], False)
    for r in range(a.rounds):
        p0 = ptr[0]
        for v in a.variants:  # every variant renders the same frames in a round
            ptr[0] = p0
            use_lib(libs[v])
            sync_now[0] = syncs[v]
            for _ in range(a.steps):
                ms, h = step(pipes[v], True)
                res[v].append(ms)
                host[v].append(h * 1e3)
    out = {v: {"fps_median": round(a.frames / (statistics.median(res[v]) / 1e3), 1),
               "fps_mean": round(a.frames * len(res[v]) / (sum(res[v]) / 1e3), 1),
               "host_ms_per_frame": round(statistics.median(host[v]) / a.frames, 4)} for v in a.variants}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
