"""A/B timing of the render stages on fixed C3 masked frames (GPU box).

Renders `--frames` frames spread over the C3 sequence, one stream, with the
5 stage events of fdgs_render_timed; prints one JSON line with the median
per-stage ms per frame (over `--reps` passes) and a checksum of the images,
so variants selected by environment variables can be compared run by run.
"""
import argparse
import hashlib
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import os  # noqa: E402

import fdgs_inputs as fi  # noqa: E402
import paper_2503_16422_b200 as fd  # noqa: E402
from paper_2503_16422_b200 import _lib  # noqa: E402

if os.environ.get("AB_LIB"):  # a variant build of libfdgs.so (tools/ab_build.sh)
    _lib.LIB_PATH = os.path.abspath(os.environ["AB_LIB"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--frames", type=int, default=40)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--unmasked", action="store_true")
    a = ap.parse_args()
    scene = fi.make_scene(a.config)
    cams = fi.make_cameras(a.config)
    frames = {"c3": 300, "c4": 300, "c2": 150}[a.config]
    interval = {"c3": 20, "c4": 20, "c2": 10}[a.config]
    times = fi.frame_times(frames)
    sc = fd.Scene.from_arrays(scene)
    kf = fd.keyframes(frames, interval)
    masks = [fd.keyframe_mask(sc, cams, float(times[k])) for k in kf]
    r = fd.Renderer(sc, cams[0].width, cams[0].height)
    sel = [(i * 7919) % (frames * len(cams)) for i in range(a.frames)]
    jobs = []
    for f in sel:
        ti, ci = divmod(f, len(cams))
        lo, hi = fd.bracket(kf, ti)
        ml = None if a.unmasked else masks[lo]
        mr = None if a.unmasked else masks[hi]
        jobs.append((cams[ci], float(times[ti]), ml, mr))
    outs = [r.new_output() for _ in jobs]
    for cam, t, ml, mr in jobs[:4]:
        r.render_checked(cam, t, ml, mr)
    names = ["preprocess", "depth_sort", "binning", "blend"]
    per = {k: [] for k in names}
    for _ in range(a.reps):
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in jobs]
        for ev in evs:
            for e in ev:
                e.record()  # materialise the CUDA events before passing their handles
        for (cam, t, ml, mr), o, ev in zip(jobs, outs, evs):
            r.render(cam, t, ml, mr, out=o, stage_events=ev)
        torch.cuda.synchronize()
        for k, nm in enumerate(names):
            per[nm].append(sum(ev[k].elapsed_time(ev[k + 1]) for ev in evs) / len(jobs))
    h = hashlib.sha256()
    for o in outs:
        h.update(o.cpu().numpy().tobytes())
    res = {k: round(float(np.median(v)), 5) for k, v in per.items()}
    res["total"] = round(sum(res.values()), 5)
    res["checksum"] = h.hexdigest()[:16]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
