"""Whole-GPU counters of the pipelined render (all kernels of 60 frames
running concurrently on the pipeline's streams) as one ncu range:

    ncu --replay-mode app-range --metrics ... python tools/range_prof.py --config c4

cudaProfilerStart/Stop bracket one step of 60 frames (after warm-up), so the
metrics are GPU-wide utilisation while frames overlap -- what a per-kernel
(serialised) capture cannot show."""
import argparse
import sys

import torch

sys.path.insert(0, ".")
import fdgs_inputs as fi  # noqa: E402
import paper_2503_16422_b200 as fd  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--frames", type=int, default=60)
    ap.add_argument("--no-graphs", action="store_true")
    ap.add_argument("--noblend", action="store_true", help="(unused placeholder for variant libs)")
    a = ap.parse_args()
    cfg = fi.CONFIGS[a.config]
    cams = fi.make_cameras(a.config)
    sc = fd.Scene.from_arrays(fi.make_scene(a.config))
    F, D = cfg["frames"], cfg["keyframe_interval"]
    times = fi.frame_times(F)
    kf = fd.keyframes(F, D)
    masks = {}
    li, ri = fd.bracket(kf, 150)
    for k in (li, ri):
        masks[k] = fd.keyframe_mask(sc, cams, float(times[kf[k]]))
    ws = sc.compact(masks[li], masks[ri], sync=False)
    pipe = fd.RenderPipeline(sc, cams[0].width, cams[0].height, depth=6, graphs=not a.no_graphs)
    jobs = []
    for k in range(a.frames):
        ti = kf[li] + (k // len(cams)) % max(1, kf[ri] - kf[li])
        jobs.append((cams[k % len(cams)], float(times[ti]), None, None, ws))
    outs = [pipe.renderers[0].new_output() for _ in jobs]
    for _ in range(3):
        pipe.render_many(jobs, outs)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    pipe.render_many(jobs, outs)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("ok")


if __name__ == "__main__":
    main()
