"""Host enqueue cost and device throughput of RenderPipeline with and without
CUDA graphs (C3 frames of one key-frame window; GPU box)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import fdgs_inputs as fi  # noqa: E402
import paper_2503_16422_b200 as fd  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = fi.CONFIGS[name]
scene = fi.make_scene(name)
cams = fi.make_cameras(name)
sc = fd.Scene.from_arrays(scene)
F = cfg["frames"]
times = fi.frame_times(F)
kf = fd.keyframes(F, cfg["keyframe_interval"])
masks = [fd.keyframe_mask(sc, cams, float(times[k])) for k in kf]
cs = [fd.camera_struct(c) for c in cams]
frames = []
for f in range(1000, 1060):
    ti, ci = divmod(f, len(cams))
    l, r = fd.bracket(kf, ti)
    frames.append((cs[ci], float(times[ti]), masks[l], masks[r]))
for graphs in (False, True, False, True):
    pipe = fd.RenderPipeline(sc, cams[0].width, cams[0].height, depth=4, graphs=graphs)
    outs = [pipe.renderers[0].new_output() for _ in frames]
    for _ in range(3):
        pipe.render_many(frames, outs)
    torch.cuda.synchronize()
    best = (1e9, 1e9)
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record()
        pipe.render_many(frames, outs)
        b.record()
        t1 = time.perf_counter()
        b.synchronize()
        best = min(best, (a.elapsed_time(b), 1e3 * (t1 - t0)))
    print(f"{name} graphs={graphs}: device {best[0]:.2f} ms = {len(frames) / best[0] * 1e3:.0f} frames/s, "
          f"host enqueue {best[1]:.2f} ms ({best[1] / len(frames) * 1e3:.1f} us/frame)")
