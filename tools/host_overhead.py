"""Host-side enqueue cost of RenderPipeline.render_many vs the device time (GPU box)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import fdgs_inputs as fi  # noqa: E402
import paper_2503_16422_b200 as fd  # noqa: E402

scene = fi.make_scene("c3")
cams = fi.make_cameras("c3")
sc = fd.Scene.from_arrays(scene)
times = fi.frame_times(300)
kf = fd.keyframes(300, 20)
masks = [fd.keyframe_mask(sc, cams, float(times[k])) for k in kf]
pipe = fd.RenderPipeline(sc, 1352, 1014, depth=4)
F = 60
outs = [pipe.renderers[0].new_output() for _ in range(F)]
cs = [fd.camera_struct(c) for c in cams]
frames = []
for f in range(F):
    ti, ci = divmod(1000 + f, 20)
    l, r = fd.bracket(kf, ti)
    frames.append((cs[ci], float(times[ti]), masks[l], masks[r]))
for _ in range(3):
    pipe.render_many(frames, outs)
torch.cuda.synchronize()
for rep in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    pipe.render_many(frames, outs)
    b.record()
    t1 = time.perf_counter()
    b.synchronize()
    t2 = time.perf_counter()
    print(f"enqueue {1e3 * (t1 - t0):.2f} ms, device {a.elapsed_time(b):.2f} ms, wall {1e3 * (t2 - t0):.2f} ms")
