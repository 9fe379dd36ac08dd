"""Small renders for compute-sanitizer (memcheck / racecheck / initcheck):
C1 frames, an overflowing workspace, a working set, the counting blend."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import fdgs_inputs as fi  # noqa: E402
import paper_2503_16422_b200 as fd  # noqa: E402

scene = fi.make_scene("c1")
cams = fi.make_cameras("c1")
sc = fd.Scene.from_arrays(scene)
m = fd.keyframe_mask(sc, cams, 0.3)
r = fd.Renderer(sc, 64, 64)
for t in (0.0, 0.5, 1.0):
    r.render_checked(cams[0], t)
    st = torch.zeros(4, dtype=torch.int64, device="cuda")
    r.render(cams[0], t, m, m, stats=st)
small = fd.Renderer(sc, 64, 64, max_entries=16)
out, s = small.render_checked(cams[0], 0.5)                 # overflow, grow, re-render
ws = sc.compact(m, m, sync=False)
r.render(cams[0], 0.3, scene=ws)
pipe = fd.RenderPipeline(sc, 64, 64, depth=3, native=True, threads=2)
outs = [r.new_output() for _ in range(6)]
pipe.render_many([(cams[0], 0.1 * k, m, m) for k in range(6)], outs)
torch.cuda.synchronize()
print("sanitize ok", s.n_entries)
