"""Host enqueue cost per frame, split into the C call and the Python around it (GPU box)."""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, ".")
import fdgs_inputs as fi  # noqa: E402
import paper_2503_16422_b200 as fd  # noqa: E402
from paper_2503_16422_b200 import api  # noqa: E402
from paper_2503_16422_b200._lib import lib  # noqa: E402

scene = fi.make_scene("c3")
cams = fi.make_cameras("c3")
sc = fd.Scene.from_arrays(scene)
times = fi.frame_times(300)
pipe = fd.RenderPipeline(sc, 1352, 1014, depth=6)
F = 60
outs = [pipe.renderers[0].new_output() for _ in range(F)]
cs = [fd.camera_struct(c) for c in cams]
frames = [(cs[f % 20], float(times[f // 20 + 100]), None, None) for f in range(F)]
for _ in range(3):
    pipe.render_many(frames, outs)
torch.cuda.synchronize()
res = {}
for rep in range(3):
    t0 = time.perf_counter()
    pipe.render_many(frames, outs)
    res.setdefault("render_many_ms_per_frame", []).append((time.perf_counter() - t0) * 1e3 / F)
    torch.cuda.synchronize()
# raw C calls, arguments prebuilt, no Python event objects
r = pipe.renderers[0]
st = torch.cuda.Stream()
bs = torch.cuda.Stream()
ev = torch.cuda.Event()
ev.record(st)
args = []
for f in range(F):
    fr = frames[f]
    args.append((C.byref(sc.struct), None, None, C.byref(fr[0]), fr[1], api._ptr(outs[f]), None, api._ptr(r.ws),
                 r.ws_bytes, r.max_entries, None, C.c_void_p(st.cuda_stream), C.c_void_p(bs.cuda_stream),
                 C.c_void_p(ev.cuda_event), None))
fn = lib().fdgs_render_split
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for a in args:
        fn(*a)
    res.setdefault("raw_c_ms_per_frame", []).append((time.perf_counter() - t0) * 1e3 / F)
torch.cuda.synchronize()
print({k: [round(x, 4) for x in v] for k, v in res.items()})
