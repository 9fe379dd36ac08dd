"""Compacted working sets of key-frame windows (fdgs_scene_compact; the filter
of P:285 realised as a dense copy of the window's active Gaussians): frames
rendered from the working set without a mask are bit-identical to masked
renders of the full scene, records report the original indices, and the
working set is exactly the oracle's active set."""
import numpy as np
import pytest
import torch

import fdgs_inputs as fi
import oracle
import paper_2503_16422_b200 as fd
from paper_2503_16422_b200 import _lib

from parity import assert_records_bit_exact, mask_bits

pytestmark = pytest.mark.gpu


def _window(name, n, W, H, f, count, frame):
    scene = fi.make_scene(name, n=n, seed=4)
    cams = fi.make_cameras(name, width=W, height=H, fx=f, count=count)
    F, D = fi.CONFIGS[name]["frames"], fi.CONFIGS[name]["keyframe_interval"]
    times = fi.frame_times(F)
    kf = fd.keyframes(F, D)
    l, r = fd.bracket(kf, frame)
    sc = fd.Scene.from_arrays(scene)
    ml = fd.keyframe_mask(sc, cams, float(times[kf[l]]))
    mr = fd.keyframe_mask(sc, cams, float(times[kf[r]]))
    return scene, cams, sc, ml, mr, float(times[frame])


@pytest.mark.parametrize("vq", [False, True])
def test_working_set_frames_equal_masked_frames(vq):
    scene, cams, sc, ml, mr, t = _window("c3", 30_000, 320, 240, 240.0, 4, 130)
    if vq:
        scene = fi.vq_scene(scene, codebook_size=300, seed=2)
        sc = fd.Scene.from_arrays(scene)
    ws = sc.compact(ml, mr)
    active = ml.cpu().numpy().view(np.uint32) | mr.cpu().numpy().view(np.uint32)
    want = np.nonzero(mask_bits(active, scene.n))[0]
    assert ws.n == want.size < scene.n
    assert np.array_equal(ws.t["gid"].cpu().numpy(), want)
    r = fd.Renderer(sc, 320, 240)
    for cam in cams:
        a, sa = r.render_checked(cam, t, ml, mr)
        a = a.clone()
        b = r.render(cam, t, scene=ws)
        torch.cuda.synchronize()
        assert torch.equal(a, b)
    views = r.debug_views()  # of the last (working-set) frame: original indices, oracle records
    assert_records_bit_exact(views, scene, cams[-1], t, active)


def test_working_sets_in_the_pipeline_and_errors():
    scene, cams, sc, ml, mr, t = _window("c3", 20_000, 200, 160, 150.0, 3, 70)
    ws = sc.compact(ml, mr)
    frames_m = [(cams[k % 3], t, ml, mr) for k in range(7)]
    frames_w = [(cams[k % 3], t, None, None, ws) for k in range(7)]
    pipe = fd.RenderPipeline(sc, 200, 160, depth=3)
    a = [pipe.renderers[0].new_output() for _ in frames_m]
    b = [pipe.renderers[0].new_output() for _ in frames_w]
    pipe.render_many(frames_w, b)
    pipe.render_many(frames_m, a)   # the full scene again: workspaces reset for the other layout
    pipe.render_many(frames_w, b)
    torch.cuda.synchronize()
    for x, y in zip(a, b):
        assert torch.equal(x, y)
    with pytest.raises(ValueError):
        ws.compact(ml, mr)
    with pytest.raises(fd.FdgsError) as e:
        fd.keyframe_mask(ws, cams, t)
    assert e.value.status == _lib.FDGS_ERR_INVALID_ARG


def test_bench_launch_configuration_full_c3():
    """BASELINE configs[2] at full size in the launch configuration bench.py
    times: RenderPipeline on 4 stream pairs, frames across a key-frame boundary
    rendered from their windows' working sets, against single-stream masked
    renders (bit-identical) and, for one frame, the oracle (sampled pixels)."""
    from parity import assert_rgb_parity
    scene = fi.make_scene("c3")
    cams = fi.make_cameras("c3")
    times = fi.frame_times(300)
    kf = fd.keyframes(300, 20)
    sc = fd.Scene.from_arrays(scene)
    masks = [fd.keyframe_mask(sc, cams, float(times[k])) for k in kf]
    seq = [(ti, ci) for ti in (99, 100, 101) for ci in (0, 7, 13)]
    sets, frames, refs = {}, [], []
    r = fd.Renderer(sc, 1352, 1014)
    for ti, ci in seq:
        l, rr = fd.bracket(kf, ti)
        if (l, rr) not in sets:
            sets[(l, rr)] = sc.compact(masks[l], masks[rr])
        frames.append((fd.camera_struct(cams[ci]), float(times[ti]), None, None, sets[(l, rr)]))
        refs.append(r.render_checked(cams[ci], float(times[ti]), masks[l], masks[rr])[0].clone())
    pipe = fd.RenderPipeline(sc, 1352, 1014, depth=4)
    outs = [pipe.renderers[0].new_output() for _ in frames]
    pipe.render_many(frames, outs)
    torch.cuda.synchronize()
    for a, b in zip(outs, refs):
        assert torch.equal(a, b)
    ti, ci = seq[4]
    l, rr = fd.bracket(kf, ti)
    active = masks[l].cpu().numpy().view(np.uint32) | masks[rr].cpu().numpy().view(np.uint32)
    pix = np.unique(np.random.default_rng(5).integers(0, 1352 * 1014, 2500))
    orc = oracle.render(scene, cams[ci], float(times[ti]), mask=active, pixels=pix)
    assert_rgb_parity(outs[4].cpu().numpy(), orc, pixels=pix)


def test_compact_on_a_side_stream():
    """Scene.compact on a non-current stream orders its
    zero-fill, kernel and count read-back on that stream; a working set whose
    count stays on the device (sync=False) renders the same frame."""
    scene = fi.make_scene("c3", n=40_000, seed=12)
    cams = fi.make_cameras("c3", width=240, height=180, fx=180.0, count=3)
    sc = fd.Scene.from_arrays(scene)
    t0, t1 = float(np.float32(0.2)), float(np.float32(0.26))
    ml, mr = fd.keyframe_mask(sc, cams, t0), fd.keyframe_mask(sc, cams, t1)
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    busy = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    with torch.cuda.stream(side):
        busy.fill_(1.0)                     # keep the side stream busy when compact starts
    a = sc.compact(ml, mr, stream=side)
    want = int(np.count_nonzero(np.unpackbits((ml.cpu().numpy().view(np.uint32) | mr.cpu().numpy().view(np.uint32))
                                              .view(np.uint8), bitorder="little")[:sc.n]))
    assert a.n == want
    b = sc.compact(ml, mr, stream=side, sync=False)
    assert b.n == sc.n and int(b.count.item()) == want
    r = fd.Renderer(sc, 240, 180)
    ref, _ = r.render_checked(cams[1], 0.23, ml, mr)
    ref = ref.clone()
    for ws in (a, b):
        out = r.render(cams[1], 0.23, scene=ws)
        torch.cuda.synchronize()
        assert torch.equal(out, ref)
