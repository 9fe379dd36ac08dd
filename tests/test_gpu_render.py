"""GPU parity of the CUDA render path (through the C-ABI) against the oracle.

Bars (BASELINE.json north_star): masks, decision records and tile lists
bit-exact; RGB max-abs <= 2e-4 and mean-abs <= 1e-5 against the oracle's
nearest admissible termination branch.  Sizes span several tiles with ragged
edges; full-size configs are checked on the launch configuration bench.py
times (sampled pixels).
"""
import math

import numpy as np
import pytest
import torch

import fdgs_inputs as fi
import oracle
import paper_2503_16422_b200 as fd
from paper_2503_16422_b200 import _lib

from parity import assert_records_bit_exact, assert_rgb_parity, assert_tile_lists_bit_exact, mask_bits

pytestmark = pytest.mark.gpu


def _np_mask(t):
    return t.cpu().numpy().view(np.uint32)


def _render(scene_arr, cam, t, mask_l=None, mask_r=None, max_entries=None):
    sc = fd.Scene.from_arrays(scene_arr)
    r = fd.Renderer(sc, cam.width, cam.height, max_entries=max_entries)
    T = torch.empty((cam.height, cam.width), dtype=torch.float32, device="cuda")
    out, stats = r.render_checked(cam, t, mask_l, mask_r, out_T=T)
    return out.cpu().numpy(), T.cpu().numpy(), stats, r


# ------------------------------------------------------------------ C1 tiny
@pytest.mark.parametrize("t", [0.0, 1 / 3, 2 / 3, 1.0])
def test_c1_full_frame_parity(t):
    scene = fi.make_scene("c1")
    cam = fi.make_cameras("c1")[0]
    t = float(np.float32(t))
    img, T, stats, r = _render(scene, cam, t)
    views = r.debug_views()
    assert_records_bit_exact(views, scene, cam, t)
    assert_tile_lists_bit_exact(views, scene, cam, t)
    orc = oracle.render(scene, cam, t)
    assert_rgb_parity(img, orc)
    assert np.abs(T.reshape(-1) - orc["T"]).max() < 2e-4
    assert stats.n_act == scene.n and stats.n_vis == orc["stats"]["n_vis"]
    # Eq. 2 work counters of the counting blend variant = the oracle's counts
    # (pairs in the pixel AABB before termination / pairs composited), up to
    # knife-edge pixels
    sc = fd.Scene.from_arrays(scene)
    rr = fd.Renderer(sc, cam.width, cam.height)
    st = torch.zeros(4, dtype=torch.int64, device="cuda")
    rr.render(cam, t, stats=st)
    s_np = st.cpu().numpy()
    knife = orc["stats"]["knife"]
    assert abs(int(s_np[2]) - orc["stats"]["evaluated"]) <= 64 * knife
    assert abs(int(s_np[3]) - orc["stats"]["blended"]) <= 64 * knife


# ------------------------------------------------------- reduced configs
SMALL = {
    # name: (n, width, height, fx, cameras, frames, interval)
    "c2": (20_000, 200, 200, 1111.0 / 4, 6, 150, 10),
    "c3": (20_000, 338, 254, 250.0, 5, 300, 20),
    "c4": (60_000, 338, 254, 250.0, 5, 300, 20),
}


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_reduced_config_masked_parity(name):
    n, W, H, f, ncam, F, D = SMALL[name]
    scene = fi.make_scene(name, n=n)
    cams = fi.make_cameras(name, width=W, height=H, fx=f, count=ncam)
    times = fi.frame_times(F)
    kf = fd.keyframes(F, D)
    frame = kf[3] + D // 2                      # mid-window
    l, r = fd.bracket(kf, frame)
    sc = fd.Scene.from_arrays(scene)
    ml = fd.keyframe_mask(sc, cams, float(times[kf[l]]))
    mr = fd.keyframe_mask(sc, cams, float(times[kf[r]]))
    torch.cuda.synchronize()
    for m, k in ((ml, kf[l]), (mr, kf[r])):
        assert np.array_equal(_np_mask(m), oracle.keyframe_mask(scene, cams, times[k]))
    active = _np_mask(ml) | _np_mask(mr)
    cam = cams[ncam // 2]
    t = float(times[frame])
    img, T, stats, rd = _render(scene, cam, t, ml, mr)
    views = rd.debug_views()
    assert stats.n_act == int(mask_bits(active, n).sum())
    assert_records_bit_exact(views, scene, cam, t, active)
    assert_tile_lists_bit_exact(views, scene, cam, t, active)
    orc = oracle.render(scene, cam, t, mask=active)
    mx, mean, used = assert_rgb_parity(img, orc)
    assert stats.n_vis == orc["stats"]["n_vis"] > 100


# --------------------------------------------------- full-size C3 (bench)
def test_c3_full_size_sampled_parity():
    scene = fi.make_scene("c3")
    cams = fi.make_cameras("c3")
    times = fi.frame_times(300)
    kf = fd.keyframes(300, 20)
    frame = 150
    l, r = fd.bracket(kf, frame)
    sc = fd.Scene.from_arrays(scene)
    ml = fd.keyframe_mask(sc, cams, float(times[kf[l]]))
    mr = fd.keyframe_mask(sc, cams, float(times[kf[r]]))
    torch.cuda.synchronize()
    assert np.array_equal(_np_mask(ml), oracle.keyframe_mask(scene, cams, times[kf[l]]))
    assert np.array_equal(_np_mask(mr), oracle.keyframe_mask(scene, cams, times[kf[r]]))
    active = _np_mask(ml) | _np_mask(mr)
    cam = cams[7]
    t = float(times[frame])
    img, T, stats, rd = _render(scene, cam, t, ml, mr)
    views = rd.debug_views()
    assert_records_bit_exact(views, scene, cam, t, active)
    assert_tile_lists_bit_exact(views, scene, cam, t, active)
    rng = np.random.default_rng(0)
    pix = np.unique(rng.integers(0, cam.width * cam.height, 4000))
    orc = oracle.render(scene, cam, t, mask=active, pixels=pix)
    assert_rgb_parity(img, orc, pixels=pix)


def test_c4_full_size_sampled_parity_unmasked():
    scene = fi.make_scene("c4")
    cam = fi.make_cameras("c4")[3]
    t = float(fi.frame_times(300)[77])
    img, T, stats, rd = _render(scene, cam, t)
    views = rd.debug_views()
    assert_records_bit_exact(views, scene, cam, t)
    assert_tile_lists_bit_exact(views, scene, cam, t)
    rng = np.random.default_rng(1)
    pix = np.unique(rng.integers(0, cam.width * cam.height, 1500))
    orc = oracle.render(scene, cam, t, pixels=pix)
    assert_rgb_parity(img, orc, pixels=pix)


def test_c4_full_size_sampled_parity_masked():
    """BASELINE configs[3] masked (the bench's --config c4 path): key-frame
    masks bit-exact against the oracle, records and tile lists bit-exact under
    the OR-ed mask, sampled RGB parity."""
    scene = fi.make_scene("c4")
    cams = fi.make_cameras("c4")
    times = fi.frame_times(300)
    kf = fd.keyframes(300, 20)
    frame = 211
    l, r = fd.bracket(kf, frame)
    sc = fd.Scene.from_arrays(scene)
    ml = fd.keyframe_mask(sc, cams, float(times[kf[l]]))
    mr = fd.keyframe_mask(sc, cams, float(times[kf[r]]))
    assert np.array_equal(_np_mask(ml), oracle.keyframe_mask(scene, cams, times[kf[l]]))
    assert np.array_equal(_np_mask(mr), oracle.keyframe_mask(scene, cams, times[kf[r]]))
    active = _np_mask(ml) | _np_mask(mr)
    cam = cams[16]
    t = float(times[frame])
    img, T, stats, rd = _render(scene, cam, t, ml, mr)
    assert stats.n_act == int(mask_bits(active, scene.n).sum()) < scene.n
    views = rd.debug_views()
    assert_records_bit_exact(views, scene, cam, t, active)
    assert_tile_lists_bit_exact(views, scene, cam, t, active)
    pix = np.unique(np.random.default_rng(2).integers(0, cam.width * cam.height, 1500))
    orc = oracle.render(scene, cam, t, mask=active, pixels=pix)
    assert_rgb_parity(img, orc, pixels=pix)


# ------------------------------------------------------------ invariants
def test_all_ones_mask_equals_unmasked_and_determinism():
    n, W, H, f = 30_000, 300, 200, 220.0
    scene = fi.make_scene("c3", n=n)
    cam = fi.make_cameras("c3", width=W, height=H, fx=f, count=3)[1]
    ones = torch.full((fd.mask_words(n),), -1, dtype=torch.int32, device="cuda")
    a, _, _, _ = _render(scene, cam, 0.4)
    b, _, _, _ = _render(scene, cam, 0.4, ones)
    c, _, _, _ = _render(scene, cam, 0.4, ones, ones)
    d, _, _, _ = _render(scene, cam, 0.4)
    assert np.array_equal(a, b) and np.array_equal(a, c)
    assert np.array_equal(a, d)                      # bit-identical reruns


def test_keyframe_soundness_on_gpu():
    n, W, H, f = 30_000, 300, 200, 220.0
    scene = fi.make_scene("c3", n=n)
    cams = fi.make_cameras("c3", width=W, height=H, fx=f, count=4)
    sc = fd.Scene.from_arrays(scene)
    tk = float(np.float32(20 / 299))
    m = fd.keyframe_mask(sc, cams, tk)
    for cam in cams:
        a, _, _, _ = _render(scene, cam, tk)
        b, _, _, _ = _render(scene, cam, tk, m)
        assert np.array_equal(a, b)


# ------------------------------------------------------------ edge cases
def test_empty_scene_and_all_zero_mask_give_background():
    cam = fi.make_cameras("c1")[0]
    cam.bg = (0.1, 0.2, 0.3)
    empty = fi.make_scene("c1", n=1).subset([])
    img, T, stats, _ = _render(empty, cam, 0.5)
    assert np.all(img == np.array(cam.bg, np.float32)[:, None, None]) and np.all(T == 1)
    scene = fi.make_scene("c1")
    zero = torch.zeros(fd.mask_words(scene.n), dtype=torch.int32, device="cuda")
    img, T, stats, _ = _render(scene, cam, 0.5, zero)
    assert stats.n_act == 0 and stats.n_vis == 0
    assert np.all(img == np.array(cam.bg, np.float32)[:, None, None])
    # the pipeline's front-end graphs (an empty layout captures no cull / slice
    # nodes) and the native batch, both submission paths
    sc = fd.Scene.from_arrays(empty)
    for native in (False, True):
        pipe = fd.RenderPipeline(sc, cam.width, cam.height, depth=2, native=native)
        outs = [pipe.renderers[0].new_output() for _ in range(3)]
        pipe.render_many([(cam, 0.5, None, None)] * 3, outs)
        torch.cuda.synchronize()
        for o in outs:
            assert np.all(o.cpu().numpy() == np.array(cam.bg, np.float32)[:, None, None])


@pytest.mark.parametrize("W,H", [(1, 1), (17, 33), (16, 16), (250, 7)])
def test_ragged_and_tiny_images(W, H):
    scene = fi.make_scene("c1", n=800, seed=9)
    cam = fi.make_cameras("c1", width=W, height=H, fx=64.0 * max(W, H) / 64)[0]
    img, T, stats, rd = _render(scene, cam, 0.5)
    views = rd.debug_views()
    assert_records_bit_exact(views, scene, cam, 0.5)
    assert_tile_lists_bit_exact(views, scene, cam, 0.5)
    assert_rgb_parity(img, oracle.render(scene, cam, 0.5))


@pytest.mark.parametrize("W,H", [(48, 4160), (2048, 2048)])
def test_large_tile_grids(W, H):
    """Edge of the tile-grid limits: more than 256 tile rows (the row partition
    then takes its second 8-bit pass) and the FDGS_MAX_TILES grid (128 x 128
    tiles).  Records and tile lists bit-exact, sampled RGB parity."""
    scene = fi.make_scene("c1", n=3000, seed=13)
    cam = fi.make_cameras("c1", width=W, height=H, fx=64.0 * max(W, H) / 64)[0]
    assert ((W + 15) // 16) * ((H + 15) // 16) <= 16384
    img, T, stats, rd = _render(scene, cam, 0.4)
    views = rd.debug_views()
    assert_records_bit_exact(views, scene, cam, 0.4)
    assert_tile_lists_bit_exact(views, scene, cam, 0.4)
    pix = np.unique(np.random.default_rng(3).integers(0, W * H, 6000))
    assert_rgb_parity(img, oracle.render(scene, cam, 0.4, pixels=pix), pixels=pix)
    if H > 4096:
        assert stats.n_vis > 100


def test_tile_grid_above_the_limit_is_unsupported():
    scene = fi.make_scene("c1", n=100)
    cam = fi.make_cameras("c1", width=2064, height=2048, fx=2000.0)[0]
    sc = fd.Scene.from_arrays(scene)
    with pytest.raises(fd.FdgsError) as e:
        fd.Renderer(sc, 2064, 2048).render_checked(cam, 0.5)
    assert e.value.status == _lib.FDGS_ERR_UNSUPPORTED


def test_single_gaussian_closed_form_on_gpu():
    """North-star pin, on the GPU: one on-axis isotropic Gaussian."""
    cam = fi.scenes._cam(65, 65, 64.0, np.eye(3), np.zeros(3), np.zeros(3), bg=(0.1, 0.2, 0.3))
    cam.cx = cam.cy = 32.5
    sc = fi.isotropic_scene([[0, 0, 4.0, 0.5]], [[0.2, 0.2, 0.2, 0.3]], [0.9], colors=[0.8, 0.4, 0.1])
    img, T, _, _ = _render(sc, cam, 0.5)
    j, i = np.mgrid[0:65, 0:65]
    s = float(sc.scale[0, 0])
    sp2 = (64.0 * s / 4.0) ** 2 + 0.3
    a_un = float(sc.opacity[0]) * np.exp(-((i + 0.5 - 32.5) ** 2 + (j + 0.5 - 32.5) ** 2) / (2 * sp2))
    alpha = np.where(a_un >= 1 / 255, np.minimum(0.99, a_un), 0.0)
    c = 0.28209479177387814 * sc.sh[0, 0].astype(np.float64) + 0.5
    bg = np.array(cam.bg, np.float32).astype(np.float64)
    expect = c[:, None, None] * alpha[None] + (1 - alpha[None]) * bg[:, None, None]
    sure = np.abs(a_un * 255 - 1) > 1e-4
    assert np.abs(img - expect)[:, sure].max() < 2e-4


def test_overflow_is_reported_and_recovered():
    scene = fi.make_scene("c1")
    cam = fi.make_cameras("c1")[0]
    sc = fd.Scene.from_arrays(scene)
    r = fd.Renderer(sc, cam.width, cam.height, max_entries=8)
    with pytest.raises(fd.FdgsError) as ei:
        r.render_checked(cam, 0.5, grow=False)
    assert ei.value.status == _lib.FDGS_ERR_OVERFLOW
    out, stats = r.render_checked(cam, 0.5)          # grows and re-renders
    assert stats.status == 0 and r.max_entries >= stats.n_entries
    assert_rgb_parity(out.cpu().numpy(), oracle.render(scene, cam, 0.5))


def test_validate_and_log255():
    scene = fi.make_scene("c3", n=50_000)
    sc = fd.Scene.from_arrays(scene)
    st, bad = fd.validate(sc)
    assert st == 0 and bad == -1
    L = fd.log255_opacity(sc.t["opacity"])
    assert np.array_equal(L.cpu().numpy().view(np.uint32), scene.log255_opacity.view(np.uint32))
    broken = fi.make_scene("c3", n=1000)
    broken.rot_l[17] *= 1.01
    broken.scale[400, 2] = 0.0
    st, bad = fd.validate(fd.Scene.from_arrays(broken))
    assert st == _lib.FDGS_ERR_INVALID_SCENE and bad == 17


def test_mask_or_and_compact_bit_exact():
    rng = np.random.default_rng(3)
    for n in (1, 31, 32, 33, 1000, 200_003):
        nw = (n + 31) // 32
        a = rng.integers(0, 2 ** 32, nw, dtype=np.uint64).astype(np.uint32)
        b = rng.integers(0, 2 ** 32, nw, dtype=np.uint64).astype(np.uint32)
        if n % 32:
            a[-1] &= (1 << (n % 32)) - 1
            b[-1] &= (1 << (n % 32)) - 1
        ta = torch.from_numpy(a.view(np.int32)).cuda()
        tb = torch.from_numpy(b.view(np.int32)).cuda()
        o = fd.mask_or(ta, tb, n)
        assert np.array_equal(_np_mask(o), a | b)
        idx = fd.mask_compact(ta, n, tb).cpu().numpy()
        want = np.nonzero(mask_bits(a | b, n))[0]
        assert np.array_equal(idx, want)
        idx = fd.mask_compact(ta, n).cpu().numpy()
        assert np.array_equal(idx, np.nonzero(mask_bits(a, n))[0])


def test_extrapolated_time_and_bad_camera():
    scene = fi.make_scene("c1")
    cam = fi.make_cameras("c1")[0]
    img, _, stats, _ = _render(scene, cam, 1.7)        # outside [0,1]: allowed
    assert_rgb_parity(img, oracle.render(scene, cam, float(np.float32(1.7))))
    bad = fi.make_cameras("c1")[0]
    bad.R = np.eye(3, dtype=np.float32) * 2
    sc = fd.Scene.from_arrays(scene)
    with pytest.raises(fd.FdgsError):
        fd.Renderer(sc, 64, 64).render(bad, 0.5)


def test_render_pipeline_matches_sequential():
    """Frame pipelining over 3 streams/workspaces gives the sequential frames bit for bit."""
    n, W, H, f = 30_000, 300, 200, 220.0
    scene = fi.make_scene("c3", n=n)
    cams = fi.make_cameras("c3", width=W, height=H, fx=f, count=4)
    sc = fd.Scene.from_arrays(scene)
    kf = fd.keyframes(300, 20)
    times = fi.frame_times(300)
    masks = [fd.keyframe_mask(sc, cams, float(times[k])) for k in kf]
    frames = []
    for fr in range(100, 124):
        l, r = fd.bracket(kf, fr)
        frames.append((cams[fr % 4], float(times[fr]), masks[l], masks[r]))
    seq = fd.Renderer(sc, W, H)
    refs = [seq.render_checked(cam, t, ml, mr)[0] for (cam, t, ml, mr) in frames]
    for split, native, threads, graphs in ((False, False, 1, True), (True, False, 1, True), (False, True, 1, True),
                                           (True, True, 3, True), (True, True, 2, True), (True, False, 1, False),
                                           (True, True, 1, False), (False, False, 1, False)):
        pipe = fd.RenderPipeline(sc, W, H, depth=3, split=split, native=native, threads=threads, graphs=graphs)
        outs = [pipe.renderers[0].new_output() for _ in frames]
        pipe.render_many(frames, outs)
        pipe.render_many(frames[::-1], outs[::-1])   # reuse every workspace again
        torch.cuda.synchronize()
        for ref, o in zip(refs, outs):
            assert torch.equal(ref, o)
        # overlapped D2H into pinned host buffers (the e2e path of bench.py)
        host = [torch.empty_like(o, device="cpu").pin_memory() for o in outs]
        pipe.render_many(frames, outs, host_outs=host)
        torch.cuda.current_stream().synchronize()
        for ref, h in zip(refs, host):
            assert torch.equal(ref.cpu(), h)


def test_interleaved_and_planar_parameters_identical():
    """fdgs_scene.param_stride: the interleaved 64-byte records (the Python
    Scene's default) and four SoA planes give bit-identical frames, masks and
    scores."""
    scene = fi.make_scene("c3", n=40_000, seed=4)
    cams = fi.make_cameras("c3", width=300, height=220, fx=222.0, count=3)
    a = fd.Scene.from_arrays(scene)
    b = fd.Scene({f: getattr(scene, f) for f in fd.api._FIELDS}, interleaved=False)
    assert a.struct.param_stride == 4 and b.struct.param_stride == 0
    t = float(np.float32(0.37))
    ma, mb = fd.keyframe_mask(a, cams, t), fd.keyframe_mask(b, cams, t)
    assert torch.equal(ma, mb)
    ra, rb = fd.Renderer(a, 300, 220), fd.Renderer(b, 300, 220)
    for cam in cams:
        x, _ = ra.render_checked(cam, t, ma, ma)
        y, _ = rb.render_checked(cam, t, mb, mb)
        assert torch.equal(x, y)
    sa = fd.stv_score(a, cams, [0.2, 0.6])["score"]
    sb = fd.stv_score(b, cams, [0.2, 0.6])["score"]
    assert torch.equal(sa, sb)


def test_native_pipeline_working_sets_without_host_sync():
    """fdgs_pipeline_render with compacted working sets whose size stays on the
    device (Scene.compact sync=False, fdgs_scene.d_n): the frames equal the
    masked renders bit for bit, with stats and status copies."""
    scene = fi.make_scene("c3", n=30_000, seed=8)
    cams = fi.make_cameras("c3", width=300, height=200, fx=220.0, count=4)
    sc = fd.Scene.from_arrays(scene)
    kf = fd.keyframes(300, 20)
    times = fi.frame_times(300)
    masks = [fd.keyframe_mask(sc, cams, float(times[k])) for k in kf]
    seq = fd.Renderer(sc, 300, 200)
    frames, refs, wsets = [], [], {}
    for fr in range(35, 65):
        l, r = fd.bracket(kf, fr)
        if (l, r) not in wsets:
            wsets[(l, r)] = sc.compact(masks[l], masks[r], sync=False)
            assert wsets[(l, r)].n == sc.n and wsets[(l, r)].struct.d_n
        frames.append((cams[fr % 4], float(times[fr]), None, None, wsets[(l, r)]))
        refs.append(seq.render_checked(cams[fr % 4], float(times[fr]), masks[l], masks[r])[0].clone())
    pipe = fd.RenderPipeline(sc, 300, 200, depth=4, native=True, threads=2)
    outs = [pipe.renderers[0].new_output() for _ in frames]
    st = pipe.render_many_checked(frames, outs)
    assert (st[:, 3] == 0).all()
    for ref, o in zip(refs, outs):
        assert torch.equal(ref, o)
    m = wsets[(1, 2)]
    exact = sc.compact(masks[1], masks[2])
    assert int(m.count.item()) == exact.n and int(st[0, 0]) == exact.n


def test_pipeline_overflow_detected_and_re_rendered():
    """render_many_checked: frames that exceed a deliberately tiny tile-entry
    capacity are flagged by their counter block and re-rendered (after growing
    the workspace) to exactly the frames of an ample sequential renderer."""
    scene = fi.make_scene("c3", n=20_000, seed=2)
    cams = fi.make_cameras("c3", width=200, height=150, fx=150.0, count=3)
    sc = fd.Scene.from_arrays(scene)
    frames = [(cams[k % 3], float(np.float32(0.1 * k)), None, None) for k in range(9)]
    seq = fd.Renderer(sc, 200, 150)
    refs = [seq.render_checked(cam, t)[0].clone() for (cam, t, _, _) in frames]
    pipe = fd.RenderPipeline(sc, 200, 150, depth=3, max_entries=4096)
    outs = [pipe.renderers[0].new_output() for _ in frames]
    st = pipe.render_many_checked(frames, outs)
    assert (st[:, 3] == 0).all() and (st[:, 2] > 4096).any()
    for ref, o in zip(refs, outs):
        assert torch.equal(ref, o)
    # the grown workspaces serve the graph path afterwards (graphs re-captured on them)
    pipe.render_many(frames, outs := [pipe.renderers[0].new_output() for _ in frames])
    torch.cuda.synchronize()
    for ref, o in zip(refs, outs):
        assert torch.equal(ref, o)


def test_cuda_graph_frames_equal_launched_frames():
    """fdgs_render_graph_*: the captured frame replayed with new arguments
    (camera, t, masks, output, working set) gives the frames of fdgs_render bit
    for bit, also inside the pipeline."""
    scene = fi.make_scene("c3", n=25_000, seed=6)
    cams = fi.make_cameras("c3", width=240, height=180, fx=180.0, count=4)
    sc = fd.Scene.from_arrays(scene)
    kf = fd.keyframes(300, 20)
    times = fi.frame_times(300)
    masks = [fd.keyframe_mask(sc, cams, float(times[k])) for k in kf]
    frames = []
    for fr in range(95, 113):
        l, r = fd.bracket(kf, fr)
        frames.append((cams[fr % 4], float(times[fr]), masks[l], masks[r]))
    seq = fd.Renderer(sc, 240, 180)
    refs = [seq.render_checked(cam, t, ml, mr)[0].clone() for (cam, t, ml, mr) in frames]
    g = fd.Renderer(sc, 240, 180)
    for (cam, t, ml, mr), ref in zip(frames, refs):
        out = g.render_graph(cam, t, ml, mr)
        torch.cuda.synchronize()
        assert torch.equal(out, ref)
    # working sets through the same graph (n_capacity keeps the layout)
    l, r = fd.bracket(kf, 100)
    ws = sc.compact(masks[l], masks[r])
    out = g.render_graph(frames[5][0], frames[5][1], scene=ws)
    torch.cuda.synchronize()
    assert torch.equal(out, refs[5])
    pipe = fd.RenderPipeline(sc, 240, 180, depth=3, graphs=True)
    outs = [pipe.renderers[0].new_output() for _ in frames]
    pipe.render_many(frames, outs)
    torch.cuda.synchronize()
    for ref, o in zip(refs, outs):
        assert torch.equal(ref, o)
    # stage events through the graph (event-record nodes re-pointed per frame),
    # then a batch without events (the nodes fall back to their own events)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in frames]
    outs = [pipe.renderers[0].new_output() for _ in frames]
    pipe.render_many(frames, outs, stage_events=evs)
    torch.cuda.synchronize()
    for ref, o, ev in zip(refs, outs, evs):
        assert torch.equal(ref, o)
        dt = [ev[k].elapsed_time(ev[k + 1]) for k in range(4)]
        assert all(x >= 0.0 for x in dt) and sum(dt) > 0.0, dt
    stamp = [ev[0].elapsed_time(ev[4]) for ev in evs]
    outs = [pipe.renderers[0].new_output() for _ in frames]
    pipe.render_many(frames, outs)
    torch.cuda.synchronize()
    for ref, o in zip(refs, outs):
        assert torch.equal(ref, o)
    assert stamp == [ev[0].elapsed_time(ev[4]) for ev in evs]  # not re-recorded
    # the native batch over the slots' graphs, with stage events
    nat = fd.RenderPipeline(sc, 240, 180, depth=3, native=True, graphs=True)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in frames]
    for row in evs:
        for e in row:
            e.record()
    outs = [nat.renderers[0].new_output() for _ in frames]
    nat.render_many(frames, outs, stage_events=evs)
    torch.cuda.synchronize()
    for ref, o, ev in zip(refs, outs, evs):
        assert torch.equal(ref, o)
        assert all(ev[k].elapsed_time(ev[k + 1]) >= 0.0 for k in range(4))


def test_aabb_redundant_flag_sound():
    """k_slice's aabb_redundant bit (rec1.w bit 31): for every flagged record of
    a C2 frame, no pixel centre outside the pixel AABB has e2 >= 0.  e2 is
    evaluated in binary64 from the fp32 record fields with the pinned chain's
    rounding budget (9 x 2^-24 of the absolute terms) added, over every pixel of
    the image outside the AABB within the record's tile-cover box + 2 px.  Also
    checks that the flag holds for the bulk of the records (the mask-free blend
    loop is the common case)."""
    scene = fi.make_scene("c2")
    cam = fi.make_cameras("c2")[3]
    t = 0.5
    _, _, _, r = _render(scene, cam, t)
    v = r.debug_views()
    n = v["n_vis"]
    r0 = v["rec0"].cpu().numpy().astype(np.float64)
    r1 = v["rec1"].cpu().numpy()
    ax = r1[:, 2].view(np.uint32)
    ay = r1[:, 3].view(np.uint32)
    flag = (ay >> 31) == 1
    assert r0.shape[0] == n and flag.mean() > 0.9, flag.mean()
    px0, px1, py0, py1 = ax & 0xFFFF, ax >> 16, ay & 0xFFFF, (ay >> 16) & 0x7FFF
    u, vv, A, B = r0.T
    C, Q2 = r1[:, 0].astype(np.float64), r1[:, 1].astype(np.float64)
    budget = 9 * 2.0 ** -24
    checked = 0
    for i in np.nonzero(flag)[0][::7]:
        x0, x1 = max(int(px0[i]) - 40, 0), min(int(px1[i]) + 40, cam.width - 1)
        y0, y1 = max(int(py0[i]) - 40, 0), min(int(py1[i]) + 40, cam.height - 1)
        X, Y = np.meshgrid(np.arange(x0, x1 + 1) + 0.5 - u[i], np.arange(y0, y1 + 1) + 0.5 - vv[i])
        q = A[i] * X * X + B[i] * X * Y + C[i] * Y * Y + Q2[i]
        err = budget * (abs(A[i]) * X * X + abs(B[i]) * abs(X * Y) + abs(C[i]) * Y * Y + abs(Q2[i]))
        gx, gy = np.meshgrid(np.arange(x0, x1 + 1), np.arange(y0, y1 + 1))
        outside = (gx < px0[i]) | (gx > px1[i]) | (gy < py0[i]) | (gy > py1[i])
        assert not np.any(outside & (q + err >= 0.0)), i
        checked += 1
    assert checked > 100


def test_counting_blend_matches_timed_blend():
    """The counting / recording variant k_blend_ws (fdgs_render with d_stats)
    and the timed k_blend_wi give the same C2 frame within the parity bar: the
    same decisions except at termination knife edges (k_blend_ws carries T,
    k_blend_wi U = T/255 with a paired stop test); k_blend_wi itself is
    parity-tested against the oracle above."""
    sc = fd.Scene.from_arrays(fi.make_scene("c2"))
    cam = fi.make_cameras("c2")[5]
    r = fd.Renderer(sc, cam.width, cam.height)
    a = r.render(cam, 0.4).clone()
    st = torch.zeros(4, dtype=torch.int64, device="cuda")
    b = r.render(cam, 0.4, stats=st)
    torch.cuda.synchronize()
    assert a.shape == (3, 800, 800)
    assert (a - b).abs().max().item() <= 2e-4
    assert int(st[2]) >= int(st[3]) > 0          # evaluated >= blended pairs


@pytest.mark.parametrize("cap", [0, 8, 100])
def test_overflow_writes_nothing_past_the_workspace(cap):
    """with more row items / entries than max_entries the
    frame must report OVERFLOW without writing past the workspace (the row
    partition is bounded by the capacity).  A guard region after the
    workspace must keep its pattern."""
    import ctypes as C
    from paper_2503_16422_b200._lib import FdgsFrameStats, lib
    scene = fi.make_scene("c1")
    cam = fi.make_cameras("c1")[0]
    sc = fd.Scene.from_arrays(scene)
    nb = lib().fdgs_render_workspace_bytes(sc.n, cam.width, cam.height, cap)
    guard = 1 << 20
    buf = torch.full((nb + guard,), 0xA5, dtype=torch.uint8, device="cuda")
    buf[:nb].zero_()
    out = torch.empty((3, cam.height, cam.width), dtype=torch.float32, device="cuda")
    hs = FdgsFrameStats()
    cs = fd.camera_struct(cam)
    for t in (0.0, 0.5, 1.0):
        st = lib().fdgs_render_checked(C.byref(sc.struct), None, None, C.byref(cs), float(np.float32(t)),
                                       C.c_void_p(out.data_ptr()), None, C.c_void_p(buf.data_ptr()), nb, cap,
                                       C.byref(hs), C.c_void_p(torch.cuda.current_stream().cuda_stream))
        assert st == _lib.FDGS_ERR_OVERFLOW
    torch.cuda.synchronize()
    assert bool((buf[nb:] == 0xA5).all())


def test_anamorphic_camera_parity():
    """fx != fy and an off-centre principal point (reading R13): records, tile
    lists bit-exact and RGB within the bar on a C3-shaped scene (the oracle's
    projection for such cameras is pinned by test_oracle_projection_pins.py)."""
    scene = fi.make_scene("c3", n=40_000, seed=14)
    cam = fi.make_cameras("c3", width=420, height=300, fx=310.0, count=5)[3]
    cam.fy = float(np.float32(0.7 * cam.fx))
    cam.cx = float(np.float32(0.43 * cam.width))
    cam.cy = float(np.float32(0.58 * cam.height))
    t = float(np.float32(0.41))
    img, T, stats, r = _render(scene, cam, t)
    views = r.debug_views()
    assert_records_bit_exact(views, scene, cam, t)
    assert_tile_lists_bit_exact(views, scene, cam, t)
    assert_rgb_parity(img, oracle.render(scene, cam, t))
    assert stats.n_vis > 1000


def test_stress_scene_parity():
    """Edge cases of the conic and the composite together, whole frame: splats
    just beyond z_near (screen-filling, Jacobian clamp active), opacity 1
    (alpha clamped at 0.99 on every layer: termination after 2-3 layers),
    sub-pixel splats (the 0.3 px^2 dilation dominates), strongly anisotropic
    ones, and Gaussians far outside the frustum."""
    rng = np.random.default_rng(29)
    parts = []
    n1 = 200    # near the camera plane: z in (0.21, 0.6)
    parts.append((np.stack([rng.uniform(-0.2, 0.2, n1), rng.uniform(-0.15, 0.15, n1), rng.uniform(0.21, 0.6, n1),
                            np.full(n1, 0.5)], 1), np.exp(rng.uniform(-4, -2, (n1, 3))), rng.uniform(0.2, 1.0, n1)))
    n2 = 3000   # opacity 1 layers
    parts.append((np.stack([rng.uniform(-2, 2, n2), rng.uniform(-1.5, 1.5, n2), rng.uniform(3, 8, n2),
                            np.full(n2, 0.5)], 1), np.exp(rng.uniform(-3, -1.5, (n2, 3))), np.ones(n2)))
    n3 = 6000   # sub-pixel
    parts.append((np.stack([rng.uniform(-2, 2, n3), rng.uniform(-1.5, 1.5, n3), rng.uniform(2, 9, n3),
                            np.full(n3, 0.5)], 1), np.exp(rng.uniform(-9, -7, (n3, 3))), rng.uniform(0.3, 1.0, n3)))
    n4 = 2000   # anisotropic (one long axis)
    s4 = np.exp(rng.uniform(-6, -4, (n4, 3)))
    s4[:, 0] = np.exp(rng.uniform(-1.5, -0.5, n4))
    parts.append((np.stack([rng.uniform(-2, 2, n4), rng.uniform(-1.5, 1.5, n4), rng.uniform(2, 9, n4),
                            np.full(n4, 0.5)], 1), s4, rng.uniform(0.3, 1.0, n4)))
    n5 = 500    # behind the camera and far to the side
    parts.append((np.stack([rng.uniform(-50, 50, n5), rng.uniform(-50, 50, n5), rng.uniform(-20, 2, n5),
                            np.full(n5, 0.5)], 1), np.exp(rng.uniform(-3, 0, (n5, 3))), rng.uniform(0.3, 1.0, n5)))
    means = np.concatenate([p[0] for p in parts])
    scales = np.concatenate([np.concatenate([p[1], np.full((len(p[1]), 1), 0.4)], 1) for p in parts])
    ops = np.concatenate([p[2] for p in parts])
    n = means.shape[0]
    ql = rng.standard_normal((n, 4))
    ql /= np.linalg.norm(ql, axis=1, keepdims=True)
    ql[:, 0] = np.abs(ql[:, 0])
    sc = fi.isotropic_scene(means, scales, ops, colors=rng.uniform(0, 1, (n, 3)), rot_l=ql,
                            rot_r=np.tile([1.0, 0, 0, 0], (n, 1)))
    cam = fi.scenes._cam(480, 360, 420.0, np.eye(3), np.zeros(3), np.zeros(3), bg=(0.3, 0.2, 0.1))
    for t in (0.5, 0.62):
        img, T, stats, r = _render(sc, cam, t)
        views = r.debug_views()
        assert_records_bit_exact(views, sc, cam, t)
        assert_tile_lists_bit_exact(views, sc, cam, t)
        orc = oracle.render(sc, cam, t)
        assert_rgb_parity(img, orc)
        assert stats.n_vis > 5000 and orc["stats"]["knife"] >= 0
