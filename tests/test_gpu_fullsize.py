"""Full-size GPU parity in bench.py's launch configuration (-m gpu).

Every pixel of whole frames of the BASELINE configs is compared with the
oracle's per-pixel Eq. 2 at the north_star bar (max-abs 2e-4
against the nearest admissible termination branch, mean-abs 1e-5):

* C3 (the metric's workload): a key-frame, a mid-window frame and the first
  frame after a window switch, rendered by RenderPipeline on 6 stream pairs
  (fdgs_pipeline_render) from each window's compacted
  working set whose size stays on the device (Scene.compact sync=False) --
  exactly what bench.py times; masks from the oracle itself (bit-exact
  against the GPU's);
* C4 masked, one whole frame, same path; C2 at full size (100k Gaussians,
  800x800, 50-camera hemisphere), two frames;
* >= 50k Gaussians at exactly one depth (the canonical order's tie rule, R8,
  carried by the onesweep sort): tile lists bit-exact, every pixel;
* the blend's record-to-strip culling (strip_stage) by brute force: no pixel
  with e2 >= 0 lies in a strip the record was not staged for.
"""
import numpy as np
import pytest
import torch

import fdgs_inputs as fi
import oracle
import paper_2503_16422_b200 as fd

from parity import assert_records_bit_exact, assert_rgb_parity, assert_tile_lists_bit_exact

pytestmark = pytest.mark.gpu


def _np(t):
    return t.cpu().numpy().view(np.uint32)


def _pipeline_frames(name, picks, fill_cams=6):
    """Render the frames of `picks` [(time index, camera)] -- each followed by
    frames of other cameras at the same time, so the 6-slot pipeline is full --
    as bench.py does; returns (scene, cams, times, kf, [(ti, ci, image)])."""
    cfg = fi.CONFIGS[name]
    scene = fi.make_scene(name)
    cams = fi.make_cameras(name)
    F, D = cfg["frames"], cfg["keyframe_interval"]
    times = fi.frame_times(F)
    kf = fd.keyframes(F, D)
    sc = fd.Scene.from_arrays(scene)
    need = sorted({k for ti, _ in picks for k in fd.bracket(kf, ti)})
    gmasks = {k: fd.keyframe_mask(sc, cams, float(times[kf[k]])) for k in need}
    torch.cuda.synchronize()
    okf = oracle.keyframes(F, D)
    assert list(okf) == list(kf)
    omasks = {k: oracle.keyframe_mask(scene, cams, times[kf[k]]) for k in need}
    for k in need:                                   # the filter's input, bit-exact
        assert np.array_equal(_np(gmasks[k]), omasks[k])
    frames, keep, wsets = [], [], {}
    for ti, ci in picks:
        li, ri = fd.bracket(kf, ti)
        if (li, ri) not in wsets:
            wsets[(li, ri)] = sc.compact(gmasks[li], gmasks[ri], sync=False)
        for c in [ci] + [(ci + 1 + j) % len(cams) for j in range(fill_cams - 1)]:
            if c == ci:
                keep.append(len(frames))
            frames.append((fd.camera_struct(cams[c]), float(times[ti]), None, None, wsets[(li, ri)]))
    pipe = fd.RenderPipeline(sc, cams[0].width, cams[0].height, depth=6)
    outs = [pipe.renderers[0].new_output() for _ in frames]
    st = pipe.render_many_checked(frames, outs)
    assert (st[:, 3] == 0).all()
    res = [(ti, ci, outs[k].cpu().numpy()) for (ti, ci), k in zip(picks, keep)]
    masks = np.stack([omasks.get(k, np.zeros_like(next(iter(omasks.values())))) for k in range(len(kf))])
    return scene, cams, times, okf, masks, res


def _check_full_frames(scene, cams, times, kf, masks, res):
    for ti, ci, img in res:
        act = oracle.active_mask(masks, kf, ti)      # the oracle's own bracketing and OR
        orc = oracle.render(scene, cams[ci], float(times[ti]), mask=act)
        mx, mean, used = assert_rgb_parity(img, orc)
        assert orc["stats"]["n_vis"] > 1000


def test_c3_bench_path_full_frames():
    """C3 (BASELINE configs[2], the metric's workload): key-frame 140, mid-window
    150, first frame after the switch at 160 -- all pixels."""
    out = _pipeline_frames("c3", [(140, 3), (150, 10), (161, 17)])
    _check_full_frames(*out)


def test_c4_masked_full_frame():
    """C4 masked (BASELINE configs[3], 3M Gaussians): one whole frame."""
    out = _pipeline_frames("c4", [(211, 16)], fill_cams=2)
    _check_full_frames(*out)


def test_c2_full_size_frames():
    """C2 at full size (100k Gaussians, 800x800, 50 hemisphere cameras,
    masks OR-ed over all 50): a mid-window frame and a key-frame."""
    out = _pipeline_frames("c2", [(75, 7), (80, 33)], fill_cams=3)
    _check_full_frames(*out)


def test_equal_depth_sheet_ties_by_index():
    """>= 50k Gaussians at exactly the same camera depth (a fronto-parallel
    sheet; identity rotors, camera R = I, so z = mean_z exactly): the depth
    sort's ties must fall back to ascending index (R8).  Records, canonical
    order and tile lists bit-exact, every pixel within the bar."""
    rng = np.random.default_rng(23)
    n = 60_000
    means = np.stack([rng.uniform(-3.2, 3.2, n), rng.uniform(-2.4, 2.4, n), np.full(n, 5.0), np.full(n, 0.5)], 1)
    s = np.exp(rng.uniform(-4.5, -3.0, n))
    # every third Gaussian on a second sheet (z = 4), interleaved in index order
    means2 = means.copy()
    means2[::3, 2] = 4.0
    sc = fi.isotropic_scene(means2, np.stack([s, s, s, np.full(n, 0.3)], 1), rng.uniform(0.05, 0.95, n),
                            colors=rng.uniform(0, 1, (n, 3)))
    cam = fi.scenes._cam(1352, 1014, 1000.0, np.eye(3), np.zeros(3), np.zeros(3), bg=(0.1, 0.1, 0.1))
    rec = oracle.records(sc, cam, 0.5)
    vis = rec["stage"] == oracle.ST_VISIBLE
    _, counts = np.unique(rec["depth_bits"][vis], return_counts=True)
    assert counts.max() >= 30_000 and vis.sum() >= 50_000
    scene = fd.Scene.from_arrays(sc)
    r = fd.Renderer(scene, 1352, 1014)
    img, stats = r.render_checked(cam, 0.5)
    views = r.debug_views()
    assert_records_bit_exact(views, sc, cam, 0.5)
    assert_tile_lists_bit_exact(views, sc, cam, 0.5)
    assert_rgb_parity(img.cpu().numpy(), oracle.render(sc, cam, 0.5))


def _strip_violations(views, reach, W, H, chunk=1 << 17):
    """Brute force in binary64 on the GPU over every (entry, pixel of its tile
    ∩ AABB): a pixel whose pinned fp32 e2 chain can be >= 0 (exact quadratic +
    the chain's rounding budget, 9 x 2^-24 of the absolute terms) must lie in a
    strip (4 rows) the entry's record was staged for.  Returns (violations,
    staged (entry, strip) pairs, (entry, strip) pairs inside the AABB)."""
    E = views["n_entries"]
    ts = views["tile_start"].long()
    T = ts.numel() - 1
    tiles_x = (W + 15) // 16
    tile = torch.repeat_interleave(torch.arange(T, device=ts.device), ts[1:] - ts[:-1])
    assert tile.numel() == E == reach.numel()
    g_all = views["entries"].long()
    r0 = views["rec0"].double()
    r1 = views["rec1"]
    bits = r1[:, 2:4].contiguous().view(torch.int32).long() & 0x7FFFFFFF
    k = torch.arange(16, device=ts.device, dtype=torch.float64)
    strip_of_row = torch.arange(16, device=ts.device) // 4
    bad = staged = pairs = 0
    for c0 in range(0, E, chunk):
        g = g_all[c0:c0 + chunk]
        t = tile[c0:c0 + chunk]
        tx, ty = (t % tiles_x).double(), (t // tiles_x).double()
        u, v, A, B = [r0[g, i][:, None, None] for i in range(4)]
        C, Q = [r1[g, i].double()[:, None, None] for i in (0, 1)]
        ax, ay = bits[g, 0], bits[g, 1]
        px0, px1 = (ax & 0xFFFF).double(), (ax >> 16).double()
        py0, py1 = (ay & 0xFFFF).double(), (ay >> 16).double()
        ii = 16 * tx[:, None] + k[None]
        jj = 16 * ty[:, None] + k[None]
        inx = (ii >= px0[:, None]) & (ii <= px1[:, None]) & (ii < W)
        iny = (jj >= py0[:, None]) & (jj <= py1[:, None]) & (jj < H)
        dx = (ii + 0.5)[:, None, :] - u
        dy = (jj + 0.5)[:, :, None] - v
        q = A * dx * dx + B * dx * dy + C * dy * dy + Q
        err = 9 * 2.0 ** -24 * (A.abs() * dx * dx + B.abs() * (dx * dy).abs() + C.abs() * dy * dy + Q.abs())
        possible = (q + err >= 0) & inx[:, None, :] & iny[:, :, None]
        rb = reach[c0:c0 + chunk].long()
        row_staged = ((rb[:, None] >> strip_of_row[None]) & 1).bool()        # [e, 16 rows]
        bad += int((possible & ~row_staged[:, :, None]).sum())
        staged += int(sum(((rb >> w) & 1).sum() for w in range(4)))
        pairs += int((iny.view(-1, 4, 4).any(2) & inx.any(1, keepdim=True)).sum())
    return bad, staged, pairs


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_blend_strip_culling_sound_brute_force(name):
    """k_blend_wi's per-row reach test (strip_stage, replayed by
    fdgs_debug_strip_reach): sound on whole frames, and it culls."""
    scene = fi.make_scene(name, n={"c2": None, "c3": None, "c4": 600_000}[name])
    cam = fi.make_cameras(name)[{"c2": 11, "c3": 5, "c4": 14}[name]]
    sc = fd.Scene.from_arrays(scene)
    r = fd.Renderer(sc, cam.width, cam.height)
    r.render_checked(cam, 0.45)
    v = r.debug_views()
    bad, staged, pairs = _strip_violations(v, r.strip_reach(), cam.width, cam.height)
    assert bad == 0
    assert v["n_entries"] > 100_000 and staged < pairs, (staged, pairs)


def test_blend_strip_culling_sound_adversarial():
    """Thin, strongly sheared and very large splats across tile edges."""
    rng = np.random.default_rng(17)
    n = 4000
    means = np.stack([rng.uniform(-3, 3, n), rng.uniform(-2, 2, n), rng.uniform(2.5, 9, n), np.full(n, 0.5)], 1)
    sx = np.exp(rng.uniform(-6, 0.5, n))
    scales = np.stack([sx, sx * np.exp(rng.uniform(-6, 0, n)), sx * np.exp(rng.uniform(-6, 0, n)),
                       np.full(n, 0.4)], 1)
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    sc = fi.isotropic_scene(means, scales, rng.uniform(0.05, 1.0, n), colors=rng.uniform(0, 1, (n, 3)),
                            rot_l=q, rot_r=np.tile([1.0, 0, 0, 0], (n, 1)))
    cam = fi.make_cameras("c3", width=640, height=480, fx=600.0, count=3)[1]
    scene = fd.Scene.from_arrays(sc)
    r = fd.Renderer(scene, cam.width, cam.height)
    img, _ = r.render_checked(cam, 0.5)
    v = r.debug_views()
    bad, staged, pairs = _strip_violations(v, r.strip_reach(), cam.width, cam.height)
    assert bad == 0 and v["n_entries"] > 10_000
    assert_rgb_parity(img.cpu().numpy(), oracle.render(sc, cam, 0.5))


def _cover_violations(views, W, H, chunk=1 << 16):
    """Brute force (binary64 on the GPU) over every (visible Gaussian, tile of
    its pixel-AABB rectangle) pair that is NOT in the tile lists: no pixel of
    tile ∩ AABB may reach e2 >= 0 (exact quadratic + the pinned fp32 chain's
    rounding budget).  Returns (violations, pairs checked, listed entries)."""
    dev = views["tile_start"].device
    tiles_x = (W + 15) // 16
    ts = views["tile_start"].long()
    T = ts.numel() - 1
    tile = torch.repeat_interleave(torch.arange(T, device=dev), ts[1:] - ts[:-1])
    g_list = views["entries"].long()
    nv = views["n_vis"]
    listed = torch.sort(tile * nv + g_list).values
    r0 = views["rec0"].double()
    r1 = views["rec1"]
    bits = r1[:, 2:4].contiguous().view(torch.int32).long() & 0x7FFFFFFF
    px0, px1 = bits[:, 0] & 0xFFFF, bits[:, 0] >> 16
    py0, py1 = bits[:, 1] & 0xFFFF, bits[:, 1] >> 16
    ntx = (px1 >> 4) - (px0 >> 4) + 1
    nty = (py1 >> 4) - (py0 >> 4) + 1
    cnt = ntx * nty
    g_of = torch.repeat_interleave(torch.arange(nv, device=dev), cnt)
    first = torch.cumsum(cnt, 0) - cnt
    k = torch.arange(g_of.numel(), device=dev) - first[g_of]
    tx = (px0[g_of] >> 4) + k % ntx[g_of]
    ty = (py0[g_of] >> 4) + k // ntx[g_of]
    key = (ty * tiles_x + tx) * nv + g_of
    pos = torch.searchsorted(listed, key).clamp(max=listed.numel() - 1)
    unl = listed[pos] != key
    g_u, tx_u, ty_u = g_of[unl], tx[unl].double(), ty[unl].double()
    kk = torch.arange(16, device=dev, dtype=torch.float64)
    bad = 0
    for c0 in range(0, g_u.numel(), chunk):
        g = g_u[c0:c0 + chunk]
        u, v, A, B = [r0[g, i][:, None, None] for i in range(4)]
        C, Q = [r1[g, i].double()[:, None, None] for i in (0, 1)]
        ii = 16 * tx_u[c0:c0 + chunk, None] + kk[None]
        jj = 16 * ty_u[c0:c0 + chunk, None] + kk[None]
        inx = (ii >= px0[g, None]) & (ii <= px1[g, None]) & (ii < W)
        iny = (jj >= py0[g, None]) & (jj <= py1[g, None]) & (jj < H)
        dx = (ii + 0.5)[:, None, :] - u
        dy = (jj + 0.5)[:, :, None] - v
        q = A * dx * dx + B * dx * dy + C * dy * dy + Q
        err = 9 * 2.0 ** -24 * (A.abs() * dx * dx + B.abs() * (dx * dy).abs() + C.abs() * dy * dy + Q.abs())
        bad += int(((q + err >= 0) & inx[:, None, :] & iny[:, :, None]).sum())
    return bad, int(g_u.numel()), int(g_list.numel())


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_tile_cover_sound_full_size(name):
    """The tile cover (reading R7b, the same definition in the oracle and the
    kernel, so bit-exact lists cannot catch a shared error): at full size, no
    tile of a splat's pixel AABB that the lists omit holds a pixel with
    e2 >= 0 -- checked independently of both, by brute force."""
    scene = fi.make_scene(name, n={"c2": None, "c3": None, "c4": 600_000}[name])
    cam = fi.make_cameras(name)[{"c2": 19, "c3": 13, "c4": 6}[name]]
    sc = fd.Scene.from_arrays(scene)
    r = fd.Renderer(sc, cam.width, cam.height)
    r.render_checked(cam, 0.55)
    bad, omitted, listed = _cover_violations(r.debug_views(), cam.width, cam.height)
    assert bad == 0
    assert listed > 100_000 and omitted > 0.1 * listed     # the cover is tighter than the AABB rectangles
