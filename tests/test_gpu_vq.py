"""GPU parity of the vector-quantised SH decode (the "Ours-PP" storage of
P:483) through the C-ABI: the render reads each visible
Gaussian's SH from a codebook entry instead of its own 192-byte record.
Bars as tests/test_gpu_render.py: decisions, records and tile lists bit-exact,
RGB within max-abs 2e-4 / mean-abs 1e-5 of the oracle."""
import numpy as np
import pytest
import torch

import fdgs_inputs as fi
import oracle
import paper_2503_16422_b200 as fd
from paper_2503_16422_b200 import _lib

from parity import assert_records_bit_exact, assert_rgb_parity, assert_tile_lists_bit_exact

pytestmark = pytest.mark.gpu


def _render(scene, cam, t, ml=None, mr=None):
    sc = fd.Scene.from_arrays(scene)
    r = fd.Renderer(sc, cam.width, cam.height)
    out, stats = r.render_checked(cam, t, ml, mr)
    return out.cpu().numpy(), stats, r


@pytest.mark.parametrize("k", [1, 256, 4096])
def test_vq_reduced_c3_parity(k):
    scene = fi.vq_scene(fi.make_scene("c3", n=20_000), codebook_size=k, seed=5)
    cam = fi.make_cameras("c3", width=338, height=254, fx=250.0, count=5)[2]
    t = float(np.float32(0.4))
    img, stats, r = _render(scene, cam, t)
    views = r.debug_views()
    assert_records_bit_exact(views, scene, cam, t)
    assert_tile_lists_bit_exact(views, scene, cam, t)
    orc = oracle.render(scene, cam, t)
    assert_rgb_parity(img, orc)
    assert stats.n_vis == orc["stats"]["n_vis"] > 100


def test_vq_equals_dense_materialised_bit_exact():
    """Same CUDA path, SH read through the codebook vs materialised per
    Gaussian: identical images bit for bit (the decode is a lookup)."""
    vq = fi.vq_scene(fi.make_scene("c2", n=30_000), codebook_size=512, seed=9)
    dense = fi.SceneArrays(vq.mean, vq.scale, vq.rot_l, vq.rot_r, vq.opacity, vq.log255_opacity,
                           np.ascontiguousarray(vq.sh[vq.sh_index.astype(np.int64)]))
    cam = fi.make_cameras("c2", width=400, height=400, fx=555.0, count=7)[3]
    a, _, _ = _render(vq, cam, 0.5)
    b, _, _ = _render(dense, cam, 0.5)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_vq_full_size_c3_masked_sampled():
    """BASELINE configs[2] size with the bench's VQ variant (K = 4096)."""
    base = fi.make_scene("c3")
    scene = fi.vq_scene(base, codebook_size=4096, seed=1)
    cams = fi.make_cameras("c3")
    times = fi.frame_times(300)
    kf = fd.keyframes(300, 20)
    l, r = fd.bracket(kf, 130)
    sc = fd.Scene.from_arrays(scene)
    ml = fd.keyframe_mask(sc, cams, float(times[kf[l]]))
    mr = fd.keyframe_mask(sc, cams, float(times[kf[r]]))
    active = ml.cpu().numpy().view(np.uint32) | mr.cpu().numpy().view(np.uint32)
    cam = cams[12]
    t = float(times[130])
    img, stats, rd = _render(scene, cam, t, ml, mr)
    assert_records_bit_exact(rd.debug_views(), scene, cam, t, active)
    pix = np.unique(np.random.default_rng(1).integers(0, cam.width * cam.height, 3000))
    orc = oracle.render(scene, cam, t, mask=active, pixels=pix)
    assert_rgb_parity(img, orc, pixels=pix)


def test_vq_index_out_of_range_is_rejected():
    scene = fi.vq_scene(fi.make_scene("c1", n=100), codebook_size=8, seed=1)
    idx = scene.sh_index.copy()
    idx[57] = 8
    bad = fi.SceneArrays(scene.mean, scene.scale, scene.rot_l, scene.rot_r, scene.opacity, scene.log255_opacity,
                         scene.sh, idx)
    st, first = fd.validate(fd.Scene.from_arrays(bad))
    assert st == _lib.FDGS_ERR_INVALID_SCENE and first == 57
    st, first = fd.validate(fd.Scene.from_arrays(scene))
    assert st == _lib.FDGS_OK
