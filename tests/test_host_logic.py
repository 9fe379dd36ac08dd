"""Host logic of the product path (no GPU): key-frame schedule and bracketing
(readings R4/R5) against the golden schedules, and the input
generator's recipe."""
import os

import numpy as np
import pytest

import fdgs_inputs as fi
from paper_2503_16422_b200 import api


def _golden():
    rows = []
    with open(os.path.join(os.path.dirname(__file__), "golden", "keyframes.txt")) as fh:
        for line in fh:
            if line.startswith("#") or not line.strip():
                continue
            lhs, rhs = line.split("->")
            F, D = map(int, lhs.split())
            rows.append((F, D, [int(x) for x in rhs.split()]))
    return rows


def test_keyframes_golden():
    for F, D, kf in _golden():
        assert api.keyframes(F, D) == kf
    with pytest.raises(ValueError):
        api.keyframes(10, 0)


def test_bracket_rules():
    kf = api.keyframes(300, 20)
    for f in range(300):
        l, r = api.bracket(kf, f)
        assert kf[l] <= f <= kf[r]
        assert r - l in (0, 1)
        assert (l == r) == (f in kf)


def test_generator_recipe_and_determinism():
    a = fi.make_scene("c3", n=5000)
    b = fi.make_scene("c3", n=5000)
    assert fi.scene_sha256(a) == fi.scene_sha256(b)
    assert a.mean.dtype == np.float32 and a.sh.shape == (5000, 16, 3)
    assert np.all(a.mean[:, 0] >= -5) and np.all(a.mean[:, 0] <= 5)
    assert np.all(a.mean[:, 2] >= 2) and np.all(a.mean[:, 2] <= 12)
    nq = np.linalg.norm(a.rot_l.astype(np.float64), axis=1)
    assert np.all(np.abs(nq - 1) < 1e-6)
    assert np.all((a.opacity > 0) & (a.opacity <= 1))
    L = np.log(255.0 * a.opacity.astype(np.float64)).astype(np.float32)
    assert np.array_equal(L, a.log255_opacity)
    # log-scale_t ~ N(-1, 0.5) for c3
    assert abs(np.log(a.scale[:, 3]).mean() + 1.0) < 0.05
    cams = fi.make_cameras("c3")
    assert len(cams) == 20 and cams[0].width == 1352 and cams[0].height == 1014
    for c in cams:
        R = c.R.astype(np.float64)
        assert np.max(np.abs(R @ R.T - np.eye(3))) < 1e-6
    t = fi.frame_times(4)
    assert np.allclose(t, [0, 1 / 3, 2 / 3, 1])
    c2 = fi.make_cameras("c2")
    assert len(c2) == 50 and all(np.linalg.norm(c.position) == pytest.approx(4.0) for c in c2)


def test_alpha_clamp_premultiply_identity_exhaustive():
    """The blend computes alpha = min(0.99, 2^e2 / 255) (Eq. 2 with the 0.99
    clamp, reading R6) as fl(min(x, c) * k) with k = fl(1/255) and
    c = 0x437c7332 (render.cu kAlphaPre).  Exhaustive over every float32 x in
    [128, 256) (2^e2 < 256 since e2 <= log2 255), where the clamp can engage;
    below 128, x k < 0.99 on both sides."""
    k = np.float32(1.0) / np.float32(255.0)
    c = np.uint32(0x437C7332).view(np.float32)
    lo, hi = np.float32(128.0).view(np.uint32), np.float32(256.0).view(np.uint32)
    x = np.arange(lo, hi, dtype=np.uint32).view(np.float32)
    want = np.minimum(np.float32(0.99), (x * k).astype(np.float32))
    got = (np.minimum(x, c) * k).astype(np.float32)
    assert np.array_equal(want.view(np.uint32), got.view(np.uint32))
