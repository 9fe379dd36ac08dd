"""Pins of the oracle's spatial-temporal variation score (Sec. 4.2.1,
P:241-273) against closed forms, finite differences and
hand-evaluated examples (SPEC S:234-263 ideas).  -m "not gpu"."""
import math

import numpy as np
import pytest

import fdgs_inputs as fi
import oracle


def cam_axis(width=33, height=33, f=32.0):
    c = fi.scenes._cam(width, height, f, np.eye(3), np.zeros(3), np.zeros(3))
    c.cx = float(np.float32(width / 2.0))
    c.cy = float(np.float32(height / 2.0))
    return c


def test_spatial_score_full_cover_is_alpha_times_pixels():
    """One huge splat with sigma = 1: alpha = 0.99 (clamp) at every pixel ->
    S^S = 0.99 * W * H (P:251 with a single Gaussian: prod over j<i is empty)."""
    cam = cam_axis(8, 8, 8.0)
    sc = fi.isotropic_scene([[0, 0, 4.0, 0.5]], [[200.0, 200.0, 200.0, 0.3]], [1.0])
    c = oracle.contrib(sc, cam, 0.5)
    assert c[0] == pytest.approx(0.99 * 64, rel=1e-9)


def test_spatial_score_two_coaxial_layers_closed_form():
    """Front alpha_f(p), back alpha_b(p): S_f = sum alpha_f, S_b = sum alpha_b (1 - alpha_f)."""
    cam = cam_axis(33, 33, 32.0)
    s = 1.5
    sc = fi.isotropic_scene([[0, 0, 4.0, 0.5], [0, 0, 8.0, 0.5]], [[s, s, s, 0.3]], [0.5])
    c = oracle.contrib(sc, cam, 0.5)
    j, i = np.mgrid[0:33, 0:33]
    rho2 = (i + 0.5 - cam.cx) ** 2 + (j + 0.5 - cam.cy) ** 2
    op = float(sc.opacity[0])
    sf = float(sc.scale[0, 0])
    a = []
    for z in (4.0, 8.0):
        sp2 = (32.0 * sf / z) ** 2 + 0.3
        au = op * np.exp(-rho2 / (2 * sp2))
        a.append(np.where(au >= 1 / 255, np.minimum(0.99, au), 0.0))
    assert c[0] == pytest.approx(a[0].sum(), rel=1e-9)
    assert c[1] == pytest.approx((a[1] * (1 - a[0])).sum(), rel=1e-9)


def test_temporal_variation_closed_forms_and_finite_difference():
    # inflection points t = mu +- sqrt(Sigma_t): p2 = 0 -> S^TV = 2
    assert oracle.tv_value(0.5 + math.sqrt(0.04), 0.5, 0.04) == pytest.approx(2.0, abs=1e-12)
    # Sigma_t = 0.01 at t = mu: |p2| = 1/Sigma_t = 100 -> S^TV ~ 1
    assert oracle.tv_value(0.5, 0.5, 0.01) == pytest.approx(1.0, abs=1e-12)
    # long lifespan: |p2| = 1/Sigma_t -> 0 -> S^TV -> 2
    assert oracle.tv_value(0.5, 0.5, 1e6) == pytest.approx(2.0, abs=1e-5)
    # p2 against a central finite difference of p(t) = exp(-(t-mu)^2 / 2 Sigma)
    rng = np.random.default_rng(0)
    for _ in range(50):
        mu, st, t = rng.uniform(0, 1), rng.uniform(0.01, 0.3), rng.uniform(0, 1)
        p = lambda x: math.exp(-(x - mu) ** 2 / (2 * st))
        h = 1e-4
        p2 = (p(t + h) - 2 * p(t) + p(t - h)) / (h * h)
        want = 1.0 / (0.5 * math.tanh(abs(p2)) + 0.5)
        assert oracle.tv_value(t, mu, st) == pytest.approx(want, rel=1e-5, abs=1e-6)


def test_volume_normalisation_percentile():
    cam = cam_axis()
    # volumes 1..100 (s = (v,1,1,1)): nearest-rank 90th percentile = 90
    means = [[3.0, 3.0, 50.0 + k, 0.5] for k in range(100)]        # far off-screen: no spatial term needed
    scales = [[float(k + 1), 1.0, 1.0, 1.0] for k in range(100)]
    sc = fi.isotropic_scene(means, scales, [0.5])
    r = oracle.stv_score(sc, [cam], [0.5])
    g = r["gamma"]
    assert g[44] == pytest.approx(45.0 / 90.0, rel=1e-12)
    assert g[99] == 1.0 and g[89] == 1.0
    # identical volumes -> all 1
    sc2 = fi.isotropic_scene(means[:10], [[0.1, 0.2, 0.3, 0.4]], [0.5])
    assert np.all(oracle.stv_score(sc2, [cam], [0.5])["gamma"] == 1.0)


def test_combined_score_time_aligned_and_absorbing_zero():
    scene = fi.make_scene("c1", n=300, seed=21)
    cams = fi.make_cameras("c1")
    ts = np.float32([0.0, 0.5, 1.0])
    r = oracle.stv_score(scene, cams, ts)
    want = (r["tv"] * r["gamma"][None] * r["spatial"]).sum(0)
    assert np.allclose(r["score"], want, rtol=1e-12, atol=0)
    assert np.all(r["tv"] >= 1.0) and np.all(r["tv"] <= 2.0)          # S^TV in (1, 2] (tanh saturates to 1 in fp64)
    zero = r["spatial"].sum(0) == 0.0
    assert zero.any() and np.all(r["score"][zero] == 0.0)            # spatial 0 -> score 0
    # per-t spatial term = the sum over views of the per-view contributions
    c0 = sum(oracle.contrib(scene, c, ts[1]) for c in cams)
    assert np.allclose(r["spatial"][1], c0, rtol=1e-12)
    # weights of a pixel sum to 1 - T: total over Gaussians = sum (1 - T)
    out = oracle.render(scene, cams[0], ts[1])
    assert oracle.contrib(scene, cams[0], ts[1]).sum() == pytest.approx((1 - out["T"]).sum(), rel=1e-9)


def test_combine_modes_closed_form_long_lifespan_full_cover():
    """One splat covering the whole image with sigma = 1 and a huge temporal
    scale: p_t ~ 1 and |p2| ~ 1/Sigma_t ~ 0, so S^TV(t) = 2 - O(1e-12) and
    S^S(t) = 0.99 W H at every t.  With gamma = 1 (a single Gaussian is its own
    percentile) and n_t timestamps:
      time-aligned (R20):   S = sum_t 2 * 0.99 W H           = 2 n_t 0.99 W H
      product of the sums:  S = (sum_t 2) (sum_t 0.99 W H)   = 2 n_t^2 0.99 W H."""
    cam = cam_axis(8, 8, 8.0)
    sc = fi.isotropic_scene([[0, 0, 4.0, 0.5]], [[200.0, 200.0, 200.0, 1e6]], [1.0])
    ts = np.float32([0.0, 0.25, 0.5, 1.0])
    a = oracle.stv_score(sc, [cam], ts, combine=0)
    b = oracle.stv_score(sc, [cam], ts, combine=1)
    assert a["gamma"][0] == 1.0
    assert a["score"][0] == pytest.approx(2 * 4 * 0.99 * 64, rel=1e-9)
    assert b["score"][0] == pytest.approx(2 * 16 * 0.99 * 64, rel=1e-9)


def _bits(words, n):
    return np.unpackbits(np.asarray(words, np.uint32).view(np.uint8), bitorder="little")[:n].astype(bool)


def test_contribution_keyframe_mask_pins():
    """Paper-literal m_{i,j}: Gaussians whose blending
    weights in the view-j render sum above a threshold, unioned over views."""
    # 1. full-cover splat: S = 0.99 W H -> set just below, clear just above
    cam = cam_axis(8, 8, 8.0)
    sc = fi.isotropic_scene([[0, 0, 4.0, 0.5]], [[200.0, 200.0, 200.0, 0.3]], [1.0])
    s = 0.99 * 64
    assert _bits(oracle.keyframe_mask_contrib(sc, [cam], 0.5, s - 1e-6), 1)[0]
    assert not _bits(oracle.keyframe_mask_contrib(sc, [cam], 0.5, s + 1e-6), 1)[0]
    # 2. occlusion: two opaque full-cover layers drive T to 1e-4 before the
    #    third Gaussian -> geometrically visible (the geometric mask of R3 sets
    #    it) but it receives no blending weight (clear in the literal mask)
    sc3 = fi.isotropic_scene([[0, 0, 4.0, 0.5], [0, 0, 5.0, 0.5], [0, 0, 6.0, 0.5]],
                             [[200.0, 200.0, 200.0, 0.3]], [1.0])
    geo = _bits(oracle.keyframe_mask(sc3, [cam], 0.5), 3)
    lit = _bits(oracle.keyframe_mask_contrib(sc3, [cam], 0.5, 0.0), 3)
    assert geo.tolist() == [True, True, True] and lit.tolist() == [True, True, False]
    # 3. random scene: literal (threshold 0) subset of geometric, union over
    #    views, monotone in the threshold
    scene = fi.make_scene("c2", n=1500, seed=4)
    cams = fi.make_cameras("c2", width=48, height=48, fx=66.0, count=3)
    n = scene.n
    g = _bits(oracle.keyframe_mask(scene, cams, 0.5), n)
    m0 = _bits(oracle.keyframe_mask_contrib(scene, cams, 0.5, 0.0), n)
    assert m0.sum() > 100 and np.all(g[m0])
    per_view = [_bits(oracle.keyframe_mask_contrib(scene, [c], 0.5, 0.0), n) for c in cams]
    assert np.array_equal(m0, np.logical_or.reduce(per_view))
    m1 = _bits(oracle.keyframe_mask_contrib(scene, cams, 0.5, 0.5), n)
    m2 = _bits(oracle.keyframe_mask_contrib(scene, cams, 0.5, 5.0), n)
    assert np.all(m0[m1]) and np.all(m1[m2]) and m2.sum() < m1.sum() < m0.sum()
    # per-view threshold (not the sum over views): a Gaussian is set iff some
    # single view's sum exceeds it
    c = np.stack([oracle.contrib(scene, cc, 0.5) for cc in cams])
    assert np.array_equal(m1, (c > 0.5).any(0))


def test_score_ablation_variants_closed_forms():
    """Variants of Table ablation_score on the full-cover splat
    (S^S = 0.99 W H at every t, gamma = 1):
      long lifespan (Sigma_t = 1e12): S^TV(p2) = S^TV(p1) = 2;
      short lifespan (Sigma_t = 0.01) at t = mu_t: p1 = 0 -> S^TV(p1) = 2,
      |p2| = 1/Sigma_t = 100 -> S^TV(p2) = 1."""
    cam = cam_axis(8, 8, 8.0)
    W = 0.99 * 64
    sc = fi.isotropic_scene([[0, 0, 4.0, 0.5]], [[200.0, 200.0, 200.0, 1e6]], [1.0])
    ts = np.float32([0.0, 0.5, 1.0])
    n = len(ts)
    v = lambda variant, combine=0: oracle.stv_score(sc, [cam], ts, variant=variant, combine=combine)["score"][0]
    assert v(0) == pytest.approx(2 * W * n, rel=1e-9)
    assert v(1) == pytest.approx(W * n, rel=1e-12)               # S^S only
    assert v(2) == pytest.approx(2 * n, rel=1e-9)                # S^T only
    assert v(3) == pytest.approx(2 * W * n, rel=1e-9)            # p1
    assert v(4) == pytest.approx(1e12 * W * n, rel=1e-6)         # Sigma_t
    assert v(1, 1) == pytest.approx(n * W * n, rel=1e-12)        # (sum_t 1)(sum_t S^S)
    sc2 = fi.isotropic_scene([[0, 0, 4.0, 0.5]], [[200.0, 200.0, 200.0, 0.1]], [1.0])
    t = np.float32([0.5])
    assert oracle.tv_value(0.5, 0.5, 0.01, order=1) == pytest.approx(2.0, abs=1e-12)
    assert oracle.tv_value(0.5, 0.5, 0.01, order=2) == pytest.approx(1.0, abs=1e-12)
    s0 = oracle.stv_score(sc2, [cam], t, variant=0)
    s3 = oracle.stv_score(sc2, [cam], t, variant=3)
    assert s3["score"][0] == pytest.approx(2.0 * s0["score"][0], rel=1e-6)


def test_prune_mask_ranking_rule():
    """keep the highest scores; equal scores ranked by ascending index
    (reading R23).  Hand example, the edges keep = 0 / n, and a brute-force
    check against numpy's stable argsort on tie-heavy scores."""
    s = np.float32([0.5, 2.0, 0.5, 3.0, 0.5, 1.0])
    m = _bits(oracle.prune_mask(s, 3), 6)
    assert m.tolist() == [False, True, False, True, False, True]
    m = _bits(oracle.prune_mask(s, 4), 6)      # one of the three 0.5s: the lowest index
    assert m.tolist() == [True, True, False, True, False, True]
    assert not _bits(oracle.prune_mask(s, 0), 6).any() and _bits(oracle.prune_mask(s, 6), 6).all()
    rng = np.random.default_rng(3)
    s = np.round(rng.random(5000) * 20).astype(np.float32)   # many ties
    for keep in (1, 777, 2500, 4999):
        want = np.zeros(5000, bool)
        want[np.argsort(-s, kind="stable")[:keep]] = True
        assert np.array_equal(_bits(oracle.prune_mask(s, keep), 5000), want)
