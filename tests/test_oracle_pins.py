"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Each test names the passage (P:n = PAPER.md line n) or DESIGN.md reading it
follows and the independent fact it checks: closed forms, invariants,
brute force on tiny inputs, or an independent construction (numpy quaternion
products, numpy block-partition conditioning).  No expected value here comes
from the CUDA path.
"""
import math

import numpy as np
import pytest

import fdgs_inputs as fi
import oracle

LN255 = math.log(255.0)


# ----------------------------------------------------------------- helpers
def qmul(a, b):
    """Hamilton product of (w,x,y,z) quaternions (independent of the oracle)."""
    w1, x1, y1, z1 = a
    w2, x2, y2, z2 = b
    return np.array([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2,
                     w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2,
                     w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2])


def rotor_by_products(ql, qr):
    """Matrix of x -> q_l * x * q_r (4D rotation of P:115 as a map), column-wise."""
    R = np.zeros((4, 4))
    for j in range(4):
        e = np.zeros(4)
        e[j] = 1.0
        R[:, j] = qmul(np.asarray(ql, np.float64), qmul(e, np.asarray(qr, np.float64)))
    return R


def cam_axis(width=65, height=65, f=64.0, bg=(0.0, 0.0, 0.0)):
    """Camera at the world origin looking down +z; principal point on a pixel centre."""
    R = np.eye(3)
    T = np.zeros(3)
    c = fi.scenes._cam(width, height, f, R, T, np.zeros(3), bg=bg)
    c.cx = float(np.float32(width / 2.0))
    c.cy = float(np.float32(height / 2.0))
    return c


def pixel_grid(cam):
    j, i = np.mgrid[0:cam.height, 0:cam.width]
    return (i + 0.5).ravel(), (j + 0.5).ravel()


# ------------------------------------------------------------ Sec. 3
def test_rotor_identity_and_hand_expanded():
    assert np.array_equal(oracle.rotor4([1, 0, 0, 0], [1, 0, 0, 0]), np.eye(4))
    c = math.cos(math.pi / 4)
    a, b = np.float32(c), np.float32(c)
    R = oracle.rotor4([a, b, 0, 0], [1, 0, 0, 0])
    a, b = float(a), float(b)
    # left-isoclinic matrix of q = (a,b,0,0), expanded by hand from q*x
    hand = np.array([[a, -b, 0, 0], [b, a, 0, 0], [0, 0, a, -b], [0, 0, b, a]])
    assert np.allclose(R, hand, atol=1e-15)


def test_rotor_matches_quaternion_products_and_is_rotation():
    rng = np.random.default_rng(1)
    for _ in range(1000):
        ql = rng.standard_normal(4); ql /= np.linalg.norm(ql)
        qr = rng.standard_normal(4); qr /= np.linalg.norm(qr)
        ql = ql.astype(np.float32); qr = qr.astype(np.float32)
        R = oracle.rotor4(ql, qr)
        ref = rotor_by_products(ql.astype(np.float64), qr.astype(np.float64))
        assert np.max(np.abs(R - ref)) < 1e-15
        # fp32-rounded unit quaternions: orthogonal to ~1e-7
        assert np.max(np.abs(R @ R.T - np.eye(4))) < 1e-6
        assert abs(np.linalg.det(R) - 1.0) < 1e-6


# ---------------------------------------------------------- Eq. 1
def _conditioning_reference(scene, i, t):
    """Generic Gaussian conditioning by block partition (np.linalg.solve)."""
    R = rotor_by_products(scene.rot_l[i].astype(np.float64), scene.rot_r[i].astype(np.float64))
    s = scene.scale[i].astype(np.float64)
    S4 = R @ np.diag(s * s) @ R.T
    mu = scene.mean[i].astype(np.float64)
    S_bb = S4[3:, 3:]
    S_ab = S4[:3, 3:]
    dt = np.array([float(np.float32(t)) - mu[3]])
    mu3 = mu[:3] + S_ab @ np.linalg.solve(S_bb, dt)
    S3 = S4[:3, :3] - S_ab @ np.linalg.solve(S_bb, S_ab.T)
    return mu3, S3, S4[3, 3]


def test_eq1_conditioning_matches_generic_block_formula():
    scene = fi.make_scene("c1", n=400, seed=3)
    cam = fi.make_cameras("c1")[0]
    for t in (0.0, 0.37, 1.0):
        rec = oracle.records(scene, cam, t)
        idx = np.nonzero(rec["stage"] >= oracle.ST_SUPPORT)[0]
        assert idx.size > 50
        for i in idx:
            mu3, S3, s44 = _conditioning_reference(scene, i, t)
            scale = float(np.max(np.abs(S3))) + 1e-30
            assert abs(rec["s44"][i] - s44) <= 1e-12 * s44
            assert np.max(np.abs(rec["mu3"][i] - mu3)) <= 1e-9 * (1 + np.max(np.abs(mu3)))
            c = rec["cov3"][i]
            got = np.array([[c[0], c[1], c[2]], [c[1], c[3], c[4]], [c[2], c[4], c[5]]])
            assert np.max(np.abs(got - S3)) <= 1e-9 * scale
            assert np.min(np.linalg.eigvalsh(got)) >= -1e-12 * scale


def test_eq1_identity_rotor_and_invariants():
    # identity rotor: mu3 = mu_xyz, Sigma3 = diag(s^2) (zero cross-covariance)
    sc = fi.isotropic_scene([[0.1, -0.2, 0.3, 0.5]], [[0.3, 0.2, 0.1, 0.4]], [0.8])
    cam = fi.make_cameras("c1")[0]
    rec = oracle.records(sc, cam, 0.6)
    s = sc.scale[0].astype(np.float64)
    assert np.array_equal(rec["mu3"][0], sc.mean[0, :3].astype(np.float64))
    c = rec["cov3"][0]
    assert np.allclose([c[0], c[3], c[5]], s[:3] ** 2, rtol=1e-15) and c[1] == c[2] == c[4] == 0.0
    # any rotor: Sigma3 independent of t, mu3 affine in t, mu3 = mu_xyz at t = mu_t
    scene = fi.make_scene("c1", n=200, seed=5)
    ts = [np.float32(0.2), np.float32(0.45), np.float32(0.7)]
    recs = [oracle.records(scene, cam, t) for t in ts]
    ok = (recs[0]["stage"] >= 1) & (recs[1]["stage"] >= 1) & (recs[2]["stage"] >= 1)
    assert ok.sum() > 20
    for a in (1, 2):
        d = np.abs(recs[a]["cov3"][ok] - recs[0]["cov3"][ok])
        assert np.all(d <= 1e-12 * (np.abs(recs[0]["cov3"][ok]).max(1, keepdims=True) + 1e-30))
    slope1 = (recs[1]["mu3"][ok] - recs[0]["mu3"][ok]) / (float(ts[1]) - float(ts[0]))
    slope2 = (recs[2]["mu3"][ok] - recs[1]["mu3"][ok]) / (float(ts[2]) - float(ts[1]))
    assert np.allclose(slope1, slope2, rtol=1e-6, atol=1e-9)
    one = scene.subset([7])
    r = oracle.records(one, cam, one.mean[0, 3])
    if r["stage"][0] >= 1:
        assert np.allclose(r["mu3"][0], one.mean[0, :3].astype(np.float64), atol=1e-15)


# ----------------------------------------------------- Eq. 3
def test_temporal_marginal_closed_forms():
    sc = fi.isotropic_scene([[0, 0, 5.0, 0.5]], [[0.2, 0.2, 0.2, 0.1]], [0.5])
    cam = cam_axis()
    s_t = float(sc.scale[0, 3])
    r = oracle.records(sc, cam, 0.5)
    assert r["amp"][0] == pytest.approx(float(sc.opacity[0]), rel=1e-15)   # p_t(mu_t) = 1
    th = 0.5 + math.sqrt(2 * math.log(2.0)) * s_t                          # half height
    r = oracle.records(sc, cam, np.float32(th))
    dt = float(np.float32(th)) - 0.5
    assert r["amp"][0] == pytest.approx(float(sc.opacity[0]) * math.exp(-dt * dt / (2 * s_t * s_t)), rel=1e-14)
    assert r["amp"][0] / float(sc.opacity[0]) == pytest.approx(0.5, abs=2e-6)


def test_single_isotropic_gaussian_profile_closed_form():
    """North-star pin: one isotropic Gaussian on the axis renders the closed form."""
    bg = (0.1, 0.2, 0.3)
    cam = cam_axis(bg=bg)
    s, z, f, sig = 0.2, 4.0, 64.0, 0.9
    rgb = np.array([0.8, 0.4, 0.1])
    sc = fi.isotropic_scene([[0, 0, z, 0.5]], [[s, s, s, 0.3]], [sig], colors=rgb)
    out = oracle.render(sc, cam, 0.5)
    px, py = pixel_grid(cam)
    s_f = float(sc.scale[0, 0])
    sp2 = (f * s_f / z) ** 2 + 0.3
    rho2 = (px - cam.cx) ** 2 + (py - cam.cy) ** 2
    a_un = float(sc.opacity[0]) * np.exp(-rho2 / (2 * sp2))
    alpha = np.minimum(0.99, a_un)
    c = 0.28209479177387814 * ((rgb - 0.5) / 0.28209479177387814).astype(np.float32).astype(np.float64) + 0.5
    expect = np.where((a_un >= 1 / 255)[:, None], c[None] * alpha[:, None] + (1 - alpha[:, None]) * np.array(bg, np.float32), np.array(bg, np.float32)[None])
    sure = np.abs(a_un * 255 - 1) > 1e-6
    assert sure.sum() > 0.99 * sure.size
    err = np.abs(out["rgb"] - expect)[sure]
    assert err.max() < 1e-12
    assert (a_un >= 1 / 255).sum() > 100              # a real splat, not a dot
    Texp = np.where(a_un >= 1 / 255, 1 - alpha, 1.0)
    assert np.abs(out["T"] - Texp)[sure].max() < 1e-12


def test_temporal_scaling_of_the_image():
    """North-star pin: at several t the image of one Gaussian scales by p_t(t)."""
    cam = cam_axis()
    sc = fi.isotropic_scene([[0, 0, 4.0, 0.5]], [[0.2, 0.2, 0.2, 0.15]], [0.6], colors=[0.9, 0.9, 0.9])
    s_t = float(sc.scale[0, 3])
    base = oracle.render(sc, cam, 0.5)["rgb"][:, 0]
    for t in (0.45, 0.6, 0.7):
        tt = float(np.float32(t))
        pt = math.exp(-(tt - 0.5) ** 2 / (2 * s_t * s_t))
        img = oracle.render(sc, cam, tt)["rgb"][:, 0]
        both = (img > 0) & (base > 0)
        assert both.sum() > 30
        assert np.allclose(img[both] / base[both], pt, rtol=1e-12)
    # beyond the 1/255 marginal: nothing at all
    far = 0.5 + 1.01 * math.sqrt(2 * LN255) * s_t
    assert np.all(oracle.render(sc, cam, far)["rgb"] == 0.0)


def test_marginal_below_threshold_contributes_nothing():
    """North-star pin: sigma*p_t < 1/255 -> exactly background; >= -> a splat."""
    bg = (0.25, 0.5, 0.75)
    cam = cam_axis(bg=bg)
    sc = fi.isotropic_scene([[0, 0, 4.0, 0.5]], [[0.2, 0.2, 0.2, 0.1]], [1.0], colors=[0.9, 0.1, 0.4])
    s_t = float(sc.scale[0, 3])
    tstar = 0.5 + math.sqrt(2 * LN255) * s_t
    t = np.float32(tstar)
    ts = [t]
    a = b = t
    for _ in range(25):
        a = np.nextafter(a, np.float32(0)); b = np.nextafter(b, np.float32(2))
        ts += [a, b]
    bgv = np.array(bg, np.float32).astype(np.float64)
    seen_in = seen_out = 0
    for tt in ts:
        dt = float(tt) - 0.5
        pt = math.exp(-dt * dt / (2 * s_t * s_t))
        img = oracle.render(sc, cam, tt)["rgb"]
        stage = oracle.records(sc, cam, tt)["stage"][0]
        if pt * 255 < 1 - 1e-6:
            assert np.all(img == bgv[None]), tt
            assert stage == oracle.ST_TEMPORAL           # the temporal cull is p_t < 1/255
            seen_out += 1
        elif pt * 255 > 1 + 1e-6:
            assert np.any(img != bgv[None]), tt
            assert stage == oracle.ST_VISIBLE
            seen_in += 1
    assert seen_in > 5 and seen_out > 5


# ---------------------------------------------------- projection
def test_projection_closed_forms():
    cam = cam_axis(width=101, height=81, f=100.0)
    s, z = 0.05, 3.0
    sc = fi.isotropic_scene([[0, 0, z, 0.5]], [[s, s, s, 0.3]], [0.9])
    r = oracle.records(sc, cam, 0.5)
    assert r["u"][0] == pytest.approx(cam.cx, abs=1e-12) and r["v"][0] == pytest.approx(cam.cy, abs=1e-12)
    sf = float(sc.scale[0, 0])
    a, b, c = r["cov2"][0]
    assert a == pytest.approx((100.0 * sf / z) ** 2 + 0.3, rel=1e-14)
    assert c == pytest.approx((100.0 * sf / z) ** 2 + 0.3, rel=1e-14)
    assert abs(b) < 1e-15
    # behind the camera / inside z_near -> near cull
    sc2 = fi.isotropic_scene([[0, 0, -1.0, 0.5], [0, 0, 0.1, 0.5]], [[s, s, s, 0.3]], [0.9])
    assert list(oracle.records(sc2, cam, 0.5)["stage"]) == [oracle.ST_NEAR, oracle.ST_NEAR]


def test_aabb_contains_closed_form_disk():
    cam = cam_axis(width=129, height=129, f=64.0)
    for s, sig in ((0.2, 0.9), (0.5, 0.3), (0.05, 0.99)):
        sc = fi.isotropic_scene([[0, 0, 4.0, 0.5]], [[s, s, s, 0.3]], [sig])
        r = oracle.records(sc, cam, 0.5)
        sf = float(sc.scale[0, 0])
        sp2 = (64.0 * sf / 4.0) ** 2 + 0.3
        rad = math.sqrt(2 * sp2 * math.log(255 * float(sc.opacity[0])))
        px0, px1, py0, py1 = r["rect"][0]
        # every pixel centre inside the alpha >= 1/255 disk lies in the AABB
        assert px0 <= math.ceil(cam.cx - rad - 0.5) and px1 >= math.floor(cam.cx + rad - 0.5)
        # and the margin is small (at most one pixel each side)
        assert px0 >= math.ceil(cam.cx - rad - 0.5) - 1 and px1 <= math.floor(cam.cx + rad - 0.5) + 1
        assert (py0, py1) == (px0, px1)


# -------------------------------------------------------- SH (P:139 c_i(d))
def test_sh_basis_orthonormal_and_pole():
    x, w = np.polynomial.legendre.leggauss(24)
    nphi = 48
    phis = 2 * np.pi * np.arange(nphi) / nphi
    G = np.zeros((16, 16))
    for ct, wt in zip(x, w):
        st = math.sqrt(1 - ct * ct)
        for ph in phis:
            Y = oracle.sh_basis([st * math.cos(ph), st * math.sin(ph), ct])
            G += np.outer(Y, Y) * wt * (2 * np.pi / nphi)
    assert np.max(np.abs(G - np.eye(16))) < 1e-12
    Y = oracle.sh_basis([0.0, 0.0, 1.0])
    assert Y[1] == 0.0 and Y[3] == 0.0 and Y[2] == pytest.approx(math.sqrt(3 / (4 * math.pi)))
    assert Y[0] == pytest.approx(0.5 / math.sqrt(math.pi))


# ----------------------------------------------------- Eq. 2
def _coaxial_scene(n, seed, tie=False):
    rng = np.random.default_rng(seed)
    zs = rng.uniform(2.0, 6.0, n)
    if tie:
        zs[1] = zs[0]
    means = np.stack([np.zeros(n), np.zeros(n), zs, np.full(n, 0.5)], 1)
    ss = rng.uniform(0.1, 0.3, n)
    scales = np.stack([ss, ss, ss, np.full(n, 0.3)], 1)
    ops = rng.uniform(0.2, 0.6, n)
    cols = rng.uniform(0.05, 0.95, (n, 3))
    return fi.isotropic_scene(means, scales, ops, colors=cols), cols


def _literal_eq2(sc, cam, order):
    """I = sum_i c_i a_i prod_{j<i}(1-a_j) + bg prod(1-a) (non-incremental)."""
    px, py = pixel_grid(cam)
    f = cam.fx
    alphas, cols, sure = [], [], np.ones(px.shape, bool)
    for i in order:
        z = float(sc.mean[i, 2])
        s = float(sc.scale[i, 0])
        sp2 = (f * s / z) ** 2 + 0.3
        a_un = float(sc.opacity[i]) * np.exp(-((px - cam.cx) ** 2 + (py - cam.cy) ** 2) / (2 * sp2))
        sure &= np.abs(a_un * 255 - 1) > 1e-6
        alphas.append(np.where(a_un >= 1 / 255, np.minimum(0.99, a_un), 0.0))
        c = 0.28209479177387814 * sc.sh[i, 0].astype(np.float64) + 0.5
        cols.append(np.maximum(c, 0.0))
    out = np.zeros((px.size, 3))
    for k in range(len(order)):
        w = alphas[k].copy()
        for j in range(k):
            w *= 1 - alphas[j]
        out += w[:, None] * cols[k][None]
    Tall = np.ones(px.size)
    for a in alphas:
        Tall *= 1 - a
    out += Tall[:, None] * np.array(cam.bg, np.float32)[None]
    return out, sure


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_compositing_order_brute_force(seed):
    cam = cam_axis(bg=(0.05, 0.1, 0.15))
    n = 8
    sc, _ = _coaxial_scene(n, seed)
    order = list(np.argsort(sc.mean[:, 2].astype(np.float64), kind="stable"))
    ref, sure = _literal_eq2(sc, cam, order)
    got = oracle.render(sc, cam, 0.5)["rgb"]
    assert sure.mean() > 0.99
    assert np.abs(got - ref)[sure].max() < 1e-12
    # swapping an adjacent overlapping pair changes the result
    sw = order.copy()
    sw[3], sw[4] = sw[4], sw[3]
    ref2, _ = _literal_eq2(sc, cam, sw)
    assert np.abs(ref2 - got)[sure].max() > 1e-4


def test_equal_depth_tie_broken_by_index():
    cam = cam_axis()
    sc, _ = _coaxial_scene(3, 7, tie=True)
    assert sc.mean[0, 2] == sc.mean[1, 2]
    others = sorted(range(2, 3), key=lambda i: float(sc.mean[i, 2]))
    # canonical order: ascending (depth, index)
    order = sorted(range(3), key=lambda i: (float(sc.mean[i, 2]), i))
    ref, sure = _literal_eq2(sc, cam, order)
    got = oracle.render(sc, cam, 0.5)["rgb"]
    assert np.abs(got - ref)[sure].max() < 1e-12
    bad = order.copy()
    a, b = bad.index(0), bad.index(1)
    bad[a], bad[b] = bad[b], bad[a]
    ref_bad, _ = _literal_eq2(sc, cam, bad)
    assert np.abs(ref_bad - got)[sure].max() > 1e-4
    assert list(oracle.canonical_order(sc, cam, 0.5)) == order
    del others


def test_termination_knife_edge_records_both_branches():
    """Two alpha=0.99 layers: T(1-a) = 1.0000000000000018e-4 ~ 1e-4 -> both outcomes."""
    cam = cam_axis(bg=(0.2, 0.2, 0.2))
    sc = fi.isotropic_scene([[0, 0, 3.0, 0.5], [0, 0, 5.0, 0.5], [0, 0, 7.0, 0.5]],
                            [[0.3, 0.3, 0.3, 0.3]], [1.0], colors=[[0.9, 0.1, 0.1], [0.1, 0.9, 0.1], [0.1, 0.1, 0.9]])
    k = (cam.height // 2) * cam.width + cam.width // 2
    r = oracle.render(sc, cam, 0.5, pixels=[k])
    c = 0.28209479177387814 * sc.sh[:, 0].astype(np.float64) + 0.5
    bg = np.array(cam.bg, np.float32).astype(np.float64)
    a = 0.99
    T1 = 1 - a
    test2 = T1 * (1 - a)
    assert test2 >= 1e-4 and abs(test2 / 1e-4 - 1) < 1e-3
    primary = c[0] * a + c[1] * a * T1 + test2 * bg          # 3rd layer stops (test < 1e-4)
    alt = c[0] * a + T1 * bg                                  # stop at the 2nd layer
    assert np.allclose(r["rgb"][0], primary, atol=1e-12)
    assert r["n_alt"][0] == 1
    assert np.allclose(r["alt"][0, 0], alt, atol=1e-12)
    assert r["stats"]["knife"] >= 1


# ------------------------------------------------- Sec. 4.2.2
def _golden_keyframes():
    import os
    rows = []
    with open(os.path.join(os.path.dirname(__file__), "golden", "keyframes.txt")) as fh:
        for line in fh:
            if line.startswith("#") or not line.strip():
                continue
            lhs, rhs = line.split("->")
            F, D = map(int, lhs.split())
            rows.append((F, D, [int(x) for x in rhs.split()]))
    return rows


def test_keyframe_schedule_golden():
    for F, D, kf in _golden_keyframes():
        assert list(oracle.keyframes(F, D)) == kf
    kf = oracle.keyframes(300, 20)
    assert len(kf) == 16
    assert oracle.bracket(kf, 0) == (0, 0)
    assert oracle.bracket(kf, 20) == (1, 1)                  # at a key-frame: its own mask
    assert oracle.bracket(kf, 25) == (1, 2)
    assert oracle.bracket(kf, 290) == (14, 15)
    assert oracle.bracket(kf, 299) == (15, 15)


def test_keyframe_mask_union_and_never_visible():
    cams = fi.make_cameras("c3", width=160, height=120, fx=120.0, count=3)
    # G0: visible from the left camera only; G1: never active in time; G2: in front of all
    p0 = cams[0].position
    R0 = cams[0].R.astype(np.float64)
    side = p0 + R0.T @ np.array([-0.64 * 0.5, 0.0, 0.5])    # near, at the left edge of the leftmost camera
    means = [[*side, 0.5], [0.0, 0.0, 7.0, 0.0], [0.0, 0.0, 7.0, 0.5]]
    sc = fi.isotropic_scene(means, [[0.05, 0.05, 0.05, 0.05]], [0.9])
    m_all = oracle.keyframe_mask(sc, cams, 0.5)
    bits = [(int(m_all[0]) >> i) & 1 for i in range(3)]
    per_cam = [[(int(oracle.keyframe_mask(sc, [c], 0.5)[0]) >> i) & 1 for i in range(3)] for c in cams]
    assert bits[1] == 0                                       # never visible -> clear
    assert bits[2] == 1 and all(pc[2] == 1 for pc in per_cam)
    assert bits[0] == 1 and sum(pc[0] for pc in per_cam) >= 1  # union semantics
    assert sum(pc[0] for pc in per_cam) < 3                   # not visible from every camera
    # union = OR of single-camera masks
    ors = np.zeros_like(m_all)
    for c in cams:
        ors |= oracle.keyframe_mask(sc, [c], 0.5)
    assert np.array_equal(ors, m_all)


def test_keyframe_soundness_and_all_ones_mask():
    scene = fi.make_scene("c1", n=600, seed=11)
    cams = fi.make_cameras("c1")
    t_key = np.float32(1.0 / 3.0)
    m = oracle.keyframe_mask(scene, cams, t_key)
    assert 0 < np.unpackbits(m.view(np.uint8)).sum() < scene.n
    a = oracle.render(scene, cams[0], t_key)["rgb"]
    b = oracle.render(scene, cams[0], t_key, mask=m)["rgb"]
    assert np.array_equal(a, b)                               # soundness at the key-frame
    ones = np.full((scene.n + 31) // 32, 0xFFFFFFFF, np.uint32)
    c = oracle.render(scene, cams[0], 0.2, mask=ones)["rgb"]
    d = oracle.render(scene, cams[0], 0.2)["rgb"]
    assert np.array_equal(c, d)                               # all-ones mask == no mask
    zero = np.zeros_like(ones)
    e = oracle.render(scene, cams[0], 0.2, mask=zero)["rgb"]
    assert np.all(e == np.array(cams[0].bg, np.float32)[None])


def test_active_set_union_dominance():
    scene = fi.make_scene("c1", n=300, seed=2)
    cams = fi.make_cameras("c1")
    kf = oracle.keyframes(10, 4)
    masks = np.stack([oracle.keyframe_mask(scene, cams, np.float32(k / 9.0)) for k in kf])
    for f in range(10):
        a = oracle.active_mask(masks, kf, f)
        l, r = oracle.bracket(kf, f)
        assert np.array_equal(a & masks[l], masks[l]) and np.array_equal(a & masks[r], masks[r])
        if l == r:
            assert np.array_equal(a, masks[l])


# ------------------------------------------------------------ tile lists
def _q_exact(f32, i, j):
    """The e2 quadratic in binary64 at pixel centre (i+.5, j+.5) (exact-ish)."""
    u, v, A, B, C, Q = (float(x) for x in f32)
    dx, dy = i + 0.5 - u, j + 0.5 - v
    return A * dx * dx + B * dx * dy + C * dy * dy + Q


def test_tile_lists_brute_force():
    """Tile lists: canonical order, a subset of the
    AABB tiles, covering every pixel whose e2 quadratic is >= 0 (brute force
    over all pixels in binary64), and strictly tighter than the AABB."""
    scene = fi.make_scene("c1", n=500, seed=4)
    cam = fi.make_cameras("c1", width=72, height=56, fx=60.0)[0]
    for t in (0.0, 0.5):
        ranges, ids = oracle.tile_lists(scene, cam, t)
        rec = oracle.records(scene, cam, t)
        order = oracle.canonical_order(scene, cam, t)
        assert np.all(rec["stage"][order] == oracle.ST_VISIBLE)
        tw, th = (cam.width + 15) // 16, (cam.height + 15) // 16
        E_aabb = 0
        for ty in range(th):
            for tx in range(tw):
                x0, x1, y0, y1 = 16 * tx, 16 * tx + 15, 16 * ty, 16 * ty + 15
                aabb = [g for g in order if rec["rect"][g, 0] <= x1 and rec["rect"][g, 1] >= x0
                        and rec["rect"][g, 2] <= y1 and rec["rect"][g, 3] >= y0]
                E_aabb += len(aabb)
                k = ty * tw + tx
                got = list(ids[ranges[k, 0]:ranges[k, 1]])
                assert set(got) <= set(aabb)                          # subset of the AABB tiles
                assert got == [g for g in aabb if g in set(got)]      # canonical order
                for g in aabb:                                        # coverage of every e2 >= 0 pixel
                    if g in set(got):
                        continue
                    px0, px1, py0, py1 = rec["rect"][g]
                    for j in range(max(y0, py0), min(y1, py1) + 1):
                        for i in range(max(x0, px0), min(x1, px1) + 1):
                            assert _q_exact(rec["f32"][g], i, j) < -1e-6, (g, i, j)
        assert ids.size < E_aabb                                       # the cover is tighter than the AABB
        # canonical order = ascending (depth bits, index)
        keys = [(int(rec["depth_bits"][g]), int(g)) for g in order]
        assert keys == sorted(keys)


def test_band_tiles_closed_form():
    """An axis-aligned isotropic splat: the cover of each band is the set of
    tiles the closed-form disc (radius sqrt(-Q2/A')) reaches, inflated by the
    margin only."""
    cam = fi.make_cameras("c1", width=129, height=129, fx=64.0)[0]
    cam.cx = cam.cy = 64.5
    sc = fi.isotropic_scene([[0, 0, 0.0, 0.5]], [[0.6, 0.6, 0.6, 0.3]], [0.9])
    rec = oracle.records(sc, cam, 0.5)
    f32 = rec["f32"][0]
    u, v, A = float(f32[0]), float(f32[1]), float(f32[2])
    Q = float(f32[5])
    r = math.sqrt(-Q / A)                                  # e2 >= 0 disc radius (pixels)
    px0, px1, py0, py1 = rec["rect"][0]
    for ty in range(py0 // 16, py1 // 16 + 1):
        band = oracle.band_tiles(f32, rec["rect"][0], ty)
        ja, jb = max(16 * ty, py0), min(16 * ty + 15, py1)
        dy = min(abs(ja + 0.5 - v), abs(jb + 0.5 - v)) if not (ja + 0.5 <= v <= jb + 0.5) else 0.0
        if dy > r + 0.05:
            assert band is None
            continue
        assert band is not None
        half = math.sqrt(max(r * r - dy * dy, 0.0))
        lo, hi = math.ceil(u - half - 0.5), math.floor(u + half - 0.5)
        lo, hi = max(lo, px0), min(hi, px1)
        if lo <= hi:
            assert band[0] <= lo // 16 and band[1] >= hi // 16         # covers the disc's columns
        assert band[0] >= (lo - 2) // 16 and band[1] <= (hi + 2) // 16  # and not much more


def test_vq_sh_decode_equals_materialised_codebook():
    """Ours-PP storage (vector quantisation of SH): rendering a scene
    whose SH are codebook entries sh_index[i] gives exactly the image of the
    dense scene with sh_i = codebook[sh_index[i]] (the decode is a lookup)."""
    scene = fi.make_scene("c1", n=400, seed=11)
    vq = fi.vq_scene(scene, codebook_size=37, seed=2)
    dense = fi.SceneArrays(vq.mean, vq.scale, vq.rot_l, vq.rot_r, vq.opacity, vq.log255_opacity,
                           np.ascontiguousarray(vq.sh[vq.sh_index.astype(np.int64)]))
    cam = fi.make_cameras("c1")[0]
    a = oracle.render(scene=vq, cam=cam, t=0.5)
    b = oracle.render(scene=dense, cam=cam, t=0.5)
    assert np.array_equal(a["rgb"], b["rgb"]) and a["stats"]["n_vis"] > 50
    # a one-entry codebook: every visible Gaussian gets the same rgb at a fixed direction
    one = fi.vq_scene(scene, codebook_size=1, seed=3)
    assert np.all(one.sh_index == 0)
    rec = oracle.records(one, cam, 0.5)
    assert np.isfinite(rec["rgb"]).all()
