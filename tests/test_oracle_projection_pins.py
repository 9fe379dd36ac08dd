"""Pins of the oracle's off-axis projection and colour (-m "not gpu").

P:139 (Sec. 3, text after Eq. 3): the conditional 3D Gaussian is projected
to a 2D Gaussian with covariance Sigma_2D (EWA splatting, readings R6/R13) and
coloured by its view-dependent SH colour c_i(d) (readings R9/R10).  The
oracle builds Sigma_2D from a hand-written Jacobian J and the camera rotation
R_c (oracle/fdgs_oracle.c or_gauss_eval); these tests rebuild every quantity
from a construction that shares none of that code:

* the pixel position by the pinhole formula on the world->camera transform;
* Sigma_2D = J_w Sigma_3 J_w^T + 0.3 I, where J_w is the COMPLEX-STEP
  derivative of the world->pixel map X -> pi(R_c X + T_c) (exact to rounding:
  pi is analytic, so Im pi(X + i h e_k) / h is the derivative with no
  cancellation), evaluated at the world point whose camera-space image has
  x/z, y/z clamped to +-1.3 tan(fov/2) (reading R6, the EWA clamp);
* the conic as numpy's matrix inverse of Sigma_2D;
* the pixel AABB against the closed-form extent of {d^T Sigma_2D^-1 d <= 2Q};
* the view direction from the generator's float64 camera centre
  (Camera.position), and the SH basis from scipy's complex spherical harmonics
  (Condon-Shortley phase) turned real: sqrt2 Re Y_l^m (m > 0), Y_l^0,
  sqrt2 Im Y_l^|m| (m < 0) -- the sign convention of reading R9.

Cameras: the C2 hemisphere rig (50 rotated cameras) and the C3 arc rig, on
>= 1000 off-axis Gaussians each, with the clamp exercised by Gaussians outside
the field of view.  No expected value comes from the CUDA path.
"""
import math

import numpy as np
import pytest
import scipy.special as sps

import fdgs_inputs as fi
import oracle

RIGS = {
    # config: (scene n, camera indices, timestamps); "c3a": the C3 arc rig with
    # anamorphic intrinsics (fy = 0.7 fx) and an off-centre principal point
    "c2": (8000, [0, 5, 9, 17, 23, 31, 41, 47], [0.25, 0.6]),
    "c3": (6000, [0, 11, 19], [0.3, 0.7]),
    "c3a": (6000, [2, 14], [0.3, 0.7]),
}


def anamorphic(cam):
    """fy = 0.7 fx, principal point at (0.43 W, 0.58 H) (reading R13 allows any)."""
    cam.fy = float(np.float32(0.7 * cam.fx))
    cam.cx = float(np.float32(0.43 * cam.width))
    cam.cy = float(np.float32(0.58 * cam.height))
    return cam


def _projected(name):
    """(scene, cam, t, rec, idx) with idx the Gaussians that reach the
    projection (stage COVER or VISIBLE: Sigma_2D and (u, v) are defined)."""
    n, cam_ids, ts = RIGS[name]
    base = "c3" if name == "c3a" else name
    scene = fi.make_scene(base, n=n, seed=21)
    cams = fi.make_cameras(base)
    if name == "c3a":
        cams = [anamorphic(c) for c in cams]
    for c in cam_ids:
        for t in ts:
            t32 = float(np.float32(t))
            rec = oracle.records(scene, cams[c], t32)
            idx = np.nonzero(rec["stage"] >= oracle.ST_COVER)[0]
            yield scene, cams[c], t32, rec, idx


def _pix_map(cam, X):
    """World points (..., 3), real or complex -> pixel (u, v) by the pinhole model."""
    R = cam.R.astype(np.float64)
    T = cam.T.astype(np.float64)
    p = X @ R.T + T
    return cam.fx * p[..., 0] / p[..., 2] + cam.cx, cam.fy * p[..., 1] / p[..., 2] + cam.cy


def _clamped_world_point(cam, X):
    """The world point whose camera-space image is X's with x/z and y/z clamped
    to +-1.3 W/(2 fx), +-1.3 H/(2 fy) (the EWA Jacobian clamp, reading R6)."""
    R = cam.R.astype(np.float64)
    T = cam.T.astype(np.float64)
    p = X @ R.T + T
    limx = 1.3 * cam.width / (2.0 * cam.fx)
    limy = 1.3 * cam.height / (2.0 * cam.fy)
    z = p[:, 2]
    pc = np.stack([np.clip(p[:, 0] / z, -limx, limx) * z, np.clip(p[:, 1] / z, -limy, limy) * z, z], 1)
    clamped = (np.abs(p[:, 0] / z) > limx) | (np.abs(p[:, 1] / z) > limy)
    # R^-1 (p - T) (R is float32-rounded, so R^T is not its exact inverse)
    return np.linalg.solve(R, (pc - T).T).T, clamped


def _complex_step_jacobian(cam, X):
    """J_w[i] = d(u, v)/dX at X[i] (2x3), by the complex step (h = 1e-30)."""
    h = 1e-30
    J = np.zeros((X.shape[0], 2, 3))
    for k in range(3):
        Xc = X.astype(np.complex128)
        Xc[:, k] += 1j * h
        u, v = _pix_map(cam, Xc)
        J[:, 0, k] = u.imag / h
        J[:, 1, k] = v.imag / h
    return J


def _cov3(rec, idx):
    c = rec["cov3"][idx]
    return np.stack([np.stack([c[:, 0], c[:, 1], c[:, 2]], 1),
                     np.stack([c[:, 1], c[:, 3], c[:, 4]], 1),
                     np.stack([c[:, 2], c[:, 4], c[:, 5]], 1)], 1)


@pytest.mark.parametrize("name", ["c2", "c3", "c3a"])
def test_pixel_position_is_the_pinhole_image(name):
    seen = 0
    for scene, cam, t, rec, idx in _projected(name):
        u, v = _pix_map(cam, rec["mu3"][idx])
        assert np.all(np.abs(rec["u"][idx] - u) <= 1e-9 * np.maximum(1.0, np.abs(u)))
        assert np.all(np.abs(rec["v"][idx] - v) <= 1e-9 * np.maximum(1.0, np.abs(v)))
        # camera-space depth (the depth key, "sorted by their depth")
        z = (rec["mu3"][idx] @ cam.R.astype(np.float64).T + cam.T.astype(np.float64))[:, 2]
        assert np.all(np.abs(rec["z"][idx] - z) <= 1e-12 * np.abs(z))
        seen += idx.size
    assert seen >= 1000


@pytest.mark.parametrize("name", ["c2", "c3", "c3a"])
def test_sigma2d_is_the_complex_step_ewa_projection(name):
    """Sigma_2D = J_w Sigma_3 J_w^T + 0.3 I (R6) to 1e-9 relative, with
    the Jacobian clamp exercised; the unclamped Jacobian would differ there."""
    seen = clamped_seen = 0
    for scene, cam, t, rec, idx in _projected(name):
        Xc, clamped = _clamped_world_point(cam, rec["mu3"][idx])
        J = _complex_step_jacobian(cam, Xc)
        S2 = J @ _cov3(rec, idx) @ np.transpose(J, (0, 2, 1)) + 0.3 * np.eye(2)
        a, b, c = rec["cov2"][idx].T
        scale = np.maximum(np.abs(S2[:, 0, 0]), np.abs(S2[:, 1, 1]))
        assert np.all(np.abs(a - S2[:, 0, 0]) <= 1e-9 * scale)
        assert np.all(np.abs(b - S2[:, 0, 1]) <= 1e-9 * scale)
        assert np.all(np.abs(c - S2[:, 1, 1]) <= 1e-9 * scale)
        # conic = Sigma_2D^-1 (power = 0.5 (A dx^2 + 2B dx dy + C dy^2))
        inv = np.linalg.inv(S2)
        A, B, C = rec["conic"][idx].T
        iscale = np.maximum(np.abs(inv[:, 0, 0]), np.abs(inv[:, 1, 1]))
        assert np.all(np.abs(A - inv[:, 0, 0]) <= 1e-9 * iscale)
        assert np.all(np.abs(B - inv[:, 0, 1]) <= 1e-9 * iscale)
        assert np.all(np.abs(C - inv[:, 1, 1]) <= 1e-9 * iscale)
        if clamped.any():  # the clamp is what the oracle applies: the raw Jacobian differs
            Jr = _complex_step_jacobian(cam, rec["mu3"][idx][clamped])
            S2r = Jr @ _cov3(rec, idx)[clamped] @ np.transpose(Jr, (0, 2, 1)) + 0.3 * np.eye(2)
            d = np.abs(S2r[:, 0, 0] - a[clamped]) + np.abs(S2r[:, 1, 1] - c[clamped])
            assert np.median(d / scale[clamped]) > 1e-3
        seen += idx.size
        clamped_seen += int(clamped.sum())
    assert seen >= 1000 and clamped_seen >= 50, (seen, clamped_seen)


@pytest.mark.parametrize("name", ["c2", "c3", "c3a"])
def test_pixel_aabb_contains_the_alpha_ellipse(name):
    """The pixel AABB of a splat (reading R7) covers the closed-form extent of
    {power <= Q} = {d^T Sigma_2D^-1 d <= 2Q}, half-widths sqrt(2Q Sigma_2D,xx)
    (from the independent Sigma_2D), with at most one pixel of margin."""
    seen = 0
    for scene, cam, t, rec, idx in _projected(name):
        vis = idx[rec["stage"][idx] == oracle.ST_VISIBLE]
        Xc, _ = _clamped_world_point(cam, rec["mu3"][vis])
        J = _complex_step_jacobian(cam, Xc)
        S2 = J @ _cov3(rec, vis) @ np.transpose(J, (0, 2, 1)) + 0.3 * np.eye(2)
        u, v = _pix_map(cam, rec["mu3"][vis])
        Q = rec["Q"][vis]
        hx, hy = np.sqrt(2 * Q * S2[:, 0, 0]), np.sqrt(2 * Q * S2[:, 1, 1])
        lo_x = np.maximum(np.ceil(u - hx - 0.5), 0)
        hi_x = np.minimum(np.floor(u + hx - 0.5), cam.width - 1)
        lo_y = np.maximum(np.ceil(v - hy - 0.5), 0)
        hi_y = np.minimum(np.floor(v + hy - 0.5), cam.height - 1)
        px0, px1, py0, py1 = rec["rect"][vis].T
        inside = (lo_x <= hi_x) & (lo_y <= hi_y)
        assert np.all(px0[inside] <= lo_x[inside]) and np.all(px1[inside] >= hi_x[inside])
        assert np.all(py0[inside] <= lo_y[inside]) and np.all(py1[inside] >= hi_y[inside])
        assert np.all(px0[inside] >= lo_x[inside] - 1) and np.all(px1[inside] <= hi_x[inside] + 1)
        seen += int(inside.sum())
    assert seen >= 500


def _real_sh_scipy(d):
    """Degree-3 real SH from scipy's complex SH with the Condon-Shortley phase:
    k = l^2 + l + m; sqrt2 Re Y_l^m (m > 0), Y_l^0, sqrt2 Im Y_l^|m| (m < 0)."""
    x, y, z = d
    polar = math.acos(max(-1.0, min(1.0, z)))
    azim = math.atan2(y, x)
    out = np.zeros(16)
    for l in range(4):
        for m in range(-l, l + 1):
            Y = complex(sps.sph_harm_y(l, abs(m), polar, azim))
            out[l * l + l + m] = (math.sqrt(2) * Y.real if m > 0 else Y.real if m == 0
                                  else math.sqrt(2) * Y.imag)
    return out


def test_sh_basis_equals_scipy_real_sh():
    """Reading R9's sign convention, pinned to an independent library: the
    oracle's closed-form basis equals scipy's complex SH turned real."""
    rng = np.random.default_rng(5)
    for _ in range(300):
        d = rng.standard_normal(3)
        d /= np.linalg.norm(d)
        assert np.max(np.abs(oracle.sh_basis(d) - _real_sh_scipy(d))) < 1e-12
    for d in ([1.0, 0, 0], [0, 1.0, 0], [0, 0, -1.0]):
        assert np.max(np.abs(oracle.sh_basis(d) - _real_sh_scipy(d))) < 1e-12


@pytest.mark.parametrize("name", ["c2", "c3", "c3a"])
def test_view_dependent_colour_from_the_camera_centre(name):
    """c_i(d) with d = (mu3 - C)/|mu3 - C|, C the generator's float64
    camera centre (reading R10), rgb = max(0, sum_k Y_k(d) sh_k + 0.5) with the
    scipy basis.  The tolerance covers the float32 rounding of R, T (the
    oracle derives C = -R^T T from them)."""
    seen = 0
    for scene, cam, t, rec, idx in _projected(name):
        vis = idx[rec["stage"][idx] == oracle.ST_VISIBLE][:150]
        for i in vis:
            d = rec["mu3"][i] - cam.position
            d /= np.linalg.norm(d)
            Y = _real_sh_scipy(d)
            rgb = np.maximum(Y @ scene.sh[i].astype(np.float64) + 0.5, 0.0)
            assert np.max(np.abs(rec["rgb"][i] - rgb)) < 2e-5, i
        seen += vis.size
    assert seen >= 500
