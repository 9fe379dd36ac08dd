"""Scene / camera / timestamp generators for the BASELINE.json configs.

Recipe:

* one ``numpy.random.default_rng(seed)`` (PCG64) per scene, seed 0 unless
  overridden, with the fixed draw order
  mean-xyz -> mu_t -> log-scale-xyz -> log-scale-t -> q_l -> q_r ->
  opacity-logit -> SH DC (N x 3) -> SH rest (N x 15 x 3);
* activation in float64 (exp for scales, sigmoid for opacity, quaternion
  normalisation), then a cast to float32 (the canonical scene arrays);
* ``log255_opacity`` L_i = fp32(ln(255 * sigma_i)) evaluated in float64 from
  the fp32 sigma.  It is a derived *input* field of the C-ABI scene
  (include/fdgs.h ``fdgs_scene``), supplied identically to both sides.

The N3V / D-NeRF datasets are not in this container; these synthetic scenes
take their shapes (resolution, frame count, camera rig) and BASELINE.json's
distributions.  No dataset content is reproduced.
"""
from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np


@dataclass
class SceneArrays:
    """Canonical fp32 SoA scene (torch-compatible shapes)."""

    mean: np.ndarray      # (N,4) x,y,z,t
    scale: np.ndarray     # (N,4) linear std-devs (>0)
    rot_l: np.ndarray     # (N,4) unit quaternion (w,x,y,z)
    rot_r: np.ndarray     # (N,4) unit quaternion (w,x,y,z)
    opacity: np.ndarray   # (N,)  sigma in (0,1]
    log255_opacity: np.ndarray  # (N,) fp32(ln(255 sigma)) computed in fp64
    sh: np.ndarray        # (N,16,3) degree-3 SH, coefficient index k*3+c; (K,16,3) codebook if sh_index
    sh_index: np.ndarray | None = None  # (N,) uint16 VQ codebook entry per Gaussian (Ours-PP)

    @property
    def n(self) -> int:
        return int(self.mean.shape[0])

    def subset(self, idx) -> "SceneArrays":
        idx = np.asarray(idx, dtype=np.int64)
        if self.sh_index is None:
            return SceneArrays(*(np.ascontiguousarray(getattr(self, f)[idx]) for f in _FIELDS))
        return SceneArrays(*(np.ascontiguousarray(getattr(self, f)[idx]) for f in _FIELDS[:-1]), self.sh,
                           np.ascontiguousarray(self.sh_index[idx]))

    def arrays(self):
        d = {f: getattr(self, f) for f in _FIELDS}
        if self.sh_index is not None:
            d["sh_index"] = self.sh_index
        return d


_FIELDS = ("mean", "scale", "rot_l", "rot_r", "opacity", "log255_opacity", "sh")


@dataclass
class Camera:
    """Pinhole camera, world->camera (OpenCV axes: x right, y down, z fwd)."""

    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    R: np.ndarray                      # (3,3) float32 row-major, world->cam
    T: np.ndarray                      # (3,)  float32
    z_near: float = 0.2
    bg: tuple = (0.0, 0.0, 0.0)
    position: np.ndarray = field(default=None, repr=False)  # float64 centre (info only)


# --------------------------------------------------------------------------
# BASELINE.json configs (index 0..4 -> c1..c5); sizes are the full sizes.
CONFIGS = {
    "c1": dict(n=1000, layout="cube1", log_s_xyz=(-3.0, 0.5), log_s_t=(-2.0, 0.5),
               rig="c1", width=64, height=64, fx=64.0, frames=4, keyframe_interval=None),
    "c2": dict(n=100_000, layout="ball1.5", log_s_xyz=(-3.0, 0.5), log_s_t=(-2.0, 0.5),
               rig="hemisphere50", width=800, height=800, fx=1111.0, frames=150,
               keyframe_interval=10),
    "c3": dict(n=200_000, layout="n3v", log_s_xyz=(-3.0, 0.5), log_s_t=(-1.0, 0.5),
               rig="arc20", width=1352, height=1014, fx=1000.0, frames=300,
               keyframe_interval=20),
    "c4": dict(n=3_000_000, layout="n3v", log_s_xyz=(-3.0, 0.5), log_s_t=(-3.0, 0.7),
               rig="arc20", width=1352, height=1014, fx=1000.0, frames=300,
               keyframe_interval=20),
}


def _sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def make_scene(name: str, n: int | None = None, seed: int = 0) -> SceneArrays:
    """Draw the scene of config ``name`` (optionally with fewer Gaussians)."""
    cfg = CONFIGS[name]
    n = int(cfg["n"] if n is None else n)
    rng = np.random.default_rng(seed)
    layout = cfg["layout"]
    # 1. mean xyz
    if layout == "cube1":
        xyz = rng.uniform(-1.0, 1.0, size=(n, 3))
    elif layout == "ball1.5":
        d = rng.standard_normal(size=(n, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        r = 1.5 * rng.uniform(0.0, 1.0, size=(n, 1)) ** (1.0 / 3.0)
        xyz = d * r
    elif layout == "n3v":
        u = rng.uniform(0.0, 1.0, size=(n, 3))
        xyz = np.stack([-5.0 + 10.0 * u[:, 0], -3.0 + 6.0 * u[:, 1], 2.0 + 10.0 * u[:, 2]], 1)
    else:
        raise ValueError(layout)
    # 2. mu_t
    mt = rng.uniform(0.0, 1.0, size=(n, 1))
    # 3./4. log-scales
    ls_xyz = rng.normal(cfg["log_s_xyz"][0], cfg["log_s_xyz"][1], size=(n, 3))
    ls_t = rng.normal(cfg["log_s_t"][0], cfg["log_s_t"][1], size=(n, 1))
    # 5./6. quaternions ~ normalised N(0, I4), (w,x,y,z)
    ql = rng.standard_normal(size=(n, 4))
    qr = rng.standard_normal(size=(n, 4))
    ql /= np.linalg.norm(ql, axis=1, keepdims=True)
    qr /= np.linalg.norm(qr, axis=1, keepdims=True)
    # 7. opacity logit
    op = _sigmoid(rng.standard_normal(size=n))
    # 8./9. SH: DC ~ N(0.5,0.2), rest ~ N(0,0.2)
    dc = rng.normal(0.5, 0.2, size=(n, 1, 3))
    rest = rng.normal(0.0, 0.2, size=(n, 15, 3))
    return _finish(np.concatenate([xyz, mt], 1), np.exp(np.concatenate([ls_xyz, ls_t], 1)),
                   ql, qr, op, np.concatenate([dc, rest], 1))


def _finish(mean, scale, ql, qr, op, sh) -> SceneArrays:
    f32 = lambda a: np.ascontiguousarray(np.asarray(a, dtype=np.float64).astype(np.float32))
    op32 = f32(op)
    op32 = np.clip(op32, np.float32(1e-7), np.float32(1.0))
    L = f32(np.log(255.0 * op32.astype(np.float64)))
    return SceneArrays(f32(mean), f32(scale), f32(ql), f32(qr), op32, L, f32(sh))


def isotropic_scene(means, scales, opacities, colors=None, rot_l=None, rot_r=None, sh=None) -> SceneArrays:
    """Hand-built scene for pins: identity rotors unless given, DC colour.

    ``colors`` are the *target* rgb of a degree-0 SH (sh0 = (rgb-0.5)/C0).
    """
    means = np.atleast_2d(np.asarray(means, dtype=np.float64))
    n = means.shape[0]
    scales = np.broadcast_to(np.asarray(scales, dtype=np.float64), (n, 4))
    ops = np.broadcast_to(np.asarray(opacities, dtype=np.float64), (n,))
    ql = np.tile([1.0, 0, 0, 0], (n, 1)) if rot_l is None else np.asarray(rot_l, np.float64)
    qr = np.tile([1.0, 0, 0, 0], (n, 1)) if rot_r is None else np.asarray(rot_r, np.float64)
    if sh is None:
        sh = np.zeros((n, 16, 3))
        if colors is not None:
            c0 = 0.28209479177387814
            sh[:, 0, :] = (np.broadcast_to(np.asarray(colors, np.float64), (n, 3)) - 0.5) / c0
    return _finish(means, scales, ql, qr, ops, sh)


# --------------------------------------------------------------------------
def look_at(position, target, down=(0.0, 1.0, 0.0)):
    """World->camera (R, T) in float64 for OpenCV axes (z toward target)."""
    p = np.asarray(position, np.float64)
    z = np.asarray(target, np.float64) - p
    z /= np.linalg.norm(z)
    d = np.asarray(down, np.float64)
    y = d - np.dot(d, z) * z
    y /= np.linalg.norm(y)
    x = np.cross(y, z)
    R = np.stack([x, y, z], 0)
    T = -R @ p
    return R, T


def _cam(width, height, fx, R, T, pos, z_near=0.2, bg=(0.0, 0.0, 0.0)):
    return Camera(width=int(width), height=int(height), fx=float(np.float32(fx)),
                  fy=float(np.float32(fx)), cx=float(np.float32(width / 2.0)),
                  cy=float(np.float32(height / 2.0)), R=np.asarray(R, np.float64).astype(np.float32),
                  T=np.asarray(T, np.float64).astype(np.float32), z_near=float(np.float32(z_near)),
                  bg=tuple(float(np.float32(b)) for b in bg), position=np.asarray(pos, np.float64))


def make_cameras(name: str, width: int | None = None, height: int | None = None,
                 fx: float | None = None, count: int | None = None) -> list:
    """The camera rig of config ``name``; resolution/focal may be scaled for tests."""
    cfg = CONFIGS[name]
    W = cfg["width"] if width is None else width
    H = cfg["height"] if height is None else height
    f = cfg["fx"] if fx is None else fx
    rig = cfg["rig"]
    cams = []
    if rig == "c1":
        cams.append(_cam(W, H, f, np.eye(3), [0.0, 0.0, 4.0], [0.0, 0.0, -4.0]))
    elif rig == "hemisphere50":
        n = 50 if count is None else count
        golden = math.pi * (3.0 - math.sqrt(5.0))
        for i in range(n):
            h = (i + 0.5) / n                 # height fraction in (0,1): avoids the pole
            rxz = math.sqrt(1.0 - h * h)
            ang = golden * i
            pos = 4.0 * np.array([rxz * math.cos(ang), -h, rxz * math.sin(ang)])  # upper = -y
            R, T = look_at(pos, [0.0, 0.0, 0.0])
            cams.append(_cam(W, H, f, R, T, pos))
    elif rig == "arc20":
        n = 20 if count is None else count
        centre = np.array([0.0, 0.0, 7.0])
        half = 0.5 / 7.0                       # 1 m of arc on a radius-7 circle
        for i in range(n):
            th = -half + (2.0 * half) * (i / (n - 1) if n > 1 else 0.5)
            pos = centre + 7.0 * np.array([math.sin(th), 0.0, -math.cos(th)])
            R, T = look_at(pos, centre)
            cams.append(_cam(W, H, f, R, T, pos))
    else:
        raise ValueError(rig)
    return cams


def frame_times(frames: int) -> np.ndarray:
    """t_f = f/(F-1) as float32 (BASELINE config 1 uses t in {0,1/3,2/3,1})."""
    if frames == 1:
        return np.zeros(1, np.float32)
    return (np.arange(frames, dtype=np.float64) / (frames - 1)).astype(np.float32)


def scene_sha256(s: SceneArrays) -> dict:
    return {k: hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest()[:16]
            for k, v in s.arrays().items()}


def vq_scene(scene: SceneArrays, codebook_size: int = 4096, seed: int = 1) -> SceneArrays:
    """The scene with vector-quantised SH storage (the "Ours-PP" decode input,
    P:483): a codebook of ``codebook_size`` SH entries drawn with the scene's
    SH distribution (DC ~ N(0.5, 0.2), rest ~ N(0, 0.2)) and a uniform uint16
    entry index per Gaussian.  Synthetic stand-in: the codebook is not fitted
    to the scene (fitting is compression-time work, out of scope)."""
    if not 1 <= codebook_size <= 65536:
        raise ValueError("codebook_size must lie in [1, 65536]")
    rng = np.random.default_rng(seed)
    dc = rng.normal(0.5, 0.2, size=(codebook_size, 1, 3))
    rest = rng.normal(0.0, 0.2, size=(codebook_size, 15, 3))
    book = np.ascontiguousarray(np.concatenate([dc, rest], 1).astype(np.float32))
    idx = rng.integers(0, codebook_size, size=scene.n).astype(np.uint16)
    return SceneArrays(scene.mean, scene.scale, scene.rot_l, scene.rot_r, scene.opacity, scene.log255_opacity,
                       book, idx)
