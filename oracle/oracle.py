"""ctypes wrapper of oracle/liboracle.so (TEST INFRASTRUCTURE ONLY; see __init__)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "fdgs_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")
MAX_LEAVES = 4
ST_TEMPORAL, ST_SUPPORT, ST_NEAR, ST_COVER, ST_VISIBLE = range(5)

_lock = threading.Lock()
_lib = None


def build_oracle(force: bool = False) -> str:
    """Compile the oracle with gcc (-ffp-contract=off, no fast-math)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp",
                               "-ffp-contract=off", "-fno-fast-math", "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB)
    return LIB


class _Scene(C.Structure):
    _fields_ = [("n", C.c_int32), ("mean", C.c_void_p), ("scale", C.c_void_p),
                ("rot_l", C.c_void_p), ("rot_r", C.c_void_p), ("opacity", C.c_void_p),
                ("log255_opacity", C.c_void_p), ("sh", C.c_void_p), ("sh_index", C.c_void_p)]


class _Camera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("R", C.c_float * 9), ("T", C.c_float * 3),
                ("z_near", C.c_float), ("bg", C.c_float * 3)]


def load():
    global _lib
    with _lock:
        if _lib is None:
            # ORACLE_LIB: a mutated build (tools/mutate_oracle.py checks that the
            # pins kill every mutant); default the in-tree liboracle.so
            alt = os.environ.get("ORACLE_LIB")
            if not alt:
                build_oracle()
            lib = C.CDLL(alt or LIB)
            P = C.c_void_p
            lib.or_records.argtypes = [P, P, C.c_float, P, P, P, P, P]
            lib.or_render.argtypes = [P, P, P, C.c_float, P, C.c_int64, P, P, P, P, P]
            lib.or_render.restype = C.c_int
            lib.or_canonical_order.argtypes = [P, P, P, C.c_float, P, C.c_int32]
            lib.or_canonical_order.restype = C.c_int
            lib.or_tile_lists.argtypes = [P, P, P, C.c_float, P, P, C.c_int64]
            lib.or_tile_lists.restype = C.c_int64
            lib.or_keyframe_mask.argtypes = [P, P, C.c_int32, C.c_float, P]
            lib.or_keyframe_mask_contrib.argtypes = [P, P, C.c_int32, C.c_float, C.c_double, P]
            lib.or_prune_mask.argtypes = [P, C.c_int32, C.c_int64, P]
            lib.or_keyframes.argtypes = [C.c_int32, C.c_int32, P]
            lib.or_keyframes.restype = C.c_int
            lib.or_bracket.argtypes = [P, C.c_int32, C.c_int32, P, P]
            lib.or_mask_or.argtypes = [P, P, C.c_int32, P]
            lib.or_rotor4.argtypes = [P, P, P]
            lib.or_sh_basis.argtypes = [P, P]
            lib.or_band_consts.argtypes = [P, C.c_int, C.c_int, C.c_int, C.c_int, P]
            lib.or_band_tiles.argtypes = [P, C.c_int, C.c_int, C.c_int, C.c_int, P, C.c_int, P, P]
            lib.or_band_tiles.restype = C.c_int
            lib.or_num_threads.restype = C.c_int
            lib.or_set_num_threads.argtypes = [C.c_int]
            lib.or_contrib.argtypes = [P, P, C.c_float, P]
            lib.or_stv_score.argtypes = [P, P, C.c_int32, P, C.c_int32, C.c_double, P, P, P, P, C.c_int, C.c_int]
            lib.or_tv_p1.argtypes = [C.c_double, C.c_double, C.c_double]
            lib.or_tv_p1.restype = C.c_double
            lib.or_tv.argtypes = [C.c_double, C.c_double, C.c_double]
            lib.or_tv.restype = C.c_double
            lib.or_sigma_t.argtypes = [P, C.c_int]
            lib.or_sigma_t.restype = C.c_double
            _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


class _SceneRef:
    """Keeps contiguous arrays alive while the struct is used."""

    def __init__(self, scene):
        self.arrs = [np.ascontiguousarray(getattr(scene, f), dtype=np.float32) for f in
                     ("mean", "scale", "rot_l", "rot_r", "opacity", "log255_opacity", "sh")]
        idx = getattr(scene, "sh_index", None)
        self.idx = None if idx is None else np.ascontiguousarray(idx, dtype=np.uint16)
        self.s = _Scene(int(scene.mean.shape[0]), *[a.ctypes.data for a in self.arrs],
                        None if self.idx is None else self.idx.ctypes.data)


def _cam(cam):
    c = _Camera()
    c.width, c.height = int(cam.width), int(cam.height)
    c.fx, c.fy, c.cx, c.cy = cam.fx, cam.fy, cam.cx, cam.cy
    c.R[:] = [float(x) for x in np.asarray(cam.R, np.float32).reshape(9)]
    c.T[:] = [float(x) for x in np.asarray(cam.T, np.float32).reshape(3)]
    c.z_near = cam.z_near
    c.bg[:] = [float(b) for b in cam.bg]
    return c


def _mask(mask):
    return None if mask is None else np.ascontiguousarray(mask, dtype=np.uint32)


def records(scene, cam, t):
    """Per-Gaussian decision records (mask not applied)."""
    lib = load()
    sr = _SceneRef(scene)
    n = sr.s.n
    stage = np.zeros(n, np.int32)
    rect = np.zeros((n, 4), np.int32)
    depth = np.zeros(n, np.uint32)
    f32 = np.zeros((n, 6), np.float32)
    f64 = np.zeros((n, 26), np.float64)
    c = _cam(cam)
    lib.or_records(C.byref(sr.s), C.byref(c), float(t), stage.ctypes.data, rect.ctypes.data,
                   depth.ctypes.data, f32.ctypes.data, f64.ctypes.data)
    return dict(stage=stage, rect=rect, depth_bits=depth, f32=f32, mu3=f64[:, 0:3],
                cov3=f64[:, 3:9], s44=f64[:, 9], Q=f64[:, 10], amp=f64[:, 11],
                rgb=f64[:, 12:15], cam=f64[:, 15:18], z=f64[:, 17], u=f64[:, 18], v=f64[:, 19],
                cov2=f64[:, 20:23], conic=f64[:, 23:26])


def render(scene, cam, t, mask=None, pixels=None):
    """Per-pixel Eq. 2 render.  Returns dict with rgb (P,3) primary, T (P,),
    alt (P,MAX_LEAVES,3) alternatives (NaN where absent), n_alt (P,), stats."""
    lib = load()
    sr = _SceneRef(scene)
    c = _cam(cam)
    m = _mask(mask)
    if pixels is None:
        P = cam.width * cam.height
        pix = None
    else:
        pix = np.ascontiguousarray(pixels, dtype=np.int64)
        P = pix.shape[0]
    rgb = np.zeros((P, 3), np.float64)
    T = np.zeros(P, np.float64)
    alt = np.zeros((P, MAX_LEAVES, 3), np.float64)
    n_alt = np.zeros(P, np.int32)
    stats = np.zeros(5, np.int64)
    lib.or_render(C.byref(sr.s), _ptr(m), C.byref(c), float(t), _ptr(pix), P,
                  rgb.ctypes.data, T.ctypes.data, alt.ctypes.data, n_alt.ctypes.data, stats.ctypes.data)
    return dict(rgb=rgb, T=T, alt=alt, n_alt=n_alt,
                stats=dict(n_act=int(stats[0]), n_vis=int(stats[1]), evaluated=int(stats[2]),
                           blended=int(stats[3]), knife=int(stats[4])))


def render_image(scene, cam, t, mask=None):
    """Full frame as CHW float64 (primary branch)."""
    r = render(scene, cam, t, mask)
    return r["rgb"].reshape(cam.height, cam.width, 3).transpose(2, 0, 1).copy(), r


def canonical_order(scene, cam, t, mask=None):
    lib = load()
    sr = _SceneRef(scene)
    c = _cam(cam)
    out = np.zeros(max(sr.s.n, 1), np.int32)
    nv = lib.or_canonical_order(C.byref(sr.s), _ptr(_mask(mask)), C.byref(c), float(t),
                                out.ctypes.data, out.shape[0])
    return out[:nv].copy()


def tile_lists(scene, cam, t, mask=None, cap=None):
    """(ranges (T,2) int64, ids (E,) int32 Gaussian indices) in canonical order."""
    lib = load()
    sr = _SceneRef(scene)
    c = _cam(cam)
    nt = ((cam.width + 15) // 16) * ((cam.height + 15) // 16)
    ranges = np.zeros((nt, 2), np.int64)
    m = _mask(mask)
    E = lib.or_tile_lists(C.byref(sr.s), _ptr(m), C.byref(c), float(t), ranges.ctypes.data, None, 0)
    ids = np.zeros(max(E, 1), np.int32)
    E2 = lib.or_tile_lists(C.byref(sr.s), _ptr(m), C.byref(c), float(t), ranges.ctypes.data,
                           ids.ctypes.data, ids.shape[0])
    assert E2 == E
    return ranges, ids[:E].copy()


def band_tiles(f32, rect, ty):
    """Tile cover of one Gaussian in tile row ty: (txa, txb) or None."""
    lib = load()
    f = np.ascontiguousarray(f32, np.float32)
    a, b = C.c_int(), C.c_int()
    bc = np.zeros(5, np.float64)
    r = [int(x) for x in rect]
    lib.or_band_consts(f.ctypes.data, r[0], r[1], r[2], r[3], bc.ctypes.data)
    ok = lib.or_band_tiles(f.ctypes.data, r[0], r[1], r[2], r[3], bc.ctypes.data, int(ty), C.byref(a), C.byref(b))
    return (a.value, b.value) if ok else None


def keyframe_mask(scene, cams, t_key):
    lib = load()
    sr = _SceneRef(scene)
    arr = (_Camera * len(cams))(*[_cam(c) for c in cams])
    out = np.zeros((sr.s.n + 31) // 32, np.uint32)
    lib.or_keyframe_mask(C.byref(sr.s), arr, len(cams), float(t_key), out.ctypes.data)
    return out


def keyframe_mask_contrib(scene, cams, t_key, threshold=0.0):
    """Paper-literal key-frame mask: union over views of {i : sum of
    Gaussian i's blending weights in the view's render at t_key > threshold}."""
    lib = load()
    sr = _SceneRef(scene)
    arr = (_Camera * len(cams))(*[_cam(c) for c in cams])
    out = np.zeros(max((sr.s.n + 31) // 32, 1), np.uint32)
    lib.or_keyframe_mask_contrib(C.byref(sr.s), arr, len(cams), float(t_key), float(threshold), out.ctypes.data)
    return out[:(sr.s.n + 31) // 32]


def prune_mask(score, keep):
    """bitmask of the `keep` highest scores (ties by ascending index)."""
    lib = load()
    sc = np.ascontiguousarray(score, np.float32)
    n = sc.shape[0]
    out = np.zeros(max((n + 31) // 32, 1), np.uint32)
    lib.or_prune_mask(sc.ctypes.data, n, int(keep), out.ctypes.data)
    return out[:(n + 31) // 32]


def keyframes(frames, interval):
    lib = load()
    out = np.zeros(frames + 1, np.int32)
    k = lib.or_keyframes(int(frames), int(interval), out.ctypes.data)
    return out[:k].copy()


def bracket(kf, frame):
    lib = load()
    kf = np.ascontiguousarray(kf, np.int32)
    l, r = C.c_int32(), C.c_int32()
    lib.or_bracket(kf.ctypes.data, kf.shape[0], int(frame), C.byref(l), C.byref(r))
    return l.value, r.value


def active_mask(masks, kf, frame):
    """Active set of frame = M(t_l) | M(t_r)."""
    lib = load()
    l, r = bracket(kf, frame)
    a = np.ascontiguousarray(masks[l], np.uint32)
    b = np.ascontiguousarray(masks[r], np.uint32)
    out = np.zeros_like(a)
    lib.or_mask_or(a.ctypes.data, b.ctypes.data, a.shape[0] * 32, out.ctypes.data)
    return out


def rotor4(ql, qr):
    lib = load()
    a = np.ascontiguousarray(ql, np.float32)
    b = np.ascontiguousarray(qr, np.float32)
    out = np.zeros(16, np.float64)
    lib.or_rotor4(a.ctypes.data, b.ctypes.data, out.ctypes.data)
    return out.reshape(4, 4)


def sh_basis(d):
    lib = load()
    d = np.ascontiguousarray(d, np.float64)
    out = np.zeros(16, np.float64)
    lib.or_sh_basis(d.ctypes.data, out.ctypes.data)
    return out


def contrib(scene, cam, t):
    """Per-Gaussian sum of blending weights of one view at t."""
    lib = load()
    sr = _SceneRef(scene)
    out = np.zeros(max(sr.s.n, 1), np.float64)
    lib.or_contrib(C.byref(sr.s), C.byref(_cam(cam)), float(t), out.ctypes.data)
    return out[:sr.s.n]


def stv_score(scene, cams, ts, percentile=0.9, combine=0, variant=0):
    """Spatial-temporal variation score: dict(score, spatial, tv, gamma).
    combine 0 = time-aligned sum_t S^T S^S (R20), 1 = product of the sums;
    variant 0 full, 1 S^S only, 2 S^T only, 3 S^TV from p1, 4 Sigma_t."""
    lib = load()
    sr = _SceneRef(scene)
    n = sr.s.n
    ts = np.ascontiguousarray(ts, np.float32)
    arr = (_Camera * len(cams))(*[_cam(c) for c in cams])
    score = np.zeros(max(n, 1))
    spatial = np.zeros((len(ts), max(n, 1)))
    tv = np.zeros((len(ts), max(n, 1)))
    gamma = np.zeros(max(n, 1))
    lib.or_stv_score(C.byref(sr.s), arr, len(cams), ts.ctypes.data, len(ts), float(percentile), score.ctypes.data,
                     spatial.ctypes.data, tv.ctypes.data, gamma.ctypes.data, int(combine), int(variant))
    return dict(score=score[:n], spatial=spatial[:, :n], tv=tv[:, :n], gamma=gamma[:n])


def tv_value(t, mu_t, sigma_t, order=2):
    """S^TV of one Gaussian at t from p2 (order 2) or p1 (order 1)."""
    f = load().or_tv if order == 2 else load().or_tv_p1
    return float(f(float(t), float(mu_t), float(sigma_t)))


def num_threads():
    return int(load().or_num_threads())


def set_num_threads(n):
    """OpenMP threads of the oracle (bench.py's single-core baseline)."""
    load().or_set_num_threads(int(n))
