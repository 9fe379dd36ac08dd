"""ctypes view of libfdgs.so (include/fdgs.h).  Argument marshalling only."""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfdgs.so")

FDGS_OK = 0
FDGS_ERR_INVALID_ARG = 1
FDGS_ERR_INVALID_SCENE = 2
FDGS_ERR_WORKSPACE_TOO_SMALL = 3
FDGS_ERR_OVERFLOW = 4
FDGS_ERR_CUDA = 5
FDGS_ERR_UNSUPPORTED = 6

# every symbol include/fdgs.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "fdgs_status_string", "fdgs_last_error", "fdgs_abi_version",
    "fdgs_scene_validate", "fdgs_scene_validate_workspace_bytes", "fdgs_log255_opacity",
    "fdgs_render_workspace_bytes", "fdgs_render", "fdgs_render_timed", "fdgs_render_split", "fdgs_render_checked",
    "fdgs_render_debug_views", "fdgs_render_graph_create", "fdgs_render_graph_launch", "fdgs_render_graph_destroy",
    "fdgs_render_graph_launch_split",
    "fdgs_render_graph_launch_timed",
    "fdgs_keyframe_workspace_bytes", "fdgs_keyframe_mask", "fdgs_mask_or",
    "fdgs_keyframe_mask_contrib_workspace_bytes", "fdgs_keyframe_mask_contrib",
    "fdgs_mask_compact_workspace_bytes", "fdgs_mask_compact", "fdgs_stv_workspace_bytes", "fdgs_stv_score",
    "fdgs_scene_compact_workspace_bytes", "fdgs_scene_compact", "fdgs_prune_workspace_bytes", "fdgs_prune_mask",
    "fdgs_pipeline_create", "fdgs_pipeline_render", "fdgs_pipeline_destroy", "fdgs_debug_strip_reach",
]


class FdgsScene(C.Structure):
    _fields_ = [("n", C.c_int32), ("mean", C.c_void_p), ("scale", C.c_void_p), ("rot_l", C.c_void_p),
                ("rot_r", C.c_void_p), ("opacity", C.c_void_p), ("log255_opacity", C.c_void_p),
                ("sh", C.c_void_p), ("sh_index", C.c_void_p), ("sh_codebook_size", C.c_int32),
                ("param_stride", C.c_int32), ("gid", C.c_void_p), ("n_capacity", C.c_int32),
                ("d_n", C.c_void_p)]


class FdgsCamera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("R", C.c_float * 9), ("T", C.c_float * 3),
                ("z_near", C.c_float), ("bg", C.c_float * 3)]


class FdgsFrameStats(C.Structure):
    _fields_ = [("n_act", C.c_uint32), ("n_vis", C.c_uint32), ("n_entries", C.c_uint32), ("status", C.c_uint32),
                ("n_evaluated", C.c_uint64), ("n_blended", C.c_uint64)]


class FdgsDebugViews(C.Structure):
    _fields_ = [("rec0", C.c_void_p), ("rec1", C.c_void_p), ("rec2", C.c_void_p), ("depth", C.c_void_p),
                ("vis", C.c_void_p), ("order", C.c_void_p), ("tile_start", C.c_void_p), ("entries", C.c_void_p),
                ("counters", C.c_void_p), ("n_tiles", C.c_int32)]


class FdgsPipelineSlot(C.Structure):
    _fields_ = [("d_ws", C.c_void_p), ("ws_bytes", C.c_size_t), ("max_entries", C.c_int64),
                ("front_stream", C.c_void_p), ("blend_stream", C.c_void_p), ("graph", C.c_void_p)]


class FdgsFrameJob(C.Structure):
    _fields_ = [("scene", FdgsScene), ("d_mask_l", C.c_void_p), ("d_mask_r", C.c_void_p), ("cam", FdgsCamera),
                ("t", C.c_float), ("d_out_rgb", C.c_void_p), ("d_out_T", C.c_void_p), ("d_stats", C.c_void_p),
                ("h_out_rgb", C.c_void_p), ("d_status", C.c_void_p), ("done_event", C.c_void_p)]


class FdgsStvOpts(C.Structure):
    _fields_ = [("volume_percentile", C.c_double), ("combine_mode", C.c_int32), ("variant", C.c_int32),
                ("max_entries", C.c_int64)]


class FdgsError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"fdgs status {status}: {msg}")
        self.status = status


_lock = threading.Lock()
_lib = None
ABI_VERSION = 2            # include/fdgs.h FDGS_ABI_VERSION this binding's structs follow
CHECK_ABI = True           # tools/ loading older A/B variant libraries turn this off


def lib():
    """Load libfdgs.so.  There is no fallback: a missing library is an error."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2503_16422_b200.build` "
                              "(the render path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        P, I32, I64, SZ, F = C.c_void_p, C.c_int32, C.c_int64, C.c_size_t, C.c_float
        sig = {
            "fdgs_status_string": ([C.c_int], C.c_char_p),
            "fdgs_last_error": ([], C.c_char_p),
            "fdgs_abi_version": ([], I32),
            "fdgs_scene_validate": ([P, P, P, SZ, P], C.c_int),
            "fdgs_scene_validate_workspace_bytes": ([], SZ),
            "fdgs_log255_opacity": ([P, I32, P, P], C.c_int),
            "fdgs_render_workspace_bytes": ([I32, I32, I32, I64], SZ),
            "fdgs_render": ([P, P, P, P, F, P, P, P, SZ, I64, P, P], C.c_int),
            "fdgs_render_timed": ([P, P, P, P, F, P, P, P, SZ, I64, P, P, P], C.c_int),
            "fdgs_render_split": ([P, P, P, P, F, P, P, P, SZ, I64, P, P, P, P, P], C.c_int),
            "fdgs_render_checked": ([P, P, P, P, F, P, P, P, SZ, I64, P, P], C.c_int),
            "fdgs_render_debug_views": ([P, SZ, I32, I32, I32, I64, P], C.c_int),
            "fdgs_render_graph_create": ([P, I32, I32, P, SZ, I64, P], C.c_int),
            "fdgs_render_graph_launch": ([P, P, P, P, P, F, P, P, P], C.c_int),
            "fdgs_render_graph_launch_split": ([P, P, P, P, P, F, P, P, P, P, P], C.c_int),
            "fdgs_render_graph_launch_timed": ([P, P, P, P, P, F, P, P, P, P, P, P], C.c_int),
            "fdgs_render_graph_destroy": ([P], C.c_int),
            "fdgs_keyframe_workspace_bytes": ([I32], SZ),
            "fdgs_keyframe_mask": ([P, P, I32, F, P, P, SZ, P], C.c_int),
            "fdgs_mask_or": ([P, P, I32, P, P], C.c_int),
            "fdgs_keyframe_mask_contrib_workspace_bytes": ([I32, P, I32, I64], SZ),
            "fdgs_keyframe_mask_contrib": ([P, P, I32, F, C.c_double, I64, P, P, SZ, P, P], C.c_int),
            "fdgs_mask_compact_workspace_bytes": ([I32], SZ),
            "fdgs_mask_compact": ([P, P, I32, P, P, P, SZ, P], C.c_int),
            "fdgs_stv_workspace_bytes": ([I32, P, I32, I64], SZ),
            "fdgs_scene_compact_workspace_bytes": ([I32], SZ),
            "fdgs_scene_compact": ([P, P, P, P, P, P, P, P, P, P, P, SZ, P], C.c_int),
            "fdgs_stv_score": ([P, P, I32, P, I32, P, P, P, P, P, SZ, P, P], C.c_int),
            "fdgs_prune_workspace_bytes": ([I32], SZ),
            "fdgs_prune_mask": ([P, I32, C.c_int64, P, P, SZ, P], C.c_int),
            "fdgs_pipeline_create": ([P, I32, P, I32, I32, P], C.c_int),
            "fdgs_pipeline_render": ([P, P, I32, P, P], C.c_int),
            "fdgs_pipeline_destroy": ([P], C.c_int),
            "fdgs_debug_strip_reach": ([P, SZ, I32, I32, I32, I64, P, P], C.c_int),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name, None)
            if f is None:  # an older build (tools/ A/B variants); tests/test_abi.py checks the exports
                continue
            f.argtypes = args
            f.restype = res
        if CHECK_ABI and L.fdgs_abi_version() != ABI_VERSION:
            raise ImportError(f"{LIB_PATH} has ABI version {L.fdgs_abi_version()}, the binding needs {ABI_VERSION}: "
                              "rebuild it (python -m paper_2503_16422_b200.build)")
        _lib = L
        return L


def check(status: int):
    if status != FDGS_OK:
        msg = lib().fdgs_last_error().decode(errors="replace")
        raise FdgsError(status, msg)
