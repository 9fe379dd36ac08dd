"""B200-native render hot path of 4DGS-1K (arXiv 2503.16422).

Rendering a frame at timestamp t from 4D Gaussians under the key-frame
temporal filter: libfdgs.so (csrc/, sm_100a CUDA) behind the C ABI of
include/fdgs.h, with this thin ctypes binding.  See DESIGN.md.
"""
from .api import (  # noqa: F401
    FrameStats,
    RenderPipeline,
    Renderer,
    Scene,
    bracket,
    camera_struct,
    default_max_entries,
    keyframe_mask,
    keyframe_mask_contrib,
    keyframes,
    log255_opacity,
    mask_compact,
    prune_mask,
    mask_or,
    mask_words,
    stv_score,
    validate,
)
from ._lib import FdgsError, lib  # noqa: F401
