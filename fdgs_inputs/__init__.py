"""Seeded synthetic inputs shared by the oracle, the tests and the bench.

This module holds NO arithmetic of the method (no slicing, projection,
culling, sorting or blending).  It only draws the scene arrays, builds the
camera rigs and the frame timestamps of BASELINE.json ``configs`` with the
recipe of SURVEY.md §8(d) d.2 / DESIGN.md "Input recipe".  Both the CUDA
path and ``oracle/`` consume what it returns; neither side imports the other.
"""
from .scenes import (  # noqa: F401
    CONFIGS,
    SceneArrays,
    Camera,
    make_scene,
    make_cameras,
    frame_times,
    look_at,
    scene_sha256,
    isotropic_scene,
    vq_scene,
)
