"""CPU oracle for the 4DGS-1K render hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2503_16422_b200``) never imports it; the two share no
code (see oracle/fdgs_oracle.c header).

Parity status per function:
  rotor4, slice (Eq. 1), temporal marginal (Eq. 3), projection, SH basis,
  per-pixel compositing (Eq. 2), masks, key-frame schedule, tile lists, VQ-SH
  lookup: pinned by tests/test_oracle_pins.py; contributions, the STV score
  (both combine readings, all variants), paper-literal masks: pinned by
  tests/test_oracle_stv.py.  Parity unpinned: the SH *sign convention* only, a
  reading (R9); orthonormality and the pole case pin everything but the signs.
"""
from .oracle import (  # noqa: F401
    build_oracle,
    load,
    records,
    render,
    render_image,
    canonical_order,
    tile_lists,
    band_tiles,
    contrib,
    stv_score,
    tv_value,
    keyframe_mask,
    keyframe_mask_contrib,
    prune_mask,
    keyframes,
    bracket,
    active_mask,
    rotor4,
    sh_basis,
    num_threads,
    MAX_LEAVES,
    ST_TEMPORAL, ST_SUPPORT, ST_NEAR, ST_COVER, ST_VISIBLE,
)
