"""CPU oracle for the 4DGS-1K render hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2503_16422_b200``) never imports it; the two share no
code (see oracle/fdgs_oracle.c header).

Parity status per function:
  rotor4, slice (Eq. 1), temporal marginal (Eq. 3), projection, SH basis,
  per-pixel compositing (Eq. 2), masks, key-frame schedule, tile lists, VQ-SH
  lookup: pinned by tests/test_oracle_pins.py; the off-axis projection
  (pinhole image, Sigma_2D against a complex-step Jacobian of the world->pixel
  map under rotated cameras with the EWA clamp exercised, conic, pixel AABB),
  the SH basis against scipy's spherical harmonics (sign convention of R9) and
  the view direction: tests/test_oracle_projection_pins.py; contributions, the
  STV score (both combine readings, all variants), paper-literal masks:
  tests/test_oracle_stv.py.  tools/mutate_oracle.py (run by
  tests/test_oracle_mutants.py) checks that every listed mutant of the oracle
  fails a pin.  No function is parity-unpinned.
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
    set_num_threads,
    MAX_LEAVES,
    ST_TEMPORAL, ST_SUPPORT, ST_NEAR, ST_COVER, ST_VISIBLE,
)
