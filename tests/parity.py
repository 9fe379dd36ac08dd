"""Helpers comparing the CUDA path (via the C-ABI binding) with the oracle."""
import numpy as np

import oracle

TOL_MAX = 2e-4      # BASELINE.json north_star: max-abs 2e-4 per pixel
TOL_MEAN = 1e-5     # mean-abs 1e-5 over all pixels


def compare_rgb(gpu_chw, orc, pixels=None, width=None):
    """gpu_chw: (3,H,W) numpy float32; orc: oracle.render() dict.
    Returns (max_err, mean_err, n_alt_used) against the nearest admissible
    branch of the two-branch termination rule (R17)."""
    g = gpu_chw.reshape(3, -1).T.astype(np.float64)
    if pixels is not None:
        g = g[np.asarray(pixels)]
    prim = orc["rgb"]
    err = np.abs(g - prim).max(1)
    chosen = prim.copy()
    used = 0
    bad = np.nonzero(err > TOL_MAX)[0]
    for k in bad:
        for a in range(orc["n_alt"][k]):
            e = np.abs(g[k] - orc["alt"][k, a]).max()
            if e < err[k]:
                err[k] = e
                chosen[k] = orc["alt"][k, a]
                used += 1
    mean = np.abs(g - chosen).mean()
    return float(err.max()) if err.size else 0.0, float(mean) if err.size else 0.0, used


def assert_rgb_parity(gpu_chw, orc, pixels=None):
    mx, mean, used = compare_rgb(gpu_chw, orc, pixels)
    assert mx <= TOL_MAX, f"max-abs {mx:.3g} > {TOL_MAX} (alternates used: {used})"
    assert mean <= TOL_MEAN, f"mean-abs {mean:.3g} > {TOL_MEAN}"
    return mx, mean, used


def gpu_records(views):
    """Decision records of the GPU visible set as numpy (ordered by slot)."""
    r0 = views["rec0"].cpu().numpy()
    r1 = views["rec1"].cpu().numpy()
    r2 = views["rec2"].cpu().numpy()
    gid = r2[:, 3].view(np.int32).copy()
    ax = r1[:, 2].view(np.uint32)
    ay = r1[:, 3].view(np.uint32)
    rect = np.stack([ax & 0xFFFF, ax >> 16, ay & 0xFFFF, (ay >> 16) & 0x7FFF], 1).astype(np.int32)
    f32 = np.stack([r0[:, 0], r0[:, 1], r0[:, 2], r0[:, 3], r1[:, 0], r1[:, 1]], 1)
    depth = views["depth"].cpu().numpy().view(np.uint32)
    order = views["order"].cpu().numpy()
    return dict(gid=gid, rect=rect, f32=f32, depth=depth, rgb=r2[:, :3], order=order)


def assert_records_bit_exact(views, scene, cam, t, mask=None):
    """Visible set, pixel AABBs, depth keys, fp32 record fields and the
    canonical order must equal the oracle's bit for bit."""
    g = gpu_records(views)
    rec = oracle.records(scene, cam, t)
    vis = rec["stage"] == oracle.ST_VISIBLE
    if mask is not None:
        bits = np.unpackbits(np.asarray(mask, np.uint32).view(np.uint8), bitorder="little")[:scene.n].astype(bool)
        vis &= bits
    want = np.nonzero(vis)[0].astype(np.int32)
    assert views["n_vis"] == want.size, (views["n_vis"], want.size)
    assert np.array_equal(g["gid"], want)
    assert np.array_equal(g["rect"], rec["rect"][want])
    assert np.array_equal(g["depth"], rec["depth_bits"][want])
    assert np.array_equal(g["f32"].view(np.uint32), rec["f32"][want].view(np.uint32))
    canon = oracle.canonical_order(scene, cam, t, mask)
    assert np.array_equal(g["gid"][g["order"]], canon)
    # value path: colour within fp32 SH evaluation error
    assert np.abs(g["rgb"] - rec["rgb"][want]).max(initial=0.0) < 1e-5
    return g


def assert_tile_lists_bit_exact(views, scene, cam, t, mask=None):
    g = gpu_records(views)
    ranges, ids = oracle.tile_lists(scene, cam, t, mask)
    ts = views["tile_start"].cpu().numpy().astype(np.int64)
    assert views["n_entries"] == ids.size
    assert np.array_equal(ts[:-1], ranges[:, 0]) and np.array_equal(ts[1:], ranges[:, 1])
    ent = views["entries"].cpu().numpy()
    assert np.array_equal(g["gid"][ent], ids)


def mask_bits(mask_words, n):
    return np.unpackbits(np.asarray(mask_words, np.uint32).view(np.uint8), bitorder="little")[:n].astype(bool)
