"""GPU parity of fdgs_prune_mask (Sec. 4.2.1 "Pruning"; SURVEY NEXT-f1
top-k select) against the oracle (oracle/fdgs_oracle.c or_prune_mask), through
the C-ABI.  Integer work: masks bit-exact, on ragged sizes spanning many
1024-element chunks, tie-heavy / signed / +-0 scores, every keep edge, and the
STV scores of a real scene; then the pruned scene (Scene.prune) renders
bit-identically to the same subset built on the host.
"""
import numpy as np
import pytest
import torch

import fdgs_inputs as fi
import oracle
import paper_2503_16422_b200 as fd

pytestmark = pytest.mark.gpu


def _gpu_mask(score, keep):
    s = torch.from_numpy(np.ascontiguousarray(score, np.float32)).cuda()
    m = fd.prune_mask(s, s.numel(), keep)
    torch.cuda.synchronize()
    return m.cpu().numpy().view(np.uint32)[: (score.size + 31) // 32]


def _scores(kind, n, rng):
    if kind == "uniform":
        return rng.random(n, dtype=np.float32)
    if kind == "ties":  # 21 distinct values
        return np.round(rng.random(n) * 20).astype(np.float32)
    if kind == "signed":  # negatives, +-0, denormals, huge values
        s = rng.standard_normal(n).astype(np.float32) * np.float32(1e3)
        s[rng.random(n) < 0.2] = 0.0
        s[rng.random(n) < 0.2] = -0.0
        s[rng.random(n) < 0.05] = np.float32(1e-42)
        s[rng.random(n) < 0.05] = np.float32(-3e38)
        return s
    if kind == "constant":
        return np.full(n, 0.5, np.float32)
    raise ValueError(kind)


@pytest.mark.parametrize("kind", ["uniform", "ties", "signed", "constant"])
@pytest.mark.parametrize("n", [1, 31, 1000, 100_003])
def test_prune_mask_bit_exact(kind, n):
    rng = np.random.default_rng(n + len(kind))
    s = _scores(kind, n, rng)
    for keep in sorted({0, 1, n // 3, n // 2, n - 1, n, n + 7}):
        if keep < 0:
            continue
        got = _gpu_mask(s, keep)
        want = oracle.prune_mask(s, keep)
        assert np.array_equal(got, want), f"{kind} n={n} keep={keep}"
        assert int(np.unpackbits(got.view(np.uint8)).sum()) == min(keep, n)


def test_prune_mask_full_size_c4():
    """BASELINE's largest scene size (3M), scores with many ties at the cut."""
    rng = np.random.default_rng(7)
    n = fi.CONFIGS["c4"]["n"]
    s = (np.round(rng.random(n) * 1000) / 1000).astype(np.float32)
    for keep in (n // 5, n // 2):
        assert np.array_equal(_gpu_mask(s, keep), oracle.prune_mask(s, keep))


def test_prune_stv_scores_and_pruned_render():
    """End to end on c1: the GPU STV score ranks the scene, the mask matches the
    oracle's selection from the same scores, and the pruned scene renders
    exactly like the host-built subset of the kept indices."""
    scene = fi.make_scene("c1")
    cams = fi.make_cameras("c1")
    sc = fd.Scene.from_arrays(scene)
    score = fd.stv_score(sc, cams, [0.0, 0.5, 1.0])["score"]
    keep = scene.n // 2
    got = fd.prune_mask(score, scene.n, keep).cpu().numpy().view(np.uint32)
    assert np.array_equal(got[: (scene.n + 31) // 32], oracle.prune_mask(score.cpu().numpy(), keep))
    pr = sc.prune(score, keep)
    kept = pr.kept.cpu().numpy()
    bits = np.unpackbits(got.view(np.uint8), bitorder="little")[: scene.n].astype(bool)
    assert np.array_equal(kept, np.nonzero(bits)[0])
    ref = fd.Scene.from_arrays(scene.subset(kept))
    w, h = cams[0].width, cams[0].height
    a = fd.Renderer(pr, w, h).render(cams[0], 0.5)
    b = fd.Renderer(ref, w, h).render(cams[0], 0.5)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    m = fd.keyframe_mask(pr, cams, 0.5)  # a standalone scene takes masks of its own
    assert m.numel() == fd.mask_words(keep)


def test_prune_mask_errors():
    s = torch.zeros(10, device="cuda")
    with pytest.raises(fd.FdgsError):
        fd.prune_mask(s, 10, -1)
    with pytest.raises(ValueError):
        fd.prune_mask(s.double(), 10, 3)
