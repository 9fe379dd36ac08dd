"""The README's usage example, verbatim in substance: the masked render of one
frame, the STV score, and the same frame through the pipelined working-set
path (bit-identical)."""
import pytest
import torch

import fdgs_inputs as fi


@pytest.mark.gpu
def test_readme_usage_example():
    import paper_2503_16422_b200 as fd
    scene = fd.Scene.from_arrays(fi.make_scene("c3"))
    cams = fi.make_cameras("c3")
    kf = fd.keyframes(300, 20)
    times = fi.frame_times(300)
    masks = [fd.keyframe_mask(scene, cams, float(times[k])) for k in kf]
    l, r = fd.bracket(kf, 150)
    img = fd.Renderer(scene, 1352, 1014).render(cams[7], float(times[150]), masks[l], masks[r])
    score = fd.stv_score(scene, cams, times[::20])["score"]
    pipe = fd.RenderPipeline(scene, 1352, 1014, depth=6)
    ws = scene.compact(masks[l], masks[r], sync=False)
    frames = [(cams[c], float(times[150]), None, None, ws) for c in range(20)]
    outs = [pipe.renderers[0].new_output() for _ in frames]
    pipe.render_many(frames, outs)
    torch.cuda.synchronize()
    assert torch.equal(outs[7], img)
    assert score.shape == (scene.n,) and bool(torch.isfinite(score).all()) and float(score.sum()) > 0
