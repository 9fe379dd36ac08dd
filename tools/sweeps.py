"""Redundancy analytics and speed sweeps on the GPU box.

Analogues, on the synthetic C3 scene, of
  * Fig. 2b "active ratio": the fraction of Gaussians active
    across all views at a moment, with "active" = receives blending weight in
    some view (the paper-literal mask, fdgs_keyframe_mask_contrib, threshold 0)
    and, beside it, the geometric visibility of reading R3;
  * Fig. 2c "activation IoU": IoU of the active set of frame 0
    and of frame t;
  * Fig. 10: FPS against the number of inactive Gaussians added to
    the active set of one timestamp;
  * the key-frame interval study: FPS and PSNR(masked, unmasked)
    against the interval Delta.
Every render is the product path (libfdgs.so through the binding); popcounts,
IoU and PSNR are host-side analysis.  Prints one JSON object.
"""
import argparse
import json
import math
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import fdgs_inputs as fi  # noqa: E402
import paper_2503_16422_b200 as fd  # noqa: E402


def bits(m, n):
    return np.unpackbits(m.cpu().numpy().view(np.uint32).view(np.uint8), bitorder="little")[:n].astype(bool)


def fps_of(pipe, frames, outs, reps=3):
    best = math.inf
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        pipe.render_many(frames, outs)
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return len(frames) / (best / 1e3)


def pruning_study(name, ratios=(0.0, 0.5, 0.8, 0.9), t_stride=10):
    """Sec. 4.2.1 end to end on the GPU (Table 3 d/e analogue, speed only): the
    STV score over the rig, prune the lowest-scored fraction, then render the
    pruned scene under its own key-frame masks.  No fine-tuning (needs
    training data): this measures speed, not quality."""
    cfg = fi.CONFIGS[name]
    scene = fi.make_scene(name)
    cams = fi.make_cameras(name)
    F = cfg["frames"]
    times = fi.frame_times(F)
    sc = fd.Scene.from_arrays(scene)
    t0 = time.perf_counter()
    score = fd.stv_score(sc, cams, [float(x) for x in times[::t_stride]])["score"]
    score_s = time.perf_counter() - t0
    seq = [(f, c) for f in range(0, F, 5) for c in range(0, len(cams), 4)]
    out = {"config": name, "n": scene.n, "score_views": len(cams) * len(times[::t_stride]),
           "score_s": round(score_s, 3), "curve": []}
    for r in ratios:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sub = sc.prune(score, max(1, int(round(scene.n * (1.0 - r)))))  # fdgs_prune_mask + fdgs_scene_compact
        prune_s = time.perf_counter() - t0
        kf = fd.keyframes(F, cfg["keyframe_interval"])
        masks = [fd.keyframe_mask(sub, cams, float(times[k])) for k in kf]
        pipe = fd.RenderPipeline(sub, cams[0].width, cams[0].height, depth=4)
        outs = [pipe.renderers[0].new_output() for _ in seq]
        frames = []
        for f, c in seq:
            lo, hi = fd.bracket(kf, f)
            frames.append((fd.camera_struct(cams[c]), float(times[f]), masks[lo], masks[hi]))
        fps_of(pipe, frames, outs, reps=1)
        out["curve"].append({"prune_ratio": r, "n": sub.n, "prune_s": round(prune_s, 4),
                             "fps_masked": round(fps_of(pipe, frames, outs), 1)})
        del pipe, outs, sub, masks
        torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--t-stride", type=int, default=10, help="timestamps sampled for the ratio / IoU curves")
    ap.add_argument("--prune-config", default="c4", help="config of the pruning study ('' to skip)")
    a = ap.parse_args()
    cfg = fi.CONFIGS[a.config]
    scene = fi.make_scene(a.config)
    cams = fi.make_cameras(a.config)
    F = cfg["frames"]
    times = fi.frame_times(F)
    n = scene.n
    sc = fd.Scene.from_arrays(scene)
    out = {"config": a.config, "n": n, "views": len(cams), "frames": F}

    # ---- Fig. 2b / 2c analogues
    ts_idx = list(range(0, F, a.t_stride))
    t0 = time.perf_counter()
    lit, geo = {}, {}
    for f in ts_idx:
        t = float(times[f])
        lit[f] = bits(fd.keyframe_mask_contrib(sc, cams, t, 0.0), n)
        geo[f] = bits(fd.keyframe_mask(sc, cams, t), n)
    torch.cuda.synchronize()
    out["mask_build_s"] = round(time.perf_counter() - t0, 3)
    iou = lambda x, y: float((x & y).sum() / max(1, (x | y).sum()))
    out["active_ratio"] = {"t_index": ts_idx, "literal": [round(float(lit[f].mean()), 4) for f in ts_idx],
                           "geometric": [round(float(geo[f].mean()), 4) for f in ts_idx]}
    # set difference of the two mask readings (R3 geometric vs R3b literal)
    out["mask_set_difference"] = {
        "t_index": ts_idx,
        "literal_not_geometric": [int((lit[f] & ~geo[f]).sum()) for f in ts_idx],
        "geometric_not_literal_fraction": [round(float((geo[f] & ~lit[f]).sum() / max(1, geo[f].sum())), 4)
                                           for f in ts_idx]}
    out["activation_iou_vs_frame0"] = {"t_index": ts_idx, "literal": [round(iou(lit[ts_idx[0]], lit[f]), 4)
                                                                      for f in ts_idx]}
    win = [iou(lit[f], lit[f + a.t_stride]) for f in ts_idx[:-1] if f + a.t_stride in lit]
    out["activation_iou_adjacent"] = {"stride_frames": a.t_stride, "mean": round(float(np.mean(win)), 4),
                                      "min": round(float(np.min(win)), 4)}

    # ---- Fig. 10 analogue: FPS vs injected inactive Gaussians at one t
    fmid = F // 2
    tmid = float(times[fmid])
    act_idx = np.nonzero(lit[(fmid // a.t_stride) * a.t_stride] if fmid % a.t_stride == 0 else
                         bits(fd.keyframe_mask_contrib(sc, cams, tmid, 0.0), n))[0]
    inact_pool = np.nonzero(~bits(fd.keyframe_mask(sc, cams, tmid), n))[0]  # not even geometrically visible
    rng = np.random.default_rng(0)
    rng.shuffle(inact_pool)
    frames_idx = list(range(len(cams)))
    fps_curve = []
    for k in [0, 50_000, 100_000, 200_000, 400_000, 800_000]:
        if k <= inact_pool.size:
            sel = np.sort(np.concatenate([act_idx, inact_pool[:k]]))
        else:  # more inactive Gaussians than the scene holds: replicate the pool with distant mu_t
            extra = inact_pool[rng.integers(0, inact_pool.size, k)]
            sel = np.sort(np.concatenate([act_idx, extra]))
        sub = scene.subset(sel)
        ssub = fd.Scene.from_arrays(sub)
        pipe = fd.RenderPipeline(ssub, cams[0].width, cams[0].height, depth=4)
        outs = [pipe.renderers[0].new_output() for _ in frames_idx]
        frames = [(fd.camera_struct(cams[c]), tmid, None, None) for c in frames_idx]
        fps_of(pipe, frames, outs, reps=1)
        fps_curve.append({"inactive_added": int(k), "n": int(sel.size), "fps": round(fps_of(pipe, frames, outs), 1)})
        del pipe, outs, ssub
        torch.cuda.empty_cache()
    out["fps_vs_inactive"] = {"t": tmid, "active": int(act_idx.size), "curve": fps_curve,
                              "note": "unmasked renders of the active set of t plus k Gaussians inactive at t"}

    # ---- interval study: FPS and PSNR(masked vs unmasked) against Delta
    seq = [(f, c) for f in range(0, F, 3) for c in range(0, len(cams), 4)]
    pipe = fd.RenderPipeline(sc, cams[0].width, cams[0].height, depth=4)
    outs_u = [pipe.renderers[0].new_output() for _ in seq]
    frames_u = [(fd.camera_struct(cams[c]), float(times[f]), None, None) for f, c in seq]
    fps_u = fps_of(pipe, frames_u, outs_u)
    res = []
    for kind, delta in [(k, d) for k in ("geometric", "literal") for d in [1, 5, 10, 20, 50, 100, F]]:
        kf = fd.keyframes(F, delta)
        if kind == "geometric":
            masks = [fd.keyframe_mask(sc, cams, float(times[k])) for k in kf]
        else:  # P:282 read literally: blending weight > 0 in some view
            masks = [fd.keyframe_mask_contrib(sc, cams, float(times[k]), 0.0) for k in kf]
        outs_m = [pipe.renderers[0].new_output() for _ in seq]
        frames_m = []
        act = []
        for f, c in seq:
            lo, hi = fd.bracket(kf, f)
            frames_m.append((fd.camera_struct(cams[c]), float(times[f]), masks[lo], masks[hi]))
            act.append(float((bits(masks[lo], n) | bits(masks[hi], n)).mean()))
        fps_m = fps_of(pipe, frames_m, outs_m)
        psnr, same = [], 0
        for x, y in zip(outs_m, outs_u):
            mse = float(((x - y) ** 2).mean())
            if mse == 0:
                same += 1
            else:
                psnr.append(10 * math.log10(1.0 / mse))
        res.append({"masks": kind, "delta": delta, "keyframes": len(kf), "fps": round(fps_m, 1),
                    "mean_active_fraction": round(float(np.mean(act)), 4),
                    "identical_frames": same,
                    "psnr_vs_unmasked_mean_of_differing": round(float(np.mean(psnr)), 2) if psnr else None,
                    "psnr_vs_unmasked_min": round(float(np.min(psnr)), 2) if psnr else None})
        del outs_m
    if a.prune_config:
        out["pruning_study"] = pruning_study(a.prune_config)
    out["interval_study"] = {"unmasked_fps": round(fps_u, 1), "frames": len(seq), "curve": res,
                             "note": "geometric (reading R3) and literal (R3b, weight > 0) key-frame masks; PSNR on [0,1] "
                                     "rgb over the frames that differ at all"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
