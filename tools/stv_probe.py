"""Probe fdgs_stv_score: parity margins against the oracle on a reduced case and
throughput on the C3 rig (GPU box).  Prints one JSON line."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import fdgs_inputs as fi  # noqa: E402
import oracle  # noqa: E402
import paper_2503_16422_b200 as fd  # noqa: E402


def margins():
    scene = fi.make_scene("c2", n=4000, seed=3)
    cams = fi.make_cameras("c2", width=96, height=72, fx=133.0, count=4)
    ts = [0.0, 0.3, 0.7, 1.0]
    r = fd.stv_score(fd.Scene.from_arrays(scene), cams, ts, spatial=True)
    ref = oracle.stv_score(scene, cams, np.float32(ts))
    sp = r["spatial"].cpu().numpy().astype(np.float64)
    e = np.abs(sp - ref["spatial"])
    rel = e / np.maximum(np.abs(ref["spatial"]), 1e-30)
    return dict(max_abs=float(e.max()), max_rel_where_ref_gt_1=float(rel[ref["spatial"] > 1].max()),
                score_max_abs=float(np.abs(r["score"].cpu().numpy() - ref["score"]).max()))


def throughput(n_ts=15):
    scene = fi.make_scene("c3")
    cams = fi.make_cameras("c3")
    ts = list(fi.frame_times(300)[:: 300 // n_ts][:n_ts])
    sc = fd.Scene.from_arrays(scene)
    fd.stv_score(sc, cams, ts[:2])  # warm up (workspace, capacity)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fd.stv_score(sc, cams, ts, max_entries=8 << 20)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    views = len(cams) * len(ts)
    return dict(views=views, s=dt, views_per_s=views / dt, ms_per_view=1e3 * dt / views,
                nonzero=int((r["score"] > 0).sum().item()))


if __name__ == "__main__":
    out = dict(margins=margins(), c3=throughput())
    print(json.dumps(out))
