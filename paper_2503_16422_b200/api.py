"""Python binding of libfdgs.so: same names as include/fdgs.h, marshalling only.

Every step of the render path runs in the CUDA kernels of libfdgs.so;
PyTorch only provides device memory and streams.  There is no CPU fallback:
if the library or a CUDA device is missing these functions raise.

Host logic that the paper states and that is not a per-pixel/per-Gaussian
computation lives here: the key-frame schedule and bracketing of
Sec. 4.2.2 (readings R4/R5).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import FdgsCamera, FdgsDebugViews, FdgsFrameJob, FdgsFrameStats, FdgsPipelineSlot, FdgsScene, check, lib

_FIELDS = ("mean", "scale", "rot_l", "rot_r", "opacity", "log255_opacity", "sh")


def _stream_ptr(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


class Scene:
    """Device-resident 4D Gaussians (fdgs_scene)."""

    def __init__(self, tensors: dict, device=None, interleaved: bool = True):
        """tensors: the _FIELDS arrays; optional "sh_index" (N,) uint16 makes
        "sh" a VQ codebook (K,16,3) (Ours-PP storage).  interleaved:
        mean/scale/rot_l/rot_r live in one (N, 4, 4) buffer, a 64-byte record per
        Gaussian (fdgs_scene.param_stride = 4), so the mask-driven sparse gather
        of the cull and slice kernels reads one DRAM burst per Gaussian."""
        dev = torch.device(device or "cuda")
        self.t = {}
        for f in _FIELDS:
            x = tensors[f]
            if isinstance(x, np.ndarray):
                x = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
            self.t[f] = x.to(device=dev, dtype=torch.float32).contiguous()
        self.n = int(self.t["mean"].shape[0])
        self.device = dev
        self.stride = 0
        if interleaved:
            self.params = torch.stack([self.t[f] for f in ("mean", "scale", "rot_l", "rot_r")], 1).contiguous()
            for k, f in enumerate(("mean", "scale", "rot_l", "rot_r")):
                self.t[f] = self.params[:, k]  # (N, 4) views with a 64-byte row stride
            self.stride = 4
        idx = tensors.get("sh_index")
        k = 0
        if idx is not None:
            if isinstance(idx, np.ndarray):
                idx = torch.from_numpy(np.ascontiguousarray(idx, dtype=np.uint16))
            self.t["sh_index"] = idx.to(device=dev, dtype=torch.uint16).contiguous()
            k = int(self.t["sh"].shape[0])
        self.struct = FdgsScene(self.n, *[self.t[f].data_ptr() for f in _FIELDS],
                                self.t["sh_index"].data_ptr() if idx is not None else None, k, self.stride, None, 0,
                                None)

    def compact(self, mask_l: torch.Tensor, mask_r: torch.Tensor | None = None, stream=None,
                standalone: bool = False, sync: bool = True) -> "Scene":
        """fdgs_scene_compact: the working set of a key-frame window (the
        Gaussians of mask_l | mask_r, ascending) as a dense Scene whose records
        report the original indices.  Render it with no mask: frames equal the
        masked renders of this scene bit for bit.  sync=True reads the count
        back (one synchronisation; `.n` is exact); sync=False keeps it on the
        device (fdgs_scene.d_n: `.n` is the capacity, the render reads the
        count itself -- no host synchronisation, bench.py's timed path).
        standalone: a new scene in its own right (a pruned scene: records,
        masks and scores index the kept Gaussians 0..m-1); `.kept` holds the
        original indices either way (standalone implies sync)."""
        if self.struct.gid:
            raise ValueError("already a compacted working set")
        n, dev = self.n, self.device
        vq = "sh_index" in self.t
        st = stream or torch.cuda.current_stream(dev)
        # every allocation, the zero-fill and the count read-back are ordered on
        # `st` (the caching allocator ties the buffers to the stream current at
        # allocation, so they are allocated with `st` current)
        with torch.cuda.stream(st):
            params = torch.empty((max(n, 1), 4, 4), dtype=torch.float32, device=dev)
            opacity = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
            L = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
            sh = None if vq else torch.empty((max(n, 1), 16, 3), dtype=torch.float32, device=dev)
            sh_index = torch.empty(max(n, 1), dtype=torch.uint16, device=dev) if vq else None
            gid = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
            count = torch.zeros(1, dtype=torch.int32, device=dev)
            nb = lib().fdgs_scene_compact_workspace_bytes(n)
            ws = torch.empty(nb, dtype=torch.uint8, device=dev)
            check(lib().fdgs_scene_compact(C.byref(self.struct), _ptr(mask_l), _ptr(mask_r), _ptr(params),
                                           _ptr(opacity), _ptr(L), _ptr(sh), _ptr(sh_index), _ptr(gid), _ptr(count),
                                           _ptr(ws), nb, _stream_ptr(st)))
            if sync or standalone:
                host = torch.empty(1, dtype=torch.int32, pin_memory=True)
                host.copy_(count, non_blocking=True)
        if sync or standalone:
            st.synchronize()
            m = int(host.item())
        else:
            m = n  # capacity; the device count decides
        out = Scene.__new__(Scene)
        out.n, out.device, out.stride = m, dev, 4
        out.params = params
        out.t = {"mean": params[:m, 0], "scale": params[:m, 1], "rot_l": params[:m, 2], "rot_r": params[:m, 3],
                 "opacity": opacity[:m], "log255_opacity": L[:m], "gid": gid[:m],
                 "sh": self.t["sh"] if vq else sh[:m]}
        if vq:
            out.t["sh_index"] = sh_index[:m]
        out.struct = FdgsScene(m, *[out.t[f].data_ptr() for f in _FIELDS],
                               out.t["sh_index"].data_ptr() if vq else None,
                               int(self.t["sh"].shape[0]) if vq else 0, 4,
                               None if standalone else gid.data_ptr(), 0 if standalone else n,
                               None if (sync or standalone) else count.data_ptr())
        out.source = self
        out.count = count  # DEVICE uint32 count (the exact size)
        out.kept = gid[:m]
        if standalone:
            del out.t["gid"]
        return out

    def prune(self, score: torch.Tensor, keep: int, stream=None) -> "Scene":
        """Pruning of Sec. 4.2.1: the scene of the `keep` highest-scored
        Gaussians (fdgs_prune_mask, ties by ascending index), compacted in index
        order (fdgs_scene_compact).  `.kept` = their original indices."""
        if self.struct.gid:
            raise ValueError("prune the full scene, not a working set")
        return self.compact(prune_mask(score, self.n, keep, stream=stream), stream=stream, standalone=True)

    @classmethod
    def from_arrays(cls, arrays, device=None):
        d = {f: getattr(arrays, f) for f in _FIELDS}
        if getattr(arrays, "sh_index", None) is not None:
            d["sh_index"] = arrays.sh_index
        return cls(d, device)

    def nbytes(self) -> int:
        return sum(v.numel() * 4 for v in self.t.values())


def camera_struct(cam) -> FdgsCamera:
    c = FdgsCamera()
    c.width, c.height = int(cam.width), int(cam.height)
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.R[:] = [float(x) for x in np.asarray(cam.R, np.float32).reshape(9)]
    c.T[:] = [float(x) for x in np.asarray(cam.T, np.float32).reshape(3)]
    c.z_near = float(cam.z_near)
    c.bg[:] = [float(b) for b in cam.bg]
    return c


def default_max_entries(n: int) -> int:
    """Entry capacity of a render workspace; render_checked grows it on overflow."""
    return int(min(2 ** 32 - 1, max(1 << 22, 24 * max(n, 1))))


def mask_words(n: int) -> int:
    return (n + 31) // 32


@dataclass
class FrameStats:
    n_act: int
    n_vis: int
    n_entries: int
    status: int
    n_evaluated: int = 0
    n_blended: int = 0


class Renderer:
    """fdgs_render with a caller-owned workspace sized for (n, width, height)."""

    def __init__(self, scene: Scene, width: int, height: int, max_entries: int | None = None):
        self.scene = scene
        self.width, self.height = int(width), int(height)
        self.max_entries = int(default_max_entries(scene.n) if max_entries is None else max_entries)
        self._alloc()

    def _alloc(self):
        nbytes = lib().fdgs_render_workspace_bytes(self.scene.n, self.width, self.height, self.max_entries)
        if nbytes == 0:
            raise ValueError("invalid render size")
        # zero-filled: the epoch-tagged look-back tables require it (include/fdgs.h)
        self._drop_graph()
        self.ws = torch.zeros(nbytes, dtype=torch.uint8, device=self.scene.device)
        self.ws_bytes = nbytes
        self._layout_n = self.scene.n

    def _drop_graph(self):
        g = getattr(self, "_graph", None)
        if g:
            lib().fdgs_render_graph_destroy(g)
        self._graph = None

    def __del__(self):
        try:
            self._drop_graph()
        except Exception:
            pass

    def _ensure_graph(self):
        """The front-end graph of this workspace (captured on first use)."""
        if not self._graph:
            h = C.c_void_p()
            base = self.scene  # the layout is the full scene's (working sets share it, n_capacity)
            check(lib().fdgs_render_graph_create(C.byref(base.struct), self.width, self.height, _ptr(self.ws),
                                                 self.ws_bytes, self.max_entries, C.byref(h)))
            self._graph = h
        return self._graph

    def render_graph(self, cam, t, mask_l=None, mask_r=None, out=None, out_T=None, stream=None, scene=None,
                     blend_stream=None, split_event=None, stage_events=None):
        """fdgs_render_graph_launch_timed: the front end as one CUDA-graph launch
        (captured on first use for this workspace) and the blend launched after
        it -- on `blend_stream` ordered by `split_event` when given; optional
        stage_events (5 torch.cuda.Event, as render()); results identical to
        render().  Async."""
        if cam.width != self.width or cam.height != self.height:
            raise ValueError("camera size differs from the renderer's")
        out = self.new_output() if out is None else out
        sc = self._scene_for(scene, stream)
        ml, mr = self._masks(mask_l, mask_r, sc)
        cs = camera_struct(cam) if not isinstance(cam, FdgsCamera) else cam
        self._ensure_graph()
        evs = None
        if stage_events is not None:
            for e in stage_events:
                if e.cuda_event == 0:
                    e.record(stream)  # materialise the CUDA event
            evs = (C.c_void_p * 5)(*[e.cuda_event for e in stage_events])
        split = None
        if blend_stream is not None:
            if split_event.cuda_event == 0:
                split_event.record(stream)
            split = C.c_void_p(split_event.cuda_event)
        check(lib().fdgs_render_graph_launch_timed(self._graph, C.byref(sc.struct), ml, mr, C.byref(cs), float(t),
                                                   _ptr(out), _ptr(out_T), _stream_ptr(stream),
                                                   None if blend_stream is None else _stream_ptr(blend_stream),
                                                   split, evs))
        return out

    def _scene_for(self, scene, stream):
        """The scene to render (default: the renderer's), resetting the workspace
        when its layout changes (another n; include/fdgs.h fdgs_render_workspace_bytes)."""
        scene = self.scene if scene is None else scene
        ln = max(scene.n, int(scene.struct.n_capacity))  # the layout fdgs_render uses
        if ln > self.scene.n:
            raise ValueError("scene larger than the workspace's")
        if ln != self._layout_n:
            with torch.cuda.stream(stream or torch.cuda.current_stream()):
                self.ws.zero_()
            self._layout_n = ln
        return scene

    def _masks(self, mask_l, mask_r, scene=None):
        scene = self.scene if scene is None else scene
        for m in (mask_l, mask_r):
            if m is not None:
                if m.dtype != torch.int32 or m.numel() != mask_words(scene.n) or not m.is_cuda:
                    raise ValueError(f"mask must be a cuda int32 tensor of {mask_words(scene.n)} words")
        return _ptr(mask_l), _ptr(mask_r)

    def new_output(self):
        return torch.empty((3, self.height, self.width), dtype=torch.float32, device=self.scene.device)

    def render(self, cam, t, mask_l=None, mask_r=None, out=None, out_T=None, stats=None, stream=None,
               stage_events=None, scene=None):
        """Async render (no host sync).  Returns the CHW float32 output tensor.
        stage_events: optional 5 torch.cuda.Event recorded at the stage boundaries.
        scene: another Scene to render in this workspace (e.g. a compacted
        working set, Scene.compact), at most the renderer's n."""
        if cam.width != self.width or cam.height != self.height:
            raise ValueError("camera size differs from the renderer's")
        out = self.new_output() if out is None else out
        sc = self._scene_for(scene, stream)
        ml, mr = self._masks(mask_l, mask_r, sc)
        cs = camera_struct(cam) if not isinstance(cam, FdgsCamera) else cam
        if stage_events is None:
            check(lib().fdgs_render(C.byref(sc.struct), ml, mr, C.byref(cs), float(t), _ptr(out),
                                    _ptr(out_T), _ptr(self.ws), self.ws_bytes, self.max_entries, _ptr(stats),
                                    _stream_ptr(stream)))
        else:
            evs = (C.c_void_p * 5)(*[e.cuda_event for e in stage_events])
            check(lib().fdgs_render_timed(C.byref(sc.struct), ml, mr, C.byref(cs), float(t), _ptr(out),
                                          _ptr(out_T), _ptr(self.ws), self.ws_bytes, self.max_entries, _ptr(stats),
                                          _stream_ptr(stream), evs))
        return out

    def render_split(self, cam, t, mask_l=None, mask_r=None, out=None, out_T=None, stats=None, stream=None,
                     blend_stream=None, split_event=None, stage_events=None, scene=None):
        """fdgs_render_split: front end on `stream`, blend on `blend_stream`."""
        out = self.new_output() if out is None else out
        sc = self._scene_for(scene, stream)
        ml, mr = self._masks(mask_l, mask_r, sc)
        cs = camera_struct(cam) if not isinstance(cam, FdgsCamera) else cam
        if split_event.cuda_event == 0:
            split_event.record(stream)  # materialise the CUDA event
        evs = None if stage_events is None else (C.c_void_p * 5)(*[e.cuda_event for e in stage_events])
        check(lib().fdgs_render_split(C.byref(sc.struct), ml, mr, C.byref(cs), float(t), _ptr(out),
                                      _ptr(out_T), _ptr(self.ws), self.ws_bytes, self.max_entries, _ptr(stats),
                                      _stream_ptr(stream), _stream_ptr(blend_stream),
                                      C.c_void_p(split_event.cuda_event), evs))
        return out

    def render_checked(self, cam, t, mask_l=None, mask_r=None, out=None, out_T=None, stream=None,
                       grow: bool = True, scene=None):
        """Synchronous render; grows the entry capacity and retries on overflow.
        scene: another Scene to render in this workspace (as render())."""
        out = self.new_output() if out is None else out
        sc = self._scene_for(scene, stream)
        ml, mr = self._masks(mask_l, mask_r, sc)
        cs = camera_struct(cam) if not isinstance(cam, FdgsCamera) else cam
        while True:
            hs = FdgsFrameStats()
            st = lib().fdgs_render_checked(C.byref(sc.struct), ml, mr, C.byref(cs), float(t), _ptr(out),
                                           _ptr(out_T), _ptr(self.ws), self.ws_bytes, self.max_entries,
                                           C.byref(hs), _stream_ptr(stream))
            if st == _lib.FDGS_ERR_OVERFLOW and grow:
                self.max_entries = int(min(2 ** 32 - 1, max(2 * self.max_entries, hs.n_entries + 1)))
                self._alloc()
                self._layout_n = max(sc.n, int(sc.struct.n_capacity))
                continue
            check(st)
            return out, FrameStats(hs.n_act, hs.n_vis, hs.n_entries, hs.status, hs.n_evaluated, hs.n_blended)

    def debug_views(self) -> dict:
        """Device views (torch tensors into the workspace) after a render."""
        v = FdgsDebugViews()
        n = self._layout_n  # the n of the last frame rendered in this workspace
        check(lib().fdgs_render_debug_views(_ptr(self.ws), self.ws_bytes, n, self.width, self.height,
                                            self.max_entries, C.byref(v)))
        base = self.ws.data_ptr()
        cnt = self._slice(v.counters, base, 16).view(torch.int32)
        n_act, n_vis, E, status = [int(x) for x in cnt.cpu()]

        def arr(ptr, count, itemsize, dtype):
            return self._slice(ptr, base, count * itemsize).view(dtype)

        # records live at survivor slots; re-index everything by the visible
        # rank (ascending Gaussian index) for the caller
        vis = arr(v.vis, n, 4, torch.int32)[:n_vis].long()
        rank = torch.full((max(n, 1),), -1, dtype=torch.long, device=self.ws.device)
        rank[vis] = torch.arange(n_vis, device=self.ws.device)
        return dict(
            n_act=n_act, n_vis=n_vis, n_entries=E, status=status,
            rec0=arr(v.rec0, n, 16, torch.float32).view(n, 4)[vis],
            rec1=arr(v.rec1, n, 16, torch.float32).view(n, 4)[vis],
            rec2=arr(v.rec2, n, 16, torch.float32).view(n, 4)[vis],
            depth=arr(v.depth, n, 4, torch.int32)[vis],
            order=rank[arr(v.order, n, 4, torch.int32)[:n_vis].long()].int(),
            tile_start=arr(v.tile_start, v.n_tiles + 1, 4, torch.int32),
            entries=rank[arr(v.entries, max(E, 1), 4, torch.int32)[:E].long()].int(),
            n_tiles=v.n_tiles,
        )

    def strip_reach(self) -> torch.Tensor:
        """fdgs_debug_strip_reach: uint8[E] strip-culling bits of the last frame
        (bit w: entry staged for warp strip w), entries in debug_views order."""
        cnt = self.debug_views()["n_entries"]
        out = torch.zeros(max(cnt, 1), dtype=torch.uint8, device=self.ws.device)
        check(lib().fdgs_debug_strip_reach(_ptr(self.ws), self.ws_bytes, self._layout_n, self.width, self.height,
                                           self.max_entries, _ptr(out), _stream_ptr(None)))
        return out[:cnt]

    def _slice(self, ptr, base, nbytes):
        off = int(ptr) - base
        return self.ws[off:off + nbytes]


class RenderPipeline:
    """Frame-pipelined rendering of a sequence: `depth` independent workspaces,
    frame k on workspace k mod depth.  Each workspace has a high-priority
    front-end stream (preprocess, sorts, binning) and a low-priority blend
    stream (fdgs_render_split), so the latency-bound front end of later frames
    is scheduled ahead of, and overlaps, the ALU-bound blends.

    graphs (default True): each frame's front end is one CUDA-graph launch
    (fdgs_render_graph_launch_timed) and its blend one kernel launch -- ~0.02
    ms of host time per frame at the device throughput of stream launches
    (DESIGN.md "CUDA graphs"); graphs=False launches the front end's kernels
    one by one (~0.065 ms per frame).  native=True: render_many submits the
    whole batch through fdgs_pipeline_render -- one C call issuing the frames
    in order on the calling thread (with graphs: each slot's graph;
    threads > 1: in parallel by that many host threads, cheaper on the host
    but slower on the device)."""

    def __init__(self, scene: Scene, width: int, height: int, depth: int = 4, max_entries: int | None = None,
                 split: bool = True, copy_streams: int = 1, graphs: bool | None = None, native: bool | None = None,
                 threads: int = 1):
        self.renderers = [Renderer(scene, width, height, max_entries) for _ in range(depth)]
        self.native = False if native is None else bool(native)
        if graphs is None:
            graphs = True
        self.threads = max(1, int(threads))
        self._handle = None
        self._handle_key = None
        self._frame_ev = []
        lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
        self.split = split
        self.graphs = graphs  # the front end as one CUDA-graph launch per frame, the blend launched after it
        self.front = [torch.cuda.Stream(device=scene.device, priority=-1 if split else 0) for _ in range(depth)]
        self.blend = [torch.cuda.Stream(device=scene.device, priority=0) for _ in range(depth)] if split else None
        self.split_ev = [torch.cuda.Event() for _ in range(depth)]
        # reused per-workspace events (created once: no event creation per frame)
        self.done_ev = [torch.cuda.Event() for _ in range(depth)]
        self.fin_ev = [torch.cuda.Event() for _ in range(depth)]
        self.start_ev = torch.cuda.Event()
        self.join_ev = [torch.cuda.Event() for _ in range(2 * depth + copy_streams)]
        # D2H of finished frames (render_many host_outs), alternating over copy streams
        self.copies = [torch.cuda.Stream(device=scene.device) for _ in range(copy_streams)]
        self.depth = depth

    @property
    def streams(self):
        return self.front + (self.blend or [])

    def __del__(self):
        try:
            self._drop_handle()
        except Exception:
            pass

    def _drop_handle(self):
        if self._handle:
            lib().fdgs_pipeline_destroy(self._handle)
        self._handle = None

    def _native_handle(self):
        """fdgs_pipeline over the current workspaces (re-created when one grew)."""
        graphs = [r._ensure_graph().value if self.graphs else None for r in self.renderers]
        key = tuple((r.ws.data_ptr(), r.ws_bytes, r.max_entries, g) for r, g in zip(self.renderers, graphs))
        if self._handle is None or key != self._handle_key:
            self._drop_handle()
            slots = (FdgsPipelineSlot * self.depth)()
            for i, r in enumerate(self.renderers):
                slots[i] = FdgsPipelineSlot(r.ws.data_ptr(), r.ws_bytes, r.max_entries, self.front[i].cuda_stream,
                                            self.blend[i].cuda_stream if self.split else None, graphs[i])
            cps = (C.c_void_p * len(self.copies))(*[c.cuda_stream for c in self.copies])
            h = C.c_void_p()
            check(lib().fdgs_pipeline_create(slots, self.depth, cps, len(self.copies), self.threads, C.byref(h)))
            self._handle, self._handle_key = h, key
        return self._handle

    def _render_native(self, frames, outs, stats, stage_events, main, host_outs, status_out, frame_done):
        n = len(frames)
        jobs = (FdgsFrameJob * max(n, 1))()
        if frame_done is not None:
            while len(self._frame_ev) < n:
                ev = torch.cuda.Event()
                ev.record(main)  # materialise the CUDA event
                self._frame_ev.append(ev)
        for k, fr in enumerate(frames):
            cam, t, ml, mr = fr[:4]
            r = self.renderers[k % self.depth]
            if cam.width != r.width or cam.height != r.height:
                raise ValueError("camera size differs from the renderer's")
            sc = r._scene_for(fr[4] if len(fr) > 4 else None, main)
            pl, pr = r._masks(ml, mr, sc)
            J = jobs[k]
            J.scene = sc.struct
            J.d_mask_l, J.d_mask_r = pl, pr
            J.cam = cam if isinstance(cam, FdgsCamera) else camera_struct(cam)
            J.t = float(t)
            J.d_out_rgb = outs[k].data_ptr()
            if stats is not None:
                J.d_stats = stats[k].data_ptr()
            if host_outs is not None:
                J.h_out_rgb = host_outs[k].data_ptr()
            if status_out is not None:
                J.d_status = status_out[k].data_ptr()
            if frame_done is not None:
                J.done_event = self._frame_ev[k].cuda_event
        evs = None
        if stage_events is not None:
            evs = (C.c_void_p * (5 * n))(*[e.cuda_event for row in stage_events[:n] for e in row])
        check(lib().fdgs_pipeline_render(self._native_handle(), jobs, n, _stream_ptr(main), evs))
        if frame_done is not None:
            for k in range(n):
                frame_done(k, outs[k], None, self._frame_ev[k])
        return outs

    def counters_view(self, i: int) -> torch.Tensor:
        """The 16-byte counter block {n_act, n_vis, n_entries, status} at the head
        of workspace i (include/fdgs.h fdgs_debug_views.counters)."""
        r = self.renderers[i]
        v = FdgsDebugViews()
        check(lib().fdgs_render_debug_views(_ptr(r.ws), r.ws_bytes, r._layout_n, r.width, r.height, r.max_entries,
                                            C.byref(v)))
        off = int(v.counters) - r.ws.data_ptr()
        return r.ws[off:off + 16]

    def render_many_checked(self, frames, outs, stream=None, host_outs=None):
        """render_many, then a check of every frame's status: frames that exceeded
        the tile-entry capacity are re-rendered (synchronously) after growing the
        workspaces.  Returns the per-frame {n_act, n_vis, n_entries, status}."""
        main = stream or torch.cuda.current_stream()
        status = torch.zeros((len(frames), 16), dtype=torch.uint8, device=self.renderers[0].ws.device)
        self.render_many(frames, outs, stream=main, host_outs=host_outs, status_out=status)
        main.synchronize()
        st = status.cpu().view(torch.int32).view(len(frames), 4)
        bad = [k for k in range(len(frames)) if int(st[k, 3]) != _lib.FDGS_OK]
        for k in bad:
            cam, t, ml, mr = frames[k][:4]
            sc = frames[k][4] if len(frames[k]) > 4 else None  # the frame's working set, if any
            r = self.renderers[k % self.depth]
            _, fs = r.render_checked(cam, t, ml, mr, out=outs[k], stream=main, scene=sc)
            st[k] = torch.tensor([fs.n_act, fs.n_vis, fs.n_entries, fs.status], dtype=torch.int32)
            if host_outs is not None:
                host_outs[k].copy_(outs[k])
        return st

    def render_many(self, frames, outs, stats=None, stage_events=None, stream=None, host_outs=None,
                    status_out=None, frame_done=None):
        """frames: list of (cam, t, mask_l, mask_r); outs: list of output tensors.
        host_outs (optional): pinned host tensors; frame k is copied D2H on a
        copy stream as soon as its blend finishes, overlapping the rendering of
        later frames.  status_out (optional): uint8 device tensor [len(frames),
        16] receiving each frame's counter block (an async device copy after
        its blend; status != 0 means the frame overflowed its tile-entry
        capacity and is undefined -- see render_many_checked).  Ordered after
        the current work of `stream` (default: current stream), and `stream`
        waits for every frame (and copy) before continuing.  frame_done
        (optional): called as frame_done(k, outs[k], s, ev) after frame k is
        enqueued: it completes where stream s is now, or (native submission)
        when event ev completes (dist.FrameGather hooks
        the multi-GPU frame gather here).  Async."""
        main = stream or torch.cuda.current_stream()
        if self.native:
            return self._render_native(frames, outs, stats, stage_events, main, host_outs, status_out, frame_done)
        start = self.start_ev
        start.record(main)
        for s in self.streams:
            s.wait_event(start)
        if host_outs is not None:
            for c in self.copies:
                c.wait_event(start)
        for k, fr in enumerate(frames):
            cam, t, ml, mr = fr[:4]
            sc = fr[4] if len(fr) > 4 else None  # optional per-frame scene (a compacted working set)
            i = k % self.depth
            r = self.renderers[i]
            graph = self.graphs and stats is None  # work counters: the counting blend, stream launches
            if graph and self.split:
                if k >= self.depth:  # the workspace is free once its previous blend is done
                    self.done_ev[i].record(self.blend[i])
                    self.front[i].wait_event(self.done_ev[i])
                r.render_graph(cam, t, ml, mr, out=outs[k], stream=self.front[i], scene=sc,
                               blend_stream=self.blend[i], split_event=self.split_ev[i],
                               stage_events=None if stage_events is None else stage_events[k])
                last = self.blend[i]
            elif graph:
                r.render_graph(cam, t, ml, mr, out=outs[k], stream=self.front[i], scene=sc,
                               stage_events=None if stage_events is None else stage_events[k])
                last = self.front[i]
            elif not self.split:
                r.render(cam, t, ml, mr, out=outs[k], stats=None if stats is None else stats[k], stream=self.front[i],
                         stage_events=None if stage_events is None else stage_events[k], scene=sc)
                last = self.front[i]
            else:
                if k >= self.depth:  # the workspace is free once its previous blend is done
                    self.done_ev[i].record(self.blend[i])
                    self.front[i].wait_event(self.done_ev[i])
                r.render_split(cam, t, ml, mr, out=outs[k], stats=None if stats is None else stats[k],
                               stream=self.front[i], blend_stream=self.blend[i], split_event=self.split_ev[i],
                               stage_events=None if stage_events is None else stage_events[k], scene=sc)
                last = self.blend[i]
            if status_out is not None:  # counters of this frame, before the workspace is reused
                with torch.cuda.stream(last):
                    status_out[k].copy_(self.counters_view(i), non_blocking=True)
            if frame_done is not None:
                frame_done(k, outs[k], last, None)
            if host_outs is not None:
                fin = self.fin_ev[i]
                fin.record(last)
                cp = self.copies[k % len(self.copies)]
                cp.wait_event(fin)
                with torch.cuda.stream(cp):
                    host_outs[k].copy_(outs[k], non_blocking=True)
        for s, e in zip(self.streams + (self.copies if host_outs is not None else []), self.join_ev):
            e.record(s)
            main.wait_event(e)
        return outs


# ----------------------------------------------------------- other entries
def validate(scene: Scene, stream=None):
    ws = torch.empty(lib().fdgs_scene_validate_workspace_bytes(), dtype=torch.uint8, device=scene.device)
    bad = C.c_int64(-1)
    st = lib().fdgs_scene_validate(C.byref(scene.struct), C.byref(bad), _ptr(ws), ws.numel(), _stream_ptr(stream))
    return st, bad.value


def log255_opacity(opacity: torch.Tensor, stream=None) -> torch.Tensor:
    out = torch.empty_like(opacity)
    check(lib().fdgs_log255_opacity(_ptr(opacity), opacity.numel(), _ptr(out), _stream_ptr(stream)))
    return out


def keyframe_mask(scene: Scene, cams, t_key: float, out=None, stream=None) -> torch.Tensor:
    """M(t_key) = OR over cams of the visibility decision."""
    out = torch.empty(mask_words(scene.n), dtype=torch.int32, device=scene.device) if out is None else out
    arr = (FdgsCamera * len(cams))(*[camera_struct(c) for c in cams])
    nb = lib().fdgs_keyframe_workspace_bytes(len(cams))
    ws = torch.empty(nb, dtype=torch.uint8, device=scene.device)
    check(lib().fdgs_keyframe_mask(C.byref(scene.struct), arr, len(cams), float(t_key), _ptr(out), _ptr(ws), nb,
                                   _stream_ptr(stream)))
    return out  # ws goes back to torch's stream-ordered cache: safe to reuse after the kernel


def keyframe_mask_contrib(scene: Scene, cams, t_key: float, threshold: float = 0.0, out=None,
                          max_entries: int | None = None, stream=None) -> torch.Tensor:
    """Paper-literal M(t_key): union over cams of {i : Gaussian i's Eq. 2
    blending weights in the view's render sum above `threshold`}.  Synchronous;
    grows the per-view entry capacity on overflow."""
    out = torch.empty(mask_words(scene.n), dtype=torch.int32, device=scene.device) if out is None else out
    arr = (FdgsCamera * len(cams))(*[camera_struct(c) for c in cams])
    cap = int(default_max_entries(scene.n) if max_entries is None else max_entries)
    while True:
        nb = lib().fdgs_keyframe_mask_contrib_workspace_bytes(scene.n, arr, len(cams), cap)
        if nb == 0:
            raise ValueError("invalid keyframe_mask_contrib arguments")
        ws = torch.empty(nb, dtype=torch.uint8, device=scene.device)
        need = C.c_uint32(0)
        st = lib().fdgs_keyframe_mask_contrib(C.byref(scene.struct), arr, len(cams), float(t_key), float(threshold),
                                              cap, _ptr(out), _ptr(ws), nb, C.byref(need), _stream_ptr(stream))
        if st == _lib.FDGS_ERR_OVERFLOW:
            cap = int(min(2 ** 32 - 1, max(2 * cap, need.value + 1)))
            continue
        check(st)
        return out


def mask_or(a: torch.Tensor, b: torch.Tensor, n: int, out=None, stream=None) -> torch.Tensor:
    out = torch.empty_like(a) if out is None else out
    check(lib().fdgs_mask_or(_ptr(a), _ptr(b), int(n), _ptr(out), _stream_ptr(stream)))
    return out


def mask_compact(a: torch.Tensor, n: int, b: torch.Tensor | None = None, stream=None):
    """Ascending indices of the set bits of a|b."""
    idx = torch.empty(max(n, 1), dtype=torch.int32, device=a.device)
    cnt = torch.zeros(1, dtype=torch.int32, device=a.device)
    nb = lib().fdgs_mask_compact_workspace_bytes(int(n))
    ws = torch.empty(nb, dtype=torch.uint8, device=a.device)
    check(lib().fdgs_mask_compact(_ptr(a), _ptr(b), int(n), _ptr(idx), _ptr(cnt), _ptr(ws), nb, _stream_ptr(stream)))
    k = int(cnt.item())
    return idx[:k]


def prune_mask(score: torch.Tensor, n: int, keep: int, out=None, stream=None) -> torch.Tensor:
    """fdgs_prune_mask: bitmask of the `keep` highest scores, ties by
    ascending index.  Asynchronous."""
    if score.dtype != torch.float32 or not score.is_cuda or not score.is_contiguous():
        raise ValueError("score must be a contiguous CUDA float32 tensor")
    out = torch.empty(max(mask_words(n), 1), dtype=torch.int32, device=score.device) if out is None else out
    nb = lib().fdgs_prune_workspace_bytes(int(n))
    ws = torch.empty(nb, dtype=torch.uint8, device=score.device)
    check(lib().fdgs_prune_mask(_ptr(score), int(n), int(keep), _ptr(out), _ptr(ws), nb, _stream_ptr(stream)))
    return out


def stv_score(scene: Scene, cams, ts, percentile: float = 0.9, combine: int = 0, spatial: bool = False,
              gamma: bool = False, max_entries: int | None = None, stream=None, variant: int = 0) -> dict:
    """fdgs_stv_score (Sec. 4.2.1): dict(score[n], spatial[n_ts][n] | None,
    gamma[n] | None) as device float32 tensors.  Synchronous; grows the per-view
    tile-entry capacity and retries on overflow."""
    n = scene.n
    dev = scene.device
    cs = [camera_struct(c) for c in cams]
    arr = (FdgsCamera * len(cs))(*cs)
    tsa = (C.c_float * max(len(ts), 1))(*[float(t) for t in ts])
    score = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
    sp = torch.empty((len(ts), max(n, 1)), dtype=torch.float32, device=dev) if spatial else None
    gm = torch.empty(max(n, 1), dtype=torch.float32, device=dev) if gamma else None
    cap = int(default_max_entries(n) if max_entries is None else max_entries)
    while True:
        opts = _lib.FdgsStvOpts(float(percentile), int(combine), int(variant), cap)
        nb = lib().fdgs_stv_workspace_bytes(n, arr, len(cs), cap)
        if nb == 0:
            raise ValueError("invalid stv_score arguments")
        ws = torch.empty(nb, dtype=torch.uint8, device=dev)
        need = C.c_uint32(0)
        st = lib().fdgs_stv_score(C.byref(scene.struct), arr, len(cs), tsa, len(ts), C.byref(opts), _ptr(score),
                                  _ptr(sp), _ptr(gm), _ptr(ws), nb, C.byref(need), _stream_ptr(stream))
        if st == _lib.FDGS_ERR_OVERFLOW:
            cap = int(min(2 ** 32 - 1, max(2 * cap, need.value + 1)))
            continue
        check(st)
        return dict(score=score[:n], spatial=None if sp is None else sp[:, :n], gamma=None if gm is None else gm[:n],
                    max_entries=int(need.value))


# ------------------------------------------------ Sec. 4.2.2 host logic
def keyframes(frames: int, interval: int) -> list:
    """Key-frame indices at an even interval, last frame appended (R5)."""
    if not (1 <= interval <= max(frames, 1)):
        raise ValueError("interval must be in [1, frames]")
    kf = list(range(0, frames, interval))
    if kf[-1] != frames - 1:
        kf.append(frames - 1)
    return kf


def bracket(kf: list, frame: int):
    """Indices (l, r) of the two bracketing key-frames t_l <= t <= t_r (R4)."""
    lo = [k for k, f in enumerate(kf) if f <= frame]
    hi = [k for k, f in enumerate(kf) if f >= frame]
    left = lo[-1] if lo else 0
    right = hi[0] if hi else len(kf) - 1
    return left, right
