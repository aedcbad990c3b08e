"""WindowPipeline — the public API a user calls for the whole hot path.

It owns the device buffers (torch CUDA tensors) and runs, on one stream and
without host synchronisation, the three C-ABI calls of libmp_b200.so:

    proxy_input(frames)     NEXT-3 full-frame downscale to the proxy's input
                                   resolution, optional
    plan(scores)            a1-a4  mp_plan_windows
    gather(frames)          a5     mp_gather_resize[_strided|_nv12] -> one batched
                                   tensor per size class
    merge(boxes, offsets)   a6-a7  mp_remap_nms

Frames are RGB24 rows (src="rgb24") or NV12 decoder output (src="nv12",
[F, H*3/2, pitch] uint8, reading R23).

Buffers are sized once (`reserve`) and reused, so a step is graph-capturable.
All arithmetic runs in the CUDA kernels; torch only provides memory/streams.
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import torch

from . import _binding as B


class _ranges:
    """Host-side range of one runner call, visible to nsys / ncu (NVTX) and to
    torch.profiler traces (record_function)."""

    def __init__(self, name):
        self.name = name
        self.rf = torch.profiler.record_function(name)

    def __enter__(self):
        torch.cuda.nvtx.range_push(self.name)
        self.rf.__enter__()

    def __exit__(self, *exc):
        self.rf.__exit__(*exc)
        torch.cuda.nvtx.range_pop()
        return False


class WindowPipeline:
    def __init__(self, W: int, H: int, sizes: Sequence[Tuple[int, int]], cost: Sequence[int],
                 out_dims: Sequence[Tuple[int, int]], b_proxy: float = 0.5, score_thr: float = 0.25,
                 iou_thr: float = 0.5, fmt: int = B.MP_OUT_F32_NCHW, cell: int = 32, device="cuda",
                 want_mask: bool = False, src: str = "rgb24", matrix: int = B.MP_BT709_LIMITED,
                 proxy_dims: Optional[Tuple[int, int]] = None):
        if src not in ("rgb24", "nv12"):
            raise ValueError("src must be 'rgb24' or 'nv12'")
        self.params = B.PlanParams(W, H, sizes, cost, b_proxy, cell, cell)
        self.W, self.H = int(W), int(H)
        self.src, self.matrix = src, int(matrix)
        self.proxy_dims = (int(proxy_dims[0]), int(proxy_dims[1])) if proxy_dims else None
        self.pitch = (3 * self.W + 15) // 16 * 16 if src == "rgb24" else (self.W + 15) // 16 * 16
        self.sizes = list(self.params.sizes)
        self.out_dims = [(int(a), int(b)) for (a, b) in out_dims]
        self.k = len(self.sizes)
        self.score_thr, self.iou_thr, self.fmt = float(score_thr), float(iou_thr), int(fmt)
        self.device = torch.device(device)
        self.want_mask = want_mask
        self.F = 0
        self.max_windows = 0
        self.caps = [0] * self.k
        self.max_boxes = 0
        self.max_out = 0
        self.status = torch.zeros(1, dtype=torch.int32, device=self.device)

    # ------------------------------------------------------------ buffers
    def reserve(self, F: int, max_windows: int, caps: Optional[Sequence[int]] = None, max_boxes: int = 0,
                max_out: Optional[int] = None):
        """Size the buffers for batches of F frames.  The window buffers only
        grow (a smaller max_windows for the same F keeps them, and the planned
        windows in them), so plan -> reserve(caps from the plan) -> gather
        works without re-planning."""
        dev = self.device
        R, C = self.params.grid
        if F != self.F or max_windows > self.max_windows:
            self.F, self.max_windows = int(F), int(max_windows)
            self.windows = torch.zeros((max(self.max_windows, 1), 7), dtype=torch.int32, device=dev)
            self.frame_off = torch.zeros(self.F + 1, dtype=torch.int32, device=dev)
            self.class_count = torch.zeros(self.k, dtype=torch.int32, device=dev)
            self.mask = (torch.zeros((self.F, R, (C + 31) // 32), dtype=torch.int32, device=dev)
                         if self.want_mask else None)
            self.plan_ws = torch.empty(max(B.mp_plan_workspace_size(self.params, self.F), 1), dtype=torch.uint8,
                                       device=dev)
            if self.proxy_dims:
                # one full-frame window per frame in a single class whose output is the proxy resolution
                pw, ph = self.proxy_dims
                f = torch.arange(self.F, dtype=torch.int32)
                z = torch.zeros_like(f)
                self.proxy_windows = torch.stack([f, z, z, z + self.W, z + self.H, z, f], 1).contiguous().to(dev) \
                    if self.F else torch.zeros((1, 7), dtype=torch.int32, device=dev)
                self.proxy_frame_off = torch.arange(self.F + 1, dtype=torch.int32).to(dev)
                self.proxy_out = torch.empty((self.F, 3, ph, pw), dtype=torch.float32, device=dev)
                self.proxy_ws = torch.empty(max(B.mp_gather_workspace_size([self.proxy_dims], [self.F]), 1),
                                            dtype=torch.uint8, device=dev)
        if caps is not None and list(caps) != self.caps:
            self.caps = [int(c) for c in caps]
            self.outs = []
            for q, (ow, oh) in enumerate(self.out_dims):
                if self.fmt == B.MP_OUT_F32_NCHW:
                    self.outs.append(torch.empty((self.caps[q], 3, oh, ow), dtype=torch.float32, device=dev))
                else:
                    self.outs.append(torch.empty((self.caps[q], oh, ow, 3), dtype=torch.uint8, device=dev))
            self.gather_ws = torch.empty(max(B.mp_gather_workspace_size(self.out_dims, self.caps), 1), dtype=torch.uint8,
                                         device=dev)
        if max_boxes and (max_boxes != self.max_boxes or F != getattr(self, "_nms_F", -1)):
            self.max_boxes = int(max_boxes)
            self._nms_F = F
            self.max_out = int(max_out if max_out is not None else max_boxes)
            self.nms_out = torch.zeros((max(self.max_out, 1), 6), dtype=torch.float32, device=dev)
            self.nms_src = torch.zeros(max(self.max_out, 1), dtype=torch.int32, device=dev)
            self.nms_frame_off = torch.zeros(self.F + 1, dtype=torch.int32, device=dev)
            self.nms_ws = torch.empty(max(B.mp_remap_nms_workspace_size(self.F, self.max_boxes), 1),
                                      dtype=torch.uint8, device=dev)

    # ------------------------------------------------------------ steps
    def plan(self, scores: torch.Tensor, stream=None):
        R, C = self.params.grid
        if tuple(scores.shape) != (self.F, R, C):
            raise ValueError(f"scores must be [{self.F}, {R}, {C}] (reserved F x grid), got {tuple(scores.shape)}")
        F = self.F
        B.mp_plan_windows(self.params, scores, F, self.mask, self.windows, self.frame_off, self.class_count,
                          self.status, self.plan_ws, stream)

    def proxy_input(self, frames: torch.Tensor, stream=None):
        """NEXT-3: every frame downscaled (R15 bilinear; NV12 converted, R23) to
        the proxy's input resolution -> self.proxy_out f32 [F, 3, ph, pw]."""
        if not self.proxy_dims:
            raise ValueError("pipeline built without proxy_dims")
        one = [(self.W, self.H)]
        if self.src == "nv12":
            B.mp_gather_resize_nv12(frames, self.W, self.H, self.proxy_windows, self.proxy_frame_off, one,
                                    [self.proxy_dims], [self.proxy_out], B.MP_OUT_F32_NCHW, self.status,
                                    self.proxy_ws, self.matrix, stream)
        else:
            B.mp_gather_resize_strided(frames, self.W, self.H, self.proxy_windows, self.proxy_frame_off, one,
                                       [self.proxy_dims], [self.proxy_out], B.MP_OUT_F32_NCHW, self.status,
                                       self.proxy_ws, stream)

    def gather(self, frames: torch.Tensor, stream=None):
        """frames: a uint8 [F, H, pitch] RGB24 batch tensor (TMA tensor path,
        mp_gather_resize_strided), an int64 [F] tensor of RGB24 frame addresses
        (pointer-array path, mp_gather_resize), or, with src="nv12", a uint8
        [F, H*3/2, pitch] NV12 batch (mp_gather_resize_nv12).  Frames may sit
        in HBM or in pinned host memory: from the host the kernels read only
        the window footprints over PCIe (zero-copy, same bits)."""
        if self.src == "nv12":
            B.mp_gather_resize_nv12(frames, self.W, self.H, self.windows, self.frame_off, self.sizes,
                                    self.out_dims, self.outs, self.fmt, self.status, self.gather_ws, self.matrix,
                                    stream)
        elif frames.dtype == torch.uint8:
            B.mp_gather_resize_strided(frames, self.W, self.H, self.windows, self.frame_off, self.sizes,
                                       self.out_dims, self.outs, self.fmt, self.status, self.gather_ws, stream)
        else:
            B.mp_gather_resize(frames, self.pitch, self.W, self.H, self.F, self.windows, self.frame_off,
                               self.sizes, self.out_dims, self.outs, self.fmt, self.status, self.gather_ws, stream)

    def merge(self, boxes: torch.Tensor, win_box_off: torch.Tensor, stream=None):
        B.mp_remap_nms(boxes, win_box_off, self.windows, self.frame_off, self.F, self.out_dims, self.W, self.H,
                       self.score_thr, self.iou_thr, self.nms_out, self.nms_src, self.nms_frame_off, self.status,
                       self.nms_ws, stream)

    def check_status(self):
        st = int(self.status.item())
        if st != B.MP_OK:
            raise B.MPError(st, "device status")

    # ------------------------------------------------------------ helpers
    @staticmethod
    def frame_ptrs(frames: torch.Tensor, device=None) -> torch.Tensor:
        """Address of each frame of a uint8 [F,H,pitch] tensor, as an int64
        tensor on `device` (default: the frames' device).  Frames in pinned
        host memory give host addresses the gather reads zero-copy (only the
        window footprints cross PCIe); their list goes to `device`."""
        F = frames.shape[0]
        step = frames.stride(0) * frames.element_size()
        if not frames.is_cuda and not frames.is_pinned():
            raise ValueError("frames must be in HBM or in pinned host memory")
        dev = frames.device if device is None else torch.device(device)
        ptrs = torch.arange(F, dtype=torch.int64, device=frames.device) * step + frames.data_ptr()
        return ptrs.to(dev).contiguous()


class PipelinedRunner:
    """Software pipeline over consecutive batches on three CUDA streams:
    plan(i+1) and remap/NMS(i-1) run while gather/resize(i) streams through HBM.

    With proxy_dims set (NEXT-3), proxy_input(i) runs on a fourth stream and
    plan(i) waits for it (the proxy consumes that downscale), so the downscale
    of batch i+1 overlaps the gather of batch i.

    Each in-flight batch owns one WindowPipeline (`depth` sets of plan/gather/
    NMS buffers), so no stage of batch i+1 overwrites a buffer a later stage of
    batch i still reads.  Ordering is enforced only with CUDA events (no host
    synchronisation):
        caller's stream -> plan(i) -> gather(i) -> [detector] -> merge(i);
        plan(i) waits merge(i-depth).

    Two ways to drive it:
      * `enqueue(scores, frames)` (plan + gather of one batch, returns its
        buffer-set index k; the detector reads `pipes[k].outs` after
        `wait_gathered(k)`), then `merge(k, boxes, win_box_off,
        detector_done=event)` once the detector has produced the boxes; the
        merge waits for `detector_done`, so the next batch that reuses set k
        cannot overwrite `outs` while the detector still reads them;
      * `step(scores, frames, boxes, win_box_off)` = both at once (stand-in
        detections known in advance, as in bench.py).
    Every call first makes the side streams wait for the caller's current
    stream (inputs written there, e.g. non_blocking H2D copies, are complete)
    and records the caller's tensors on the side streams (record_stream), so
    the caching allocator does not hand their memory out while they are read.
    """

    def __init__(self, pipes, device="cuda", merge_on_gather_stream: bool = False, side_streams: int = 1,
                 plan_priority: bool = True, gather_sm_reserve: Optional[int] = None):
        self.pipes = list(pipes)
        # SMs the persistent gather leaves to the co-running planner of the
        # next batch (mp_gather_set_sm_reserve, a process-wide launch setting,
        # set here when given; None leaves it as it is): only for plan-bound
        # steps (4K dense frames, u8 output, DESIGN 6f)
        self.gather_sm_reserve = gather_sm_reserve
        if gather_sm_reserve is not None:
            B.mp_gather_set_sm_reserve(int(gather_sm_reserve))
        self.depth = len(self.pipes)
        self.dev = torch.device(device)
        dev = self.dev
        # side_streams > 1: plan and remap/NMS of consecutive batches run on
        # their own streams (set k uses stream k mod side_streams), so the
        # plans (and merges) of two batches may overlap each other
        n = max(1, min(int(side_streams), self.depth))
        # plan(i+1) gates gather(i+1): with plan_priority its streams have the
        # highest priority, so the block scheduler places its CTAs before the
        # remap/NMS CTAs that compete for the SM space the gather leaves
        prio = torch.cuda.Stream.priority_range()[1] if plan_priority else 0
        self.s_plans = [torch.cuda.Stream(dev, priority=prio) for _ in range(n)]
        self.s_plan = self.s_plans[0]
        self.s_gather = torch.cuda.Stream(dev)
        # merge_on_gather_stream: remap/NMS(i) runs right after gather(i) on the
        # gather stream instead of concurrently with gather(i+1)
        self.s_merges = [self.s_gather] if merge_on_gather_stream else [torch.cuda.Stream(dev) for _ in range(n)]
        self.s_merge = self.s_merges[0]
        self.s_proxy = torch.cuda.Stream(dev) if self.pipes[0].proxy_dims else None
        self.done = [None] * self.depth       # merge(i) finished -> set k reusable
        self.gathered = [None] * self.depth   # gather(i) finished -> set k's outs readable
        self.pending = [False] * self.depth   # set k enqueued, merge not yet enqueued
        self.static = None                    # graph mode: runner-owned inputs per set
        self.i = 0
        self._capturing = False
        self.g_steps = None                   # capture_steps(): U whole steps as one graph

    # ------------------------------------------------------------ graphs
    def capture_graphs(self, scores, boxes=None, win_box_off=None):
        """Capture each buffer set's plan and merge calls (latency-bound
        launches) as CUDA graphs over runner-OWNED static input tensors
        (copies of the examples given here).  `enqueue`/`merge` then copy each
        batch's inputs into them before the replay — or skip the copy when the
        caller already wrote into `inputs(k)` in place.  The gather stays a
        plain launch so its duration can be timed with events on its stream."""
        if any(self.pending):
            raise RuntimeError("capture_graphs with batches in flight")
        torch.cuda.synchronize(self.dev)
        self.g_plan, self.g_merge, self.static = [], [], []
        for k, p in enumerate(self.pipes):
            sp, sm = self.s_plans[k % len(self.s_plans)], self.s_merges[k % len(self.s_merges)]
            st = {"scores": scores.detach().clone(),
                  "boxes": None if boxes is None else boxes.detach().clone(),
                  "win_box_off": None if win_box_off is None else win_box_off.detach().clone()}
            self.static.append(st)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=sp):
                p.plan(st["scores"], stream=sp)
            self.g_plan.append(g)
            if boxes is not None:
                g2 = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g2, stream=sm):
                    p.merge(st["boxes"], st["win_box_off"], stream=sm)
                self.g_merge.append(g2)
        torch.cuda.synchronize(self.dev)

    def capture_steps(self, batches, gather_events=None):
        """Capture len(batches) consecutive whole steps — plan, gather and
        remap/NMS of each batch on the runner's streams, with the same
        cross-batch event ordering as `step` — as ONE CUDA graph;
        `replay_steps()` then issues all of them with a single launch (small
        batches, e.g. configs[0]'s 30 frames, are otherwise bound by the
        host-side issue of ~20 launches and events per step).

        batches: [(scores, frames, boxes, win_box_off), ...]; the graph keeps
        reading these tensors (and the frames' addresses, baked into the TMA
        descriptors), so the caller keeps them alive and rewrites them in place
        between replays.  gather_events: optional [(start, end)] per batch,
        created with torch.cuda.Event(enable_timing=True, external=True) so
        they are recorded as graph nodes on every replay.  A replay starts
        after all earlier work of the capture stream and ends with every
        stream joined (no overlap across replays)."""
        if any(self.pending):
            raise RuntimeError("capture_steps with batches in flight")
        if self.static is not None:
            raise RuntimeError("capture_steps and capture_graphs are exclusive")
        torch.cuda.synchronize(self.dev)
        self.done = [None] * self.depth
        self.gathered = [None] * self.depth
        self.i = 0
        cap = torch.cuda.Stream(self.dev)
        g = torch.cuda.CUDAGraph()
        self._capturing = True
        try:
            with torch.cuda.graph(g, stream=cap):
                for u, (sc, fr, bx, wbo) in enumerate(batches):
                    ev = gather_events[u] if gather_events is not None else None
                    self.step(sc, fr, bx, wbo, gather_events=ev)
                self.wait_all(cap)
        finally:
            self._capturing = False
            self.done = [None] * self.depth
            self.gathered = [None] * self.depth
            self.pending = [False] * self.depth
            self.i = 0
        torch.cuda.synchronize(self.dev)
        self.g_steps = g
        self.n_graph_steps = len(batches)
        return g

    def replay_steps(self):
        """Launch the captured steps on the current stream (see capture_steps)."""
        if self.g_steps is None:
            raise RuntimeError("replay_steps needs capture_steps()")
        self.g_steps.replay()

    def inputs(self, k: Optional[int] = None):
        """Graph mode: the static (scores, boxes, win_box_off) tensors of
        buffer set k (default: the set the next `enqueue` uses).  A caller that
        writes its inputs there in place (on its current stream) saves the
        per-batch copy."""
        if self.static is None:
            raise RuntimeError("inputs() needs capture_graphs()")
        st = self.static[self.i % self.depth if k is None else k]
        return st["scores"], st["boxes"], st["win_box_off"]

    # ------------------------------------------------------------ helpers
    def _caller_ready(self):
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.dev))
        return ev

    def _use(self, t, stream):
        if t is not None and t.is_cuda and not self._capturing:
            t.record_stream(stream)

    @staticmethod
    def _stage(dst, src, stream):
        """Copy a caller tensor into a static graph input on `stream` (no-op
        when the caller passed the static tensor itself)."""
        if src is None or dst is None or src.data_ptr() == dst.data_ptr():
            return
        if src.shape != dst.shape or src.dtype != dst.dtype:
            raise ValueError(f"graph input shape/dtype changed: {tuple(src.shape)} {src.dtype} vs captured "
                             f"{tuple(dst.shape)} {dst.dtype}")
        with torch.cuda.stream(stream):
            dst.copy_(src, non_blocking=True)
        if src.is_cuda:
            src.record_stream(stream)

    # ------------------------------------------------------------ pipeline
    def enqueue(self, scores, frames, gather_events=None, proxy_events=None) -> int:
        """Enqueue plan + gather of one batch; returns its buffer set k.
        gather_events / proxy_events: optional (start, end) CUDA events
        recorded around the gather / the proxy-input downscale."""
        k = self.i % self.depth
        if self.pending[k]:
            raise RuntimeError(f"buffer set {k} still awaits merge() of batch {self.i - self.depth}")
        with _ranges(f"mp.enqueue set {k}"):
            return self._enqueue(k, scores, frames, gather_events, proxy_events)

    def _enqueue(self, k, scores, frames, gather_events, proxy_events) -> int:
        p = self.pipes[k]
        s_plan = self.s_plans[k % len(self.s_plans)]
        ready = self._caller_ready()
        for s in (s_plan, self.s_gather) + ((self.s_proxy,) if self.s_proxy is not None else ()):
            s.wait_event(ready)
            if self.done[k] is not None:
                s.wait_event(self.done[k])   # set k's buffers (windows, outs) are free again
        if self.s_proxy is not None:
            if proxy_events is not None:
                proxy_events[0].record(self.s_proxy)
            p.proxy_input(frames, stream=self.s_proxy)
            self._use(frames, self.s_proxy)
            if proxy_events is not None:
                proxy_events[1].record(self.s_proxy)
            downscaled = torch.cuda.Event()
            downscaled.record(self.s_proxy)
            s_plan.wait_event(downscaled)
        if self.static is not None:
            self._stage(self.static[k]["scores"], scores, s_plan)
            with torch.cuda.stream(s_plan):
                self.g_plan[k].replay()
        else:
            p.plan(scores, stream=s_plan)
            self._use(scores, s_plan)
        planned = torch.cuda.Event()
        planned.record(s_plan)
        self.s_gather.wait_event(planned)
        if gather_events is not None:
            gather_events[0].record(self.s_gather)
        p.gather(frames, stream=self.s_gather)
        self._use(frames, self.s_gather)
        if gather_events is not None:
            gather_events[1].record(self.s_gather)
        gathered = torch.cuda.Event()
        gathered.record(self.s_gather)
        self.gathered[k] = gathered
        self.pending[k] = True
        self.i += 1
        return k

    def wait_gathered(self, k: int, stream=None):
        """Make `stream` (default: current) wait until set k's class tensors
        (pipes[k].outs, the detector's inputs) are written."""
        s = torch.cuda.current_stream(self.dev) if stream is None else stream
        s.wait_event(self.gathered[k])

    def merge(self, k: int, boxes=None, win_box_off=None, detector_done=None):
        """Enqueue remap/NMS of buffer set k's batch (boxes None: no merge, the
        set is just released).  detector_done: event recorded after the
        detector's last read of pipes[k].outs and write of the boxes."""
        if not self.pending[k]:
            raise RuntimeError(f"buffer set {k} has no batch awaiting merge")
        with _ranges(f"mp.merge set {k}"):
            self._merge(k, boxes, win_box_off, detector_done)

    def _merge(self, k, boxes, win_box_off, detector_done):
        p = self.pipes[k]
        s_merge = self.s_merges[k % len(self.s_merges)]
        s_merge.wait_event(self.gathered[k])
        s_merge.wait_event(self._caller_ready())
        if detector_done is not None:
            s_merge.wait_event(detector_done)
        if boxes is not None:
            if self.static is not None and self.g_merge:
                self._stage(self.static[k]["boxes"], boxes, s_merge)
                self._stage(self.static[k]["win_box_off"], win_box_off, s_merge)
                with torch.cuda.stream(s_merge):
                    self.g_merge[k].replay()
            else:
                p.merge(boxes, win_box_off, stream=s_merge)
                self._use(boxes, s_merge)
                self._use(win_box_off, s_merge)
        done = torch.cuda.Event()
        done.record(s_merge)
        self.done[k] = done
        self.pending[k] = False

    def step(self, scores, frames, boxes=None, win_box_off=None, gather_events=None, proxy_events=None):
        """enqueue + merge of one batch whose detector output is already known
        (`boxes`/`win_box_off`; None skips the merge).  Returns its pipeline."""
        k = self.enqueue(scores, frames, gather_events, proxy_events)
        self.merge(k, boxes, win_box_off)
        return self.pipes[k]

    def wait_all(self, stream=None):
        """Make `stream` (default: current) wait for everything enqueued."""
        s = torch.cuda.current_stream(self.dev) if stream is None else stream
        for e in self.done + self.gathered:
            if e is not None:
                s.wait_event(e)
