"""WindowPipeline — the public API a user calls for the whole hot path.

It owns the device buffers (torch CUDA tensors) and runs, on one stream and
without host synchronisation, the three C-ABI calls of libmp_b200.so:

    plan(scores)            a1-a4  mp_plan_windows
    gather(frames)          a5     mp_gather_resize -> one batched tensor per size class
    merge(boxes, offsets)   a6-a7  mp_remap_nms

Buffers are sized once (`reserve`) and reused, so a step is graph-capturable.
All arithmetic runs in the CUDA kernels; torch only provides memory/streams.
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import torch

from . import _binding as B


class WindowPipeline:
    def __init__(self, W: int, H: int, sizes: Sequence[Tuple[int, int]], cost: Sequence[int],
                 out_dims: Sequence[Tuple[int, int]], b_proxy: float = 0.5, score_thr: float = 0.25,
                 iou_thr: float = 0.5, fmt: int = B.MP_OUT_F32_NCHW, cell: int = 32, device="cuda",
                 want_mask: bool = False):
        self.params = B.PlanParams(W, H, sizes, cost, b_proxy, cell, cell)
        self.W, self.H = int(W), int(H)
        self.pitch = (3 * self.W + 15) // 16 * 16
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
        dev = self.device
        R, C = self.params.grid
        if F != self.F or max_windows != self.max_windows:
            self.F, self.max_windows = int(F), int(max_windows)
            self.windows = torch.zeros((max(self.max_windows, 1), 7), dtype=torch.int32, device=dev)
            self.frame_off = torch.zeros(self.F + 1, dtype=torch.int32, device=dev)
            self.class_count = torch.zeros(self.k, dtype=torch.int32, device=dev)
            self.mask = (torch.zeros((self.F, R, (C + 31) // 32), dtype=torch.int32, device=dev)
                         if self.want_mask else None)
            self.plan_ws = torch.empty(max(B.mp_plan_workspace_size(self.params, self.F), 1), dtype=torch.uint8,
                                       device=dev)
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
        F = scores.shape[0]
        B.mp_plan_windows(self.params, scores, F, self.mask, self.windows, self.frame_off, self.class_count,
                          self.status, self.plan_ws, stream)

    def gather(self, frames: torch.Tensor, stream=None):
        """frames: either a uint8 [F, H, pitch] batch tensor (TMA tensor path,
        mp_gather_resize_strided) or an int64 [F] tensor of frame addresses
        (pointer-array path, mp_gather_resize)."""
        if frames.dtype == torch.uint8:
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
    def frame_ptrs(frames: torch.Tensor) -> torch.Tensor:
        """Device address of each frame of a uint8 [F,H,pitch] tensor."""
        F = frames.shape[0]
        step = frames.stride(0) * frames.element_size()
        return (torch.arange(F, dtype=torch.int64, device=frames.device) * step + frames.data_ptr()).contiguous()
