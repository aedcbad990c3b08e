"""Thin ctypes binding of libmp_b200.so (include/mp.h).

Argument marshalling only: every step of the path runs in the CUDA kernels of
the library.  Device buffers are torch CUDA tensors; the library never
allocates.  There is no CPU fallback: if the library is missing this module
raises at import time.

Tensor conventions (byte-identical to the C structs):
  windows   int32  [n, 7]  (frame, x, y, w, h, size_idx, slot)      = mp_window
  boxes     float32 [n, 6] (x1, y1, x2, y2, score, cls-as-int32-bits) = mp_box
  sizes     list of (w, h)
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Sequence

import numpy as _np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# MP_LIB (development A/B runs only) points the binding at another build of
# the same library; by default the in-tree libmp_b200.so is loaded.
LIB_PATH = os.environ.get("MP_LIB") or os.path.join(_HERE, "libmp_b200.so")

MP_OK, MP_ERR_INVALID, MP_ERR_CUDA, MP_ERR_CAPACITY, MP_ERR_UNSUPPORTED = 0, 1, 2, 3, 4
MP_OUT_F32_NCHW, MP_OUT_U8_NHWC = 0, 1
MP_BT709_LIMITED, MP_BT601_LIMITED, MP_BT709_FULL, MP_BT601_FULL = 0, 1, 2, 3


class MPError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: {_lib.mp_status_string(code).decode()} (code {code})")
        self.code = code


class mp_size(C.Structure):
    _fields_ = [("w", C.c_int32), ("h", C.c_int32)]


class mp_plan_params(C.Structure):
    _fields_ = [("W", C.c_int32), ("H", C.c_int32), ("cell_w", C.c_int32), ("cell_h", C.c_int32),
                ("b_proxy", C.c_float), ("k", C.c_int32), ("sizes", C.POINTER(mp_size)),
                ("cost", C.POINTER(C.c_int64))]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(nvcc, sm_100a).  There is no CPU fallback.")
    L = C.CDLL(LIB_PATH)
    vp, sz, i32, f32 = C.c_void_p, C.c_size_t, C.c_int32, C.c_float
    L.mp_status_string.restype = C.c_char_p
    L.mp_status_string.argtypes = [C.c_int]
    L.mp_launches_per_call.restype = i32
    L.mp_launches_per_call.argtypes = [i32]
    L.mp_gather_set_sm_reserve.restype = C.c_int
    L.mp_gather_set_sm_reserve.argtypes = [i32]
    L.mp_plan_workspace_size.restype = sz
    L.mp_plan_workspace_size.argtypes = [C.POINTER(mp_plan_params), i32]
    L.mp_plan_windows.restype = C.c_int
    L.mp_plan_windows.argtypes = [C.POINTER(mp_plan_params), vp, i32, vp, vp, i32, vp, vp, vp, vp, sz, vp]
    L.mp_gather_workspace_size.restype = sz
    L.mp_gather_workspace_size.argtypes = [i32, vp, vp]
    L.mp_gather_resize.restype = C.c_int
    L.mp_gather_resize.argtypes = [vp, i32, i32, i32, i32, vp, vp, i32, i32, vp, vp, vp, vp, C.c_int, vp, vp, sz, vp]
    L.mp_gather_resize_strided.restype = C.c_int
    L.mp_gather_resize_strided.argtypes = [vp, C.c_int64, i32, i32, i32, i32, vp, vp, i32, i32, vp, vp, vp, vp, C.c_int,
                                           vp, vp, sz, vp]
    L.mp_gather_resize_nv12.restype = C.c_int
    L.mp_gather_resize_nv12.argtypes = [vp, C.c_int64, i32, i32, i32, i32, vp, vp, i32, i32, vp, vp, vp, vp, C.c_int,
                                        C.c_int, vp, vp, sz, vp]
    L.mp_proxy_sweep_workspace_size.restype = sz
    L.mp_proxy_sweep_workspace_size.argtypes = [C.POINTER(mp_plan_params), i32]
    L.mp_proxy_sweep.restype = C.c_int
    L.mp_proxy_sweep.argtypes = [C.POINTER(mp_plan_params), vp, i32, vp, i32, vp, vp, vp, vp, sz, vp]
    L.mp_window_set_cost.restype = C.c_int
    L.mp_window_set_cost.argtypes = [C.POINTER(mp_plan_params), vp, i32, vp, vp, i32, vp, vp, vp]
    L.mp_hungarian_workspace_size.restype = sz
    L.mp_hungarian_workspace_size.argtypes = [i32]
    L.mp_hungarian.restype = C.c_int
    L.mp_hungarian.argtypes = [vp, vp, i32, C.c_float, i32, vp, vp, vp, vp, vp, sz, vp]
    dbl = C.c_double
    L.mp_track_resample.restype = C.c_int
    L.mp_track_resample.argtypes = [vp, vp, i32, i32, vp, vp, vp]
    L.mp_dbscan_workspace_size.restype = sz
    L.mp_dbscan_workspace_size.argtypes = [i32]
    L.mp_dbscan.restype = C.c_int
    L.mp_dbscan.argtypes = [vp, i32, i32, dbl, i32, vp, vp, vp, vp, sz, vp]
    L.mp_cluster_centers.restype = C.c_int
    L.mp_cluster_centers.argtypes = [vp, i32, i32, vp, vp, i32, vp, vp, vp, vp]
    L.mp_refine_workspace_size.restype = sz
    L.mp_refine_workspace_size.argtypes = [i32, i32, dbl, i32, i32]
    L.mp_refine_tracks.restype = C.c_int
    L.mp_refine_tracks.argtypes = [vp, vp, i32, i32, vp, vp, vp, i32, i32, i32, dbl, i32, i32, vp, vp, vp, vp, sz,
                                   vp]
    L.mp_remap_nms_workspace_size.restype = sz
    L.mp_remap_nms_workspace_size.argtypes = [i32, i32]
    L.mp_remap_nms.restype = C.c_int
    L.mp_remap_nms.argtypes = [vp, vp, vp, vp, i32, i32, i32, vp, i32, i32, f32, f32, vp, vp, i32, vp, vp, i32, vp,
                               sz, vp]
    return L


_lib = _load()

EXPORTED = ("mp_plan_workspace_size", "mp_plan_windows", "mp_gather_workspace_size", "mp_gather_resize",
            "mp_gather_resize_strided", "mp_proxy_sweep_workspace_size", "mp_proxy_sweep",
            "mp_window_set_cost",
            "mp_remap_nms_workspace_size", "mp_remap_nms", "mp_status_string", "mp_launches_per_call",
            "mp_gather_set_sm_reserve")


def lib():
    return _lib


def status_string(code: int) -> str:
    return _lib.mp_status_string(code).decode()


def launches_per_call(which: int) -> int:
    return int(_lib.mp_launches_per_call(which))


def mp_gather_set_sm_reserve(sms: int) -> None:
    """Process-wide launch setting of the persistent gather: SMs left out of
    its grid for co-running planner CTAs (mp.h; 0 = every SM)."""
    st = _lib.mp_gather_set_sm_reserve(int(sms))
    if st != MP_OK:
        raise MPError(st, "mp_gather_set_sm_reserve")


def _p(t) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


def _dev(t, dtype, name):
    if t is None:
        return
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def _frames_ok(frames, what):
    """Frames may be a CUDA tensor or a page-locked host tensor (zero-copy:
    the gather reads only the window footprints over PCIe)."""
    if frames.dtype != torch.uint8 or frames.dim() != 3 or not (frames.is_cuda or frames.is_pinned()):
        raise ValueError(f"frames must be a uint8 CUDA or pinned host tensor {what}")
    if frames.stride(2) != 1 or frames.stride(1) != frames.shape[2]:
        raise ValueError("frames rows must be contiguous with pitch = shape[2]")


def _stream(stream):
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def _nwin(windows) -> int:
    """Capacity (records) of an int32 [n, 7] windows tensor."""
    if windows is None:
        return 0
    if windows.dim() != 2 or windows.shape[1] != 7:
        raise ValueError("windows must be int32 [n, 7] (mp_window records)")
    return int(windows.shape[0])


def _sizes(sizes: Sequence) -> C.Array:
    arr = (mp_size * len(sizes))()
    for i, (w, h) in enumerate(sizes):
        arr[i].w, arr[i].h = int(w), int(h)
    return arr


class PlanParams:
    """Host-side planner parameters (mp_plan_params); keeps its arrays alive."""

    def __init__(self, W, H, sizes, cost, b_proxy=0.5, cell_w=32, cell_h=32):
        self.W, self.H, self.cell_w, self.cell_h = int(W), int(H), int(cell_w), int(cell_h)
        self.b_proxy = float(b_proxy)
        self.sizes = [(int(w), int(h)) for (w, h) in sizes]
        self.cost = [int(c) for c in cost]
        self._sz = _sizes(self.sizes)
        self._cost = (C.c_int64 * len(self.cost))(*self.cost)
        self.c = mp_plan_params(self.W, self.H, self.cell_w, self.cell_h, C.c_float(self.b_proxy),
                                len(self.sizes), self._sz, self._cost)

    @property
    def grid(self):
        return (-(-self.H // self.cell_h), -(-self.W // self.cell_w))

    def with_b(self, b_proxy: float) -> "PlanParams":
        return PlanParams(self.W, self.H, self.sizes, self.cost, b_proxy, self.cell_w, self.cell_h)


def mp_plan_workspace_size(params: PlanParams, F: int) -> int:
    return int(_lib.mp_plan_workspace_size(C.byref(params.c), int(F)))


def mp_plan_windows(params: PlanParams, scores, F, mask, windows, frame_off, class_count, status, ws,
                    stream=None) -> None:
    """a1-a4.  scores float32 [F,R,C]; mask uint32-as-int32 [F,R,words] or None;
    windows int32 [max,7]; frame_off int32 [F+1]; class_count int32 [k];
    status int32 [1]; ws uint8 workspace."""
    _dev(scores, torch.float32, "scores")
    _dev(mask, torch.int32, "mask")
    _dev(windows, torch.int32, "windows")
    _dev(frame_off, torch.int32, "frame_off")
    _dev(class_count, torch.int32, "class_count")
    _dev(status, torch.int32, "status")
    _dev(ws, torch.uint8, "ws")
    R, Cc = params.grid
    if scores.numel() < int(F) * R * Cc:
        raise ValueError(f"scores must hold F x {R} x {Cc} cells (got {scores.numel()} for F = {F})")
    if mask is not None and mask.numel() < int(F) * R * ((Cc + 31) // 32):
        raise ValueError("mask too small for F frames")
    if frame_off.numel() < int(F) + 1:
        raise ValueError("frame_off needs F + 1 entries")
    max_w = _nwin(windows)
    st = _lib.mp_plan_windows(C.byref(params.c), _p(scores), int(F), _p(mask), _p(windows), max_w,
                              _p(frame_off), _p(class_count), _p(status), _p(ws),
                              0 if ws is None else ws.numel(), _stream(stream))
    if st != MP_OK:
        raise MPError(st, "mp_plan_windows")


def mp_gather_workspace_size(out_dims: Sequence, out_cap: Sequence[int]) -> int:
    cap = (C.c_int32 * len(out_cap))(*[int(c) for c in out_cap])
    return int(_lib.mp_gather_workspace_size(len(out_cap), _sizes(out_dims), cap))


def mp_gather_resize(frame_ptrs, pitch, W, H, F, windows, frame_off, sizes, out_dims, outs, fmt, status, ws,
                     stream=None) -> None:
    """a5.  frame_ptrs int64 CUDA tensor [F] of device-accessible addresses
    (HBM or pinned host) of uint8 [H][pitch] frames; outs = list of k class tensors (f32 [cap,3,oh,ow] or
    u8 [cap,oh,ow,3]); capacity = outs[k].shape[0]."""
    _dev(frame_ptrs, torch.int64, "frame_ptrs")
    if frame_ptrs.numel() < int(F):
        raise ValueError("frame_ptrs needs F entries")
    _dev(windows, torch.int32, "windows")
    _dev(frame_off, torch.int32, "frame_off")
    _dev(status, torch.int32, "status")
    _dev(ws, torch.uint8, "ws")
    k = len(sizes)
    if len(outs) != k or len(out_dims) != k:
        raise ValueError("sizes, out_dims and outs must have one entry per size class")
    odt = torch.float32 if fmt == MP_OUT_F32_NCHW else torch.uint8
    for q, o in enumerate(outs):
        _dev(o, odt, f"outs[{q}]")
    ptrs = (C.c_void_p * k)(*[o.data_ptr() for o in outs])
    cap = (C.c_int32 * k)(*[int(o.shape[0]) for o in outs])
    st = _lib.mp_gather_resize(_p(frame_ptrs), int(pitch), int(W), int(H), int(F), _p(windows), _p(frame_off),
                               _nwin(windows), k,
                               _sizes(sizes), _sizes(out_dims), ptrs, cap, int(fmt), _p(status), _p(ws),
                               ws.numel(), _stream(stream))
    if st != MP_OK:
        raise MPError(st, "mp_gather_resize")


def mp_gather_resize_strided(frames, W, H, windows, frame_off, sizes, out_dims, outs, fmt, status, ws,
                             stream=None) -> None:
    """a5 on a frame batch: frames uint8 tensor [F, H, pitch] in HBM or pinned
    host memory (rows contiguous, pitch % 16 == 0); frame stride taken from
    the tensor."""
    _dev(windows, torch.int32, "windows")
    _dev(frame_off, torch.int32, "frame_off")
    _dev(status, torch.int32, "status")
    _dev(ws, torch.uint8, "ws")
    _frames_ok(frames, "[F, H, pitch]")
    F, Hh, pitch = frames.shape
    k = len(sizes)
    if len(outs) != k or len(out_dims) != k:
        raise ValueError("sizes, out_dims and outs must have one entry per size class")
    odt = torch.float32 if fmt == MP_OUT_F32_NCHW else torch.uint8
    for q, o in enumerate(outs):
        _dev(o, odt, f"outs[{q}]")
    ptrs = (C.c_void_p * k)(*[o.data_ptr() for o in outs])
    cap = (C.c_int32 * k)(*[int(o.shape[0]) for o in outs])
    st = _lib.mp_gather_resize_strided(_p(frames), int(frames.stride(0)), int(pitch), int(W), int(H), int(F),
                                       _p(windows), _p(frame_off), _nwin(windows), k, _sizes(sizes), _sizes(out_dims),
                                       ptrs, cap, int(fmt), _p(status), _p(ws), ws.numel(), _stream(stream))
    if st != MP_OK:
        raise MPError(st, "mp_gather_resize_strided")


def mp_gather_resize_nv12(frames, W, H, windows, frame_off, sizes, out_dims, outs, fmt, status, ws,
                          matrix=MP_BT709_LIMITED, stream=None) -> None:
    """a5 from NV12 decoder output (NEXT-3, R23): frames uint8 CUDA (or pinned
    host, zero-copy) tensor
    [F, H*3/2, pitch] (Y rows then interleaved UV rows, pitch % 16 == 0)."""
    _dev(windows, torch.int32, "windows")
    _dev(frame_off, torch.int32, "frame_off")
    _dev(status, torch.int32, "status")
    _dev(ws, torch.uint8, "ws")
    _frames_ok(frames, "[F, H*3/2, pitch]")
    F, rows, pitch = frames.shape
    if rows != int(H) + int(H) // 2:
        raise ValueError("NV12 frames need H*3/2 rows")
    k = len(sizes)
    if len(outs) != k or len(out_dims) != k:
        raise ValueError("sizes, out_dims and outs must have one entry per size class")
    odt = torch.float32 if fmt == MP_OUT_F32_NCHW else torch.uint8
    for q, o in enumerate(outs):
        _dev(o, odt, f"outs[{q}]")
    ptrs = (C.c_void_p * k)(*[o.data_ptr() for o in outs])
    cap = (C.c_int32 * k)(*[int(o.shape[0]) for o in outs])
    st = _lib.mp_gather_resize_nv12(_p(frames), int(frames.stride(0)), int(pitch), int(W), int(H), int(F),
                                    _p(windows), _p(frame_off), _nwin(windows), k, _sizes(sizes), _sizes(out_dims),
                                    ptrs, cap, int(fmt), int(matrix), _p(status), _p(ws), ws.numel(), _stream(stream))
    if st != MP_OK:
        raise MPError(st, "mp_gather_resize_nv12")


def mp_remap_nms_workspace_size(F: int, max_boxes: int) -> int:
    return int(_lib.mp_remap_nms_workspace_size(int(F), int(max_boxes)))


def mp_remap_nms(boxes, win_box_off, windows, frame_off, F, out_dims, W, H, score_thr, iou_thr, out, out_src,
                 out_frame_off, status, ws, stream=None) -> None:
    """a6-a7.  boxes float32 [max_boxes,6]; win_box_off int32 [n_win+1];
    out float32 [max_out,6]; out_src int32 [max_out]; out_frame_off int32 [F+1]."""
    _dev(boxes, torch.float32, "boxes")
    _dev(win_box_off, torch.int32, "win_box_off")
    _dev(windows, torch.int32, "windows")
    _dev(frame_off, torch.int32, "frame_off")
    _dev(out, torch.float32, "out")
    _dev(out_src, torch.int32, "out_src")
    _dev(out_frame_off, torch.int32, "out_frame_off")
    _dev(status, torch.int32, "status")
    _dev(ws, torch.uint8, "ws")
    st = _lib.mp_remap_nms(_p(boxes), _p(win_box_off), _p(windows), _p(frame_off), _nwin(windows), int(F),
                           len(out_dims),
                           _sizes(out_dims), int(W), int(H), C.c_float(score_thr), C.c_float(iou_thr), _p(out),
                           _p(out_src), int(out.shape[0]), _p(out_frame_off), _p(status),
                           int(boxes.shape[0]), _p(ws), ws.numel(), _stream(stream))
    if st != MP_OK:
        raise MPError(st, "mp_remap_nms")


def mp_proxy_sweep_workspace_size(params: PlanParams, F: int) -> int:
    return int(_lib.mp_proxy_sweep_workspace_size(C.byref(params.c), int(F)))


def mp_proxy_sweep(params: PlanParams, scores, F, thresholds, dets, det_off, out, ws, stream=None) -> None:
    """NEXT-1 proxy-module sweep.  scores float32 [F,R,C];
    thresholds: host sequence of J floats; dets float32 [n,4] frame px;
    det_off int32 [F+1]; out int64 [J,5] (cost_sum, windows, full_frames,
    dets_covered, dets_touched)."""
    _dev(scores, torch.float32, "scores")
    _dev(dets, torch.float32, "dets")
    _dev(det_off, torch.int32, "det_off")
    _dev(out, torch.int64, "out")
    _dev(ws, torch.uint8, "ws")
    th = (C.c_float * len(thresholds))(*[float(t) for t in thresholds])
    st = _lib.mp_proxy_sweep(C.byref(params.c), _p(scores), int(F), th, len(thresholds), _p(dets), _p(det_off),
                             _p(out), _p(ws), ws.numel(), _stream(stream))
    if st != MP_OK:
        raise MPError(st, "mp_proxy_sweep")


def mp_window_set_cost(params: PlanParams, scores, F, cand, cand_cost, tot, status, stream=None) -> None:
    """NEXT-2 greedy-step objective: tot[c] = sum_t
    est(R(I_t; S + {cand[c]})).  cand int32 CUDA tensor [n_cand, 2] (w, h);
    cand_cost int64 CUDA [n_cand]; tot int64 CUDA [n_cand]; status int32
    CUDA [1] (MP_ERR_INVALID for invalid candidates, whose tot = INT64_MAX)."""
    _dev(scores, torch.float32, "scores")
    _dev(cand, torch.int32, "cand")
    _dev(cand_cost, torch.int64, "cand_cost")
    _dev(tot, torch.int64, "tot")
    _dev(status, torch.int32, "status")
    n = int(cand.shape[0])
    if cand.dim() != 2 or cand.shape[1] != 2 or cand_cost.numel() < n or tot.numel() < n:
        raise ValueError("cand must be [n, 2] int32 with n costs and n totals")
    st = _lib.mp_window_set_cost(C.byref(params.c), _p(scores), int(F), _p(cand), _p(cand_cost), n, _p(tot),
                                 _p(status), _stream(stream))
    if st != MP_OK:
        raise MPError(st, "mp_window_set_cost")


# --------------------------------------------------------------------------- NEXT-4a

ASSIGN_PROBLEM_DTYPE = _np.dtype([("score_off", "<i8"), ("m", "<i4"), ("n", "<i4"), ("row_off", "<i4"),
                                  ("col_off", "<i4")])   # = mp_assign_problem, 24 bytes


def assign_problems(ms, ns):
    """Host-side packing of a batch of [m_b][n_b] score matrices laid out back
    to back: returns (mp_assign_problem records as a numpy structured array,
    total score count, total rows, total columns)."""
    ms = _np.asarray(ms, _np.int64)
    ns = _np.asarray(ns, _np.int64)
    rec = _np.zeros(len(ms), ASSIGN_PROBLEM_DTYPE)
    so = _np.concatenate([[0], _np.cumsum(ms * ns)])
    ro = _np.concatenate([[0], _np.cumsum(ms)])
    co = _np.concatenate([[0], _np.cumsum(ns)])
    rec["score_off"], rec["m"], rec["n"] = so[:-1], ms, ns
    rec["row_off"], rec["col_off"] = ro[:-1], co[:-1]
    return rec, int(so[-1]), int(ro[-1]), int(co[-1])


def mp_hungarian_workspace_size(B: int) -> int:
    return int(_lib.mp_hungarian_workspace_size(int(B)))


def mp_hungarian(scores, problems, B, floor_, max_dim, row_match, col_match, total, status, ws,
                 stream=None) -> None:
    """NEXT-4a batched matching (R24).  scores float32 CUDA [total]; problems
    uint8 CUDA [B*24] (ASSIGN_PROBLEM_DTYPE records); row_match / col_match
    int32 CUDA; total float64 CUDA [B]."""
    _dev(scores, torch.float32, "scores")
    _dev(problems, torch.uint8, "problems")
    _dev(row_match, torch.int32, "row_match")
    _dev(col_match, torch.int32, "col_match")
    _dev(total, torch.float64, "total")
    _dev(status, torch.int32, "status")
    _dev(ws, torch.uint8, "ws")
    if problems.numel() < 24 * int(B):
        raise ValueError("problems must hold B mp_assign_problem records")
    st = _lib.mp_hungarian(_p(scores), _p(problems), int(B), float(floor_), int(max_dim), _p(row_match),
                           _p(col_match), _p(total), _p(status), _p(ws), ws.numel(), _stream(stream))
    if st != MP_OK:
        raise MPError(st, "mp_hungarian")


# --------------------------------------------------------------------------- NEXT-4b
def mp_track_resample(boxes, track_off, T, N, paths, ends=None, stream=None) -> None:
    """R25: boxes float32 CUDA [n_det, 4]; track_off int32 [T+1]; paths float64
    [T, N, 2]; ends float64 [T, 4] or None."""
    _dev(boxes, torch.float32, "boxes")
    _dev(track_off, torch.int32, "track_off")
    _dev(paths, torch.float64, "paths")
    _dev(ends, torch.float64, "ends")
    st = _lib.mp_track_resample(_p(boxes), _p(track_off), int(T), int(N), _p(paths), _p(ends), _stream(stream))
    if st != MP_OK:
        raise MPError(st, "mp_track_resample")


def mp_dbscan_workspace_size(T: int) -> int:
    return int(_lib.mp_dbscan_workspace_size(int(T)))


def mp_dbscan(paths, T, N, eps, min_pts, labels, is_core, nclust, ws, stream=None) -> None:
    """R26: labels int32 [T]; is_core uint8 [T] or None; nclust int32 [2]."""
    _dev(paths, torch.float64, "paths")
    _dev(labels, torch.int32, "labels")
    _dev(is_core, torch.uint8, "is_core")
    _dev(nclust, torch.int32, "nclust")
    _dev(ws, torch.uint8, "ws")
    st = _lib.mp_dbscan(_p(paths), int(T), int(N), float(eps), int(min_pts), _p(labels), _p(is_core), _p(nclust),
                        _p(ws), ws.numel(), _stream(stream))
    if st != MP_OK:
        raise MPError(st, "mp_dbscan")


def mp_cluster_centers(paths, T, N, labels, nclust, C_max, centers, counts, status, stream=None) -> None:
    _dev(paths, torch.float64, "paths")
    _dev(labels, torch.int32, "labels")
    _dev(nclust, torch.int32, "nclust")
    _dev(centers, torch.float64, "centers")
    _dev(counts, torch.int32, "counts")
    _dev(status, torch.int32, "status")
    st = _lib.mp_cluster_centers(_p(paths), int(T), int(N), _p(labels), _p(nclust), int(C_max), _p(centers),
                                 _p(counts), _p(status), _stream(stream))
    if st != MP_OK:
        raise MPError(st, "mp_cluster_centers")


def mp_refine_workspace_size(W, H, cell, C_max, N) -> int:
    return int(_lib.mp_refine_workspace_size(int(W), int(H), float(cell), int(C_max), int(N)))


def mp_refine_tracks(paths, ends, Q, N, centers, counts, nclust, C_max, W, H, cell, k, max_cand, out, taken, status,
                     ws, stream=None) -> None:
    """R27: out float64 [Q, 4]; taken int32 [Q]."""
    for t, dt, nm in ((paths, torch.float64, "paths"), (ends, torch.float64, "ends"), (centers, torch.float64,
                      "centers"), (counts, torch.int32, "counts"), (nclust, torch.int32, "nclust"),
                      (out, torch.float64, "out"), (taken, torch.int32, "taken"), (status, torch.int32, "status"),
                      (ws, torch.uint8, "ws")):
        _dev(t, dt, nm)
    st = _lib.mp_refine_tracks(_p(paths), _p(ends), int(Q), int(N), _p(centers), _p(counts), _p(nclust),
                               int(C_max), int(W), int(H), float(cell), int(k), int(max_cand), _p(out), _p(taken),
                               _p(status), _p(ws), ws.numel(), _stream(stream))
    if st != MP_OK:
        raise MPError(st, "mp_refine_tracks")
