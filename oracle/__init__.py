"""CPU ORACLE for the MultiScope proxy-guided window path (test infrastructure).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_2103_14695_b200``) never imports it and shares no code with it.

This module is a ctypes wrapper over ``oracle/mp_oracle.c`` (plain C99, fp64,
built with ``-O2 -ffp-contract=off``); every function there cites the PAPER.md
passage or DESIGN.md reading it follows.  Arrays are numpy.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mp_oracle.c")
_LIB = os.path.join(_HERE, "libmp_oracle.so")

BOX_DTYPE = np.dtype([("x1", "<f4"), ("y1", "<f4"), ("x2", "<f4"), ("y2", "<f4"),
                      ("score", "<f4"), ("cls", "<i4")])
WINDOW_FIELDS = ("frame", "x", "y", "w", "h", "size_idx", "slot")

F32_NCHW, U8_NHWC, F64_NCHW = 0, 1, 2
OK, ERR_INVALID, ERR_CAPACITY = 0, 1, 3


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, no SIMD intrinsics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-std=c99", "-O2", "-ffp-contract=off", "-fno-fast-math",
                               "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        p = C.c_void_p
        i32, i64, f32 = C.c_int32, C.c_int64, C.c_float
        L.mpo_threshold.restype = i64
        L.mpo_threshold.argtypes = [p, i32, i32, f32, p]
        L.mpo_pack_mask.restype = None
        L.mpo_pack_mask.argtypes = [p, i32, i32, p]
        L.mpo_components.restype = i32
        L.mpo_components.argtypes = [p, i32, i32, p, p]
        L.mpo_smallest_window.restype = i32
        L.mpo_smallest_window.argtypes = [p, i32, i32, i32]
        L.mpo_plan_windows.restype = i32
        L.mpo_plan_windows.argtypes = [i32, i32, i32, i32, f32, i32, p, p, p, i32, p, p, i32,
                                       p, p, p]
        L.mpo_taps.restype = None
        L.mpo_taps.argtypes = [i32, i32, i32, p, p, p]
        L.mpo_gather_resize.restype = i32
        L.mpo_gather_resize.argtypes = [p, i32, i32, i32, i32, p, i32, i32, p, p, p, p, i32]
        L.mpo_yuv_to_rgb.restype = i32
        L.mpo_yuv_to_rgb.argtypes = [C.c_double, C.c_double, C.c_double, i32, p]
        L.mpo_gather_resize_nv12.restype = i32
        L.mpo_gather_resize_nv12.argtypes = [p, i32, i32, i32, i32, p, i32, i32, p, p, p, p, i32, i32]
        L.mpo_iou.restype = f32
        L.mpo_iou.argtypes = [BoxC, BoxC]
        L.mpo_remap_box.restype = i32
        L.mpo_remap_box.argtypes = [BoxC, i32, i32, i32, i32, i32, i32, f32, p]
        L.mpo_proxy_sweep.restype = i32
        L.mpo_proxy_sweep.argtypes = [i32, i32, i32, i32, i32, p, p, p, i32, p, i32, p, p, p]
        L.mpo_window_set_cost.restype = i32
        L.mpo_window_set_cost.argtypes = [i32, i32, i32, i32, f32, i32, p, p, p, i32, p, p, i32, p]
        L.mpo_hungarian.restype = i32
        L.mpo_hungarian.argtypes = [p, i32, i32, f32, p, p, p]
        d = C.c_double
        L.mpo_track_resample.restype = None
        L.mpo_track_resample.argtypes = [p, i32, i32, p]
        L.mpo_track_distance.restype = d
        L.mpo_track_distance.argtypes = [p, p, i32]
        L.mpo_dbscan.restype = i32
        L.mpo_dbscan.argtypes = [p, i32, i32, d, i32, p, p, p]
        L.mpo_cluster_centers.restype = None
        L.mpo_cluster_centers.argtypes = [p, i32, i32, p, i32, p, p]
        L.mpo_refine_track.restype = i32
        L.mpo_refine_track.argtypes = [p, i32, p, p, p, p, i32, d, i32, p]
        L.mpo_remap_nms.restype = i32
        L.mpo_remap_nms.argtypes = [p, p, p, p, i32, i32, p, i32, i32, f32, f32, p, p, i32, p]
        _lib = L
    return _lib


class BoxC(C.Structure):
    _fields_ = [("x1", C.c_float), ("y1", C.c_float), ("x2", C.c_float), ("y2", C.c_float),
                ("score", C.c_float), ("cls", C.c_int32)]


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


def _sizes_arr(sizes) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(sizes, dtype=np.int32).reshape(-1, 2))


# --------------------------------------------------------------------------- a1/a2
def threshold(scores: np.ndarray, b_proxy: float) -> np.ndarray:
    s = np.ascontiguousarray(scores, dtype=np.float32)
    R, Cc = s.shape
    pos = np.zeros((R, Cc), np.uint8)
    lib().mpo_threshold(_ptr(s), R, Cc, float(b_proxy), _ptr(pos))
    return pos


def pack_mask(pos: np.ndarray) -> np.ndarray:
    p = np.ascontiguousarray(pos, dtype=np.uint8)
    R, Cc = p.shape
    m = np.zeros((R, (Cc + 31) // 32), np.uint32)
    lib().mpo_pack_mask(_ptr(p), R, Cc, _ptr(m))
    return m


def components(pos: np.ndarray):
    """Returns (labels[R,C] int32 with -1 for background, bbox[n,4] (c0,r0,c1,r1))."""
    p = np.ascontiguousarray(pos, dtype=np.uint8)
    R, Cc = p.shape
    labels = np.empty((R, Cc), np.int32)
    bbox = np.empty((max(R * Cc, 1), 4), np.int32)
    n = lib().mpo_components(_ptr(p), R, Cc, _ptr(labels), _ptr(bbox))
    return labels, bbox[:n].copy()


def smallest_window(sizes, bw: int, bh: int) -> int:
    s = _sizes_arr(sizes)
    return lib().mpo_smallest_window(_ptr(s), len(s), bw, bh)


# --------------------------------------------------------------------------- a1-a4
def plan_windows(W, H, cell_w, cell_h, b_proxy, sizes, cost, scores, max_windows=None):
    """Batched plan (ABI semantics).  scores: float32 [F][R][C].
    Returns dict(status, mask[F,R,words], windows[n,7] int32, frame_off[F+1],
    class_count[k], passes[F])."""
    s = np.ascontiguousarray(scores, dtype=np.float32)
    F = s.shape[0]
    R, Cc = (H + cell_h - 1) // cell_h, (W + cell_w - 1) // cell_w
    assert s.shape[1:] == (R, Cc), (s.shape, R, Cc)
    sz = _sizes_arr(sizes)
    k = len(sz)
    cs = np.ascontiguousarray(np.asarray(cost, dtype=np.int64))
    if max_windows is None:
        max_windows = max(F * ((R * Cc + 1) // 2 + 1), 1)
    mask = np.zeros((F, R, (Cc + 31) // 32), np.uint32)
    win = np.zeros((max(max_windows, 1), 7), np.int32)
    frame_off = np.zeros(F + 1, np.int32)
    cc = np.zeros(k, np.int32)
    passes = np.zeros(max(F, 1), np.int32)
    st = lib().mpo_plan_windows(W, H, cell_w, cell_h, float(b_proxy), k, _ptr(sz), _ptr(cs),
                                _ptr(s), F, _ptr(mask), _ptr(win), max_windows, _ptr(frame_off),
                                _ptr(cc), _ptr(passes))
    n = int(frame_off[F]) if st != ERR_INVALID else 0
    return dict(status=st, mask=mask, windows=win[:min(n, max_windows)].copy(),
                frame_off=frame_off, class_count=cc, passes=passes[:F].copy())


# --------------------------------------------------------------------------- a5
def taps(n_in: int, n_out: int, d: int):
    i0, i1, lam = C.c_int32(), C.c_int32(), C.c_double()
    lib().mpo_taps(n_in, n_out, d, C.byref(i0), C.byref(i1), C.byref(lam))
    return i0.value, i1.value, lam.value


def gather_resize(frames, pitch, W, H, windows, sizes, out_dims, out_cap, fmt=F32_NCHW):
    """frames: list/array of uint8 [H][pitch] host frames (index = window.frame).
    Returns (status, [class tensors])."""
    fr = [np.ascontiguousarray(f, dtype=np.uint8) for f in frames]
    F = len(fr)
    ptrs = (C.c_void_p * max(F, 1))(*[f.ctypes.data for f in fr])
    win = np.ascontiguousarray(np.asarray(windows, dtype=np.int32).reshape(-1, 7))
    sz = _sizes_arr(sizes)
    od = _sizes_arr(out_dims)
    k = len(sz)
    cap = np.ascontiguousarray(np.asarray(out_cap, dtype=np.int32))
    outs = []
    for i in range(k):
        ow, oh = int(od[i, 0]), int(od[i, 1])
        if fmt == U8_NHWC:
            outs.append(np.zeros((cap[i], oh, ow, 3), np.uint8))
        else:
            outs.append(np.zeros((cap[i], 3, oh, ow), np.float64 if fmt == F64_NCHW else np.float32))
    optrs = (C.c_void_p * k)(*[o.ctypes.data for o in outs])
    st = lib().mpo_gather_resize(ptrs, pitch, W, H, F, _ptr(win), len(win), k, _ptr(sz),
                                 _ptr(od), optrs, _ptr(cap), fmt)
    return st, outs


# --------------------------------------------------------------------------- NEXT-3
BT709_LIMITED, BT601_LIMITED, BT709_FULL, BT601_FULL = 0, 1, 2, 3


def yuv_to_rgb(Y, U, V, matrix=BT709_LIMITED):
    """R23 colour conversion of one (Y, U, V) triple -> clamped fp64 (R, G, B)."""
    out = np.zeros(3, np.float64)
    st = lib().mpo_yuv_to_rgb(float(Y), float(U), float(V), int(matrix), _ptr(out))
    if st:
        raise ValueError("bad matrix")
    return out


def gather_resize_nv12(frames, pitch, W, H, windows, sizes, out_dims, out_cap, fmt=F32_NCHW,
                       matrix=BT709_LIMITED):
    """frames: list/array of uint8 [H*3/2][pitch] NV12 host frames (Y rows then
    interleaved UV rows).  Returns (status, [class tensors]) like gather_resize."""
    fr = [np.ascontiguousarray(f, dtype=np.uint8) for f in frames]
    for f in fr:
        if f.shape != (H + H // 2, pitch):
            raise ValueError("NV12 frame must be [H*3/2][pitch]")
    F = len(fr)
    ptrs = (C.c_void_p * max(F, 1))(*[f.ctypes.data for f in fr])
    win = np.ascontiguousarray(np.asarray(windows, dtype=np.int32).reshape(-1, 7))
    sz = _sizes_arr(sizes)
    od = _sizes_arr(out_dims)
    k = len(sz)
    cap = np.ascontiguousarray(np.asarray(out_cap, dtype=np.int32))
    outs = []
    for i in range(k):
        ow, oh = int(od[i, 0]), int(od[i, 1])
        if fmt == U8_NHWC:
            outs.append(np.zeros((cap[i], oh, ow, 3), np.uint8))
        else:
            outs.append(np.zeros((cap[i], 3, oh, ow), np.float64 if fmt == F64_NCHW else np.float32))
    optrs = (C.c_void_p * k)(*[o.ctypes.data for o in outs])
    st = lib().mpo_gather_resize_nv12(ptrs, pitch, W, H, F, _ptr(win), len(win), k, _ptr(sz),
                                      _ptr(od), optrs, _ptr(cap), fmt, int(matrix))
    return st, outs


# --------------------------------------------------------------------------- a6/a7
def _boxc(b) -> BoxC:
    return BoxC(float(b["x1"]), float(b["y1"]), float(b["x2"]), float(b["y2"]),
                float(b["score"]), int(b["cls"]))


def iou(a, b) -> float:
    return float(lib().mpo_iou(_boxc(a), _boxc(b)))


def remap_box(box, window, out_dim, score_thr):
    out = np.zeros(1, BOX_DTYPE)
    x, y, w, h = (int(v) for v in window[1:5]) if len(window) == 7 else (int(v) for v in window)
    ok = lib().mpo_remap_box(_boxc(box), x, y, w, h, int(out_dim[0]), int(out_dim[1]),
                             float(score_thr), _ptr(out))
    return out[0] if ok else None


def remap_nms(boxes, win_box_off, windows, frame_off, out_dims, W, H, score_thr, iou_thr,
              max_out=None):
    """Returns dict(status, boxes (BOX_DTYPE), src int32, frame_off[F+1])."""
    bx = np.ascontiguousarray(np.asarray(boxes, dtype=BOX_DTYPE))
    wbo = np.ascontiguousarray(np.asarray(win_box_off, dtype=np.int32))
    win = np.ascontiguousarray(np.asarray(windows, dtype=np.int32).reshape(-1, 7))
    fo = np.ascontiguousarray(np.asarray(frame_off, dtype=np.int32))
    od = _sizes_arr(out_dims)
    F = len(fo) - 1
    if max_out is None:
        max_out = max(len(bx), 1)
    out = np.zeros(max(max_out, 1), BOX_DTYPE)
    src = np.zeros(max(max_out, 1), np.int32)
    ofo = np.zeros(F + 1, np.int32)
    if len(bx) == 0:
        bx = np.zeros(1, BOX_DTYPE)
    st = lib().mpo_remap_nms(_ptr(bx), _ptr(wbo), _ptr(win), _ptr(fo), F, len(od), _ptr(od), W, H,
                             float(score_thr), float(iou_thr), _ptr(out), _ptr(src), max_out,
                             _ptr(ofo))
    n = min(int(ofo[F]), max_out)
    return dict(status=st, boxes=out[:n].copy(), src=src[:n].copy(), frame_off=ofo)


# --------------------------------------------------------------------------- NEXT-1
SWEEP_FIELDS = ("cost_sum", "windows", "full_frames", "dets_covered", "dets_touched")


def proxy_sweep(W, H, cell_w, cell_h, sizes, cost, scores, thresholds, dets, det_off):
    """Per-threshold totals.  dets float32 [n,4] frame px,
    det_off int32 [F+1].  Returns (status, int64 [J,5])."""
    s = np.ascontiguousarray(scores, dtype=np.float32)
    F = s.shape[0]
    sz = _sizes_arr(sizes)
    cs = np.ascontiguousarray(np.asarray(cost, dtype=np.int64))
    th = np.ascontiguousarray(np.asarray(thresholds, dtype=np.float32))
    d = np.ascontiguousarray(np.asarray(dets, dtype=np.float32).reshape(-1, 4))
    if len(d) == 0:
        d = np.zeros((1, 4), np.float32)
    do = np.ascontiguousarray(np.asarray(det_off, dtype=np.int32))
    out = np.zeros((len(th), 5), np.int64)
    st = lib().mpo_proxy_sweep(W, H, cell_w, cell_h, len(sz), _ptr(sz), _ptr(cs), _ptr(s), F, _ptr(th), len(th),
                               _ptr(d), _ptr(do), _ptr(out))
    return st, out


# --------------------------------------------------------------------------- NEXT-2
def window_set_cost(W, H, cell_w, cell_h, b_proxy, sizes, cost, scores, cand, cand_cost):
    """tot[c] = sum_t est(R(I_t; S + {cand[c]}))."""
    s = np.ascontiguousarray(scores, dtype=np.float32)
    sz = _sizes_arr(sizes)
    cs = np.ascontiguousarray(np.asarray(cost, dtype=np.int64))
    cd = _sizes_arr(cand)
    cc = np.ascontiguousarray(np.asarray(cand_cost, dtype=np.int64))
    tot = np.zeros(max(len(cd), 1), np.int64)
    st = lib().mpo_window_set_cost(W, H, cell_w, cell_h, float(b_proxy), len(sz), _ptr(sz), _ptr(cs), _ptr(s),
                                   s.shape[0], _ptr(cd), _ptr(cc), len(cd), _ptr(tot))
    return st, tot[:len(cd)].copy()


def select_window_sizes(W, H, cell_w, cell_h, scores, k, cost_fn, b_proxy=0.5, step=32):
    """The greedy of PAPER.md:193-195: S = {full frame}; k-1 times add the
    candidate (w, h), multiples of `step` no larger than the frame (not the full
    frame, not already in S), minimising tot_time(S + {(w,h)}); ties -> smaller
    area, then smaller w (reading R22).  Returns (sizes, [tot per step])."""
    S = [(W, H)]
    hist = []
    for _ in range(k - 1):
        cand = [(w, h) for w in range(step, W + 1, step) for h in range(step, H + 1, step)
                if (w, h) != (W, H) and (w, h) not in S]
        if not cand:
            break
        st, tot = window_set_cost(W, H, cell_w, cell_h, b_proxy, S, [cost_fn(*s) for s in S], scores, cand,
                                  [cost_fn(*c) for c in cand])
        assert st == OK, st
        best = min(range(len(cand)), key=lambda i: (int(tot[i]), cand[i][0] * cand[i][1], cand[i][0]))
        S.append(cand[best])
        hist.append(int(tot[best]))
    return S, hist


# --------------------------------------------------------------------------- NEXT-4
def hungarian(scores, floor=0.5):
    """R24 matching of track prefixes (rows) to detections (columns): maximum
    total score over pairs with score >= floor.  Returns (status, row_match,
    col_match, total)."""
    s = np.ascontiguousarray(np.asarray(scores, dtype=np.float32))
    if s.ndim != 2:
        s = s.reshape(0, 0) if s.size == 0 else s.reshape(s.shape[0], -1)
    m, n = s.shape
    rm = np.full(max(m, 1), -1, np.int32)
    cm = np.full(max(n, 1), -1, np.int32)
    tot = np.zeros(1, np.float64)
    st = lib().mpo_hungarian(_ptr(s) if s.size else None, m, n, float(floor), _ptr(rm), _ptr(cm), _ptr(tot))
    return st, rm[:m].copy(), cm[:n].copy(), float(tot[0])


# --------------------------------------------------------------------------- NEXT-4b
TRACK_N = 20   # P:244 "In our implementation, N = 20"


def box_centers(boxes):
    """R25: a track's path = its detections' box centres ((x1+x2)/2, (y1+y2)/2)
    in fp64.  boxes: [n][4] (x1, y1, x2, y2)."""
    b = np.asarray(boxes, np.float64).reshape(-1, 4)
    return np.ascontiguousarray(np.stack([(b[:, 0] + b[:, 2]) / 2, (b[:, 1] + b[:, 3]) / 2], 1))


def track_resample(points, N=TRACK_N):
    p = np.ascontiguousarray(np.asarray(points, np.float64).reshape(-1, 2))
    out = np.zeros((N, 2), np.float64)
    lib().mpo_track_resample(_ptr(p), len(p), N, _ptr(out))
    return out


def track_distance(a, b):
    a = np.ascontiguousarray(np.asarray(a, np.float64).reshape(-1, 2))
    b = np.ascontiguousarray(np.asarray(b, np.float64).reshape(-1, 2))
    assert a.shape == b.shape
    return float(lib().mpo_track_distance(_ptr(a), _ptr(b), len(a)))


def dbscan(paths, eps, min_pts):
    """R26 DBSCAN over resampled paths [T][N][2].  Returns (labels, is_core,
    n_dbscan_clusters, n_clusters incl. noise singletons)."""
    P = np.ascontiguousarray(np.asarray(paths, np.float64))
    T, N = P.shape[0], P.shape[1]
    lab = np.zeros(max(T, 1), np.int32)
    core = np.zeros(max(T, 1), np.uint8)
    nd = np.zeros(1, np.int32)
    Cn = lib().mpo_dbscan(_ptr(P), T, N, float(eps), int(min_pts), _ptr(lab), _ptr(core), _ptr(nd))
    return lab[:T].copy(), core[:T].astype(bool), int(nd[0]), int(Cn)


def cluster_centers(paths, labels, C):
    P = np.ascontiguousarray(np.asarray(paths, np.float64))
    T, N = P.shape[0], P.shape[1]
    lab = np.ascontiguousarray(np.asarray(labels, np.int32))
    ctr = np.zeros((max(C, 1), N, 2), np.float64)
    cnt = np.zeros(max(C, 1), np.int32)
    lib().mpo_cluster_centers(_ptr(P), T, N, _ptr(lab), C, _ptr(ctr), _ptr(cnt))
    return ctr[:C].copy(), cnt[:C].copy()


def refine_track(path, first, last, centers, counts, cell=32.0, k=10):
    """R27 refinement of one track: returns (clusters taken, (sx, sy, ex, ey))."""
    path = np.ascontiguousarray(np.asarray(path, np.float64))
    f = np.ascontiguousarray(np.asarray(first, np.float64))
    l = np.ascontiguousarray(np.asarray(last, np.float64))
    ctr = np.ascontiguousarray(np.asarray(centers, np.float64))
    cnt = np.ascontiguousarray(np.asarray(counts, np.int32))
    out = np.zeros(4, np.float64)
    C = len(cnt)
    n = lib().mpo_refine_track(_ptr(path), path.shape[0], _ptr(f), _ptr(l), _ptr(ctr) if C else None,
                               _ptr(cnt) if C else None, C, float(cell), int(k), _ptr(out))
    return int(n), out
