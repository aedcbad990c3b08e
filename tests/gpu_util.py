"""Helpers for the -m gpu parity tests: run the CUDA path (through the C-ABI
binding) on numpy inputs and bring the results back as numpy."""
import numpy as np
import torch

import paper_2103_14695_b200 as mp
from paper_2103_14695_b200 import _binding as B

DEV = torch.device("cuda:0")


def gpu_plan(W, H, cw, ch, b, sizes, cost, scores, max_windows=None, want_mask=True):
    scores = np.ascontiguousarray(scores, np.float32)
    F = scores.shape[0]
    p = B.PlanParams(W, H, sizes, cost, b, cw, ch)
    R, C = p.grid
    if max_windows is None:
        max_windows = max(F * ((R * C + 1) // 2 + 1), 1)
    win = torch.full((max(max_windows, 1), 7), -7, dtype=torch.int32, device=DEV)
    fo = torch.full((F + 1,), -7, dtype=torch.int32, device=DEV)
    cc = torch.full((len(sizes),), -7, dtype=torch.int32, device=DEV)
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    mask = torch.full((max(F, 1), R, (C + 31) // 32), -7, dtype=torch.int32, device=DEV) if want_mask else None
    ws = torch.empty(max(B.mp_plan_workspace_size(p, F), 1), dtype=torch.uint8, device=DEV)
    sc = torch.from_numpy(scores).to(DEV) if F else torch.zeros((1, R, C), device=DEV)
    B.mp_plan_windows(p, sc, F, mask if F else None, win if max_windows else None, fo, cc, st, ws)
    torch.cuda.synchronize()
    n = int(fo[F].item())
    return dict(status=int(st.item()), windows=win[:min(n, max_windows)].cpu().numpy(), frame_off=fo.cpu().numpy(),
                class_count=cc.cpu().numpy(),
                mask=(mask[:F].cpu().numpy().view(np.uint32) if want_mask else None))


def gpu_gather(frames_np_or_t, pitch, W, H, windows, sizes, out_dims, caps, fmt=mp.MP_OUT_F32_NCHW,
               strided=True, host=False):
    """host=True: frames in pinned host memory (zero-copy reads over PCIe)."""
    if isinstance(frames_np_or_t, torch.Tensor):
        fr = frames_np_or_t
    else:
        fr = torch.from_numpy(np.stack(frames_np_or_t))
        fr = fr.pin_memory() if host else fr.to(DEV)
    F = fr.shape[0]
    win = np.asarray(windows, np.int32).reshape(-1, 7)
    # a CSR over frames consistent with the (frame-sorted) window list
    fo = np.searchsorted(win[:, 0], np.arange(F + 1), side="left").astype(np.int32) if len(win) else \
        np.zeros(F + 1, np.int32)
    fo[F] = len(win)
    wt = torch.from_numpy(win if len(win) else np.zeros((1, 7), np.int32)).to(DEV)
    fot = torch.from_numpy(fo).to(DEV)
    outs = []
    for q, (ow, oh) in enumerate(out_dims):
        if fmt == mp.MP_OUT_F32_NCHW:
            outs.append(torch.full((caps[q], 3, oh, ow), -1.0, dtype=torch.float32, device=DEV))
        else:
            outs.append(torch.zeros((caps[q], oh, ow, 3), dtype=torch.uint8, device=DEV))
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    ws = torch.empty(B.mp_gather_workspace_size(out_dims, caps), dtype=torch.uint8, device=DEV)
    if strided:
        B.mp_gather_resize_strided(fr, W, H, wt, fot, sizes, out_dims, outs, fmt, st, ws)
    else:
        ptrs = mp.WindowPipeline.frame_ptrs(fr, device=DEV)
        B.mp_gather_resize(ptrs, pitch, W, H, F, wt, fot, sizes, out_dims, outs, fmt, st, ws)
    torch.cuda.synchronize()
    return int(st.item()), [o.cpu().numpy() for o in outs]


def gpu_gather_nv12(frames_np_or_t, W, H, windows, sizes, out_dims, caps, fmt=mp.MP_OUT_F32_NCHW,
                    matrix=mp.MP_BT709_LIMITED, host=False):
    if isinstance(frames_np_or_t, torch.Tensor):
        fr = frames_np_or_t
    else:
        fr = torch.from_numpy(np.stack(frames_np_or_t))
        fr = fr.pin_memory() if host else fr.to(DEV)
    F = fr.shape[0]
    win = np.asarray(windows, np.int32).reshape(-1, 7)
    fo = np.searchsorted(win[:, 0], np.arange(F + 1), side="left").astype(np.int32) if len(win) else \
        np.zeros(F + 1, np.int32)
    fo[F] = len(win)
    wt = torch.from_numpy(win if len(win) else np.zeros((1, 7), np.int32)).to(DEV)
    fot = torch.from_numpy(fo).to(DEV)
    outs = []
    for q, (ow, oh) in enumerate(out_dims):
        if fmt == mp.MP_OUT_F32_NCHW:
            outs.append(torch.full((caps[q], 3, oh, ow), -1.0, dtype=torch.float32, device=DEV))
        else:
            outs.append(torch.zeros((caps[q], oh, ow, 3), dtype=torch.uint8, device=DEV))
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    ws = torch.empty(B.mp_gather_workspace_size(out_dims, caps), dtype=torch.uint8, device=DEV)
    B.mp_gather_resize_nv12(fr, W, H, wt, fot, sizes, out_dims, outs, fmt, st, ws, matrix)
    torch.cuda.synchronize()
    return int(st.item()), [o.cpu().numpy() for o in outs]


def boxes_to_t(boxes):
    if len(boxes) == 0:
        return torch.zeros((1, 6), dtype=torch.float32, device=DEV)
    return torch.from_numpy(np.ascontiguousarray(boxes).view(np.float32).reshape(-1, 6).copy()).to(DEV)


def gpu_remap_nms(boxes, win_box_off, windows, frame_off, out_dims, W, H, score_thr, iou_thr, max_out=None):
    F = len(frame_off) - 1
    n_box = len(boxes)
    max_out = max(n_box, 1) if max_out is None else max_out
    win = np.asarray(windows, np.int32).reshape(-1, 7)
    wt = torch.from_numpy(win if len(win) else np.zeros((1, 7), np.int32)).to(DEV)
    out = torch.full((max(max_out, 1), 6), -3.0, dtype=torch.float32, device=DEV)
    src = torch.full((max(max_out, 1),), -3, dtype=torch.int32, device=DEV)
    ofo = torch.full((F + 1,), -3, dtype=torch.int32, device=DEV)
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    bx = boxes_to_t(boxes)
    ws = torch.empty(B.mp_remap_nms_workspace_size(F, max(n_box, 1)), dtype=torch.uint8, device=DEV)
    B.mp_remap_nms(bx, torch.from_numpy(np.asarray(win_box_off, np.int32)).to(DEV), wt,
                   torch.from_numpy(np.asarray(frame_off, np.int32)).to(DEV), F, out_dims, W, H, score_thr,
                   iou_thr, out[:max(max_out, 1)] if max_out else out, src, ofo, st, ws)
    torch.cuda.synchronize()
    n = min(int(ofo[F].item()), max_out)
    return dict(status=int(st.item()), boxes=out[:n].cpu().numpy(), src=src[:n].cpu().numpy(),
                frame_off=ofo.cpu().numpy())


def gpu_hungarian(mats, floor=0.5, max_dim=None):
    """Run mp_hungarian on a list of float32 [m][n] matrices; returns
    (status, [row_match], [col_match], totals)."""
    ms = [int(a.shape[0]) for a in mats]
    ns = [int(a.shape[1]) for a in mats]
    rec, ns_tot, nr, nc = B.assign_problems(ms, ns)
    flat = np.concatenate([np.ascontiguousarray(a, np.float32).ravel() for a in mats]) if ns_tot else \
        np.zeros(1, np.float32)
    sc = torch.from_numpy(flat if len(flat) else np.zeros(1, np.float32)).to(DEV)
    pr = torch.from_numpy(rec.view(np.uint8).copy() if len(rec) else np.zeros(24, np.uint8)).to(DEV)
    rm = torch.full((max(nr, 1),), -9, dtype=torch.int32, device=DEV)
    cm = torch.full((max(nc, 1),), -9, dtype=torch.int32, device=DEV)
    tot = torch.full((max(len(mats), 1),), -1.0, dtype=torch.float64, device=DEV)
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    ws = torch.empty(max(B.mp_hungarian_workspace_size(len(mats)), 1), dtype=torch.uint8, device=DEV)
    md = max([max(m, n) for m, n in zip(ms, ns)] + [0]) if max_dim is None else max_dim
    B.mp_hungarian(sc, pr, len(mats), floor, md, rm, cm, tot, st, ws)
    torch.cuda.synchronize()
    rmh, cmh = rm.cpu().numpy(), cm.cpu().numpy()
    rows = [rmh[rec["row_off"][b]:rec["row_off"][b] + ms[b]] for b in range(len(mats))]
    cols = [cmh[rec["col_off"][b]:rec["col_off"][b] + ns[b]] for b in range(len(mats))]
    return int(st.item()), rows, cols, tot.cpu().numpy()[:len(mats)]


def gpu_refine_pipeline(train_boxes, query_boxes, eps, min_pts, N=20, W=1920, H=1080, cell=32.0, k=10,
                        max_cand=1024, C_max=None):
    """NEXT-4b end to end on the GPU: resample train + query tracks, DBSCAN the
    training paths, cluster centres, refine the queries.  Returns a dict of
    numpy arrays."""
    def pack(tr):
        off = np.concatenate([[0], np.cumsum([len(b) for b in tr])]).astype(np.int32)
        bx = np.concatenate([np.asarray(b, np.float32).reshape(-1, 4) for b in tr]) if off[-1] else \
            np.zeros((1, 4), np.float32)
        return torch.from_numpy(bx).to(DEV), torch.from_numpy(off).to(DEV)

    T, Q = len(train_boxes), len(query_boxes)
    tb, to = pack(train_boxes)
    qb, qo = pack(query_boxes)
    tp = torch.empty((max(T, 1), N, 2), dtype=torch.float64, device=DEV)
    te = torch.empty((max(T, 1), 4), dtype=torch.float64, device=DEV)
    qp = torch.empty((max(Q, 1), N, 2), dtype=torch.float64, device=DEV)
    qe = torch.empty((max(Q, 1), 4), dtype=torch.float64, device=DEV)
    B.mp_track_resample(tb, to, T, N, tp, te)
    B.mp_track_resample(qb, qo, Q, N, qp, qe)
    lab = torch.full((max(T, 1),), -9, dtype=torch.int32, device=DEV)
    core = torch.zeros((max(T, 1),), dtype=torch.uint8, device=DEV)
    ncl = torch.zeros(2, dtype=torch.int32, device=DEV)
    ws = torch.empty(max(B.mp_dbscan_workspace_size(T), 1), dtype=torch.uint8, device=DEV)
    B.mp_dbscan(tp, T, N, eps, min_pts, lab, core, ncl, ws)
    C_max = max(T, 1) if C_max is None else C_max
    ctr = torch.zeros((max(C_max, 1), N, 2), dtype=torch.float64, device=DEV)
    cnt = torch.zeros((max(C_max, 1),), dtype=torch.int32, device=DEV)
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    B.mp_cluster_centers(tp, T, N, lab, ncl, C_max, ctr, cnt, st)
    out = torch.full((max(Q, 1), 4), -1.0, dtype=torch.float64, device=DEV)
    taken = torch.full((max(Q, 1),), -1, dtype=torch.int32, device=DEV)
    rws = torch.empty(max(B.mp_refine_workspace_size(W, H, cell, C_max, N), 1), dtype=torch.uint8, device=DEV)
    B.mp_refine_tracks(qp, qe, Q, N, ctr, cnt, ncl, C_max, W, H, cell, k, max_cand, out, taken, st, rws)
    torch.cuda.synchronize()
    C = int(ncl[1].item())
    return dict(status=int(st.item()), train_paths=tp[:T].cpu().numpy(), train_ends=te[:T].cpu().numpy(),
                query_paths=qp[:Q].cpu().numpy(), query_ends=qe[:Q].cpu().numpy(), labels=lab[:T].cpu().numpy(),
                is_core=core[:T].cpu().numpy().astype(bool), nclust=ncl.cpu().numpy(),
                centers=ctr[:min(C, C_max)].cpu().numpy(), counts=cnt[:min(C, C_max)].cpu().numpy(),
                out=out[:Q].cpu().numpy(), taken=taken[:Q].cpu().numpy())
