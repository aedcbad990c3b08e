"""Quick start: the public Python API on one batch of synthetic 540p frames.

    python examples/quickstart.py        (needs a B200 and the built library)

Plan detector windows from proxy scores (a1-a4), gather + resize the crops
into per-size detector batches (a5), hand them to a detector (here a stand-in
that emits jittered boxes), then remap + NMS the detections into frame
coordinates (a6-a7).  Every step runs in libmp_b200.so's CUDA kernels.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_14695_b200 as mp  # noqa: E402
from workloads import synth as S  # noqa: E402


def main():
    cfg = S.CONFIGS["c1_540p"]              # 960x540, S = {256x256, full frame}
    dev = torch.device("cuda:0")
    F = cfg.frames
    scene = S.make_scene(cfg, 0, F)
    scores = torch.from_numpy(S.score_grids(cfg, 0, scene)).to(dev)          # proxy output [F][R][C]
    frames = S.frame_pixels_torch([S.frame_seed(0, f) for f in range(F)], cfg.H, cfg.pitch, device=dev)

    pipe = mp.WindowPipeline(cfg.W, cfg.H, cfg.sizes, cfg.cost, cfg.out_dims, b_proxy=cfg.b_proxy,
                             score_thr=cfg.score_thr, iou_thr=cfg.iou_thr, device=dev)
    R, C = cfg.grid
    pipe.reserve(F, F * R * ((C + 1) // 2))
    pipe.plan(scores)                                                           # a1-a4
    torch.cuda.synchronize()
    pipe.check_status()
    n = int(pipe.frame_off[F].item())
    counts = pipe.class_count.cpu().tolist()
    print(f"{F} frames -> {n} windows, per size {dict(zip(map(tuple, cfg.sizes), counts))}")

    windows = pipe.windows[:n].cpu().numpy()
    boxes, wbo = S.standin_boxes(cfg, 0, scene, windows)                        # the detector (stand-in)
    pipe.reserve(F, n, caps=counts, max_boxes=max(len(boxes), 1))
    pipe.gather(frames)                                                         # a5
    for q, t in enumerate(pipe.outs):
        print(f"  size {cfg.sizes[q]} -> detector batch {tuple(t.shape)} {t.dtype}")
    pipe.merge(torch.from_numpy(boxes.view(np.float32).reshape(-1, 6).copy()).to(dev),
               torch.from_numpy(wbo).to(dev))                                   # a6-a7
    torch.cuda.synchronize()
    pipe.check_status()
    kept = int(pipe.nms_frame_off[F].item())
    print(f"{len(boxes)} raw detections -> {kept} kept after remap + per-frame NMS")
    if kept:
        row = pipe.nms_out[0].cpu()
        print("first kept box: x1 y1 x2 y2 =", [round(v, 2) for v in row[:4].tolist()],
              "score", round(float(row[4]), 3), "class", int(row[5:6].view(torch.int32).item()))


if __name__ == "__main__":
    main()
