"""Dev tool: time the gather kernels alone (CUDA events, after warm-up) for the
c2 workload — the NV12 / RGB crop gather and the NEXT-3 proxy-input
downscale.  Prints one JSON line per measurement.  Used to sweep the
MP_GATHER_* experiment knobs, which the library reads only when built with
-DMP_EXPERIMENT_KNOBS (e.g. nvcc ... -DMP_EXPERIMENT_KNOBS into a copy of
libmp_b200.so); not part of the bench contract."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2103_14695_b200 as mp  # noqa: E402
from workloads import synth as S  # noqa: E402


FMT = int(os.environ.get("FMT", "0"))   # 0 f32 NCHW, 1 u8 NHWC (crop gathers only)


def timeit(fn, n=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def main():
    cfg = S.CONFIGS[os.environ.get("CFG", "c2_1080p_sparse")]
    F = int(os.environ.get("FRAMES", cfg.frames))
    what = os.environ.get("WHAT", "proxy_nv12,crops_nv12,crops_rgb,proxy_rgb").split(",")
    dev = torch.device("cuda:0")
    scene = S.make_scene(cfg, 0, F)
    scores = torch.from_numpy(S.score_grids(cfg, 0, scene)).to(dev)
    seeds = [S.frame_seed(0, f) for f in range(F)]
    tag = os.environ.get("TAG", "")
    for src in ("nv12", "rgb24"):
        if not any(w.endswith("nv12" if src == "nv12" else "rgb") for w in what):
            continue
        if src == "nv12":
            frames = S.frame_pixels_torch(seeds, cfg.H + cfg.H // 2, cfg.pitch_nv12, device=dev)
        else:
            frames = S.frame_pixels_torch(seeds, cfg.H, cfg.pitch, device=dev)
        p = mp.WindowPipeline(cfg.W, cfg.H, cfg.sizes, cfg.cost, cfg.out_dims, cfg.b_proxy, cfg.score_thr,
                              cfg.iou_thr, device=dev, src=src, proxy_dims=cfg.proxy_dims, fmt=FMT)
        R, C = cfg.grid
        p.reserve(F, F * R * ((C + 1) // 2))
        p.plan(scores)
        torch.cuda.synchronize()
        caps = p.class_count.cpu().tolist()
        p.reserve(F, p.max_windows, caps=caps)
        bpp = 1.5 if src == "nv12" else 3
        short = "nv12" if src == "nv12" else "rgb"
        if f"proxy_{short}" in what:
            ms = timeit(lambda: p.proxy_input(frames))
            p.check_status()
            pw, ph = cfg.proxy_dims
            frame_b = F * cfg.W * cfg.H * bpp
            out_b = F * pw * ph * 12
            print(json.dumps({"tag": tag, "what": f"proxy_{short}", "ms": ms,
                              "GBps_frame+out": (frame_b + out_b) / ms / 1e6}), flush=True)
        if f"crops_{short}" in what:
            ms = timeit(lambda: p.gather(frames))
            p.check_status()
            n = int(p.frame_off[F].item())
            w = p.windows[:n].cpu().numpy()
            out_b = sum((12 if FMT == 0 else 3) * cfg.out_dims[q][0] * cfg.out_dims[q][1] for q in w[:, 5])
            rd = bpp * sum(int(x[3]) * int(x[4]) for x in w)
            print(json.dumps({"tag": tag, "cfg": cfg.name, "rep": os.environ.get("REP"), "what": f"crops_{short}",
                              "fmt": FMT, "ms": ms,
                              "GBps_sum": (out_b + rd) / ms / 1e6}), flush=True)
        del frames, p
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
