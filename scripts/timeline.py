"""Dev tool: per-stream timeline of the PipelinedRunner (plan / gather /
merge start-end from CUDA events) for one config, to see which stage sits on
the critical path.  Not part of the bench contract."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2103_14695_b200 as mp  # noqa: E402
from workloads import synth as S  # noqa: E402


def main():
    cfg = S.CONFIGS[os.environ.get("CFG", "c4_4k_drone")]
    depth = int(os.environ.get("DEPTH", "2"))
    dev = torch.device("cuda:0")
    F = cfg.frames
    scene = S.make_scene(cfg, 0, F)
    scores_np = S.score_grids(cfg, 0, scene)
    scores = torch.from_numpy(scores_np).to(dev)
    frames = S.frame_pixels_torch([S.frame_seed(0, f) for f in range(F)], cfg.H, cfg.pitch, device=dev)
    pipes = []
    R, C = cfg.grid
    fmt = int(os.environ.get("FMT", "0"))   # 0 f32 NCHW, 1 u8 NHWC
    mp.mp_gather_set_sm_reserve(int(os.environ.get("RSV", "0")))   # SMs the gather leaves free
    p0 = mp.WindowPipeline(cfg.W, cfg.H, cfg.sizes, cfg.cost, cfg.out_dims, cfg.b_proxy, cfg.score_thr, cfg.iou_thr,
                           fmt=fmt, device=dev)
    p0.reserve(F, F * R * ((C + 1) // 2))
    p0.plan(scores)
    torch.cuda.synchronize()
    n = int(p0.frame_off[F].item())
    # the plan alone (nothing co-running): median of 20
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        p0.plan(scores)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"plan alone: {sorted(ts)[10]:.3f} ms")
    caps = p0.class_count.cpu().tolist()
    w = p0.windows[:n].cpu().numpy()
    boxes, wbo = S.standin_boxes(cfg, 0, scene, w)
    bt = torch.from_numpy(boxes.view(np.float32).reshape(-1, 6).copy()).to(dev)
    wt = torch.from_numpy(wbo).to(dev)
    for _ in range(depth):
        p = mp.WindowPipeline(cfg.W, cfg.H, cfg.sizes, cfg.cost, cfg.out_dims, cfg.b_proxy, cfg.score_thr,
                              cfg.iou_thr, fmt=fmt, device=dev)
        p.reserve(F, n, caps=caps, max_boxes=len(boxes))
        pipes.append(p)
    run = mp.PipelinedRunner(pipes, device=dev, merge_on_gather_stream=bool(int(os.environ.get("MOG", "0"))))
    ev = lambda: torch.cuda.Event(enable_timing=True)
    steps = 8
    rec = []
    t0 = ev()
    for i in range(steps + 3):
        if i == 3:
            torch.cuda.synchronize()
            t0.record(torch.cuda.current_stream())
            run.s_plan.wait_stream(torch.cuda.current_stream())
        k = run.i % run.depth
        p = run.pipes[k]
        if run.done[k] is not None:
            run.s_plan.wait_event(run.done[k])
        e = [ev() for _ in range(6)]
        e[0].record(run.s_plan)
        p.plan(scores, stream=run.s_plan)
        e[1].record(run.s_plan)
        run.s_gather.wait_event(e[1])
        e[2].record(run.s_gather)
        p.gather(frames, stream=run.s_gather)
        e[3].record(run.s_gather)
        run.s_merge.wait_event(e[3])
        e[4].record(run.s_merge)
        p.merge(bt, wt, stream=run.s_merge)
        e[5].record(run.s_merge)
        run.done[k] = e[5]
        run.i += 1
        if i >= 3:
            rec.append(e)
    run.wait_all()
    torch.cuda.synchronize()
    for i, e in enumerate(rec):
        t = [t0.elapsed_time(x) for x in e]
        print(f"step {i}: plan {t[0]:7.3f}-{t[1]:7.3f}  gather {t[2]:7.3f}-{t[3]:7.3f}  merge {t[4]:7.3f}-{t[5]:7.3f}")


if __name__ == "__main__":
    main()
