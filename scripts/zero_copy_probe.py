"""Dev tool: can the gather read window footprints straight out of pinned host
memory (zero-copy over PCIe) instead of copying whole frames H2D first?

Runs the c2 crop gather three ways on the same frames and compares bits:
  dev      frames resident in HBM (the bench's device path)
  host_ptr pointer-array path, frame addresses inside a pinned host pool
  host_tma strided TMA path over a pinned host batch
and times each beside a plain H2D copy of the same frames.  Prints JSON lines."""
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2103_14695_b200 as mp  # noqa: E402
from paper_2103_14695_b200 import _binding as B  # noqa: E402
from workloads import synth as S  # noqa: E402


def timeit(fn, n=5, warm=2):
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
    F = int(os.environ.get("FRAMES", 256))
    dev = torch.device("cuda:0")
    scene = S.make_scene(cfg, 0, F)
    scores = torch.from_numpy(S.score_grids(cfg, 0, scene)).to(dev)
    seeds = [S.frame_seed(0, f) for f in range(F)]
    frames_d = S.frame_pixels_torch(seeds, cfg.H, cfg.pitch, device=dev)
    frames_h = frames_d.cpu().pin_memory()
    p = mp.WindowPipeline(cfg.W, cfg.H, cfg.sizes, cfg.cost, cfg.out_dims, cfg.b_proxy, cfg.score_thr,
                          cfg.iou_thr, device=dev)
    R, Cc = cfg.grid
    p.reserve(F, F * R * ((Cc + 1) // 2))
    p.plan(scores)
    torch.cuda.synchronize()
    p.reserve(F, p.max_windows, caps=p.class_count.cpu().tolist())
    n = int(p.frame_off[F].item())
    w = p.windows[:n].cpu().numpy()
    crop = 3 * sum(int(x[3]) * int(x[4]) for x in w)
    frame_b = frames_h.numel()

    p.gather(frames_d)
    torch.cuda.synchronize()
    ref = [o.clone() for o in p.outs]
    ms = timeit(lambda: p.gather(frames_d))
    print(json.dumps({"what": "dev", "ms": ms, "frames": F}), flush=True)

    ms = timeit(lambda: frames_d.copy_(frames_h, non_blocking=True))
    print(json.dumps({"what": "h2d_copy", "ms": ms, "GBps": frame_b / ms / 1e6}), flush=True)

    def same():
        return all(torch.equal(a, b) for a, b in zip(ref, p.outs))

    # pointer-array path over host addresses
    step = frames_h.stride(0)
    ptrs = (torch.arange(F, dtype=torch.int64) * step + frames_h.data_ptr()).to(dev)
    for o in p.outs:
        o.zero_()
    try:
        p.gather(ptrs)
        torch.cuda.synchronize()
        p.check_status()
        ok = same()
        ms = timeit(lambda: p.gather(ptrs))
        print(json.dumps({"what": "host_ptr", "ok": ok, "ms": ms, "crop_GBps": crop / ms / 1e6,
                          "frame_equiv_GBps": frame_b / ms / 1e6}), flush=True)
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"what": "host_ptr", "error": repr(e)}), flush=True)

    # strided TMA path over the pinned host batch (bypass the binding's is_cuda check)
    for o in p.outs:
        o.zero_()
    k = p.k
    optrs = (C.c_void_p * k)(*[o.data_ptr() for o in p.outs])
    cap = (C.c_int32 * k)(*[int(o.shape[0]) for o in p.outs])

    def tma():
        st = B._lib.mp_gather_resize_strided(
            C.c_void_p(frames_h.data_ptr()), int(frames_h.stride(0)), int(cfg.pitch), cfg.W, cfg.H, F,
            B._p(p.windows), B._p(p.frame_off), B._nwin(p.windows), k, B._sizes(p.sizes), B._sizes(p.out_dims), optrs, cap,
            int(p.fmt), B._p(p.status), B._p(p.gather_ws), p.gather_ws.numel(), B._stream(None))
        if st != 0:
            raise B.MPError(st, "strided host")
    try:
        tma()
        torch.cuda.synchronize()
        p.check_status()
        ok = same()
        ms = timeit(tma)
        print(json.dumps({"what": "host_tma", "ok": ok, "ms": ms, "crop_GBps": crop / ms / 1e6,
                          "frame_equiv_GBps": frame_b / ms / 1e6}), flush=True)
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"what": "host_tma", "error": repr(e)}), flush=True)


if __name__ == "__main__":
    main()
