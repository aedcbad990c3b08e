"""Dev tool (needs a -DMP_PLAN_PROF build in MP_LIB): cycles per phase of the
cooperative merge (plan_full_kernel) for the c4 workload, (a) plan alone and
(b) inside the pipelined step beside the persistent gather."""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2103_14695_b200 as mp  # noqa: E402
from paper_2103_14695_b200 import _binding as B  # noqa: E402
from workloads import synth as S  # noqa: E402

lib = B._lib if hasattr(B, "_lib") else ctypes.CDLL(os.environ["MP_LIB"])
fn = lib.mp_debug_plan_prof
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]


def read(reset=1):
    a = (ctypes.c_ulonglong * 4)()
    torch.cuda.synchronize()
    assert fn(a, reset) == 0
    return list(a)


def show(tag, a):
    st = max(a[3], 1)
    print(f"{tag}: steps {a[3]}  cycles/step argmin {a[0] / st:.0f}  fit {a[1] / st:.0f}  walk+publish {a[2] / st:.0f}",
          flush=True)


cfg = S.CONFIGS[os.environ.get("CFG", "c4_4k_drone")]
dev = torch.device("cuda:0")
F = cfg.frames
scene = S.make_scene(cfg, 0, F)
scores = torch.from_numpy(S.score_grids(cfg, 0, scene)).to(dev)
frames = S.frame_pixels_torch([S.frame_seed(0, f) for f in range(F)], cfg.H, cfg.pitch, device=dev)
R, C = cfg.grid
pipes = []
for _ in range(3):
    p = mp.WindowPipeline(cfg.W, cfg.H, cfg.sizes, cfg.cost, cfg.out_dims, cfg.b_proxy, cfg.score_thr, cfg.iou_thr,
                          device=dev)
    p.reserve(F, F * R * ((C + 1) // 2))
    pipes.append(p)
pipes[0].plan(scores)
torch.cuda.synchronize()
n = int(pipes[0].frame_off[F].item())
caps = pipes[0].class_count.cpu().tolist()
for p in pipes:
    p.reserve(F, n, caps=caps)
read()
for _ in range(5):
    pipes[0].plan(scores)
show("alone", read())
runner = mp.PipelinedRunner(pipes, device=dev)
for _ in range(3):
    runner.step(scores, frames)
runner.wait_all()
read()
for _ in range(12):
    runner.step(scores, frames)
runner.wait_all()
show("beside the gather (pipelined, 12 steps)", read())
