"""Multi-process (gloo, world size 2, CPU) tests of the clip-sharding driver:
clip assignment covers every clip exactly once, per-(clip, frame) results are
independent of the sharding, and the counter all-reduce equals the
single-process totals.  The per-clip work here is the CPU oracle (the GPU path
cannot run in this container); the sharding logic is the same code bench.py
uses with NCCL."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp_

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _clip_counters(clip, frames=12):
    import oracle as O
    from paper_2103_14695_b200.sharding import Counters
    from workloads import synth as S
    cfg = S.CONFIGS["c5_1080p_clips"]
    scene = S.make_scene(cfg, clip, frames)
    scores = S.score_grids(cfg, clip, scene)
    res = O.plan_windows(cfg.W, cfg.H, 32, 32, cfg.b_proxy, cfg.sizes, cfg.cost, scores)
    w = res["windows"]
    boxes, wbo = S.standin_boxes(cfg, clip, scene, w)
    nms = O.remap_nms(boxes, wbo, w, res["frame_off"], cfg.out_dims, cfg.W, cfg.H, cfg.score_thr, cfg.iou_thr)
    full = len(cfg.sizes) - 1
    c = Counters(frames=frames, windows=len(w), fallback_frames=int((w[:, 5] == full).sum()),
                 crop_bytes=int(sum(3 * x[3] * x[4] for x in w)),
                 out_bytes=int(sum(12 * cfg.out_dims[x[5]][0] * cfg.out_dims[x[5]][1] for x in w)),
                 boxes_in=len(boxes), boxes_kept=len(nms["boxes"]), clips=1)
    digest = (w.tobytes(), nms["src"].tobytes(), nms["boxes"].tobytes())
    return c, digest


def _worker(rank, world, port, n_clips, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2103_14695_b200.sharding import Counters, assign_clips, reduce_counters
    mine = assign_clips(n_clips, world, rank)
    tot = Counters()
    digests = {}
    for clip in mine:
        c, d = _clip_counters(clip)
        tot.add(c)
        digests[clip] = d
    g, emax = reduce_counters(tot, elapsed_ms=10.0 + rank)
    out[rank] = (mine, g, emax, digests)
    dist.barrier()
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def libs_available():
    # the gloo test imports the package (for sharding) which needs the built .so to exist
    sys.path.insert(0, ROOT)
    import __graft_entry__ as g
    g.build_cuda()


def test_assign_clips_partition(libs_available):
    from paper_2103_14695_b200 import sharding as sh
    for world in (1, 2, 4, 8):
        got = sorted(c for r in range(world) for c in sh.assign_clips(1000, world, r))
        assert got == list(range(1000))
        assert sh.assign_clips(1000, world, 0)[:2] == [0, world]
    rng = np.random.default_rng(0)
    cost = rng.uniform(1, 10, 50)
    for world in (2, 3, 8):
        parts = [sh.assign_clips(50, world, r, cost) for r in range(world)]
        assert sorted(c for p in parts for c in p) == list(range(50))
        loads = [sum(cost[p]) for p in parts]
        assert max(loads) - min(loads) <= cost.max() + 1e-9      # LPT bound


@pytest.mark.parametrize("world,n_clips", [(2, 5), (4, 6)])
def test_gloo_counters_and_results_match_single_process(libs_available, world, n_clips):
    port = _free_port()
    manager = mp_.get_context("spawn").Manager()
    out = manager.dict()
    ctx = mp_.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_clips, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
        assert p.exitcode == 0
    res = [out[r] for r in range(world)]
    mine = [m for (m, _, _, _) in res]
    assert sorted(c for m in mine for c in m) == list(range(n_clips))
    assert sum(len(m) for m in mine) == n_clips                      # each clip on exactly one rank
    g = [x[1] for x in res]
    e = [x[2] for x in res]
    assert all(gi == g[0] for gi in g) and all(ei == 10.0 + world - 1 for ei in e)   # SUM / MAX reductions
    # single-process reference
    from paper_2103_14695_b200.sharding import Counters
    ref = Counters()
    digests = {}
    for (_, _, _, d) in res:
        digests.update(d)
    for clip in range(n_clips):
        c, d = _clip_counters(clip)
        ref.add(c)
        assert digests[clip] == d     # per-clip outputs independent of the sharding
    assert g[0] == ref
