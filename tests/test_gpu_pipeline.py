"""GPU tests of the public pipeline API (WindowPipeline / PipelinedRunner)
under the conditions a real caller creates, against the CPU oracle:

* different inputs on every batch, written on the caller's stream with
  non_blocking H2D copies into freshly allocated tensors that are dropped
  right after the call (stream ordering + record_stream), with and without
  CUDA graphs (graph mode copies each batch into runner-owned static inputs);
* the split enqueue / merge API with the detector between them (merge waits
  for a detector-done event);
* a plan that overflows its window buffer, followed by gather and remap/NMS
  on the same buffers: MP_ERR_CAPACITY, no read past the buffers, and the
  stored prefix of windows is gathered and merged correctly.

Tolerances as everywhere: windows / kept boxes bit-exact,
f32 pixels <= 1e-3."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
from workloads import synth as S  # noqa: E402

F32_TOL = 1e-3


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import gpu_util
    return gpu_util


def _clip_inputs(cfg, clip, F):
    scene = S.make_scene(cfg, clip, F)
    scores = S.score_grids(cfg, clip, scene)
    ref = O.plan_windows(cfg.W, cfg.H, 32, 32, cfg.b_proxy, cfg.sizes, cfg.cost, scores)
    boxes, wbo = S.standin_boxes(cfg, clip, scene, ref["windows"], extra_edge_cases=True)
    r = O.remap_nms(boxes, wbo, ref["windows"], ref["frame_off"], cfg.out_dims, cfg.W, cfg.H, cfg.score_thr,
                    cfg.iou_thr)
    frames = np.stack([S.frame_pixels_np(S.frame_seed(clip, f), cfg.H, cfg.pitch) for f in range(F)])
    return dict(scores=scores, ref=ref, boxes=boxes, wbo=wbo, nms=r, frames=frames)


def _check_batch(cfg, inp, snap, rng, n_pix=6):
    ref, r = inp["ref"], inp["nms"]
    n = len(ref["windows"])
    assert snap["status"] == 0
    assert np.array_equal(snap["frame_off"], ref["frame_off"])
    assert np.array_equal(snap["windows"][:n], ref["windows"])
    nk = int(snap["nms_frame_off"][-1])
    assert np.array_equal(snap["nms_frame_off"], r["frame_off"])
    assert np.array_equal(snap["nms_src"][:nk], r["src"])
    assert np.array_equal(snap["nms_out"][:nk].view(np.uint32), r["boxes"].view(np.float32).reshape(-1, 6).view(np.uint32))
    for wi in rng.choice(n, size=min(n_pix, n), replace=False):
        w = ref["windows"][wi].copy()
        f, q, slot = int(w[0]), int(w[5]), int(w[6])
        one = w.copy(); one[0] = 0; one[6] = 0
        caps1 = [1 if qq == q else 0 for qq in range(len(cfg.sizes))]
        st, o = O.gather_resize([inp["frames"][f]], cfg.pitch, cfg.W, cfg.H, one[None], cfg.sizes, cfg.out_dims, caps1)
        assert np.abs(snap["outs"][q][slot].astype(np.float64) - o[q][0]).max() <= F32_TOL, (wi, q)


@pytest.mark.parametrize("graphs,reserve", [(False, 0), (True, 0), (False, 16), (True, 140)],
                         ids=["eager", "graphs", "eager-reserve16", "graphs-reserve140"])
@pytest.mark.parametrize("depth", [2, 3])
def test_runner_new_inputs_every_batch(G, graphs, reserve, depth, request):
    """Batches from 3 different clips in rotation, each batch's inputs copied
    H2D (non_blocking, pinned) into NEW tensors on the caller's stream and
    released right after the call; each batch's results are snapshotted on a
    reader stream that waits for its merge.  Every snapshot equals the
    oracle for its own clip (also with the gather leaving SMs to the
    planner: mp_gather_set_sm_reserve 16, and 140 of 148 — an 8-CTA grid
    that must still cover every tile)."""
    import paper_2103_14695_b200 as mp
    request.addfinalizer(lambda: mp.mp_gather_set_sm_reserve(0))
    cfg = S.CONFIGS["c1_540p"]
    F = cfg.frames
    clips = [_clip_inputs(cfg, c, F) for c in (11, 12, 13)]
    n_max = max(len(c["ref"]["windows"]) for c in clips)
    caps = [max(int(c["ref"]["class_count"][q]) for c in clips) for q in range(len(cfg.sizes))]
    nb = max(max(len(c["boxes"]) for c in clips), 1)
    pipes = []
    for _ in range(depth):
        p = mp.WindowPipeline(cfg.W, cfg.H, cfg.sizes, cfg.cost, cfg.out_dims, cfg.b_proxy, cfg.score_thr,
                              cfg.iou_thr, device=G.DEV)
        p.reserve(F, n_max + 4, caps=caps, max_boxes=nb)
        pipes.append(p)
    runner = mp.PipelinedRunner(pipes, device=G.DEV, gather_sm_reserve=reserve)

    def pad_boxes(c):
        b = np.zeros((nb, 6), np.float32)
        if len(c["boxes"]):
            b[:len(c["boxes"])] = c["boxes"].view(np.float32).reshape(-1, 6)
        w = np.full(n_max + 4 + 1, c["wbo"][-1], np.int32)
        w[:len(c["wbo"])] = c["wbo"]
        return torch.from_numpy(b).pin_memory(), torch.from_numpy(w).pin_memory()

    host = [(torch.from_numpy(c["scores"]).pin_memory(), torch.from_numpy(c["frames"]).pin_memory()) + pad_boxes(c)
            for c in clips]
    if graphs:
        sc0 = torch.empty(host[0][0].shape, dtype=torch.float32, device=G.DEV)
        bx0 = torch.zeros((nb, 6), dtype=torch.float32, device=G.DEV)
        wb0 = torch.zeros(n_max + 5, dtype=torch.int32, device=G.DEV)
        runner.capture_graphs(sc0, bx0, wb0)
    reader = torch.cuda.Stream(G.DEV)
    snaps = []
    order = [0, 1, 2, 1, 0, 2, 2, 0, 1]
    for i, ci in enumerate(order):
        hs, hf, hb, hw = host[ci]
        sc = hs.to(G.DEV, non_blocking=True)
        fr = hf.to(G.DEV, non_blocking=True)
        bx = hb.to(G.DEV, non_blocking=True)
        wb = hw.to(G.DEV, non_blocking=True)
        k = runner.enqueue(sc, fr)
        # the "detector" runs on the caller's stream after the gather
        runner.wait_gathered(k)
        det_done = torch.cuda.Event()
        det_done.record(torch.cuda.current_stream(G.DEV))
        runner.merge(k, bx, wb, detector_done=det_done)
        del sc, fr, bx, wb                      # caller drops its tensors at once
        p = pipes[k]
        reader.wait_event(runner.done[k])
        with torch.cuda.stream(reader):
            snaps.append((ci, dict(frame_off=p.frame_off.clone(), windows=p.windows.clone(),
                                   nms_frame_off=p.nms_frame_off.clone(), nms_src=p.nms_src.clone(),
                                   nms_out=p.nms_out.clone(), outs=[o.clone() for o in p.outs],
                                   status=p.status.clone())))
        # the next enqueue into set k waits for runner.done[k]; the reader
        # stream's clones must finish first too
        ev = torch.cuda.Event()
        ev.record(reader)
        torch.cuda.current_stream(G.DEV).wait_event(ev)
    runner.wait_all()
    torch.cuda.synchronize()
    rng = np.random.default_rng(99)
    for ci, snap in snaps:
        s = {k: (v.cpu().numpy() if torch.is_tensor(v) else [o.cpu().numpy() for o in v]) for k, v in snap.items()}
        s["status"] = int(s["status"][0])
        _check_batch(cfg, clips[ci], s, rng)


def test_runner_enqueue_merge_protocol(G):
    """enqueue() twice into the same buffer set without merge() in between is
    refused (the detector may still read that set's outputs)."""
    import paper_2103_14695_b200 as mp
    cfg = S.CONFIGS["c1_540p"]
    F = 4
    inp = _clip_inputs(cfg, 21, F)
    p = mp.WindowPipeline(cfg.W, cfg.H, cfg.sizes, cfg.cost, cfg.out_dims, cfg.b_proxy, cfg.score_thr,
                          cfg.iou_thr, device=G.DEV)
    p.reserve(F, len(inp["ref"]["windows"]) + 2, caps=[max(1, int(c)) for c in inp["ref"]["class_count"]],
              max_boxes=max(len(inp["boxes"]), 1))
    runner = mp.PipelinedRunner([p], device=G.DEV)
    sc = torch.from_numpy(inp["scores"]).to(G.DEV)
    fr = torch.from_numpy(inp["frames"]).to(G.DEV)
    k = runner.enqueue(sc, fr)
    with pytest.raises(RuntimeError):
        runner.enqueue(sc, fr)
    runner.merge(k, G.boxes_to_t(inp["boxes"]), torch.from_numpy(inp["wbo"]).to(G.DEV))
    with pytest.raises(RuntimeError):
        runner.merge(k)
    runner.wait_all()
    torch.cuda.synchronize()
    p.check_status()
    with pytest.raises(ValueError):        # scores not shaped [F, R, C]
        p.plan(sc[:2])


@pytest.mark.parametrize("cap_frac", [0.0, 0.37, 0.8])
def test_plan_overflow_then_gather_and_merge(G, cap_frac):
    """the plan overflows its window buffer (frame_off[F]
    reports the true total); gather and remap/NMS on the same buffers must
    read nothing past them.  The stored prefix of windows (and its slots) is
    exactly the oracle's prefix, the gathered pixels of those windows are
    correct, and frames whose windows all fit keep exactly the oracle's
    boxes; status = MP_ERR_CAPACITY."""
    import paper_2103_14695_b200 as mp
    cfg = S.CONFIGS["c1_540p"]
    F = cfg.frames
    inp = _clip_inputs(cfg, 23, F)
    ref = inp["ref"]
    n = len(ref["windows"])
    cap = int(cap_frac * n)
    p = mp.WindowPipeline(cfg.W, cfg.H, cfg.sizes, cfg.cost, cfg.out_dims, cfg.b_proxy, cfg.score_thr,
                          cfg.iou_thr, device=G.DEV)
    p.reserve(F, max(cap, 1), caps=[int(c) for c in ref["class_count"]], max_boxes=max(len(inp["boxes"]), 1))
    if cap == 0:   # reserve keeps >= 1 record; make the capacity truly 0 through the binding
        p.windows = p.windows[:0]
    sc = torch.from_numpy(inp["scores"]).to(G.DEV)
    fr = torch.from_numpy(inp["frames"]).to(G.DEV)
    p.plan(sc)
    p.gather(fr)
    # win_box_off sized for the windows that exist (the stored prefix)
    wbo = torch.from_numpy(inp["wbo"][:cap + 1].copy()).to(G.DEV)
    p.merge(G.boxes_to_t(inp["boxes"]), wbo)
    torch.cuda.synchronize()
    assert int(p.status.item()) == mp.MP_ERR_CAPACITY
    fo = p.frame_off.cpu().numpy()
    assert np.array_equal(fo, ref["frame_off"])                        # true offsets
    assert np.array_equal(p.windows[:cap].cpu().numpy(), ref["windows"][:cap])
    rng = np.random.default_rng(3)
    for wi in rng.choice(cap, size=min(8, cap), replace=False) if cap else []:
        w = ref["windows"][wi].copy()
        f, q, slot = int(w[0]), int(w[5]), int(w[6])
        one = w.copy(); one[0] = 0; one[6] = 0
        caps1 = [1 if qq == q else 0 for qq in range(len(cfg.sizes))]
        st, o = O.gather_resize([inp["frames"][f]], cfg.pitch, cfg.W, cfg.H, one[None], cfg.sizes, cfg.out_dims,
                                caps1)
        assert np.abs(p.outs[q][slot].cpu().numpy().astype(np.float64) - o[q][0]).max() <= F32_TOL
    # frames entirely inside the stored prefix keep exactly the oracle's boxes
    r = inp["nms"]
    kfo = p.nms_frame_off.cpu().numpy()
    src = p.nms_src.cpu().numpy()
    for f in range(F):
        if ref["frame_off"][f + 1] <= cap:
            a, b = r["frame_off"][f], r["frame_off"][f + 1]
            assert np.array_equal(src[kfo[f]:kfo[f + 1]], r["src"][a:b]), f
        elif ref["frame_off"][f] >= cap:
            assert kfo[f + 1] == kfo[f], f                              # its windows do not exist


@pytest.mark.parametrize("replays", [1, 3])
def test_runner_capture_steps_whole_step_graphs(G, replays):
    """PipelinedRunner.capture_steps (the bench's mode for small batches):
    three whole pipelined steps (plan / gather / merge of three clips on the
    runner's streams) captured as ONE CUDA graph and replayed; after the
    last replay buffer set u holds batch u, and every set equals the oracle
    for its clip.  The gather events recorded as graph nodes (external
    events) time every replayed gather."""
    import paper_2103_14695_b200 as mp
    cfg = S.CONFIGS["c1_540p"]
    F = cfg.frames
    clips = [_clip_inputs(cfg, c, F) for c in (21, 22, 23)]
    n_max = max(len(c["ref"]["windows"]) for c in clips)
    caps = [max(int(c["ref"]["class_count"][q]) for c in clips) for q in range(len(cfg.sizes))]
    nb = max(max(len(c["boxes"]) for c in clips), 1)
    pipes = []
    for _ in range(3):
        p = mp.WindowPipeline(cfg.W, cfg.H, cfg.sizes, cfg.cost, cfg.out_dims, cfg.b_proxy, cfg.score_thr,
                              cfg.iou_thr, device=G.DEV)
        p.reserve(F, n_max + 4, caps=caps, max_boxes=nb)
        pipes.append(p)
    runner = mp.PipelinedRunner(pipes, device=G.DEV)
    batches = []
    for c in clips:
        b = np.zeros((nb, 6), np.float32)
        if len(c["boxes"]):
            b[:len(c["boxes"])] = c["boxes"].view(np.float32).reshape(-1, 6)
        w = np.full(n_max + 5, c["wbo"][-1], np.int32)
        w[:len(c["wbo"])] = c["wbo"]
        batches.append((torch.from_numpy(c["scores"]).to(G.DEV), torch.from_numpy(c["frames"]).to(G.DEV),
                        torch.from_numpy(b).to(G.DEV), torch.from_numpy(w).to(G.DEV)))
    evs = [(torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True))
           for _ in batches]
    runner.capture_steps(batches, evs)
    for p in pipes:                                  # capture only records: nothing ran yet
        p.status.zero_()
        p.nms_frame_off.fill_(-3)
    for _ in range(replays):
        runner.replay_steps()
    torch.cuda.synchronize()
    assert all(a.elapsed_time(b) > 0.0 for a, b in evs)
    rng = np.random.default_rng(7)
    for u, c in enumerate(clips):
        p = pipes[u]
        s = dict(frame_off=p.frame_off.cpu().numpy(), windows=p.windows.cpu().numpy(),
                 nms_frame_off=p.nms_frame_off.cpu().numpy(), nms_src=p.nms_src.cpu().numpy(),
                 nms_out=p.nms_out.cpu().numpy(), outs=[o.cpu().numpy() for o in p.outs],
                 status=int(p.status.item()))
        _check_batch(cfg, c, s, rng)
    # the runner is reusable eagerly after a capture
    k = runner.enqueue(*batches[0][:2])
    runner.merge(k, batches[0][2], batches[0][3])
    runner.wait_all()
    torch.cuda.synchronize()
    assert int(pipes[k].status.item()) == 0
