"""NEXT-2 host driver: the greedy window-size selection of PAPER.md:190-195.

"we first initialize S to only contain the size corresponding to the entire
video frame ... on each iteration, we select the size (w,h) that minimizes
tot_time(S + {(w,h)}).  We try all possible dimension (w,h) that are smaller
than the video frame and where w and h are both multiples of 32."

Each greedy step evaluates every candidate on every training frame with ONE
mp_window_set_cost launch (frames x candidate blocks on the GPU).  Across
GPUs (one process per GPU) the candidates are split
round-robin over the ranks; each rank takes the arg-min of its share and one
all-gather of the per-rank (tot, area, w, h) keys per greedy step picks the
global arg-min (ties: smaller area, then smaller w — reading R22; the key is
total, so the choice does not depend on the split).
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple

import torch

from . import _binding as B

_INF = (1 << 63) - 1


def candidate_sizes(W: int, H: int, S: Sequence[Tuple[int, int]], step: int = 32) -> List[Tuple[int, int]]:
    return [(w, h) for w in range(step, W + 1, step) for h in range(step, H + 1, step)
            if (w, h) != (W, H) and (w, h) not in S]


def gpu_evaluator(scores: torch.Tensor, W: int, H: int, cell: int = 32, b_proxy: float = 0.5, stream=None):
    """tot(S, costs, cand, cand_cost) -> list of int on the scores' GPU (one
    mp_window_set_cost call)."""
    def evaluate(S, S_cost, cand, cand_cost):
        if not cand:
            return []
        dev = scores.device
        p = B.PlanParams(W, H, S, S_cost, b_proxy, cell, cell)
        c = torch.tensor(cand, dtype=torch.int32).to(dev, non_blocking=True)
        cc = torch.tensor(cand_cost, dtype=torch.int64).to(dev, non_blocking=True)
        tot = torch.empty(len(cand), dtype=torch.int64, device=dev)
        st = torch.zeros(1, dtype=torch.int32, device=dev)
        B.mp_window_set_cost(p, scores, scores.shape[0], c, cc, tot, st, stream)
        out = tot.cpu().tolist()
        if int(st.item()) != B.MP_OK:
            raise B.MPError(int(st.item()), "mp_window_set_cost (device status)")
        return out
    return evaluate


def _world(group):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def _global_best(key: List[int], group, device) -> List[int]:
    """Lexicographic min of the per-rank keys [tot, area, w, h] (one
    all-gather; NCCL needs device tensors, gloo host tensors)."""
    import torch.distributed as dist
    world, _ = _world(group)
    if world == 1:
        return key
    dev = device if dist.get_backend(group) == "nccl" else torch.device("cpu")
    mine = torch.tensor(key, dtype=torch.int64, device=dev)
    allk = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(allk, mine, group=group)
    return min(tuple(int(x) for x in t.tolist()) for t in allk)


def select_window_sizes(scores: Optional[torch.Tensor], W: int, H: int, k: int, cost_fn: Callable[[int, int], int],
                        cell: int = 32, b_proxy: float = 0.5, step: int = 32, stream=None, group=None,
                        evaluate=None):
    """scores: float32 CUDA tensor [F, R, C] of perfect-proxy grids (1 where a
    cell intersects a theta_best detection), this rank's copy of the training
    frames.  With a process group, rank r evaluates candidates r, r+world, ...
    Returns (S, tot per step), identical on every rank and for any world size.
    `evaluate` (tests) replaces the GPU evaluation."""
    if evaluate is None:
        evaluate = gpu_evaluator(scores, W, H, cell, b_proxy, stream)
    world, rank = _world(group)
    device = scores.device if scores is not None else torch.device("cpu")
    S = [(W, H)]
    hist = []
    for _ in range(k - 1):
        cand = candidate_sizes(W, H, S, step)
        if not cand:
            break
        mine = cand[rank::world]
        tot = evaluate(S, [cost_fn(*s) for s in S], mine, [cost_fn(*c) for c in mine])
        best = [_INF, _INF, _INF, _INF]
        for (w, h), t in zip(mine, tot):
            best = min(best, [int(t), w * h, w, h])
        t, _, w, h = _global_best(best, group, device)
        if t == _INF:
            break
        S.append((w, h))
        hist.append(t)
    return S, hist
