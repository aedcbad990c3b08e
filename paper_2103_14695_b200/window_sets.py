"""NEXT-2 host driver: the greedy window-size selection of PAPER.md:190-195.

"we first initialize S to only contain the size corresponding to the entire
video frame ... on each iteration, we select the size (w,h) that minimizes
tot_time(S + {(w,h)}).  We try all possible dimension (w,h) that are smaller
than the video frame and where w and h are both multiples of 32."

Each greedy step evaluates every candidate on every training frame with ONE
mp_window_set_cost launch (frames x candidate blocks on the GPU); the host
keeps only the arg-min (ties: smaller area, then smaller w — reading R22).
"""
from __future__ import annotations

from typing import Callable, List, Sequence, Tuple

import torch

from . import _binding as B


def candidate_sizes(W: int, H: int, S: Sequence[Tuple[int, int]], step: int = 32) -> List[Tuple[int, int]]:
    return [(w, h) for w in range(step, W + 1, step) for h in range(step, H + 1, step)
            if (w, h) != (W, H) and (w, h) not in S]


def select_window_sizes(scores: torch.Tensor, W: int, H: int, k: int, cost_fn: Callable[[int, int], int],
                        cell: int = 32, b_proxy: float = 0.5, step: int = 32, stream=None):
    """scores: float32 CUDA tensor [F, R, C] of perfect-proxy grids (1 where a
    cell intersects a theta_best detection).  Returns (S, tot per step)."""
    S = [(W, H)]
    hist = []
    F = scores.shape[0]
    for _ in range(k - 1):
        cand = candidate_sizes(W, H, S, step)
        if not cand:
            break
        p = B.PlanParams(W, H, S, [cost_fn(*s) for s in S], b_proxy, cell, cell)
        tot = torch.empty(len(cand), dtype=torch.int64, device=scores.device)
        ws = torch.empty(B.mp_window_set_cost_workspace_size(len(cand)), dtype=torch.uint8, device=scores.device)
        B.mp_window_set_cost(p, scores, F, cand, [cost_fn(*c) for c in cand], tot, ws, stream)
        t = tot.cpu().tolist()
        best = min(range(len(cand)), key=lambda i: (t[i], cand[i][0] * cand[i][1], cand[i][0]))
        S.append(cand[best])
        hist.append(t[best])
    return S, hist
