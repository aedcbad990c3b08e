"""Clip sharding across GPUs (one process per GPU) and the end-of-run counter
reduction — the only cross-GPU traffic of the path.

Every frame is independent for steps a1-a7 (PAPER.md:184 plans one frame at a
time; NMS is per frame), so the job is partitioned by video clip with no
data-path collective: clip c runs on rank c mod world (or by longest-processing
-time balancing when per-clip cost estimates are given).  At the end one
all-reduce(SUM) of int64 counters and one all-reduce(MAX) of the elapsed time
run over NCCL (NVLink/NVSwitch) — or gloo in the CPU tests.
"""
from __future__ import annotations

import dataclasses
import heapq
from typing import List, Optional, Sequence

import torch

COUNTER_FIELDS = ("frames", "windows", "fallback_frames", "crop_bytes", "out_bytes", "boxes_in", "boxes_kept",
                  "clips")


def assign_clips(n_clips: int, world: int, rank: int, cost: Optional[Sequence[float]] = None) -> List[int]:
    """Clips handled by `rank`.  Round-robin (c mod world) by default; with
    per-clip cost estimates, greedy longest-processing-time assignment
    (deterministic: ties broken by clip id, then rank)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if cost is None:
        return list(range(rank, n_clips, world))
    if len(cost) != n_clips:
        raise ValueError("one cost per clip")
    heap = [(0.0, r) for r in range(world)]
    owner = [0] * n_clips
    for c in sorted(range(n_clips), key=lambda c: (-float(cost[c]), c)):
        load, r = heapq.heappop(heap)
        owner[c] = r
        heapq.heappush(heap, (load + float(cost[c]), r))
    return [c for c in range(n_clips) if owner[c] == rank]


@dataclasses.dataclass
class Counters:
    frames: int = 0
    windows: int = 0
    fallback_frames: int = 0
    crop_bytes: int = 0
    out_bytes: int = 0
    boxes_in: int = 0
    boxes_kept: int = 0
    clips: int = 0

    def add(self, other: "Counters") -> "Counters":
        for f in COUNTER_FIELDS:
            setattr(self, f, getattr(self, f) + getattr(other, f))
        return self

    def tensor(self, device="cpu") -> torch.Tensor:
        return torch.tensor([getattr(self, f) for f in COUNTER_FIELDS], dtype=torch.int64, device=device)

    @classmethod
    def from_tensor(cls, t: torch.Tensor) -> "Counters":
        v = t.tolist()
        return cls(**{f: int(x) for f, x in zip(COUNTER_FIELDS, v)})


def reduce_counters(c: Counters, elapsed_ms: float, device="cpu", group=None):
    """All-reduce the run's counters (SUM) and elapsed time (MAX) over the
    default process group (NCCL on GPUs, gloo in tests).  Returns
    (global Counters, max elapsed ms)."""
    import torch.distributed as dist
    t = c.tensor(device)
    e = torch.tensor([float(elapsed_ms)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(e, op=dist.ReduceOp.MAX, group=group)
    return Counters.from_tensor(t.cpu()), float(e.item())
