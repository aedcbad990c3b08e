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


# --------------------------------------------------------------------------- host placement
def gpu_numa_node(device_index: int, sysfs: str = "/sys") -> Optional[int]:
    """NUMA node of a CUDA device (from its PCI bus id in sysfs), or None when
    unknown (no GPU, no NUMA info, or a single-node host reporting -1)."""
    try:
        props = torch.cuda.get_device_properties(device_index)
        bus = "%04x:%02x:%02x.0" % (props.pci_domain_id, props.pci_bus_id, props.pci_device_id)
    except Exception:   # no CUDA device / attribute missing
        return None
    return pci_numa_node(bus, sysfs)


def pci_numa_node(bus_id: str, sysfs: str = "/sys") -> Optional[int]:
    import os
    try:
        v = int(open(os.path.join(sysfs, "bus", "pci", "devices", bus_id.lower(), "numa_node")).read().strip())
    except (OSError, ValueError):
        return None
    return v if v >= 0 else None


def node_cpus(node: int, sysfs: str = "/sys") -> List[int]:
    """CPU ids of a NUMA node from its sysfs cpulist ("0-15,64-79")."""
    import os
    txt = open(os.path.join(sysfs, "devices", "system", "node", f"node{node}", "cpulist")).read().strip()
    cpus: List[int] = []
    for part in filter(None, txt.split(",")):
        a, _, b = part.partition("-")
        cpus.extend(range(int(a), int(b or a) + 1))
    return cpus


def bind_host_to_gpu(device_index: int, sysfs: str = "/sys") -> dict:
    """Restrict this process's host threads to the CPUs of the GPU's NUMA
    node, so pinned host buffers allocated afterwards (first touch) sit on
    the socket whose PCIe root complex serves that GPU — zero-copy frame
    reads (the e2e leg) then never cross the inter-socket link.  Returns a
    record of what was done (no-op without NUMA information)."""
    import os
    node = gpu_numa_node(device_index, sysfs)
    if node is None:
        return {"numa_node": None, "bound": False}
    try:
        cpus = sorted(set(node_cpus(node, sysfs)) & set(os.sched_getaffinity(0)))
        if cpus:
            os.sched_setaffinity(0, cpus)
        return {"numa_node": node, "bound": bool(cpus), "cpus": len(cpus)}
    except (OSError, AttributeError, ValueError):
        return {"numa_node": node, "bound": False}
