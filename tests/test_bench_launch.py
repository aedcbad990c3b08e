"""CPU tests of bench.py's multi-rank plumbing (the contract's
`bench.py --gpus N` form, which the driver runs without an outer launcher)
and of the host-placement helpers in sharding.py."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None, timeout=600):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT", "LOCAL_WORLD_SIZE"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          timeout=timeout, env=e, cwd=ROOT)


def _json_lines(out):
    return [json.loads(x) for x in out.splitlines() if x.startswith("{")]


def test_bench_gpus2_starts_two_ranks_itself():
    """`bench.py --gpus 2` with no WORLD_SIZE re-launches itself as 2 ranks
    (torch.distributed.run, rendezvous on 127.0.0.1); in --dry-run the ranks
    use gloo: they shard configs[4]'s 1000 clips with assign_clips (LPT over
    per-clip cost estimates), all-reduce a coverage vector and the counters,
    and rank 0 alone prints one line."""
    r = _run(["--gpus", "2", "--dry-run"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1, r.stdout
    d = lines[0]
    assert d["n_gpus"] == 2 and d["coverage_ok"] and d["clips"] == 1000
    assert d["frames"] == 1000 * 1800 * 9
    lo, hi = min(d["rank_loads"]), max(d["rank_loads"])
    assert hi - lo <= 0.01 * hi          # LPT balances the estimated cost


def test_bench_single_rank_dry_run_matches():
    r = _run(["--dry-run"])
    assert r.returncode == 0, r.stderr[-2000:]
    d = _json_lines(r.stdout)[0]
    assert d["n_gpus"] == 1 and d["coverage_ok"] and d["clips"] == 1000


def test_bench_world_size_mismatch_fails_loudly():
    r = _run(["--gpus", "4", "--dry-run"], env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2 and "WORLD_SIZE=2" in r.stderr


def test_numa_helpers_from_sysfs(tmp_path):
    from paper_2103_14695_b200 import sharding as SH
    dev = tmp_path / "bus" / "pci" / "devices" / "0000:1b:00.0"
    dev.mkdir(parents=True)
    (dev / "numa_node").write_text("1\n")
    node = tmp_path / "devices" / "system" / "node" / "node1"
    node.mkdir(parents=True)
    (node / "cpulist").write_text("8-11,40,42-43\n")
    assert SH.pci_numa_node("0000:1B:00.0", str(tmp_path)) == 1
    assert SH.node_cpus(1, str(tmp_path)) == [8, 9, 10, 11, 40, 42, 43]
    (dev / "numa_node").write_text("-1\n")
    assert SH.pci_numa_node("0000:1b:00.0", str(tmp_path)) is None
    assert SH.pci_numa_node("0000:ff:00.0", str(tmp_path)) is None
    # without a CUDA device binding is a recorded no-op
    rec = SH.bind_host_to_gpu(0, str(tmp_path))
    assert rec["bound"] is False


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_lpt_assignment_covers_each_clip_once(world):
    from paper_2103_14695_b200.sharding import assign_clips
    from workloads import synth as S
    cfg = S.CONFIGS["c5_1080p_clips"]
    cost = [S.clip_cost_estimate(cfg, c % 8) for c in range(1000)]
    seen = sorted(c for r in range(world) for c in assign_clips(1000, world, r, cost))
    assert seen == list(range(1000))


def test_gather_sm_reserve_auto_rule():
    """bench.py's auto rule for the SMs the gather leaves to the side kernels
    (DESIGN 6f): u8 1, u8 on 4K grids 16, f32 0; an explicit value wins."""
    import argparse
    import bench
    ns = lambda fmt, k=-1: argparse.Namespace(fmt=fmt, gather_sm_reserve=k)
    assert bench.gather_sm_reserve(ns("u8"), 34, 60) == 1          # 1080p at 32-px cells
    assert bench.gather_sm_reserve(ns("u8"), 68, 120) == 16        # 4K
    assert bench.gather_sm_reserve(ns("f32"), 68, 120) == 0
    assert bench.gather_sm_reserve(ns("f32", 5), 34, 60) == 5
    assert bench.gather_sm_reserve(ns("u8", 0), 68, 120) == 0
